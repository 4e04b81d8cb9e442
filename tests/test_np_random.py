"""The oracle's restatement of the reference's random stream (oracle/np_random.py:
SeedSequence -> PCG64 -> ziggurat standard_normal, linalg.py:20-27, 67-74) against
numpy itself, bit for bit, including the ziggurat's wedge and tail paths."""

import numpy as np
import pytest

from oracle import np_random as R

KEYS = [(0, ()), (17, (5, 3)), (2**40 + 5, (6, 1, 7)), (123456789, (6, 0, 0)), (7, (5,)),
        (0xDEADBEEFCAFE1234ABCD, (1, 2, 3, 4, 5, 6)), (2**32, (2**33, 1)), (5, (0,))]


@pytest.mark.parametrize("seed,key", KEYS)
def test_seed_sequence_pcg64_state(seed, key):
    st = np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=key)).state["state"]
    assert R.pcg64_seed(seed, key) == (st["state"], st["inc"])


@pytest.mark.parametrize("seed,key", KEYS)
def test_raw_stream(seed, key):
    bg = np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=key))
    g = R.PCG64(*R.pcg64_seed(seed, key))
    assert [g.next64() for _ in range(64)] == [int(v) for v in bg.random_raw(64)]


def test_gaussian_matrix_bit_exact_with_slow_paths():
    before = dict(R.PATHS)
    for seed, key in KEYS + [(s, (6, d, t)) for s in (3, 11) for d in range(4) for t in range(1, 4)]:
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=key)))
        ref = (rng.standard_normal((3072, 8), dtype=np.float64) * 1.0).astype(np.float32)  # la:73-74
        assert R.gaussian_matrix(seed, key, 3072, 8).tobytes() == ref.tobytes()
    assert R.PATHS["wedge"] > before["wedge"] and R.PATHS["tail"] > before["tail"]
