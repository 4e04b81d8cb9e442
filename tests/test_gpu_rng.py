"""Device draw of the low-rank start block (csrc/rng.cu, cc_gaussian_keyed) against
numpy itself: float32(Generator(PCG64(SeedSequence(seed, spawn_key))).standard_normal)
is the reference's Q0 (compressors.py:407, linalg.py:25-27, 67-74)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _draw(key, rows, cols):
    from paper_2507_17511_b200 import _lib

    lib = _lib.load()
    out = torch.empty(rows, cols, dtype=torch.float32, device="cuda")
    ws = torch.empty(_lib.check(lib.cc_gaussian_workspace_bytes(rows, cols)), dtype=torch.uint8, device="cuda")
    _lib.check(lib.cc_gaussian_keyed(rows, cols, _lib.ptr(key.words), key.nwords, key.step_word, _lib.ptr(out),
                                     _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "gaussian")
    return out.cpu().numpy()


def _ref(seed, key, rows, cols):
    from paper_2507_17511_b200 import linalg as la

    return la.gaussian_matrix(la.spawn_rng(seed, *key), rows, cols)


KEYS = [(0, ()), (17, (5, 3)), (2**40 + 5, (6, 1, 7)), (123456789, (6, 0, 0)), (7, (5,)),
        (0xDEADBEEFCAFE1234ABCD, (1, 2, 3, 4, 5, 6)), (2**32, (2**33, 1))]


@pytest.mark.parametrize("seed,key", KEYS)
@pytest.mark.parametrize("shape", [(1, 1), (7, 3), (3072, 8), (1024, 16), (3072, 32), (4096, 4)])
def test_gaussian_keyed_bit_exact(seed, key, shape):
    from paper_2507_17511_b200 import linalg as la

    got = _draw(la.DeviceKey(seed, *key), *shape)
    assert got.tobytes() == _ref(seed, key, *shape).tobytes()


def test_gaussian_many_keys():
    """200 mesh-style keys (seed, 6, device, t): exercises the wedge / tail paths."""
    from paper_2507_17511_b200 import linalg as la

    for d in range(4):
        for t in range(1, 51):
            assert _draw(la.DeviceKey(99, 6, d, t), 3072, 8).tobytes() == _ref(99, (6, d, t), 3072, 8).tobytes()


def test_advancing_key_and_graph_replay():
    """step_word: each draw advances the key's last element, also across CUDA-graph replays."""
    from paper_2507_17511_b200 import _lib
    from paper_2507_17511_b200 import linalg as la

    lib = _lib.load()
    key = la.DeviceKey(5, 6, 2, 10, advance=True)
    assert _draw(key, 3072, 8).tobytes() == _ref(5, (6, 2, 10), 3072, 8).tobytes()
    assert _draw(key, 3072, 8).tobytes() == _ref(5, (6, 2, 11), 3072, 8).tobytes()
    out = torch.empty(3072, 8, dtype=torch.float32, device="cuda")
    ws = torch.empty(lib.cc_gaussian_workspace_bytes(3072, 8), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        _lib.check(lib.cc_gaussian_keyed(3072, 8, _lib.ptr(key.words), key.nwords, key.step_word, _lib.ptr(out),
                                         _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "gaussian")
    for t in (12, 13, 14):
        g.replay()
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == _ref(5, (6, 2, t), 3072, 8).tobytes()


def test_lowrank_device_key_equals_host_rng():
    """encode_lowrank with a DeviceKey produces the same body as with the host
    Generator of the same key (the only difference is where Q0 is drawn)."""
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import linalg as la

    rng = np.random.default_rng(3)
    a = torch.from_numpy((rng.standard_normal((512, 3072)) * rng.random((1, 3072))).astype(np.float32)).cuda()
    for r, int4 in ((8, False), (16, True)):
        spec = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=r, iterations=2, int4_factors=int4)
        ph = cx.encode_lowrank(a, spec, la.spawn_rng(11, 6, 0, 4))
        pd = cx.encode_lowrank(a, spec, la.DeviceKey(11, 6, 0, 4))
        assert ph.body_bytes() == pd.body_bytes()
