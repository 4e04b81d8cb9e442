"""Hand-derived known answers for the repo-defined extensions in the oracle
(4-bit element quantizer, per-token / per-channel scales; oracle/cc_oracle.py).
They follow the reference's 1/2-bit conventions (cx:135-149, cx:379-391), so the
KATs mirror the reference's own (T/test_compressors.py:21-31, 76-82)."""

import numpy as np

from oracle import cc_oracle as O


def test_scale_modes_kat():
    x = np.array([[1, -1], [2, -2]], np.float32)  # T/test_compressors.py:21-25
    u, v = O.scales(x, "rank1")
    assert np.allclose(u, [2 / 3, 4 / 3]) and np.allclose(v, [1.5, 1.5])
    u, v = O.scales(x, "per_token")
    assert u.tolist() == [1.0, 2.0] and v.tolist() == [1.0, 1.0]
    u, v = O.scales(x, "per_channel")
    assert u.tolist() == [1.0, 1.0] and v.tolist() == [1.5, 1.5]


def test_quant4_constant_input_tie_to_smaller_level():
    # constant c: u = 1, v = c, x / (u v) = 1.0 sits between levels 0.75 and 1.25:
    # the tie goes to the smaller magnitude (code 9), like 2-bit's tie -> +0.5 (:76-82)
    x = np.full((3, 5), 0.7, np.float32)
    u, v = O.scales(x)
    assert O.quant4_codes(x, u, v).tolist() == [9] * 15
    dec = O.quant4_decode(O.quant_body(x, O.QUANT4), 3, 5)
    assert np.array_equal(dec, np.full((3, 5), np.float32(0.75 * np.float64(np.float32(0.7)))))


def test_quant4_zero_and_negative_zero():
    x = np.zeros((2, 3), np.float32)
    x[0, 1] = -0.0
    u, v = O.scales(x)
    assert u.tolist() == [1.0, 1.0] and v.tolist() == [0.0, 0.0, 0.0]
    assert O.quant4_codes(x, u, v).tolist() == [8] * 6
    assert np.array_equal(O.quant4_decode(O.quant_body(x, O.QUANT4), 2, 3), np.zeros((2, 3), np.float32))
    # -0.0 with a live scale is not negative (as the sign rule t < 0, cx:375)
    y = np.array([[-0.0, 1.0]], np.float32)
    assert O.quant4_codes(y, np.ones(1, np.float32), np.ones(2, np.float32)).tolist() == [8, 9]


def test_quant4_levels_and_boundaries():
    u, v = np.ones(1, np.float32), np.ones(16, np.float32)
    # |x| on each boundary k/2 takes the lower level; just above takes the next
    bnd = np.array([[0.5 * k for k in range(1, 8)] + [0.0] * 9], np.float32)
    assert O.quant4_codes(bnd, u, v)[:7].tolist() == [8 + k - 1 for k in range(1, 8)]
    above = np.nextafter(bnd, np.float32(np.inf))
    assert O.quant4_codes(above, u, v)[:7].tolist() == [8 + k for k in range(1, 8)]
    assert O.quant4_codes(-above, u, v)[:7].tolist() == [7 - k for k in range(1, 8)]
    big = np.array([[100.0, -100.0] + [0.0] * 14], np.float32)
    assert O.quant4_codes(big, u, v)[:2].tolist() == [15, 0]
    assert np.array_equal(O.LEVELS_4BIT, -O.LEVELS_4BIT[::-1])
    assert O.LEVELS_4BIT[8] == 0.25 and O.LEVELS_4BIT[15] == 3.75


def test_quant4_body_layout():
    x = np.array([[0.1, -3.0, 2.0], [0.0, 1.0, -0.2]], np.float32)
    body = O.quant_body(x, O.QUANT4)
    assert len(body) == O.body_bytes(O.QUANT4, 2, 3) == 3 + 4 * 5
    codes = O.quant4_codes(x, *O.scales(x))
    assert body[0] == (codes[0] | (codes[1] << 4))  # low nibble first
    assert body[2] == codes[4] | (codes[5] << 4)
    u, v = O.scales(x)
    assert body[3:] == u.astype("<f4").tobytes() + v.astype("<f4").tobytes()


def test_per_token_sign_round_trip_protocol():
    """Extensions run through the same residual protocol (pl:84-165): sender and
    receiver stay bit-identical, feedback = target - decoded exactly."""
    rng = np.random.default_rng(3)
    codec = O.Codec(O.QUANT4, scale_mode="per_token")
    snd = O.Channel(O.WITH_FEEDBACK, 1, np.zeros((6, 10), np.float32))
    rcv = O.Channel(O.WITH_FEEDBACK, 1, np.zeros((6, 10), np.float32))
    for t in range(1, 6):
        x = rng.standard_normal((6, 10)).astype(np.float32)
        target = (x - snd.base) + snd.fb if t > 1 else x
        tag, body, _ = O.send(snd, x, codec)
        O.receive(rcv, t, t == 1, tag, body, codec)
        assert np.array_equal(rcv.base, snd.base)
        if t > 1:
            dec = O.decode_body(body, codec, 6, 10)
            assert np.array_equal(snd.fb, target - dec)
