"""Pins of the oracle's fp8 option (O2", reading R28): e4m3 rounding against torch's
float8_e4m3fn conversion (a library routine) and the value table's structure; the power-of-two
scale rule; and the scale invariance of Eq. 3 that makes per-token / per-hash scaling free."""
import math

import numpy as np
import torch

import oracle as O


def test_e4m3_table_structure():
    tab = O.e4m3_values()
    assert len(tab) == 127 and tab[0] == 0 and tab[-1] == 448.0 and tab[1] == 2.0 ** -9
    assert np.all(np.diff(tab) > 0)
    codes = torch.arange(0, 0x7F, dtype=torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    assert np.array_equal(codes, tab)                       # same bit -> value map as torch


def test_round_e4m3_matches_torch():
    rng = np.random.default_rng(0)
    a = np.concatenate([rng.uniform(-448, 448, 20000), rng.standard_normal(20000) * 1e-2,
                        rng.standard_normal(20000), O.e4m3_values(), -O.e4m3_values(),
                        (O.e4m3_values()[:-1] + O.e4m3_values()[1:]) / 2])      # exact ties
    a32 = a.astype(np.float32).astype(np.float64)           # torch converts from fp32
    want = torch.from_numpy(a32).to(torch.float32).to(torch.float8_e4m3fn).to(torch.float64).numpy()
    assert np.array_equal(O.round_e4m3(a32), want)


def test_pow2_scale_rule():
    for vmax in (1e-30, 0.001, 0.5, 0.875, 0.87500001, 1.0, 3.0, 448.0, 500.0, 1e6):
        s = O.pow2_scale_e4m3(vmax)
        assert math.log2(s) == int(math.log2(s))
        assert vmax * s <= 448 and vmax * s * 2 > 448
    assert O.pow2_scale_e4m3(0.0) == 1.0


def test_quantized_codes_scale_invariant():
    """Eq. 3 on quantised values: scaling a token by 2^j before quantisation changes nothing."""
    rng = np.random.default_rng(1)
    X = rng.standard_normal((50, 16))
    R = O.to_stored(O.rotation(16, 2, 99, "f32"), "f32")
    Rq = O.quantize_rotation_e4m3(R)
    a, _ = O.cp_hash(O.quantize_tokens_e4m3(X), Rq)
    b, _ = O.cp_hash(O.quantize_tokens_e4m3(X * 8.0), Rq)
    assert np.array_equal(a, b)
    assert np.abs(O.quantize_tokens_e4m3(X)).max(axis=1).max() <= 448


def test_quantize_rotation_one_scale_per_hash():
    """Reading R28 fixes ONE power-of-two scale per R_j (from max |R_j|), not per row and not one
    for all q hashes.  Hand-built R (q = 2, d = 2) whose rows and hashes have very different
    maxima; every expected value below is worked out by hand from e4m3's grid (steps of 2^(e-3)
    in [2^e, 2^(e+1))):
      R_0 = [[100, 1], [0.5, 0.25]]: max 100 -> scale 2^2 (400 <= 448 < 800) -> 400 is the exact
            midpoint of the grid points 384 (mantissa 100b) and 416 (101b) in [256, 512): ties to
            the even mantissa -> 384; then [4], [2, 1] exact -> [[384, 4], [2, 1]]
            (a per-row scale would put row 1 at 2^9: [256, 128]);
      R_1 = [[3, 0.3], [-1.1, 0]]:   max 3 -> scale 2^7 (384 <= 448 < 768) -> 3*128 = 384 (exact,
            1.5*2^8), 0.3*128 = 38.4 -> 40 (grid 36, 40 in [32, 64)), -1.1*128 = -140.8 -> -144
            (grid 128, 144 in [128, 256)), 0 -> 0 (a global scale 2^2 would give [12, 1.25], ...)."""
    R32 = np.array([[[100.0, 1.0], [0.5, 0.25]], [[3.0, 0.3], [-1.1, 0.0]]], dtype=np.float32)
    got = O.quantize_rotation_e4m3(R32.astype(np.float64))
    want = np.array([[[384.0, 4.0], [2.0, 1.0]], [[384.0, 40.0], [-144.0, 0.0]]])
    assert np.array_equal(got, want)


def test_quantize_tokens_one_scale_per_token():
    """Per-token scale (R28): x = [0.01, 1] and [300, -7] -> scales 2^8 (256 <= 448 < 512) and
    2^0 (300 <= 448 < 600): [2.56 -> 2.5 (grid 2.5, 2.75 in [2, 4)), 256] and [288 (grid 288, 320
    in [256, 512); 300 - 288 = 12 < 20), -7]."""
    X = np.array([[0.01, 1.0], [300.0, -7.0]])
    assert np.array_equal(O.quantize_tokens_e4m3(X), np.array([[2.5, 256.0], [288.0, -7.0]]))
