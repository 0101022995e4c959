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
