"""Pins for oracle O1 (random rotation of Eq. 3) and the storage roundings.

Pinned against: published SplitMix64 outputs, orthogonality, numpy.linalg.qr's
Householder QR with positive diagonal (MGS computes the same Q in exact arithmetic), the d=1
closed form, torch's bf16 conversion, and hand-checked IEEE ties."""
import numpy as np
import pytest
import torch

import oracle as O
from oracle import lshmoe_oracle as OL


def test_splitmix64_reference_outputs(golden):
    z = O.splitmix64_stream(0, 3)
    assert [int(v) for v in z] == [int(h, 16) for h in golden["splitmix64_seed0"]["outputs_hex"]]


def test_irwin_hall_moments_and_range():
    g = O.irwin_hall_gaussian(12345, 200_000)
    assert abs(g.mean()) < 0.01 and abs(g.var() - 1.0) < 0.01
    assert g.min() > -6.0 and g.max() < 6.0


@pytest.mark.parametrize("d", [2, 8, 64, 256])
def test_rotation_orthogonal(d):
    R = O.rotation_fp64(d, 0, 7)
    assert np.abs(R @ R.T - np.eye(d)).max() <= 1e-10


def test_rotation_d1_is_pm1():
    for seed in range(5):
        R = O.rotation_fp64(1, 0, seed)
        assert R.shape == (1, 1) and abs(R[0, 0]) == 1.0


@pytest.mark.parametrize("d,seed,j", [(16, 3, 0), (64, 11, 1), (200, 5, 2)])
def test_rotation_equals_householder_qr(d, seed, j):
    """Gram-Schmidt on the columns of G == Householder QR with a positive-diagonal R factor."""
    G = O.irwin_hall_gaussian(OL._hash_state(seed, j), d * d).reshape(d, d)
    Qh, Rh = np.linalg.qr(G)
    Qh = Qh * np.sign(np.diag(Rh))[None, :]
    R = O.rotation_fp64(d, j, seed)
    assert np.abs(R.T - Qh).max() < 1e-9


def test_rotation_deterministic_and_distinct_per_hash():
    a = O.rotation(32, 3, 99, "bf16")
    b = O.rotation(32, 3, 99, "bf16")
    assert a.dtype == np.uint16 and np.array_equal(a, b)
    assert not np.array_equal(a[0], a[1]) and not np.array_equal(a[1], a[2])
    # prefix property: R_j does not depend on q (S:L141 prefix construction)
    assert np.array_equal(O.rotation(32, 2, 99, "bf16"), a[:2])


def test_f32_to_bf16_matches_torch():
    x = np.random.default_rng(0).standard_normal(100_000).astype(np.float32) * 10
    mine = O.f32_to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(mine, ref)


def test_round_to_dtype_bf16_ties_and_no_double_rounding(golden):
    for exps, want in golden["bf16_rounding"]["cases"]:
        x = 1.0 + sum(2.0 ** e for e in exps)
        assert O.round_to_dtype(np.array([x]), "bf16")[0] == want
        assert O.round_to_dtype(np.array([-x]), "bf16")[0] == -want


def test_round_to_dtype_bf16_matches_torch_on_fp32_values():
    x = (np.random.default_rng(1).standard_normal(50_000) * 3).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.round_to_dtype(x.astype(np.float64), "bf16"), ref)
    assert O.round_to_dtype(np.array([0.0]), "bf16")[0] == 0.0


def test_ulp_bf16():
    assert O.ulp_bf16(np.array([1.0]))[0] == 2.0 ** -7
    assert O.ulp_bf16(np.array([1.5]))[0] == 2.0 ** -7
    assert O.ulp_bf16(np.array([2.0]))[0] == 2.0 ** -6
