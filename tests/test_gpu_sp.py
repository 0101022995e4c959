"""GPU parity of NEXT-3, lshmoe_sp_hash (spherical-plane hashing, §4.5; SPEC's sign-bit
construction S:L124-132, reading R26), against the oracle's fp64 sp_hash.

Tier 1: codes bit-exact except (token, hash) pairs whose oracle margin min_i |n_i.x|/(|n_i||x|) is
below 1e-5 (reported).  Then the SP codes drive lshmoe_compress exactly like CP codes."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import CONFIGS, NEAR_TIE, f64, make_case, oracle_rotation, small_cfg
from lshmoe_inputs import make_tokens, rotation_seed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2411_08446_b200 as L
    return L


def _sp_case(L, cfg, b, seed, X=None):
    X = make_tokens(cfg, seed) if X is None else X
    R_lib = L.rotation(cfg.d, cfg.q, rotation_seed(seed), X.dtype)
    R64 = oracle_rotation(cfg.d, cfg.q, rotation_seed(seed), cfg.dtype)
    assert np.array_equal(f64(R_lib), R64)
    Nrm = L.sp_normals(R_lib.cuda(), b)
    codes_o, margins = O.sp_hash(f64(X), O.sp_normals(R64, b), cfg.q, b)
    return X, Nrm, codes_o, margins


def _check(L, X, Nrm, q, b, codes_o, margins, label):
    got = L.sp_hash(X.cuda(), Nrm, q, b).cpu().numpy()
    mism = got != codes_o
    near = margins < NEAR_TIE
    bad = mism & ~near
    print(f"[sp {label}] n={X.shape[0]} d={X.shape[1]} q={q} b={b} mismatches={int(mism.sum())} "
          f"near-ties={int(near.sum())} outside band={int(bad.sum())}")
    assert not bad.any(), np.argwhere(bad)[:10]
    assert got.min() >= 0 and got.max() < (1 << b)
    return got


@pytest.mark.parametrize("n,d,q,b,dtype", [(300, 64, 2, 8, "f32"), (129, 64, 3, 15, "f32"), (1000, 128, 3, 5, "bf16"),
                                           (777, 256, 16, 15, "bf16"), (1, 64, 1, 1, "bf16"), (4100, 768, 6, 12, "bf16")])
def test_sp_hash_shapes(L, n, d, q, b, dtype):
    cfg = small_cfg(n=n, d=d, q=q, dtype=dtype)
    X, Nrm, codes_o, margins = _sp_case(L, cfg, b, seed=3)
    _check(L, X, Nrm, q, b, codes_o, margins, f"{dtype} n={n}")


def test_sp_hash_c2_full_size(L):
    cfg = CONFIGS["C2"]
    X, Nrm, codes_o, margins = _sp_case(L, cfg, 12, seed=0)
    _check(L, X, Nrm, cfg.q, 12, codes_o, margins, "C2")


def test_sp_identity_normals_spec_example(L, golden):
    """S:L129 through the GPU (f32 path): normals = I, x = (1, -1, 0) -> bits (1, 0, 1)."""
    g = golden["sp_hash_identity_normals"]
    X = torch.tensor([g["x"] + [0.0]], dtype=torch.float32).cuda()          # pad d = 3 -> 4
    Nrm = torch.zeros((L.sp_rows(1, 3), 4), dtype=torch.float32)
    Nrm[:3, :3] = torch.eye(3)
    code = int(L.sp_hash(X, Nrm.cuda(), 1, 3).item())
    assert code == sum(bit << i for i, bit in enumerate(g["bits"]))


def test_sp_codes_drive_compress(L):
    """SP codes (oracle's) as the composite key of lshmoe_compress: bit-exact buckets vs the oracle."""
    cfg = CONFIGS["C2"]
    case = make_case(L, cfg, seed=0, sanitize=False)
    R64 = oracle_rotation(cfg.d, cfg.q, rotation_seed(0), cfg.dtype)
    codes, _ = O.sp_hash(f64(case.X), O.sp_normals(R64, 12), cfg.q, 12)
    out = L.compress(case.X.cuda(), torch.from_numpy(codes).cuda(), case.zeta.cuda(), cfg.E)
    b = O.bucketize(codes, case.zeta.numpy(), cfg.E)
    print(f"[sp compress C2] m={b.m} ratio={b.m / cfg.n:.3f}")
    assert int(out.num_rows.item()) == b.m
    assert np.array_equal(out.bucket.cpu().numpy(), b.bucket)
    assert np.array_equal(out.perm.cpu().numpy(), b.perm)
