"""GPU parity of a3-a5, lshmoe_compress (Alg. 1 L3-L12), against the oracle.

Stage-isolated: both sides bucket the ORACLE's codes, so integer outputs are compared
bit-exactly (tier 1: bucket, perm, row_start, expert_rows, m); centroids_f32 within 1e-5
row-max-relative (tier 2) and the wire centroids within 1 ulp of the dtype."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import CONFIGS, f64, make_case, row_rel_err, small_cfg
from lshmoe_inputs import make_tokens

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2411_08446_b200 as L
    return L


def _compress_and_check(L, X, codes, zeta, E, dtype, label, repeat=True):
    Xd, cd, zd = X.cuda(), torch.from_numpy(codes).cuda(), zeta.cuda()
    out = L.compress(Xd, cd, zd, E, with_f32=True)
    torch.cuda.synchronize()
    L.check_device_error()
    b = O.bucketize(codes, zeta.numpy(), E)
    m = int(out.num_rows.item())
    n, k = zeta.shape
    print(f"[compress {label}] n={n} k={k} E={E} m={m} ratio={m / max(1, n * k):.4f}")
    assert m == b.m
    assert np.array_equal(out.expert_rows.cpu().numpy(), b.expert_rows)
    assert np.array_equal(out.bucket.cpu().numpy(), b.bucket)
    assert np.array_equal(out.perm.cpu().numpy(), b.perm)
    assert np.array_equal(out.row_start.cpu().numpy()[:m + 1], b.row_start)
    C = O.centroids(f64(X), b, k)
    c32 = out.centroids_f32[:m].cpu().numpy().astype(np.float64)
    assert row_rel_err(c32, C) <= 1e-5
    ct = f64(out.centroids[:m])
    if dtype == "bf16":          # reading R23: wire value within 1 bf16 ulp of RNE(exact mean)
        ref = O.round_to_dtype(C, dtype)
        assert np.all(np.abs(ct - ref) <= O.ulp_bf16(ref) + 1e-30)
    # the wire value is exactly the RNE of the GPU's own fp32 mean
    assert np.array_equal(ct, O.round_to_dtype(c32, dtype))
    if repeat:   # determinism: bit-identical on a second run
        out2 = L.compress(Xd, cd, zd, E, with_f32=True)
        assert torch.equal(out2.perm, out.perm) and torch.equal(out2.bucket, out.bucket)
        assert torch.equal(out2.centroids_f32[:m], out.centroids_f32[:m])
    return out, b


@pytest.mark.parametrize("cfgname", ["C1", "C2"])
def test_compress_configs(L, cfgname):
    case = make_case(L, CONFIGS[cfgname], seed=0, sanitize=False)
    _compress_and_check(L, case.X, case.codes, case.zeta, case.cfg.E, case.cfg.dtype, cfgname)


@pytest.mark.parametrize("n,k,E,q,d", [(1000, 2, 4, 3, 128), (1, 1, 1, 1, 64), (33, 3, 3, 2, 64), (4100, 2, 8, 2, 64)])
def test_compress_shapes(L, n, k, E, q, d):
    cfg = small_cfg(n=n, k=k, E=E, q=q, d=d, C=8, rho=0.05)
    case = make_case(L, cfg, seed=5, sanitize=False)
    _compress_and_check(L, case.X, case.codes, case.zeta, E, "bf16", f"n={n},k={k},E={E}")


def test_compress_all_identical_giant_bucket(L):
    """All tokens identical => one bucket per expert group spanning many 32-entry chunks."""
    cfg = small_cfg(n=5000, k=2, E=3, q=3, d=128)
    x = make_tokens(cfg, 0, n=1)
    X = x.repeat(5000, 1).contiguous()
    case = make_case(L, cfg, seed=0, sanitize=False, X=X)
    out, b = _compress_and_check(L, case.X, case.codes, case.zeta, 3, "bf16", "identical")
    assert b.m == int((b.expert_rows > 0).sum())


def test_compress_iid_tokens_every_bucket_singleton(L):
    cfg = small_cfg(n=2000, k=1, E=4, q=6, d=128)
    X = make_tokens(cfg, 0, iid=True)
    case = make_case(L, cfg, seed=0, sanitize=False, X=X)
    out, b = _compress_and_check(L, case.X, case.codes, case.zeta, 4, "bf16", "iid")
    assert b.m == 2000
    # singleton rows: centroid == token exactly
    m = b.m
    assert torch.equal(out.centroids[:m].cpu(), case.X[torch.from_numpy(b.perm.astype(np.int64))])


def test_compress_skewed_hot_expert(L):
    cfg = small_cfg(n=6000, k=2, E=8, q=4, d=192, C=40, rho=0.05)
    case = make_case(L, cfg, seed=6, sanitize=False)
    zeta = case.zeta.clone()
    hot = torch.arange(6000) % 10 < 3                       # 30% of tokens' first slot -> expert 7
    zeta[hot, 1] = 7
    zeta[hot, 0] = torch.where(zeta[hot, 0] == 7, torch.zeros_like(zeta[hot, 0]), zeta[hot, 0])
    zeta = torch.sort(zeta, dim=1).values.contiguous()
    _compress_and_check(L, case.X, case.codes, zeta, 8, "bf16", "skew")


def test_compress_k_equals_E(L):
    cfg = small_cfg(n=700, k=4, E=4, q=2, d=64)
    case = make_case(L, cfg, seed=7, sanitize=False)
    out, b = _compress_and_check(L, case.X, case.codes, case.zeta, 4, "bf16", "k=E")
    assert np.array_equal(b.expert_rows, b.expert_rows[0] * np.ones(4, np.int32))


def test_compress_f32_small(L):
    cfg = small_cfg(n=513, k=2, E=5, q=2, d=64, dtype="f32")
    case = make_case(L, cfg, seed=8, sanitize=False)
    _compress_and_check(L, case.X, case.codes, case.zeta, 5, "f32", "f32")


def test_invalid_expert_raises_device_error(L):
    cfg = small_cfg(n=100, k=1, E=4, q=2, d=64)
    case = make_case(L, cfg, seed=9, sanitize=False)
    zeta = case.zeta.clone()
    zeta[17, 0] = 9
    L.compress(case.X.cuda(), torch.from_numpy(case.codes).cuda(), zeta.cuda(), 4)
    with pytest.raises(L.LshmoeError) as ei:
        L.check_device_error()
    assert ei.value.status == L.EDEVICE
    L.check_device_error()          # cleared


@pytest.mark.parametrize("cfgname", ["C3", "C4", "C5"])
def test_compress_full_size_synthetic_codes(L, cfgname):
    """Full C3/C4/C5 shapes (k=2, d=1024, E up to 64; groups up to ~8K copies), stage-isolated on
    synthetic codes with the workloads' bucket structure (hashing them in the fp64 oracle would
    take minutes).  Expected values come from the oracle's bucketize/centroids only."""
    from lshmoe_inputs import make_codes
    cfg = CONFIGS[cfgname]
    X = make_tokens(cfg, 0)
    codes = make_codes(cfg.n, cfg.q, cfg.d, 0, C=cfg.C, p_noise=0.08)
    from lshmoe_inputs import make_gate
    zeta, _ = make_gate(cfg, 0, X)
    _compress_and_check(L, X, codes, zeta, cfg.E, cfg.dtype, cfgname, repeat=False)


def test_compress_group_larger_than_shared_memory(L):
    """Two groups of ~20K copies: phase A keeps its arrays in the workspace, not shared memory."""
    from lshmoe_inputs import make_codes, make_zipf_gate
    cfg = small_cfg(n=40000, k=1, E=2, q=3, d=64, dtype="f32")
    X = make_tokens(cfg, 1)
    codes = make_codes(cfg.n, cfg.q, cfg.d, 1, C=64, p_noise=0.05)
    zeta = make_zipf_gate(cfg.n, 1, 2, 1)
    _compress_and_check(L, X, codes, zeta, 2, "f32", "big-group")


def test_compress_iid_group_counters_in_workspace(L):
    """One group of 60K distinct keys: the per-(warp, row) counters no longer fit shared memory."""
    from lshmoe_inputs import make_codes
    cfg = small_cfg(n=60000, k=1, E=1, q=4, d=64, dtype="f32")
    X = make_tokens(cfg, 2, iid=True)
    codes = make_codes(cfg.n, cfg.q, cfg.d, 2, iid=True)
    zeta = torch.zeros((cfg.n, 1), dtype=torch.int32)
    out, b = _compress_and_check(L, X, codes, zeta, 1, "f32", "iid-60K", repeat=False)
    assert b.m == len({tuple(r) for r in codes.tolist()})


def test_compress_hot_expert_full_c2(L):
    """C2 with 30% of tokens forced onto one expert (SURVEY §8d.1 stress 3)."""
    from lshmoe_inputs import make_codes, make_zipf_gate
    cfg = CONFIGS["C2"]
    X = make_tokens(cfg, 3)
    codes = make_codes(cfg.n, cfg.q, cfg.d, 3, C=cfg.C, p_noise=0.08)
    zeta = make_zipf_gate(cfg.n, 1, cfg.E, 3, hot=0.3)
    _compress_and_check(L, X, codes, zeta, cfg.E, "bf16", "C2-hot", repeat=False)


def test_compress_leaves_workspace_at_rest(L):
    """The contract of include/lshmoe.h: the workspace is 0xFF-filled before first use and every call
    leaves its header (arrival counters) and hash table back at 0xFF, so calls need no clearing."""
    cfg = CONFIGS["C2"]
    case = make_case(L, cfg, seed=1, sanitize=False)
    ws = torch.full((L.compress_workspace_bytes(cfg.n, 1, cfg.E, cfg.q, cfg.d, torch.bfloat16),), 255,
                    dtype=torch.uint8, device="cuda")
    Xd, cd, zd = case.X.cuda(), torch.from_numpy(case.codes).cuda(), case.zeta.cuda()
    a = L.compress(Xd, cd, zd, cfg.E, workspace=ws)
    perm_a = a.perm.clone()
    torch.cuda.synchronize()
    hdr_ints = 64 + 2048 + 512 + 16 * 512            # compress.cu kHdr
    tsize = 1024
    while tsize < 2 * cfg.n:
        tsize *= 2
    rest = ws[:4 * (hdr_ints + tsize)]
    assert int((rest != 255).sum()) == 0
    b = L.compress(Xd, cd, zd, cfg.E, workspace=ws)
    assert torch.equal(b.perm, perm_a)


def test_compress_max_q_and_many_experts(L):
    """The envelope: q = LSHMOE_MAX_Q = 16 hash functions per key, E = 255 experts (one expert
    digit short of the tile grouping's 256), k = 3."""
    from lshmoe_inputs import make_codes, make_zipf_gate
    n, k, E, q = 6000, 3, 255, 16
    cfg = small_cfg(n=n, k=k, E=E, q=q, d=128)
    X = make_tokens(cfg, 4)
    codes = make_codes(n, q, 128, 4, C=40, p_noise=0.02)
    zeta = make_zipf_gate(n, k, E, 4)
    _compress_and_check(L, X, codes, zeta, E, "bf16", "q=16,E=255")
