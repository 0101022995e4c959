"""GPU parity of NEXT-1 (reading R27): lshmoe_grad_compress and lshmoe_grad_restore against the
oracle's grad_compress / grad_restore on the same seeded inputs.  Stage-isolated: the forward's
buckets come from the oracle's bucketize (bit-exact with the GPU's, test_gpu_compress), and H
(the expert backward) is the oracle's expert_ffn_vjp, rounded to the dtype.
Tolerances: f32 tier 2 (1e-5 row-max-relative); bf16 G: fp32 sums within 1e-5 and the wire value
within 1 bf16 ulp of RNE(exact); bf16 dX / dg: 1e-2 row-max-relative (inputs are bf16-rounded
gradients of O(1) magnitude; the fp32 kernel sum differs from fp64 by ~1e-6 relative, the final
bf16 rounding of dX adds 2^-9)."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import CONFIGS, f64, make_case, row_rel_err, small_cfg
from lshmoe_inputs import make_experts

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2411_08446_b200 as L
    return L


def _run(L, cfg, seed, with_g):
    case = make_case(L, cfg, seed=seed, sanitize=False, with_weights=with_g)
    X, zeta, g = case.X, case.zeta, case.g
    dt = X.dtype
    b = O.bucketize(case.codes, zeta.numpy(), cfg.E)
    k = cfg.k
    comp = L.compress(X.cuda(), torch.from_numpy(case.codes).cuda(), zeta.cuda(), cfg.E)
    assert np.array_equal(comp.bucket.cpu().numpy(), b.bucket)
    m = b.m
    rng = np.random.default_rng(seed + 100)
    dY = torch.from_numpy(rng.standard_normal(X.shape)).to(torch.float32).to(dt)
    gd = g.cuda() if g is not None else None
    # B1 on the GPU vs the oracle
    G32 = torch.empty((cfg.n * k, cfg.d), dtype=torch.float32, device="cuda")
    G = L.grad_compress(dY.cuda(), comp, gd, out_f32=G32)
    torch.cuda.synchronize()
    Go = O.grad_compress(f64(dY), b, k, None if g is None else g.numpy())
    e32 = row_rel_err(G32[:m].cpu().numpy().astype(np.float64), Go)
    assert e32 <= 1e-5, e32
    Gw = f64(G[:m])
    assert np.array_equal(Gw, O.round_to_dtype(G32[:m].cpu().numpy().astype(np.float64), cfg.dtype))
    # forward quantities (oracle) and the expert backward H (oracle, rounded to the dtype)
    ex = make_experts(cfg, seed)
    oex = {e: tuple(f64(t) for t in ex[e]) for e in range(cfg.E)}
    C = O.centroids(f64(X), b, k)
    Ct = O.round_to_dtype(C, cfg.dtype)
    ret = np.zeros_like(Ct)
    H = np.zeros_like(Ct)
    off = 0
    for e, me in enumerate(b.expert_rows):
        if me:
            ret[off:off + me] = O.expert_ffn(Ct[off:off + me], *oex[e])
            H[off:off + me] = O.expert_ffn_vjp(Ct[off:off + me], oex[e][0], oex[e][1], oex[e][2], Gw[off:off + me])
        off += me
    ret = O.round_to_dtype(ret, cfg.dtype)
    H = O.round_to_dtype(H, cfg.dtype)
    to = lambda a: torch.from_numpy(a).to(torch.float32).to(dt).cuda()   # noqa: E731
    dx, dg = L.grad_restore(dY.cuda(), X.cuda(), to(Ct), to(ret), G[:m].contiguous(), to(H), comp, gd,
                            want_dgate=True)
    torch.cuda.synchronize()
    dXo, dgo = O.grad_restore(f64(dY), f64(X), Ct, ret, Gw, H, b, None if g is None else g.numpy())
    tol = 1e-5 if cfg.dtype == "f32" else 1e-2
    ex_ = row_rel_err(f64(dx), dXo)
    eg = float(np.abs(dg.cpu().numpy() - dgo).max() / max(1e-30, np.abs(dgo).max()))
    print(f"[backward {cfg.name} g={with_g}] m={m} G32 err={e32:.2e} dX err={ex_:.2e} dg err={eg:.2e}")
    assert ex_ <= tol and eg <= tol


@pytest.mark.parametrize("with_g", [False, True])
def test_backward_f32_c1(L, with_g):
    _run(L, CONFIGS["C1"], 0, with_g)


@pytest.mark.parametrize("with_g", [False, True])
def test_backward_bf16_c2(L, with_g):
    _run(L, CONFIGS["C2"], 0, with_g)


def test_backward_bf16_topk2_small(L):
    _run(L, small_cfg(n=3000, d=256, E=6, k=2, q=3, C=30, rho=0.05), 4, True)


def test_backward_f32_giant_bucket_spans_ctas(L):
    """All tokens identical: one bucket per expert spanning many CTA ranges (cut-row merge)."""
    cfg = small_cfg(n=6000, d=64, E=2, k=1, q=2, dtype="f32")
    from lshmoe_inputs import make_tokens
    x = make_tokens(cfg, 0, n=1)
    case_X = x.repeat(6000, 1).contiguous()
    case = make_case(L, cfg, seed=1, sanitize=False, X=case_X)
    comp = L.compress(case.X.cuda(), torch.from_numpy(case.codes).cuda(), case.zeta.cuda(), 2)
    b = O.bucketize(case.codes, case.zeta.numpy(), 2)
    dY = torch.randn(case.X.shape, generator=torch.Generator().manual_seed(3))
    G = L.grad_compress(dY.cuda(), comp)
    Go = O.grad_compress(f64(dY), b, 1)
    assert row_rel_err(f64(G[:b.m]), Go) <= 1e-5
    G2 = L.grad_compress(dY.cuda(), comp)
    assert torch.equal(G[:b.m], G2[:b.m])            # deterministic (rows past m are unused)


@pytest.mark.parametrize("cfgname", ["C1", "C2"])
def test_expert_ffn_backward(L, cfgname):
    """lshmoe_expert_ffn_backward (H = J_E(c~)^T G, the dX path of the expert's backward) vs the
    oracle's expert_ffn_vjp on the same received rows (world 1: recv = centroid layout).  A hidden
    unit whose fp64 pre-activation lies within 1e-5 (relative to the row's max) of zero is a relu'
    near-tie: the GPU's fp32 pre-activation may take the other side, so both values of that unit's
    mask are correct.  Every row is compared: a row with c near-tie units must match, within the
    tier tolerance, one of the 2^c oracle results with those units' masks flipped or kept (the
    flip of unit j adds or removes (W2^T G)_j * W1[j, :]); no row is dropped."""
    cfg = CONFIGS[cfgname]
    case = make_case(L, cfg, seed=0, sanitize=True)
    b = O.bucketize(case.codes, case.zeta.numpy(), cfg.E)
    Ct = O.round_to_dtype(O.centroids(f64(case.X), b, cfg.k), cfg.dtype)
    m = b.m
    dt = case.X.dtype
    ex = make_experts(cfg, 0)
    W1 = torch.stack([ex[e][0] for e in range(cfg.E)]).cuda()
    b1 = torch.stack([ex[e][1] for e in range(cfg.E)]).cuda()
    W2 = torch.stack([ex[e][2] for e in range(cfg.E)]).cuda()
    b2 = torch.stack([ex[e][3] for e in range(cfg.E)]).cuda()
    W2T = W2.transpose(1, 2).contiguous()
    W1T = W1.transpose(1, 2).contiguous()
    rr = torch.from_numpy(b.expert_rows.astype(np.int32)).view(cfg.E, 1).cuda()
    rng = np.random.default_rng(7)
    Gh = torch.from_numpy(rng.standard_normal((m, cfg.d))).to(torch.float32).to(dt)
    recv = torch.from_numpy(Ct).to(torch.float32).to(dt).cuda()
    hid = torch.empty((m, cfg.d_ffn), dtype=dt, device="cuda")
    L.expert_ffn(recv, rr, W1, b1, W2, b2, hidden=hid)
    H = L.expert_ffn_backward(Gh.cuda(), rr, W2T, W1T, hid)
    torch.cuda.synchronize()
    Ho = np.zeros((m, cfg.d))
    Hg = f64(H)
    tol = 1e-5 if cfg.dtype == "f32" else 2e-2
    n_near, worst = 0, 0.0
    off = 0
    for e, me in enumerate(b.expert_rows):
        if me:
            w1, bb1, w2, _ = (f64(t) for t in ex[e])
            Ge = f64(Gh[off:off + me])
            Ho[off:off + me] = O.expert_ffn_vjp(Ct[off:off + me], w1, bb1, w2, Ge)
            pre = Ct[off:off + me] @ w1.T + bb1
            near = np.abs(pre) < 1e-5 * np.abs(pre).max(axis=1, keepdims=True)
            back = Ge @ w2                                   # (W2^T G) per hidden unit
            for r in range(me):
                ref = Ho[off + r]
                js = np.nonzero(near[r])[0]
                n_near += len(js)
                assert len(js) <= 8, "implausibly many relu' near-ties in one row"
                best = np.inf
                for bits in range(1 << len(js)):             # every admissible mask of the near-tie units
                    alt = ref.copy()
                    for u, j in enumerate(js):
                        if (bits >> u) & 1:
                            alt += (-1.0 if pre[r, j] > 0 else 1.0) * back[r, j] * w1[j]
                    best = min(best, np.abs(Hg[off + r] - alt).max() / max(np.abs(alt).max(), 1e-30))
                worst = max(worst, best)
        off += me
    print(f"[expert bwd {cfgname}] m={m} relu' near-tie units={n_near} worst row err={worst:.2e}")
    assert worst <= tol
