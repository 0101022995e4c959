"""A/B of the restore kernel variants (LSHMOE_RESTORE_VAR) timed as bench.py times its stages: K
launches back to back in one CUDA graph over S copies of x / y larger than 2x L2 (no flush tax),
us per launch; outputs must be bit-identical to variant 0.
Usage: python scripts/restore_ab2.py C2,C5 0,2,4,12,14"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08446_b200 as L  # noqa: E402
from lshmoe_inputs import CONFIGS, make_rank_inputs, rotation_seed  # noqa: E402

K = 24
for cfgname in sys.argv[1].split(","):
    cfg = CONFIGS[cfgname]
    X, zeta, _ = make_rank_inputs(cfg, 0, 0)
    X, zeta = X.cuda(), zeta.cuda()
    R = L.rotation(cfg.d, cfg.q, rotation_seed(0), X.dtype).cuda()
    comp = L.compress(X, L.hash(X, R), zeta, cfg.E)
    m = int(comp.num_rows.item())
    ret = (comp.centroids.float() * 0.5 + 0.25).to(X.dtype)
    S = max(4, int(2 * 126e6 // (2 * X.numel() * X.element_size())) + 1)
    xs = [X.clone() for _ in range(S)]
    ys = [torch.empty_like(X) for _ in range(S)]
    nb = 2 * X.numel() * X.element_size() + 2 * m * cfg.d * X.element_size() + 4 * cfg.n * cfg.k
    ref = None
    for var in sys.argv[2].split(","):
        os.environ["LSHMOE_RESTORE_VAR"] = var
        for i in range(S):
            L.restore(xs[i], comp.centroids, ret, comp.bucket, y=ys[i])
        torch.cuda.synchronize()
        if ref is None:
            ref = ys[0].clone()
        same = torch.equal(ref, ys[0])
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(K):
                L.restore(xs[i % S], comp.centroids, ret, comp.bucket, y=ys[i % S])
        g.replay()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e3 / K)
        print(f"{cfgname} restore var={var}: {best:.2f} us/launch  {nb / best / 1e3:.0f} GB/s "
              f"({nb / best / 1e3 / 6543:.3f} of HBM)  identical={same}", flush=True)
    os.environ.pop("LSHMOE_RESTORE_VAR")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(K):
            ys[i % S].copy_(xs[i % S])
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / K
    nb2 = 2 * X.numel() * X.element_size()
    print(f"{cfgname} torch copy x->y: {us:.2f} us/launch  {nb2 / us / 1e3:.0f} GB/s", flush=True)
