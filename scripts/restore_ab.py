"""A/B of the restore kernel variants (LSHMOE_RESTORE_VAR) on a config's real compressed rows:
graph-replayed, L2 flushed before each replay; outputs must be bit-identical to variant 0."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08446_b200 as L  # noqa: E402
from lshmoe_inputs import CONFIGS, make_rank_inputs, rotation_seed  # noqa: E402
from ab_bench import timeit  # noqa: E402

for cfgname in sys.argv[1].split(","):
    cfg = CONFIGS[cfgname]
    X, zeta, _ = make_rank_inputs(cfg, 0, 0)
    X, zeta = X.cuda(), zeta.cuda()
    R = L.rotation(cfg.d, cfg.q, rotation_seed(0), X.dtype).cuda()
    comp = L.compress(X, L.hash(X, R), zeta, cfg.E)
    m = int(comp.num_rows.item())
    ret = (comp.centroids.float() * 0.5 + 0.25).to(X.dtype)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    nb = 2 * X.numel() * X.element_size() + 2 * m * cfg.d * X.element_size() + 4 * cfg.n * cfg.k
    ref = None
    for var in sys.argv[2].split(","):
        os.environ["LSHMOE_RESTORE_VAR"] = var
        y = torch.empty_like(X)
        y.copy_(X)
        med, mn = timeit(lambda: L.restore(X, comp.centroids, ret, comp.bucket, y=y), flush=flush)
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        same = torch.equal(ref, y)
        print(f"{cfgname} restore var={var}: median {med:.2f} us  min {mn:.2f}  {nb / med / 1e3:.0f} GB/s "
              f"({nb / med / 1e3 / 6454:.3f} of HBM)  identical={same}", flush=True)
    os.environ.pop("LSHMOE_RESTORE_VAR")
    y = torch.empty_like(X)
    med, mn = timeit(lambda: y.copy_(X), flush=flush)
    nb2 = 2 * X.numel() * X.element_size()
    print(f"{cfgname} torch copy x->y: median {med:.2f} us  {nb2 / med / 1e3:.0f} GB/s", flush=True)
