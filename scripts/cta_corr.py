"""Per-CTA centroid-phase duration vs the CTA's segment count (C2), for tuning."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08446_b200 as L  # noqa: E402
from lshmoe_inputs import CONFIGS, make_rank_inputs, rotation_seed  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
X, zeta, _ = make_rank_inputs(cfg, 0, 0)
X, zeta = X.cuda(), zeta.cuda()
R = L.rotation(cfg.d, cfg.q, rotation_seed(0), X.dtype).cuda()
codes = L.hash(X, R)
ws = torch.empty(L.compress_workspace_bytes(cfg.n, cfg.k, cfg.E, cfg.q, cfg.d, X.dtype), dtype=torch.uint8, device="cuda")
comp = L.alloc_compressed(cfg.n, cfg.k, cfg.E, cfg.d, X.dtype, "cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
durs = []
for it in range(10):
    if not os.environ.get('NOFLUSH'):
        flush.zero_()
    L.compress(X, codes, zeta, cfg.E, out=comp, workspace=ws)
    torch.cuda.synchronize()
    hdr = ws[:4 * 2112].cpu().view(torch.int32).numpy().astype(np.int64) & 0xFFFFFFFF
    G = torch.cuda.get_device_properties(0).multi_processor_count
    durs.append((hdr[65:65 + 2 * G:2] - hdr[64:64 + 2 * G:2]) / 1e3)
dur = np.median(np.stack(durs), axis=0)
m = int(comp.num_rows.item())
nk = cfg.n * cfg.k
rs = comp.row_start[:m + 1].cpu().numpy()
rows = np.repeat(np.arange(m), np.diff(rs))
segs = np.array([len(np.unique(rows[b * nk // G:(b + 1) * nk // G])) for b in range(G)])
print("corr(dur, segs) =", np.corrcoef(dur, segs)[0, 1])
order = np.argsort(segs)
for b in order[::max(1, G // 20)]:
    print(f"cta {b:3d} segs {segs[b]:3d} dur {dur[b]:.2f}")
A = np.vstack([segs, np.ones(G)]).T
coef = np.linalg.lstsq(A, dur, rcond=None)[0]
print(f"fit: dur = {coef[1]:.2f} us + {coef[0] * 1e3:.1f} ns * segs")
