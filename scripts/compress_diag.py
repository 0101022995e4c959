"""Diagnostics (not a test): per-CTA phase stamps of lshmoe_compress on a config's inputs.
Prints, per phase boundary, the max over CTAs and the critical CTA's sub-step times (us)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2411_08446_b200 as L  # noqa: E402
from lshmoe_inputs import CONFIGS, make_gate, make_tokens, rotation_seed  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
fused = len(sys.argv) > 2 and sys.argv[2] == "fused"   # lshmoe_compress_p2p at world 1
cfg = CONFIGS[name]
X = make_tokens(cfg, 0)
zeta, _ = make_gate(cfg, 0, X)
Xd, zd = X.cuda(), zeta.cuda()
R = L.rotation(cfg.d, cfg.q, rotation_seed(0), X.dtype).cuda()
codes = L.hash(Xd, R)
nk = cfg.n * cfg.k
ws = torch.full((L.compress_workspace_bytes(cfg.n, cfg.k, cfg.E, cfg.q, cfg.d, X.dtype),), 255, dtype=torch.uint8, device="cuda")
out = L.alloc_compressed(cfg.n, cfg.k, cfg.E, cfg.d, X.dtype, "cuda")
G = torch.cuda.get_device_properties(0).multi_processor_count
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
comm = L.Comm(1, 0).p2p_init(nk, nk, cfg.d, X.dtype, cfg.E) if fused else None
run = (lambda: L.compress_p2p(comm, Xd, codes, zd, cfg.E, out=out, workspace=ws)) if fused else \
    (lambda: L.compress(Xd, codes, zd, cfg.E, out=out, workspace=ws))
# K compress calls back to back in one CUDA graph over S copies of x at distinct addresses (tokens
# never L2-resident), events around the replay: us per call (the bench's method)
S = max(4, -(-2 * 126 * 10 ** 6 // (2 * Xd.numel() * Xd.element_size())))
Xs = [Xd] + [Xd.clone() for _ in range(S - 1)]
K = 4 * S
runs = [((lambda xx=xx: L.compress_p2p(comm, xx, codes, zd, cfg.E, out=out, workspace=ws)) if fused else
         (lambda xx=xx: L.compress(xx, codes, zd, cfg.E, out=out, workspace=ws))) for xx in Xs]
for r in runs:
    r()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(K):
        runs[i % S]()
g.replay()
times = []
for it in range(5):
    ev[0].record()
    g.replay()
    ev[1].record()
    torch.cuda.synchronize()
    times.append(ev[0].elapsed_time(ev[1]) * 1e3 / K)
print(f"{name}: compress graph time per call (K={K}, S={S} token sets): median {np.median(times):.1f} us "
      f"min {min(times):.1f}")
L.set_diagnostics(True)
run()
torch.cuda.synchronize()
L.set_diagnostics(False)
print("kernel spans", L.compress_phase_times(ws))
m = int(out.num_rows.item())
print(f"m={m} expert_rows max={int(out.expert_rows.max())}")
gsz = torch.bincount(zd.flatten().long(), minlength=cfg.E).cpu().numpy()
print(f"group sizes: max {int(gsz.max())} (expert {int(gsz.argmax())}), median {int(np.median(gsz))}; "
      f"rows of the largest group {int(out.expert_rows[int(gsz.argmax())])}")
for kern, st in L.compress_diag(ws).items():
    D = {k: np.array(v) for k, v in st.items()}
    if np.all(np.isnan(D["end"])):
        continue
    print(kern)
    for k, v in D.items():
        if np.all(np.isnan(v)):
            continue
        print(f"  {k:12s} max {np.nanmax(v):7.2f}  med {np.nanmedian(v):7.2f}  min {np.nanmin(v):7.2f}  argmax {int(np.nanargmax(v))}")
    crit = int(np.nanargmax(D["end"]))
    print("  critical CTA", crit, {k: round(float(D[k][crit]), 2) for k in D})
if fused:
    comm.p2p_check()                          # raises if any row was dropped (capacity)
    recv, _, rr = comm.p2p_buffers()
    m = int(out.num_rows.item())
    print("fused: rows delivered match the centroids:", bool(torch.equal(recv[:m], out.centroids[:m])))
