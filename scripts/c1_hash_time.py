import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2411_08446_b200 as L
from lshmoe_inputs import CONFIGS, make_tokens, rotation_seed
cfg = CONFIGS["C1"]
X = make_tokens(cfg, 0).cuda()
R = L.rotation(cfg.d, cfg.q, rotation_seed(0), X.dtype).cuda()
codes = L.hash(X, R)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(50):
        L.hash(X, R, codes=codes)
g.replay(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); g.replay(); b.record(); torch.cuda.synchronize()
print(f"C1 f32 SIMT hash (n={cfg.n}, d={cfg.d}, q={cfg.q}): {a.elapsed_time(b) * 1e3 / 50:.2f} us per launch (graph of 50)")
