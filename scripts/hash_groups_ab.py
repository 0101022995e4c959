"""A/B of the hash kernel's cluster shapes on one workload (default C2): MMA group (1 CTA, M = 128 /
CTA pair, M = 256) x groups per cluster (LSHMOE_HASH_GROUPS: MMA groups on adjacent token tiles that
walk the same (j, slice) chunk sequence, so their B loads coincide).  Timing as bench.py: K launches
back to back in one CUDA graph over S token copies larger than 2x L2; codes compared with the
default configuration's.  Usage: python scripts/hash_groups_ab.py [C2|C3|C4|C5] [K]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08446_b200 as L  # noqa: E402
from lshmoe_inputs import CONFIGS, make_rank_inputs, rotation_seed  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    X, _, _ = make_rank_inputs(cfg, 0, 0)
    X = X.cuda()
    S = max(4, int(2 * 126e6 // (X.numel() * X.element_size())) + 1)
    xs = [X.clone() for _ in range(S)]
    R = L.rotation(cfg.d, cfg.q, rotation_seed(0), X.dtype).cuda()
    ws = L.hash_workspace(cfg.n, cfg.d, cfg.q, X.dtype, X.device)
    flops = 2.0 * cfg.n * cfg.q * cfg.d * cfg.d
    ref = L.hash(X, R, workspace=ws).clone()
    codes = torch.empty_like(ref)
    shapes = [(c, g) for c in ("1", "2") for g in ("1", "2", "4")]
    if len(sys.argv) > 3:
        shapes = [tuple(s.split("x")) for s in sys.argv[3].split(",")]
    for cta, groups in shapes:
        os.environ["LSHMOE_HASH_CTA"] = cta
        os.environ["LSHMOE_HASH_GROUPS"] = groups
        try:
            codes.zero_()
            L.hash(X, R, codes, workspace=ws)
            torch.cuda.synchronize()
            mism = int((codes != ref).sum().item())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(K):
                    L.hash(xs[i % S], R, codes, workspace=ws)
            for _ in range(2):
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
            print(f"{cfg.name} hash cta={cta} groups={groups}: {best:.1f} us/launch  {flops / best / 1e6:.0f} TFLOP/s  "
                  f"code mismatches vs default {mism}", flush=True)
        except Exception as ex:   # noqa: BLE001
            print(f"cta={cta} groups={groups}: FAILED {str(ex)[:300]}", flush=True)
            torch.cuda.synchronize()


if __name__ == "__main__":
    main()
