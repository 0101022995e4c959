"""Expert-FFN probe (tuning aid): grouped FFN on synthetic received rows shaped like a config's
centroids (E experts, ~m/E rows each), random weights made on the device; times GEMM 1 / GEMM 2 /
both (graph replays, events) -- and is short enough to run under ncu."""
import os
import sys

import torch
os.environ.setdefault("LSHMOE_EXPERIMENTS", "1")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08446_b200 as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
E, d, dff, m = {"C2": (16, 768, 3072, 3128), "C3": (32, 1024, 4096, 12558), "C4": (64, 1024, 16384, 13389)}[cfg]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g = torch.Generator(device="cuda").manual_seed(0)
rows = torch.full((E, 1), m // E, dtype=torch.int32)
rows[: m % E] += 1
rr = rows.cuda()
x = torch.randn((m, d), device="cuda", generator=g).to(torch.bfloat16)
W1 = (torch.randn((E, dff, d), device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
b1 = torch.zeros((E, dff), device="cuda", dtype=torch.bfloat16)
W2 = (torch.randn((E, d, dff), device="cuda", generator=g) / dff ** 0.5).to(torch.bfloat16)
b2 = torch.zeros((E, d), device="cuda", dtype=torch.bfloat16)
out = torch.empty_like(x)
hid = torch.empty((m, dff), device="cuda", dtype=torch.bfloat16)
fl = 4.0 * m * d * dff
wbytes = 2 * E * d * dff * 2
for only in (os.environ.get("ONLY", "1,2,0").split(",")):
    if only != "0":
        os.environ["LSHMOE_FFN_ONLY"] = only
    else:
        os.environ.pop("LSHMOE_FFN_ONLY", None)
    L.expert_ffn(x, rr, W1, b1, W2, b2, out=out, hidden=hid)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        L.expert_ffn(x, rr, W1, b1, W2, b2, out=out, hidden=hid)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    f = fl / 2 if only != "0" else fl
    wb = wbytes / 2 if only != "0" else wbytes
    print(f"{cfg} ffn gemm={only or 'both'}: {us:.1f} us  {f / us / 1e6:.0f} TFLOP/s  weights {wb / us / 1e3:.0f} GB/s", flush=True)
