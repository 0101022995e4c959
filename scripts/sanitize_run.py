"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
the hash with its slice merge, the three compress kernels (C1 f32 and a small bf16 top-2 case with a
giant bucket), the expert FFN, restore, the phase-2 exchange in a local group of 2 virtual ranks,
the fused compress+dispatch at world 1, the NEXT-1 backward kernels, SP / e4m3 / hd3 hashes.
Prints one line per stage; any sanitizer finding is reported by the tool itself."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08446_b200 as L  # noqa: E402
from lshmoe_inputs import CONFIGS, LayerConfig, make_experts, make_gate, make_tokens, rotation_seed  # noqa: E402


def layer(cfg, seed=0, giant=False):
    X = make_tokens(cfg, seed)
    if giant:
        X[: cfg.n // 2] = X[0]
    zeta, g = make_gate(cfg, seed, X, True)
    Xd, zd = X.cuda(), zeta.cuda()
    R = L.rotation(cfg.d, cfg.q, rotation_seed(seed), X.dtype).cuda()
    codes = L.hash(Xd, R)
    out = L.compress(Xd, codes, zd, cfg.E)
    ex = make_experts(cfg, seed)
    W = [torch.stack([ex[e][i] for e in range(cfg.E)]).cuda() for i in range(4)]
    rr = torch.empty((cfg.E, 1), dtype=torch.int32, device="cuda")
    recv = torch.empty_like(out.centroids)
    L.dispatch(None, out.centroids, out.expert_rows, cfg.E, recv, rr)
    hid = torch.empty((recv.shape[0], cfg.d_ffn), dtype=X.dtype, device="cuda")
    eo = L.expert_ffn(recv, rr, *W, hidden=hid)
    ret = torch.empty_like(out.centroids)
    L.combine(None, eo, out.expert_rows, cfg.E, ret)
    y = L.restore(Xd, out.centroids, ret, out.bucket, g.cuda())
    dY = torch.randn_like(Xd)
    G = L.grad_compress(dY, out, g.cuda())
    if X.dtype == torch.bfloat16:
        H = L.expert_ffn_backward(G, rr, W[2].transpose(1, 2).contiguous(), W[0].transpose(1, 2).contiguous(), hid)
    else:
        H = G
    L.grad_restore(dY, Xd, out.centroids, ret, G, H, out, g.cuda(), want_dgate=True)
    torch.cuda.synchronize()
    L.check_device_error()
    print(f"{cfg.name}: layer fwd+bwd ok (m={int(out.num_rows.item())})", flush=True)
    return Xd, zd, codes


layer(CONFIGS["C1"])
small = LayerConfig("S-bf16", 3000, 768, 8, 2, 6, "bf16", 512, 24, 0.1)
Xd, zd, codes = layer(small, giant=True)
layer(LayerConfig("S-bf16-k1", 2000, 768, 8, 1, 6, "bf16", 512, 24, 0.1))   # two-row restore, group path k = 1
layer(LayerConfig("S-f32-tiles", 17000, 64, 4, 1, 2, "f32", 256, 16, 0.1))   # n*k > 16K: the tiles compress path
# NEXT-2/3/4 hashes
L.sp_hash(Xd, L.sp_normals(L.rotation(768, 6, 3, torch.bfloat16).cuda(), 12), 6, 12)
L.hash_e4m3(L.quantize_e4m3(Xd), L.rotation_e4m3(768, 6, 3).cuda())
L.hash_hd3(Xd, L.hd3_signs(6, 3).cuda())
torch.cuda.synchronize()
print("sp / e4m3 / hd3 hashes ok", flush=True)
# NEXT-2 gate + hash, then compress on the same stream (the gate map is read after the dependency
# wait here; the plain compress calls above read it before)
Wg = (torch.randn((small.E, 768)) / 768 ** 0.5).to(torch.bfloat16)
RG = L.rotation_gate(L.rotation(768, 6, 3, torch.bfloat16), Wg).cuda()
gcodes, gzeta, _ = L.gate_hash(Xd, RG, 6, small.E, 2)
L.compress(Xd, gcodes, gzeta, small.E)
torch.cuda.synchronize()
print("gate_hash -> compress ok", flush=True)
# phase 2: local group of 2 virtual ranks (each on its own stream), then the fused compress at world 1
E, d = 8, 768
comms = L.Comm.local_group(2, 4000, 4000, d, torch.bfloat16, E)
streams = [torch.cuda.Stream() for _ in range(2)]
C = [torch.randn((300, d), device="cuda").to(torch.bfloat16) for _ in range(2)]
er = [torch.tensor([40] * 7 + [20], dtype=torch.int32, device="cuda") for _ in range(2)]
torch.cuda.synchronize()
for r in range(2):
    with torch.cuda.stream(streams[r]):
        L.dispatch_p2p(comms[r], C[r], er[r], grid=4, stream=streams[r])
torch.cuda.synchronize()
for r in range(2):
    recv, _, _ = comms[r].p2p_buffers()
    with torch.cuda.stream(streams[r]):
        L.combine_p2p(comms[r], recv[:300], grid=4, stream=streams[r])
torch.cuda.synchronize()
for c in comms:
    c.p2p_check()
    c.close()
comm = L.Comm(1, 0).p2p_init(3000 * 2, 3000 * 2, d, torch.bfloat16, small.E)
L.compress_p2p(comm, Xd, codes, zd, small.E)
torch.cuda.synchronize()
comm.p2p_check()
comm.close()
print("phase-2 exchange + fused compress ok", flush=True)
