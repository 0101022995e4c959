"""GPU parity of NEXT-2's gate + hash (reading R29): one lshmoe_gate_hash pass gives the same codes
as lshmoe_hash / the oracle's cp_hash and the oracle's gate_topk (ids bit-exact except tokens whose
score margin at the k-th place is below 1e-5; weights within 1e-4)."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import CONFIGS, NEAR_TIE, f64, make_case, small_cfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2411_08446_b200 as L
    return L


@pytest.mark.parametrize("cfg", [small_cfg(n=1000, d=128, E=6, k=2, q=3), small_cfg(n=700, d=256, E=64, k=4, q=2),
                                 CONFIGS["C2"], CONFIGS["C3"].with_(n=4096)], ids=["small", "E64k4", "C2", "C3-4K"])
def test_gate_hash(L, cfg):
    case = make_case(L, cfg, seed=4, sanitize=False)
    rng = np.random.default_rng(3)
    Wg = torch.from_numpy(rng.standard_normal((cfg.E, cfg.d)) / np.sqrt(cfg.d)).to(torch.float32).to(case.X.dtype)
    RG = L.rotation_gate(case.R_lib, Wg).cuda()
    codes, zeta, gw = L.gate_hash(case.X.cuda(), RG, cfg.q, cfg.E, cfg.k)
    torch.cuda.synchronize()
    got = codes.cpu().numpy()
    bad_codes = (got != case.codes) & (case.margins >= NEAR_TIE)
    assert not bad_codes.any()
    z_o, g_o, margin = O.gate_topk(f64(case.X), f64(Wg), cfg.k)
    clean = margin >= NEAR_TIE
    z = zeta.cpu().numpy()
    mism = (z != z_o).any(axis=1)
    print(f"[gate_hash {cfg.name} E={cfg.E} k={cfg.k}] gate mismatches={int(mism.sum())} "
          f"near-ties={int((~clean).sum())}")
    assert not (mism & clean).any()
    assert np.abs(gw.cpu().numpy()[clean] - g_o[clean]).max() <= 1e-4


def test_gate_hash_then_compress_ordering(L):
    """compress reads the gate map before griddepcontrol.wait unless the preceding kernel on the stream
    is lshmoe_gate_hash (which writes it): gate_hash -> compress back to back on one stream, with the
    gate map changing between calls (reversed tokens), must equal the same compress after a full
    synchronisation (compress.cu early_gate; lshmoe.h ordering note)."""
    cfg = CONFIGS["C2"]
    case = make_case(L, cfg, seed=5, sanitize=False)
    rng = np.random.default_rng(7)
    Wg = torch.from_numpy(rng.standard_normal((cfg.E, cfg.d)) / np.sqrt(cfg.d)).to(torch.float32).to(case.X.dtype)
    RG = L.rotation_gate(case.R_lib, Wg).cuda()
    n, d = case.X.shape
    ws = L.compress_workspace(n, cfg.k, cfg.E, cfg.q, d, case.X.dtype, "cuda")
    outs = [L.alloc_compressed(n, cfg.k, cfg.E, d, case.X.dtype, "cuda") for _ in range(2)]
    X0 = case.X.cuda()
    xs = [X0, X0.flip(0).contiguous()]
    torch.cuda.synchronize()
    inputs = []
    for X, out in zip(xs, outs):
        codes, zeta, _ = L.gate_hash(X, RG, cfg.q, cfg.E, cfg.k)
        L.compress(X, codes, zeta, cfg.E, out=out, workspace=ws)   # no launch in between
        inputs.append((X, codes, zeta))
    torch.cuda.synchronize()
    for (X, codes, zeta), out in zip(inputs, outs):
        ref = L.compress(X, codes, zeta, cfg.E)
        torch.cuda.synchronize()
        m = int(ref.num_rows.item())
        assert int(out.num_rows.item()) == m
        for f in ("bucket", "perm", "expert_rows"):
            assert torch.equal(getattr(out, f), getattr(ref, f)), f
        assert torch.equal(out.row_start[:m + 1], ref.row_start[:m + 1])
        assert torch.equal(out.centroids[:m], ref.centroids[:m])
