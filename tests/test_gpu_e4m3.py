"""GPU parity of NEXT-2's fp8 option (reading R28): the e4m3 rotation bytes (host library vs the
oracle's independent rounding), the per-token e4m3 quantisation (bit-exact), and the codes of
lshmoe_hash_e4m3 against Eq. 3 evaluated exactly (fp64) on the quantised values — tier 1 with the
oracle's near-ties (< 1e-5) reported."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import CONFIGS, NEAR_TIE, f64, small_cfg
from lshmoe_inputs import make_tokens, rotation_seed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2411_08446_b200 as L
    return L


def _e4m3_values(u8: torch.Tensor) -> np.ndarray:
    return u8.view(torch.float8_e4m3fn).to(torch.float64).cpu().numpy()


@pytest.mark.parametrize("cfg", [small_cfg(n=1000, d=128, q=3), small_cfg(n=777, d=256, q=2), CONFIGS["C2"]],
                         ids=["d128", "d256", "C2"])
def test_hash_e4m3_parity(L, cfg):
    X = make_tokens(cfg, 2)
    seed = rotation_seed(2)
    R8 = L.rotation_e4m3(cfg.d, cfg.q, seed)
    Rq = O.quantize_rotation_e4m3(O.to_stored(O.rotation(cfg.d, cfg.q, seed, "f32"), "f32"))
    assert np.array_equal(_e4m3_values(R8), Rq), "library e4m3 rotation != oracle"
    x8 = L.quantize_e4m3(X.cuda())
    Xq = O.quantize_tokens_e4m3(f64(X))
    assert np.array_equal(_e4m3_values(x8), Xq), "GPU e4m3 quantisation != oracle"
    codes = L.hash_e4m3(x8, R8.cuda()).cpu().numpy()
    want, margins = O.cp_hash(Xq, Rq)
    mism = codes != want
    near = margins < NEAR_TIE
    print(f"[hash e4m3 d={cfg.d} q={cfg.q} n={cfg.n}] mismatches={int(mism.sum())} near-ties={int(near.sum())}")
    assert not (mism & ~near).any()
    # the fp8 codes are a different hash of x than the bf16 one; report how often they agree
    full, _ = O.cp_hash(f64(X), O.to_stored(O.rotation(cfg.d, cfg.q, seed, "bf16"), "bf16"))
    print(f"    agreement with the bf16 CP codes: {float((full == want).mean()):.3f}")
