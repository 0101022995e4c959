"""Calibrate the generator's noise rho so q=6 gives the paper's compression rates
(~20% at q~6; 11.7% on Swin).  Calls only oracle/ and lshmoe_inputs/."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle as O
from lshmoe_inputs import CONFIGS, make_rank_inputs, rotation_seed

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C2"
rhos = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [None]
nsub = int(sys.argv[3]) if len(sys.argv) > 3 else None
cfg = CONFIGS[cfg_name]
t = time.time()
R = O.to_stored(O.rotation(cfg.d, 8, rotation_seed(0), cfg.dtype), cfg.dtype)
print("rotation", time.time() - t, flush=True)
for rho in rhos:
    c = cfg if rho is None else cfg.with_(rho=rho)
    if nsub: c = c.with_(n=nsub)
    X, zeta, _ = make_rank_inputs(c, 0, 0)
    Xf = X.to(__import__("torch").float64).numpy()
    codes, margins = O.cp_hash(Xf, R)
    rs = []
    for q in range(1, 9):
        b = O.bucketize(codes[:, :q], zeta.numpy(), c.E)
        rs.append(round(b.m / zeta.numel(), 4))
    print(cfg_name, "rho", c.rho, "r(q=1..8)", rs, "near-ties(<1e-5)", int((margins[:, :6] < 1e-5).sum()), flush=True)
