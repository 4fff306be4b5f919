import os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2305_15661_b200 import configs
from paper_2305_15661_b200.eqp import WeightVector
from paper_2305_15661_b200.lm import LmConfig, lm_solve_batched
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases
for which in ("3", "5"):
    case = configs.cfg3() if which == "3" else configs.cfg5_rom(256)
    op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)
    res = lm_solve_batched(op, case.mus, case.W[0], None, WeightVector(case.rho), LmConfig(max_iters=30 if which == "3" else 10))
    al = np.concatenate([r.history[:, 5] for r in res])
    al = al[np.isfinite(al)]
    vals, cnt = np.unique(al, return_counts=True)
    print("cfg", which, "rows", al.size, dict(zip(vals.tolist(), cnt.tolist())))
    print(" reasons", {r.reason for r in res}, "evals mean", np.mean([r.n_iters for r in res]))
