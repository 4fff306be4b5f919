"""Diagnostics for the config-4 / config-5 bench paths (non-finite LP rows, failed candidates)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_15661_b200 import _lib, configs, sharded
from paper_2305_15661_b200.eqp import WeightVector
from paper_2305_15661_b200.greedy import indicators
from paper_2305_15661_b200.lm import LmConfig, lm_solve_batched
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

which = sys.argv[1]
if which == "4":
    case = configs.cfg4_case()
    op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)
    ne = case.mesh.num_elements
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    mus, U, X = sharded.snapshot_fields_device(case, np.arange(S), 4, op.device)
    print("fields finite", bool(torch.isfinite(U).all()), bool(torch.isfinite(X).all()), mus.ravel())
    rows = op.contributions_at_snapshots(U, X, mus, "lprows")
    bad = ~torch.isfinite(rows)
    print("rows", tuple(rows.shape), "non-finite", int(bad.sum()))
    if bad.any():
        idx = torch.nonzero(bad)[:10].cpu().numpy()
        print("first bad (s, row, e):", idx.tolist())
        degen = torch.zeros(S, dtype=torch.int32, device=op.device)
        W = torch.zeros((S, 20), dtype=torch.float64, device=op.device)
        T = torch.zeros((S, 10), dtype=torch.float64, device=op.device)
        _lib.check(_lib.load().strom_set_offsets(op._h, U.data_ptr(), U.shape[1], X.data_ptr(), X.shape[1]), "off")
        out, _ = op.eval_batched(_lib.RESNORM2, W, T, torch.as_tensor(mus).cuda(), None, degen=degen)
        print("resnorm2", out.cpu().numpy(), "degen", degen.cpu().numpy())
else:
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    case = configs.cfg5_rom(P)
    if len(sys.argv) > 3:  # distortion weight override (cfg5_rom default: 1.0)
        case.kappa = float(sys.argv[3])
        print("kappa", case.kappa)
    op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)
    res = lm_solve_batched(op, case.mus, case.W[0], None, WeightVector(case.rho), LmConfig(max_iters=10))
    W = np.stack([r.w for r in res]); T = np.stack([r.tau for r in res])
    reasons = {}
    for r in res:
        reasons[r.reason] = reasons.get(r.reason, 0) + 1
    print("reasons", reasons, "objective finite", sum(np.isfinite(r.objective) for r in res))
    print("|tau| quantiles", np.quantile(np.linalg.norm(T, axis=1), [0, 0.5, 1]))
    ind = indicators(op, case.mus, W, T)
    print("indicators finite", int(np.isfinite(ind).sum()), "of", P, "quantiles", np.quantile(ind[np.isfinite(ind)], [0, 0.5, 1]) if np.isfinite(ind).any() else None)
    dx = case.psi @ T.T
    print("max |Psi tau| node displacement", np.abs(dx).max(), "h ~", 1.0 / 400)
