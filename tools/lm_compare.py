import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from cases import build
from test_gpu_lm import gpu_op, leading_agreement
from paper_2305_15661_b200.eqp import WeightVector
from paper_2305_15661_b200.lm import LmConfig, lm_solve_batched
for name in ["strip", "sector"]:
    case, g = build(name)
    op = gpu_op(case)
    cfg = LmConfig(max_iters=int(g["lm_max_iters"]))
    w0 = case.W[0] if name == "sector" else None
    res = lm_solve_batched(op, case.mus[:2], w0, None, WeightVector(case.rho), cfg)
    for i, r in enumerate(res):
        hr = g[f"lm{i}_hist"]
        print(name, i, "rows", len(r.history), len(hr), "agree", leading_agreement(r.history, hr), r.reason, str(g[f"lm{i}_reason"]),
              "w err", np.max(np.abs(r.w - g[f"lm{i}_w"])), "obj", r.objective, float(g[f"lm{i}_obj"]))
