"""Where the time of a batched LM solve goes (cfg3): wall vs device kernel time per kernel."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_15661_b200 import configs
from paper_2305_15661_b200.eqp import WeightVector
from paper_2305_15661_b200.lm import LmConfig, lm_solve_batched
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

which = sys.argv[1] if len(sys.argv) > 1 else "3"
case = configs.cfg3() if which == "3" else (configs.cfg5_rom(256) if which == "5" else configs.strip_case())
op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)
rho = WeightVector(case.rho)
W0 = case.W[0] if which in ("3", "5") else None
cfg = LmConfig(max_iters=10 if which == "5" else 30)
lm_solve_batched(op, case.mus, W0, None, rho, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = lm_solve_batched(op, case.mus, W0, None, rho, cfg)
dt = time.perf_counter() - t0
print(f"wall {dt*1e3:.2f} ms, iters {np.mean([r.n_iters for r in res]):.1f}")
import ctypes
from paper_2305_15661_b200 import _lib
st = (ctypes.c_int32 * 3)()
_lib.load().strom_lm_stats(op._h, st)
print("rounds, derivative passes, objective passes:", list(st))
tm = (ctypes.c_double * 4)()
_lib.load().strom_lm_timing(op._h, tm)
print("device ms: control %.2f, after d-only rounds %.2f, o-only %.2f, d+o %.2f" % tuple(tm))
rw = (ctypes.c_double * 2)()
_lib.load().strom_lm_rows(op._h, rw)
print("rows evaluated: derivatives %d (%.1f per mu), objective trials %d (%.1f per mu)" % (rw[0], rw[0] / len(res), rw[1], rw[1] / len(res)))
# per-kernel times of the graph's kernel nodes: run under
#   ncu --metrics gpu__time_duration.sum --csv python tools/prof_lm.py 3  (tools/launch_summary.py)
