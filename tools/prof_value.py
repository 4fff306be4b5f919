# profile target: cfg5-shaped full-mesh indicator (value_mu_kernel), smaller P for ncu
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_15661_b200 import configs
from paper_2305_15661_b200.greedy import indicators
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases
case = configs.cfg5_rom(P=128)
op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)
rng = np.random.default_rng(0)
W = case.W + 0.01 * rng.standard_normal(case.W.shape)
Tau = 1e-3 * rng.standard_normal((128, 12))
for _ in range(3):
    ind = indicators(op, case.mus, W, Tau)
torch.cuda.synchronize()
import time; t0 = time.perf_counter(); ind = indicators(op, case.mus, W, Tau); torch.cuda.synchronize()
print("indicator 160k x 128:", time.perf_counter() - t0, "s", ind[:3])
