"""Standalone device times of the batched passes an LM round launches on config 3 (800 EQP elements):
K2 objective over P trial rows and K1 derivatives over P rows, CUDA events over 200 launches."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_15661_b200 import _lib, configs
from paper_2305_15661_b200.eqp import WeightVector
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

case = configs.cfg3()
op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)
rho = WeightVector(case.rho)
dev = op.device
for mode, name, Ps in ((_lib.OBJECTIVE, "K2 objective", (32, 64, 128, 256)), (_lib.DERIVS, "K1 derivatives", (8, 16, 32, 64))):
    for P in Ps:
        W = torch.as_tensor(np.tile(case.W[0], (P, 1))).to(dev)
        Tau = torch.zeros((P, op.k_x), dtype=torch.float64, device=dev)
        Mu = torch.as_tensor(np.resize(case.mus, (P, 1)).astype(float)).to(dev)
        out = None
        for _ in range(5):
            out, _ = op.eval_batched(mode, W, Tau, Mu, rho, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            op.eval_batched(mode, W, Tau, Mu, rho, out=out)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} P={P}: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us per pass (incl. its reduction kernel and launch gaps)")
