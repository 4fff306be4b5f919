"""cfg3 derivs pass timing (800 active x P mu) for grid-shape experiments."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_15661_b200 import _lib, configs
from paper_2305_15661_b200.eqp import WeightVector
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases
case = configs.cfg3()
op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)
rho = WeightVector(case.rho)
K = 30
for P in (64, 16):
    W = torch.as_tensor(case.W[:P]).cuda(); Tau = torch.as_tensor(case.Tau[:P]).cuda(); Mu = torch.as_tensor(case.mus[:P]).cuda()
    out = torch.empty(P * (1 + K + K * K), dtype=torch.float64, device="cuda")
    f = lambda: op.eval_batched(_lib.DERIVS, W, Tau, Mu, rho, out=out)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record(); torch.cuda.synchronize()
    print(f"P={P} UPW={os.environ.get('STROM_MMA_UPW','-')}: {e0.elapsed_time(e1)/10*1e3:.1f} us per pass")
