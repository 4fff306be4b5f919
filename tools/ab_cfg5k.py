"""cfg5 derivatives-pass timing (4800 active x P candidates, k_u=24, k_x=12)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_15661_b200 import _lib, configs
from paper_2305_15661_b200.eqp import WeightVector
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases
case = configs.cfg5_rom(256)
op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)
rho = WeightVector(case.rho)
K = 36
for P in (256, 32):
    W = torch.as_tensor(case.W[:P]).cuda(); Tau = torch.zeros((P, 12), dtype=torch.float64, device="cuda")
    Mu = torch.as_tensor(case.mus[:P]).cuda()
    out = torch.empty(P * (1 + K + K * K), dtype=torch.float64, device="cuda")
    f = lambda: op.eval_batched(_lib.DERIVS, W, Tau, Mu, rho, out=out)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record(); torch.cuda.synchronize()
    print(f"{os.environ.get('TAG','')} cfg5 P={P}: {e0.elapsed_time(e1)/5*1e3:.1f} us per pass")
