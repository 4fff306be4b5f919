"""K1 derivatives-pass time on config 2 for the numerical-flux / wall variants (Euler LLF,
Euler Roe; cfg3 sector with extrapolated vs slip wall)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_15661_b200 import _lib, configs, laws as L
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases


def time_pass(case, P=1, reps=20):
    op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist,
                            state_offset=case.state_offset)
    ku, kx = op.k_u, op.k_x
    K = ku + kx
    W = torch.as_tensor(np.tile(case.W[0], (P, 1))).cuda()
    Tau = torch.zeros((P, kx), dtype=torch.float64, device="cuda")
    Mu = torch.as_tensor(np.tile(case.mus[0], (P, 1))).cuda()
    out = torch.empty(P * (1 + K + K * K), dtype=torch.float64, device="cuda")
    rho = None if case.rho is None else __import__("paper_2305_15661_b200.eqp", fromlist=["x"]).WeightVector(case.rho)
    for _ in range(3):
        op.eval_batched(_lib.DERIVS, W, Tau, Mu, rho, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        op.eval_batched(_lib.DERIVS, W, Tau, Mu, rho, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


c = configs.euler_square_case(n=256)
print("cfg2 LLF  ms", round(time_pass(c), 4))
c.law = L.euler(tags={t: "freestream" for t in ("left", "right", "bottom", "top")}, flux="roe")
print("cfg2 Roe  ms", round(time_pass(c), 4))
for wall in ("extrapolate", "slip"):
    s = configs.sector_rom_case(wall=wall)
    print(f"cfg3 {wall:11s} 64 mu ms", round(time_pass(s, P=64), 4))
s = configs.sector_rom_case(wall="slip", flux="roe")
print("cfg3 slip+Roe 64 mu ms", round(time_pass(s, P=64), 4))
