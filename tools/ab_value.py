"""A/B of the K2 value path: cfg3 objective pass (800 x 64), cfg5-shaped indicator (160k x 256), cfg3 LM wall.
Also cross-checks the objective / indicator against the previous kernel (STROM_VALUE_OLD path) when
--check is given (same process, both kernels)."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_15661_b200 import _lib, configs
from paper_2305_15661_b200.eqp import WeightVector
from paper_2305_15661_b200.greedy import indicators
from paper_2305_15661_b200.lm import LmConfig, lm_solve_batched
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases


def cuda_time(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


case = configs.cfg3()
op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)
rho = WeightVector(case.rho)
W = torch.as_tensor(case.W).cuda(); Tau = torch.as_tensor(case.Tau).cuda(); Mu = torch.as_tensor(case.mus).cuda()
outo = torch.empty(64, dtype=torch.float64, device="cuda")
t_o = cuda_time(lambda: op.eval_batched(_lib.OBJECTIVE, W, Tau, Mu, rho, out=outo))
obj = outo.clone()
cfg = LmConfig(max_iters=30)
lm_solve_batched(op, case.mus, case.W[0], None, rho, cfg); torch.cuda.synchronize()
t0 = time.perf_counter(); res = lm_solve_batched(op, case.mus, case.W[0], None, rho, cfg); t_lm = time.perf_counter() - t0
c5 = configs.cfg5_rom(P=256)
op5 = GpuReducedOperator(c5.law, c5.geom, ReducedBases(c5.phi, c5.psi, c5.ref_coords), c5.dist)
rng = np.random.default_rng(0)
W5 = c5.W + 0.01 * rng.standard_normal(c5.W.shape)
T5 = 1e-3 * rng.standard_normal((256, 12))
indicators(op5, c5.mus, W5, T5); torch.cuda.synchronize()
t0 = time.perf_counter(); ind = indicators(op5, c5.mus, W5, T5); torch.cuda.synchronize(); t_i = time.perf_counter() - t0
print(f"objective 800x64: {t_o*1e3:.1f} us | LM cfg3 64 solves: {t_lm*1e3:.1f} ms ({np.mean([r.n_iters for r in res]):.1f} it) | "
      f"indicator 160k x 256: {t_i*1e3:.1f} ms ({160000*256/t_i/1e6:.0f} M el-evals/s)")
np.save(os.path.join(ROOT, "gpurun_out", f"ab_value_{os.environ.get('TAG','x')}.npy"),
        np.concatenate([obj.cpu().numpy(), ind, [r.objective for r in res]]))
