#!/usr/bin/env python
"""Measure the BASELINE.json configs beyond the headline (configs 1, 3, 4, 5) on one GPU.

Prints one JSON object per config (and writes profiles/configs_r01.json with --out).
All inputs are seeded synthetic (paper_2305_15661_b200.configs); config 4's
snapshots are generated on the device with a seeded torch generator (5 GB of
states; same distribution as configs.snapshot_fields).  Times are CUDA-event
/ wall clocks around device-resident work after a warm-up.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2305_15661_b200 import _lib, configs, laws as L  # noqa: E402
from paper_2305_15661_b200.eqp import WeightVector  # noqa: E402
from paper_2305_15661_b200.lm import LmConfig, lm_solve_batched  # noqa: E402
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases  # noqa: E402
import bench  # noqa: E402


def op_of(case, **kw):
    return GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist, **kw)


def cuda_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def lm_stats(res):
    it = np.array([r.n_iters for r in res])
    reasons = {}
    for r in res:
        reasons[r.reason] = reasons.get(r.reason, 0) + 1
    return {"iters_mean": float(it.mean()), "iters_max": int(it.max()), "reasons": reasons,
            "converged": int(sum(r.converged for r in res))}


def cfg1():
    case = configs.strip_case()
    op = op_of(case)
    rho = WeightVector(case.rho)
    cfg = LmConfig()
    lm_solve_batched(op, case.mus, None, None, rho, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = lm_solve_batched(op, case.mus, None, None, rho, cfg)
    dt = time.perf_counter() - t0
    return {"config": "cfg1 strip Burgers, 128 tri, k=4/2, 10 active, 8 mu", "lm_solves_per_s": len(res) / dt,
            "batch_wall_s": dt, **lm_stats(res)}


def cfg3(max_iters):
    case = configs.cfg3()
    op = op_of(case)
    rho = WeightVector(case.rho)
    K = case.phi.shape[1] + case.psi.shape[1]
    # one batched derivatives pass: 800 active x 64 mu
    W = torch.as_tensor(case.W).cuda()
    Tau = torch.as_tensor(case.Tau).cuda()
    Mu = torch.as_tensor(case.mus).cuda()
    out = torch.empty(64 * (1 + K + K * K), dtype=torch.float64, device="cuda")
    t_d = cuda_time(lambda: op.eval_batched(_lib.DERIVS, W, Tau, Mu, rho, out=out), 5)
    outo = torch.empty(64, dtype=torch.float64, device="cuda")
    t_o = cuda_time(lambda: op.eval_batched(_lib.OBJECTIVE, W, Tau, Mu, rho, out=outo), 5)
    units = 800 * 64
    cfg = LmConfig(max_iters=max_iters)
    lm_solve_batched(op, case.mus, case.W[0], None, rho, LmConfig(max_iters=2))  # workspace for all 64 mu
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = lm_solve_batched(op, case.mus, case.W[0], None, rho, cfg)
    dt = time.perf_counter() - t0
    F = bench.flops_per_element(12, 6, 4, 4, 3, 6, 20, 10)
    return {"config": "cfg3 half cylinder 40k tri, k=20/10, 800 active (2%), 64 mu",
            "derivs_pass_ms": t_d * 1e3, "derivs_units_per_s": units / t_d, "derivs_tflops_model": F * units / t_d / 1e12,
            "objective_pass_ms": t_o * 1e3, "objective_units_per_s": units / t_o,
            "gn_solves_per_s": len(res) / dt, "lm_batch_wall_s": dt, "lm_max_iters": max_iters, **lm_stats(res)}


def cfg4(S):
    case = configs.sector_rom_case(320, 625, 20, 10, 0.02, 50.0, 1, seed=4, name="cfg4")
    op = op_of(case)
    ne, nu_g = case.mesh.num_elements, case.maps.n_global_state
    g = torch.Generator(device="cuda").manual_seed(4)
    mus = torch.rand(S, 1, generator=g, device="cuda", dtype=torch.float64) * 2.0 + 2.0
    gam = 1.4
    ff = torch.stack([torch.ones_like(mus[:, 0]), mus[:, 0], torch.zeros_like(mus[:, 0]),
                      (1.0 / gam) / (gam - 1.0) + 0.5 * mus[:, 0] ** 2], 1)  # (S, 4)
    U = (1.0 + 0.1 * (torch.rand(S, ne * 6, 4, generator=g, device="cuda", dtype=torch.float64) - 0.5)) * ff[:, None, :]
    U = U.reshape(S, nu_g)
    nodes = torch.as_tensor(case.mesh.nodes).cuda()
    X = nodes.reshape(1, -1).repeat(S, 1)
    h = 1.0 / 320
    for _ in range(4):
        k = torch.randint(1, 5, (S, 2), generator=g, device="cuda").double()
        ph = torch.rand(S, 1, generator=g, device="cuda", dtype=torch.float64) * 2 * np.pi
        th = torch.rand(S, 1, generator=g, device="cuda", dtype=torch.float64) * 2 * np.pi
        sv = torch.sin(2 * np.pi * (k[:, :1] * nodes[None, :, 0] + k[:, 1:] * nodes[None, :, 1]) + ph)
        X[:, 0::2] += 0.05 * h * torch.cos(th) * sv
        X[:, 1::2] += 0.05 * h * torch.sin(th) * sv
    K = 30
    out = torch.empty(S * (K + 1) * ne, dtype=torch.float64, device="cuda")
    mus_np = mus.cpu().numpy()
    t = cuda_time(lambda: op.contributions_at_snapshots(U, X, mus_np, "lprows", out=out), 3)
    return {"config": f"cfg4 EQP constraint matrix, 400k tri, {S} snapshots, (K+1)=31 rows each",
            "matrix_shape": [S * (K + 1), ne], "matrix_gb": S * (K + 1) * ne * 8 / 1e9, "pass_ms": t * 1e3,
            "element_snapshots_per_s": S * ne / t}


def cfg5(P, max_iters):
    case = configs.cfg5_rom(P)
    op = op_of(case)
    rho = WeightVector(case.rho)
    from paper_2305_15661_b200.greedy import indicators, local_argmax

    cfg = LmConfig(max_iters=max_iters)
    lm_solve_batched(op, case.mus, case.W[0], None, rho, LmConfig(max_iters=1))  # workspace for all P
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = lm_solve_batched(op, case.mus, case.W[0], None, rho, cfg)
    t_lm = time.perf_counter() - t0
    W = np.stack([r.w for r in res])
    Tau = np.stack([r.tau for r in res])
    indicators(op, case.mus[:8], W[:8], Tau[:8])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ind = indicators(op, case.mus, W, Tau)
    t_ind = time.perf_counter() - t0
    v, i = local_argmax(np.where([np.isfinite(r.objective) for r in res], ind, np.inf), np.arange(P))
    ne = case.mesh.num_elements
    return {"config": f"cfg5 greedy sweep, 160k tri, {P} candidates, k=24/12, 4800 active (3%)",
            "rom_solves_per_s": P / t_lm, "lm_wall_s": t_lm, "lm_max_iters": max_iters, **lm_stats(res),
            "indicator_wall_s": t_ind, "indicator_element_evals_per_s": ne * P / t_ind, "argmax": [float(v), int(i)]}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="1,3,4,5")
    ap.add_argument("--cfg3-iters", type=int, default=30)
    ap.add_argument("--cfg4-snapshots", type=int, default=64)
    ap.add_argument("--cfg5-candidates", type=int, default=1024)
    ap.add_argument("--cfg5-iters", type=int, default=10)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    results = {}
    for c in a.only.split(","):
        t0 = time.perf_counter()
        if c == "1":
            r = cfg1()
        elif c == "3":
            r = cfg3(a.cfg3_iters)
        elif c == "4":
            r = cfg4(a.cfg4_snapshots)
        elif c == "5":
            r = cfg5(a.cfg5_candidates, a.cfg5_iters)
        r["total_wall_s"] = time.perf_counter() - t0
        results[f"cfg{c}"] = r
        print(json.dumps({f"cfg{c}": r}), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(results, fh, indent=1)
