#!/usr/bin/env python
"""Benchmark: element residual + Jacobian + projection evals/s (fp64), config 2.

Workload (BASELINE.json configs[1]): 2-D Euler, DG p=2, 12/4-point rules,
unit square 2x256x256 = 131,072 triangles, explicit perturbed freestream
state and sinusoidally displaced mesh, Phi (N_u x 16), Psi (N_x x 8)
seeded orthonormal; one step = one full reduced derivatives pass
(R_e, J_e = [dR/dU Phi | dR/dx Psi], Gram/gradient/objective reduced over
all elements, rho = 1) — ``ReducedOperator.derivatives`` (strom/reduced.py:
209-229).

Arms:
  default            this repo's CUDA path; ``value`` = elements/s with inputs
                     resident in HBM (Phi alone is 403 MB > 126 MB L2, so no
                     L2 flush is needed); ``e2e`` = the same metric through
                     GpuReducedOperator.derivatives with host numpy inputs
                     (H2D of w, tau, mu and D2H of J,S,T,H inside the timed
                     region).
  --impl reference   the reference algorithm on the host CPU: the oracle port
                     (numpy restatement of strom's dual-number path,
                     oracle/) on a bounded sample of config-2 elements, one
                     process per host core.
Multi-GPU (torchrun): elements are split into contiguous ranges, each rank
reduces its range and the 1+K+K^2 sums are all-reduced over NCCL
(strong scaling; max-over-ranks device time).
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "element residual+Jacobian+projection evals/sec (fp64)"
UNIT = "elements/s"
FP64_PEAK_TFLOPS = None  # filled from profiles/fp64_peak_r01.json


def flops_per_element(nq, nb, m, ns, nf, nx, ku, kx, d=2):
    """SURVEY §8(d) algorithmic flop model F1 (FMA = 2) per element per mu."""
    nu, K = nb * m, ku + kx
    return (2 * nq * (nb * m * m * d + nb * nb * m * m) + 2 * nq * nb * m * nx * (d + 1)
            + 3 * ns * 4 * nf * nf * m * m + 3 * ns * 2 * nf * m * nx
            + 2 * nu * (nu * ku + 3 * nf * m * ku + nx * kx)
            + nu * K * (K + 1) + 2 * nu * K + 2 * nu
            + (2 * nq * nb * m + 2 * nq * m * d * d + 2 * nq * nb * m * (d + 1) + 3 * ns * 6 * nf * m)
            + 2 * nx * kx + kx * (kx + 1))


def bytes_per_pass(ne, nv, nu, ku, kx):
    """Compulsory HBM bytes of one derivatives pass (SURVEY §8(d) B_alg)."""
    Nu, Nx = ne * nu, 2 * nv
    return 8 * (Nu * ku + Nu + Nx * kx + 2 * Nx + ne) + ne * 3 * (4 + 4 + 1)


def fp64_peak():
    path = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
    with open(path) as fh:
        d = json.load(fh)
    return max(d["dfma_tflops_t1024"], d["dfma_tflops_t512"]), "measured DFMA loop (tools/fp64_peak.cu, profiles/fp64_peak_r01.json)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------
_WORKER = {}


def _cpu_init(n, seed):
    """Pool initializer: build a cfg2-shaped oracle problem once per process."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import oracle.dual  # noqa: F401
    from oracle.element import OracleGeometry, OracleReducedOperator
    from paper_2305_15661_b200 import configs

    case = configs.euler_square_case(n=n, seed=seed)
    geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
    op = OracleReducedOperator(case.law, geom, case.phi, case.psi, case.ref_coords, case.kappa, case.eps,
                               state_offset=case.state_offset)
    op.derivatives(case.W[0], case.Tau[0], case.mus[0], None)  # warm caches (eta_ref, einsum paths)
    _WORKER.update(case=case, op=op)


def _cpu_step(_):
    case, op = _WORKER["case"], _WORKER["op"]
    t0 = time.perf_counter()
    op.derivatives(case.W[0], case.Tau[0], case.mus[0], None)
    return case.mesh.num_elements, time.perf_counter() - t0


class CpuArm:
    """Oracle port (numpy restatement of strom's dual-number derivatives) on all host cores.

    Each process owns a 2 n^2-element config-2-shaped mesh (same p, rules,
    k_u, k_x, law -> same per-element work as config 2); one step = one
    derivatives pass in every process.
    """

    def __init__(self, cores=None, n=16):
        import multiprocessing as mp

        self.cores = cores or os.cpu_count() or 1
        self.n = n
        self.pool = mp.get_context("spawn").Pool(self.cores, initializer=_cpu_init, initargs=(n, 100))

    def step(self):
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_step, range(self.cores), chunksize=1)
        return sum(r[0] for r in res), time.perf_counter() - t0, res

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, steps):
        return (f"{self.cores} processes x {steps} derivatives pass(es) over {2 * self.n * self.n} cfg2-shaped elements "
                f"each (Euler p=2, 12/4 rules, k_u=16, k_x=8)")


def cpu_baseline(n=16, steps=3):
    arm = CpuArm(n=n)
    try:
        arm.step()
        elems, wall = 0, 0.0
        for _ in range(steps):
            e, t, _ = arm.step()
            elems, wall = elems + e, wall + t
    finally:
        arm.close()
    return {"value": elems / wall, "unit": UNIT, "cores": arm.cores, "kind": "port",
            "sample": arm.describe(steps) + f"; {elems} element evals in {wall:.1f}s wall"}


# ---------------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    arm = CpuArm(n=args.cpu_n)
    try:
        for _ in range(args.warmup):
            arm.step()
        elems, wall = 0, 0.0
        for _ in range(args.steps):
            e, t, _ = arm.step()
            elems, wall = elems + e, wall + t
    finally:
        arm.close()
    value = elems / wall
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "impl": "reference",
            "config": {"workload": "cfg2: Euler p=2, 12/4-point rules, k_u=16, k_x=8 — bounded CPU sample of cfg2-shaped elements",
                       "sample_elements_per_step": elems // args.steps},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": arm.cores, "kind": "port",
                             "sample": arm.describe(args.steps)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_mine(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if os.environ.get("BENCH_ONE_DEVICE"):  # functional test of the N>1 code path on a 1-GPU box (gloo)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2305_15661_b200 import _lib, configs
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases, ReducedCoords
    from paper_2305_15661_b200.eqp import WeightVector

    n = args.n
    case = configs.euler_square_case(n=n)
    ne = case.mesh.num_elements
    bases = ReducedBases(case.phi, case.psi, case.ref_coords)
    op = GpuReducedOperator(case.law, case.geom, bases, case.dist, device=dev, state_offset=case.state_offset)
    ku, kx = bases.k_u, bases.k_x
    K = ku + kx
    # element range of this rank (contiguous, strong scaling); BENCH_SIM_WORLD=N runs rank 0's
    # share of an N-GPU job on one GPU (per-rank kernel time for scaling estimates; no collective)
    sim = int(os.environ.get("BENCH_SIM_WORLD", "0"))
    sw, sr = (sim, 0) if (sim > 1 and world == 1) else (world, rank)
    lo, hi = ne * sr // sw, ne * (sr + 1) // sw
    rho = None if sw == 1 else WeightVector(np.where((np.arange(ne) >= lo) & (np.arange(ne) < hi), 1.0, 0.0))
    W = torch.zeros((1, ku), dtype=torch.float64, device=dev)
    Tau = torch.zeros((1, kx), dtype=torch.float64, device=dev)
    Mu = torch.as_tensor(case.mus, dtype=torch.float64).to(dev)
    out = torch.empty(1 + K + K * K, dtype=torch.float64, device=dev)
    degen = torch.zeros(1, dtype=torch.int32, device=dev)

    def step():
        op.eval_batched(_lib.DERIVS, W, Tau, Mu, rho, out=out, degen=degen)
        if world > 1:
            dist.all_reduce(out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = Clocks(local)
    lib = _lib.load()
    lib.strom_profile(op._h, 1)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nl = _lib.C.c_int32()
    kern_ms = lib.strom_profile_ms(op._h, _lib.C.byref(nl))
    lib.strom_profile(op._h, 0)
    clocks = clk.stop()
    if world > 1:
        t = torch.tensor([ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms, kern_ms = float(t[0]), float(t[1])
    # sanity: the reduced sums are finite and identical across steps
    host = out.cpu().numpy()
    assert np.all(np.isfinite(host)), "non-finite reduced sums"

    # e2e through the public API with host buffers (H2D coords, D2H J,S,T,H)
    coords = ReducedCoords(np.zeros(ku), np.zeros(kx))
    e2e_value = None
    if world == 1:
        for _ in range(max(1, args.warmup)):
            op.derivatives(coords, case.mus[0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            op.derivatives(coords, case.mus[0])
        e2e_s = time.perf_counter() - t0
        e2e_value = ne * args.steps / e2e_s
        e2e_io = (8 * (ku + kx + op.n_mu), 8 * (1 + K + K * K) + 4)
    else:
        # each rank: the public derivatives call on its element range (host in, host out), then
        # the 1+K+K^2 sums all-reduced over NCCL and read back; wall time, max over ranks
        def e2e_step():
            J, S, T, Hww, Hwt, Htt = op.derivatives(coords, case.mus[0], rho)
            v = torch.as_tensor(np.concatenate([[J], S, T, Hww.ravel(), Hwt.ravel(), Htt.ravel()])).to(dev)
            dist.all_reduce(v)
            return v.cpu()

        for _ in range(max(1, args.warmup)):
            e2e_step()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_value = ne * args.steps / float(tt[0])
        n_out = 1 + ku + kx + ku * ku + ku * kx + kx * kx
        e2e_io = (8 * (ku + kx + op.n_mu) + 8 * n_out, 2 * 8 * n_out + 4)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    nu, nq, ns = 24, 12, 4
    F = flops_per_element(nq, 6, 4, ns, 3, 6, ku, kx)
    per_launch_flops = F * (hi - lo)
    kern_avg_s = kern_ms / max(1, nl.value) / 1e3
    peak, peak_src = fp64_peak()
    achieved = per_launch_flops / kern_avg_s / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "derivs_traffic_r01.json")
    if os.path.exists(tp) and n == 256:  # the ncu capture is of the full config-2 pass
        with open(tp) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch") * (hi - lo) / ne
    value = ne * args.steps / (ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded: perturbed freestream state, sinusoidal mesh displacement, Gaussian-QR bases)",
        "config": {"workload": "cfg2: Euler p=2, 12/4-point rules, 2x%dx%d triangles, k_u=%d, k_x=%d, rho=1, one derivatives pass per step" % (n, n, ku, kx),
                   "elements": ne, "n_u": nu, "K": K, "l2": "inputs larger than L2 (Phi %.0f MB)" % (case.phi.nbytes / 1e6),
                   "parallelism": f"element-range x{world}" + (" + NCCL all_reduce of 1+K+K^2 sums" if world > 1 else "")},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "derivs_mma_kernel<Euler,12,16,8>",
                     "flops_per_element": F, "flops_per_launch": per_launch_flops,
                     "kernel_ms_avg": kern_avg_s * 1e3, "peak_source": peak_src,
                     "hbm_bytes_per_launch": bytes_per_pass(ne, case.mesh.num_nodes, nu, ku, kx) * (hi - lo) / ne},
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
    }
    if e2e_value is not None:
        line["e2e"] = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": e2e_io[0], "d2h_bytes_per_step": e2e_io[1]}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(n=args.cpu_n)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--cells", "--n", dest="n", type=int, default=256, help="cells per side of the unit square (cfg2: 256)")
    ap.add_argument("--cpu-n", type=int, default=16, help="CPU-baseline sample: cells per side per process")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
