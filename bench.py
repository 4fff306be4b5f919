#!/usr/bin/env python
"""Benchmark: element residual + Jacobian + projection evals/s (fp64), config 2.

Workload (BASELINE.json configs[1]): 2-D Euler, DG p=2, 12/4-point rules,
unit square 2x256x256 = 131,072 triangles, explicit perturbed freestream
state and sinusoidally displaced mesh, Phi (N_u x 16), Psi (N_x x 8)
seeded orthonormal; one step = one full reduced derivatives pass
(R_e, J_e = [dR/dU Phi | dR/dx Psi], Gram/gradient/objective reduced over
all elements, rho = 1) — ``ReducedOperator.derivatives`` (strom/reduced.py:
209-229).

The same JSON line carries "gn": the second half of BASELINE.json's metric,
ROM Gauss-Newton solves/s on config 3 (40k-triangle half-cylinder sector with
a slip wall, k_u=20, k_x=10, 800 EQP elements, 64 mu per batch, LM
max_iters=30), and "cfg4" / "cfg5": the sharded training configs (EQP LP rows
of 64 snapshots over 400k triangles; one 1,024-candidate greedy step).  The
timed config-2 step is replayed as one CUDA graph (``--no-graph``: eager).

Arms:
  default            this repo's CUDA path; ``value`` = elements/s with inputs
                     resident in HBM (Phi alone is 403 MB > 126 MB L2, so no
                     L2 flush is needed); ``e2e`` = the same metric through
                     GpuReducedOperator.derivatives with host numpy inputs
                     (H2D of w, tau, mu and D2H of J,S,T,H inside the timed
                     region).  ``cpu_baseline`` (rank 0, N=1): the arm below on a
                     bounded sample.
  --impl reference   the reference's CPU path on all host cores: the UNMODIFIED
                     strom installed in baseline/_ref (oracle/strom_ref.py),
                     ``ReducedOperator.derivatives`` on a bounded sample of
                     config-2-generator elements per process, and stock
                     ``lm_solve`` on config-3 mu for "gn"; the oracle port
                     (oracle/) only if the install is missing.
Multi-GPU (torchrun): config 2's elements are split into contiguous ranges,
each rank reduces its range and the 1+K+K^2 sums are all-reduced over NCCL
(strong scaling; max-over-ranks device time); config 3 runs one 64-mu batch per
rank (weak); configs 4 / 5 shard snapshots / candidates (sharded.py, greedy.py).
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

METRIC = "element residual+Jacobian+projection evals/sec (fp64)"  # first half of BASELINE.json's metric; GN solves/s in "gn"
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


def fp64_peak(gpu=0):
    """FP64 roofline denominator: the DFMA / DMMA issue-bound loops of tools/fp64_peak.cu run
    on this GPU in this run (clocks sampled while they run), else the round-1 measurement."""
    tool = os.path.join(ROOT, "tools", "fp64_peak")
    if os.path.exists(tool):
        clk = Clocks(gpu)
        try:
            out = subprocess.run([tool], capture_output=True, text=True, timeout=120).stdout
            d = json.loads(out.strip().splitlines()[-1])
        except (OSError, ValueError, IndexError, subprocess.SubprocessError):
            d = None
        c = clk.stop()
        if d and d.get("err") == "no error":
            dfma = max(v for k, v in d.items() if k.startswith("dfma_tflops"))
            dmma = max(v for k, v in d.items() if k.startswith("dmma_tflops"))
            return max(dfma, dmma), (f"measured in this run by tools/fp64_peak.cu: DFMA {dfma:.2f}, DMMA {dmma:.2f} "
                                     f"TFLOP/s at {c.get('sm_mhz')} MHz (reasons {c.get('reasons')})")
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


def _cpu_init(n, seed, kind):
    """Pool initializer: build a cfg2-shaped problem once per process (stock reference or port)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from paper_2305_15661_b200 import configs

    case = configs.euler_square_case(n=n, seed=seed)
    if kind == "reference":
        from oracle import strom_ref

        op = strom_ref.operator(case)
        c = strom_ref.coords(case.W[0], case.Tau[0])
        call = lambda: op.derivatives(c, case.mus[0])  # noqa: E731  (reduced.py:209-229, stock)
    else:
        import oracle.dual  # noqa: F401
        from oracle.element import OracleGeometry, OracleReducedOperator

        geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
        op = OracleReducedOperator(case.law, geom, case.phi, case.psi, case.ref_coords, case.kappa, case.eps,
                                   state_offset=case.state_offset)
        call = lambda: op.derivatives(case.W[0], case.Tau[0], case.mus[0], None)  # noqa: E731
    call()  # warm caches (element slices, geometry tables, einsum paths)
    _WORKER.update(case=case, call=call)


def _cpu_step(_):
    case, call = _WORKER["case"], _WORKER["call"]
    t0 = time.perf_counter()
    call()
    return case.mesh.num_elements, time.perf_counter() - t0


def cpu_kind():
    """"reference" when the unmodified strom is importable (baseline/_ref), else "port"."""
    from oracle import strom_ref

    return "reference" if strom_ref.locate() else "port"


class CpuArm:
    """The reference's CPU derivatives path on all host cores.

    kind "reference": the unmodified ``strom`` installed in baseline/_ref,
    ``ReducedOperator.derivatives`` on its own dual numbers (oracle/strom_ref.py
    lists the plugin-level additions: Euler law spec, 12-point rule, state
    offset); kind "port": the oracle restatement (oracle/), used only when the
    install is missing.  Each process owns a 2 n^2-element config-2-shaped mesh
    (same p, rules, k_u, k_x, law, generator -> same per-element work as
    config 2); one step = one derivatives pass in every process.
    """

    def __init__(self, cores=None, n=16, kind=None):
        import multiprocessing as mp

        self.cores = cores or os.cpu_count() or 1
        self.n = n
        self.kind = kind or cpu_kind()
        self.pool = mp.get_context("spawn").Pool(self.cores, initializer=_cpu_init, initargs=(n, 100, self.kind))

    def step(self):
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_step, range(self.cores), chunksize=1)
        return sum(r[0] for r in res), time.perf_counter() - t0, res

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, steps):
        what = "stock strom ReducedOperator.derivatives" if self.kind == "reference" else "oracle port of strom's derivatives"
        return (f"{what}: {self.cores} processes x {steps} pass(es) over {2 * self.n * self.n} cfg2-generator elements "
                f"each (Euler p=2, 12/4 rules, k_u=16, k_x=8, W=Tau=0)")


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
    return {"value": elems / wall, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
            "sample": arm.describe(steps) + f"; {elems} element evals in {wall:.1f}s wall"}


# -- ROM Gauss-Newton solves (config 3), the second half of the BASELINE metric ----------------
GN_METRIC = "ROM Gauss-Newton solves/sec (fp64)"
GN_UNIT = "solves/s"
GN_ITERS = 30


def _gn_init(kind):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from paper_2305_15661_b200 import configs

    # the reference has no slip wall (conslaw.py:20-29): its arm runs the same mesh, bases, sample
    # and solver with the cylinder wall extrapolated (identical work per element and face)
    case = configs.cfg3(wall="extrapolate")
    if kind == "reference":
        from oracle import strom_ref

        op = strom_ref.operator(case)
        solve = lambda mu: strom_ref.lm_solve(op, mu, case.rho, case.W[0], GN_ITERS)  # noqa: E731 (lm.py:164, stock)
        op.objective(strom_ref.coords(case.W[0], case.Tau[0]), case.mus[0], strom_ref.weights(case.rho))  # slices
    else:
        import oracle.dual  # noqa: F401
        from oracle import lm as olm
        from oracle.element import OracleGeometry, OracleReducedOperator

        op = OracleReducedOperator(case.law, OracleGeometry(case.mesh, case.maps, case.quad_order), case.phi,
                                   case.psi, case.ref_coords, case.kappa, case.eps)
        solve = lambda mu: olm.lm_solve(olm.OracleProblem(op, mu, case.rho, case.W[0]), olm.LmConfig(max_iters=GN_ITERS))  # noqa: E731
    _WORKER.update(gn_case=case, gn_solve=solve)


def _gn_step(i):
    case, solve = _WORKER["gn_case"], _WORKER["gn_solve"]
    t0 = time.perf_counter()
    r = solve(case.mus[i])
    return time.perf_counter() - t0, int(r.n_iters), str(r.reason)


def gn_cpu_baseline(max_procs=16):
    """Stock ``strom.lm.lm_solve`` (max_iters=30) on the first min(cores, 16) config-3 mu, one
    full solve per process, all in parallel: solves / wall seconds."""
    import multiprocessing as mp

    kind = cpu_kind()
    n = max(1, min(os.cpu_count() or 1, max_procs))
    pool = mp.get_context("spawn").Pool(n, initializer=_gn_init, initargs=(kind,))
    try:
        pool.map(time.sleep, [0.0] * n, chunksize=1)  # initializers done
        t0 = time.perf_counter()
        res = pool.map(_gn_step, range(n), chunksize=1)
        wall = time.perf_counter() - t0
    finally:
        pool.close()
        pool.join()
    it = [r[1] for r in res]
    what = "stock strom lm_solve" if kind == "reference" else "oracle port of strom lm_solve"
    return {"value": n / wall, "unit": GN_UNIT, "cores": n, "kind": kind,
            "sample": f"{what}: {n} of the 64 config-3 mu (cylinder wall extrapolated: the reference has no slip wall), "
                      f"one full solve (max_iters={GN_ITERS}, w0 lsq) per process, "
                      f"{wall:.1f}s wall; iterations mean {np.mean(it):.1f}; per-solve {np.mean([r[0] for r in res]):.1f}s"}


# ---------------------------------------------------------------------------------
def cfg2_config(n, ku, kx, world):
    return {"workload": "cfg2: Euler p=2, 12/4-point rules, 2x%dx%d triangles, k_u=%d, k_x=%d, rho=1, one derivatives pass per step" % (n, n, ku, kx),
            "elements": 2 * n * n, "n_u": 24, "K": ku + kx,
            "state": "freestream x (1+U(-0.05,0.05)) per DG node and component (no LLF wavespeed ties; DESIGN.md §6)",
            "l2": "inputs larger than L2 (Phi %.0f MB)" % (2 * n * n * 24 * ku * 8 / 1e6),
            "parallelism": f"element-range x{world}" + (" + NCCL all_reduce of 1+K+K^2 sums" if world > 1 else "")}


def gn_config(world):
    return {"workload": "cfg3: half-cylinder sector 100x200 quads = 40,000 triangles, Euler p=2, k_u=20, k_x=10, "
                        "800 EQP elements (2%%), 64 mu ~ U[2,4] per batch, LM max_iters=%d, w0 = Phi^T U_ff(3) + lsq state init" % GN_ITERS,
            "parallelism": f"mu batches x{world} (each rank its own 64-mu batch, no collective)"}


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
    cfg = cfg2_config(args.n, 16, 8, 1)
    cfg["sample_elements_per_step"] = elems // args.steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "impl": "reference", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
                             "sample": arm.describe(args.steps)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_gn:
        g = gn_cpu_baseline()
        line["gn"] = {"metric": GN_METRIC, "value": g["value"], "unit": GN_UNIT, "higher_is_better": True,
                      "config": gn_config(1), "cpu_baseline": g,
                      "e2e": {"value": g["value"], "unit": GN_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_gn(args, dev, world, rank, local):
    """Config 3: batched ROM Gauss-Newton (LM) solves of 64 mu per step on this rank.

    value: device-resident (strom_lm_solve on device buffers; W reset from w0 inside the
    timed region), CUDA events on the launching stream, max over ranks; e2e: the public
    ``lm_solve_batched`` with host numpy mu / w0 in and LmResult objects out, wall clock."""
    import torch
    import torch.distributed as dist

    from paper_2305_15661_b200 import configs
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.lm import REASONS, LmConfig, lm_solve_batched, lm_solve_device
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

    case = configs.cfg3()
    mus = case.mus if rank == 0 else np.random.default_rng(1000 + rank).uniform(2.0, 4.0, size=case.mus.shape)
    op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist, device=dev)
    rho = WeightVector(case.rho)
    cfg = LmConfig(max_iters=GN_ITERS)
    P, ku, kx = len(mus), op.k_u, op.k_x
    Mu = torch.as_tensor(mus, dtype=torch.float64).to(dev)
    W0 = torch.as_tensor(np.tile(case.W[0], (P, 1))).to(dev)
    W = torch.empty_like(W0)
    Tau = torch.zeros((P, kx), dtype=torch.float64, device=dev)
    status = torch.zeros((P, 8), dtype=torch.float64, device=dev)

    def step():
        W.copy_(W0)
        Tau.zero_()
        lm_solve_device(op, W, Tau, Mu, rho, cfg, status)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    steps = max(3, args.gn_steps)
    clk = Clocks(local)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    stat = status.cpu().numpy()
    lm_stats = _lm_stats(op)
    # e2e through the public API (host numpy in, LmResult out)
    lm_solve_batched(op, mus, case.W[0], None, rho, cfg, want_history=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        res = lm_solve_batched(op, mus, case.W[0], None, rho, cfg, want_history=False)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([ms, e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1])
    reasons = {}
    for r in stat[:, 5]:
        reasons[REASONS[int(r)]] = reasons.get(REASONS[int(r)], 0) + 1
    assert all(np.isfinite(r.objective) for r in res)
    return {"metric": GN_METRIC, "value": world * P * steps / (ms / 1e3), "unit": GN_UNIT, "higher_is_better": True,
            "steps": steps, "warmup": args.warmup, "ms_per_step": ms / steps, "solves_per_step": world * P,
            "config": gn_config(world), "scaling": "weak",
            "iterations": {"mean": float(stat[:, 4].mean()), "max": int(stat[:, 4].max()), "reasons": reasons},
            "lm_graph_last_batch": lm_stats, "clocks": clocks,
            "e2e": {"value": world * P * steps / e2e_s, "unit": GN_UNIT, "h2d_bytes_per_step": 8 * P * (1 + ku + kx),
                    "d2h_bytes_per_step": 8 * P * (ku + kx + 8)}}


def _sync_max(world, dev, *vals):
    """Max over ranks of host-side numbers (timing)."""
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return tuple(float(v) for v in t)


def run_cfg4(args, dev, world, rank, local):
    """Config 4: EQP constraint rows of 64 training snapshots over the 400k-triangle sector,
    snapshots sharded over the ranks (s mod G = r, no collective in the compute; the row
    blocks are gathered to rank 0 for the LP afterwards, timed separately)."""
    import torch
    import torch.distributed as dist

    from paper_2305_15661_b200 import configs, sharded
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

    S = 64
    case = configs.cfg4_case()
    op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist, device=dev)
    ne, K = case.mesh.num_elements, op.k_u + op.k_x
    ids = sharded.snapshot_ids(S, rank, world)
    mus, U, X = sharded.snapshot_fields_device(case, ids, 4, dev)
    out = torch.empty(len(ids) * (K + 1) * ne, dtype=torch.float64, device=dev)

    def step():
        if len(ids):
            op.contributions_at_snapshots(U, X, mus, "lprows", out=out)

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    steps = max(1, args.cfg_steps)
    clk = Clocks(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    e0.record(st)
    for _ in range(steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / steps
    t0 = time.perf_counter()
    full = sharded.gather_rows(out.view(len(ids), K + 1, ne), S, rank, world)
    torch.cuda.synchronize()
    gather_ms = 1e3 * (time.perf_counter() - t0)
    ms, gather_ms = _sync_max(world, dev, ms, gather_ms)
    ok = bool(torch.isfinite(full).all()) if full is not None else True
    return {"metric": "EQP constraint-row element-snapshot evals/sec (fp64)", "value": S * ne / (ms / 1e3),
            "unit": "element-snapshots/s", "higher_is_better": True, "scaling": "strong", "ms_per_step": ms,
            "steps": steps, "gather_to_rank0_ms": gather_ms if world > 1 else 0.0, "finite": ok,
            "config": {"workload": "cfg4: 400,000-triangle sector, 64 snapshots x (k_u+k_x+1) = 31 rows, k_u=20, k_x=10",
                       "matrix": [S * (K + 1), ne], "parallelism": f"snapshots s mod {world} per rank, no compute collective"},
            "clocks": clocks}


def run_cfg5(args, dev, world, rank, local, group=None):
    """Config 5: one greedy search step over 1024 candidates (batched ROM LM solves, k_u=24,
    k_x=12, 3% EQP elements, then full-mesh residual-norm indicators and the argmax),
    candidates interleaved over the ranks, one all-gather of (indicator, index) winners."""
    import torch
    import torch.distributed as dist

    from paper_2305_15661_b200 import configs
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.greedy import greedy_step
    from paper_2305_15661_b200.lm import LmConfig
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

    case = configs.cfg5_rom(1024)
    op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist, device=dev)
    rho = WeightVector(case.rho)
    cfg = LmConfig(max_iters=10)

    st = {}

    def step():
        return greedy_step(op, case.mus, [], rho, case.W[0], None, cfg, rank, world, group, stats=st)

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    steps = max(1, args.cfg_steps)
    clk = Clocks(local)
    t0 = time.perf_counter()
    for _ in range(steps):
        v, i = step()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps
    clocks = clk.stop()
    (wall,) = _sync_max(world, dev, wall)
    return {"metric": "greedy candidate evaluations/sec (ROM LM solve + full-mesh indicator, fp64)",
            "value": len(case.mus) / wall, "unit": "candidates/s", "higher_is_better": True, "scaling": "strong",
            "ms_per_step": 1e3 * wall, "steps": steps, "argmax": [float(v), int(i)],
            "rank0_failed_candidates": st.get("failed"), "rank0_candidates": st.get("candidates"),
            "failed_note": "a candidate fails (+inf, SPEC.md:492) when its reconstructed full mesh inverts an element "
                           "(reference: DegenerateMappingError); with untrained seeded bases most do",
            "config": {"workload": "cfg5: 160,000-triangle sector, 1024 candidate mu ~ U[2,4], k_u=24, k_x=12, "
                                   "4,800 EQP elements (3%), LM max_iters=10, indicator ||R||_2 on the full mesh",
                       "parallelism": f"candidates interleaved over {world} rank(s) + all_gather argmax",
                       "timing": "wall clock of the public greedy_step (host in / out), max over ranks"},
            "clocks": clocks}


def _fullspace_case(n_radial, n_circ, seed=6):
    from paper_2305_15661_b200 import configs, laws as L

    case = configs.sector_rom_case(n_radial, n_circ, 2, 1, 0.5, 2.0, 1, seed=seed, name="fullspace", wall="extrapolate")
    rng = np.random.default_rng(seed)
    ne = case.mesh.num_elements
    U = np.tile(L.euler_freestream(3.0), ne * 6) * (1.0 + 0.03 * rng.standard_normal(ne * 24))
    return case, U, case.ref_coords.copy(), np.array([3.0])


def _fullspace_cpu(_):
    """Stock reference assemble_enriched (dg.py:275-326) on a 400-triangle sector: elements/s."""
    from oracle import strom_ref

    strom_ref.load()
    import strom.dg as sdg

    case, U, x, mu = _fullspace_case(10, 20)
    rop = strom_ref.operator(case)
    t0 = time.perf_counter()
    sdg.assemble_enriched(case.law, rop.geom.mesh, rop.geom.maps, U, x, mu)
    return case.mesh.num_elements / (time.perf_counter() - t0)


def run_fullspace(args, dev, local):
    """SURVEY §8f-3 measurement: one enriched full-space assembly (dg.py:275-326: residual against
    the degree-3 test space with dR/dU, dR/dx blocks, N_e and dN_e/dx) of a 4,000-triangle
    sector. Device time of the K1 pass (CUDA events), e2e of the public assemble_enriched (host
    state in, scipy CSR out: H2D of U and x, D2H of the records, host scatter)."""
    import torch

    from paper_2305_15661_b200 import _lib, fullspace
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

    case, U, x, mu = _fullspace_case(25, 80)
    ne = case.mesh.num_elements
    geom = case.geom
    op = GpuReducedOperator(case.law, geom, ReducedBases(np.zeros((U.size, 0)), np.zeros((x.size, 0)), x),
                            fullspace._NoDistortion(), device=dev, state_offset=U)
    phi_t, dphi_t, trace_t = fullspace.test_space_tables(op.dm.tabs, 3)
    _lib.check(op._lib.strom_set_test_space(op._h, 10, phi_t.ctypes.data, dphi_t.ctypes.data, trace_t.ctypes.data),
               "strom_set_test_space")
    rec = 40 * (1 + 4 * 24 + 6) + 7
    out = torch.empty(ne * rec, dtype=torch.float64, device=dev)
    W = torch.zeros((1, 1), dtype=torch.float64, device=dev)
    Mu = torch.as_tensor(mu[None]).to(dev)
    for _ in range(3):
        op.eval_batched(_lib.ELEMJAC_ENRICHED, W, W, Mu, None, out=out)
    torch.cuda.synchronize()
    steps = 10
    clk = Clocks(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    e0.record(st)
    for _ in range(steps):
        op.eval_batched(_lib.ELEMJAC_ENRICHED, W, W, Mu, None, out=out)
    e1.record(st)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / steps
    fullspace.assemble_enriched(case.law, case.mesh, case.maps, U, x, mu, geom=geom, device=dev)
    t0 = time.perf_counter()
    for _ in range(3):
        Rb, JU, JX = fullspace.assemble_enriched(case.law, case.mesh, case.maps, U, x, mu, geom=geom, device=dev)
    e2e_s = (time.perf_counter() - t0) / 3
    wbytes = ne * rec * 8.0
    rbytes = ne * (24 * 8.0 * 4 + 64)  # own + neighbor state rows, indices, coordinates (approx.)
    peak = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        peak = 6500.0
    res = {"metric": "full-space enriched element Jacobian evals/sec (fp64)", "value": ne / (ms / 1e3),
           "unit": "elements/s", "higher_is_better": True, "ms_per_step": ms, "steps": steps,
           "config": {"workload": "4,000-triangle half-cylinder sector, Euler p=2, degree-3 test space (40 rows/element), "
                                  "one STROM_ELEMJAC_ENRICHED pass: 4,127 doubles written per element"},
           "roofline": {"bound": "hbm", "achieved": (wbytes + rbytes) / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": (wbytes + rbytes) / (ms / 1e3) / 1e9 / peak, "traffic": None,
                        "bytes_per_launch": wbytes + rbytes,
                        "note": "one warp per element, plain per-lane contraction loops: an offline path, far from the HBM bound"},
           "e2e": {"value": ne / e2e_s, "unit": "elements/s", "h2d_bytes_per_step": 8 * (U.size + x.size),
                   "d2h_bytes_per_step": 8 * (int(JU.nnz) + int(JX.nnz) + ne * 47), "csr_nnz": [int(JU.nnz), int(JX.nnz)],
                   "note": "assemble_enriched on a warm operator: H2D of U and x, K1 pass, device gather of the CSR values "
                           "on the cached pattern, D2H of the nnz values, residual rows and distortion columns"},
           "clocks": clocks}
    if not args.no_cpu_baseline:
        try:
            import concurrent.futures as cf

            n = min(16, os.cpu_count() or 1)
            with cf.ProcessPoolExecutor(max_workers=n) as ex:
                t0 = time.perf_counter()
                rates = list(ex.map(_fullspace_cpu, range(n)))
                wall = time.perf_counter() - t0
            res["cpu_baseline"] = {"value": n * 400 / wall, "unit": "elements/s", "cores": n, "kind": "reference",
                                   "sample": f"stock strom.dg.assemble_enriched on a 400-triangle sector per process x {n} "
                                             f"processes (wall incl. geometry set-up); per-process rate {np.mean(rates):.0f} el/s"}
        except Exception as exc:  # the reference is test infrastructure: absent -> no baseline
            res["cpu_baseline"] = {"unavailable": str(exc)[:200]}
    return res


def _lm_stats(op):
    """(control rounds, derivative passes, objective passes) of the op's last batched solve."""
    import ctypes

    from paper_2305_15661_b200 import _lib

    out = (ctypes.c_int32 * 3)()
    _lib.check(_lib.load().strom_lm_stats(op._h, out), "strom_lm_stats")
    return {"rounds": out[0], "derivative_passes": out[1], "objective_passes": out[2]}


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
    # the step (counter memsets, K1, finalize, and the NCCL all-reduce for N > 1) captured once
    # as a CUDA graph and replayed: no per-kernel launch gaps (eager with --no-graph or when the
    # capture is not possible, e.g. the gloo functional runs)
    graph, graph_note = None, "eager launches"
    if not args.no_graph and (world == 1 or dist.get_backend() == "nccl"):
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
            torch.cuda.synchronize()
            graph_note = "one CUDA graph per step (memsets, K1, finalize" + (", NCCL all-reduce)" if world > 1 else ")")
        except Exception as exc:  # noqa: BLE001
            graph, graph_note = None, f"eager launches (graph capture failed: {type(exc).__name__})"
    run = graph.replay if graph is not None else step
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = Clocks(local)
    lib = _lib.load()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(args.steps):
        run()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clocks = clk.stop()
    # K1 kernel time: events around every K1 launch of the same number of eager steps
    lib.strom_profile(op._h, 1)
    for _ in range(args.steps):
        op.eval_batched(_lib.DERIVS, W, Tau, Mu, rho, out=out, degen=degen)
    nl = _lib.C.c_int32()
    kern_ms = lib.strom_profile_ms(op._h, _lib.C.byref(nl))
    lib.strom_profile(op._h, 0)
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
        e2e_io = (8 * (ku + kx + op.n_mu), 8 * (1 + K + K * K) + 8)  # inputs; outputs + degenerate counter slot
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
    gn = None if args.no_gn else run_gn(args, dev, world, rank, local)
    fs = None
    if rank == 0 and world == 1 and not args.no_fullspace:
        fs = run_fullspace(args, dev, local)
    cfg4 = cfg5 = None
    if not args.no_sharded:
        cfg4 = run_cfg4(args, dev, world, rank, local)
        torch.cuda.empty_cache()
        cfg5 = run_cfg5(args, dev, world, rank, local)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    nu, nq, ns = 24, 12, 4
    F = flops_per_element(nq, 6, 4, ns, 3, 6, ku, kx)
    per_launch_flops = F * (hi - lo)
    kern_avg_s = kern_ms / max(1, nl.value) / 1e3
    peak, peak_src = fp64_peak(local)
    achieved = per_launch_flops / kern_avg_s / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "derivs_traffic_r02.json")
    if os.path.exists(tp) and n == 256:  # the ncu capture is of the full config-2 pass
        with open(tp) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch") * (hi - lo) / ne
    value = ne * args.steps / (ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded: perturbed freestream state, sinusoidal mesh displacement, Gaussian-QR bases)",
        "config": cfg2_config(n, ku, kx, world),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "derivs_mma_kernel<Euler,12,16,8>",
                     "flops_per_element": F, "flops_per_launch": per_launch_flops,
                     "kernel_ms_avg": kern_avg_s * 1e3, "peak_source": peak_src,
                     "hbm_bytes_per_launch": bytes_per_pass(ne, case.mesh.num_nodes, nu, ku, kx) * (hi - lo) / ne},
        "gpu_launches": 2 * args.steps, "step_launch": graph_note,
        "clocks": clocks,
    }
    if e2e_value is not None:
        line["e2e"] = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": e2e_io[0], "d2h_bytes_per_step": e2e_io[1]}
    if gn is not None:
        line["gn"] = gn
    if cfg4 is not None:
        line["cfg4"], line["cfg5"] = cfg4, cfg5
    if fs is not None:
        line["fullspace"] = fs
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(n=args.cpu_n)
        if gn is not None:
            gn["cpu_baseline"] = gn_cpu_baseline()
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
    ap.add_argument("--no-gn", action="store_true", help="skip the config-3 Gauss-Newton solves/s measurement")
    ap.add_argument("--gn-steps", type=int, default=20, help="timed 64-mu LM batches of the GN measurement")
    ap.add_argument("--no-sharded", action="store_true", help="skip the config-4 / config-5 sharded measurements")
    ap.add_argument("--no-fullspace", action="store_true", help="skip the full-space enriched assembly measurement")
    ap.add_argument("--no-graph", action="store_true", help="time the config-2 step with eager launches")
    ap.add_argument("--cfg-steps", type=int, default=3, help="timed steps of the config-4 / config-5 measurements")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
