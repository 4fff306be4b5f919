"""The sharded config-4 / config-5 paths with two ranks on one device (gloo host
collectives, each rank's kernels independent of the other's) reproduce the single-rank
results bit for bit: snapshot-sharded LP rows gathered in snapshot order, and the
candidate-sharded greedy step's (indicator, argmax)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def small_case():
    from paper_2305_15661_b200 import configs

    return configs.sector_rom_case(n_radial=4, n_circ=8, ku=6, kx=4, frac_active=0.25, rho_scale=4.0, P=5, seed=61)


def gpu_op(case):
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

    return GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist)


def _work(rank, world, S):
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.greedy import greedy_step
    from paper_2305_15661_b200.lm import LmConfig
    from paper_2305_15661_b200.sharded import gather_rows, snapshot_rows

    case = small_case()
    op = gpu_op(case)
    ids, rows = snapshot_rows(op, case, S, seed=8, rank=rank, world=world)
    full = gather_rows(rows, S, rank, world) if world > 1 else rows
    full = None if full is None else full.cpu().numpy()
    g = greedy_step(op, case.mus, [2], WeightVector(case.rho), case.W[0], None, LmConfig(max_iters=8), rank, world)
    return full, g


def _worker(rank, world, port, S, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank,) + _work(rank, world, S))
    finally:
        dist.destroy_process_group()


def test_two_ranks_match_single_rank():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    S = 5
    full1, g1 = _work(0, 1, S)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, S, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (f, g) for r, f, g in (q.get(timeout=600) for _ in procs)}
    for p in procs:
        p.join(timeout=120)
    assert res[1][0] is None
    assert np.array_equal(res[0][0], full1)  # snapshot rows, bit for bit, in snapshot order
    for r in (0, 1):  # both ranks hold the global winner, identical to the single-rank search
        assert res[r][1][1] == g1[1] and (res[r][1][0] == g1[0] or (np.isnan(res[r][1][0]) and np.isnan(g1[0])))
