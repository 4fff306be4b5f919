"""Multi-process (gloo, world_size 2) tests of the sharding and NCCL-argmax logic on CPU."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_15661_b200.greedy import global_argmax, local_argmax, shard


def test_shard_partitions():
    for n, world in [(10, 3), (1024, 8), (5, 8), (0, 2)]:
        for mode in ("interleaved", "contiguous"):
            allids = np.concatenate([shard(n, r, world, mode) for r in range(world)])
            assert sorted(allids.tolist()) == list(range(n))


def test_local_argmax_rules():
    assert local_argmax([1.0, 3.0, 3.0], [4, 7, 5]) == (3.0, 5)           # tie -> smallest id
    assert local_argmax([1.0, np.nan, 2.0], [0, 1, 2]) == (np.inf, 1)      # failed -> +inf
    assert local_argmax([9.0, 3.0], [0, 1], selected=[0]) == (3.0, 1)      # excluded
    assert local_argmax([], []) == (-np.inf, -1)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    vals = rng.random(37)
    vals[[3, 20]] = vals.max() + 1.0  # tie across ranks
    ids = shard(len(vals), rank, world)
    got = global_argmax(vals[ids], ids, selected=[11])
    # all-reduce of reduced sums (element sharding, config 2): sum of rank partials == total
    part = torch.tensor(vals[ids].sum(), dtype=torch.float64)
    dist.all_reduce(part)
    q.put((rank, got, float(part)))
    dist.destroy_process_group()


def test_global_argmax_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    rng = np.random.default_rng(0)
    vals = rng.random(37)
    vals[[3, 20]] = vals.max() + 1.0
    want = local_argmax(vals, np.arange(37), selected=[11])
    for rank, got, total in res:
        assert got == want == (vals[3], 3)
        assert abs(total - vals.sum()) < 1e-12


# -- config 4 snapshot sharding (paper_2305_15661_b200.sharded) ----------------------------
def test_snapshot_fields_rank_independent():
    """A snapshot's fields do not depend on which rank (which id subset) generates it."""
    from paper_2305_15661_b200 import configs
    from paper_2305_15661_b200.sharded import snapshot_fields_device, snapshot_ids

    case = configs.sector_rom_case(n_radial=3, n_circ=4, ku=4, kx=2, frac_active=0.5, rho_scale=2.0, P=1, seed=9)
    S = 5
    mus, U, X = snapshot_fields_device(case, np.arange(S), 7, "cpu")
    for world in (2, 3):
        for r in range(world):
            ids = snapshot_ids(S, r, world)
            m, u, x = snapshot_fields_device(case, ids, 7, "cpu")
            assert np.array_equal(m, mus[ids]) and torch.equal(u, U[ids]) and torch.equal(x, X[ids])
    # freestream x (1 + U(-0.05, 0.05)) per node and component, Mach in [2, 4]
    ff = U.view(S, -1, 4)
    assert np.all((mus >= 2.0) & (mus <= 4.0))
    assert torch.all((ff[:, :, 0] > 0.95 - 1e-12) & (ff[:, :, 0] < 1.05 + 1e-12))
    assert torch.allclose(X.view(S, -1, 2).mean(0), torch.as_tensor(case.mesh.nodes), atol=0.05 / 2)


def _rows_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_15661_b200.sharded import gather_rows, snapshot_ids

    S = 7
    ids = snapshot_ids(S, rank, world)
    rows = torch.stack([torch.full((3, 4), float(s)) + torch.arange(12.0).view(3, 4) for s in ids])
    full = gather_rows(rows, S, rank, world)
    q.put((rank, None if full is None else full.numpy()))
    dist.destroy_process_group()


def test_gather_rows_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_rows_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    want = np.stack([np.full((3, 4), float(s)) + np.arange(12.0).reshape(3, 4) for s in range(7)])
    assert res[1] is None and np.array_equal(res[0], want)
