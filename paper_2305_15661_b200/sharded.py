"""Multi-GPU sharding of the training configurations.

One process per GPU (``torchrun``; ``torch.distributed`` over NCCL, or gloo in
the CPU tests).  Only the data-parallel axes the reference's algorithm has are
sharded, and only its real exchange steps are collectives:

* config 4, EQP constraint rows (eqp.build_lp, eqp.py:82-124): training
  snapshots are independent — rank r of G owns snapshots {s : s mod G = r},
  evaluates their element contributions with no communication, and the row
  blocks are gathered to the LP host (``gather_rows``) in snapshot order;
* config 5, greedy search: candidates are interleaved over
  the ranks (``greedy.greedy_step``) and the argmax is one all-gather of the
  per-rank (indicator, index) winners (``greedy.global_argmax``).

Snapshot fields are generated per snapshot from a seed derived from the
snapshot index (``snapshot_fields_device``), so a rank builds only the
snapshots it owns and every snapshot is bit-identical whichever rank builds it.
"""

import numpy as np
import torch

from .greedy import shard


def snapshot_ids(S, rank, world):
    """Snapshots owned by ``rank`` of ``world`` (interleaved: s = rank, rank + world, ...)."""
    return shard(S, rank, world, "interleaved")


def snapshot_fields_device(case, ids, seed, device, jitter=0.05, amp=0.05, mach_range=(2.0, 4.0), gamma=1.4):
    """Config 4 training snapshots (state and mesh perturbations as in config 2) for the
    snapshot indices ``ids``, generated on ``device``: (mus (S, 1) host, U (S, N_u), X (S, N_x)).

    Snapshot s uses its own generator (seed * 1_000_003 + s): freestream(Mach mu_s) perturbed
    per DG node in its primitive variables, rho, u and p times (1 + U(-jitter, jitter)) and
    v = u U(-jitter, jitter) (conservative per-component jitter makes the pressure negative at
    Mach ~4), and the reference coordinates plus four sinusoid modes of amplitude amp * h
    (configs.displacement)."""
    mesh = case.mesh
    ne, nb = mesh.num_elements, 6
    nodes = torch.as_tensor(mesh.nodes, dtype=torch.float64, device=device)
    h = 1.0 / max(1, int(round(np.sqrt(ne / 2))))
    ids = np.asarray(ids, dtype=np.int64)
    S = len(ids)
    mus = np.zeros((S, 1))
    U = torch.empty((S, ne * nb * 4), dtype=torch.float64, device=device)
    X = torch.empty((S, 2 * mesh.num_nodes), dtype=torch.float64, device=device)
    for j, s in enumerate(ids):
        g = torch.Generator(device=device).manual_seed(int(seed) * 1_000_003 + int(s))
        mu = float(mach_range[0] + (mach_range[1] - mach_range[0]) * torch.rand(1, generator=g, device=device,
                                                                                  dtype=torch.float64))
        mus[j, 0] = mu
        d = jitter * (2.0 * torch.rand((ne * nb, 4), generator=g, device=device, dtype=torch.float64) - 1.0)
        rho, u = 1.0 + d[:, 0], mu * (1.0 + d[:, 1])
        v, p = mu * d[:, 2], (1.0 / gamma) * (1.0 + d[:, 3])
        U[j] = torch.stack([rho, rho * u, rho * v, p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)], 1).reshape(-1)
        x = nodes.clone()
        for _ in range(4):
            k = torch.randint(1, 5, (2,), generator=g, device=device).double()
            ph, th = (2 * np.pi * torch.rand(2, generator=g, device=device, dtype=torch.float64)).unbind()
            sv = torch.sin(2 * np.pi * (k[0] * nodes[:, 0] + k[1] * nodes[:, 1]) + ph)
            x[:, 0] += amp * h * torch.cos(th) * sv
            x[:, 1] += amp * h * torch.sin(th) * sv
        X[j] = x.reshape(-1)
    return mus, U, X


def snapshot_rows(op, case, S, seed, rank=0, world=1, layout="lprows", out=None):
    """This rank's share of the config-4 constraint rows: (ids, rows (len(ids), K+1, ne))."""
    ids = snapshot_ids(S, rank, world)
    if len(ids) == 0:
        K = op.k_u + op.k_x
        return ids, torch.empty((0, K + 1, op.dm.ne), dtype=torch.float64, device=op.device)
    mus, U, X = snapshot_fields_device(case, ids, seed, op.device)
    return ids, op.contributions_at_snapshots(U, X, mus, layout, out=out)


def gather_rows(rows, S, rank, world, group=None, dst=0):
    """Row blocks of all ranks, in snapshot order, on rank ``dst`` (None elsewhere).

    rows: this rank's (len(snapshot_ids(S, rank, world)), ...) block.  One all-gather of
    blocks padded to ceil(S / world) snapshots (the collective the LP host needs)."""
    import torch.distributed as dist

    if world == 1:
        return rows
    per = (S + world - 1) // world
    dev = rows.device if dist.get_backend(group) == "nccl" else torch.device("cpu")  # gloo: host tensors
    rows = rows.to(dev)
    pad = torch.zeros((per,) + tuple(rows.shape[1:]), dtype=rows.dtype, device=dev)
    pad[: rows.shape[0]] = rows
    allb = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(allb, pad, group=group)
    if rank != dst:
        return None
    full = torch.empty((S,) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
    for r in range(world):
        ids = snapshot_ids(S, r, world)
        full[torch.as_tensor(ids, device=rows.device)] = allb[r][: len(ids)]
    return full
