"""Greedy-training error indicator and the multi-GPU candidate / snapshot sharding.

SPEC.md:489-497 (no reference code): for every candidate mu not yet
selected, solve the hyperreduced ROM, reconstruct (U, x) and take the
full-mesh residual norm ||R(U, x; mu)||_2 as the error indicator; the next
training point is the argmax, first index on ties, failed solves count as
+inf, already-selected candidates are excluded
(SPEC.md:534).  Candidates and training snapshots are embarrassingly
parallel: rank r of G owns candidates {i : i mod G = r} (interleaved for
load balance) and the global argmax is one all-gather of (value, index)
pairs per rank.
"""

import math

import numpy as np


def shard(n, rank, world, mode="interleaved"):
    """Indices of ``n`` work items owned by ``rank`` of ``world``."""
    if mode == "interleaved":
        return np.arange(rank, n, world)
    lo, hi = n * rank // world, n * (rank + 1) // world
    return np.arange(lo, hi)


def local_argmax(values, ids, selected=()):
    """(value, id) of the largest indicator; NaN/failed -> +inf; ties -> smallest id."""
    best_v, best_i = -math.inf, -1
    sel = set(int(s) for s in selected)
    for v, i in zip(np.asarray(values, dtype=float), np.asarray(ids)):
        i = int(i)
        if i in sel:
            continue
        v = math.inf if not np.isfinite(v) else float(v)
        if v > best_v or (v == best_v and (best_i < 0 or i < best_i)):
            best_v, best_i = v, i
    return best_v, best_i


def global_argmax(values, ids, selected=(), group=None):
    """Argmax over all ranks: all-gather of the per-rank (value, id) winners."""
    import torch
    import torch.distributed as dist

    v, i = local_argmax(values, ids, selected)
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return v, i
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = torch.tensor([v, float(i)], dtype=torch.float64, device=dev)
    allv = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    pairs = [(float(t[0]), int(t[1])) for t in allv]
    return local_argmax([p[0] for p in pairs if p[1] >= 0], [p[1] for p in pairs if p[1] >= 0], selected)


def indicators(op, mus, W, Tau):
    """Full-mesh residual norms ||R(Phi w, X + Psi tau; mu)||_2 for a batch (GPU)."""
    import torch

    from . import _lib

    Mu = torch.as_tensor(np.stack([op._mu(m) for m in np.atleast_2d(mus)])).to(op.device)
    W = torch.as_tensor(np.asarray(W, float)).to(op.device)
    Tau = torch.as_tensor(np.asarray(Tau, float)).to(op.device)
    degen = torch.zeros(Mu.shape[0], dtype=torch.int32, device=op.device)
    out, _ = op.eval_batched(_lib.RESNORM2, W, Tau, Mu, None, degen=degen)
    # a degenerate reconstructed mesh is a failed candidate: the reference's
    # assemble_global raises DegenerateMappingError there (dg.py:177-178)
    ind = torch.sqrt(out).cpu().numpy()
    return np.where(degen.cpu().numpy() > 0, np.inf, ind)


def greedy_step(op, cand_mus, selected, rho, W0=None, Tau0=None, lm_config=None, rank=0, world=1, group=None,
                stats=None):
    """One greedy search over this rank's candidate shard -> global (indicator, index).
    ``stats`` (dict, optional) receives this rank's candidate / failed-candidate counts."""
    from .lm import lm_solve_batched

    ids = shard(len(cand_mus), rank, world)
    ids = np.array([i for i in ids if i not in set(selected)], dtype=np.int64)
    if len(ids) == 0:
        return global_argmax([], [], selected, group)
    res = lm_solve_batched(op, np.asarray(cand_mus)[ids], W0, Tau0, rho, lm_config)
    W = np.stack([r.w for r in res])
    Tau = np.stack([r.tau for r in res])
    ind = indicators(op, np.asarray(cand_mus)[ids], W, Tau)
    # per-candidate solver failures count as +inf: a non-finite objective or a
    # solve that ended on a degenerate mapping (lm.py:150,231 catch DegenerateMappingError)
    failed = np.array([(not np.isfinite(r.objective)) or r.reason == "degenerate" for r in res])
    ind = np.where(failed, np.inf, ind)
    if stats is not None:
        stats.update(candidates=len(ids), failed=int(np.sum(~np.isfinite(ind))))
    return global_argmax(ind, ids, selected, group)
