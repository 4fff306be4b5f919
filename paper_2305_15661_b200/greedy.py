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


# -- Algorithm 1 (SPEC.md greedy-driver, no reference code) ---------------
class BasisInSpanError(ValueError):
    """New column numerically inside the span of the basis (strom/reduced.py:20-22)."""


class CandidateSetExhausted(RuntimeError):
    """Every candidate parameter is already a training parameter (SPEC greedy_search errors)."""


def gram_schmidt_append(basis, new_column, tol=1e-10):
    """Append one column to an orthonormal basis: modified Gram-Schmidt with one
    re-orthogonalisation pass, BasisInSpanError below ``tol`` times the column norm
    (semantics of strom/reduced.py:88-113)."""
    col = np.asarray(new_column, dtype=float).reshape(-1).copy()
    nrm0 = np.linalg.norm(col)
    if nrm0 == 0.0:
        raise BasisInSpanError("zero column")
    basis = np.asarray(basis, dtype=float)
    if basis.size == 0:
        return (col / nrm0)[:, None]
    basis = basis.reshape(col.shape[0], -1)
    v = col
    for _ in range(2):
        v = v - basis @ (basis.T @ v)
    nrm = np.linalg.norm(v)
    if nrm < tol * nrm0:
        raise BasisInSpanError(f"column inside span (residual {nrm:.3e} vs norm {nrm0:.3e})")
    return np.column_stack([basis, v / nrm])


def seed_index(cand_mus):
    """mu_1 = argmin ||mu - centroid|| over the candidate set, first index on ties (SPEC seed)."""
    mus = np.atleast_2d(np.asarray(cand_mus, dtype=float))
    d = np.linalg.norm(mus - mus.mean(axis=0), axis=1)
    return int(np.flatnonzero(d == d.min())[0])


class GreedyState:
    """Training state of Algorithm 1 (SPEC GreedyState): selected candidate indices, bases,
    weights, snapshots and one metrics record per iteration."""

    def __init__(self, phi, psi, ref_coords, weights, selected, snapshots):
        from .reduced import ReducedBases

        self.bases = ReducedBases(phi, psi, ref_coords)
        self.weights = weights
        self.selected = list(selected)
        self.snapshots = list(snapshots)
        self.metrics = []

    @property
    def j(self):
        return len(self.selected)


# -- full-space callbacks of Algorithm 1 on the GPU-assembled blocks ----------
def tracking_alignment(law, geom, dist_config, lm_config=None, device=None):
    """``align(bases, mu) -> x*``: SPEC snapshot_alignment (Eq. align0) — the alignment problem
    over (w in R^j, sliding deformation) solved by ``lm.lm_solve`` on a
    ``tracking.TrackingProblem`` with the current state basis; the state coefficients are
    discarded.  A solve that fails or does not reduce the objective falls back to x = X with a
    warning (the snapshot is then added unaligned)."""
    import warnings

    from .lm import LmConfig, lm_solve
    from .reduced import DegenerateMappingError
    from .tracking import TrackingProblem

    def align(bases, mu, w0=None):
        X = np.asarray(geom.mesh.nodes, dtype=float).ravel()
        if w0 is None:  # the law's initial guess at mu projected on the state basis (w = 0 is no state)
            from .fullspace import initial_state

            w0 = bases.phi.T @ initial_state(law, geom.mesh, geom.maps, X, mu, geom)
        try:
            prob = TrackingProblem(law, geom.mesh, geom.maps, mu, dist_config, state_basis=bases.phi, w0=w0,
                                   geom=geom, device=device)
            j0 = prob.objective(*prob.initial_guess())
            res = lm_solve(prob, lm_config or LmConfig(max_iters=20), w0_mode="lsq")
        except (DegenerateMappingError, np.linalg.LinAlgError) as exc:
            warnings.warn(f"snapshot alignment at mu={np.asarray(mu).tolist()} failed ({exc}); x = X")
            return X
        if not np.isfinite(res.objective) or res.objective > j0:
            warnings.warn(f"snapshot alignment at mu={np.asarray(mu).tolist()} did not reduce the objective; x = X")
            return X
        return prob.coords_from(res.tau)

    return align


def tracking_snapshot(law, geom, dist_config, lm_config=None, track=True, hdm_tol=1e-10, device=None):
    """``hdm_snapshot(mu, x_aligned) -> (U*, x*)``: with ``track``, the full-space tracking solve
    on the enriched residual from the law's initial guess on the aligned mesh (tracking.py:41-150;
    SPEC seed: Phi = I, Psi = I, rho = 1), then the HDM solve on the tracked mesh
    (``fullspace.solve_hdm``, dg.py:343-400: plain Newton suffices on a feature-aligned mesh) —
    both on GPU-assembled residuals and sparse Jacobians.  An HDM solve that does not converge
    keeps the tracked state with a warning."""
    import warnings

    from .fullspace import HdmSolveError, initial_state, solve_hdm
    from .lm import LmConfig, lm_solve
    from .tracking import TrackingProblem

    def hdm_snapshot(mu, x_aligned, U_init=None):
        mesh, maps = geom.mesh, geom.maps
        x = np.asarray(x_aligned, dtype=float).copy()
        U = initial_state(law, mesh, maps, x, mu, geom) if U_init is None else np.asarray(U_init, dtype=float)
        if track:
            prob = TrackingProblem(law, mesh, maps, mu, dist_config, U0=U, x0=x, geom=geom, device=device)
            res = lm_solve(prob, lm_config or LmConfig(max_iters=50), w0_mode="keep")
            U, x = res.w, prob.coords_from(res.tau)
        try:
            U = solve_hdm(law, mesh, maps, x, mu, U_init=U, tol=hdm_tol, geom=geom, device=device)
        except HdmSolveError as exc:
            warnings.warn(f"HDM solve at mu={np.asarray(mu).tolist()} stopped at |R| = {exc.residual_norm:.2e}; "
                          "the tracked state is kept")
        return U, x

    return hdm_snapshot


def greedy_train(law, geom, cand_mus, hdm_snapshot, n_iter, dist_config, train_weights, lm_config=None, align=None,
                 rank=0, world=1, group=None, device=None):
    """Greedy training (Algorithm 1): seed, then per iteration greedy search (GPU, candidates
    sharded over ranks), snapshot alignment, HDM snapshot, basis growth by Gram-Schmidt and
    EQP weight retraining with the previous weights as the guess.

    The full-space solves are callbacks: ``hdm_snapshot(mu, x_aligned) -> (U*, x*)`` (None:
    ``tracking_snapshot``, the GPU-assembled HDM + full-space tracking solve) and
    ``align(bases, mu) -> x_aligned`` (None: x = X, SPEC's no-alignment fallback; "tracking":
    ``tracking_alignment``, the alignment problem of Eq. align0).
    ``train_weights(bases, guess, selected_mus) -> WeightVector`` is the EQP LP (e.g. the
    reference's strom.eqp.train_weights with the GPU operator swapped in, dropin.install).
    Seed (SPEC): mu_1 nearest the candidate centroid, Phi_1 = U*(mu_1)/||U*||,
    Psi_1 = X/||X||, rho_1 trained from the all-ones guess.
    """
    import time

    from .eqp import WeightVector
    from .lm import LmConfig
    from .reduced import GpuReducedOperator

    cand_mus = np.atleast_2d(np.asarray(cand_mus, dtype=float))
    X = np.asarray(geom.mesh.nodes, dtype=float).ravel()
    if hdm_snapshot is None:
        hdm_snapshot = tracking_snapshot(law, geom, dist_config, device=device)
    if isinstance(align, str):
        if align != "tracking":
            raise ValueError(f"unknown alignment {align!r}")
        align = tracking_alignment(law, geom, dist_config, device=device)
    i1 = seed_index(cand_mus)
    U1, _ = hdm_snapshot(cand_mus[i1], X)
    phi = gram_schmidt_append(np.zeros((len(U1), 0)), U1)
    psi = gram_schmidt_append(np.zeros((len(X), 0)), X)
    state = GreedyState(phi, psi, X, None, [i1], [(np.asarray(U1), X)])
    t0 = time.perf_counter()
    state.weights = train_weights(state.bases, WeightVector.ones(geom.mesh.num_elements), cand_mus[state.selected])
    state.metrics.append({"j": 1, "mu": cand_mus[i1].tolist(), "T_rho": time.perf_counter() - t0,
                          "active": int(len(state.weights.active))})
    for _ in range(1, n_iter):
        if len(state.selected) >= len(cand_mus):
            raise CandidateSetExhausted("all candidate parameters are training parameters")
        op = GpuReducedOperator(law, geom, state.bases, dist_config, device=device)
        t0 = time.perf_counter()
        w0 = state.bases.phi.T @ state.snapshots[-1][0]  # projection of the latest snapshot
        v, i = greedy_step(op, cand_mus, state.selected, state.weights, w0, None, lm_config or LmConfig(), rank,
                           world, group)
        t_gs = time.perf_counter() - t0
        if i < 0:
            raise CandidateSetExhausted("no selectable candidate")
        x_al = align(state.bases, cand_mus[i]) if align is not None else X
        U, x = hdm_snapshot(cand_mus[i], x_al)
        state.bases.phi = gram_schmidt_append(state.bases.phi, U)
        try:  # an unaligned snapshot (x* = X, SPEC's alignment fallback) adds no mesh motion
            state.bases.psi = gram_schmidt_append(state.bases.psi, np.asarray(x, dtype=float) - X)
            psi_grown = True
        except BasisInSpanError:
            import warnings

            warnings.warn(f"mesh snapshot at mu={cand_mus[i].tolist()} adds no new motion; Psi not grown")
            psi_grown = False
        state.selected.append(int(i))
        state.snapshots.append((np.asarray(U), np.asarray(x)))
        t0 = time.perf_counter()
        state.weights = train_weights(state.bases, state.weights, cand_mus[state.selected])
        state.metrics.append({"j": state.j, "mu": cand_mus[i].tolist(), "indicator": v, "T_gs": t_gs,
                              "T_rho": time.perf_counter() - t0, "active": int(len(state.weights.active)),
                              "psi_grown": psi_grown})
    return state
