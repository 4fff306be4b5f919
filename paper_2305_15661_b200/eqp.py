"""EQP weights (strom/eqp.py:28-50) and weighted reduced sums on the GPU.

``WeightVector`` mirrors the reference (rho >= 0, ``active =
flatnonzero(rho > 0)`` ascending, ``sparsity``, ``touched_elements``);
``weighted_residuals`` / ``weighted_objective`` mirror eqp.py:66-79 on the
GPU operator.
"""

import numpy as np

from .mesh import get_geometry


class WeightVector:
    def __init__(self, rho):
        self.rho = np.asarray(rho, dtype=float)
        if np.any(self.rho < 0.0):
            raise ValueError("weights must be non-negative")
        self.active = np.flatnonzero(self.rho > 0.0)

    @classmethod
    def ones(cls, n_elements):
        return cls(np.ones(n_elements))

    @property
    def sparsity(self):
        return len(self.active) / len(self.rho)

    def touched_elements(self, mesh):
        nbr, _, _, _ = mesh.neighbor_tables()
        n = nbr[self.active].ravel()
        return np.unique(np.concatenate([self.active, n[n >= 0]]))


def weighted_residuals(law, mesh, maps, bases, weights, coords, mu, dist_config, stats=None):
    from .reduced import GpuReducedOperator

    op = GpuReducedOperator(law, get_geometry(mesh, maps), bases, dist_config)
    out = op.residuals(coords, mu, rho=weights)
    if stats is not None:
        stats.update(op.stats)
        stats["elements_touched"] = len(weights.touched_elements(mesh))
    return out


def weighted_objective(law, mesh, maps, bases, weights, coords, mu, dist_config):
    from .reduced import GpuReducedOperator

    return GpuReducedOperator(law, get_geometry(mesh, maps), bases, dist_config).objective(coords, mu, rho=weights)


# -- weight-training LP rows (eqp.py:82-124) ------------------------------------------
from dataclasses import dataclass, field


@dataclass
class LpProblem:
    """Mirror of strom.simplex.LpProblem fields used by build_lp (simplex.py:20-60)."""

    c: np.ndarray
    A: np.ndarray
    lo_row: np.ndarray
    hi_row: np.ndarray
    lb: np.ndarray
    row_labels: list = field(default_factory=list)
    fallback: np.ndarray = None


@dataclass
class EqpTrainingConfig:
    delta: float
    xi: np.ndarray

    def __post_init__(self):
        self.xi = np.atleast_2d(np.asarray(self.xi, dtype=float))
        if self.delta <= 0.0:
            raise ValueError("delta must be positive")
        if len(self.xi) == 0:
            raise ValueError("training set must be nonempty")


def build_lp(law, mesh, maps, bases, guess_weights, training_solutions, config, dist_config, op=None):
    """Weight-training LP at frozen training solutions (eqp.py:82-124), built
    with one batched GPU pass over all training parameters.

    Row 0: element areas in [(1-delta)|Omega|, (1+delta)|Omega|]; then for
    each training parameter and each part (sr-vol, sr-face, dr-vol, dr-face)
    and component, the column of per-element contributions with bounds
    (sum +- delta/|Xi|).
    """
    import torch

    from .reduced import GpuReducedOperator, _lib

    geom = get_geometry(mesh, maps)
    if op is None:
        op = GpuReducedOperator(law, geom, bases, dist_config)
    ku, kx, ne = op.k_u, op.k_x, mesh.num_elements
    P = len(config.xi)
    W = torch.as_tensor(np.stack([np.asarray(c.w, float) for c in training_solutions])).to(op.device)
    Tau = torch.as_tensor(np.stack([np.asarray(c.tau, float) for c in training_solutions])).to(op.device)
    Mu = torch.as_tensor(np.stack([op._mu(m) for m in config.xi])).to(op.device)
    out, _ = op.eval_batched(_lib.CONTRIB_SPLIT, W, Tau, Mu, None)
    parts = out.view(P, ne, 2 * (ku + kx)).cpu().numpy()
    areas = mesh.element_areas()
    total = float(np.sum(areas))
    rows, lo, hi, labels = [areas], [(1.0 - config.delta) * total], [(1.0 + config.delta) * total], [("dv",)]
    bound = config.delta / P
    offs = {"sr-vol": (0, ku), "sr-face": (ku, ku), "dr-vol": (2 * ku, kx), "dr-face": (2 * ku + kx, kx)}
    for j in range(P):
        for name in ("sr-vol", "sr-face", "dr-vol", "dr-face"):
            o, n = offs[name]
            for comp in range(n):
                col = parts[j, :, o + comp]
                center = float(np.sum(col))
                rows.append(col)
                lo.append(center - bound)
                hi.append(center + bound)
                labels.append((name, j, comp))
    return LpProblem(c=np.ones(ne), A=np.asarray(rows), lo_row=np.asarray(lo), hi_row=np.asarray(hi),
                     lb=np.zeros(ne), row_labels=labels, fallback=np.asarray(guess_weights.rho, dtype=float).copy())
