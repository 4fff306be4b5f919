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
