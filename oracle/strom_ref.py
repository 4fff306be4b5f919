"""Loader for the UNMODIFIED reference package — TEST / BASELINE INFRASTRUCTURE ONLY.

The reference ``strom`` (pure Python/NumPy) is installed once, unmodified,
into ``baseline/_ref`` (``pip install --no-index --no-build-isolation
--no-deps --target baseline/_ref <copy of /root/reference/pkg>``; DESIGN.md
§5) so it travels to the GPU box; in the dev container ``/root/reference``
is used when the install is absent.  ``bench.py --impl reference`` and its
``cpu_baseline`` leg time the stock code path through this module:
``strom.reduced.ReducedOperator.derivatives`` (reduced.py:209-229) and
``strom.lm.lm_solve`` (lm.py:164-271) on the reference's own dual numbers,
element kernel and distortion.

What is added around the stock path, all through the reference's own
extension points (the same ones tests/golden/make_golden.py uses):

* the Euler law as a ``ConservationLawSpec``-compatible object whose
  callables use the reference's dual namespace (``paper_2305_15661_b200.laws``
  with the reference ``Dual`` registered as the backend; the reference ships
  no Euler law, SURVEY §8c ii);
* the 12-point degree-6 triangle rule injected into
  ``strom.quadrature._TRI_RULES[6]`` (SURVEY §8c iii);
* meshes built by this package and handed over as ``ReferenceMesh`` fields
  (connectivity identical to the reference mesher, tests/test_host.py);
* config 2's explicit state enters as an affine offset ``U = U0 + Phi w``
  added in a three-line ``_inputs`` override (SURVEY §8c iv).
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def locate():
    """Directory holding the reference ``strom`` package, or None."""
    for d in CANDIDATES:
        if os.path.isfile(os.path.join(d, "strom", "reduced.py")):
            return d
    return None


def load():
    """Import the reference modules (raises ImportError when the reference is absent)."""
    d = locate()
    if d is None:
        raise ImportError("reference strom not installed (baseline/_ref) and /root/reference absent")
    if d not in sys.path:
        sys.path.insert(0, d)
    from strom import conslaw, distortion, dual, geometry, lm, meshing, quadrature, reduced  # noqa: F401
    from strom import eqp

    from paper_2305_15661_b200 import laws as L, tables

    L.register_dual_backend(dual.Dual, dual)
    tables.install_degree6_rule(quadrature)
    return dict(conslaw=conslaw, distortion=distortion, dual=dual, geometry=geometry, lm=lm, meshing=meshing,
                reduced=reduced, eqp=eqp, path=d)


def operator(case):
    """Stock ``strom.reduced.ReducedOperator`` (with the affine state offset) for a ``configs.Case``."""
    S = load()
    smesh, sgeom, sred, sdist, sdual = S["meshing"], S["geometry"], S["reduced"], S["distortion"], S["dual"]

    class OffsetOperator(sred.ReducedOperator):
        def __init__(self, *a, u0=None):
            super().__init__(*a)
            self.u0 = u0

        def _inputs(self, els, coords, seeded):
            out = super()._inputs(els, coords, seeded)
            if self.u0 is None:
                return out
            g = self.geom
            B, nb, m = len(els), g.n_basis, g.n_comp
            oe = self.u0[g.maps.state_map[els]].reshape(B, nb, m)
            nm = g.maps.neighbor_map[els]
            on = np.where(nm >= 0, self.u0[np.clip(nm, 0, None)], 0.0).reshape(B, 3, nb, m)
            Ue, Un, xe = out
            if seeded:
                return sdual.Dual(Ue.val + oe, Ue.tan), sdual.Dual(Un.val + on, Un.tan), xe
            return Ue + oe, Un + on, xe

    mesh, maps = case.mesh, case.maps
    rm = smesh.ReferenceMesh(dim=2, degree_geo=1, nodes=mesh.nodes.copy(), elements=mesh.elements.copy(),
                             interior_faces=mesh.interior_faces.copy(), boundary_faces=mesh.boundary_faces.copy(),
                             boundary_tags=dict(mesh.boundary_tags))
    rm.validate()
    rmaps = smesh.build_assembly_maps(rm, degree_sol=maps.degree_sol, n_comp=maps.n_comp)
    geom = sgeom.Geometry(rm, rmaps, quad_order=case.quad_order)
    rm._geometry_cache = {(rmaps.degree_sol, rmaps.n_comp, None): geom}
    bases = sred.ReducedBases(case.phi, case.psi, case.ref_coords)
    return OffsetOperator(case.law, geom, bases, sdist.DistortionConfig(case.kappa, case.eps), u0=case.state_offset)


def coords(w, tau):
    return load()["reduced"].ReducedCoords(np.asarray(w, float), np.asarray(tau, float))


def weights(rho):
    return None if rho is None else load()["eqp"].WeightVector(np.asarray(rho, float))


def lm_solve(op, mu, rho=None, w0=None, max_iters=200):
    """Stock ``strom.lm.lm_solve`` on a ``ReducedTrackingProblem`` (reduced.py:254-281)."""
    S = load()
    prob = S["reduced"].ReducedTrackingProblem(op, np.asarray(mu, float), rho=weights(rho), w0=w0)
    return S["lm"].lm_solve(prob, S["lm"].LmConfig(max_iters=max_iters))
