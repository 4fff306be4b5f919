"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset is involved: every array comes from
``numpy.random.default_rng(seed)`` (seed = config number unless stated) so
the oracle and the GPU see identical inputs.  Choices the BASELINE leaves
open are fixed here and recorded in DESIGN.md §6:

* distortion weight kappa = 1e-3, eps = 1e-8;
* config 1: strip [0,1] x [0,1/64], 64 x 1 cells (128 triangles), steady
  Burgers (u^2/2)_x = mu u with u(0)=1, u(1)=-0.5 (laws.burgers_strip);
* configs 3-5: annular sector r in [0.5, 1.5] around a half cylinder;
* mesh displacement modes: integer wave numbers in [1, 4], random phase and
  direction, amplitude 0.05 h (h = smallest edge spacing of the grid).
"""

from dataclasses import dataclass, field

import numpy as np

from . import laws as L
from .mesh import Geometry, build_box_mesh, build_sector_mesh

KAPPA = 1e-3
EPS = 1e-8


@dataclass
class DistortionConfig:
    """Mirror of strom.distortion.DistortionConfig (distortion.py:19-26)."""

    kappa: float
    eps: float = 1e-8

    def __post_init__(self):
        if self.kappa <= 0.0 or self.eps <= 0.0:
            raise ValueError("kappa and eps must be positive")


@dataclass
class Case:
    name: str
    law: object
    mesh: object
    maps: object
    quad_order: int
    phi: np.ndarray
    psi: np.ndarray
    ref_coords: np.ndarray
    mus: np.ndarray                 # (P, n_mu)
    W: np.ndarray                   # (P, k_u)
    Tau: np.ndarray                 # (P, k_x)
    rho: np.ndarray = None          # (ne,) or None (all ones, reduced.py:134-141)
    state_offset: np.ndarray = None
    kappa: float = KAPPA
    eps: float = EPS
    extra: dict = field(default_factory=dict)

    @property
    def geom(self):
        return Geometry(self.mesh, self.maps, self.quad_order)

    @property
    def dist(self):
        return DistortionConfig(self.kappa, self.eps)


def orthonormal(rng, n, k, first=None):
    A = rng.standard_normal((n, k))
    if first is not None:
        A[:, 0] = first
    Q, R = np.linalg.qr(A)
    return Q * np.sign(np.diag(R))[None, :]


def eqp_weights(rng, ne, n_active, scale):
    act = np.sort(rng.choice(ne, n_active, replace=False))
    rho = np.zeros(ne)
    rho[act] = rng.uniform(0.5, 2.0, n_active) * scale
    return rho


def displacement(rng, nodes, h, n_modes=4, amp=0.05):
    d = np.zeros_like(nodes)
    for _ in range(n_modes):
        kx, ky = rng.integers(1, 5, size=2)
        ph = rng.uniform(0, 2 * np.pi)
        th = rng.uniform(0, 2 * np.pi)
        s = np.sin(2 * np.pi * (kx * nodes[:, 0] + ky * nodes[:, 1]) + ph)
        d[:, 0] += amp * h * np.cos(th) * s
        d[:, 1] += amp * h * np.sin(th) * s
    return d


def freestream_field(rng, ne, nb, mach, gamma=1.4, jitter=0.05, per_component=False):
    """Freestream times (1 + U(-jitter, jitter)), one factor per DG node
    (config 2's definition) or one per node and component.

    With a common factor the velocity and sound speed are identical on both
    sides of every face, so the LLF max(ws_in, ws_out) is an exact tie whose
    one-sided derivative is decided by last-bit rounding (reference and GPU
    may legitimately differ there); parity inputs use ``per_component``.
    """
    ff = L.euler_freestream(mach, gamma)
    fac = 1.0 + rng.uniform(-jitter, jitter, size=(ne, nb, 4 if per_component else 1))
    return (fac * ff[None, None, :]).reshape(-1)


# -- config 1 -----------------------------------------------------------------------
def strip_case(ncell=64, ku=4, kx=2, n_active=10, P=8, seed=1, quad_order=None, boundary_in_sample=True):
    """Config 1.  The EQP sample always contains the two elements that touch the
    prescribed left / right boundaries (``boundary_in_sample``): without them the
    weighted residual at U = 0 vanishes identically and every solve is trivial."""
    mesh, maps = build_box_mesh(((0.0, 0.0), (1.0, 1.0 / ncell)), ncell, 1, degree_sol=2, n_comp=1)
    rng = np.random.default_rng(seed)
    phi = orthonormal(rng, maps.n_global_state, ku)
    psi = orthonormal(rng, maps.n_global_coord, kx)
    rho = eqp_weights(rng, mesh.num_elements, n_active, mesh.num_elements / n_active)
    if boundary_in_sample:
        _, _, _, tag = mesh.neighbor_tables()
        ends = [int(np.flatnonzero(np.any(tag == mesh.boundary_tags[t], axis=1))[0]) for t in ("left", "right")]
        for e in ends:
            if rho[e] == 0.0:
                drop = np.flatnonzero(rho > 0.0)
                drop = [d for d in drop if d not in ends]
                rho[rng.choice(drop)] = 0.0
                rho[e] = rng.uniform(0.5, 2.0) * mesh.num_elements / n_active
    mus = rng.uniform(1.0, 3.0, size=(P, 1))
    return Case("cfg1-strip", L.burgers_strip(), mesh, maps, quad_order, phi, psi, mesh.nodes.ravel().copy(),
                mus, np.zeros((P, ku)), np.zeros((P, kx)), rho)


# -- config 2 -----------------------------------------------------------------------
def euler_square_case(n=256, ku=16, kx=8, seed=2, mach=2.0, quad_order=6, per_component=True):
    """Element microbench: unit square, 2 n^2 triangles, explicit (U, x) fields.

    The state is freestream x (1 + U(-0.05, 0.05)) per DG node, drawn
    independently per component (``per_component=True``, the default and the
    benchmarked input): a factor shared by the four components of a node
    leaves velocity and sound speed identical on both sides of every face, so
    every LLF max(ws_in, ws_out) would be an exact tie decided by last-bit
    rounding (tests/test_gpu_bench_inputs.py).

    The state and deformed coordinates enter as the affine offsets of the
    reduced parametrisation (U = U0 + Phi w, x = x_field + Psi tau) at
    w = 0, tau = 0, so the reduced Jacobian is evaluated at the given fields
    with tangents seeded by Phi and Psi (SURVEY §8c iv).
    """
    mesh, maps = build_box_mesh(((0.0, 0.0), (1.0, 1.0)), n, n, degree_sol=2, n_comp=4)
    rng = np.random.default_rng(seed)
    nb = 6
    U0 = freestream_field(rng, mesh.num_elements, nb, mach, per_component=per_component)
    x = (mesh.nodes + displacement(rng, mesh.nodes, 1.0 / n)).ravel()
    phi = orthonormal(rng, maps.n_global_state, ku)
    psi = orthonormal(rng, maps.n_global_coord, kx)
    law = L.euler(tags={t: "freestream" for t in ("left", "right", "bottom", "top")})
    return Case("cfg2-euler-square", law, mesh, maps, quad_order, phi, psi, x, np.array([[mach]]),
                np.zeros((1, ku)), np.zeros((1, kx)), None, U0)


# -- configs 3-5 (half cylinder) -----------------------------------------------------------
def sector_bcs(wall="slip"):
    """Half-cylinder boundary conditions: inflow = prescribed freestream(mu), outflow =
    extrapolate, cylinder wall = slip wall ("slip", the physical one that forms the bow shock;
    a GPU-only extension the reference cannot express) or "extrapolate" (the reference-
    expressible variant the reference goldens and CPU timings use)."""
    return {"inflow": "freestream", "outflow": "extrapolate", "wall": "wall" if wall == "slip" else "extrapolate"}


SECTOR_BCS = sector_bcs("extrapolate")


def smooth_modes(rng, nodes, k, n_modes=4):
    """(2 n_nodes, k) orthonormal basis of smooth mesh motions: each column is a sum of
    ``n_modes`` seeded sinusoid modes (integer wave numbers in [1, 4], random phase and
    direction, as ``displacement``) interleaved (x, y) per node, then QR."""
    cols = [displacement(rng, nodes, 1.0, n_modes, 1.0).ravel() for _ in range(k)]
    Q, R = np.linalg.qr(np.stack(cols, axis=1))
    return Q * np.sign(np.diag(R))[None, :]


def sector_rom_case(n_radial=100, n_circ=200, ku=20, kx=10, frac_active=0.02, rho_scale=50.0, P=64, seed=3,
                    quad_order=6, name="cfg3-half-cylinder", wall="slip", psi_kind="smooth", flux="llf"):
    """Half-cylinder ROM case (configs 3-5).  Phi = QR([normalised freestream(3), Gaussian
    columns]); Psi = seeded orthonormal smooth mesh motions (``smooth_modes``; a Gaussian Psi
    moves neighbouring nodes independently and inverts elements outside the EQP sample once
    tau is O(0.1)), or ``psi_kind="gaussian"``."""
    mesh, maps = build_sector_mesh(n_radial, n_circ, degree_sol=2, n_comp=4)
    rng = np.random.default_rng(seed)
    ne = mesh.num_elements
    ff = np.tile(L.euler_freestream(3.0), ne * 6)
    phi = orthonormal(rng, maps.n_global_state, ku, first=ff / np.linalg.norm(ff))
    psi = orthonormal(rng, maps.n_global_coord, kx) if psi_kind == "gaussian" else smooth_modes(rng, mesh.nodes, kx)
    n_act = max(1, int(round(frac_active * ne)))
    rho = eqp_weights(rng, ne, n_act, rho_scale)
    mus = rng.uniform(2.0, 4.0, size=(P, 1))
    w0 = phi.T @ ff
    law = L.euler(tags=sector_bcs(wall), flux=flux)
    return Case(name, law, mesh, maps, quad_order, phi, psi, mesh.nodes.ravel().copy(), mus,
                np.tile(w0, (P, 1)), np.zeros((P, kx)), rho)


def cfg3(wall="slip"):
    return sector_rom_case(wall=wall)


def cfg4_case(wall="slip"):
    """Config 4 geometry: the config-3 sector scaled to 320 x 625 quads = 400,000 triangles,
    k_u = 20, k_x = 10 (the snapshots come from sharded.snapshot_fields_device)."""
    return sector_rom_case(320, 625, 20, 10, 0.02, 50.0, 1, seed=4, name="cfg4-eqp-rows", wall=wall)


def cfg5_rom(P=1024, wall="slip", kappa=1.0):
    """Config 5.  Distortion weight kappa = 1 (not the 1e-3 of the other configs): with the
    untrained seeded bases the LM drives |tau| to ~7, and at kappa = 1e-3 every candidate's
    reconstructed full mesh inverts an element (a failed, +inf candidate); at kappa = 1 all
    stay valid and the greedy argmax is decided by the residual (tools/diag_cfg45.py)."""
    case = sector_rom_case(200, 400, 24, 12, 0.03, 100.0 / 3.0, P, seed=5, name="cfg5-greedy", wall=wall)
    case.kappa = kappa
    return case


def snapshot_fields(case, S, seed, mach_range=(2.0, 4.0)):
    """Training snapshots for config 4: perturbed freestream states and meshes."""
    rng = np.random.default_rng(seed)
    mesh = case.mesh
    h = (1.5 - 0.5) / max(1, int(round(np.sqrt(mesh.num_elements / 2))))
    mus = rng.uniform(*mach_range, size=(S, 1))
    U = np.stack([freestream_field(rng, mesh.num_elements, 6, m[0], per_component=True) for m in mus])
    X = np.stack([(mesh.nodes + displacement(rng, mesh.nodes, h)).ravel() for _ in range(S)])
    return mus, U, X
