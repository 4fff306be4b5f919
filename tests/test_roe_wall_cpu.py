"""CPU checks of the Roe flux and slip-wall host specs the GPU extensions restate (no GPU)."""

import numpy as np

import oracle.dual as D
from oracle.element import OracleGeometry, OracleReducedOperator, reflect_state
from paper_2305_15661_b200 import configs, laws as L

L.register_dual_backend(D.Dual, D)


def test_slip_wall_has_no_mass_flux():
    """The mass component of the face flux vanishes on a slip wall, for LLF and Roe."""
    rng = np.random.default_rng(5)
    law_llf, law_roe = L.euler(flux="llf"), L.euler(flux="roe")
    for _ in range(5):
        u = L.euler_freestream(rng.uniform(2, 4)) * (1 + 0.1 * rng.standard_normal(4))
        th = rng.uniform(0, 2 * np.pi)
        n = np.array([np.cos(th), np.sin(th)])
        ug = reflect_state(u[None], n[None])[0]
        fn = (np.einsum("ci,i->c", law_llf.flux(u[None], None, None)[0], n)
              + np.einsum("ci,i->c", law_llf.flux(ug[None], None, None)[0], n))
        lam = law_llf.wavespeed(u[None], n[None], None)[0]
        H_llf = 0.5 * fn - 0.5 * lam * (ug - u)
        H_roe = 0.5 * fn - 0.5 * law_roe.numflux(u[None], ug[None], n[None], None)[0]
        assert abs(H_llf[0]) <= 1e-12 * np.abs(u).max() and abs(H_roe[0]) <= 1e-12 * np.abs(u).max()


def test_roe_property_and_consistency():
    """delta = 0: D = A_roe (uR - uL) equals F(uR).n - F(uL).n when every wave moves one way
    (supersonic normal flow); D(u, u) = 0 for any delta."""
    rng = np.random.default_rng(2)
    law = L.euler()
    Dz, Dd = L.roe_dissipation(1.4, 0.0), L.roe_dissipation(1.4)
    for _ in range(5):
        uL = L.euler_freestream(3.0) * (1 + 0.05 * rng.standard_normal(4))
        uR = L.euler_freestream(3.2) * (1 + 0.05 * rng.standard_normal(4))
        th = rng.uniform(-0.3, 0.3)
        n = np.array([np.cos(th), np.sin(th)])
        dF = np.einsum("ci,i->c", law.flux(uR[None], None, None)[0] - law.flux(uL[None], None, None)[0], n)
        assert np.allclose(Dz(uL[None], uR[None], n[None], None)[0], dF, rtol=1e-12, atol=1e-12)
        assert np.all(Dd(uL[None], uL[None], n[None], None) == 0.0)


def test_oracle_derivatives_match_finite_differences():
    """The oracle's dual-number gradient (S, T) through the Roe flux and the slip wall matches
    central differences of its objective (validates the dual paths the GPU is checked against)."""
    case = configs.sector_rom_case(n_radial=3, n_circ=5, ku=5, kx=3, frac_active=0.4, rho_scale=2.0, P=1, seed=91,
                                   wall="slip", flux="roe")
    op = OracleReducedOperator(case.law, OracleGeometry(case.mesh, case.maps, case.quad_order), case.phi, case.psi,
                               case.ref_coords, case.kappa, case.eps)
    rng = np.random.default_rng(4)
    w, tau = case.W[0] + 0.05 * rng.standard_normal(5), 0.02 * rng.standard_normal(3)
    mu = case.mus[0]
    _, S, T, *_ = op.derivatives(w, tau, mu, None)
    g = np.concatenate([S, T])
    z = np.concatenate([w, tau])
    for _ in range(3):
        v = rng.standard_normal(8)
        v /= np.linalg.norm(v)
        h = 1e-6 * np.linalg.norm(z)
        J = lambda zz: op.objective(zz[:5], zz[5:], mu, None)  # noqa: E731
        fd = (J(z + h * v) - J(z - h * v)) / (2 * h)
        assert abs(fd - g @ v) <= 1e-6 * np.linalg.norm(g)
