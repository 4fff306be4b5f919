"""GPU full-space assembly (fullspace.assemble_global, dg.py:228-272) vs the reference's element
Jacobian goldens (dg.py:197-225, stored by make_golden.py) and vs the oracle's dual-number
assembly over every element."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle.dual as D
from oracle.element import OracleGeometry, element_eval

from cases import build, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def fields(case, g):
    U = case.phi @ g["w"] + (case.state_offset if case.state_offset is not None else 0.0)
    x = case.ref_coords + case.psi @ g["tau"]
    return U, x


@pytest.mark.parametrize("name", ["euler_square_q6", "euler_square_default", "sector"])
def test_element_jacobians_match_reference_goldens(name):
    from paper_2305_15661_b200.fullspace import element_jacobians

    case, g = build(name)
    U, x = fields(case, g)
    res, js, jn, jx = element_jacobians(case.law, case.geom, U, x, case.mus[0])
    elems = sorted({int(k[4:].split("_")[0]) for k in g if k.startswith("elem") and k.endswith("_res")})
    assert elems
    for e in elems:
        scale = np.max(np.abs(g[f"elem{e}_jself"]))
        assert rel_err(res[e], g[f"elem{e}_res"]) < 1e-10
        assert rel_err(js[e], g[f"elem{e}_jself"]) < 1e-10
        assert rel_err(jn[e], g[f"elem{e}_jneigh"], scale) < 1e-10  # off-face reference entries are ~1e-16
        assert rel_err(jx[e], g[f"elem{e}_jcoord"]) < 1e-10


def test_assemble_global_matches_oracle():
    from paper_2305_15661_b200.fullspace import assemble_global

    case, g = build("sector")
    U, x = fields(case, g)
    mu = case.mus[0]
    R, dRdU, dRdx = assemble_global(case.law, case.mesh, case.maps, U, x, mu, geom=case.geom)
    # oracle: every element seeded with identity tangents [U_e | U_nbr | x_e] (dg.py:184-195)
    geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
    els = np.arange(case.mesh.num_elements)
    Ue, Un = geom.gather_state(U, els)
    xe = geom.gather_coords(x, els)
    nu, ng = 24, 3
    T = 4 * nu + 2 * ng
    out = element_eval(case.law, geom, els, D.seed_identity(Ue, 0, T), D.seed_identity(Un, nu, T),
                       D.seed_identity(xe, 4 * nu, T), mu)
    tan = out.res.tan
    maps = case.maps
    Ju = np.zeros((maps.n_global_state, maps.n_global_state))
    Jx = np.zeros((maps.n_global_state, maps.n_global_coord))
    sm, nm, cm = maps.state_map, maps.neighbor_map, maps.coord_map
    for e in els:
        np.add.at(Ju, (sm[e][:, None], sm[e][None, :]), tan[e][:, :nu])
        ok = nm[e] >= 0
        np.add.at(Ju, (sm[e][:, None], nm[e][ok][None, :]), tan[e][:, nu:4 * nu][:, ok])
        np.add.at(Jx, (sm[e][:, None], cm[e][None, :]), tan[e][:, 4 * nu:])
    assert rel_err(R, out.res.val.reshape(-1)) < 1e-10
    assert rel_err(dRdU.toarray(), Ju) < 1e-10 and rel_err(dRdx.toarray(), Jx) < 1e-10
    assert dRdU.shape == (maps.n_global_state, maps.n_global_state)


def test_assemble_distortion_matches_oracle():
    """fullspace.assemble_distortion (distortion.py:71-92) vs the oracle's dual-number
    distortion residuals and their coordinate gradients."""
    from oracle.element import distortion_eval
    from paper_2305_15661_b200.configs import DistortionConfig
    from paper_2305_15661_b200.fullspace import assemble_distortion

    case, g = build("sector")
    _, x = fields(case, g)
    cfg = DistortionConfig(case.kappa, case.eps)
    N, jac = assemble_distortion(case.mesh, case.maps, x, cfg, geom=case.geom)
    geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
    els = np.arange(case.mesh.num_elements)
    xe = geom.gather_coords(x, els)
    out = distortion_eval(geom, els, D.seed_identity(xe, 0, 6), case.kappa, case.eps)
    assert rel_err(N, D.val(out)) < 1e-10
    want = np.zeros((len(els), case.maps.n_global_coord))
    for e in els:
        np.add.at(want, (e, case.maps.coord_map[e]), out.tan[e])
    assert rel_err(jac.toarray(), want) < 1e-10


def test_solve_hdm_converges_and_matches_reference():
    """fullspace.solve_hdm (dg.py:343-400 on GPU-assembled Jacobians) converges to the target and
    to the reference's own solve_hdm state (stock code path, when the reference is installed)."""
    from paper_2305_15661_b200 import configs, laws as L
    from paper_2305_15661_b200.fullspace import assemble_global, solve_hdm

    case = configs.sector_rom_case(n_radial=3, n_circ=6, ku=2, kx=1, frac_active=0.5, rho_scale=2.0, P=1, seed=95,
                                   wall="extrapolate")
    mu = np.array([3.0])
    rng = np.random.default_rng(2)
    U0 = np.tile(L.euler_freestream(3.0), case.mesh.num_elements * 6) * (1.0 + 0.02 * rng.standard_normal(
        case.mesh.num_elements * 24))
    x = case.ref_coords
    U = solve_hdm(case.law, case.mesh, case.maps, x, mu, U_init=U0, geom=case.geom)
    R0 = assemble_global(case.law, case.mesh, case.maps, U0, x, mu, want_jacobians=False, geom=case.geom)[0]
    R = assemble_global(case.law, case.mesh, case.maps, U, x, mu, want_jacobians=False, geom=case.geom)[0]
    assert np.linalg.norm(R) <= 1e-10 * max(1.0, np.linalg.norm(R0))
    try:
        from oracle import strom_ref

        S = strom_ref.load()
    except ImportError:
        return
    import strom.dg as sdg

    rop = strom_ref.operator(case)  # the reference geometry (12-point rule) for this mesh
    st = sdg.solve_hdm(case.law, rop.geom.mesh, rop.geom.maps, x, mu, U_init=U0)
    assert rel_err(U, st.values) < 1e-8
