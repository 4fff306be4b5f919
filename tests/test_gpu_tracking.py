"""GPU enriched assembly (fullspace.assemble_enriched, dg.py:275-326) and the full-space
tracking / snapshot-alignment problems (tracking.TrackingProblem, tracking.py:41-150) vs
goldens from the unmodified reference (tests/golden/tracking_*.npz) and vs the pinned oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle.dual  # noqa: F401
from oracle.element import OracleGeometry, enriched_blocks

from cases import build, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", ["tracking_q6", "tracking_default"])
def test_assemble_enriched_matches_reference(name):
    from paper_2305_15661_b200.fullspace import assemble_enriched, enriched_records

    case, g = build(name)
    mu = case.mus[0]
    Rb, JU, JX = assemble_enriched(case.law, case.mesh, case.maps, g["U"], g["x"], mu, geom=case.geom)
    ne = case.mesh.num_elements
    assert Rb.shape == (ne * 40,) and JU.shape == (ne * 40, case.maps.n_global_state)
    assert JX.shape == (ne * 40, case.maps.n_global_coord)
    assert rel_err(Rb, g["enr_R"]) < TOL
    assert rel_err(JU @ g["v_u"], g["enr_JU_v"]) < TOL and rel_err(JU.T @ g["u_r"], g["enr_JUt_u"]) < TOL
    assert rel_err(JX @ g["v_x"], g["enr_JX_v"]) < TOL and rel_err(JX.T @ g["u_r"], g["enr_JXt_u"]) < TOL
    assert [JU.nnz, JX.nnz] == g["enr_nnz"].tolist()
    res, js, jn, jc, _, _ = enriched_records(case.law, case.geom, g["U"], g["x"], mu)
    for e in (0, 9, 31):
        tan = g[f"enr_elem{e}_tan"]
        scale = np.max(np.abs(tan))
        assert rel_err(res[e], g[f"enr_elem{e}_res"]) < TOL
        assert rel_err(js[e], tan[:, :24], scale) < TOL
        ok = np.repeat(case.maps.neighbor_map[e].reshape(3, 24)[:, 0] >= 0, 24)
        assert rel_err(jn[e][:, ok], tan[:, 24:96][:, ok], scale) < TOL
        assert rel_err(jc[e], tan[:, 96:], scale) < TOL
    # value-only path: same residual, no Jacobians copied back
    R2, a, b = assemble_enriched(case.law, case.mesh, case.maps, g["U"], g["x"], mu, want_jacobians=False,
                                 geom=case.geom)
    assert a is None and b is None and np.array_equal(R2, Rb)


@pytest.mark.parametrize("flux,wall", [("llf", "slip"), ("roe", "slip"), ("roe", "extrapolate")])
def test_enriched_blocks_match_oracle_roe_wall(flux, wall):
    """The GPU-only extensions (Roe flux, slip wall) through the enriched contraction, against
    the oracle's dual-number blocks on the half-cylinder sector."""
    from paper_2305_15661_b200 import configs, laws as L
    from paper_2305_15661_b200.fullspace import enriched_records

    case = configs.sector_rom_case(n_radial=3, n_circ=5, ku=4, kx=2, frac_active=0.5, rho_scale=2.0, P=1, seed=71,
                                   wall=wall)
    law = L.euler(tags=configs.sector_bcs(wall), flux=flux)
    rng = np.random.default_rng(72)
    ne = case.mesh.num_elements
    U = np.tile(L.euler_freestream(3.0), ne * 6) * (1.0 + 0.03 * rng.standard_normal(ne * 24))
    x = case.ref_coords + 2e-3 * rng.standard_normal(case.ref_coords.size)
    mu = np.array([3.0])
    res, js, jn, jc, _, _ = enriched_records(law, case.geom, U, x, mu)
    geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
    ores, otan = enriched_blocks(law, geom, U, x, mu)
    scale = np.max(np.abs(otan))
    assert rel_err(res, ores) < TOL
    assert rel_err(js, otan[:, :, :24], scale) < TOL and rel_err(jc, otan[:, :, 96:], scale) < TOL
    ok = np.repeat(case.maps.neighbor_map.reshape(ne, 3, 24)[:, :, 0] >= 0, 24, axis=1)
    assert rel_err(jn * ok[:, None, :], otan[:, :, 24:96] * ok[:, None, :], scale) < TOL


def _problem(case, g, kind):
    from paper_2305_15661_b200.configs import DistortionConfig
    from paper_2305_15661_b200.tracking import TrackingProblem

    dist = DistortionConfig(case.kappa, case.eps)
    kw = dict(geom=case.geom)
    if kind == "al":
        return TrackingProblem(case.law, case.mesh, case.maps, case.mus[0], dist, state_basis=g["al_B"],
                               w0=g["al_w0"], x0=g["x"], **kw)
    return TrackingProblem(case.law, case.mesh, case.maps, case.mus[0], dist, U0=g["U"], x0=g["x"],
                           enrich=kind == "fs", **kw)


@pytest.mark.parametrize("kind", ["fs", "fsplain"])
def test_tracking_problem_matches_reference(kind):
    case, g = build("tracking_q6")
    prob = _problem(case, g, kind)
    assert np.array_equal(prob.free, g[f"{kind}_free"])
    w0, z0 = prob.initial_guess()
    assert np.array_equal(z0, g[f"{kind}_z0"]) and prob.nw == g["U"].size and prob.ntau == len(prob.free)
    assert rel_err(prob.objective(w0, z0), g[f"{kind}_obj"]) < TOL
    J, S, T, Hww, Hwt, Htt = prob.derivatives(w0, z0)
    a, b = g[f"{kind}_a"], g[f"{kind}_b"]
    assert rel_err(J, g[f"{kind}_J"]) < TOL and rel_err(S, g[f"{kind}_S"]) < TOL and rel_err(T, g[f"{kind}_T"]) < TOL
    assert rel_err(Hww @ a, g[f"{kind}_Hww_a"]) < TOL and rel_err(Hwt @ b, g[f"{kind}_Hwt_b"]) < TOL
    assert rel_err(Htt @ b, g[f"{kind}_Htt_b"]) < TOL and rel_err(Htt.diagonal(), g[f"{kind}_Htt_diag"]) < TOL


def test_alignment_problem_matches_reference():
    case, g = build("tracking_q6")
    prob = _problem(case, g, "al")
    w0, z0 = prob.initial_guess()
    J, S, T, Hww, Hwt, Htt = prob.derivatives(w0, z0)
    assert rel_err(J, g["al_J"]) < TOL and rel_err(S, g["al_S"]) < TOL and rel_err(T, g["al_T"]) < TOL
    assert rel_err(Hww, g["al_Hww"]) < TOL
    assert rel_err(Hwt @ g["al_b"], g["al_Hwt_b"]) < TOL and rel_err(Htt @ g["al_b"], g["al_Htt_b"]) < TOL


@pytest.mark.parametrize("kind,iters", [("fs", 3), ("al", 4)])
def test_tracking_lm_histories_match_reference(kind, iters):
    """lm.lm_solve (protocol path, GPU-assembled sparse blocks) reproduces the reference
    lm_solve on the reference TrackingProblem: same step lengths and damping row for row."""
    from paper_2305_15661_b200.lm import LmConfig, lm_solve

    case, g = build("tracking_q6")
    res = lm_solve(_problem(case, g, kind), LmConfig(max_iters=iters), w0_mode="keep")
    hist, ref = res.history, g[f"{kind}_lm_hist"]
    assert hist.shape == ref.shape and str(res.reason) == str(g[f"{kind}_lm_reason"])
    assert np.array_equal(hist[:, 0], ref[:, 0]) and np.array_equal(hist[:, 5], ref[:, 5])  # iteration, alpha
    assert rel_err(hist[:, 4], ref[:, 4]) < 1e-9  # lambda
    assert rel_err(hist[:, 1], ref[:, 1]) < 1e-8 and rel_err(hist[:, 2:4], ref[:, 2:4]) < 1e-6
    assert rel_err(res.objective, g[f"{kind}_lm_obj"]) < 1e-8
    assert rel_err(res.w, g[f"{kind}_lm_w"]) < 1e-8
    assert rel_err(res.tau, g[f"{kind}_lm_tau"], scale=max(np.max(np.abs(g[f"{kind}_lm_tau"])), 1e-3)) < 1e-6


def test_reference_lm_runs_on_gpu_tracking_problem():
    """Drop-in: the unmodified reference's lm_solve drives the GPU TrackingProblem (its protocol)
    and lands on the same iterates as the reference problem did."""
    try:
        from oracle import strom_ref

        S = strom_ref.load()
    except ImportError:
        pytest.skip("reference strom not installed")
    case, g = build("tracking_q6")
    res = S["lm"].lm_solve(_problem(case, g, "fs"), S["lm"].LmConfig(max_iters=3), w0_mode="keep")
    assert np.array_equal(res.history[:, 5], g["fs_lm_hist"][:, 5])
    assert rel_err(res.objective, g["fs_lm_obj"]) < 1e-8 and rel_err(res.w, g["fs_lm_w"]) < 1e-8


def test_enriched_mode_argument_errors():
    """C-ABI error behaviour of the enriched mode: no test space bound, more than one
    parameter point, an active set — all rejected with a negative code (RuntimeError here)."""
    from paper_2305_15661_b200 import _lib
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.fullspace import _NoDistortion, test_space_tables
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

    case, g = build("tracking_q6")
    ne = case.mesh.num_elements
    op = GpuReducedOperator(case.law, case.geom, ReducedBases(np.zeros((g["U"].size, 0)), np.zeros((g["x"].size, 0)), g["x"]),
                            _NoDistortion(), state_offset=g["U"])
    rec = 40 * (1 + 24 + 72 + 6) + 7
    out = torch.empty(ne * rec, dtype=torch.float64, device=op.device)
    W = torch.zeros((2, 1), dtype=torch.float64, device=op.device)
    Mu = torch.full((2, 1), 2.0, dtype=torch.float64, device=op.device)
    with pytest.raises(RuntimeError, match="test space not set"):
        op.eval_batched(_lib.ELEMJAC_ENRICHED, W[:1], W[:1], Mu[:1], None, out=out, sync=True)
    phi_t, dphi_t, trace_t = test_space_tables(op.dm.tabs, 3)
    assert phi_t.shape == (12, 10) and dphi_t.shape == (12, 10, 2) and trace_t.shape == (3, 4, 10)
    _lib.check(op._lib.strom_set_test_space(op._h, 10, phi_t.ctypes.data, dphi_t.ctypes.data, trace_t.ctypes.data),
               "set_test_space")
    with pytest.raises(RuntimeError, match="one parameter point"):
        op.eval_batched(_lib.ELEMJAC_ENRICHED, W, W, Mu, None, out=out, sync=True)
    with pytest.raises(RuntimeError, match="all elements"):
        op.eval_batched(_lib.ELEMJAC_ENRICHED, W[:1], W[:1], Mu[:1], WeightVector(np.ones(ne)), out=out, sync=True)
    with pytest.raises(RuntimeError, match="bad arguments"):
        _lib.check(op._lib.strom_set_test_space(op._h, 0, phi_t.ctypes.data, dphi_t.ctypes.data, trace_t.ctypes.data),
                   "set_test_space")
    with pytest.raises(ValueError):
        op.eval_batched(_lib.ELEMJAC_ENRICHED, W[:1], W[:1], Mu[:1], None)  # needs a caller-sized output


# -- the reference's own scalar laws (with sources), p = 1 and 2: the warp kernel's contraction ----
def _scalar_case(name):
    from cases import load
    from paper_2305_15661_b200 import laws as L
    from paper_2305_15661_b200.mesh import build_box_mesh, get_geometry

    g = load(name)
    nx, ny = (int(v) for v in g["nxny"])
    mesh, maps = build_box_mesh(g["box"], nx, ny, degree_sol=int(g["p"]), n_comp=1)
    law = L.burgers_spacetime() if "burgers" in name else L.linear_advection((1.0, 0.5))
    return g, law, mesh, maps, get_geometry(mesh, maps)


SCALAR = ["tracking_burgers_p2", "tracking_burgers_p1", "tracking_linadv_p1"]


@pytest.mark.parametrize("name", SCALAR)
def test_scalar_law_assembly_matches_reference(name):
    """assemble_global / assemble_enriched / assemble_distortion for the reference's scalar laws
    (position-dependent source included) vs the reference's CSR products."""
    from paper_2305_15661_b200.configs import DistortionConfig
    from paper_2305_15661_b200.fullspace import assemble_distortion, assemble_enriched, assemble_global

    g, law, mesh, maps, geom = _scalar_case(name)
    U, x, mu = g["U"], g["x"], g["mu"]
    R, JU, JX = assemble_global(law, mesh, maps, U, x, mu, geom=geom)
    assert rel_err(R, g["glob_R"]) < TOL
    assert rel_err(JU @ g["v_u"], g["glob_JU_v"]) < TOL and rel_err(JU.T @ g["u_r"], g["glob_JUt_u"]) < TOL
    assert rel_err(JX @ g["v_x"], g["glob_JX_v"]) < TOL and rel_err(JX.T @ g["u_r"], g["glob_JXt_u"]) < TOL
    Rb, EU, EX = assemble_enriched(law, mesh, maps, U, x, mu, geom=geom)
    assert rel_err(Rb, g["enr_R"]) < TOL
    assert rel_err(EU @ g["v_u"], g["enr_JU_v"]) < TOL and rel_err(EU.T @ g["u_e"], g["enr_JUt_u"]) < TOL
    assert rel_err(EX @ g["v_x"], g["enr_JX_v"]) < TOL and rel_err(EX.T @ g["u_e"], g["enr_JXt_u"]) < TOL
    N, JN = assemble_distortion(mesh, maps, x, DistortionConfig(1e-3), geom=geom)
    assert rel_err(N, g["dist_N"], max(np.max(np.abs(g["dist_N"])), 1e-12)) < 1e-8  # N = kappa (eta - eta_ref): a difference
    assert rel_err(JN @ g["v_x"], g["dist_JN_v"]) < TOL


@pytest.mark.parametrize("name", ["burgers_st_p1", "burgers_st_p2", "linadv_p1", "linadv_p2", "linadv_ms_p1", "linadv_ms_p2", "strip"])
def test_scalar_element_jacobians_match_reference_goldens(name):
    """fullspace.element_jacobians for the scalar laws vs the reference's elemental_residual
    blocks stored in the round-1 goldens (dg.py:197-225)."""
    from paper_2305_15661_b200.fullspace import element_jacobians

    case, g = build(name)
    U = case.phi @ g["w"] + (case.state_offset if case.state_offset is not None else 0.0)
    x = case.ref_coords + case.psi @ g["tau"]
    res, js, jn, jx = element_jacobians(case.law, case.geom, U, x, case.mus[0])
    elems = sorted({int(k[4:].split("_")[0]) for k in g if k.startswith("elem") and k.endswith("_res")})
    assert elems
    for e in elems:
        scale = np.max(np.abs(g[f"elem{e}_jself"]))
        assert rel_err(res[e], g[f"elem{e}_res"], max(np.max(np.abs(g[f"elem{e}_res"])), 1e-8 * scale)) < 1e-9
        assert rel_err(js[e], g[f"elem{e}_jself"]) < TOL
        assert rel_err(jn[e], g[f"elem{e}_jneigh"], scale) < TOL
        assert rel_err(jx[e], g[f"elem{e}_jcoord"], max(np.max(np.abs(g[f"elem{e}_jcoord"])), 1e-8 * scale)) < 1e-9


@pytest.mark.parametrize("name", SCALAR)
def test_scalar_tracking_lm_matches_reference(name):
    """Full-space tracking of the reference's Burgers / advection problems: Gauss-Newton blocks
    and the lm_solve history row for row against the reference."""
    from paper_2305_15661_b200.configs import DistortionConfig
    from paper_2305_15661_b200.lm import LmConfig, lm_solve
    from paper_2305_15661_b200.tracking import TrackingProblem

    g, law, mesh, maps, geom = _scalar_case(name)
    prob = TrackingProblem(law, mesh, maps, g["mu"], DistortionConfig(1e-3), U0=g["U"], x0=g["x"], geom=geom)
    w0, z0 = prob.initial_guess()
    assert rel_err(prob.objective(w0, z0), g["fs_obj"]) < TOL
    J, S, T, Hww, Hwt, Htt = prob.derivatives(w0, z0)
    assert rel_err(J, g["fs_J"]) < TOL and rel_err(S, g["fs_S"]) < TOL and rel_err(T, g["fs_T"]) < TOL
    assert rel_err(Hww @ g["fs_a"], g["fs_Hww_a"]) < TOL and rel_err(Hwt @ g["fs_b"], g["fs_Hwt_b"]) < TOL
    assert rel_err(Htt @ g["fs_b"], g["fs_Htt_b"]) < TOL
    res = lm_solve(prob, LmConfig(max_iters=3), w0_mode="keep")
    hist, ref = res.history, g["fs_lm_hist"]
    assert hist.shape == ref.shape and str(res.reason) == str(g["fs_lm_reason"])
    assert np.array_equal(hist[:, 5], ref[:, 5]) and rel_err(hist[:, 4], ref[:, 4]) < 1e-8
    assert rel_err(hist[:, 1], ref[:, 1], np.max(np.abs(ref[:, 1]))) < 1e-8
    assert rel_err(res.w, g["fs_lm_w"]) < 1e-7


@pytest.mark.parametrize("kind", ["euler_p1", "strip_p2", "burgers_p1_default"])
def test_warp_kernel_blocks_match_oracle(kind):
    """The warp kernel's element-block contraction on the cases the goldens do not reach: Euler at
    p = 1 (4 components, 3 nodes), the strip law (state-dependent source) and the space-time
    Burgers law (position-dependent source) on the default 2q+2p+1 rule — plain (trial = test)
    and enriched (p + 1) blocks against the oracle's dual-number tangents."""
    from oracle.element import element_eval
    import oracle.dual as D
    from paper_2305_15661_b200 import laws as L
    from paper_2305_15661_b200.fullspace import element_blocks
    from paper_2305_15661_b200.mesh import build_box_mesh, get_geometry

    rng = np.random.default_rng(33)
    if kind == "euler_p1":
        mesh, maps = build_box_mesh(((0.0, 0.0), (1.0, 1.0)), 3, 2, degree_sol=1, n_comp=4)
        law = L.euler(tags={"left": "freestream", "bottom": "freestream", "right": "extrapolate", "top": "extrapolate"})
        U = np.tile(L.euler_freestream(2.5), mesh.num_elements * 3) * (1.0 + 0.03 * rng.standard_normal(mesh.num_elements * 12))
        mu, qo = np.array([2.5]), None
    elif kind == "strip_p2":
        mesh, maps = build_box_mesh(((0.0, 0.0), (1.0, 0.125)), 8, 1, degree_sol=2, n_comp=1)
        law, mu, qo = L.burgers_strip(), np.array([2.0]), None
        U = 0.5 + 0.3 * rng.standard_normal(maps.n_global_state)
    else:
        mesh, maps = build_box_mesh(((0.0, 0.0), (2.0, 1.0)), 3, 2, degree_sol=1, n_comp=1)
        law, mu, qo = L.burgers_spacetime(), np.array([5.0, 0.05]), None
        U = 3.0 + 0.5 * rng.standard_normal(maps.n_global_state)
    geom = get_geometry(mesh, maps, qo)
    x = mesh.nodes.ravel() + 0.01 * rng.standard_normal(mesh.nodes.size) * np.min(np.ptp(mesh.nodes, axis=0)) / 8
    og = OracleGeometry(mesh, maps, qo)
    els = np.arange(mesh.num_elements)
    Ue, Un = og.gather_state(U, els)
    xe = og.gather_coords(x, els)
    nu = og.n_basis * og.n_comp
    T = 4 * nu + 6
    seeds = (D.seed_identity(Ue, 0, T), D.seed_identity(Un, nu, T), D.seed_identity(xe, 4 * nu, T))
    ok = np.repeat(maps.neighbor_map.reshape(len(els), 3, nu)[:, :, 0] >= 0, nu, axis=1)
    for deg in (None, maps.degree_sol + 1):
        out = element_eval(law, og, els, *seeds, mu, test=None if deg is None else og.test_space(deg))
        res, js, jn, jc, _, _ = element_blocks(law, geom, U, x, mu, deg)
        tan = out.res.tan
        scale = np.max(np.abs(tan))
        assert rel_err(res, out.res.val, max(np.max(np.abs(out.res.val)), 1e-6 * scale)) < 1e-9
        assert rel_err(js, tan[:, :, :nu], scale) < TOL and rel_err(jc, tan[:, :, 4 * nu:], scale) < TOL
        assert rel_err(jn * ok[:, None, :], tan[:, :, nu:4 * nu] * ok[:, None, :], scale) < TOL
