"""Pin the CPU oracle against golden vectors from the unmodified reference."""

import numpy as np
import pytest

import oracle.dual  # noqa: F401  (registers the oracle dual backend for the laws)
from oracle.element import (DegenerateMappingError, OracleGeometry, OracleReducedOperator, assemble_residual,
                            elemental_residual)
from oracle.lm import LmConfig, OracleProblem, lm_solve

from cases import EVAL_CASES, build, rel_err

TOL = 1e-12


def oracle_op(case):
    geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
    return OracleReducedOperator(case.law, geom, case.phi, case.psi, case.ref_coords, case.kappa, case.eps,
                                 state_offset=case.state_offset), geom


@pytest.mark.parametrize("name", EVAL_CASES)
def test_oracle_matches_reference(name):
    case, g = build(name)
    op, geom = oracle_op(case)
    w, tau, mu = g["w"], g["tau"], case.mus[0]
    assert rel_err(op.objective(w, tau, mu), g["obj_all"]) < TOL
    J, S, T, Hww, Hwt, Htt = op.derivatives(w, tau, mu)
    for k, v in dict(J=J, S=S, T=T, Hww=Hww, Hwt=Hwt, Htt=Htt).items():
        assert rel_err(v, g[f"der_all_{k}"]) < TOL, k
    if case.rho is not None:
        assert rel_err(op.objective(w, tau, mu, case.rho), g["obj_rho"]) < TOL
        J, S, T, Hww, Hwt, Htt = op.derivatives(w, tau, mu, case.rho)
        for k, v in dict(J=J, S=S, T=T, Hww=Hww, Hwt=Hwt, Htt=Htt).items():
            assert rel_err(v, g[f"der_rho_{k}"]) < TOL, k
    for k, v in zip(("Se", "Te"), op.elemental_contributions(w, tau, mu)):
        assert rel_err(v, g[f"contrib_{k}"]) < TOL, k
    for k, v in zip(("Sv", "Sf", "Tv", "Tf"), op.elemental_contributions(w, tau, mu, split=True)):
        assert rel_err(v, g[f"split_{k}"]) < TOL, k
    U = op.phi @ w + (case.state_offset if case.state_offset is not None else 0.0)
    x = case.ref_coords + op.psi @ tau
    assert rel_err(assemble_residual(case.law, geom, U, x, mu), g["resid"]) < TOL
    for key in g:
        if key.startswith("elem") and key.endswith("_res"):
            e = int(key[4:-4])
            Ue, Un = geom.gather_state(U, np.array([e]))
            xe = geom.gather_coords(x, np.array([e]))
            r = elemental_residual(case.law, geom, e, Ue, Un, xe, mu, want_jacobians=True)
            assert rel_err(r["res"], g[key]) < TOL
            for blk in ("jself", "jneigh", "jcoord"):
                ref = g[f"elem{e}_{blk}"]
                mine = r[{"jself": "jac_self", "jneigh": "jac_neigh", "jcoord": "jac_coord"}[blk]]
                assert rel_err(mine, ref) < 1e-11, blk


@pytest.mark.parametrize("name", ["tracking_q6", "tracking_default"])
def test_oracle_enriched_matches_reference(name):
    """The oracle's enriched (degree p+1 test space) element blocks vs the reference's
    assemble_enriched (dg.py:275-326): residual, element tangents, CSR products."""
    from oracle.element import enriched_blocks

    case, g = build(name)
    geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
    res, tan = enriched_blocks(case.law, geom, g["U"], g["x"], case.mus[0])
    assert rel_err(res.reshape(-1), g["enr_R"]) < TOL
    for e in (0, 9, 31):
        assert rel_err(res[e], g[f"enr_elem{e}_res"]) < TOL
        assert rel_err(tan[e], g[f"enr_elem{e}_tan"]) < 1e-11
    # products of the assembled Jacobians with the stored vectors, from the element blocks
    maps, (ne, nt) = case.maps, res.shape
    Jv, Jx = np.zeros(ne * nt), np.zeros(ne * nt)
    for e in range(ne):
        ok = maps.neighbor_map[e] >= 0
        rows = slice(e * nt, (e + 1) * nt)
        Jv[rows] = tan[e][:, :24] @ g["v_u"][maps.state_map[e]] + tan[e][:, 24:96][:, ok] @ g["v_u"][maps.neighbor_map[e][ok]]
        Jx[rows] = tan[e][:, 96:] @ g["v_x"][maps.coord_map[e]]
    assert rel_err(Jv, g["enr_JU_v"]) < 1e-11 and rel_err(Jx, g["enr_JX_v"]) < 1e-11


def test_oracle_degenerate_elements():
    case, g = build("degenerate")
    op, _ = oracle_op(case)
    with pytest.raises(DegenerateMappingError) as ei:
        op.objective(np.zeros(4), np.zeros(2), case.mus[0])
    assert np.array_equal(np.asarray(ei.value.elements), g["degenerate_elements"])


@pytest.mark.parametrize("name", ["strip", "sector"])
def test_oracle_lm_matches_reference(name):
    case, g = build(name)
    op, _ = oracle_op(case)
    cfg = LmConfig(max_iters=int(g["lm_max_iters"]))
    w0 = case.W[0] if name == "sector" else None
    for i in range(2):
        key = f"lm{i}_w"
        if key not in g:
            continue
        res = lm_solve(OracleProblem(op, case.mus[i], rho=case.rho, w0=w0), cfg)
        assert bool(res.converged) == bool(g[f"lm{i}_conv"])
        assert res.n_iters == int(g[f"lm{i}_iters"])
        assert str(res.reason) == str(g[f"lm{i}_reason"])
        assert rel_err(res.w, g[f"lm{i}_w"]) < 1e-9
        assert rel_err(res.tau, g[f"lm{i}_tau"], scale=max(1.0, np.max(np.abs(g[f"lm{i}_tau"])))) < 1e-9
        h, hr = res.history, g[f"lm{i}_hist"]
        assert h.shape == hr.shape
        assert np.allclose(h[:, [0, 4, 5]], hr[:, [0, 4, 5]], rtol=1e-8, atol=0, equal_nan=True)
