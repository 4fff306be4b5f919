"""Generate golden vectors from the UNMODIFIED reference (run in the dev container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference ``strom`` package read-only and evaluates it on small
seeded cases built by ``paper_2305_15661_b200.configs``; writes one ``.npz``
per case holding the inputs (bases, coordinates, weights, parameters) and
the reference outputs.  Test-side extensions of the reference:
the 12-point degree-6 rule injected into ``strom.quadrature._TRI_RULES``,
laws written against the pluggable dual namespace (Euler, Burgers strip),
the half-cylinder ``ReferenceMesh`` built from its dataclass fields, and an
affine state offset added inside ``ReducedOperator._inputs`` for the
explicit-field cases.  Nothing here is used by the product or on the GPU box.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from strom import dg as sdg  # noqa: E402
from strom import distortion as sdist  # noqa: E402
from strom import dual as sdual  # noqa: E402
from strom import geometry as sgeom  # noqa: E402
from strom import lm as slm  # noqa: E402
from strom import meshing as smesh  # noqa: E402
from strom import quadrature as squad  # noqa: E402
from strom import reduced as sred  # noqa: E402
from strom import conslaw as slaw  # noqa: E402
from strom.eqp import WeightVector  # noqa: E402

from paper_2305_15661_b200 import configs, laws as L, tables  # noqa: E402

L.register_dual_backend(sdual.Dual, sdual)
tables.install_degree6_rule(squad)
OUT = os.environ.get("GOLDEN_OUT", os.path.dirname(os.path.abspath(__file__)))


class OffsetOperator(sred.ReducedOperator):
    """ReducedOperator with U = U0 + Phi w (test-side emulation of the offset)."""

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


def ref_mesh(mesh, maps):
    rm = smesh.ReferenceMesh(dim=2, degree_geo=1, nodes=mesh.nodes.copy(), elements=mesh.elements.copy(),
                             interior_faces=mesh.interior_faces.copy(), boundary_faces=mesh.boundary_faces.copy(),
                             boundary_tags=dict(mesh.boundary_tags))
    rm.validate()
    return rm, smesh.build_assembly_maps(rm, degree_sol=maps.degree_sol, n_comp=maps.n_comp)


def operator(case, law=None):
    rm, rmaps = ref_mesh(case.mesh, case.maps)
    geom = sgeom.Geometry(rm, rmaps, quad_order=case.quad_order)
    # assemble_global / elemental_residual look the geometry up with the default
    # rule key (dg.py:203,234); point that key at the case's rule
    rm._geometry_cache = {(rmaps.degree_sol, rmaps.n_comp, None): geom}
    bases = sred.ReducedBases(case.phi, case.psi, case.ref_coords)
    op = OffsetOperator(law or case.law, geom, bases, sdist.DistortionConfig(case.kappa, case.eps), u0=case.state_offset)
    return op, rm, rmaps, geom


def inputs_of(case, w, tau):
    d = dict(phi=case.phi, psi=case.psi, ref_coords=case.ref_coords, mus=case.mus, w=w, tau=tau,
             rho=case.rho if case.rho is not None else np.zeros(0), quad_order=-1 if case.quad_order is None else case.quad_order,
             kappa=case.kappa, eps=case.eps)
    if case.state_offset is not None:
        d["state_offset"] = case.state_offset
    return d


def evaluate(case, op, geom, w, tau, mu, tag, out, elems=(0,)):
    coords = sred.ReducedCoords(w, tau)
    rho = WeightVector(case.rho) if case.rho is not None else None
    out[f"{tag}obj_all"] = op.objective(coords, mu)
    J, S, T, Hww, Hwt, Htt = op.derivatives(coords, mu)
    out.update({f"{tag}der_all_J": J, f"{tag}der_all_S": S, f"{tag}der_all_T": T, f"{tag}der_all_Hww": Hww,
                f"{tag}der_all_Hwt": Hwt, f"{tag}der_all_Htt": Htt})
    if rho is not None:
        out[f"{tag}obj_rho"] = op.objective(coords, mu, rho)
        J, S, T, Hww, Hwt, Htt = op.derivatives(coords, mu, rho)
        out.update({f"{tag}der_rho_J": J, f"{tag}der_rho_S": S, f"{tag}der_rho_T": T, f"{tag}der_rho_Hww": Hww,
                    f"{tag}der_rho_Hwt": Hwt, f"{tag}der_rho_Htt": Htt})
    for k, v in zip(("Se", "Te"), op.elemental_contributions(coords, mu)):
        out[f"{tag}contrib_{k}"] = v
    for k, v in zip(("Sv", "Sf", "Tv", "Tf"), op.elemental_contributions(coords, mu, split=True)):
        out[f"{tag}split_{k}"] = v
    U, x = sred.reconstruct(op.bases, coords)
    if case.state_offset is not None:
        U = U + case.state_offset
    R, _, _ = sdg.assemble_global(op.law, geom.mesh, geom.maps, U, x, mu, want_jacobians=False)
    out[f"{tag}resid"] = R
    # element-level Jacobian blocks (dg.py:197-225) for the oracle's self-check
    g = geom
    for e in elems:
        Ue, Un = g.gather_state(U, np.array([e]))
        xe = g.gather_coords(x, np.array([e]))
        r = sdg.elemental_residual(op.law, g.mesh, g.maps, e, Ue.ravel(), Un.ravel(), xe.ravel(), mu, want_jacobians=True)
        out[f"{tag}elem{e}_res"] = r.res
        out[f"{tag}elem{e}_jself"] = r.jac_self
        out[f"{tag}elem{e}_jneigh"] = r.jac_neigh
        out[f"{tag}elem{e}_jcoord"] = r.jac_coord


def lm_runs(case, op, mus, out, w0=None, max_iters=30):
    cfg = slm.LmConfig(max_iters=max_iters)
    rho = WeightVector(case.rho) if case.rho is not None else None
    for i, mu in enumerate(mus):
        prob = sred.ReducedTrackingProblem(op, mu, rho=rho, w0=w0)
        res = slm.lm_solve(prob, cfg)
        out[f"lm{i}_w"] = res.w
        out[f"lm{i}_tau"] = res.tau
        out[f"lm{i}_hist"] = res.history
        out[f"lm{i}_conv"] = res.converged
        out[f"lm{i}_obj"] = res.objective
        out[f"lm{i}_iters"] = res.n_iters
        out[f"lm{i}_reason"] = res.reason
    out["lm_max_iters"] = max_iters


def save(name, d):
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **{k: np.asarray(v) for k, v in d.items()})
    print("wrote", path, os.path.getsize(path))


def case_strip():
    case = configs.strip_case(ncell=16, n_active=10, P=3, seed=11, boundary_in_sample=False)
    rng = np.random.default_rng(111)
    w = rng.standard_normal(4) * 3.0
    tau = rng.standard_normal(2) * 1e-2
    op, rm, rmaps, geom = operator(case)
    out = inputs_of(case, w, tau)
    evaluate(case, op, geom, w, tau, case.mus[0], "", out, elems=(0, 5, 31))
    lm_runs(case, op, case.mus[:2], out)
    save("strip", out)


def case_euler_square(quad_order, name):
    case = configs.euler_square_case(n=4, ku=16, kx=8, seed=12, quad_order=quad_order, per_component=False)
    rng = np.random.default_rng(112)
    w = rng.standard_normal(16) * 0.05
    tau = rng.standard_normal(8) * 1e-3
    case.rho = configs.eqp_weights(rng, case.mesh.num_elements, 7, 3.0)
    op, rm, rmaps, geom = operator(case)
    out = inputs_of(case, w, tau)
    evaluate(case, op, geom, w, tau, case.mus[0], "", out, elems=(0, 9, 31))
    save(name, out)


def case_sector():
    case = configs.sector_rom_case(n_radial=4, n_circ=6, ku=6, kx=4, frac_active=0.25, rho_scale=4.0, P=2, seed=13,
                                   wall="extrapolate")
    rng = np.random.default_rng(113)
    w = case.W[0] + rng.standard_normal(6) * 0.02
    tau = rng.standard_normal(4) * 1e-3
    op, rm, rmaps, geom = operator(case)
    out = inputs_of(case, w, tau)
    evaluate(case, op, geom, w, tau, case.mus[0], "", out, elems=(0, 7, 47))
    lm_runs(case, op, case.mus[:2], out, w0=case.W[0], max_iters=15)
    save("sector", out)


def case_reference_law(law, name, p, box, nx, ny, mu, ku, kx, seed):
    from paper_2305_15661_b200.mesh import build_box_mesh

    mesh, maps = build_box_mesh(box, nx, ny, degree_sol=p, n_comp=1)
    rng = np.random.default_rng(seed)
    phi = configs.orthonormal(rng, maps.n_global_state, ku)
    psi = configs.orthonormal(rng, maps.n_global_coord, kx)
    rho = configs.eqp_weights(rng, mesh.num_elements, max(1, mesh.num_elements // 4), 2.0)
    case = configs.Case(name, law, mesh, maps, None, phi, psi, mesh.nodes.ravel().copy(), np.array([mu]),
                        np.zeros((1, ku)), np.zeros((1, kx)), rho)
    w = 1.0 + rng.standard_normal(ku) * 2.0
    tau = rng.standard_normal(kx) * 1e-2
    op, rm, rmaps, geom = operator(case)
    out = inputs_of(case, w, tau)
    out["p"] = p
    out["box"] = np.asarray(box, dtype=float)
    out["nxny"] = np.array([nx, ny])
    evaluate(case, op, geom, w, tau, np.asarray(mu, dtype=float), "", out, elems=(0, 3))
    save(name, out)


def case_degenerate():
    case = configs.euler_square_case(n=4, ku=4, kx=2, seed=14, quad_order=6, per_component=False)
    x = case.ref_coords.reshape(-1, 2).copy()
    node = 1 * 5 + 2  # interior node (i=2, j=1)
    x[node, 0] += 0.6  # pushed across the neighbouring cells -> inverted triangles
    case.ref_coords = x.ravel()
    op, rm, rmaps, geom = operator(case)
    out = inputs_of(case, np.zeros(4), np.zeros(2))
    try:
        op.objective(sred.ReducedCoords(np.zeros(4), np.zeros(2)), case.mus[0])
        raise SystemExit("expected DegenerateMappingError")
    except sdg.DegenerateMappingError as exc:
        out["degenerate_elements"] = exc.elements
    save("degenerate", out)


def case_cfg1():
    """Config 1 exactly as BASELINE states it: 64 cells, 10 EQP elements, 8 mu, full LM solves."""
    case = configs.strip_case()
    op, rm, rmaps, geom = operator(case)
    out = inputs_of(case, case.W[0], case.Tau[0])
    lm_runs(case, op, case.mus, out, max_iters=200)
    save("cfg1", out)


def case_sector_shape(name, n_radial, n_circ, ku, kx, frac, P, seed, max_iters):
    """Config 3 / 5 reduced dimensions (K = 30 / 36, the specialised DMMA kernels) on a reduced
    sector mesh: LM histories of the reference for P mu."""
    case = configs.sector_rom_case(n_radial=n_radial, n_circ=n_circ, ku=ku, kx=kx, frac_active=frac,
                                   rho_scale=1.0 / frac, P=P, seed=seed, wall="extrapolate")
    op, rm, rmaps, geom = operator(case)
    out = inputs_of(case, case.W[0], case.Tau[0])
    out["nrnc"] = np.array([n_radial, n_circ])
    lm_runs(case, op, case.mus, out, w0=case.W[0], max_iters=max_iters)
    save(name, out)


def case_lprows():
    """Config 4 LP rows at (k_u, k_x) = (20, 10): per snapshot s the element contributions
    S_e, T_e (reduced.py:231-251) and 0.5 (|R_e|^2 + N_e^2) at explicit (U_s, x_s)."""
    case = configs.sector_rom_case(n_radial=6, n_circ=10, ku=20, kx=10, frac_active=0.2, rho_scale=5.0, P=2, seed=41,
                                   wall="extrapolate")
    mus, U, X = configs.snapshot_fields(case, 3, seed=42)
    ne = case.mesh.num_elements
    out = inputs_of(case, np.zeros(20), np.zeros(10))
    out.update(snap_mus=mus, snap_U=U, snap_X=X)
    rows = np.zeros((3, 31, ne))
    for s in range(3):
        case.state_offset, case.ref_coords = U[s], X[s]
        op, rm, rmaps, geom = operator(case)
        c = sred.ReducedCoords(np.zeros(20), np.zeros(10))
        Se, Te = op.elemental_contributions(c, mus[s])
        rows[s, :20], rows[s, 20:30] = Se.T, Te.T
        for e in range(ne):  # the element objective: the weighted objective at a one-hot weight
            wv = np.zeros(ne)
            wv[e] = 1.0
            rows[s, 30, e] = op.objective(c, mus[s], WeightVector(wv))
    out["lprows"] = rows
    save("lprows", out)


def case_tracking(quad_order, name, with_problem):
    """Full-space assembly against the enriched (degree p+1) test space (dg.py:275-326) and the
    full-space tracking / snapshot-alignment problems on top (tracking.py:41-150), from the
    reference: residuals, element tangent blocks, products of the CSR Jacobians and of the
    Gauss-Newton blocks with seeded vectors, and a short reference lm_solve history."""
    from strom import tracking as strack

    case = configs.euler_square_case(n=4, ku=16, kx=8, seed=61, quad_order=quad_order)
    case.law = L.euler(tags={"left": "freestream", "bottom": "freestream", "right": "extrapolate", "top": "extrapolate"})
    op, rm, rmaps, geom = operator(case)
    rng = np.random.default_rng(161)
    mu = case.mus[0]
    U = case.state_offset + case.phi @ (rng.standard_normal(16) * 0.05)
    x = case.ref_coords.copy()
    out = inputs_of(case, np.zeros(16), np.zeros(8))
    out.update(U=U, x=x)
    Rb, JU, JX = sdg.assemble_enriched(case.law, rm, rmaps, U, x, mu)
    v_u, v_x, u_r = rng.standard_normal(JU.shape[1]), rng.standard_normal(JX.shape[1]), rng.standard_normal(JU.shape[0])
    out.update(enr_R=Rb, v_u=v_u, v_x=v_x, u_r=u_r, enr_JU_v=JU @ v_u, enr_JUt_u=JU.T @ u_r, enr_JX_v=JX @ v_x,
               enr_JXt_u=JX.T @ u_r, enr_nnz=np.array([JU.nnz, JX.nnz]))
    test = geom.test_space(rmaps.degree_sol + 1)
    for e in (0, 9, 31):  # element tangent blocks [U_e | U_nbr | x_e] of the enriched rows
        els = np.array([e])
        Ue, Un = geom.gather_state(U, els)
        xe = geom.gather_coords(x, els)
        o = sdg.element_eval(case.law, geom, els, *sdg.seed_elemental(geom, Ue, Un, xe), mu, test=test)
        out[f"enr_elem{e}_res"] = o.res.val[0]
        out[f"enr_elem{e}_tan"] = o.res.tan[0]
    if with_problem:
        dist = sdist.DistortionConfig(case.kappa, case.eps)
        X = rm.nodes.ravel()
        for tag, enrich in (("fs", True), ("fsplain", False)):
            prob = strack.TrackingProblem(case.law, rm, rmaps, mu, dist, U0=U, x0=x, enrich=enrich)
            w0, z0 = prob.initial_guess()
            J, S, T, Hww, Hwt, Htt = prob.derivatives(w0, z0)
            a, b = rng.standard_normal(len(w0)), rng.standard_normal(len(z0))
            out.update({f"{tag}_free": prob.free, f"{tag}_z0": z0, f"{tag}_obj": prob.objective(w0, z0), f"{tag}_J": J,
                        f"{tag}_S": S, f"{tag}_T": T, f"{tag}_a": a, f"{tag}_b": b, f"{tag}_Hww_a": Hww @ a,
                        f"{tag}_Hwt_b": Hwt @ b, f"{tag}_Htt_b": Htt @ b, f"{tag}_Htt_diag": Htt.diagonal()})
        # snapshot alignment: a small state basis holding the state, full-dimensional deformation
        B = np.linalg.qr(np.column_stack([U, case.phi[:, :3]]))[0]
        wB = B.T @ U + rng.standard_normal(4) * 1e-3
        prob = strack.TrackingProblem(case.law, rm, rmaps, mu, dist, state_basis=B, w0=wB, x0=x)
        w0, z0 = prob.initial_guess()
        J, S, T, Hww, Hwt, Htt = prob.derivatives(w0, z0)
        b = rng.standard_normal(len(z0))
        out.update(al_B=B, al_w0=w0, al_J=J, al_S=S, al_T=T, al_Hww=Hww, al_Hwt_b=Hwt @ b, al_Htt_b=Htt @ b, al_b=b)
        res = slm.lm_solve(prob, slm.LmConfig(max_iters=4), w0_mode="keep")
        out.update(al_lm_w=res.w, al_lm_tau=res.tau, al_lm_hist=res.history, al_lm_obj=res.objective,
                   al_lm_reason=res.reason)
        # full-space tracking: three LM iterations of the reference solver on the enriched objective
        prob = strack.TrackingProblem(case.law, rm, rmaps, mu, dist, U0=U, x0=x)
        res = slm.lm_solve(prob, slm.LmConfig(max_iters=3), w0_mode="keep")
        out.update(fs_lm_w=res.w, fs_lm_tau=res.tau, fs_lm_hist=res.history, fs_lm_obj=res.objective,
                   fs_lm_reason=res.reason)
    save(name, out)


def case_tracking_scalar(name, law, p, box, nx, ny, mu, seed):
    """The reference's own scalar laws through the full-space path: assemble_global Jacobian
    products, assemble_enriched (dg.py:275-326) and the full-space TrackingProblem with a
    short lm_solve history (tracking.py:41-150)."""
    from strom import tracking as strack

    from paper_2305_15661_b200.mesh import build_box_mesh

    mesh, maps = build_box_mesh(box, nx, ny, degree_sol=p, n_comp=1)
    rm, rmaps = ref_mesh(mesh, maps)
    rng = np.random.default_rng(seed)
    mu = np.asarray(mu, dtype=float)
    X = rm.nodes.ravel()
    z = 0.02 * min((box[1][0] - box[0][0]) / nx, (box[1][1] - box[0][1]) / ny) * rng.standard_normal(X.size)
    free = strack.boundary_slide_dofs(rm)
    x = X.copy()
    x[free] += z[free]
    U = sdg.initial_state(law, rm, rmaps, x, mu) * (1.0 + 0.02 * rng.standard_normal(rmaps.n_global_state))
    out = dict(p=p, box=np.asarray(box, dtype=float), nxny=np.array([nx, ny]), mu=mu, U=U, x=x)
    R, JU, JX = sdg.assemble_global(law, rm, rmaps, U, x, mu)
    Rb, EU, EX = sdg.assemble_enriched(law, rm, rmaps, U, x, mu)
    v_u, v_x = rng.standard_normal(JU.shape[1]), rng.standard_normal(JX.shape[1])
    u_r, u_e = rng.standard_normal(JU.shape[0]), rng.standard_normal(EU.shape[0])
    out.update(v_u=v_u, v_x=v_x, u_r=u_r, u_e=u_e, glob_R=R, glob_JU_v=JU @ v_u, glob_JUt_u=JU.T @ u_r,
               glob_JX_v=JX @ v_x, glob_JXt_u=JX.T @ u_r, enr_R=Rb, enr_JU_v=EU @ v_u, enr_JUt_u=EU.T @ u_e,
               enr_JX_v=EX @ v_x, enr_JXt_u=EX.T @ u_e)
    dist = sdist.DistortionConfig(1e-3)
    N, JN = sdist.assemble_distortion(rm, rmaps, x, dist)
    out.update(dist_N=N, dist_JN_v=JN @ v_x)
    prob = strack.TrackingProblem(law, rm, rmaps, mu, dist, U0=U, x0=x)
    w0, z0 = prob.initial_guess()
    J, S, T, Hww, Hwt, Htt = prob.derivatives(w0, z0)
    a, b = rng.standard_normal(len(w0)), rng.standard_normal(len(z0))
    out.update(fs_obj=prob.objective(w0, z0), fs_J=J, fs_S=S, fs_T=T, fs_a=a, fs_b=b, fs_Hww_a=Hww @ a,
               fs_Hwt_b=Hwt @ b, fs_Htt_b=Htt @ b)
    res = slm.lm_solve(prob, slm.LmConfig(max_iters=3), w0_mode="keep")
    out.update(fs_lm_w=res.w, fs_lm_tau=res.tau, fs_lm_hist=res.history, fs_lm_obj=res.objective,
               fs_lm_reason=res.reason)
    save(name, out)


if __name__ == "__main__":
    case_strip()
    case_euler_square(6, "euler_square_q6")
    case_euler_square(None, "euler_square_default")
    case_sector()
    case_reference_law(slaw.burgers_spacetime(), "burgers_st_p1", 1, ((0.0, 0.0), (2.0, 1.0)), 5, 3, (5.0, 0.05), 5, 3, 15)
    case_reference_law(slaw.burgers_spacetime(), "burgers_st_p2", 2, ((0.0, 0.0), (2.0, 1.0)), 4, 3, (4.0, 0.03), 6, 3, 16)
    case_reference_law(slaw.linear_advection((1.0, 0.5)), "linadv_p2", 2, ((0.0, 0.0), (1.0, 1.0)), 3, 3, (0.5,), 5, 3, 17)
    case_reference_law(slaw.linear_advection((-0.7, 1.0)), "linadv_p1", 1, ((0.0, 0.0), (1.0, 1.0)), 4, 2, (0.5,), 4, 2, 18)
    # the verification law with a manufactured solution (position-dependent source and inflow ghosts)
    ms = L.ExpManufactured()
    case_reference_law(slaw.linear_advection((1.0, 0.5), manufactured=(ms.u, ms.grad)), "linadv_ms_p2", 2,
                       ((0.0, 0.0), (1.0, 1.0)), 3, 3, (0.5,), 5, 3, 19)
    case_reference_law(slaw.linear_advection((-0.7, 1.0), manufactured=(ms.u, ms.grad)), "linadv_ms_p1", 1,
                       ((0.0, 0.0), (1.0, 1.0)), 4, 2, (0.5,), 4, 2, 20)
    case_degenerate()
    case_cfg1()
    case_sector_shape("sector_k30", 6, 12, 20, 10, 0.25, 4, 51, 30)
    case_sector_shape("sector_k36", 6, 12, 24, 12, 0.25, 3, 52, 15)
    case_lprows()
    case_tracking(6, "tracking_q6", True)
    case_tracking(None, "tracking_default", False)
    case_tracking_scalar("tracking_burgers_p2", slaw.burgers_spacetime(), 2, ((0.0, 0.0), (2.0, 1.0)), 4, 3, (5.0, 0.05), 171)
    case_tracking_scalar("tracking_burgers_p1", slaw.burgers_spacetime(), 1, ((0.0, 0.0), (2.0, 1.0)), 5, 3, (4.0, 0.03), 172)
    case_tracking_scalar("tracking_linadv_p1", slaw.linear_advection((1.0, 0.5)), 1, ((0.0, 0.0), (1.0, 1.0)), 3, 3, (0.5,), 173)
