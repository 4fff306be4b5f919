"""Oracle restatement of the DG element kernel and the reduced operator.

Follows, line by line in meaning (not in text):
  * per-element tabulations        strom/geometry.py:40-139
  * element_eval                   strom/dg.py:82-181 (incl. the richer test space, dg.py:92-102)
  * Geometry.test_space            strom/geometry.py:162-196
  * assemble_enriched              strom/dg.py:275-326
  * seed_elemental / elemental_residual  strom/dg.py:184-225
  * assemble_global (value path)   strom/dg.py:228-240
  * distortion_integral/_eval      strom/distortion.py:33-68
  * ReducedOperator                strom/reduced.py:116-251
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from dataclasses import dataclass

import numpy as np

from paper_2305_15661_b200.tables import LOCAL_EDGES, interval_rule, lagrange_basis, lagrange_nodes, triangle_rule

from . import dual as D


class DegenerateMappingError(RuntimeError):
    """g <= 0 at a quadrature point (strom/dg.py:26-33)."""

    def __init__(self, elements):
        self.elements = np.atleast_1d(np.asarray(elements))
        super().__init__(f"mapping degeneracy (g <= 0) on elements {self.elements[:8].tolist()}")


class OracleGeometry:
    """Per-element tables, as strom/geometry.py:29-139 builds them."""

    def __init__(self, mesh, maps, quad_order=None):
        self.mesh, self.maps = mesh, maps
        p, q = maps.degree_sol, mesh.degree_geo
        self.quad_order = 2 * q + 2 * p + 1 if quad_order is None else quad_order
        vr, fr = triangle_rule(self.quad_order), interval_rule(self.quad_order)
        self.n_basis = lagrange_nodes(p).shape[0]
        self.n_geo = mesh.elements.shape[1]
        self.n_comp = maps.n_comp
        self.wq = vr.weights
        self.phi, self.dphi = lagrange_basis(p, vr.points)
        self.gphi, self.gdphi = lagrange_basis(q, vr.points)
        s = fr.points
        self.ws = fr.weights
        verts = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
        ns = s.size
        self.phi_face = np.empty((3, ns, self.n_basis))
        self.gphi_face = np.empty((3, ns, self.n_geo))
        self.gdphi_face = np.empty((3, ns, self.n_geo, 2))
        for f, (a, b) in enumerate(LOCAL_EDGES):
            pts = (1.0 - s)[:, None] * verts[a] + s[:, None] * verts[b]
            self.phi_face[f], _ = lagrange_basis(p, pts)
            self.gphi_face[f], self.gdphi_face[f] = lagrange_basis(q, pts)
        opp = np.stack([self.phi_face, self.phi_face[:, ::-1]], axis=1)  # (3, 2, ns, nb)

        v = mesh.vertex_coords()
        jac = np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]], axis=-1)
        det = jac[:, 0, 0] * jac[:, 1, 1] - jac[:, 0, 1] * jac[:, 1, 0]
        inv = np.stack([np.stack([jac[:, 1, 1], -jac[:, 0, 1]], -1),
                        np.stack([-jac[:, 1, 0], jac[:, 0, 0]], -1)], -2) / det[:, None, None]
        self.det_ref, self.inv_jac_ref = det, inv
        self.areas = 0.5 * det
        self.total_area = float(np.sum(self.areas))
        ne = mesh.num_elements
        self.face_normal = np.empty((ne, 3, 2))
        self.face_length = np.empty((ne, 3))
        for f, (a, b) in enumerate(LOCAL_EDGES):
            t = v[:, b] - v[:, a]
            ln = np.hypot(t[:, 0], t[:, 1])
            self.face_length[:, f] = ln
            self.face_normal[:, f, 0] = t[:, 1] / ln
            self.face_normal[:, f, 1] = -t[:, 0] / ln
        dphi0 = np.einsum("qnk,ekj->eqnj", self.dphi, inv)
        self.wdphi0 = dphi0 * (self.wq[None, :, None, None] * det[:, None, None, None])
        self.wphi = self.phi[None] * (self.wq[None, :, None] * det[:, None, None])
        self.wphi_face = self.ws[None, None, :, None] * self.face_length[:, :, None, None] * self.phi_face[None]
        nbr, nface, flip, tag = mesh.neighbor_tables()
        self.nbr_elem, self.face_tag = nbr, tag
        self.phi_opp = opp[np.where(nbr >= 0, nface, 0), flip.astype(np.int64)]
        self.extras = {}

    def test_space(self, degree):
        """Tabulations of a richer nodal test space (strom/geometry.py:162-196): weighted
        reference gradients (ne, nq, n_t, 2), weighted values, weighted face traces."""
        key = ("test_space", degree)
        if key not in self.extras:
            vr, fr = triangle_rule(self.quad_order), interval_rule(self.quad_order)
            phi_t, dphi_t = lagrange_basis(degree, vr.points)
            det = self.det_ref
            wdphi0 = np.einsum("qnk,ekj->eqnj", dphi_t, self.inv_jac_ref) * (self.wq[None, :, None, None] * det[:, None, None, None])
            wphi = phi_t[None] * (self.wq[None, :, None] * det[:, None, None])
            verts = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
            s = fr.points
            face = np.stack([lagrange_basis(degree, (1.0 - s)[:, None] * verts[a] + s[:, None] * verts[b])[0]
                             for a, b in LOCAL_EDGES])
            wphi_face = self.ws[None, None, :, None] * self.face_length[:, :, None, None] * face[None]
            self.extras[key] = EnrichedTabs(degree, phi_t.shape[1], wdphi0, wphi, wphi_face)
        return self.extras[key]

    def gather_state(self, U, els):
        nb, m = self.n_basis, self.n_comp
        U = np.asarray(U)
        Ue = U[self.maps.state_map[els]].reshape(len(els), nb, m)
        idx = self.maps.neighbor_map[els]
        Un = np.where(idx >= 0, U[np.clip(idx, 0, None)], 0.0).reshape(len(els), 3, nb, m)
        return Ue, Un

    def gather_coords(self, x, els):
        return np.asarray(x)[self.maps.coord_map[els]].reshape(len(els), self.n_geo, 2)


@dataclass
class EnrichedTabs:
    degree: int
    n_basis: int
    wdphi0: np.ndarray
    wphi: np.ndarray
    wphi_face: np.ndarray


def _det(G):
    return G[..., 0, 0] * G[..., 1, 1] - G[..., 0, 1] * G[..., 1, 0]


def _adj(G):
    return D.stack([D.stack([G[..., 1, 1], -G[..., 0, 1]], -1),
                    D.stack([-G[..., 1, 0], G[..., 0, 0]], -1)], -2)


@dataclass
class KernelOut:
    res: object
    res_vol: object
    res_face: object


def element_eval(law, geom, els, Ue, Un, xe, mu, check_degenerate=True, test=None):
    """Batched elemental DG residual (strom/dg.py:82-181); ``test`` swaps the test-side
    tabulations for a richer nodal space, the trial side untouched (dg.py:92-102)."""
    els = np.asarray(els)
    B, m, nb = len(els), geom.n_comp, geom.n_basis if test is None else test.n_basis
    wdphi0, wphi, wphi_face = (geom.wdphi0, geom.wphi, geom.wphi_face) if test is None else (
        test.wdphi0, test.wphi, test.wphi_face)
    bad = set()
    # volume (dg.py:105-125)
    Jx = D.einsum("qgj,bgi->bqij", geom.gdphi, xe)
    G = D.einsum("bkj,bqik->bqij", geom.inv_jac_ref[els], Jx)
    g = _det(G)
    if check_degenerate:
        hit = np.any(D.val(g) <= 0.0, axis=1)
        bad.update(els[hit].tolist())
    adj = _adj(G)
    u = D.einsum("qn,bnc->bqc", geom.phi, Ue)
    pos = D.einsum("qg,bgi->bqi", geom.gphi, xe)
    f = law.flux(u, None, mu)
    F = D.einsum("bqci,bqji->bqcj", f, adj)
    S = D.expand(g, 1) * law.source(pos, u, None, mu)
    res_vol = -(D.einsum("bqnj,bqcj->bnc", wdphi0[els], F) + D.einsum("bqn,bqc->bnc", wphi[els], S))
    # faces (dg.py:127-175)
    tag_name = {tid: name for name, tid in geom.mesh.boundary_tags.items()}
    res_face = None
    for fi in range(3):
        GF = D.einsum("bkj,bsik->bsij", geom.inv_jac_ref[els], D.einsum("sgj,bgi->bsij", geom.gdphi_face[fi], xe))
        gF = _det(GF)
        if check_degenerate:
            bad.update(els[np.any(D.val(gF) <= 0.0, axis=1)].tolist())
        ntil = D.einsum("bsji,bj->bsi", _adj(GF), geom.face_normal[els, fi])
        sigma = D.sqrt(ntil[..., 0] ** 2 + ntil[..., 1] ** 2)
        nhat = ntil / D.expand(sigma, 1)
        u_in = D.einsum("sn,bnc->bsc", geom.phi_face[fi], Ue)
        u_out = D.einsum("bsn,bnc->bsc", geom.phi_opp[els, fi], Un[:, fi])
        tags = geom.face_tag[els, fi]
        posF = None
        for tid in np.unique(tags):
            if tid < 0:
                continue
            bc = law.bc(tag_name[int(tid)])
            mask = tags == tid
            if bc.kind == "extrapolate":  # copies value and tangent (dg.py:149-150)
                if isinstance(u_out, D.Dual):
                    u_out.val[mask] = np.broadcast_to(D.val(u_in), u_out.val.shape)[mask]
                    u_out.tan[mask] = np.broadcast_to(u_in.tan, u_out.tan.shape)[mask]
                else:
                    u_out[mask] = D.val(u_in)[mask]
            elif bc.kind == "reflect":  # slip wall (GPU-only extension): u_g = R(nhat) u_in
                refl = reflect_state(u_in, nhat)
                if isinstance(u_out, D.Dual):
                    u_out.val[mask] = np.broadcast_to(D.val(refl), u_out.val.shape)[mask]
                    u_out.tan[mask] = np.broadcast_to(refl.tan, u_out.tan.shape)[mask]
                else:
                    u_out[mask] = D.val(refl)[mask]
            else:  # prescribed ghost at deformed positions, zero tangent (dg.py:151-161)
                if posF is None:
                    posF = D.val(D.einsum("sg,bgi->bsi", geom.gphi_face[fi], xe))
                ghost = np.asarray(bc.value(posF[mask], mu), dtype=float)
                if isinstance(u_out, D.Dual):
                    u_out.val[mask] = ghost
                    u_out.tan[mask] = 0.0
                else:
                    u_out[mask] = ghost
        fn = D.einsum("bsci,bsi->bsc", law.flux(u_in, None, mu), ntil) + D.einsum(
            "bsci,bsi->bsc", law.flux(u_out, None, mu), ntil)
        numflux = getattr(law, "numflux", None)
        if numflux is not None:  # matrix dissipation (Roe, GPU-only extension): H = fn/2 - sigma D/2
            H = 0.5 * fn - 0.5 * D.expand(sigma, 1) * numflux(u_in, u_out, nhat, mu)
        else:
            ws_in, ws_out = law.wavespeed(u_in, nhat, mu), law.wavespeed(u_out, nhat, mu)
            wall = np.isin(tags, [tid for tid in np.unique(tags)
                                  if tid >= 0 and law.bc(tag_name[int(tid)]).kind == "reflect"])
            if np.any(wall):  # ws(R u) = ws(u) exactly in exact arithmetic: use ws_in (no rounding tie)
                if isinstance(ws_out, D.Dual):
                    ws_out.val[wall] = D.val(ws_in)[wall]
                    ws_out.tan[wall] = ws_in.tan[wall]
                else:
                    ws_out[wall] = ws_in[wall]
            lam = D.maximum(ws_in, ws_out)
            H = 0.5 * fn - 0.5 * D.expand(lam * sigma, 1) * (u_out - u_in)
        c = D.einsum("bsn,bsc->bnc", wphi_face[els, fi], H)
        res_face = c if res_face is None else res_face + c
    if bad:
        raise DegenerateMappingError(sorted(bad))
    res_vol = D.reshape(res_vol, (B, nb * m))
    res_face = D.reshape(res_face, (B, nb * m))
    return KernelOut(res_vol + res_face, res_vol, res_face)


def enriched_blocks(law, geom, U, x, mu, test_degree=None):
    """Enriched residual rows and their element tangent blocks [U_e | U_nbr | x_e] over every
    element: the quantities strom/dg.py:275-326 scatters (res (ne, n_t m), tan (ne, n_t m, T))."""
    test = geom.test_space(geom.maps.degree_sol + 1 if test_degree is None else test_degree)
    els = np.arange(geom.mesh.num_elements)
    Ue, Un = geom.gather_state(U, els)
    xe = geom.gather_coords(x, els)
    nu = geom.n_basis * geom.n_comp
    T = 4 * nu + 2 * geom.n_geo
    out = element_eval(law, geom, els, D.seed_identity(Ue, 0, T), D.seed_identity(Un, nu, T),
                       D.seed_identity(xe, 4 * nu, T), mu, test=test)
    return out.res.val, out.res.tan


def reflect_state(u, nhat):
    """Slip-wall ghost of 2-D Euler states: momentum mirrored in the wall, m - 2 (m . n) n."""
    mn = u[..., 1] * nhat[..., 0] + u[..., 2] * nhat[..., 1]
    return D.stack([u[..., 0], u[..., 1] - 2.0 * mn * nhat[..., 0], u[..., 2] - 2.0 * mn * nhat[..., 1], u[..., 3]],
                   axis=-1)


# -- distortion (strom/distortion.py:33-68) -----------------------------------------
def distortion_integral(geom, els, xe, eps):
    Jx = D.einsum("qgj,bgi->bqij", geom.gdphi, xe)
    G = D.einsum("bqik,bkj->bqij", Jx, geom.inv_jac_ref[els])
    g = _det(G)
    fro2 = G[..., 0, 0] ** 2 + G[..., 0, 1] ** 2 + G[..., 1, 0] ** 2 + G[..., 1, 1] ** 2
    ratio = fro2 / D.maximum(g, eps)  # d = 2: exponent 2/d = 1
    weff = geom.wq[None, :] * geom.det_ref[els, None]
    return D.einsum("bq,bq->b", weff, ratio ** 2)


def reference_distortion(geom, eps):
    key = ("eta_ref", float(eps))
    if key not in geom.extras:
        els = np.arange(geom.mesh.num_elements)
        geom.extras[key] = distortion_integral(geom, els, geom.gather_coords(geom.mesh.nodes.ravel(), els), eps)
    return geom.extras[key]


def distortion_eval(geom, els, xe, kappa, eps):
    return kappa * (distortion_integral(geom, els, xe, eps) - reference_distortion(geom, eps)[els])


# -- element-level API (strom/dg.py:184-240) ---------------------------------------------
def elemental_residual(law, geom, elem, Ue, Uneigh, xe, mu, want_jacobians=False):
    nb, m, ng = geom.n_basis, geom.n_comp, geom.n_geo
    nu = nb * m
    Ue = np.asarray(Ue, dtype=float).reshape(1, nb, m)
    Un = np.asarray(Uneigh, dtype=float).reshape(1, 3, nb, m)
    xe = np.asarray(xe, dtype=float).reshape(1, ng, 2)
    els = np.array([elem])
    if not want_jacobians:
        out = element_eval(law, geom, els, Ue, Un, xe, mu)
        return {"res": out.res[0], "res_vol": out.res_vol[0], "res_face": out.res_face[0]}
    T = 4 * nu + 2 * ng
    out = element_eval(law, geom, els, D.seed_identity(Ue, 0, T), D.seed_identity(Un, nu, T),
                       D.seed_identity(xe, 4 * nu, T), mu)
    t = out.res.tan[0]
    return {"res": out.res.val[0], "res_vol": out.res_vol.val[0], "res_face": out.res_face.val[0],
            "jac_self": t[:, :nu].copy(), "jac_neigh": t[:, nu:4 * nu].copy(), "jac_coord": t[:, 4 * nu:].copy()}


def assemble_residual(law, geom, U, x, mu):
    """Global residual vector, element-major (assemble_global value path)."""
    els = np.arange(geom.mesh.num_elements)
    Ue, Un = geom.gather_state(U, els)
    return element_eval(law, geom, els, Ue, Un, geom.gather_coords(x, els), mu).res.reshape(-1)


# -- reduced operator (strom/reduced.py:116-251) -----------------------------------------
class OracleReducedOperator:
    def __init__(self, law, geom, phi, psi, ref_coords, kappa, eps=1e-8, state_offset=None):
        self.law, self.geom = law, geom
        self.u0 = None if state_offset is None else np.asarray(state_offset, dtype=float)
        self.phi = np.asarray(phi, dtype=float).reshape(geom.maps.n_global_state, -1)
        self.psi = np.asarray(psi, dtype=float).reshape(geom.maps.n_global_coord, -1)
        self.X = np.asarray(ref_coords, dtype=float)
        self.kappa, self.eps = kappa, eps
        self.stats = {"kernel_calls": 0, "elements_evaluated": 0}
        maps = geom.maps
        self.phi_e = self.phi[maps.state_map]
        nm = maps.neighbor_map
        self.phi_n = np.where((nm >= 0)[:, :, None], self.phi[np.clip(nm, 0, None)], 0.0)
        self.psi_e = self.psi[maps.coord_map]
        self.X_e = self.X[maps.coord_map]

    @property
    def k_u(self):
        return self.phi.shape[1]

    @property
    def k_x(self):
        return self.psi.shape[1]

    def _batch(self, rho):
        if rho is None:
            return np.arange(self.geom.mesh.num_elements), None
        rho = np.asarray(rho, dtype=float)
        act = np.flatnonzero(rho > 0.0)
        return act, rho[act]

    def _inputs(self, els, w, tau, seeded):
        g = self.geom
        B, nb, m, ng = len(els), g.n_basis, g.n_comp, g.n_geo
        ku, kx = self.k_u, self.k_x
        Ue = (self.phi_e[els] @ w).reshape(B, nb, m)
        Un = (self.phi_n[els] @ w).reshape(B, 3, nb, m)
        if self.u0 is not None:  # affine state offset U = U0 + Phi w (explicit-field driver, SURVEY §8c iv)
            Ue = Ue + self.u0[g.maps.state_map[els]].reshape(B, nb, m)
            nm = g.maps.neighbor_map[els]
            Un = Un + np.where(nm >= 0, self.u0[np.clip(nm, 0, None)], 0.0).reshape(B, 3, nb, m)
        xe = (self.X_e[els] + (self.psi_e[els] @ tau if kx else 0.0)).reshape(B, ng, 2)
        if not seeded:
            return Ue, Un, xe
        T = ku + kx
        tUe = np.zeros((B, nb, m, T)); tUe[..., :ku] = self.phi_e[els].reshape(B, nb, m, ku)
        tUn = np.zeros((B, 3, nb, m, T)); tUn[..., :ku] = self.phi_n[els].reshape(B, 3, nb, m, ku)
        txe = np.zeros((B, ng, 2, T)); txe[..., ku:] = self.psi_e[els].reshape(B, ng, 2, kx)
        return D.Dual(Ue, tUe), D.Dual(Un, tUn), D.Dual(xe, txe)

    def _count(self, els):
        self.stats["kernel_calls"] += 1
        self.stats["elements_evaluated"] += len(els)

    def objective(self, w, tau, mu, rho=None):
        els, wts = self._batch(rho)
        if len(els) == 0:
            return 0.0
        Ue, Un, xe = self._inputs(els, w, tau, False)
        self._count(els)
        out = element_eval(self.law, self.geom, els, Ue, Un, xe, mu)
        N = distortion_eval(self.geom, els, xe, self.kappa, self.eps)
        r2 = np.sum(out.res ** 2, axis=1) + N ** 2
        return 0.5 * float(np.sum(r2) if wts is None else np.dot(wts, r2))

    def _dual(self, w, tau, mu, rho):
        els, wts = self._batch(rho)
        Ue, Un, xe = self._inputs(els, w, tau, True)
        self._count(els)
        out = element_eval(self.law, self.geom, els, Ue, Un, xe, mu)
        N = distortion_eval(self.geom, els, xe, self.kappa, self.eps)
        return (np.ones(len(els)) if wts is None else wts), out, N

    def derivatives(self, w, tau, mu, rho=None):
        ku = self.k_u
        r, out, N = self._dual(w, tau, mu, rho)
        Jw, Jt, dN, R = out.res.tan[:, :, :ku], out.res.tan[:, :, ku:], N.tan[:, ku:], out.res.val
        S = np.einsum("b,bik,bi->k", r, Jw, R)
        T = np.einsum("b,bik,bi->k", r, Jt, R) + np.einsum("b,bk,b->k", r, dN, N.val)
        Hww = np.einsum("b,bik,bil->kl", r, Jw, Jw)
        Hwt = np.einsum("b,bik,bil->kl", r, Jw, Jt)
        Htt = np.einsum("b,bik,bil->kl", r, Jt, Jt) + np.einsum("b,bk,bl->kl", r, dN, dN)
        J = 0.5 * float(np.dot(r, np.sum(R ** 2, axis=1) + N.val ** 2))
        return J, S, T, Hww, Hwt, Htt

    def residuals(self, w, tau, mu, rho=None):
        ku, kx = self.k_u, self.k_x
        if self.geom.mesh.num_elements == 0 or (ku == 0 and kx == 0):
            return np.zeros(ku), np.zeros(kx)
        _, S, T, _, _, _ = self.derivatives(w, tau, mu, rho)
        return S, T

    def elemental_contributions(self, w, tau, mu, split=False):
        ku = self.k_u
        _, out, N = self._dual(w, tau, mu, None)
        Jw, Jt, dN = out.res.tan[:, :, :ku], out.res.tan[:, :, ku:], N.tan[:, ku:]
        if not split:
            return (np.einsum("bik,bi->bk", Jw, out.res.val),
                    np.einsum("bik,bi->bk", Jt, out.res.val) + dN * N.val[:, None])
        return (np.einsum("bik,bi->bk", Jw, out.res_vol.val),
                np.einsum("bik,bi->bk", Jw, out.res_face.val),
                np.einsum("bik,bi->bk", Jt, out.res_vol.val) + dN * N.val[:, None],
                np.einsum("bik,bi->bk", Jt, out.res_face.val))


def elemental_objective(op, w, tau, mu):
    """Per-element 0.5(|R_e|^2 + N_e^2) over all elements (the LP 'output' row of
    config 4; the summand of reduced.py:181-184)."""
    els = np.arange(op.geom.mesh.num_elements)
    Ue, Un, xe = op._inputs(els, w, tau, False)
    out = element_eval(op.law, op.geom, els, Ue, Un, xe, mu)
    N = distortion_eval(op.geom, els, xe, op.kappa, op.eps)
    return 0.5 * (np.sum(out.res ** 2, axis=1) + N ** 2)
