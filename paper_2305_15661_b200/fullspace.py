"""Full-space assembly on the GPU: ``assemble_global`` with the sparse
Jacobians dR/dU and dR/dx (strom/dg.py:228-272), ``assemble_distortion``
(distortion.py:71-92) and the HDM Newton / PTC solve ``solve_hdm`` (dg.py:343-400) on top.

The element blocks — residual, dR_e/dU_e, dR_e/dU_nbr and dR_e/dx_e, i.e. what
``elemental_residual(..., want_jacobians=True)`` returns (dg.py:197-225) — come from the K1
element kernel in its STROM_ELEMJAC mode (the same local Jacobians the reduced path projects,
written out instead of projected); the scatter into CSR uses the reference's own index
construction.  ``assemble_enriched`` (dg.py:275-326) tests the same weak form against the
degree p+1 nodal space: K1's STROM_ELEMJAC_ENRICHED mode contracts its pointwise flux /
Jacobian records with the test tabulations bound by ``strom_set_test_space``; with the trial
space bound as the test space the same mode gives the plain blocks for every compiled law and
degree (the scalar laws with their sources, Euler at p = 1).  Full-space tracking on top:
``tracking.py``.
"""

import numpy as np
import scipy.sparse as sp

from . import _lib
from .reduced import EJ_SIZE, GpuReducedOperator, ReducedBases


class _NoDistortion:
    kappa, eps = 1.0, 1e-8


def test_space_tables(tabs, degree):
    """Values (nq, n_test), reference gradients (nq, n_test, 2) and face traces (3, ns, n_test)
    of the degree ``degree`` nodal basis at the element tables' volume / face points
    (geometry.py:162-196)."""
    from .tables import LOCAL_EDGES, lagrange_basis, triangle_rule

    verts = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    phi_t, dphi_t = lagrange_basis(degree, triangle_rule(tabs.quad_order).points)
    s = np.asarray(tabs.s)
    trace_t = np.stack([lagrange_basis(degree, (1.0 - s)[:, None] * verts[a] + s[:, None] * verts[b])[0]
                        for a, b in LOCAL_EDGES])
    return np.ascontiguousarray(phi_t), np.ascontiguousarray(dphi_t), np.ascontiguousarray(trace_t)


def _element_records(law, geom, U, x, mu, dist=None, device=None, raise_degenerate=True, test_degree=None,
                     columns=None, on_device=False):
    """Element records at the global state U and coordinates x: (ne, EJ_SIZE) STROM_ELEMJAC
    records (4-component laws, p = 2), or with ``test_degree`` the STROM_ELEMJAC_ENRICHED records
    (ne, NT (1 + 4 n_u + 6) + 7) for any compiled law and degree.  ``columns`` limits what is
    copied back to the host."""
    import torch

    mesh, maps = geom.mesh, geom.maps
    if test_degree is None and (maps.n_comp != 4 or maps.degree_sol != 2):
        raise NotImplementedError("STROM_ELEMJAC records: 4-component laws with p = 2 (pass test_degree)")
    U = np.asarray(U, dtype=float).reshape(-1)
    x = np.asarray(x, dtype=float).reshape(-1)
    # one operator per (geometry, law, distortion constants, device): later calls only refresh the
    # state and coordinate vectors in place (an LM tracking solve evaluates dozens of times)
    d = dist or _NoDistortion()
    cache = geom.__dict__.setdefault("_b200_fullspace_ops", {})
    key = (id(law), float(d.kappa), float(d.eps), str(device))
    op = cache.get(key)
    if op is None or op.law is not law:
        bases = ReducedBases(np.zeros((U.size, 0)), np.zeros((x.size, 0)), x)
        op = cache[key] = GpuReducedOperator(law, geom, bases, d, device=device, state_offset=U)
        op._test_degree = None
    else:
        op.u0.copy_(torch.as_tensor(U))
        op.ref_coords.copy_(torch.as_tensor(x))
    W = torch.zeros((1, op.k_u), dtype=torch.float64, device=op.device)
    Tau = torch.zeros((1, 1), dtype=torch.float64, device=op.device)
    Mu = torch.as_tensor(op._mu(mu)[None]).to(op.device)
    mode, rec = _lib.ELEMJAC, EJ_SIZE
    if test_degree is not None:
        from .tables import lagrange_nodes

        nbt = lagrange_nodes(test_degree).shape[0]
        if op._test_degree != test_degree:
            phi_t, dphi_t, trace_t = test_space_tables(op.dm.tabs, test_degree)
            _lib.check(op._lib.strom_set_test_space(op._h, nbt, phi_t.ctypes.data, dphi_t.ctypes.data,
                                                    trace_t.ctypes.data), "strom_set_test_space")
            op._test_degree = test_degree
        nu = op.dm.nu
        mode, rec = _lib.ELEMJAC_ENRICHED, maps.n_comp * nbt * (1 + 4 * nu + 6) + 7
    out = torch.empty(mesh.num_elements * rec, dtype=torch.float64, device=op.device)
    out, rc = op.eval_batched(mode, W, Tau, Mu, None, out=out, sync=True)
    if rc == 1 and raise_degenerate:  # g <= 0 somewhere: raised after the whole batch, as dg.py:177-178
        from .reduced import degenerate_error

        n = op._lib.strom_degenerate_elements(op._h, 0, None, 0)
        ids = np.zeros(max(n, 1), dtype=np.int32)
        op._lib.strom_degenerate_elements(op._h, 0, ids.ctypes.data, n)
        raise degenerate_error(ids[:n].astype(np.int64))
    out = out.view(mesh.num_elements, rec)
    if on_device:
        return out
    return (out if columns is None else out[:, columns].contiguous()).cpu().numpy()


def element_blocks(law, geom, U, x, mu, test_degree=None, dist=None, want_jacobians=True, device=None,
                   raise_degenerate=True):
    """Element blocks of the DG residual in one K1 pass over the mesh:
    (res (ne, NT), dR/dU_e (ne, NT, n_u), dR/dU_nbr (ne, NT, 3 n_u), dR/dx_e (ne, NT, 6), N (ne,),
    dN/dx_e (ne, 6)) — what ``elemental_residual(..., want_jacobians=True)`` returns per element
    (dg.py:197-225) plus the distortion residual and its gradient (distortion.py:53-68).
    ``test_degree`` None: the trial space tests the residual (NT = n_u); otherwise the nodal
    space of that degree (``assemble_enriched``: p + 1).  The Jacobian blocks are None (and never
    copied back) when ``want_jacobians`` is false."""
    from .tables import lagrange_nodes

    maps = geom.maps
    m, p = maps.n_comp, maps.degree_sol
    nu = lagrange_nodes(p).shape[0] * m
    if test_degree is None and m == 4 and p == 2:  # the DMMA local-Jacobian path (STROM_ELEMJAC)
        cols = None if want_jacobians else np.r_[0:24, 2472:2479]
        o = _element_records(law, geom, U, x, mu, dist=dist, device=device, raise_degenerate=raise_degenerate,
                             columns=cols)
        if not want_jacobians:
            return o[:, :24], None, None, None, o[:, 24], o[:, 25:]
        return (o[:, :24], o[:, 24:600].reshape(-1, 24, 24), o[:, 600:2328].reshape(-1, 24, 72),
                o[:, 2328:2472].reshape(-1, 24, 6), o[:, 2472], o[:, 2473:2479])
    deg = p if test_degree is None else test_degree
    NT = lagrange_nodes(deg).shape[0] * m
    rec = NT * (1 + 4 * nu + 6)
    if not want_jacobians:  # residual rows and the distortion scalar only
        cols = np.r_[0:NT, rec:rec + 7]
        o = _element_records(law, geom, U, x, mu, dist=dist, device=device, raise_degenerate=raise_degenerate,
                             test_degree=deg, columns=cols)
        return o[:, :NT], None, None, None, o[:, NT], o[:, NT + 1:]
    o = _element_records(law, geom, U, x, mu, dist=dist, device=device, raise_degenerate=raise_degenerate,
                         test_degree=deg)
    a, b, c = NT, NT + NT * nu, NT + NT * 4 * nu
    return (o[:, :a], o[:, a:b].reshape(-1, NT, nu), o[:, b:c].reshape(-1, NT, 3 * nu), o[:, c:rec].reshape(-1, NT, 6),
            o[:, rec], o[:, rec + 1:rec + 7])


def element_jacobians(law, geom, U, x, mu, device=None):
    """(res (ne, n_u), jac_self (ne, n_u, n_u), jac_neigh (ne, n_u, 3 n_u), jac_coord (ne, n_u, 6)) at
    the global state U and coordinates x (dg.py:197-225, batched over all elements)."""
    return element_blocks(law, geom, U, x, mu, device=device)[:4]


def _any_law(mesh, maps):
    """A compiled law with the mesh's component count whose boundaries all extrapolate (the
    distortion residual does not depend on the law or the state) and an admissible state."""
    import dataclasses

    from . import laws as L

    tags = {t: L.BoundaryCondition("extrapolate") for t in mesh.boundary_tags}
    if maps.n_comp == 4:
        return L.euler(tags={t: "extrapolate" for t in mesh.boundary_tags}), L.euler_freestream(2.0)
    if maps.n_comp == 1:
        return dataclasses.replace(L.linear_advection(), boundary_data=tags), np.ones(1)
    raise NotImplementedError(f"no compiled law with {maps.n_comp} components")


def assemble_distortion(mesh, maps, x, config, want_jacobian=True, geom=None, device=None):
    """Elemental distortion residuals N (ne,) and the CSR gradient dN/dx (ne, N_x):
    strom/distortion.py:71-92 (never raises: eps floors the Jacobian determinant)."""
    from .mesh import get_geometry

    geom = geom or get_geometry(mesh, maps)
    law, u1 = _any_law(mesh, maps)
    nb = maps.state_map.shape[1] // maps.n_comp
    U = np.tile(u1, mesh.num_elements * nb)  # the state does not enter N
    _, _, _, _, N, dN = element_blocks(law, geom, U, x, np.array([2.0]), dist=config, want_jacobians=False,
                                       device=device, raise_degenerate=False)
    N = N.copy()
    if not want_jacobian:
        return N, None
    rows = np.repeat(np.arange(mesh.num_elements), 6)
    jac = sp.coo_matrix((dN.ravel(), (rows, maps.coord_map.ravel())),
                        shape=(mesh.num_elements, maps.n_global_coord)).tocsr()
    return N, jac


def assemble_global(law, mesh, maps, U, x, mu, want_jacobians=True, geom=None, device=None):
    """Residual and CSR Jacobians dR/dU (N_u x N_u), dR/dx (N_u x N_x): strom/dg.py:228-272."""
    from .mesh import get_geometry

    geom = geom or get_geometry(mesh, maps)
    if not want_jacobians:  # residual rows only (the same cached operator, nothing but the rows copied back)
        return element_blocks(law, geom, U, x, mu, want_jacobians=False, device=device)[0].reshape(-1).copy(), None, None
    res, dRdU, dRdx, _, _ = assemble_blocks_csr(law, geom, U, x, mu, None, device=device, rows=maps.state_map)
    return res.reshape(-1).copy(), dRdU, dRdx


def _csr_pattern(r, c, shape):
    """Sorted, duplicate-free CSR structure of the COO coordinates (r, c): (order, starts,
    indptr, indices) with data_csr = add.reduceat(data_coo[order], starts) — what
    ``coo_matrix(...).tocsr()`` computes, with the sort done once per mesh."""
    key = r.astype(np.int64) * shape[1] + c
    order = np.argsort(key, kind="stable")
    ks = key[order]
    first = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    rows = (ks[first] // shape[1]).astype(np.int64)
    indices = (ks[first] % shape[1]).astype(np.int32)
    indptr = np.zeros(shape[0] + 1, dtype=np.int32)
    np.cumsum(np.bincount(rows, minlength=shape[0]), out=indptr[1:])
    return order, first, indptr, indices


def _scatter_csr(maps, rows, jac_self, jac_neigh, jac_coord, n_rows):
    """CSR dR/dU and dR/dx from element blocks: the index construction of dg.py:246-271 (self and
    neighbor blocks concatenated, entries of missing neighbors masked to zero at column 0,
    duplicates summed); the sorted structure is cached on ``maps`` per block shape."""
    cache = maps.__dict__.setdefault("_b200_csr_patterns", {})
    ck = (jac_self.shape, n_rows, int(rows[0, 0, 0]), int(rows[-1, -1, 0]))
    nmap = maps.neighbor_map
    valid = nmap >= 0
    if ck not in cache:
        r1 = np.broadcast_to(rows, jac_self.shape).ravel()
        c1 = np.broadcast_to(maps.state_map[:, None, :], jac_self.shape).ravel()
        r2 = np.broadcast_to(rows, jac_neigh.shape).ravel()
        c2 = np.broadcast_to(np.clip(nmap, 0, None)[:, None, :], jac_neigh.shape).ravel()
        r3 = np.broadcast_to(rows, jac_coord.shape).ravel()
        c3 = np.broadcast_to(maps.coord_map[:, None, :], jac_coord.shape).ravel()
        cache[ck] = (_csr_pattern(np.concatenate([r1, r2]), np.concatenate([c1, c2]), (n_rows, maps.n_global_state)),
                     _csr_pattern(r3, c3, (n_rows, maps.n_global_coord)))
    (ou, su, pu, iu), (ox, sx, px, ix) = cache[ck]
    vals = np.concatenate([jac_self.ravel(), (jac_neigh * valid[:, None, :]).ravel()])
    dRdU = sp.csr_matrix((np.add.reduceat(vals[ou], su), iu, pu), shape=(n_rows, maps.n_global_state))
    dRdx = sp.csr_matrix((np.add.reduceat(jac_coord.ravel()[ox], sx), ix, px), shape=(n_rows, maps.n_global_coord))
    return dRdU, dRdx


def assemble_blocks_csr(law, geom, U, x, mu, test_degree=None, dist=None, device=None, rows=None):
    """One K1 pass and the CSR Jacobians straight from the device records:
    (res (ne, NT), dR/dU csr, dR/dx csr, N (ne,), dN/dx_e (ne, 6)).

    The sorted CSR structure of dg.py:246-271 is fixed per (mesh, test space), so it is built once
    (``_csr_pattern``) together with, for every stored entry, the record position that holds its
    value: duplicates of the reference's COO list are only the masked entries of missing
    neighbors (exact zeros in the records), so a device gather of one position per entry equals
    the reference's duplicate sum.  Per call the GPU gathers the nnz values and only they, the
    residual rows and the distortion columns cross to the host.  ``rows`` (ne, NT) global row ids
    (default: element-major test rows, ``assemble_enriched``; ``maps.state_map`` for
    ``assemble_global``)."""
    import torch

    from .tables import lagrange_nodes

    maps = geom.maps
    m, p, ne = maps.n_comp, maps.degree_sol, geom.mesh.num_elements
    nu = lagrange_nodes(p).shape[0] * m
    plain_mma = test_degree is None and m == 4 and p == 2
    deg = p if test_degree is None else test_degree
    NT = lagrange_nodes(deg).shape[0] * m
    out = _element_records(law, geom, U, x, mu, dist=dist, device=device, test_degree=None if plain_mma else deg,
                           on_device=True)
    rec = out.shape[1]
    a, b, c, d = NT, NT + NT * nu, NT + 4 * NT * nu, NT * (1 + 4 * nu + 6)
    if rows is None:
        rows = (np.arange(ne)[:, None] * NT + np.arange(NT)[None, :]).astype(np.int64)
        n_rows = ne * NT
    else:
        n_rows = maps.n_global_state
    cache = maps.__dict__.setdefault("_b200_csr_device", {})
    ck = (NT, nu, n_rows, int(rows[0, 0]), int(rows[-1, -1]), str(out.device))
    if ck not in cache:
        base = (np.arange(ne, dtype=np.int64) * rec)[:, None, None]
        rr = rows[:, :, None]
        pos_s = base + a + (np.arange(NT)[None, :, None] * nu + np.arange(nu)[None, None, :])
        pos_n = base + b + (np.arange(NT)[None, :, None] * 3 * nu + np.arange(3 * nu)[None, None, :])
        pos_x = base + c + (np.arange(NT)[None, :, None] * 6 + np.arange(6)[None, None, :])
        nmap = maps.neighbor_map
        r_u = np.concatenate([np.broadcast_to(rr, pos_s.shape).ravel(), np.broadcast_to(rr, pos_n.shape).ravel()])
        c_u = np.concatenate([np.broadcast_to(maps.state_map[:, None, :], pos_s.shape).ravel(),
                              np.broadcast_to(np.clip(nmap, 0, None)[:, None, :], pos_n.shape).ravel()])
        real = np.concatenate([np.ones(pos_s.size, bool), np.broadcast_to((nmap >= 0)[:, None, :], pos_n.shape).ravel()])
        src = np.concatenate([pos_s.ravel(), pos_n.ravel()])
        # real entries first within a duplicate group (stable sort on (key, not real))
        key = r_u.astype(np.int64) * maps.n_global_state + c_u
        order = np.lexsort((~real, key))
        ks = key[order]
        first = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
        n_real = np.add.reduceat(real[order].astype(np.int64), first)
        if np.any(n_real > 1):
            raise NotImplementedError("two element blocks share a Jacobian entry (not a conforming mesh)")
        indptr = np.zeros(n_rows + 1, dtype=np.int32)
        np.cumsum(np.bincount(ks[first] // maps.n_global_state, minlength=n_rows), out=indptr[1:])
        pu = (torch.as_tensor(src[order][first]).to(out.device), indptr, (ks[first] % maps.n_global_state).astype(np.int32))
        ox, fx, px, ix = _csr_pattern(np.broadcast_to(rr, pos_x.shape).ravel(),
                                      np.broadcast_to(maps.coord_map[:, None, :], pos_x.shape).ravel(),
                                      (n_rows, maps.n_global_coord))
        if len(fx) != pos_x.size:
            raise NotImplementedError("duplicate coordinate columns within an element")
        cache[ck] = (pu, (torch.as_tensor(pos_x.ravel()[ox]).to(out.device), px, ix))
    (gu, pu_, iu), (gx, px, ix) = cache[ck]
    flat = out.view(-1)
    small = torch.cat([out[:, :NT].reshape(-1), out[:, d:d + 7].reshape(-1)])
    host = torch.cat([flat[gu], flat[gx], small]).cpu().numpy()
    nu_, nx_ = gu.numel(), gx.numel()
    dRdU = sp.csr_matrix((host[:nu_], iu, pu_), shape=(n_rows, maps.n_global_state))
    dRdx = sp.csr_matrix((host[nu_:nu_ + nx_], ix, px), shape=(n_rows, maps.n_global_coord))
    res = host[nu_ + nx_:nu_ + nx_ + ne * NT].reshape(ne, NT)
    nd = host[nu_ + nx_ + ne * NT:].reshape(ne, 7)
    return res, dRdU, dRdx, nd[:, 0], nd[:, 1:]


def enriched_records(law, geom, U, x, mu, test_degree=None, dist=None, want_jacobians=True, device=None,
                     raise_degenerate=True):
    """``element_blocks`` against the degree p+1 (or ``test_degree``) test space (dg.py:275-326)."""
    deg = geom.maps.degree_sol + 1 if test_degree is None else test_degree
    return element_blocks(law, geom, U, x, mu, deg, dist, want_jacobians, device, raise_degenerate)


def assemble_enriched(law, mesh, maps, U, x, mu, test_degree=None, want_jacobians=True, geom=None, device=None):
    """Residual tested against the degree p+1 nodal space, with CSR dRbar/dU (ne n_t x N_u)
    and dRbar/dx (ne n_t x N_x): strom/dg.py:275-326 (rows element-major)."""
    from .mesh import get_geometry

    geom = geom or get_geometry(mesh, maps)
    deg = maps.degree_sol + 1 if test_degree is None else test_degree
    if not want_jacobians:
        res = element_blocks(law, geom, U, x, mu, deg, want_jacobians=False, device=device)[0]
        return res.reshape(-1).copy(), None, None
    res, dRdU, dRdx, _, _ = assemble_blocks_csr(law, geom, U, x, mu, deg, device=device)
    return res.reshape(-1).copy(), dRdU, dRdx


class HdmSolveError(RuntimeError):
    """Mirror of strom.dg.HdmSolveError (dg.py:336-340)."""

    def __init__(self, message, residual_norm, state):
        super().__init__(message)
        self.residual_norm = residual_norm
        self.state = state


def state_positions(geom, x):
    """Positions of all solution nodes under the mapping coefficients x (geometry.py:156-160;
    straight elements: barycentric combinations of the deformed vertices)."""
    from .tables import lagrange_nodes

    mesh, maps = geom.mesh, geom.maps
    xi = lagrange_nodes(maps.degree_sol)  # (nb, 2) reference nodes
    bary = np.stack([1.0 - xi[:, 0] - xi[:, 1], xi[:, 0], xi[:, 1]], axis=1)  # P1 shape functions
    x_e = np.asarray(x, dtype=float)[maps.coord_map].reshape(mesh.num_elements, -1, 2)[:, :3]
    return np.einsum("ng,egi->eni", bary, x_e)


def initial_state(law, mesh, maps, x, mu, geom=None):
    """Law-provided initial guess sampled at the deformed solution nodes (dg.py:329-333)."""
    from .mesh import get_geometry

    pos = state_positions(geom or get_geometry(mesh, maps), x)
    return np.asarray(law.initial_state(pos, mu), dtype=float).reshape(-1)


def solve_hdm(law, mesh, maps, x, mu, U_init=None, tol=1e-10, max_iters=80, geom=None, device=None):
    """Damped Newton / pseudo-transient-continuation solve of the DG system on a frozen mesh
    (dg.py:343-400): the residual and its sparse Jacobian are assembled on the GPU, the
    linear systems factored with SuperLU on the host like the reference.  Returns the state
    vector; raises HdmSolveError when it does not converge."""
    import scipy.sparse.linalg as spla

    from .mesh import get_geometry
    from .reduced import DegenerateMappingError

    geom = geom or get_geometry(mesh, maps)
    U = initial_state(law, mesh, maps, x, mu, geom) if U_init is None else np.asarray(U_init, dtype=float).copy()
    R, J, _ = assemble_global(law, mesh, maps, U, x, mu, geom=geom, device=device)
    rnorm0 = np.linalg.norm(R)
    target = tol * max(1.0, rnorm0)
    rnorm = rnorm0
    ptc = 0.0  # inverse pseudo-timestep; 0 = plain Newton
    ident = sp.identity(maps.n_global_state, format="csr")
    for _ in range(max_iters):
        if rnorm <= target:
            return U
        A = J + ptc * ident if ptc > 0.0 else J
        try:
            dU = spla.splu(A.tocsc()).solve(-R)
        except RuntimeError:
            ptc = max(10.0 * ptc, 1e-4 * rnorm)
            continue
        alpha, best = 1.0, None
        for _ in range(30):
            try:
                Rt, _, _ = assemble_global(law, mesh, maps, U + alpha * dU, x, mu, want_jacobians=False, geom=geom,
                                           device=device)
                nt = np.linalg.norm(Rt)
            except DegenerateMappingError:
                nt = np.inf
            if nt < (1.0 - 1e-4 * alpha) * rnorm or nt <= target:
                best = (alpha, nt)
                break
            alpha *= 0.5
        if best is None:  # line search stalled: engage / strengthen pseudo-transient damping
            ptc = max(4.0 * ptc, 1e-3 * max(rnorm, 1.0))
            continue
        U = U + best[0] * dU
        rnorm = best[1]
        if ptc > 0.0:  # relax damping as the residual drops
            ptc = ptc / 4.0 if best[0] == 1.0 else ptc
            if ptc < 1e-12 * max(rnorm, 1.0):
                ptc = 0.0
        R, J, _ = assemble_global(law, mesh, maps, U, x, mu, geom=geom, device=device)
        rnorm = np.linalg.norm(R)
    if rnorm <= target:
        return U
    raise HdmSolveError(f"HDM solve did not converge: |R| = {rnorm:.3e} (target {target:.3e})", rnorm, U)
