"""Drop-in GPU ``ReducedOperator`` (strom/reduced.py:116-251) over the C ABI.

``GpuReducedOperator(law, geom, bases, dist_config)`` has the reference's
constructor and methods — ``objective``, ``residuals``, ``derivatives``,
``elemental_contributions``, ``stats`` — with the same argument meaning,
return types and error behaviour (``DegenerateMappingError`` carrying the
sorted element ids, raised after the whole batch is evaluated,
dg.py:177-178).  Reference callers that construct ``ReducedOperator`` by
module-global name can be pointed at it (``strom.eqp.ReducedOperator =
GpuReducedOperator``); ``reduced_objective`` / ``reduced_residuals`` mirror
reduced.py:284-296.

Extensions (no reference counterpart): batched device-resident evaluation
over many parameter points (``eval_batched``), the full-mesh residual and
its norm for the greedy indicator (``global_residual``,
``residual_norm``), an affine state offset ``U = U0 + Phi w`` (explicit
state fields for the element microbenchmark), and LP-row contributions.

PyTorch is used for device memory and streams only.  There is no CPU
fallback: without the CUDA library or a GPU every method raises.
"""

import sys
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, laws as L, tables


class DegenerateMappingError(RuntimeError):
    """Mapping Jacobian non-positive at a quadrature point (dg.py:26-33)."""

    def __init__(self, elements):
        self.elements = np.atleast_1d(np.asarray(elements))
        RuntimeError.__init__(self, f"mapping degeneracy (g <= 0) on elements {self.elements[:8].tolist()}")


def degenerate_error(elements):
    """Instance catchable as this class and, when loaded, as the reference's."""
    ref = sys.modules.get("strom.dg")
    cls = DegenerateMappingError
    if ref is not None and hasattr(ref, "DegenerateMappingError"):
        cls = type("DegenerateMappingError", (DegenerateMappingError, ref.DegenerateMappingError), {})
    return cls(elements)


@dataclass
class ReducedCoords:
    w: np.ndarray
    tau: np.ndarray


class ReducedBases:
    """Orthonormal state / deformation bases (reduced.py:30-64)."""

    def __init__(self, phi, psi, ref_coords):
        phi = np.asarray(phi, dtype=float)
        psi = np.asarray(psi, dtype=float)
        self.phi = phi[:, None] if phi.ndim == 1 else phi
        self.psi = psi[:, None] if psi.ndim == 1 else psi
        self.ref_coords = np.asarray(ref_coords, dtype=float)

    @property
    def k_u(self):
        return self.phi.shape[1]

    @property
    def k_x(self):
        return self.psi.shape[1]

    def check_orthonormal(self, tol=1e-12):
        for mat in (self.phi, self.psi):
            if mat.shape[1] == 0:
                continue
            err = np.max(np.abs(mat.T @ mat - np.eye(mat.shape[1])))
            if err > tol:
                raise ValueError(f"basis not orthonormal (deviation {err:.2e})")
        return True


def reconstruct(bases, coords):
    """(Phi w, X + Psi tau), reduced.py:81-85."""
    U = bases.phi @ coords.w if bases.k_u else np.zeros(bases.phi.shape[0])
    x = bases.ref_coords + (bases.psi @ coords.tau if bases.k_x else 0.0)
    return U, x


EJ_SIZE = 24 + 24 * 24 + 24 * 72 + 24 * 6 + 7  # STROM_ELEMJAC record per element (include/strom_b200.h)


def _as_f64(a, device):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(device)


class DeviceMesh:
    """Mesh connectivity + discretisation tables resident on one device."""

    def __init__(self, geom, law, device):
        mesh, maps = geom.mesh, geom.maps
        if getattr(mesh, "degree_geo", 1) != 1:
            raise NotImplementedError("the B200 kernels support straight (q = 1) geometry only")
        self.device = device
        self.ne = mesh.num_elements
        self.nv = mesh.nodes.shape[0]
        self.p = maps.degree_sol
        self.m = maps.n_comp
        self.tabs = tables.element_tables(self.p, 1, getattr(geom, "quad_order", None))
        self.nu = self.tabs.nb * self.m
        self.dlaw = L.device_law(law, mesh.boundary_tags)
        if self.dlaw.n_comp != self.m:
            raise ValueError("law component count does not match the assembly maps")
        nbr, nface, flip, tag = mesh.neighbor_tables()
        code_of_tag = np.zeros(max(list(mesh.boundary_tags.values()) + [0]) + 1, dtype=np.int64)
        for name, tid in mesh.boundary_tags.items():
            code_of_tag[tid] = self.dlaw.bc_code_by_tag[name]
        bc = np.where(tag >= 0, code_of_tag[np.clip(tag, 0, None)], 0)
        if np.any((nbr < 0) & (bc == 0)):
            raise ValueError("boundary face without a boundary condition")
        finfo = (np.where(nbr >= 0, nface, 0) | (flip.astype(np.int64) << 2) | (bc << 3)).astype(np.uint8)
        self.elem_nodes = torch.as_tensor(np.ascontiguousarray(mesh.elements[:, :3], dtype=np.int32)).to(device)
        self.nodes = _as_f64(mesh.nodes, device)
        self.nbr = torch.as_tensor(np.ascontiguousarray(nbr, dtype=np.int32)).to(device)
        self.finfo = torch.as_tensor(finfo).to(device)
        t = self.tabs
        self._host = [np.ascontiguousarray(a, dtype=np.float64) for a in (t.phi, t.dphi, t.wq, t.bary, t.trace, t.ws, t.s)]
        self._fn = np.ascontiguousarray(t.fnodes, dtype=np.int32)

    def descriptors(self):
        md = _lib.MeshDesc(self.ne, self.nv, self.elem_nodes.data_ptr(), self.nodes.data_ptr(),
                           self.nbr.data_ptr(), self.finfo.data_ptr())
        t = self.tabs
        ptr = [a.ctypes.data for a in self._host]
        qd = _lib.QuadDesc(t.p, t.nb, t.nq, t.ns, t.fnodes.shape[1], *ptr, self._fn.ctypes.data)
        return md, qd


class GpuReducedOperator:
    """B200 replacement of ``strom.reduced.ReducedOperator``."""

    def __init__(self, law, geom, bases, dist_config, device=None, state_offset=None, n_mu=None):
        lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("GpuReducedOperator needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.law, self.geom, self.bases, self.dist = law, geom, bases, dist_config
        self.stats = {"kernel_calls": 0, "elements_evaluated": 0}
        with torch.cuda.device(self.device):
            self.dm = DeviceMesh(geom, law, self.device)
            pd = np.atleast_2d(np.asarray(getattr(law, "param_domain", np.zeros((1, 2)))))
            self.n_mu = int(n_mu if n_mu is not None else max(1, pd.shape[0]))
            params = np.zeros(8)
            params[: len(self.dm.dlaw.params)] = self.dm.dlaw.params
            ld = _lib.LawDesc(self.dm.dlaw.law_id, self.dm.m, self.n_mu, (C_double8(params)))
            md, qd = self.dm.descriptors()
            dd = _lib.DistDesc(float(dist_config.kappa), float(dist_config.eps))
            h = _lib.C.c_void_p()
            _lib.check(lib.strom_create(_lib.C.byref(md), _lib.C.byref(ld), _lib.C.byref(qd), _lib.C.byref(dd),
                                        self.device.index, _lib.C.byref(h)), "strom_create")
            self._h = h
            # k_u = 0 (no state basis, reduced.py:197-199): the device runs one zero column,
            # which contributes exact zeros, and the public methods strip it
            self._pad = 1 if bases.k_u == 0 else 0
            self.k_u, self.k_x = bases.k_u + self._pad, bases.k_x
            nu_g = self.dm.ne * self.dm.nu
            self.phi = _as_f64(np.zeros((nu_g, 1)) if self._pad else np.asarray(bases.phi).reshape(nu_g, self.k_u),
                               self.device)
            self.psi = _as_f64(np.asarray(bases.psi).reshape(2 * self.dm.nv, self.k_x), self.device)
            self.ref_coords = _as_f64(bases.ref_coords, self.device)
            self.u0 = None if state_offset is None else _as_f64(state_offset, self.device)
            _lib.check(lib.strom_set_bases(h, self.phi.data_ptr() if self.k_u else None, self.k_u,
                                           self.psi.data_ptr() if self.k_x else None, self.k_x,
                                           self.ref_coords.data_ptr(),
                                           self.u0.data_ptr() if self.u0 is not None else None), "strom_set_bases")
            _lib.check(lib.strom_reserve(h, 1, self.dm.ne), "strom_reserve")
        self._rho_cache = (None, None, None)
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.strom_destroy(h)
            self._h = None

    # -- weights -----------------------------------------------------------------
    def _weights(self, rho):
        """(active device int32, rho device f64, A) or (None, None, ne)."""
        if rho is None:
            return None, None, self.dm.ne
        key = id(rho)
        if self._rho_cache[0] == key:
            return self._rho_cache[1]
        r = np.asarray(rho.rho if hasattr(rho, "rho") else rho, dtype=float)
        act = np.asarray(rho.active) if hasattr(rho, "active") else np.flatnonzero(r > 0.0)
        act_d = torch.as_tensor(act.astype(np.int32)).to(self.device)
        rho_d = _as_f64(r[act], self.device)
        out = (act_d, rho_d, len(act))
        self._rho_cache = (key, out, rho)
        return out

    def _mu(self, mu):
        m = np.zeros(self.n_mu)
        v = np.atleast_1d(np.asarray(mu, dtype=float)).reshape(-1)
        m[: min(len(v), self.n_mu)] = v[: self.n_mu]
        return m

    # -- core call -----------------------------------------------------------------
    def eval_batched(self, mode, W, Tau, Mu, rho=None, out=None, degen=None, sync=False):
        """Device-resident batched evaluation; W (P,ku), Tau (P,kx), Mu (P,n_mu)
        are cuda float64 tensors.  Returns the output tensor (see strom_eval)."""
        P = int(Mu.shape[0])
        act, rw, A = self._weights(rho)
        K = self.k_u + self.k_x
        ne = self.dm.ne
        size = {
            _lib.OBJECTIVE: P, _lib.RESNORM2: P, _lib.DERIVS: P * (1 + K + K * K),
            _lib.CONTRIB: P * ne * K, _lib.CONTRIB_SPLIT: P * ne * 2 * K,
            _lib.RESIDUAL: P * ne * self.dm.nu, _lib.CONTRIB_LPROWS: P * (K + 1) * ne,
            _lib.ELEMJAC: P * ne * EJ_SIZE,
        }.get(mode)
        if size is None and out is None:
            raise ValueError("this mode needs a caller-sized output tensor")
        if out is None:
            out = torch.empty(size, dtype=torch.float64, device=self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        rc = self._lib.strom_eval(self._h, mode, W.data_ptr() if self.k_u else None,
                                  Tau.data_ptr() if self.k_x else None, Mu.data_ptr(), P,
                                  act.data_ptr() if act is not None else None,
                                  rw.data_ptr() if rw is not None else None, A, out.data_ptr(),
                                  degen.data_ptr() if degen is not None else None, stream, 1 if sync else 0)
        _lib.check(rc, "strom_eval")
        self.stats["kernel_calls"] += 1
        self.stats["elements_evaluated"] += A * P
        return out, rc

    def _single(self, mode, coords, mu, rho):
        """One parameter point through the public API: one C call (strom_eval_host) stages the
        host inputs in pinned memory, copies them with one H2D, evaluates, and returns the result
        and the degenerate flag with one D2H and one stream synchronisation (the element ids
        only on the rare degenerate path)."""
        ku, kx = self.k_u, self.k_x
        w = np.zeros(ku) if self._pad else np.ascontiguousarray(coords.w, dtype=np.float64).reshape(-1)
        tau = np.ascontiguousarray(coords.tau, dtype=np.float64).reshape(-1)
        mu_v = np.ascontiguousarray(self._mu(mu), dtype=np.float64)
        if w.size != ku or tau.size != kx:
            raise ValueError(f"coordinates have sizes ({w.size}, {tau.size}), expected ({ku - self._pad}, {kx})")
        act, rw, A = self._weights(rho)
        K, ne = ku + kx, self.dm.ne
        n_out = {
            _lib.OBJECTIVE: 1, _lib.RESNORM2: 1, _lib.DERIVS: 1 + K + K * K, _lib.CONTRIB: ne * K,
            _lib.CONTRIB_SPLIT: ne * 2 * K, _lib.RESIDUAL: ne * self.dm.nu, _lib.CONTRIB_LPROWS: (K + 1) * ne,
            _lib.ELEMJAC: ne * EJ_SIZE,
        }[mode]
        out = np.empty(n_out)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        rc = self._lib.strom_eval_host(self._h, mode, w.ctypes.data if ku else None, tau.ctypes.data if kx else None,
                                       mu_v.ctypes.data, 1, act.data_ptr() if act is not None else None,
                                       rw.data_ptr() if rw is not None else None, A, out.ctypes.data, n_out, None,
                                       stream)
        _lib.check(rc, "strom_eval_host")
        self.stats["kernel_calls"] += 1
        self.stats["elements_evaluated"] += A
        if rc == 1:
            n = self._lib.strom_degenerate_elements(self._h, 0, None, 0)
            ids = np.zeros(max(n, 1), dtype=np.int32)
            self._lib.strom_degenerate_elements(self._h, 0, ids.ctypes.data, n)
            raise degenerate_error(ids[:n].astype(np.int64))
        return out

    # -- reference API -------------------------------------------------------------
    def objective(self, coords, mu, rho=None):
        """Half squared norm of the (weighted) stacked residual (reduced.py:172-184)."""
        if rho is not None and len(np.asarray(rho.active if hasattr(rho, "active") else np.flatnonzero(np.asarray(rho) > 0))) == 0:
            return 0.0
        return float(self._single(_lib.OBJECTIVE, coords, mu, rho)[0])

    def _derivs(self, coords, mu, rho):
        ku, kx, a = self.k_u, self.k_x, self._pad  # device columns [a, ku) are the API's state columns
        if rho is not None and self._weights(rho)[2] == 0:
            self.stats["kernel_calls"] += 1
            n = ku - a
            return 0.0, np.zeros(n), np.zeros(kx), np.zeros((n, n)), np.zeros((n, kx)), np.zeros((kx, kx))
        o = self._single(_lib.DERIVS, coords, mu, rho)
        K = ku + kx
        H = o[1 + K:].reshape(K, K)
        return (float(o[0]), o[1 + a:1 + ku].copy(), o[1 + ku:1 + K].copy(), H[a:ku, a:ku].copy(), H[a:ku, ku:].copy(),
                H[ku:, ku:].copy())

    def residuals(self, coords, mu, rho=None):
        """First-order optimality residuals (S, T) (reduced.py:195-207)."""
        ku, kx = self.k_u - self._pad, self.k_x
        if self.geom.mesh.num_elements == 0 or (ku == 0 and kx == 0):
            return np.zeros(ku), np.zeros(kx)
        _, S, T, _, _, _ = self._derivs(coords, mu, rho)
        return S, T

    def derivatives(self, coords, mu, rho=None):
        """(J, S, T, H_ww, H_wt, H_tt) in one pass (reduced.py:209-229)."""
        return self._derivs(coords, mu, rho)

    def elemental_contributions(self, coords, mu, split=False):
        """Per-element contributions over all elements (reduced.py:231-251)."""
        ku, kx, ne, a = self.k_u, self.k_x, self.dm.ne, self._pad
        if not split:
            o = self._single(_lib.CONTRIB, coords, mu, None).reshape(ne, ku + kx)
            return o[:, a:ku].copy(), o[:, ku:].copy()
        o = self._single(_lib.CONTRIB_SPLIT, coords, mu, None).reshape(ne, 2 * (ku + kx))
        return (o[:, a:ku].copy(), o[:, ku + a:2 * ku].copy(), o[:, 2 * ku:2 * ku + kx].copy(), o[:, 2 * ku + kx:].copy())

    # -- extensions ----------------------------------------------------------------
    def global_residual(self, coords, mu):
        """R(Phi w, X + Psi tau) over the whole mesh, element-major
        (dg.assemble_global(..., want_jacobians=False), dg.py:238-240)."""
        return self._single(_lib.RESIDUAL, coords, mu, None)

    def contributions_at_snapshots(self, U, X, mus, layout="lprows", out=None):
        """Element contributions at S explicit training snapshots in one batched pass.

        ``U`` (S, N_u) states and ``X`` (S, N_x) deformed coordinates (cuda
        float64 tensors) enter as per-snapshot affine offsets at w = 0,
        tau = 0; ``layout``: "lprows" -> (S, K+1, ne) rows S_e, T_e and
        0.5(|R_e|^2 + N_e^2) (config 4), "split" -> (S, ne, 2K) (Sv, Sf, Tv,
        Tf) as in eqp.build_lp (eqp.py:104-114), "total" -> (S, ne, K).
        """
        S = int(X.shape[0])
        mode = {"lprows": _lib.CONTRIB_LPROWS, "split": _lib.CONTRIB_SPLIT, "total": _lib.CONTRIB}[layout]
        lib = self._lib
        U = None if U is None else U.contiguous()
        X = X.contiguous()
        _lib.check(lib.strom_set_offsets(self._h, U.data_ptr() if U is not None else None,
                                         int(U.shape[1]) if U is not None else 0, X.data_ptr(), int(X.shape[1])),
                   "strom_set_offsets")
        try:
            W = torch.zeros((S, max(self.k_u, 1)), dtype=torch.float64, device=self.device)
            Tau = torch.zeros((S, max(self.k_x, 1)), dtype=torch.float64, device=self.device)
            Mu = torch.as_tensor(np.stack([self._mu(m) for m in np.atleast_2d(mus)])).to(self.device)
            res, _ = self.eval_batched(mode, W, Tau, Mu, None, out=out)
        finally:
            _lib.check(lib.strom_set_offsets(self._h, self.u0.data_ptr() if self.u0 is not None else None, 0,
                                             self.ref_coords.data_ptr(), 0), "strom_set_offsets")
        K = self.k_u + self.k_x
        ne = self.dm.ne
        shape = {"lprows": (S, K + 1, ne), "split": (S, ne, 2 * K), "total": (S, ne, K)}[layout]
        res = res.view(shape)
        if self._pad:  # strip the zero state column of a k_u = 0 operator
            ku = self.k_u
            if layout == "lprows":
                res = res[:, 1:]
            elif layout == "total":
                res = res[:, :, 1:]
            else:
                res = torch.cat([res[:, :, 1:ku], res[:, :, ku + 1:]], dim=2)
        return res

    def residual_norm(self, coords, mu):
        """||R||_2 of the full-mesh residual (greedy error indicator)."""
        return float(np.sqrt(self._single(_lib.RESNORM2, coords, mu, None)[0]))


def C_double8(v):
    arr = (_lib.C.c_double * 8)()
    for i, x in enumerate(v[:8]):
        arr[i] = float(x)
    return arr


def _operator(law, mesh, maps, bases, dist_config):
    from .mesh import get_geometry

    return GpuReducedOperator(law, get_geometry(mesh, maps), bases, dist_config)


def reduced_objective(law, mesh, maps, bases, coords, mu, dist_config):
    return _operator(law, mesh, maps, bases, dist_config).objective(coords, mu)


def reduced_residuals(law, mesh, maps, bases, coords, mu, dist_config):
    return _operator(law, mesh, maps, bases, dist_config).residuals(coords, mu)
