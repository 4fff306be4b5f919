"""Batched Levenberg-Marquardt on the GPU (strom/lm.py:30-271 semantics).

``lm_solve(problem, config, w0_mode)`` keeps the reference signature and
result type; ``problem`` must be a ``ReducedTrackingProblem`` over a
``GpuReducedOperator`` (the whole solve then runs as the device-side state
machine of csrc/lm_kernels.cuh).  ``lm_solve_batched`` solves many
parameter points at once — the online EQP-IFT solve of SURVEY §8 row a21
with P parameters in flight.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .reduced import GpuReducedOperator, degenerate_error

REASONS = {0: "first-order", 1: "max-iters", 2: "line-search-failure", 3: "degenerate"}


@dataclass
class LmConfig:
    """Mirror of strom.lm.LmConfig (lm.py:30-51)."""

    eps1: float = 1e-8
    eps2: float = 1e-8
    lambda0: float = None
    lambda_inc: float = 2.0
    lambda_dec: float = 1.0 / 3.0
    ratio_hi: float = 0.75
    ratio_lo: float = 0.25
    max_iters: int = 200
    wolfe_c1: float = 1e-4
    wolfe_c2: float = 0.9
    max_backtracks: int = 30
    lambda_cap: float = 1e14
    w0_inner_tol: float = 1e-10
    w0_inner_iters: int = 50

    def __post_init__(self):
        if self.eps1 <= 0 or self.eps2 <= 0:
            raise ValueError("termination tolerances must be positive")
        if not (0.0 < self.wolfe_c1 < self.wolfe_c2 < 1.0):
            raise ValueError("need 0 < c1 < c2 < 1")

    def packed(self, w0_mode):
        lam0 = -1.0 if self.lambda0 is None else float(self.lambda0)
        return np.array([self.eps1, self.eps2, lam0, self.lambda_inc, self.lambda_dec, self.ratio_hi, self.ratio_lo,
                         self.max_iters, self.wolfe_c1, self.wolfe_c2, self.max_backtracks, self.lambda_cap,
                         self.w0_inner_tol, self.w0_inner_iters, 1.0 if w0_mode == "lsq" else 0.0], dtype=np.float64)


@dataclass
class LmResult:
    """Mirror of strom.lm.LmResult (lm.py:54-64)."""

    w: np.ndarray
    tau: np.ndarray
    converged: bool
    objective: float
    grad_w_norm: float
    grad_tau_norm: float
    n_iters: int
    history: np.ndarray
    reason: str = ""


class ReducedTrackingProblem:
    """LM problem over reduced coordinates at one parameter (reduced.py:254-281)."""

    def __init__(self, operator, mu, rho=None, w0=None, tau0=None):
        self.op = operator
        self.mu = np.asarray(mu, dtype=float)
        self.rho = rho
        self._w0 = np.zeros(operator.bases.k_u) if w0 is None else np.asarray(w0, dtype=float)
        self._tau0 = np.zeros(operator.bases.k_x) if tau0 is None else np.asarray(tau0, dtype=float)

    @property
    def nw(self):
        return self.op.bases.k_u

    @property
    def ntau(self):
        return self.op.bases.k_x

    def initial_guess(self):
        return self._w0.copy(), self._tau0.copy()

    def objective(self, w, tau):
        from .reduced import ReducedCoords

        return self.op.objective(ReducedCoords(w, tau), self.mu, self.rho)

    def derivatives(self, w, tau):
        from .reduced import ReducedCoords

        return self.op.derivatives(ReducedCoords(w, tau), self.mu, self.rho)


def as_config(config):
    """This package's LmConfig from any object with LmConfig's fields (e.g. strom.lm.LmConfig,
    which the reference's train_weights passes to a swapped-in lm_solve, eqp.py:158)."""
    if config is None or isinstance(config, LmConfig):
        return config or LmConfig()
    from dataclasses import fields

    return LmConfig(**{f.name: getattr(config, f.name) for f in fields(LmConfig) if hasattr(config, f.name)})


def lm_solve_device(op, W, Tau, Mu, rho, config, status, hist=None, w0_mode="lsq"):
    """Device-resident batched solve: W (P, k_u) / Tau (P, k_x) cuda float64 tensors are
    overwritten with the solutions, ``status`` (P, 8) and ``hist`` (P, max_iters+1, 6) filled;
    stream-ordered on the current stream (strom_lm_solve, include/strom_b200.h)."""
    P, kx = int(Mu.shape[0]), op.k_x
    act, rw, A = op._weights(rho)
    packed = as_config(config).packed(w0_mode)
    stream = torch.cuda.current_stream(op.device).cuda_stream
    rc = _lib.load().strom_lm_solve(op._h, W.data_ptr(), Tau.data_ptr() if kx else W.data_ptr(), Mu.data_ptr(), P,
                                    act.data_ptr() if act is not None else None,
                                    rw.data_ptr() if rw is not None else None, A, packed.ctypes.data,
                                    status.data_ptr(), hist.data_ptr() if hist is not None else None, stream)
    _lib.check(rc, "strom_lm_solve")
    op.stats["lm_solves"] = op.stats.get("lm_solves", 0) + P


def lm_solve_batched(op, mus, W0=None, Tau0=None, rho=None, config=None, w0_mode="lsq", want_history=True,
                     raise_degenerate=False):
    """Solve P reduced problems (one per row of ``mus``) on the GPU at once."""
    if not isinstance(op, GpuReducedOperator):
        raise TypeError("lm_solve_batched needs a GpuReducedOperator")
    if getattr(op, "_pad", 0):
        raise NotImplementedError("the batched device LM needs k_u >= 1; the tau-only problem runs through lm_solve (protocol loop)")
    if w0_mode not in ("lsq", "keep"):
        raise ValueError(f"unknown w0_mode {w0_mode!r}")
    cfg = as_config(config)
    mus = np.atleast_2d(np.asarray(mus, dtype=float))
    P, ku, kx = mus.shape[0], op.k_u, op.k_x
    dev = op.device
    Mu = torch.as_tensor(np.stack([op._mu(m) for m in mus])).to(dev)
    W = torch.as_tensor(np.zeros((P, ku)) if W0 is None else np.broadcast_to(np.asarray(W0, float), (P, ku)).copy()).to(dev)
    Tau = torch.as_tensor(np.zeros((P, kx)) if Tau0 is None else np.broadcast_to(np.asarray(Tau0, float), (P, kx)).copy()).to(dev)
    status = torch.zeros((P, 8), dtype=torch.float64, device=dev)
    hist = torch.zeros((P, cfg.max_iters + 1, 6), dtype=torch.float64, device=dev) if want_history else None
    lm_solve_device(op, W, Tau, Mu, rho, cfg, status, hist, w0_mode)
    Wh, Th, st = W.cpu().numpy(), Tau.cpu().numpy(), status.cpu().numpy()
    H = hist.cpu().numpy() if hist is not None else None
    out = []
    for p in range(P):
        conv = bool(st[p, 0])
        reason = REASONS[int(st[p, 5])]
        if reason == "degenerate" and raise_degenerate:
            raise degenerate_error(np.zeros(0, dtype=np.int64))
        n = int(st[p, 4])
        rows = n + 1 if conv else n
        out.append(LmResult(Wh[p].copy(), Th[p].copy(), conv, float(st[p, 1]), float(st[p, 2]), float(st[p, 3]), n,
                            H[p, :rows].copy() if H is not None else None, reason))
    return out


# -- protocol path: any problem with (nw, ntau, initial_guess, objective, derivatives) ----------
# The full-space tracking / alignment problems (tracking.TrackingProblem) have sparse blocks
# with thousands of unknowns; their residuals and Jacobians are assembled on the GPU, the
# damped normal equations are factored on the host (SuperLU), as strom/lm.py:77-126 does.


def _trial_objective(problem, w, tau):
    from .reduced import DegenerateMappingError

    try:
        return problem.objective(w, tau)
    except DegenerateMappingError:
        return np.inf


def _normal_step(H_ww, H_wt, H_tt, S, T, lam):
    """(dw, dtau) of the normal equations damped on the deformation block only
    (lm.py:77-126); numpy.linalg.LinAlgError when singular."""
    import scipy.linalg
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    nw, nt = len(S), len(T)
    if nw + nt == 0:
        return np.zeros(0), np.zeros(0)
    rhs = -np.concatenate([S, T])
    if any(sp.issparse(M) for M in (H_ww, H_wt, H_tt) if M is not None):
        damped = None if nt == 0 else sp.csr_matrix(H_tt) + lam * sp.identity(nt, format="csr")
        if nt == 0:
            K = sp.csc_matrix(H_ww)
        elif nw == 0:
            K = damped.tocsc()
        else:
            C = sp.csr_matrix(H_wt)
            K = sp.bmat([[sp.csr_matrix(H_ww), C], [C.T, damped]], format="csc")
        try:
            dz = spla.splu(K).solve(rhs)
        except RuntimeError as exc:
            raise np.linalg.LinAlgError(str(exc)) from exc
    else:
        if nt == 0:
            K = np.atleast_2d(H_ww)
        elif nw == 0:
            K = np.atleast_2d(H_tt) + lam * np.eye(nt)
        else:
            C = np.atleast_2d(H_wt)
            K = np.block([[np.atleast_2d(H_ww), C], [C.T, np.atleast_2d(H_tt) + lam * np.eye(nt)]])
        dz = scipy.linalg.solve(K, rhs, assume_a="sym")
    if not np.all(np.isfinite(dz)):
        raise np.linalg.LinAlgError("singular regularized system")
    return dz[:nw], dz[nw:]


def _state_init_protocol(problem, w, tau, cfg):
    """Gauss-Newton on the state block at frozen deformation (lm.py:129-161)."""
    _, S, _, H_ww, _, _ = problem.derivatives(w, tau)
    target = cfg.w0_inner_tol * max(1.0, np.linalg.norm(S))
    J = None
    for _ in range(cfg.w0_inner_iters):
        if np.linalg.norm(S) <= target:
            break
        try:
            dw, _ = _normal_step(H_ww, None, None, S, np.zeros(0), 0.0)
        except (np.linalg.LinAlgError, RuntimeError):
            break
        J = problem.objective(w, tau) if J is None else J
        sdw = float(S @ dw)
        alpha, Jt = 1.0, np.inf
        for _ in range(30):
            Jt = _trial_objective(problem, w + alpha * dw, tau)
            if Jt <= J + 1e-4 * alpha * sdw:
                break
            alpha *= 0.5
        else:
            break
        w, J = w + alpha * dw, Jt
        _, S, _, H_ww, _, _ = problem.derivatives(w, tau)
    return w


def lm_solve_protocol(problem, config=None, w0_mode="lsq"):
    """The reference LM (lm.py:164-271) over the problem protocol, host loop: lambda on the
    deformation block, Armijo backtracking, gain-ratio + weak-Wolfe damping update, lambda
    escalation on singular systems / failed searches, best-iterate fallback."""
    import scipy.sparse as sp

    cfg = as_config(config)
    if w0_mode not in ("lsq", "keep"):
        raise ValueError(f"unknown w0_mode {w0_mode!r}")
    w, tau = (np.asarray(v, dtype=float).copy() for v in problem.initial_guess())
    if w0_mode == "lsq" and len(w):
        w = _state_init_protocol(problem, w, tau, cfg)
    lam, lam_floor = cfg.lambda0, 0.0
    rows, best, reason, n_done = [], None, "max-iters", 0
    J, S, T, H_ww, H_wt, H_tt = problem.derivatives(w, tau)
    for it in range(cfg.max_iters):
        nS, nT = np.linalg.norm(S), np.linalg.norm(T)
        if best is None or J < best[0]:
            best = (J, w.copy(), tau.copy(), nS, nT)
        if lam is None:  # lambda0 = 1e-4 trace(H_tt) / k_x
            tr = (H_tt.diagonal().sum() if sp.issparse(H_tt) else np.trace(np.atleast_2d(H_tt))) if len(tau) else 0.0
            lam = 1e-4 * tr / len(tau) if len(tau) else 0.0
            lam_floor = 1e-10 * lam if lam > 0 else 0.0
        if nS <= cfg.eps1 and nT <= cfg.eps2:
            rows.append((it, J, nS, nT, lam, 0.0))
            return LmResult(w, tau, True, J, nS, nT, it, np.array(rows), "first-order")
        rows.append((it, J, nS, nT, lam, np.nan))
        n_done = it + 1
        step = None
        for _ in range(60):  # lambda escalation until a descent step passes the Armijo test
            grow = 4.0
            try:
                dw, dtau = _normal_step(H_ww, H_wt, H_tt, S, T, lam)
                gdot = float(S @ dw + T @ dtau)
                if np.isfinite(gdot) and gdot < 0.0:
                    alpha = 1.0
                    for _ in range(cfg.max_backtracks):
                        Jt = _trial_objective(problem, w + alpha * dw, tau + alpha * dtau)
                        if Jt <= J + cfg.wolfe_c1 * alpha * gdot:
                            step = (dw, dtau, gdot, alpha, Jt)
                            break
                        alpha *= 0.5
                if step is not None:
                    break
                lam = max(grow * lam, 1e-12)
            except np.linalg.LinAlgError:
                lam = max(2.0 * lam, 1e-12) * 10.0
            if lam > cfg.lambda_cap:
                break
        if step is None:
            reason = "line-search-failure"
            break
        dw, dtau, gdot, alpha, J_new = step
        w, tau = w + alpha * dw, tau + alpha * dtau
        pred = -0.5 * alpha * gdot
        ratio = (J - J_new) / pred if pred > 0 else 1.0
        J_prev = J
        J, S, T, H_ww, H_wt, H_tt = problem.derivatives(w, tau)
        J = J_new if np.isfinite(J_new) else J
        curv_ok = float(S @ dw + T @ dtau) >= cfg.wolfe_c2 * gdot
        if alpha < 0.25 or ratio < cfg.ratio_lo:
            lam *= cfg.lambda_inc
        elif alpha == 1.0 and ratio > cfg.ratio_hi and curv_ok:
            lam *= cfg.lambda_dec
        lam = min(max(lam, lam_floor), cfg.lambda_cap)
        rows[-1] = (it, J_prev, rows[-1][2], rows[-1][3], lam, alpha)
    nS, nT = np.linalg.norm(S), np.linalg.norm(T)
    if best is not None and best[0] < J:
        J, w, tau, nS, nT = best
    return LmResult(w, tau, False, J, nS, nT, n_done, np.array(rows), reason)


def lm_solve(problem, config=None, w0_mode="lsq"):
    """Reference-signature LM solve (lm.py:164).  A problem over a ``GpuReducedOperator`` runs
    as the device-resident batched state machine; any other protocol problem (full-space
    tracking, alignment: GPU-assembled sparse blocks) runs the host loop above."""
    op = getattr(problem, "op", None)
    if not isinstance(op, GpuReducedOperator) or getattr(op, "_pad", 0):
        # protocol problems, and the tau-only reduced problem (k_u = 0, reduced.py:197-199: the
        # batched device LM needs a state block): host loop over the GPU evaluations
        if all(hasattr(problem, a) for a in ("initial_guess", "objective", "derivatives")):
            return lm_solve_protocol(problem, config, w0_mode)
        raise NotImplementedError("lm_solve needs a GpuReducedOperator problem or a protocol problem")
    w0, tau0 = problem.initial_guess()
    res = lm_solve_batched(op, [problem.mu], w0[None], tau0[None], problem.rho, config, w0_mode,
                           raise_degenerate=True)
    return res[0]


def history_csv(history, path):
    """Mirror of strom.lm.history_csv (lm.py:67-70): rows (iter, J, |S|, |T|, lambda, alpha)."""
    from .io import history_csv as _h

    _h(history, path)
