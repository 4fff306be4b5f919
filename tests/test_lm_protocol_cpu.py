"""The protocol path of lm.lm_solve (host loop over GPU-assembled blocks; here a synthetic
problem, no GPU) against the oracle's dense LM (pinned to the reference, test_oracle_golden.py)
and, where the reference is present, against strom.lm.lm_solve itself — dense and sparse blocks."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import lm as olm
from paper_2305_15661_b200.lm import LmConfig, lm_solve, lm_solve_protocol


class Synthetic:
    """Nonlinear least squares over split coordinates: r = A w + B tau + c sin(D w) . (E tau) - y."""

    def __init__(self, nw=5, nt=3, m=14, seed=3, sparse=False):
        rng = np.random.default_rng(seed)
        self.A, self.B = rng.standard_normal((m, nw)), rng.standard_normal((m, nt))
        self.D, self.E = rng.standard_normal((m, nw)) * 0.3, rng.standard_normal((m, nt)) * 0.5
        self.y = rng.standard_normal(m)
        self.nw, self.ntau, self.sparse = nw, nt, sparse

    def initial_guess(self):
        return np.full(self.nw, 0.1), np.full(self.ntau, -0.2)

    def _r(self, w, t):
        return self.A @ w + self.B @ t + np.sin(self.D @ w) * (self.E @ t) - self.y

    def objective(self, w, t):
        r = self._r(w, t)
        return 0.5 * float(r @ r)

    def derivatives(self, w, t):
        r = self._r(w, t)
        Jw = self.A + (np.cos(self.D @ w) * (self.E @ t))[:, None] * self.D
        Jt = self.B + np.sin(self.D @ w)[:, None] * self.E
        blocks = (Jw.T @ Jw, Jw.T @ Jt, Jt.T @ Jt)
        if self.sparse:
            blocks = tuple(sp.csr_matrix(b) for b in blocks)
        return (0.5 * float(r @ r), Jw.T @ r, Jt.T @ r, *blocks)


@pytest.mark.parametrize("w0_mode", ["lsq", "keep"])
def test_protocol_lm_matches_oracle_dense(w0_mode):
    p = Synthetic()
    got = lm_solve(p, LmConfig(max_iters=40), w0_mode=w0_mode)  # dispatches to the protocol path
    ref = olm.lm_solve(p, olm.LmConfig(max_iters=40), w0_mode=w0_mode)
    assert got.converged == ref.converged and got.n_iters == ref.n_iters and got.reason == ref.reason
    assert np.array_equal(got.history[:, [0, 5]], ref.history[:, [0, 5]], equal_nan=True)
    assert np.allclose(got.history[:, 1:5], ref.history[:, 1:5], rtol=1e-9, atol=1e-14)
    assert np.allclose(got.w, ref.w, rtol=1e-10, atol=1e-12) and np.allclose(got.tau, ref.tau, rtol=1e-10, atol=1e-12)


def test_protocol_lm_sparse_blocks_agree_with_dense():
    d = lm_solve_protocol(Synthetic(sparse=False), LmConfig(max_iters=25))
    s = lm_solve_protocol(Synthetic(sparse=True), LmConfig(max_iters=25))
    # sysv vs SuperLU round differently: same solution, iteration counts within one near the tolerance
    assert abs(d.n_iters - s.n_iters) <= 1 and d.reason == s.reason == "first-order"
    assert np.allclose(d.w, s.w, rtol=1e-8, atol=1e-10) and np.allclose(d.tau, s.tau, rtol=1e-8, atol=1e-10)


def test_protocol_lm_matches_reference_solver():
    try:
        from oracle import strom_ref

        S = strom_ref.load()
    except ImportError:
        pytest.skip("reference strom not installed")
    for sparse in (False, True):
        p = Synthetic(nw=6, nt=4, m=20, seed=9, sparse=sparse)
        got = lm_solve_protocol(p, LmConfig(max_iters=30))
        ref = S["lm"].lm_solve(p, S["lm"].LmConfig(max_iters=30))
        assert got.converged == ref.converged and got.n_iters == ref.n_iters and got.reason == ref.reason
        assert np.array_equal(got.history, ref.history, equal_nan=True)
        assert np.array_equal(got.w, ref.w) and np.array_equal(got.tau, ref.tau)


def test_protocol_lm_line_search_failure_and_bad_mode():
    class Flat(Synthetic):
        def objective(self, w, t):  # never decreases: every Armijo test fails
            return 1.0 + float(w @ w)

    res = lm_solve_protocol(Flat(), LmConfig(max_iters=5, lambda_cap=1e3), w0_mode="keep")
    assert not res.converged and res.reason == "line-search-failure"
    with pytest.raises(ValueError):
        lm_solve_protocol(Synthetic(), w0_mode="nope")
