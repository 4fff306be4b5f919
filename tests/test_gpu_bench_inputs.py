"""Parity at exactly bench.py's inputs (config 2 generator, W = Tau = 0, rho = 1).

bench.py times ``configs.euler_square_case(n=256)`` at w = 0, tau = 0; the
same generator at n = 16 / 32 is compared here with the oracle through the
public API (``ReducedOperator.derivatives``, strom/reduced.py:209-229) at the
1e-10 contract.  A second test documents the tie point of the literal
"one factor per node shared by the four components" reading of config 2:
every LLF max(ws_in, ws_out) (strom/dg.py:170-172, dual.py:167-176) is then
an exact tie whose one-sided derivative is decided by last-bit rounding, so
only tie-insensitive quantities are held to 1e-10 there and the measured
deviation of the rest is reported.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle.dual as D
from oracle import element as OE
from oracle.element import OracleGeometry, OracleReducedOperator

from cases import rel_err

TOL = 1e-10
NAMES = ("J", "S", "T", "Hww", "Hwt", "Htt")


def _oracle(case):
    geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
    return OracleReducedOperator(case.law, geom, case.phi, case.psi, case.ref_coords, case.kappa, case.eps,
                                 state_offset=case.state_offset)


def _gpu(case):
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

    return GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist,
                              state_offset=case.state_offset)


def _llf_gaps(case):
    """Relative gaps |ws_in - ws_out| / ws of every LLF max the oracle takes at W = Tau = 0."""
    gaps = []
    orig = D.maximum

    def spy(a, b):
        va, vb = D.val(a), D.val(b)
        if np.ndim(va) == 2:  # the (B, n_s) wavespeed pair; distortion's max(g, eps) is (B, n_q) with a scalar
            if np.ndim(vb) == 2:
                gaps.append((np.abs(va - vb) / np.maximum(np.abs(va), 1e-300)).ravel())
        return orig(a, b)

    D.maximum = spy
    try:
        _oracle(case).objective(case.W[0], case.Tau[0], case.mus[0])
    finally:
        D.maximum = orig
    return np.concatenate(gaps)


def test_bench_inputs_have_no_llf_ties():
    """CPU: at the benchmarked inputs no LLF wavespeed pair is within 1e-12 (no rounding-decided branch)."""
    from paper_2305_15661_b200 import configs

    case = configs.euler_square_case(n=8)
    g = _llf_gaps(case)
    assert g.size > 0
    assert np.min(g) > 1e-12, np.min(g)
    tie = configs.euler_square_case(n=8, per_component=False)
    gt = _llf_gaps(tie)
    # interior faces of the shared-factor reading are exact ties up to rounding
    assert np.mean(gt < 1e-14) > 0.5


@pytest.mark.gpu
@pytest.mark.parametrize("n", [16, 32])
def test_bench_inputs_match_oracle(n):
    """GPU vs oracle at bench.py's generator and coordinates (n cells per side)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_15661_b200 import configs
    from paper_2305_15661_b200.reduced import ReducedCoords

    case = configs.euler_square_case(n=n)
    got = _gpu(case).derivatives(ReducedCoords(case.W[0], case.Tau[0]), case.mus[0])
    ref = _oracle(case).derivatives(case.W[0], case.Tau[0], case.mus[0], None)
    for k, a, b in zip(NAMES, got, ref):
        assert rel_err(a, b) < TOL, (k, rel_err(a, b))
    # and through the batched entry point bench.py times
    from paper_2305_15661_b200 import _lib

    op = _gpu(case)
    ku, kx = case.phi.shape[1], case.psi.shape[1]
    K = ku + kx
    out = torch.empty(1 + K + K * K, dtype=torch.float64, device="cuda")
    W = torch.zeros((1, ku), dtype=torch.float64, device="cuda")
    Tau = torch.zeros((1, kx), dtype=torch.float64, device="cuda")
    Mu = torch.as_tensor(case.mus, dtype=torch.float64).cuda()
    op.eval_batched(_lib.DERIVS, W, Tau, Mu, None, out=out)
    o = out.cpu().numpy()
    assert rel_err(o[0], ref[0]) < TOL
    assert rel_err(o[1:1 + ku], ref[1]) < TOL and rel_err(o[1 + ku:1 + K], ref[2]) < TOL
    H = o[1 + K:].reshape(K, K)
    assert rel_err(H[:ku, :ku], ref[3]) < TOL and rel_err(H[:ku, ku:], ref[4]) < TOL
    assert rel_err(H[ku:, ku:], ref[5]) < TOL


@pytest.mark.gpu
def test_shared_factor_tie_point_documented(capsys):
    """The literal shared-factor reading (not benchmarked): values agree, tie-decided derivatives may not."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_15661_b200 import configs
    from paper_2305_15661_b200.reduced import ReducedCoords

    case = configs.euler_square_case(n=8, per_component=False)
    c = ReducedCoords(case.W[0], case.Tau[0])
    gpu, ora = _gpu(case), _oracle(case)
    # values are tie-insensitive (max(a, a) = a): objective and the global residual hold 1e-10
    assert rel_err(gpu.objective(c, case.mus[0]), ora.objective(case.W[0], case.Tau[0], case.mus[0])) < TOL
    U = case.state_offset
    R = OE.assemble_residual(case.law, ora.geom, U, case.ref_coords, case.mus[0])
    assert rel_err(gpu.global_residual(c, case.mus[0]), R) < TOL
    got = gpu.derivatives(c, case.mus[0])
    ref = ora.derivatives(case.W[0], case.Tau[0], case.mus[0], None)
    assert rel_err(got[0], ref[0]) < TOL  # J is a value
    dev = {k: rel_err(a, b) for k, a, b in zip(NAMES[1:], got[1:], ref[1:])}
    with capsys.disabled():
        print("\n[tie point, n=8] relative deviation of tie-decided derivatives:",
              ", ".join(f"{k}={v:.2e}" for k, v in dev.items()))
    # one-sided LLF derivatives: a flipped tie moves S/H by O(1e-2) at most (VERDICT r01 measured 1.6e-2)
    assert all(np.isfinite(v) and v < 0.1 for v in dev.values()), dev
