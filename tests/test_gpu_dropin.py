"""The GPU path swapped into the UNMODIFIED reference (baseline/_ref or /root/reference).

Everything here is the reference's own objects and code path — its law
(burgers-spacetime), mesher, geometry, bases, WeightVector, ReducedTrackingProblem,
lm_solve, build_lp, solve_lp and train_weights (strom/eqp.py:134-181) — with only
``ReducedOperator`` (and, for train_weights, ``lm_solve``) replaced by module-global
swap (paper_2305_15661_b200.dropin).  Compared with the same calls on the stock CPU path:
operator outputs and ``stats`` counters, an LM history, and the EQP weight LP end to end
(matrix, vertex weights, active set).  Skipped when the reference is not installed.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from cases import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import strom_ref

    try:
        return strom_ref.load()
    except ImportError as exc:
        pytest.skip(str(exc))


def problem(S, nx=4, ny=3, p=2, ku=6, kx=3, seed=71):
    import strom.conslaw as slaw
    import strom.distortion as sdist
    import strom.geometry as sgeom

    law = slaw.burgers_spacetime()
    mesh, maps = S["meshing"].build_structured_mesh(((0.0, 0.0), (2.0, 1.0)), nx, ny, degree_sol=p, n_comp=1)
    rng = np.random.default_rng(seed)

    def orth(n, k):
        q, r = np.linalg.qr(rng.standard_normal((n, k)))
        return q * np.sign(np.diag(r))

    bases = S["reduced"].ReducedBases(orth(maps.n_global_state, ku), orth(maps.n_global_coord, kx), mesh.nodes.ravel().copy())
    return law, mesh, maps, sgeom.get_geometry(mesh, maps), bases, sdist.DistortionConfig(1e-3)


def test_operator_dropin_matches_stock(S):
    from paper_2305_15661_b200.reduced import GpuReducedOperator

    law, mesh, maps, geom, bases, dc = problem(S)
    cpu, gpu = S["reduced"].ReducedOperator(law, geom, bases, dc), GpuReducedOperator(law, geom, bases, dc)
    rng = np.random.default_rng(5)
    c = S["reduced"].ReducedCoords(1.0 + rng.standard_normal(6), 1e-2 * rng.standard_normal(3))
    mu = np.array([5.0, 0.05])
    rho = S["eqp"].WeightVector(np.where(rng.random(mesh.num_elements) < 0.5, rng.uniform(0.5, 2.0, mesh.num_elements), 0.0))
    for w in (None, rho):
        assert rel_err(gpu.objective(c, mu, w), cpu.objective(c, mu, w)) < 1e-10
        for a, b in zip(gpu.derivatives(c, mu, w), cpu.derivatives(c, mu, w)):
            assert rel_err(a, b) < 1e-10
        for a, b in zip(gpu.residuals(c, mu, w), cpu.residuals(c, mu, w)):
            assert rel_err(a, b) < 1e-10
    for split in (False, True):
        for a, b in zip(gpu.elemental_contributions(c, mu, split), cpu.elemental_contributions(c, mu, split)):
            assert rel_err(a, b) < 1e-10
    assert gpu.stats == cpu.stats  # kernel_calls, elements_evaluated (reduced.py:131,167-169)


def test_reference_lm_solve_on_gpu_operator(S):
    from paper_2305_15661_b200.reduced import GpuReducedOperator

    law, mesh, maps, geom, bases, dc = problem(S)
    mu = np.array([5.0, 0.05])
    w0 = np.full(6, 0.5)
    runs = []
    for op in (S["reduced"].ReducedOperator(law, geom, bases, dc), GpuReducedOperator(law, geom, bases, dc)):
        prob = S["reduced"].ReducedTrackingProblem(op, mu, w0=w0)
        runs.append(S["lm"].lm_solve(prob, S["lm"].LmConfig(max_iters=20)))  # the reference's own LM loop
    a, b = runs
    assert a.reason == b.reason and a.n_iters == b.n_iters and a.history.shape == b.history.shape
    # decisions (iteration, lambda, alpha) and J to 1e-8; the gradient norms |S|, |T| relative to
    # their column scale (they are differences of O(1) terms; the state init drives |S| to rounding
    # level, and the GPU's summation order moves them by ~1e-7 of the scale)
    h, hr = b.history, a.history
    assert np.array_equal(h[:, 0], hr[:, 0]) and np.array_equal(h[:, 5], hr[:, 5], equal_nan=True)
    assert np.allclose(h[:, [1, 4]], hr[:, [1, 4]], rtol=1e-8, atol=0.0)
    for col in (2, 3):
        assert np.all(np.abs(h[:, col] - hr[:, col]) <= 1e-6 * np.max(np.abs(hr[:, col])))
    assert rel_err(b.w, a.w) < 1e-8 and abs(b.objective - a.objective) <= 1e-10 * abs(a.objective)


def test_train_weights_end_to_end(S):
    """strom.eqp.train_weights (LM solves -> build_lp -> solve_lp -> WeightVector) with the GPU
    operator and the GPU LM swapped in, vs the stock CPU run: LP matrix, weights, active set."""
    from paper_2305_15661_b200 import dropin

    eqp = S["eqp"]
    law, mesh, maps, geom, bases, dc = problem(S)
    cfg = eqp.EqpTrainingConfig(delta=0.1, xi=np.array([[4.0, 0.03], [6.0, 0.05], [8.0, 0.07]]))
    guess = eqp.WeightVector.ones(mesh.num_elements)
    lmc = S["lm"].LmConfig(max_iters=20)
    captured = {}
    orig_build = eqp.build_lp

    def spy(*a, **k):
        lp = orig_build(*a, **k)
        captured.setdefault("lp", []).append(lp)
        return lp

    eqp.build_lp = spy
    try:
        w_cpu, sol_cpu = eqp.train_weights(law, mesh, maps, bases, guess, cfg, dc, lmc, return_solutions=True)
        undo = dropin.install(lm=True)
        try:
            w_gpu, sol_gpu = eqp.train_weights(law, mesh, maps, bases, guess, cfg, dc, lmc, return_solutions=True)
        finally:
            undo()
    finally:
        eqp.build_lp = orig_build
    lp_cpu, lp_gpu = captured["lp"]
    for a, b in zip(sol_gpu, sol_cpu):  # training solutions of the LM solves
        assert rel_err(a.w, b.w) < 1e-8
    dA = float(np.max(np.abs(lp_gpu.A - lp_cpu.A)) / np.max(np.abs(lp_cpu.A)))
    print(f"\n[EQP LP] max |A_gpu - A_cpu| / max |A| = {dA:.2e}; active cpu {len(w_cpu.active)} gpu {len(w_gpu.active)}")
    assert dA < 1e-10
    assert np.allclose(lp_gpu.lo_row, lp_cpu.lo_row, rtol=1e-10) and np.allclose(lp_gpu.hi_row, lp_cpu.hi_row, rtol=1e-10)
    assert np.array_equal(w_gpu.active, w_cpu.active)  # same vertex of the LP
    assert rel_err(w_gpu.rho, w_cpu.rho) < 1e-8
