"""Config-shape parity against the unmodified reference (tests/golden/make_golden.py):

* cfg1 exactly as BASELINE states it (64 cells, 10 EQP elements, 8 mu): full LM
  histories of strom.lm.lm_solve (lm.py:164-271), row for row;
* K = 30 and K = 36 (the specialised <20,10> / <24,12> DMMA kernels of configs 3
  and 5) on a reduced half-cylinder sector: LM histories row for row;
* config 4's LP rows at (k_u, k_x) = (20, 10) over three explicit snapshots.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from cases import load, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def gpu_op(case):
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

    return GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist,
                              state_offset=case.state_offset)


def with_inputs(case, g):
    case.phi, case.psi, case.ref_coords, case.mus = g["phi"], g["psi"], g["ref_coords"], g["mus"]
    case.rho = g["rho"] if g["rho"].size else None
    return case


def same_decision(a, b, jtol=1e-8):
    """History rows (it, J, |S|, |T|, lambda, alpha): identical discrete decisions (iteration,
    step length alpha, damping lambda), objective to jtol."""
    return (a[0] == b[0] and np.isclose(a[4], b[4], rtol=1e-8, atol=0.0)
            and ((np.isnan(a[5]) and np.isnan(b[5])) or a[5] == b[5])
            and np.isclose(a[1], b[1], rtol=jtol, atol=0.0))


# ROM-solution tolerance per case.  K = 36 is ill-conditioned enough that the reference's own
# 15-iteration trajectory moves by up to ~6e-8 in the objective when each evaluation carries
# 1-ulp noise (tests/test_lm_sensitivity.py measures this floor with the oracle, which is
# bit-identical to the reference); no implementation that sums in a different order can hold
# 1e-10 there, so that case is held to 3e-7.
OBJ_TOL = {"cfg1": 1e-10, "sector_k30": 1e-10, "sector_k36": 3e-7}
# intermediate history objectives at K = 36 sit further from convergence and move more (measured
# 1.4e-7 at row 10 while every decision and the final objective agree)
HIST_TOL = {"cfg1": 1e-8, "sector_k30": 1e-8, "sector_k36": 1e-6}


def check_lm(case, g, w0, P, obj_tol=1e-10, hist_tol=1e-8):
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.lm import LmConfig, lm_solve_batched

    op = gpu_op(case)
    cfg = LmConfig(max_iters=int(g["lm_max_iters"]))
    res = lm_solve_batched(op, case.mus[:P], w0, None, WeightVector(case.rho), cfg)
    for i, r in enumerate(res):
        hr = g[f"lm{i}_hist"]
        assert len(r.history) == len(hr), (i, len(r.history), len(hr))
        for row, (a, b) in enumerate(zip(r.history, hr)):
            assert same_decision(a, b, hist_tol), (i, row, a, b)
        assert r.reason == str(g[f"lm{i}_reason"]) and r.n_iters == int(g[f"lm{i}_iters"])
        assert r.converged == bool(g[f"lm{i}_conv"])
        assert rel_err(r.w, g[f"lm{i}_w"]) < 1e-8 and rel_err(r.tau, g[f"lm{i}_tau"], max(1e-12, np.max(np.abs(g[f"lm{i}_tau"])))) < 1e-6
        assert abs(r.objective - float(g[f"lm{i}_obj"])) <= obj_tol * abs(float(g[f"lm{i}_obj"]))


def test_cfg1_lm_histories_match_reference():
    from paper_2305_15661_b200 import configs

    g = load("cfg1")
    case = with_inputs(configs.strip_case(), g)
    assert case.mesh.num_elements == 128 and int(np.count_nonzero(case.rho)) == 10 and len(case.mus) == 8
    check_lm(case, g, None, 8, OBJ_TOL["cfg1"], HIST_TOL["cfg1"])


@pytest.mark.parametrize("name,ku,kx,P,seed", [("sector_k30", 20, 10, 4, 51), ("sector_k36", 24, 12, 3, 52)])
def test_sector_lm_histories_match_reference(name, ku, kx, P, seed):
    from paper_2305_15661_b200 import configs

    g = load(name)
    nr, nc = (int(v) for v in g["nrnc"])
    case = with_inputs(configs.sector_rom_case(n_radial=nr, n_circ=nc, ku=ku, kx=kx, frac_active=0.25, rho_scale=4.0,
                                               P=P, seed=seed, wall="extrapolate"), g)
    check_lm(case, g, g["w"], P, OBJ_TOL[name], HIST_TOL[name])  # w0 = Phi^T U_ff(3), as configs.sector_rom_case


def test_cfg4_lprows_match_reference():
    from paper_2305_15661_b200 import configs

    g = load("lprows")
    case = with_inputs(configs.sector_rom_case(n_radial=6, n_circ=10, ku=20, kx=10, frac_active=0.2, rho_scale=5.0,
                                               P=2, seed=41, wall="extrapolate"), g)
    op = gpu_op(case)
    U, X = torch.as_tensor(g["snap_U"]).cuda(), torch.as_tensor(g["snap_X"]).cuda()
    rows = op.contributions_at_snapshots(U, X, g["snap_mus"], "lprows").cpu().numpy()
    want = g["lprows"]
    assert rows.shape == want.shape
    for s in range(want.shape[0]):
        for k in range(want.shape[1]):
            assert rel_err(rows[s, k], want[s, k], np.max(np.abs(want[s, :-1])) if k < want.shape[1] - 1 else None) < 1e-10, (s, k)
