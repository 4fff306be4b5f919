"""Output guard bands for every strom_eval mode (compute-sanitizer is not usable on this GPU
pool): each mode writes into a slice of a larger sentinel-filled buffer; afterwards the bands on
both sides are untouched and the slice holds no sentinel (every output entry was written).  Run
for the DMMA kernel (Euler p = 2, generic and specialised reduced dimensions, 12- and 25-point
rules) and the warp kernel (scalar laws, p = 1 and 2), single and batched parameter points."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
GUARD = 4096
SENT = -7.25e300


def _check(op, mode, n, W, Tau, Mu, rho=None):
    big = torch.full((n + 2 * GUARD,), SENT, dtype=torch.float64, device=op.device)
    out = big[GUARD:GUARD + n]
    op.eval_batched(mode, W, Tau, Mu, rho, out=out, sync=True)
    torch.cuda.synchronize()
    assert bool((big[:GUARD] == SENT).all()) and bool((big[GUARD + n:] == SENT).all()), f"mode {mode}: guard band written"
    assert not bool((out == SENT).any()), f"mode {mode}: output entries left unwritten"
    assert bool(torch.isfinite(out).all())


@pytest.mark.parametrize("kind", ["euler_16_8", "euler_generic_q25", "sector_20_10_wall", "burgers_p2", "linadv_p1"])
def test_eval_modes_stay_inside_their_outputs(kind):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_15661_b200 import _lib, configs, laws as L
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.fullspace import test_space_tables
    from paper_2305_15661_b200.mesh import build_box_mesh, get_geometry
    from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases

    rng = np.random.default_rng(21)
    if kind == "euler_16_8":
        case = configs.euler_square_case(n=5, ku=16, kx=8, seed=3)
    elif kind == "euler_generic_q25":
        case = configs.euler_square_case(n=3, ku=7, kx=3, seed=4, quad_order=None)
    elif kind == "sector_20_10_wall":
        case = configs.sector_rom_case(n_radial=4, n_circ=7, ku=20, kx=10, frac_active=0.3, rho_scale=3.0, P=3, seed=5)
    else:
        p = 2 if kind == "burgers_p2" else 1
        mesh, maps = build_box_mesh(((0.0, 0.0), (2.0, 1.0)), 4, 3, degree_sol=p, n_comp=1)
        law = L.burgers_spacetime() if kind == "burgers_p2" else L.linear_advection((1.0, 0.5))
        ku, kx = 5, 3
        case = configs.Case(kind, law, mesh, maps, None, configs.orthonormal(rng, maps.n_global_state, ku),
                            configs.orthonormal(rng, maps.n_global_coord, kx), mesh.nodes.ravel().copy(),
                            np.array([[5.0, 0.05]]) if p == 2 else np.array([[0.5]]), None, None, None)
    op = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, case.ref_coords), case.dist,
                            state_offset=case.state_offset)
    ku, kx, ne, nu = op.k_u, op.k_x, case.mesh.num_elements, op.dm.nu
    K = ku + kx
    scalar = case.maps.n_comp == 1
    for P in (1, 3, 9):  # 9 >= 8: the many-point K2 path
        w0 = np.zeros(ku) if case.W is None else case.W[0]
        W = torch.as_tensor(np.tile(w0, (P, 1)) + (1.0 if scalar else 0.0) + 0.01 * rng.standard_normal((P, ku))).to(op.device)
        Tau = torch.as_tensor(1e-3 * rng.standard_normal((P, kx))).to(op.device)
        Mu = torch.as_tensor(np.resize(np.asarray(case.mus, dtype=float), (P, op.n_mu))).to(op.device)
        rho = None
        if case.rho is not None:
            rho = WeightVector(case.rho)
        sizes = {_lib.OBJECTIVE: P, _lib.RESNORM2: P, _lib.DERIVS: P * (1 + K + K * K), _lib.CONTRIB: P * ne * K,
                 _lib.CONTRIB_SPLIT: P * ne * 2 * K, _lib.RESIDUAL: P * ne * nu, _lib.CONTRIB_LPROWS: P * (K + 1) * ne}
        for mode, n in sizes.items():
            weighted = mode in (_lib.OBJECTIVE, _lib.DERIVS)
            _check(op, mode, n, W, Tau, Mu, rho if weighted else None)
    # element Jacobian records: plain (4-component p = 2 only) and against a bound test space
    W1, T1, M1 = W[:1].contiguous(), Tau[:1].contiguous(), Mu[:1].contiguous()
    if not scalar:
        _check(op, _lib.ELEMJAC, ne * (24 * 103 + 7), W1, T1, M1)
    for deg in (case.maps.degree_sol, case.maps.degree_sol + 1):
        phi_t, dphi_t, trace_t = test_space_tables(op.dm.tabs, deg)
        nbt = phi_t.shape[1]
        _lib.check(op._lib.strom_set_test_space(op._h, nbt, phi_t.ctypes.data, dphi_t.ctypes.data, trace_t.ctypes.data),
                   "strom_set_test_space")
        NT = nbt * case.maps.n_comp
        _check(op, _lib.ELEMJAC_ENRICHED, ne * (NT * (1 + 4 * nu + 6) + 7), W1, T1, M1)
