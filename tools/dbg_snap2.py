import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_configs import small_sector
import oracle.dual
from oracle.element import OracleGeometry, OracleReducedOperator, assemble_residual
from paper_2305_15661_b200 import configs
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases, ReducedCoords
case = small_sector()
mus, U, X = configs.snapshot_fields(case, 3, seed=4)
geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
for s in range(1):
    o2 = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, X[s]), case.dist, state_offset=U[s])
    c = ReducedCoords(np.zeros(6), np.zeros(4))
    R = o2.global_residual(c, mus[s])
    Rr = assemble_residual(case.law, geom, U[s], X[s], mus[s])
    print("resid", np.max(np.abs(R - Rr)), np.max(np.abs(Rr)))
    ref = OracleReducedOperator(case.law, geom, case.phi, case.psi, X[s], case.kappa, case.eps, state_offset=U[s])
    print("obj", o2.objective(c, mus[s]), ref.objective(np.zeros(6), np.zeros(4), mus[s]))
    a = o2.derivatives(c, mus[s]); b = ref.derivatives(np.zeros(6), np.zeros(4), mus[s])
    for x, y, n in zip(a, b, "J S T Hww Hwt Htt".split()):
        print(n, np.max(np.abs(np.asarray(x) - y)) / max(np.max(np.abs(y)), 1e-300))
    # per element: which elements differ in residual
    d = np.abs(R - Rr).reshape(-1, 24).max(1)
    bad = np.nonzero(d > 1e-12 * np.max(np.abs(Rr)))[0]
    print("bad elements", bad, case.mesh.neighbor_tables()[3][bad] if len(bad) else None)
