import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_configs import small_sector
import oracle.dual
from oracle.element import OracleGeometry, OracleReducedOperator
from paper_2305_15661_b200 import configs, laws as L
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases, ReducedCoords
case = small_sector()
mus, U, X = configs.snapshot_fields(case, 3, seed=4)
geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
ne = case.mesh.num_elements
ff = np.tile(L.euler_freestream(mus[0][0]), ne * 6)
rng = np.random.default_rng(0)
variants = {
 "uniform_ff_nodisp": (ff, case.mesh.nodes.ravel()),
 "jitter_nodisp": (U[0], case.mesh.nodes.ravel()),
 "uniform_disp": (ff, X[0]),
 "jitter_disp": (U[0], X[0]),
 "jitter_v_nodisp": (U[0] + np.tile([0, 0, 0.1, 0], ne * 6) * rng.random(ne*24), case.mesh.nodes.ravel()),
}
for name, (u0, x) in variants.items():
    o2 = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, x), case.dist, state_offset=u0)
    a = o2.derivatives(ReducedCoords(np.zeros(6), np.zeros(4)), mus[0])
    ref = OracleReducedOperator(case.law, geom, case.phi, case.psi, x, case.kappa, case.eps, state_offset=u0)
    b = ref.derivatives(np.zeros(6), np.zeros(4), mus[0])
    print(name, " ".join("%s:%.1e" % (n, np.max(np.abs(np.asarray(p) - q)) / max(np.max(np.abs(q)), 1e-300)) for p, q, n in zip(a, b, "J S T Hww Hwt Htt".split())))
