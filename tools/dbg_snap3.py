import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_configs import small_sector
import oracle.dual
from oracle.element import OracleGeometry, OracleReducedOperator
from paper_2305_15661_b200 import configs
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases, ReducedCoords
case = small_sector()
mus, U, X = configs.snapshot_fields(case, 3, seed=4)
geom = OracleGeometry(case.mesh, case.maps, case.quad_order)
s = 0
o2 = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, X[s]), case.dist, state_offset=U[s])
c = ReducedCoords(np.zeros(6), np.zeros(4))
Sv, Sf, Tv, Tf = o2.elemental_contributions(c, mus[s], split=True)
ref = OracleReducedOperator(case.law, geom, case.phi, case.psi, X[s], case.kappa, case.eps, state_offset=U[s])
rSv, rSf, rTv, rTf = ref.elemental_contributions(np.zeros(6), np.zeros(4), mus[s], split=True)
nbr, nf, flip, tag = case.mesh.neighbor_tables()
dv = np.abs(Sv - rSv).max(1) / np.abs(rSv).max(); df = np.abs(Sf - rSf).max(1) / np.abs(rSf).max()
for e in range(case.mesh.num_elements):
    if dv[e] > 1e-10 or df[e] > 1e-10:
        print(e, "dv %.2e df %.2e" % (dv[e], df[e]), "nbr", nbr[e], "tag", tag[e], "flip", flip[e])
print("max", dv.max(), df.max())
