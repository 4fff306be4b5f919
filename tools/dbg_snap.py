import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_configs import small_sector, gpu_op
from paper_2305_15661_b200 import configs
from paper_2305_15661_b200.reduced import GpuReducedOperator, ReducedBases, ReducedCoords
case = small_sector()
mus, U, X = configs.snapshot_fields(case, 3, seed=4)
op = gpu_op(case)
rows = op.contributions_at_snapshots(torch.as_tensor(U).cuda(), torch.as_tensor(X).cuda(), mus, "total").cpu().numpy()
for s in range(3):
    o2 = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, X[s]), case.dist, state_offset=U[s])
    Se, Te = o2.elemental_contributions(ReducedCoords(np.zeros(6), np.zeros(4)), mus[s])
    print(s, np.max(np.abs(rows[s][:, :6] - Se)), np.max(np.abs(Se)))
    for mm in range(3):
        o3 = GpuReducedOperator(case.law, case.geom, ReducedBases(case.phi, case.psi, X[s]), case.dist, state_offset=U[s])
        Se3, _ = o3.elemental_contributions(ReducedCoords(np.zeros(6), np.zeros(4)), mus[mm])
        print("   mu", mm, np.max(np.abs(rows[s][:, :6] - Se3)))
