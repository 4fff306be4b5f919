"""The paper's Burgers workflow end to end on the GPU (SPEC greedy-driver; §4.1): seed
by a full-space tracking solve, greedy search over a candidate grid, snapshot alignment, HDM
solve + tracking, Gram-Schmidt growth, EQP weights (all-ones here: the LP needs the reference)."""
import os, sys, time, warnings
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_15661_b200 import configs, laws as L
from paper_2305_15661_b200.eqp import WeightVector
from paper_2305_15661_b200.fullspace import assemble_global
from paper_2305_15661_b200.greedy import greedy_train, tracking_alignment, tracking_snapshot
from paper_2305_15661_b200.lm import LmConfig
from paper_2305_15661_b200.mesh import build_box_mesh, get_geometry

nx, ny = int(os.environ.get("NX", 8)), int(os.environ.get("NY", 6))
mesh, maps = build_box_mesh(((0.0, 0.0), (2.0, 1.0)), nx, ny, degree_sol=2, n_comp=1)
law = L.burgers_spacetime()
geom, ne = get_geometry(mesh, maps), mesh.num_elements
dist = configs.DistortionConfig(1e-3)
cands = np.array([[a, b] for a in (3.0, 6.0, 9.0) for b in (0.02, 0.0475, 0.075)])
train = lambda bases, guess, mus: WeightVector.ones(ne)  # noqa: E731
t0 = time.perf_counter()
with warnings.catch_warnings(record=True) as wlist:
    warnings.simplefilter("always")
    st = greedy_train(law, geom, cands, tracking_snapshot(law, geom, dist, LmConfig(max_iters=int(os.environ.get('TRACK_ITERS', 60)))), 3, dist, train,
                      LmConfig(max_iters=10), align=tracking_alignment(law, geom, dist, LmConfig(max_iters=10)))
print(f"greedy: {time.perf_counter() - t0:.1f} s, selected {[cands[i].tolist() for i in st.selected]}")
print("warnings:", [str(w.message)[:90] for w in wlist][:6])
X = mesh.nodes.ravel()
for (U, x), i in zip(st.snapshots, st.selected):
    R = assemble_global(law, mesh, maps, U, x, cands[i], want_jacobians=False, geom=geom)[0]
    print(f" mu={cands[i].tolist()} |R|={np.linalg.norm(R):.2e} max|x-X|={np.max(np.abs(x - X)):.3e} u in [{U.min():.3f}, {U.max():.3f}]")
print("metrics:", [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in m.items()} for m in st.metrics])
