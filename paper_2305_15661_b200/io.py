"""Persistence and interop: the reference's plain-text ``stmesh`` format
(strom/meshing.py:385-456), the LM history CSV (strom/lm.py:67-70), and the greedy driver's
metrics CSV and model bundle (SPEC greedy-driver "External Interfaces").

The formats are the reference's, byte for byte where it defines them, so meshes and
histories move between the two implementations (tests/test_io.py round-trips them through
the unmodified reference).
"""

import numpy as np

from .mesh import MeshError, ReferenceMesh

HISTORY_HEADER = "iter,objective,grad_w_norm,grad_tau_norm,lambda,alpha"
METRICS_COLUMNS = ("j", "mu", "e_rom", "e_eqp", "r_rom", "r_eqp", "T_gs", "T_rho", "T_tst_rom", "T_tst_eqp",
                   "sparsity")


def save_mesh(mesh, path):
    """stmesh: "stmesh <dim> <q> <N_v> <N_e>", node rows (repr floats), 0-based connectivity
    rows, "tags <n>" + "<name> <id>" rows (by id), "faces <n_int> <n_bnd>", "i eL fL eR fR"
    and "b e f tag" rows."""
    lines = [f"stmesh {mesh.dim} {mesh.degree_geo} {mesh.num_nodes} {mesh.num_elements}"]
    lines += [" ".join(repr(float(c)) for c in p) for p in np.asarray(mesh.nodes)]
    lines += [" ".join(str(int(i)) for i in conn) for conn in np.asarray(mesh.elements)]
    lines.append(f"tags {len(mesh.boundary_tags)}")
    lines += [f"{name} {tag}" for name, tag in sorted(mesh.boundary_tags.items(), key=lambda kv: kv[1])]
    lines.append(f"faces {len(mesh.interior_faces)} {len(mesh.boundary_faces)}")
    lines += ["i " + " ".join(str(int(v)) for v in row) for row in np.asarray(mesh.interior_faces)]
    lines += ["b " + " ".join(str(int(v)) for v in row) for row in np.asarray(mesh.boundary_faces)]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def load_mesh(path):
    """Read an stmesh file into a validated ReferenceMesh (blank lines ignored)."""
    with open(path) as fh:
        lines = [ln.strip() for ln in fh if ln.strip()]
    head = lines[0].split()
    if head[0] != "stmesh":
        raise MeshError("not an stmesh file")
    dim, q, nv, ne = (int(v) for v in head[1:5])
    k = 1
    nodes = np.array([[float(v) for v in lines[k + i].split()] for i in range(nv)]).reshape(nv, -1)
    k += nv
    elements = np.array([[int(v) for v in lines[k + i].split()] for i in range(ne)], dtype=np.int64).reshape(ne, -1)
    k += ne
    ntags = int(lines[k].split()[1])
    k += 1
    tags = {}
    for i in range(ntags):
        name, tid = lines[k + i].split()
        tags[name] = int(tid)
    k += ntags
    nif, nbf = (int(v) for v in lines[k].split()[1:3])
    k += 1
    interior, boundary = [], []
    for ln in lines[k:k + nif + nbf]:
        parts = ln.split()
        (interior if parts[0] == "i" else boundary).append([int(v) for v in parts[1:]])
    mesh = ReferenceMesh(dim=dim, degree_geo=q, nodes=nodes, elements=elements,
                         interior_faces=np.asarray(interior, dtype=np.int64).reshape(-1, 4),
                         boundary_faces=np.asarray(boundary, dtype=np.int64).reshape(-1, 3), boundary_tags=tags)
    mesh.validate()
    return mesh


def history_csv(history, path):
    """LM convergence history rows (iter, J, |S|, |T|, lambda, alpha) as CSV (lm.py:67-70)."""
    np.savetxt(path, np.atleast_2d(history), delimiter=",", header=HISTORY_HEADER, comments="")


def greedy_metrics_csv(metrics, path):
    """greedy_metrics.csv (SPEC greedy-driver): one row per iteration; columns the driver did not
    measure (test-set errors, which need the HDM reference solutions) are left empty."""
    with open(path, "w") as fh:
        fh.write(",".join(METRICS_COLUMNS) + "\n")
        for m in metrics:
            row = []
            for c in METRICS_COLUMNS:
                v = m.get(c, m.get("active") if c == "sparsity" else None)
                if c == "mu" and v is not None:
                    v = " ".join(repr(float(x)) for x in np.atleast_1d(v))
                row.append("" if v is None else str(v))
            fh.write(",".join(row) + "\n")


def save_model(path, mesh, bases, weights, selected=None, snapshots=None):
    """Model bundle (SPEC greedy-driver): mesh fields, bases, EQP weights, training indices and
    snapshots in one .npz."""
    d = dict(nodes=mesh.nodes, elements=mesh.elements, interior_faces=mesh.interior_faces,
             boundary_faces=mesh.boundary_faces, tag_names=np.array(list(mesh.boundary_tags), dtype=str),
             tag_ids=np.array(list(mesh.boundary_tags.values()), dtype=np.int64), dim=mesh.dim, q=mesh.degree_geo,
             phi=bases.phi, psi=bases.psi, ref_coords=bases.ref_coords, rho=np.asarray(weights.rho),
             selected=np.asarray(selected if selected is not None else [], dtype=np.int64))
    for i, (U, x) in enumerate(snapshots or []):
        d[f"snapshot{i}_U"], d[f"snapshot{i}_x"] = U, x
    np.savez_compressed(path, **d)


def load_model(path):
    """(mesh, bases, weights, selected, snapshots) from a bundle written by save_model."""
    from .eqp import WeightVector
    from .reduced import ReducedBases

    with np.load(path) as z:
        mesh = ReferenceMesh(dim=int(z["dim"]), degree_geo=int(z["q"]), nodes=z["nodes"], elements=z["elements"],
                             interior_faces=z["interior_faces"], boundary_faces=z["boundary_faces"],
                             boundary_tags={str(n): int(t) for n, t in zip(z["tag_names"], z["tag_ids"])})
        bases = ReducedBases(z["phi"], z["psi"], z["ref_coords"])
        snaps, i = [], 0
        while f"snapshot{i}_U" in z.files:
            snaps.append((z[f"snapshot{i}_U"], z[f"snapshot{i}_x"]))
            i += 1
        return mesh, bases, WeightVector(z["rho"]), z["selected"].tolist(), snaps
