"""Host logic of the full-space path (no GPU): sliding-boundary DoF selection, test-space
tabulations and the cached CSR scatter, against the reference where it is installed and against
scipy's own COO -> CSR conversion."""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2305_15661_b200 import fullspace as F
from paper_2305_15661_b200.mesh import build_box_mesh, build_sector_mesh
from paper_2305_15661_b200.tables import element_tables
from paper_2305_15661_b200.tracking import boundary_slide_dofs


def _ref():
    try:
        from oracle import strom_ref

        return strom_ref.load()
    except ImportError:
        return None


def test_boundary_slide_dofs_box_and_reference():
    mesh, _ = build_box_mesh(((0.0, 0.0), (2.0, 1.0)), 4, 3, degree_sol=2, n_comp=1)
    free = boundary_slide_dofs(mesh)
    pts = mesh.nodes
    nx, ny = 5, 4
    assert len(free) == 2 * (nx - 2) * (ny - 2) + 2 * (nx - 2) + 2 * (ny - 2)  # interior both, edges tangential
    fixed = np.setdiff1d(np.arange(2 * len(pts)), free)
    for d in fixed:  # every pinned DoF is the normal coordinate of a boundary node
        v, i = divmod(int(d), 2)
        assert pts[v, i] in (pts[:, i].min(), pts[:, i].max())
    assert np.all(np.diff(free) > 0)
    S = _ref()
    if S is not None:
        import strom.tracking as strack

        rmesh, _ = S["meshing"].build_structured_mesh(((0.0, 0.0), (2.0, 1.0)), 4, 3, degree_sol=2, n_comp=1)
        assert np.array_equal(free, strack.boundary_slide_dofs(rmesh))


@pytest.mark.parametrize("p,qo", [(2, 6), (2, None), (1, None)])
def test_test_space_tables_match_reference_geometry(p, qo):
    tabs = element_tables(p, 1, qo)
    phi_t, dphi_t, trace_t = F.test_space_tables(tabs, p + 1)
    nbt = (p + 2) * (p + 3) // 2
    assert phi_t.shape == (tabs.nq, nbt) and dphi_t.shape == (tabs.nq, nbt, 2) and trace_t.shape == (3, tabs.ns, nbt)
    assert np.allclose(phi_t.sum(axis=1), 1.0) and np.allclose(dphi_t.sum(axis=1), 0.0, atol=1e-12)  # partition of unity
    assert np.allclose(trace_t.sum(axis=2), 1.0)
    # the trial space bound as its own test space reproduces the element tables
    phi_p, dphi_p, trace_p = F.test_space_tables(tabs, p)
    assert np.allclose(phi_p, tabs.phi, atol=1e-14) and np.allclose(dphi_p, tabs.dphi, atol=1e-13)
    for f in range(3):
        assert np.allclose(trace_p[f][:, tabs.fnodes[f]], tabs.trace[f], atol=1e-14)
    S = _ref()
    if S is not None and qo is None:
        rmesh, rmaps = S["meshing"].build_structured_mesh(((0.0, 0.0), (1.0, 1.0)), 2, 2, degree_sol=p, n_comp=1)
        g = S["geometry"].Geometry(rmesh, rmaps)
        ts = g.test_space(p + 1)
        e = 0  # undo the per-element weights: wphi = phi wq det_ref, wphi_face = ws len phi_face
        assert np.allclose(ts.wphi[e] / (g.wq[:, None] * g.det_ref[e]), phi_t, atol=1e-13)
        for f in range(3):
            assert np.allclose(ts.wphi_face[e, f] / (g.ws[:, None] * g.face_length[e, f]), trace_t[f], atol=1e-13)


@pytest.mark.parametrize("kind", ["box", "sector"])
def test_cached_csr_scatter_equals_scipy(kind):
    if kind == "box":
        mesh, maps = build_box_mesh(((0.0, 0.0), (1.0, 1.0)), 3, 2, degree_sol=2, n_comp=4)
    else:
        mesh, maps = build_sector_mesh(3, 4, degree_sol=2, n_comp=4)
    ne, rng = mesh.num_elements, np.random.default_rng(0)
    enriched = (np.arange(ne)[:, None] * 40 + np.arange(40)[None, :])[:, :, None]
    for NT, rows in ((24, maps.state_map[:, :, None]), (40, enriched)):
        n_rows = ne * NT
        for _ in range(2):  # the second call reuses the cached pattern with new values
            js, jn, jc = (rng.standard_normal((ne, NT, k)) for k in (24, 72, 6))
            A, B = F._scatter_csr(maps, rows, js, jn, jc, n_rows)
            nm = maps.neighbor_map
            r1, c1 = np.broadcast_to(rows, js.shape).ravel(), np.broadcast_to(maps.state_map[:, None, :], js.shape).ravel()
            r2 = np.broadcast_to(rows, jn.shape).ravel()
            c2 = np.broadcast_to(np.clip(nm, 0, None)[:, None, :], jn.shape).ravel()
            ref = sp.coo_matrix((np.concatenate([js.ravel(), (jn * (nm >= 0)[:, None, :]).ravel()]),
                                 (np.concatenate([r1, r2]), np.concatenate([c1, c2]))),
                                shape=(n_rows, maps.n_global_state)).tocsr()
            r3, c3 = np.broadcast_to(rows, jc.shape).ravel(), np.broadcast_to(maps.coord_map[:, None, :], jc.shape).ravel()
            refx = sp.coo_matrix((jc.ravel(), (r3, c3)), shape=(n_rows, maps.n_global_coord)).tocsr()
            assert A.nnz == ref.nnz and np.array_equal(A.indptr, ref.indptr) and np.array_equal(A.indices, ref.indices)
            assert np.allclose(A.data, ref.data, rtol=0, atol=1e-15)
            assert B.nnz == refx.nnz and abs(B - refx).max() == 0.0
