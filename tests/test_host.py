"""CPU-only tests: C-ABI exports, host tables, meshes, law descriptors, bench model."""

import os
import re

import numpy as np
import pytest

from paper_2305_15661_b200 import _lib, laws as L, tables
from paper_2305_15661_b200.mesh import build_box_mesh, build_sector_mesh, discover_faces

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "strom_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|double|void|const char\*)\s+(strom_\w+)\(", src, re.M)))


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.SO_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTS)


def test_degree6_rule_exact():
    pts, wts = tables._TRI[6]
    pts, wts = np.asarray(pts), np.asarray(wts)
    assert len(wts) == 12 and np.all(wts > 0)
    for i in range(7):
        for j in range(7 - i):
            assert abs(np.dot(wts, pts[:, 0] ** i * pts[:, 1] ** j) - tables._tri_moment(i, j)) < 1e-15


@pytest.mark.parametrize("order,nq,ns", [(5, 7, 3), (6, 12, 4), (7, 25, 4)])
def test_rule_sizes(order, nq, ns):
    assert tables.triangle_rule(order).points.shape[0] == nq
    assert tables.interval_rule(order).points.size == ns


def test_lagrange_basis_partition_of_unity_and_nodal():
    for p in (1, 2, 3):
        nodes = tables.lagrange_nodes(p)
        phi, dphi = tables.lagrange_basis(p, nodes)
        assert np.allclose(phi, np.eye(len(nodes)), atol=1e-13)
        pts = np.random.default_rng(0).random((9, 2)) * 0.5
        v, g = tables.lagrange_basis(p, pts)
        assert np.allclose(v.sum(1), 1.0) and np.allclose(g.sum(1), 0.0, atol=1e-12)


def test_face_trace_table_is_edge_lagrange():
    et = tables.element_tables(2, quad_order=6)
    s = et.s
    # nodes at s = 0 (start), 1 (end), 1/2 (mid)
    L0 = 2 * (s - 0.5) * (s - 1.0)
    L1 = 2 * s * (s - 0.5)
    Lm = -4 * s * (s - 1.0)
    for f in range(3):
        assert np.allclose(et.trace[f], np.stack([L0, L1, Lm], 1), atol=1e-14)
    # reversing the points equals swapping the two vertex nodes (used for flipped neighbors)
    assert np.allclose(et.trace[0][::-1], et.trace[0][:, [1, 0, 2]], atol=1e-14)


def test_box_mesh_counts_and_orientation():
    mesh, maps = build_box_mesh(((0, 0), (100, 50)), 20, 10, degree_sol=2, n_comp=4)
    assert mesh.num_elements == 400
    assert len(mesh.boundary_faces) == 2 * (20 + 10)
    assert np.all(mesh.element_areas() > 0)
    assert abs(mesh.element_areas().sum() - 5000.0) < 1e-9
    mesh.validate()
    nbr, nface, flip, tag = mesh.neighbor_tables()
    # every interior adjacency is symmetric
    e, f = np.nonzero(nbr >= 0)
    assert np.all(nbr[nbr[e, f], nface[e, f]] == e)
    assert np.all(flip[nbr >= 0])  # consistently oriented box mesh: neighbors traverse faces reversed


def test_box_mesh_matches_reference_mesher():
    """Connectivity, faces and neighbor tables equal the reference mesher's
    (only where the reference is importable, i.e. in the dev container)."""
    import sys

    if not os.path.isdir("/root/reference/pkg/src"):
        pytest.skip("reference not available")
    sys.path.insert(0, "/root/reference/pkg/src")
    smesh = pytest.importorskip("strom.meshing")
    for nx, ny in [(1, 1), (3, 2), (7, 4)]:
        rm, rmaps = smesh.build_structured_mesh(((0, 0), (2, 1)), nx, ny, degree_sol=2, n_comp=4)
        mm, mmaps = build_box_mesh(((0, 0), (2, 1)), nx, ny, degree_sol=2, n_comp=4)
        assert np.array_equal(rm.elements, mm.elements)
        assert np.array_equal(rm.interior_faces, mm.interior_faces)
        assert np.array_equal(rm.boundary_faces, mm.boundary_faces)
        for a, b in zip(rm.neighbor_tables(), mm.neighbor_tables()):
            assert np.array_equal(a, b)
        assert np.array_equal(rmaps.neighbor_map, mmaps.neighbor_map)
        assert np.array_equal(rmaps.coord_map, mmaps.coord_map)


def test_sector_mesh():
    mesh, maps = build_sector_mesh(6, 8)
    mesh.validate()
    assert mesh.num_elements == 96
    tags = np.bincount(mesh.boundary_faces[:, 2], minlength=3)
    assert list(tags) == [8, 12, 8]  # inflow arc, two cuts, wall arc
    assert np.all(mesh.element_areas() > 0)


def test_discover_faces_detects_nonmanifold():
    el = np.array([[0, 1, 2], [1, 0, 3], [0, 1, 4]])
    with pytest.raises(ValueError):
        discover_faces(el)


def test_device_law_descriptors():
    d = L.device_law(L.euler(tags={"inflow": "freestream", "outflow": "extrapolate", "wall": "extrapolate"}),
                     {"inflow": 0, "outflow": 1, "wall": 2})
    assert d.law_id == L.LAW_EULER and d.bc_code_by_tag == {"inflow": 2, "outflow": 1, "wall": 1}
    d = L.device_law(L.burgers_spacetime(), {"left": 0, "right": 1, "bottom": 2, "top": 3})
    assert d.bc_code_by_tag == {"left": 2, "right": 1, "bottom": 3, "top": 1}
    with pytest.raises(NotImplementedError):
        L.device_law(type("X", (), {"name": "mystery", "dissipation": None, "needs_gradient": False})(), {})


def test_euler_flux_consistency():
    law = L.euler()
    u = L.euler_freestream(2.5)[None, :] * np.array([[1.0, 1.1, 0.0, 1.05]])
    u[0, 2] = 0.3
    f = law.flux(u, None, np.array([2.5]))
    assert f.shape == (1, 4, 2)
    rho, mx, my, E = u[0]
    p = 0.4 * (E - 0.5 * (mx * mx + my * my) / rho)
    assert np.allclose(f[0, :, 0], [mx, mx * mx / rho + p, mx * my / rho, (E + p) * mx / rho])


def test_flop_model_matches_survey():
    import bench

    assert bench.flops_per_element(12, 6, 4, 4, 3, 6, 16, 8) == 105144
