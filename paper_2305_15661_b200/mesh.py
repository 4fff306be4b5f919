"""Reference meshes, assembly maps and the light geometry handle.

Mirrors the data model of ``strom/meshing.py`` (``ReferenceMesh``
:23-163, ``neighbor_tables`` :83-110, ``AssemblyMaps`` :166-220) with the
same attribute names, so reference objects and these can be passed to the
GPU operator interchangeably.  Face discovery is vectorised (sort of the
edge keys) instead of a Python dict walk, which matters at 400k
triangles; per-(element, face) adjacency is identical to the reference's.

Mesh generators: the reference box mesher ordering (meshing.py:281-334),
a 64x1 strip for config 1, and the body-fitted annular sector around a
half cylinder (configs 3-5), which the reference cannot express through
its box-only face tagger (meshing.py:361-362).
"""

from dataclasses import dataclass, field

import numpy as np

from .tables import LOCAL_EDGES, lagrange_nodes

BOX_TAGS = {"left": 0, "right": 1, "bottom": 2, "top": 3}
SECTOR_TAGS = {"inflow": 0, "outflow": 1, "wall": 2}


class MeshError(ValueError):
    pass


def _edge_table(elements):
    """(ne*3, 2) sorted node pairs, in (element, local face) order."""
    e = np.asarray(elements)[:, :3]
    a = np.stack([e[:, f0] for f0, _ in LOCAL_EDGES], axis=1).reshape(-1)
    b = np.stack([e[:, f1] for _, f1 in LOCAL_EDGES], axis=1).reshape(-1)
    return np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1)


def discover_faces(elements):
    """Interior pairs (el, fl, er, fr) and boundary (e, f) sorted by node key."""
    keys = _edge_table(elements)
    order = np.lexsort((keys[:, 1], keys[:, 0]))  # stable: element order kept
    k = keys[order]
    same = np.all(k[1:] == k[:-1], axis=1)
    if np.any(same[1:] & same[:-1]):
        raise MeshError("an edge is shared by more than two elements")
    first = np.flatnonzero(same)
    pair_a, pair_b = order[first], order[first + 1]
    in_pair = np.zeros(len(order), dtype=bool)
    in_pair[first] = True
    in_pair[first + 1] = True
    single = order[~in_pair]
    interior = np.stack([pair_a // 3, pair_a % 3, pair_b // 3, pair_b % 3], axis=1)
    boundary = np.stack([single // 3, single % 3], axis=1)
    return interior.astype(np.int64), boundary.astype(np.int64)


@dataclass
class ReferenceMesh:
    dim: int
    degree_geo: int
    nodes: np.ndarray
    elements: np.ndarray
    interior_faces: np.ndarray
    boundary_faces: np.ndarray
    boundary_tags: dict = field(default_factory=dict)

    def __post_init__(self):
        self.nodes = np.asarray(self.nodes, dtype=float)
        self.elements = np.asarray(self.elements, dtype=np.int64)
        self.interior_faces = np.asarray(self.interior_faces, dtype=np.int64).reshape(-1, 4)
        self.boundary_faces = np.asarray(self.boundary_faces, dtype=np.int64).reshape(-1, 3)
        self._neighbor_cache = None

    @property
    def num_nodes(self):
        return self.nodes.shape[0]

    @property
    def num_elements(self):
        return self.elements.shape[0]

    def vertex_coords(self):
        return self.nodes[self.elements[:, :3]]

    def element_areas(self):
        v = self.vertex_coords()
        d1, d2 = v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]
        return 0.5 * (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0])

    def neighbor_tables(self):
        """(nbr_elem, nbr_face, nbr_flip, face_tag), each (ne, 3); meshing.py:83-110."""
        if self._neighbor_cache is not None:
            return self._neighbor_cache
        ne = self.num_elements
        nbr_elem = -np.ones((ne, 3), dtype=np.int64)
        nbr_face = -np.ones((ne, 3), dtype=np.int64)
        nbr_flip = np.zeros((ne, 3), dtype=bool)
        face_tag = -np.ones((ne, 3), dtype=np.int64)
        if len(self.interior_faces):
            el, fl, er, fr = self.interior_faces.T
            nbr_elem[el, fl], nbr_face[el, fl] = er, fr
            nbr_elem[er, fr], nbr_face[er, fr] = el, fl
            start = np.array([a for a, _ in LOCAL_EDGES])
            flip = self.elements[el, start[fl]] != self.elements[er, start[fr]]
            nbr_flip[el, fl] = flip
            nbr_flip[er, fr] = flip
        if len(self.boundary_faces):
            e, f, t = self.boundary_faces.T
            face_tag[e, f] = t
        self._neighbor_cache = (nbr_elem, nbr_face, nbr_flip, face_tag)
        return self._neighbor_cache

    def validate(self):
        if self.dim != 2:
            raise MeshError("only 2D simplex meshes are supported")
        areas = self.element_areas()
        if np.any(areas <= 0.0):
            raise MeshError(f"element {int(np.argmin(areas))} has non-positive orientation")
        interior, boundary = discover_faces(self.elements)
        if len(interior) != len(self.interior_faces) or len(boundary) != len(self.boundary_faces):
            raise MeshError("face records inconsistent with element connectivity")
        return True


class AssemblyMaps:
    """State / neighbor / coordinate index maps (meshing.py:166-220).

    The maps are materialised lazily: the GPU path never needs them (it
    derives every index from the element id and the neighbor table), only
    the CPU oracle and reference-compatible callers do.
    """

    def __init__(self, mesh, degree_sol=1, n_comp=1):
        self._mesh = mesh
        self.degree_sol = int(degree_sol)
        self.n_comp = int(n_comp)
        self.n_basis = lagrange_nodes(self.degree_sol).shape[0]
        self.n_u = self.n_basis * self.n_comp
        self.n_global_state = mesh.num_elements * self.n_u
        self.n_global_coord = 2 * mesh.num_nodes
        self._state = self._neighbor = self._coord = None

    @property
    def state_map(self):
        if self._state is None:
            ne = self._mesh.num_elements
            self._state = np.arange(ne, dtype=np.int64)[:, None] * self.n_u + np.arange(self.n_u)[None, :]
        return self._state

    @property
    def neighbor_map(self):
        if self._neighbor is None:
            nbr, _, _, _ = self._mesh.neighbor_tables()
            out = -np.ones((self._mesh.num_elements, 3 * self.n_u), dtype=np.int64)
            for f in range(3):
                has = nbr[:, f] >= 0
                out[has, f * self.n_u:(f + 1) * self.n_u] = self.state_map[nbr[has, f]]
            self._neighbor = out
        return self._neighbor

    @property
    def coord_map(self):
        if self._coord is None:
            el = self._mesh.elements
            out = np.empty((el.shape[0], 2 * el.shape[1]), dtype=np.int64)
            out[:, 0::2] = 2 * el
            out[:, 1::2] = 2 * el + 1
            self._coord = out
        return self._coord


def build_assembly_maps(mesh, degree_sol=1, n_comp=1):
    return AssemblyMaps(mesh, degree_sol, n_comp)


def _tag_boundary(boundary, elements, tag_of_edge):
    e, f = boundary[:, 0], boundary[:, 1]
    start = np.array([a for a, _ in LOCAL_EDGES])[f]
    end = np.array([b for _, b in LOCAL_EDGES])[f]
    na, nb = elements[e, start], elements[e, end]
    tags = tag_of_edge(na, nb)
    return np.stack([e, f, tags], axis=1).astype(np.int64)


def build_box_mesh(domain_box, nx, ny, degree_sol=1, n_comp=1):
    """Box split into 2*nx*ny triangles, reference ordering (meshing.py:281-334).

    Cell (i, j) yields elements (v00, v10, v11) and (v00, v11, v01); node
    id j*(nx+1)+i; straight (q=1) geometry only.
    """
    box = np.asarray(domain_box, dtype=float).reshape(2, 2)
    (x0, y0), (x1, y1) = box
    if nx < 1 or ny < 1:
        raise ValueError("nx and ny must be >= 1")
    if abs((x1 - x0) * (y1 - y0)) < 1e-300:
        raise ValueError("degenerate domain box (zero area)")
    xs, ys = np.linspace(x0, x1, nx + 1), np.linspace(y0, y1, ny + 1)
    X, Y = np.meshgrid(xs, ys, indexing="xy")
    nodes = np.column_stack([X.ravel(), Y.ravel()])
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    v00 = (j * (nx + 1) + i).ravel()
    v10, v11, v01 = v00 + 1, v00 + nx + 2, v00 + nx + 1
    elements = np.empty((2 * nx * ny, 3), dtype=np.int64)
    elements[0::2] = np.stack([v00, v10, v11], axis=1)
    elements[1::2] = np.stack([v00, v11, v01], axis=1)
    interior, bnd = discover_faces(elements)
    tol = 1e-9 * max(abs(x1 - x0), abs(y1 - y0))

    def tag(na, nb):
        mid = 0.5 * (nodes[na] + nodes[nb])
        t = np.full(len(na), -1, dtype=np.int64)
        for name, test in (("top", abs(mid[:, 1] - y1) < tol), ("bottom", abs(mid[:, 1] - y0) < tol),
                           ("right", abs(mid[:, 0] - x1) < tol), ("left", abs(mid[:, 0] - x0) < tol)):
            t[test] = BOX_TAGS[name]  # later names win, matching the reference's if-chain order
        if np.any(t < 0):
            raise MeshError("boundary face not on the box boundary")
        return t

    boundary = _tag_boundary(bnd, elements, tag)
    mesh = ReferenceMesh(2, 1, nodes, elements, interior, boundary, dict(BOX_TAGS))
    return mesh, build_assembly_maps(mesh, degree_sol, n_comp)


def build_sector_mesh(n_radial, n_circ, r_inner=0.5, r_outer=1.5, degree_sol=2, n_comp=4):
    """Body-fitted annular sector upstream of a half cylinder.

    r in [r_inner, r_outer], theta in [pi/2, 3pi/2] (flow along +x hits the
    cylinder at theta = pi).  Node (i, j) = radial i, circumferential j,
    id j*(n_radial+1)+i; quads split like the box mesher, which keeps every
    triangle counter-clockwise because (r, theta) -> (x, y) has det r > 0.
    Tags: inner arc "wall", outer arc "inflow", the two cuts "outflow".
    """
    nr, nc = int(n_radial), int(n_circ)
    r = np.linspace(r_inner, r_outer, nr + 1)
    th = np.linspace(0.5 * np.pi, 1.5 * np.pi, nc + 1)
    TH, R = np.meshgrid(th, r, indexing="ij")  # (nc+1, nr+1): j-major
    nodes = np.column_stack([(R * np.cos(TH)).ravel(), (R * np.sin(TH)).ravel()])
    j, i = np.meshgrid(np.arange(nc), np.arange(nr), indexing="ij")
    v00 = (j * (nr + 1) + i).ravel()
    v10, v11, v01 = v00 + 1, v00 + nr + 2, v00 + nr + 1
    elements = np.empty((2 * nr * nc, 3), dtype=np.int64)
    elements[0::2] = np.stack([v00, v10, v11], axis=1)
    elements[1::2] = np.stack([v00, v11, v01], axis=1)
    interior, bnd = discover_faces(elements)

    def tag(na, nb):
        ia, ja = na % (nr + 1), na // (nr + 1)
        ib, jb = nb % (nr + 1), nb // (nr + 1)
        t = np.full(len(na), -1, dtype=np.int64)
        t[(ia == 0) & (ib == 0)] = SECTOR_TAGS["wall"]
        t[(ia == nr) & (ib == nr)] = SECTOR_TAGS["inflow"]
        t[((ja == 0) & (jb == 0)) | ((ja == nc) & (jb == nc))] = SECTOR_TAGS["outflow"]
        if np.any(t < 0):
            raise MeshError("sector boundary face not on a boundary arc or cut")
        return t

    boundary = _tag_boundary(bnd, elements, tag)
    mesh = ReferenceMesh(2, 1, nodes, elements, interior, boundary, dict(SECTOR_TAGS))
    return mesh, build_assembly_maps(mesh, degree_sol, n_comp)


class Geometry:
    """Light geometry handle: the mesh, maps and rule order the GPU needs.

    The reference's ``Geometry`` (geometry.py:29-196) precomputes
    O(ne*nq*nb) per-element tables; the GPU recomputes every per-element
    quantity from the nodal coordinates, so this handle only carries the
    identity of the discretisation.  A reference ``Geometry`` is accepted
    wherever this one is.
    """

    def __init__(self, mesh, maps, quad_order=None):
        self.mesh = mesh
        self.maps = maps
        p, q = maps.degree_sol, mesh.degree_geo
        self.quad_order = 2 * q + 2 * p + 1 if quad_order is None else int(quad_order)
        self.n_basis = lagrange_nodes(p).shape[0]
        self.n_comp = maps.n_comp
        self.n_geo = mesh.elements.shape[1]
        self.extras = {}

    @property
    def areas(self):
        return self.mesh.element_areas()

    @property
    def total_area(self):
        return float(np.sum(self.areas))


def get_geometry(mesh, maps, quad_order=None):
    key = (maps.degree_sol, maps.n_comp, quad_order)
    cache = mesh.__dict__.setdefault("_b200_geometry_cache", {})
    if key not in cache:
        cache[key] = Geometry(mesh, maps, quad_order)
    return cache[key]
