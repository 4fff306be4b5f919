"""Host-side reference-element tabulation: nodes, bases, quadrature.

Restates the reference's nodal Lagrange basis (``strom/basis.py:6-60``),
its quadrature rules (``strom/quadrature.py:46-104``) and the default rule
order ``2q+2p+1`` (``strom/geometry.py:46-47``), and adds the symmetric
degree-6, 12-point triangle rule the B200 configs use (SURVEY gap 4).
These tables are computed once on the host and copied into the CUDA
constant bank; nothing here runs on the hot path.
"""

from dataclasses import dataclass

import numpy as np

# local face f runs from vertex f to vertex (f+1)%3 (strom/meshing.py:16)
LOCAL_EDGES = ((0, 1), (1, 2), (2, 0))
_VERTS = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])


def lagrange_nodes(p):
    """Vertices, then edge nodes in edge order, then interior (basis.py:6-30)."""
    if p < 1:
        raise ValueError("degree must be >= 1")
    out = [_VERTS]
    if p >= 2:
        t = np.arange(1, p, dtype=float)[:, None] / p
        for a, b in LOCAL_EDGES:
            out.append((1.0 - t) * _VERTS[a] + t * _VERTS[b])
        inner = [(i / p, j / p) for i in range(1, p) for j in range(1, p - i)]
        if inner:
            out.append(np.array(inner, dtype=float))
    return np.vstack(out)


def _monomial_table(p, pts):
    x, y = pts[:, 0], pts[:, 1]
    v, vx, vy = [], [], []
    for i in range(p + 1):
        for j in range(p + 1 - i):
            v.append(x**i * y**j)
            vx.append(i * x ** max(i - 1, 0) * y**j if i else np.zeros_like(x))
            vy.append(j * x**i * y ** max(j - 1, 0) if j else np.zeros_like(x))
    return np.column_stack(v), np.column_stack(vx), np.column_stack(vy)


def lagrange_basis(p, pts):
    """Nodal basis values (npts, nb) and reference gradients (npts, nb, 2).

    Monomial Vandermonde inversion, as in basis.py:33-60.
    """
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    V, _, _ = _monomial_table(p, lagrange_nodes(p))
    C = np.linalg.inv(V)
    M, Mx, My = _monomial_table(p, pts)
    return M @ C, np.stack([Mx @ C, My @ C], axis=-1)


@dataclass(frozen=True)
class Rule:
    points: np.ndarray
    weights: np.ndarray
    order: int


def _s21(a):
    b = 1.0 - 2.0 * a
    return [(a, a), (b, a), (a, b)]


def _s111(a, b):
    c = 1.0 - a - b
    return [(b, c), (c, b), (a, c), (c, a), (a, b), (b, a)]


# published symmetric rules (weights relative to total 1), quadrature.py:46-64
_TRI = {
    1: ([(1.0 / 3.0, 1.0 / 3.0)], [1.0]),
    2: ([(1.0 / 6.0, 1.0 / 6.0), (2.0 / 3.0, 1.0 / 6.0), (1.0 / 6.0, 2.0 / 3.0)], [1.0 / 3.0] * 3),
    4: (_s21(0.445948490915965) + _s21(0.091576213509771),
        [0.223381589678011] * 3 + [0.109951743655322] * 3),
    5: ([(1.0 / 3.0, 1.0 / 3.0)] + _s21(0.470142064105115) + _s21(0.101286507323456),
        [0.225] + [0.132394152788506] * 3 + [0.125939180544827] * 3),
}


def _moment_residual(z):
    # unknowns: a1, w1, a2, w2, b1, c1, w3 of orbits S21, S21, S111
    a1, w1, a2, w2, b1, c1, w3 = z
    pts = np.array(_s21(a1) + _s21(a2) + _s111(b1, c1))
    wts = np.array([w1] * 3 + [w2] * 3 + [w3] * 6)
    res = []
    for i in range(7):
        for j in range(7 - i):
            exact = _tri_moment(i, j)
            res.append(np.dot(wts, pts[:, 0] ** i * pts[:, 1] ** j) - exact)
    return np.array(res)


def _tri_moment(i, j):
    # int over unit triangle of x^i y^j dx dy, normalised to total measure 1
    from math import factorial

    return 2.0 * factorial(i) * factorial(j) / factorial(i + j + 2)


def degree6_rule():
    """Symmetric 12-point rule exact to degree 6 (orbits S21, S21, S111).

    Solved here from the moment equations by Gauss-Newton, starting near
    the classical Strang-Fix/Dunavant values, so the tabulated numbers are
    exact to machine precision rather than to 15 printed digits.
    """
    z = np.array([0.2492867, 0.1167863, 0.0630890, 0.0508449, 0.0531450, 0.3103525, 0.0828511])
    for _ in range(50):
        r = _moment_residual(z)
        if np.max(np.abs(r)) < 1e-16:
            break
        Jm = np.empty((r.size, z.size))
        h = 1e-7
        for k in range(z.size):
            zp = z.copy(); zp[k] += h
            zm = z.copy(); zm[k] -= h
            Jm[:, k] = (_moment_residual(zp) - _moment_residual(zm)) / (2 * h)
        z = z - np.linalg.lstsq(Jm, r, rcond=None)[0]
    a1, w1, a2, w2, b1, c1, w3 = z
    pts = _s21(a1) + _s21(a2) + _s111(b1, c1)
    wts = [w1] * 3 + [w2] * 3 + [w3] * 6
    return pts, wts


_TRI[6] = degree6_rule()


def interval_rule(order):
    """Gauss-Legendre on [0, 1] exact to ``order`` (quadrature.py:67-73)."""
    n = max(1, (order + 2) // 2)
    x, w = np.polynomial.legendre.leggauss(n)
    return Rule(0.5 * (x + 1.0), 0.5 * w, 2 * n - 1)


def _collapsed_rule(order):
    # Duffy square (quadrature.py:76-89): (x, y) = (s, t(1-s)), jac (1-s)
    n = max(1, (order + 3) // 2)
    x, w = np.polynomial.legendre.leggauss(n)
    s, ws = 0.5 * (x + 1.0), 0.5 * w
    S, T = np.meshgrid(s, s, indexing="ij")
    WS, WT = np.meshgrid(ws, ws, indexing="ij")
    pts = np.column_stack([S.ravel(), (T * (1.0 - S)).ravel()])
    return Rule(pts, (WS * WT * (1.0 - S)).ravel(), order)


def triangle_rule(order):
    """Positive symmetric rule exact to ``order`` (quadrature.py:92-104)."""
    order = max(order, 1)
    for deg in sorted(_TRI):
        if deg >= order:
            pts, wts = _TRI[deg]
            return Rule(np.asarray(pts, dtype=float), 0.5 * np.asarray(wts, dtype=float), deg)
    return _collapsed_rule(order)


def install_degree6_rule(quadrature_module):
    """Inject the 12-point rule into a reference ``strom.quadrature`` module.

    Test-side helper for the oracle pins (SURVEY §8c iii); never used by
    the product path.
    """
    quadrature_module._TRI_RULES[6] = (list(map(tuple, _TRI[6][0])), list(_TRI[6][1]))


def face_nodes(p):
    """Element-local node ids on each face, ordered start vertex, end vertex,
    then edge-interior nodes along the edge (lagrange_nodes layout)."""
    out = []
    for f, (a, b) in enumerate(LOCAL_EDGES):
        out.append([a, b] + [3 + f * (p - 1) + i for i in range(p - 1)])
    return np.array(out, dtype=np.int64)


@dataclass
class ElementTables:
    """All reference-element constants the CUDA kernel needs.

    ``phi[q, n]``, ``dphi[q, n, k]``, ``wq[q]`` on the volume rule;
    ``trace[f, s, j]`` = value at face point s of face f of the j-th face
    node (``face_nodes``), ``ws[s]``, face points ``s``; ``bary[q, 3]`` the
    linear-geometry shape functions at volume points (positions).
    """

    p: int
    nb: int
    nq: int
    ns: int
    quad_order: int
    phi: np.ndarray
    dphi: np.ndarray
    wq: np.ndarray
    bary: np.ndarray
    s: np.ndarray
    ws: np.ndarray
    trace: np.ndarray
    fnodes: np.ndarray
    sol_nodes: np.ndarray


def element_tables(p, q=1, quad_order=None):
    if q != 1:
        raise NotImplementedError("B200 element kernel supports straight (q=1) geometry only")
    if quad_order is None:
        quad_order = 2 * q + 2 * p + 1
    vr = triangle_rule(quad_order)
    fr = interval_rule(quad_order)
    phi, dphi = lagrange_basis(p, vr.points)
    bary, _ = lagrange_basis(1, vr.points)
    fn = face_nodes(p)
    trace = np.empty((3, fr.points.size, fn.shape[1]))
    for f, (a, b) in enumerate(LOCAL_EDGES):
        pts = (1.0 - fr.points)[:, None] * _VERTS[a] + fr.points[:, None] * _VERTS[b]
        ph, _ = lagrange_basis(p, pts)
        trace[f] = ph[:, fn[f]]
    return ElementTables(
        p=p, nb=lagrange_nodes(p).shape[0], nq=vr.points.shape[0], ns=fr.points.size,
        quad_order=quad_order, phi=phi, dphi=dphi, wq=vr.weights, bary=bary,
        s=fr.points, ws=fr.weights, trace=trace, fnodes=fn, sol_nodes=lagrange_nodes(p),
    )
