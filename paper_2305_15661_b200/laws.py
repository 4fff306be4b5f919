"""Conservation laws: host specs (reference plugin API) + device law ids.

The reference's law plugin is ``ConservationLawSpec`` (``strom/conslaw.py
:32-57``): Python callables ``flux``, ``source``, ``wavespeed`` and a BC
table keyed by mesh tag name.  Python callables cannot cross the C ABI, so
every law the GPU supports exists twice: (1) a reference-API spec whose
callables are written against a pluggable dual-number namespace (so the
reference kernel, the CPU oracle and plain numpy can all evaluate it), and
(2) a compiled device functor selected by ``law_id`` with a small double
parameter block.  ``device_law`` maps either one of these specs or one of
the reference's own law objects (by ``law.name``) to the
device descriptor; anything else raises ``NotImplementedError`` — there
is no CPU fallback.

Laws:
  * ``linear-advection``  (conslaw.py:174-253, no manufactured source)
  * ``burgers-spacetime`` (conslaw.py:94-163)
  * ``burgers-strip``     steady Burgers on a thin strip (config 1)
  * ``euler``             2-D compressible Euler (configs 2-5)
"""

from dataclasses import dataclass, field

import numpy as np

# device law ids / boundary codes (must match csrc/laws.cuh)
LAW_LINEAR_ADVECTION = 0
LAW_BURGERS_SPACETIME = 1
LAW_BURGERS_STRIP = 2
LAW_EULER = 3
LAW_EULER_ROE = 4
LAW_EULER_WALL = 5  # Euler (LLF) instantiated with slip-wall support (chosen when the mesh has walls)
LAW_LINADV_MS = 6   # linear advection with the manufactured solution ExpManufactured

BC_INTERIOR = 0
BC_EXTRAPOLATE = 1
BC_GHOST0 = 2  # prescribed ghost k -> BC_GHOST0 + k
BC_REFLECT = 31  # slip wall (Euler): ghost = state with the momentum mirrored in the face


# -- pluggable dual namespace -------------------------------------------------
_BACKENDS = {}


def register_dual_backend(cls, module):
    """Route math on instances of ``cls`` to ``module`` (exp, sqrt, ...)."""
    _BACKENDS[cls] = module


def _backend(*xs):
    for x in xs:
        mod = _BACKENDS.get(type(x))
        if mod is not None:
            return mod
    return None


def is_dual(x):
    return _backend(x) is not None


def value(x):
    return x.val if is_dual(x) else np.asarray(x)


def sqrt(x):
    b = _backend(x)
    return b.sqrt(x) if b else np.sqrt(x)


def exp(x):
    b = _backend(x)
    return b.exp(x) if b else np.exp(x)


def absolute(x):
    b = _backend(x)
    return b.absolute(x) if b else np.abs(x)


def stack(parts, axis):
    b = _backend(*parts)
    return b.stack(parts, axis=axis) if b else np.stack(parts, axis=axis)


def _comp_last(x):
    """(..., ) -> (..., 1): append a value axis keeping the tangent axis last."""
    b = _backend(x)
    if b is None:
        return np.asarray(x)[..., None]
    return b.expand(x, 1)


def _flux_from_rows(rows):
    """rows: list over components of (fx, fy) -> (..., m, 2)."""
    per_comp = [stack([fx, fy], axis=-1) for fx, fy in rows]
    return stack(per_comp, axis=-2)


# -- reference-API objects -----------------------------------------------------
@dataclass
class BoundaryCondition:
    kind: str  # "prescribed" | "extrapolate" | "reflect" (slip wall, GPU-only extension)
    value: object = None
    ghost_id: int = -1  # device ghost selector for prescribed kinds


@dataclass
class LawSpec:
    """Drop-in for ``ConservationLawSpec`` plus the device descriptor."""

    name: str
    n_comp: int
    dim: int
    flux: object
    source: object
    flux_jac: object
    wavespeed: object
    boundary_data: dict
    param_domain: np.ndarray
    initial_state: object = None
    needs_gradient: bool = False
    dissipation: object = None
    extra_dissipation: float = 0.0
    # extension (no reference counterpart): matrix dissipation D(u_in, u_out, nhat, mu), (..., m),
    # with H = (f_in + f_out).ntil / 2 - sigma D / 2 (Roe); None = the reference's LLF
    numflux: object = None
    law_id: int = -1
    params: tuple = ()

    def bc(self, tag_name):
        return self.boundary_data[tag_name]


def _const_state(pos, vals):
    vals = np.asarray(vals, dtype=float)
    return np.broadcast_to(vals, np.shape(pos)[:-1] + vals.shape).copy()


def _zero_like(x):
    return 0.0 * x


class ExpManufactured:
    """Manufactured solution u(x, y) = a0 + a1 exp(k1 x + k2 y) with a compiled device counterpart.

    ``u`` and ``grad`` are the (dual-safe) callables the reference takes as
    ``linear_advection(..., manufactured=(m.u, m.grad))`` (conslaw.py:174-225); a law built from
    them — here or by the reference's own factory — maps to the device functor ``LinAdvMS``."""

    def __init__(self, a0=1.0, a1=0.5, k1=0.7, k2=-0.4):
        self.params = (float(a0), float(a1), float(k1), float(k2))

    def _e(self, pos):
        a0, a1, k1, k2 = self.params
        return a1 * exp(k1 * pos[..., 0] + k2 * pos[..., 1])

    def u(self, pos):
        return self.params[0] + self._e(pos)

    def grad(self, pos):
        e = self._e(pos)
        return (self.params[2] * e, self.params[3] * e)


def _manufactured_of(obj):
    """The ExpManufactured behind ``obj`` (the object, its (u, grad) pair, or a callable closing
    over its bound methods — the reference's source / bc_value closures), or None."""
    if isinstance(obj, ExpManufactured):
        return obj
    if isinstance(obj, (tuple, list)):
        for o in obj:
            m = _manufactured_of(o)
            if m is not None:
                return m
        return None
    owner = getattr(obj, "__self__", None)
    if isinstance(owner, ExpManufactured):
        return owner
    for cell in getattr(obj, "__closure__", None) or ():
        try:
            m = _manufactured_of(cell.cell_contents)
        except ValueError:  # empty cell
            m = None
        if m is not None:
            return m
    return None


def linear_advection(velocity=(1.0, 1.0), manufactured=None):
    """Constant-velocity advection (conslaw.py:174-253).  ``manufactured``: an ``ExpManufactured``
    (or its ``(u, grad)`` pair): the source becomes c . grad u_exact and the inflow boundaries
    prescribe u_exact at the deformed face points (conslaw.py:214-225)."""
    c = np.asarray(velocity, dtype=float)
    ms = _manufactured_of(manufactured) if manufactured is not None else None
    if manufactured is not None and ms is None:
        raise NotImplementedError("manufactured solutions other than laws.ExpManufactured have no device functor")

    def flux(u, grad_u, mu):
        uc = u[..., 0]
        return _flux_from_rows([(c[0] * uc, c[1] * uc)])

    def source(pos, u, grad_u, mu):
        if ms is None:
            return _comp_last(_zero_like(pos[..., 0]))
        gx = ms.grad(pos)
        return _comp_last(c[0] * gx[0] + c[1] * gx[1])

    def wavespeed(u, nhat, mu):
        ws = absolute(c[0] * nhat[..., 0] + c[1] * nhat[..., 1])
        if is_dual(u) and not is_dual(ws):
            ws = ws + _zero_like(u[..., 0])
        return ws

    def bc_value(pos, mu):
        if ms is None:
            return _const_state(pos, [1.0])
        return np.asarray(ms.u(np.asarray(pos, dtype=float)))[..., None]

    bcs = {}
    for name, normal in (("left", (-1, 0)), ("right", (1, 0)), ("bottom", (0, -1)), ("top", (0, 1))):
        if c @ np.asarray(normal, dtype=float) < 0:
            bcs[name] = BoundaryCondition("prescribed", bc_value, 0)
        else:
            bcs[name] = BoundaryCondition("extrapolate")
    if ms is None:
        return LawSpec("linear-advection", 1, 2, flux, source, None, wavespeed, bcs,
                       np.array([[0.0, 1.0]]), lambda pos, mu: _const_state(pos, [1.0]),
                       law_id=LAW_LINEAR_ADVECTION, params=(float(c[0]), float(c[1])))
    return LawSpec("linear-advection", 1, 2, flux, source, None, wavespeed, bcs,
                   np.array([[0.0, 1.0]]), lambda pos, mu: _const_state(pos, [1.0]),
                   law_id=LAW_LINADV_MS, params=(float(c[0]), float(c[1]), *ms.params))


def burgers_spacetime():
    def flux(u, grad_u, mu):
        uc = u[..., 0]
        return _flux_from_rows([(0.5 * uc * uc, uc)])

    def source(pos, u, grad_u, mu):
        return _comp_last(0.02 * exp(mu[1] * pos[..., 0]))

    def wavespeed(u, nhat, mu):
        v = u[..., 0] * nhat[..., 0] + nhat[..., 1]
        return sqrt(v * v + 1e-6)

    bcs = {
        "left": BoundaryCondition("prescribed", lambda pos, mu: _const_state(pos, [mu[0]]), 0),
        "bottom": BoundaryCondition("prescribed", lambda pos, mu: _const_state(pos, [1.0]), 1),
        "right": BoundaryCondition("extrapolate"),
        "top": BoundaryCondition("extrapolate"),
    }
    def initial_state(pos, mu):
        """Inflow characteristic behind the straight shock line x = (a + 1) t / 2, the slab value 1
        ahead of it (conslaw.py:136-144)."""
        a, b = mu
        x, t = pos[..., 0], pos[..., 1]
        behind = np.sqrt(a * a + (0.04 / b) * (np.exp(b * x) - 1.0))
        return np.where(x <= 0.5 * (a + 1.0) * t, behind, 1.0)[..., None]

    return LawSpec("burgers-spacetime", 1, 2, flux, source, None, wavespeed, bcs,
                   np.array([[3.0, 9.0], [0.02, 0.075]]), initial_state, law_id=LAW_BURGERS_SPACETIME)


def burgers_strip(u_left=1.0, u_right=-0.5):
    """Steady inviscid Burgers (u^2/2)_x = mu*u on a thin strip (config 1).

    Both branches satisfy u_x = mu: left u = u_left + mu x, right
    u = u_right - mu (1 - x).  Rankine-Hugoniot (u_l = -u_r) puts the single
    stationary shock at x_s = (mu - u_left - u_right) / (2 mu), which for the
    defaults moves from 0.25 (mu=1) to 0.42 (mu=3).  Top/bottom faces
    extrapolate (zero y-flux, zero jump).
    """
    def flux(u, grad_u, mu):
        uc = u[..., 0]
        return _flux_from_rows([(0.5 * uc * uc, _zero_like(uc))])

    def source(pos, u, grad_u, mu):
        return mu[0] * u

    def wavespeed(u, nhat, mu):
        v = u[..., 0] * nhat[..., 0]
        return sqrt(v * v + 1e-6)

    def initial_state(pos, mu):
        x = pos[..., 0]
        xs = (mu[0] - u_left - u_right) / (2.0 * mu[0])
        return np.where(x <= xs, u_left + mu[0] * x, u_right - mu[0] * (1.0 - x))[..., None]

    bcs = {
        "left": BoundaryCondition("prescribed", lambda pos, mu: _const_state(pos, [u_left]), 0),
        "right": BoundaryCondition("prescribed", lambda pos, mu: _const_state(pos, [u_right]), 1),
        "bottom": BoundaryCondition("extrapolate"),
        "top": BoundaryCondition("extrapolate"),
    }
    return LawSpec("burgers-strip", 1, 2, flux, source, None, wavespeed, bcs,
                   np.array([[1.0, 3.0]]), initial_state,
                   law_id=LAW_BURGERS_STRIP, params=(float(u_left), float(u_right)))


def euler_freestream(mach, gamma=1.4):
    """(rho, rho u, rho v, E) for rho=1, u=Mach, v=0, p=1/gamma (sound speed 1)."""
    p = 1.0 / gamma
    return np.array([1.0, mach, 0.0, p / (gamma - 1.0) + 0.5 * mach * mach])


ROE_DELTA = 0.1  # entropy correction |lambda| -> sqrt(lambda^2 + (ROE_DELTA c)^2)


def roe_dissipation(gamma=1.4, delta=ROE_DELTA):
    """Roe matrix dissipation D = |A_roe(nhat)| (u_out - u_in) for 2-D Euler, written against the
    pluggable dual namespace (Roe-averaged state, three wave families, smooth entropy correction
    |lambda|_d = sqrt(lambda^2 + (delta c)^2) on every family).  D(u, u) = 0, so the flux is
    consistent and equals LLF at matched states.  Device twin: laws.cuh roe_diss."""
    g = float(gamma)

    def D(uL, uR, nhat, mu):
        rl, rr = uL[..., 0], uR[..., 0]
        sl, sr = sqrt(rl), sqrt(rr)
        vxl, vyl, vxr, vyr = uL[..., 1] / rl, uL[..., 2] / rl, uR[..., 1] / rr, uR[..., 2] / rr
        pl = (g - 1.0) * (uL[..., 3] - 0.5 * (uL[..., 1] * vxl + uL[..., 2] * vyl))
        pr = (g - 1.0) * (uR[..., 3] - 0.5 * (uR[..., 1] * vxr + uR[..., 2] * vyr))
        hl, hr = (uL[..., 3] + pl) / rl, (uR[..., 3] + pr) / rr
        den = sl + sr
        ux, uy, ht = (sl * vxl + sr * vxr) / den, (sl * vyl + sr * vyr) / den, (sl * hl + sr * hr) / den
        q2 = ux * ux + uy * uy
        c2 = (g - 1.0) * (ht - 0.5 * q2)
        c = sqrt(c2)
        rt = sl * sr
        nx, ny = nhat[..., 0], nhat[..., 1]
        un = ux * nx + uy * ny
        dr, dp, dvx, dvy = rr - rl, pr - pl, vxr - vxl, vyr - vyl
        dun = dvx * nx + dvy * ny
        a1 = (dp - rt * c * dun) / (2.0 * c2)
        a3 = (dp + rt * c * dun) / (2.0 * c2)
        a2 = dr - dp / c2
        d2 = (delta * delta) * c2
        l1, l2, l3 = sqrt((un - c) * (un - c) + d2), sqrt(un * un + d2), sqrt((un + c) * (un + c) + d2)
        w1, w3 = l1 * a1, l3 * a3
        return stack([
            w1 + l2 * a2 + w3,
            w1 * (ux - c * nx) + l2 * (a2 * ux + rt * (dvx - dun * nx)) + w3 * (ux + c * nx),
            w1 * (uy - c * ny) + l2 * (a2 * uy + rt * (dvy - dun * ny)) + w3 * (uy + c * ny),
            w1 * (ht - un * c) + l2 * (0.5 * a2 * q2 + rt * (ux * dvx + uy * dvy - un * dun)) + w3 * (ht + un * c),
        ], axis=-1)

    return D


def euler(gamma=1.4, tags=None, flux="llf"):
    """Compressible Euler, conservative variables (rho, rho u, rho v, E).

    ``tags`` maps mesh tag name -> "freestream" | "extrapolate" | "wall"; the
    freestream ghost is ``euler_freestream(mu[0])`` (mu[0] = Mach number), "wall"
    a slip wall (ghost with the momentum mirrored in the face; GPU-only extension,
    its LLF wavespeed is the interior one).  ``flux``: "llf" (local Lax-Friedrichs,
    wavespeed |v.n| + c, the reference's numerical flux) or "roe" (``roe_dissipation``,
    GPU-only extension).
    """
    g = float(gamma)
    if flux not in ("llf", "roe"):
        raise ValueError(f"unknown numerical flux {flux!r}")
    roe = flux == "roe"  # (the name `flux` is the physical flux function below)

    def _primitive(u):
        rho, mx, my, E = u[..., 0], u[..., 1], u[..., 2], u[..., 3]
        vx, vy = mx / rho, my / rho
        p = (g - 1.0) * (E - 0.5 * (mx * vx + my * vy))
        return rho, mx, my, E, vx, vy, p

    def flux(u, grad_u, mu):
        rho, mx, my, E, vx, vy, p = _primitive(u)
        return _flux_from_rows([
            (mx, my),
            (mx * vx + p, mx * vy),
            (my * vx, my * vy + p),
            ((E + p) * vx, (E + p) * vy),
        ])

    def source(pos, u, grad_u, mu):
        return _zero_like(u)

    def wavespeed(u, nhat, mu):
        rho, mx, my, E, vx, vy, p = _primitive(u)
        vn = vx * nhat[..., 0] + vy * nhat[..., 1]
        return absolute(vn) + sqrt(g * p / rho)

    def initial_state(pos, mu):
        return _const_state(pos, euler_freestream(mu[0], g))

    tags = tags or {"left": "freestream", "right": "freestream", "bottom": "freestream", "top": "freestream"}
    bcs = {}
    for name, kind in tags.items():
        if kind == "freestream":
            bcs[name] = BoundaryCondition(
                "prescribed", lambda pos, mu: _const_state(pos, euler_freestream(mu[0], g)), 0)
        elif kind == "extrapolate":
            bcs[name] = BoundaryCondition("extrapolate")
        elif kind == "wall":
            bcs[name] = BoundaryCondition("reflect")
        else:
            raise ValueError(f"unknown Euler boundary kind {kind!r}")
    return LawSpec("euler-roe" if roe else "euler", 4, 2, flux, source, None, wavespeed, bcs,
                   np.array([[2.0, 4.0]]), initial_state, numflux=roe_dissipation(g) if roe else None,
                   law_id=LAW_EULER_ROE if roe else LAW_EULER, params=(g, ROE_DELTA) if roe else (g,))


# -- device descriptor ------------------------------------------------------------
@dataclass
class DeviceLaw:
    law_id: int
    n_comp: int
    params: np.ndarray
    bc_code_by_tag: dict = field(default_factory=dict)


def _reference_law_id(law):
    """Map one of the reference's own law objects (by name) to a device law."""
    name = getattr(law, "name", None)
    if name == "burgers-spacetime":
        ghosts = {"left": 0, "bottom": 1}
        return LAW_BURGERS_SPACETIME, (), ghosts
    if name == "linear-advection":
        if getattr(law, "needs_gradient", False):
            raise NotImplementedError("gradient-dependent laws have no device functor")
        probe = np.asarray(law.flux(np.ones((1, 1)), None, np.zeros(1)), dtype=float).reshape(-1)
        src = np.asarray(law.source(np.full((1, 2), 0.37), np.ones((1, 1)), None, np.zeros(1)), dtype=float)
        ghosts = {t: 0 for t, bc in law.boundary_data.items() if bc.kind == "prescribed"}
        if np.any(src != 0.0):  # manufactured = (u_exact, grad_exact), conslaw.py:214-225
            ms = _manufactured_of(law.source)
            if ms is None:
                raise NotImplementedError("manufactured linear-advection sources other than laws.ExpManufactured "
                                          "have no device functor")
            return LAW_LINADV_MS, (float(probe[0]), float(probe[1]), *ms.params), ghosts
        return LAW_LINEAR_ADVECTION, (float(probe[0]), float(probe[1])), ghosts
    raise NotImplementedError(f"no compiled device law for {name!r}")


def device_law(law, boundary_tags):
    """Descriptor for ``law`` on a mesh with ``boundary_tags`` (name -> id)."""
    if getattr(law, "dissipation", None) is not None or getattr(law, "needs_gradient", False):
        raise NotImplementedError("custom dissipation / gradient laws have no device functor")
    if getattr(law, "numflux", None) is not None and not (isinstance(law, LawSpec) and law.law_id == LAW_EULER_ROE):
        raise NotImplementedError("custom numerical fluxes have no device functor (Euler Roe only)")
    if isinstance(law, LawSpec):
        law_id, params = law.law_id, law.params
        ghosts = {t: bc.ghost_id for t, bc in law.boundary_data.items() if bc.kind == "prescribed"}
    else:
        law_id, params, ghosts = _reference_law_id(law)
    codes = {}
    for tag in boundary_tags:
        bc = law.bc(tag)
        if bc.kind == "extrapolate":
            codes[tag] = BC_EXTRAPOLATE
        elif bc.kind == "reflect":
            if law_id not in (LAW_EULER, LAW_EULER_ROE):
                raise NotImplementedError("slip walls are implemented for Euler only")
            codes[tag] = BC_REFLECT
        elif bc.kind == "prescribed":
            if tag not in ghosts or ghosts[tag] < 0:
                raise NotImplementedError(f"prescribed BC on tag {tag!r} has no device ghost")
            codes[tag] = BC_GHOST0 + int(ghosts[tag])
        else:
            raise NotImplementedError(f"boundary kind {bc.kind!r}")
    if law_id == LAW_EULER and BC_REFLECT in codes.values():
        law_id = LAW_EULER_WALL  # the wall-free Euler kernels carry no wall code
    return DeviceLaw(int(law_id), int(law.n_comp), np.asarray(params, dtype=float), codes)


LAW_FACTORIES = {
    "linear-advection": linear_advection,
    "burgers-spacetime": burgers_spacetime,
    "burgers-strip": burgers_strip,
    "euler": euler,
}


def make_law(name, **kwargs):
    try:
        return LAW_FACTORIES[name](**kwargs)
    except KeyError:
        raise ValueError(f"unknown conservation law {name!r}") from None
