"""Forward-mode dual numbers with a trailing tangent axis (oracle only).

Restates the semantics of ``strom/dual.py:31-242``: Leibniz products,
``maximum`` ties go to the first argument (:167-176), ``absolute`` uses
sign(0)=0 (:161-163), ``einsum`` contracts the value once and the tangent
once per dual operand (:190-207).
"""

import numpy as np

from paper_2305_15661_b200 import laws as _laws


def _bt(t, shape):
    want = tuple(shape) + (t.shape[-1],)
    return t if t.shape == want else np.broadcast_to(t, want)


class Dual:
    __slots__ = ("val", "tan")

    def __init__(self, val, tan):
        self.val = np.asarray(val, dtype=float)
        self.tan = np.asarray(tan, dtype=float)

    @property
    def ntan(self):
        return self.tan.shape[-1]

    @property
    def shape(self):
        return self.val.shape

    def __getitem__(self, idx):
        t = idx if isinstance(idx, tuple) else (idx,)
        return Dual(self.val[idx], self.tan[t + (slice(None),)])

    def __neg__(self):
        return Dual(-self.val, -self.tan)

    def _lift(self, o):
        return o if isinstance(o, Dual) else None

    def __add__(self, o):
        d = self._lift(o)
        if d is None:
            v = self.val + np.asarray(o)
            return Dual(v, _bt(self.tan, v.shape))
        v = self.val + d.val
        return Dual(v, _bt(self.tan, v.shape) + _bt(d.tan, v.shape))

    __radd__ = __add__

    def __sub__(self, o):
        return self + (-o if isinstance(o, Dual) else -np.asarray(o))

    def __rsub__(self, o):
        return (-self) + o

    def __mul__(self, o):
        d = self._lift(o)
        if d is None:
            o = np.asarray(o)
            v = self.val * o
            return Dual(v, _bt(self.tan, v.shape) * o[..., None])
        v = self.val * d.val
        return Dual(v, _bt(self.tan, v.shape) * d.val[..., None] + self.val[..., None] * _bt(d.tan, v.shape))

    __rmul__ = __mul__

    def __truediv__(self, o):
        d = self._lift(o)
        if d is None:
            o = np.asarray(o)
            v = self.val / o
            return Dual(v, _bt(self.tan, v.shape) / o[..., None])
        r = 1.0 / d.val
        v = self.val * r
        return Dual(v, (_bt(self.tan, v.shape) - v[..., None] * _bt(d.tan, v.shape)) * r[..., None])

    def __rtruediv__(self, o):
        r = 1.0 / self.val
        v = np.asarray(o) * r
        return Dual(v, -(v * r)[..., None] * _bt(self.tan, v.shape))

    def __pow__(self, k):
        return Dual(self.val ** k, (k * self.val ** (k - 1))[..., None] * self.tan)


def val(x):
    return x.val if isinstance(x, Dual) else np.asarray(x)


def _tan_or_zero(x, shape, n):
    if isinstance(x, Dual):
        return _bt(x.tan, shape)
    return np.zeros(tuple(shape) + (n,))


def sqrt(x):
    if isinstance(x, Dual):
        r = np.sqrt(x.val)
        return Dual(r, (0.5 / r)[..., None] * x.tan)
    return np.sqrt(x)


def exp(x):
    if isinstance(x, Dual):
        r = np.exp(x.val)
        return Dual(r, r[..., None] * x.tan)
    return np.exp(x)


def absolute(x):
    if isinstance(x, Dual):
        return Dual(np.abs(x.val), np.sign(x.val)[..., None] * x.tan)
    return np.abs(x)


def maximum(a, b):
    """Ties pick ``a`` (strom/dual.py:171)."""
    av, bv = val(a), val(b)
    if not (isinstance(a, Dual) or isinstance(b, Dual)):
        return np.maximum(av, bv)
    first = av >= bv
    v = np.where(first, av, bv)
    n = a.ntan if isinstance(a, Dual) else b.ntan
    return Dual(v, np.where(first[..., None], _tan_or_zero(a, v.shape, n), _tan_or_zero(b, v.shape, n)))


def stack(parts, axis):
    if not any(isinstance(p, Dual) for p in parts):
        return np.stack(parts, axis=axis)
    n = next(p.ntan for p in parts if isinstance(p, Dual))
    vs = [val(p) for p in parts]
    ax = axis if axis >= 0 else vs[0].ndim + 1 + axis
    return Dual(np.stack(vs, axis=ax), np.stack([_tan_or_zero(p, v.shape, n) for p, v in zip(parts, vs)], axis=ax))


def einsum(spec, a, b):
    lhs, out = spec.split("->")
    sa, sb = lhs.split(",")
    v = np.einsum(spec, val(a), val(b), optimize=True)
    if not (isinstance(a, Dual) or isinstance(b, Dual)):
        return v
    t = None
    if isinstance(a, Dual):
        t = np.einsum(f"{sa}z,{sb}->{out}z", a.tan, val(b), optimize=True)
    if isinstance(b, Dual):
        tb = np.einsum(f"{sa},{sb}z->{out}z", val(a), b.tan, optimize=True)
        t = tb if t is None else t + tb
    return Dual(v, t)


def expand(x, k=1):
    if isinstance(x, Dual):
        v, t = x.val, x.tan
        for _ in range(k):
            v, t = v[..., None], t[..., None, :]
        return Dual(v, t)
    x = np.asarray(x)
    for _ in range(k):
        x = x[..., None]
    return x


def reshape(x, shape):
    if isinstance(x, Dual):
        return Dual(x.val.reshape(shape), x.tan.reshape(tuple(shape) + (x.ntan,)))
    return np.asarray(x).reshape(shape)


def seed_identity(v, offset, n):
    """Per-row identity tangents in slots offset.. (strom/dual.py:231-242)."""
    v = np.asarray(v, dtype=float)
    k = int(np.prod(v.shape[1:], dtype=int))
    t = np.zeros((k, n))
    t[np.arange(k), offset + np.arange(k)] = 1.0
    return Dual(v, np.broadcast_to(t.reshape(v.shape[1:] + (n,)), v.shape + (n,)).copy())


import sys as _sys

_laws.register_dual_backend(Dual, _sys.modules[__name__])
