"""Kernel expression trees with the reference's public surface (minigp/kernels.py).

Same classes, fields, validation, operator sugar (``k1 + k2``, ``k1 * k2``),
hyper-parameter coordinates (positive values, natural-log flattening in
pre-order, kernels.py:403-424), s-expression grammar (kernels.py:445-519) and
node protocol (``_params / _rebuild / _slab_buffers / _sexpr / _gram /
_diag``). What changes is evaluation: a tree is *lowered* (``lower``) to the
pre-order node program of the C ABI and evaluated by CUDA kernels that the
library generates for that tree; ``_gram`` / ``_diag`` / ``kernel_eval`` /
``kernel_diag`` run on the GPU in FP64.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatchError, KernelParseError, NonFiniteError
from .linalg import as_matrix, tracked


def _check_positive(name, value):
    v = float(value)
    if not (math.isfinite(v) and v > 0.0):
        raise ValueError(f"{name} must be positive and finite, got {value!r}")
    return v


@dataclass(frozen=True)
class Kernel:
    """Base of all kernel nodes (instantiate the subclasses)."""

    def __add__(self, other):
        return Sum(self, other) if isinstance(other, Kernel) else NotImplemented

    def __mul__(self, other):
        return Product(self, other) if isinstance(other, Kernel) else NotImplemented

    # ---- device evaluation (kernel_eval / kernel_diag semantics)
    def _gram(self, x, y):
        return _device_gram(self, x, y)

    def _diag(self, x):
        return _device_diag(self, x)


class _Leaf(Kernel):
    _FORM = ""
    _FIELDS = ()

    def _params(self):
        return tuple(getattr(self, f) for f in self._FIELDS)

    def _rebuild(self, it):
        return type(self)(*[next(it) for _ in self._FIELDS])

    def _sexpr(self):
        return "(" + " ".join([self._FORM] + [repr(getattr(self, f)) for f in self._FIELDS]) + ")"

    def __post_init__(self):
        for f in self._FIELDS:
            object.__setattr__(self, f, _check_positive(f, getattr(self, f)))


@dataclass(frozen=True)
class RBF(_Leaf):
    """exp(-r^2 / (2 l^2))  (kernels.py:56-83)."""

    lengthscale: float = 1.0
    _FORM = "rbf"
    _FIELDS = ("lengthscale",)

    def _slab_buffers(self):
        return 1


@dataclass(frozen=True)
class Matern12(_Leaf):
    """exp(-r / l)  (kernels.py:86-114)."""

    lengthscale: float = 1.0
    _FORM = "matern12"
    _FIELDS = ("lengthscale",)

    def _slab_buffers(self):
        return 1


@dataclass(frozen=True)
class Matern32(_Leaf):
    """(1 + t) exp(-t), t = sqrt(3) r / l  (kernels.py:117-151)."""

    lengthscale: float = 1.0
    _FORM = "matern32"
    _FIELDS = ("lengthscale",)

    def _slab_buffers(self):
        return 2


@dataclass(frozen=True)
class Matern52(_Leaf):
    """(1 + t + t^2/3) exp(-t), t = sqrt(5) r / l  (kernels.py:154-189)."""

    lengthscale: float = 1.0
    _FORM = "matern52"
    _FIELDS = ("lengthscale",)

    def _slab_buffers(self):
        return 2


@dataclass(frozen=True)
class Periodic(_Leaf):
    """exp(-2 sum_d sin^2(pi (x_d - y_d) / p) / l^2)  (kernels.py:192-235)."""

    lengthscale: float = 1.0
    period: float = 1.0
    _FORM = "periodic"
    _FIELDS = ("lengthscale", "period")

    def _slab_buffers(self):
        return 2


@dataclass(frozen=True)
class Linear(_Leaf):
    """v * (x . y), no offset  (kernels.py:238-273)."""

    variance: float = 1.0
    _FORM = "linear"
    _FIELDS = ("variance",)

    def _slab_buffers(self):
        return 1


@dataclass(frozen=True)
class Scale(Kernel):
    """s * child(x, y), s a variance  (kernels.py:276-308)."""

    outputscale: float
    child: Kernel

    def __post_init__(self):
        object.__setattr__(self, "outputscale", _check_positive("outputscale", self.outputscale))
        if not isinstance(self.child, Kernel):
            raise TypeError("Scale child must be a kernel")

    def _params(self):
        return (self.outputscale,) + self.child._params()

    def _rebuild(self, it):
        s = next(it)
        return Scale(s, self.child._rebuild(it))

    def _slab_buffers(self):
        return self.child._slab_buffers()

    def _sexpr(self):
        return f"(scale {self.outputscale!r} {self.child._sexpr()})"


@dataclass(frozen=True)
class _Binary(Kernel):
    left: Kernel
    right: Kernel
    _OP = ""

    def __post_init__(self):
        if not (isinstance(self.left, Kernel) and isinstance(self.right, Kernel)):
            raise TypeError(f"{type(self).__name__} children must be kernels")

    def _params(self):
        return self.left._params() + self.right._params()

    def _rebuild(self, it):
        a = self.left._rebuild(it)
        return type(self)(a, self.right._rebuild(it))

    def _slab_buffers(self):
        # kernels.py:339-340 / 374-375: the right child runs while the left's
        # slab is alive
        return max(self.left._slab_buffers(), 1 + self.right._slab_buffers())

    def _sexpr(self):
        return f"({self._OP} {self.left._sexpr()} {self.right._sexpr()})"


@dataclass(frozen=True)
class Sum(_Binary):
    """left + right  (kernels.py:311-343)."""

    _OP = "+"


@dataclass(frozen=True)
class Product(_Binary):
    """left * right, pointwise  (kernels.py:346-378)."""

    _OP = "*"


_LEAVES = {"rbf": RBF, "matern12": Matern12, "matern32": Matern32, "matern52": Matern52,
           "periodic": Periodic, "linear": Linear}
_CLASS_FORM = {"RBF": "rbf", "Matern12": "matern12", "Matern32": "matern32",
               "Matern52": "matern52", "Periodic": "periodic", "Linear": "linear",
               "Scale": "scale", "Sum": "+", "Product": "*"}
_OWN_CLASSES = {RBF, Matern12, Matern32, Matern52, Periodic, Linear, Scale, Sum, Product}


# ---------------------------------------------------------------- lowering

def lower(kernel):
    """Pre-order node program ``[(form, params), ...]`` of a kernel tree.

    Accepts this package's classes and, for drop-in use, the reference's own
    ``minigp`` kernel objects (matched by class and field names). Subclasses
    that override the evaluation (``_gram``) cannot be compiled for the GPU
    and raise ``TypeError`` — there is no CPU path to run them on.
    """
    out = []

    def walk(k):
        cls = type(k)
        form = None
        if cls in _OWN_CLASSES:
            form = _CLASS_FORM[cls.__name__]
        elif cls.__module__.split(".")[0] == "minigp" and cls.__name__ in _CLASS_FORM:
            form = _CLASS_FORM[cls.__name__]
        else:
            for base in cls.__mro__[1:]:
                if base in _OWN_CLASSES and base.__name__ in _CLASS_FORM:
                    if cls._gram is base._gram and cls._diag is base._diag:
                        form = _CLASS_FORM[base.__name__]
                    break
        if form is None:
            raise TypeError(
                f"kernel class {cls.__module__}.{cls.__name__} cannot be lowered to the "
                "device kernel-tree program (custom evaluation is not supported)")
        if form in _LEAVES:
            out.append((form, tuple(float(getattr(k, f)) for f in _LEAVES[form]._FIELDS)))
        elif form == "scale":
            out.append((form, (float(k.outputscale),)))
            walk(k.child)
        else:
            out.append((form, ()))
            walk(k.left)
            walk(k.right)

    walk(kernel)
    return out


_PROGRAMS = {}


def program(kernel):
    """The library handle of a kernel tree (cached by structure + values)."""
    nodes = lower(kernel)
    key = tuple(nodes)
    prog = _PROGRAMS.get(key)
    if prog is None:
        kinds = [_lib.NODE_KINDS[f] for f, _ in nodes]
        params = [v for _, p in nodes for v in p]
        prog = _lib.KernelProgram(kinds, params)
        if len(_PROGRAMS) > 256:
            _PROGRAMS.clear()
        _PROGRAMS[key] = prog
    return prog


def _device_gram(kernel, x, y):
    ctx = _lib.default_context()
    px = _lib.DevicePoints(ctx, x)
    py = px if y is x else _lib.DevicePoints(ctx, y)
    out = np.empty((px.n, py.n))
    _lib.check(_lib.lib().lgp_gram(ctx.handle, program(kernel).handle, px.handle, py.handle,
                                   _lib.vptr(out), 0))
    return tracked(out)


def _device_diag(kernel, x):
    ctx = _lib.default_context()
    px = _lib.DevicePoints(ctx, x)
    out = np.empty(px.n)
    _lib.check(_lib.lib().lgp_diag(ctx.handle, program(kernel).handle, px.handle,
                                   _lib.vptr(out), 0))
    return tracked(out)


# --------------------------------------------------------------- functions

def kernel_eval(kernel, x, y=None):
    """k(x_i, y_j); y=None (or y is x) gives the exactly symmetric square Gram."""
    same = y is None or y is x
    xv = as_matrix(x, "X")
    yv = xv if same else as_matrix(y, "Y")
    if yv.shape[1] != xv.shape[1]:
        raise DimensionMismatchError(f"X has {xv.shape[1]} columns, Y has {yv.shape[1]}")
    return kernel._gram(xv, yv)


def kernel_diag(kernel, x):
    """diag k(x_i, x_i) in O(N D)."""
    return kernel._diag(as_matrix(x, "X"))


def n_params(kernel):
    return len(kernel._params())


def flatten_params(kernel):
    """log(hyper-parameters), pre-order."""
    return tracked(np.log(np.asarray(kernel._params(), dtype=np.float64)))


def unflatten_params(kernel, values):
    """Tree of the same shape with hyper-parameters exp(values)."""
    v = np.asarray(values, dtype=np.float64)
    if v.ndim != 1:
        raise DimensionMismatchError("parameter vector must be 1-d")
    want = n_params(kernel)
    if v.shape[0] != want:
        raise DimensionMismatchError(f"expected {want} parameters, got {v.shape[0]}")
    if not np.isfinite(v).all():
        raise NonFiniteError("parameter vector contains non-finite values")
    return kernel._rebuild(iter(np.exp(v).tolist()))


def is_stationary(kernel):
    """Every leaf depends only on x - y (Linear does not)."""
    return all(form != "linear" for form, _ in lower(kernel))


def slab_buffer_count(kernel):
    return kernel._slab_buffers()


# ------------------------------------------------------------------ grammar

def parse_kernel(text):
    """s-expression -> kernel tree; forms as in kernels.py:14-17."""
    if not isinstance(text, str):
        raise KernelParseError("kernel expression must be a string")
    toks = text.replace("(", " ( ").replace(")", " ) ").split()
    if not toks:
        raise KernelParseError("empty kernel expression")
    state = {"i": 0}

    def nxt():
        if state["i"] >= len(toks):
            raise KernelParseError("unexpected end of kernel expression")
        t = toks[state["i"]]
        state["i"] += 1
        return t

    def num(head):
        t = nxt()
        try:
            return float(t)
        except ValueError:
            raise KernelParseError(f"expected a number in {head!r} form", token=t) from None

    def build(head, fn):
        try:
            return fn()
        except ValueError as exc:
            raise KernelParseError(str(exc), token=head) from None

    def node():
        t = nxt()
        if t != "(":
            raise KernelParseError("expected '('", token=t)
        head = nxt()
        if head in _LEAVES:
            cls = _LEAVES[head]
            vals = [num(head) for _ in cls._FIELDS]
            k = build(head, lambda: cls(*vals))
        elif head == "scale":
            s = num(head)
            child = node()
            k = build(head, lambda: Scale(s, child))
        elif head in ("+", "*"):
            a = node()
            b = node()
            k = Sum(a, b) if head == "+" else Product(a, b)
        else:
            raise KernelParseError(f"unknown kernel form {head!r}", token=head)
        t = nxt()
        if t != ")":
            raise KernelParseError("expected ')'", token=t)
        return k

    k = node()
    if state["i"] != len(toks):
        raise KernelParseError("trailing tokens after kernel expression", token=toks[state["i"]])
    return k


def format_kernel(kernel):
    """Canonical text; parse_kernel(format_kernel(k)) == k."""
    return kernel._sexpr()
