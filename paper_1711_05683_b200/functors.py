"""Parametric function expressions and their lowering to device programs.

Public surface mirrors the reference (functors.py:33-318): ParamSet,
FunctorExpr with + - * / algebra, GaussianShape, ExponentialShape, Closure,
Composition, Coordinate and the factory functions.  ``eval`` on host arrays
keeps the reference semantics for scalar/API use (``expr(x)``,
``Pdf.value``).

The hot path never calls ``eval``.  Instead an expression -- composed with
the user's ``arg_builder`` -- is *lowered* to an ``hk_program_t``: an SSA
register program the sm_100a kernels interpret per event (warp-uniform op
stream).  ``arg_builder`` callables and ``wrap_closure`` bodies are traced
symbolically: they run once on :class:`Sym` placeholders that record the
numpy operations applied to them (+ - * / **2, sqrt/exp/log/square,
ones_like...).  Anything that cannot be traced raises ``NotImplementedError``
-- there is no CPU fallback (hard part 4).
"""

from __future__ import annotations

import math
from typing import Callable, Iterable, Sequence

import numpy as np

from . import _lib
from .kinematics import Parameter

_SQRT_2PI = math.sqrt(2.0 * math.pi)   # functors.py:26


class EvaluationError(ValueError):
    """An expression could not be evaluated at a concrete point."""


class ParamSet:
    """Ordered, name-addressable parameter collection (functors.py:33-76)."""

    def __init__(self, params: Iterable[Parameter] = ()):
        self._params: list[Parameter] = []
        self._index: dict[str, int] = {}
        for p in params:
            self.add(p)

    def add(self, param: Parameter) -> None:
        if param.name in self._index:
            raise ValueError(f"duplicate parameter name {param.name!r}")
        self._index[param.name] = len(self._params)
        self._params.append(param)

    def __len__(self) -> int:
        return len(self._params)

    def __iter__(self):
        return iter(self._params)

    def __contains__(self, name: str) -> bool:
        return name in self._index

    def __getitem__(self, key: str | int) -> Parameter:
        return self._params[self._index[key]] if isinstance(key, str) else self._params[key]

    @property
    def names(self) -> tuple[str, ...]:
        return tuple(p.name for p in self._params)

    def values(self) -> tuple[float, ...]:
        return tuple(p.value for p in self._params)

    def set_values(self, values: Sequence[float]) -> None:
        if len(values) != len(self._params):
            raise ValueError("value count does not match parameter count")
        for p, v in zip(self._params, values):
            p.set(v)

    def free(self) -> list[Parameter]:
        return [p for p in self._params if not p.fixed]


# ---------------------------------------------------------------------------
# symbolic tracing: a DAG of hash-consed tuples
#   ("col", c) ("const", v) (op, a, b) (unary, a) ("gauss", a, mu, s) ...

_BINARY = {"add", "sub", "mul", "div", "udiv"}
_UNARY = {"neg", "sqrt", "exp", "log", "square", "add0"}


class Sym:
    """Placeholder for a per-event value inside traced numpy code."""

    __array_priority__ = 1000

    def __init__(self, node):
        self.node = node

    @staticmethod
    def wrap(v) -> "Sym":
        if isinstance(v, Sym):
            return v
        if isinstance(v, (bool, np.bool_)):
            raise NotImplementedError("boolean values cannot be lowered to the device")
        if np.ndim(v) == 0 and isinstance(v, (int, float, np.integer, np.floating)):
            return Sym(("const", float(v)))
        raise NotImplementedError(f"cannot lower value of type {type(v).__name__} to the device")

    def _bin(self, op, other, swap=False):
        o = Sym.wrap(other)
        a, b = (o, self) if swap else (self, o)
        return Sym((op, a.node, b.node))

    def __add__(self, o): return self._bin("add", o)
    def __radd__(self, o): return self._bin("add", o, True)
    def __sub__(self, o): return self._bin("sub", o)
    def __rsub__(self, o): return self._bin("sub", o, True)
    def __mul__(self, o): return self._bin("mul", o)
    def __rmul__(self, o): return self._bin("mul", o, True)
    # numpy division in traced code never raises (inf / nan, as in the
    # reference's closures and arg_builders): unchecked "udiv"
    def __truediv__(self, o): return self._bin("udiv", o)
    def __rtruediv__(self, o): return self._bin("udiv", o, True)
    def __neg__(self): return Sym(("neg", self.node))
    def __pos__(self): return self

    def __pow__(self, k):
        if isinstance(k, (int, float, np.integer, np.floating)):
            if float(k) == 2.0:
                return Sym(("square", self.node))
            if float(k) == 0.5:
                return Sym(("sqrt", self.node))
            if float(k) == 1.0:
                return self
        raise NotImplementedError(f"x ** {k!r} is not supported on the device")

    def __bool__(self):
        raise NotImplementedError("data-dependent control flow cannot be lowered to the device")

    _UFUNCS = {"add": "add", "subtract": "sub", "multiply": "mul", "divide": "udiv",
               "true_divide": "udiv", "negative": "neg", "sqrt": "sqrt", "exp": "exp",
               "log": "log", "square": "square", "power": "power", "positive": None}

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        if method != "__call__" or kwargs.get("out") is not None:
            return NotImplemented
        name = ufunc.__name__
        if name not in self._UFUNCS:
            raise NotImplementedError(f"numpy.{name} is not supported on the device")
        op = self._UFUNCS[name]
        args = [Sym.wrap(x) for x in inputs]
        if op is None:
            return args[0]
        if op == "power":
            return args[0] ** inputs[1]
        if len(args) == 1:
            return Sym((op, args[0].node))
        return Sym((op, args[0].node, args[1].node))

    def __array_function__(self, func, types, args, kwargs):
        name = func.__name__
        if name in ("ones_like", "zeros_like", "full_like"):
            fill = {"ones_like": 1.0, "zeros_like": 0.0}.get(name)
            if fill is None:
                fill = float(args[1] if len(args) > 1 else kwargs["fill_value"])
            return Sym(("const", fill))
        if name in ("square", "sqrt", "exp", "log"):
            return getattr(np, name)(*args)
        raise NotImplementedError(f"numpy.{name} is not supported on the device")


def _sym_columns(names: Sequence[str]) -> dict[str, Sym]:
    return {name: Sym(("col", i)) for i, name in enumerate(names)}


def trace_arg_builder(arg_builder, names: Sequence[str]) -> list:
    """Run arg_builder once on symbolic columns; returns the argument nodes."""
    try:
        out = arg_builder(_sym_columns(names))
    except NotImplementedError:
        raise
    except Exception as exc:  # noqa: BLE001 -- any failure means "not traceable"
        raise NotImplementedError(
            f"arg_builder could not be traced for the device ({type(exc).__name__}: {exc}); "
            "use + - * / ** 2 and numpy sqrt/exp/log/square on the column arrays") from exc
    if isinstance(out, Sym) or np.ndim(out) == 0:
        out = (out,)
    return [Sym.wrap(a).node for a in out]


# ---------------------------------------------------------------------------
# symbolic-parameter tracing (the FCN's per-call fast path, fitting.lower_density)
#
# A model is lowered once with every Parameter as an IR leaf ("pv", k) instead
# of its current value; each later call only reads the parameters' values
# into the program's constant slots.  Anything that needs a concrete
# parameter value while tracing (math.* on it, float(), Python control flow)
# raises NotImplementedError, and the caller falls back to tracing with the
# current values on every call.

class ParamTrace:
    """Collects the parameters met while lowering with symbolic parameters,
    and the value checks the builtin shapes would run (sigma > 0, tau != 0)."""

    def __init__(self):
        self.params: list[Parameter] = []
        self.leaves: dict[int, tuple] = {}
        self.checks: list[Callable[[], float]] = []

    def leaf(self, p: Parameter) -> tuple:
        node = self.leaves.get(id(p))
        if node is None:
            node = self.leaves[id(p)] = ("pv", len(self.params))
            self.params.append(p)
        return node


_PTRACE: ParamTrace | None = None


def _reads_only_args(fn) -> bool:
    """True when a closure's code reads nothing but its arguments and global
    modules (numpy): no captured cells, no other globals, no nested code.
    Only such a closure is a pure function of (x, p), so it can be traced
    once with symbolic parameters; anything else (a captured Parameter read
    directly, a module-level constant the user may rebind) is re-traced at
    the current values on every call."""
    import dis
    import types

    code = getattr(fn, "__code__", None)
    if code is None or code.co_freevars or code.co_cellvars:
        return False
    if any(isinstance(c, types.CodeType) for c in code.co_consts):
        return False
    glb = getattr(fn, "__globals__", {})
    for ins in dis.get_instructions(code):
        if ins.opname in ("LOAD_DEREF", "LOAD_CLASSDEREF", "LOAD_NAME", "STORE_GLOBAL", "LOAD_FROM_DICT_OR_DEREF"):
            return False
        if ins.opname == "LOAD_GLOBAL" and not isinstance(glb.get(ins.argval), types.ModuleType):
            return False
    return True


class _SymParam:
    """What a closure sees as p[name] while tracing with symbolic parameters."""

    def __init__(self, param: Parameter, trace: ParamTrace):
        self._param, self._trace = param, trace
        self.name = param.name

    @property
    def value(self) -> "Sym":
        return Sym(self._trace.leaf(self._param))


class _SymParamSet:
    def __init__(self, params: ParamSet, trace: ParamTrace):
        self._params, self._trace = params, trace

    def __getitem__(self, key):
        return _SymParam(self._params[key], self._trace)

    def __getattr__(self, name):
        raise NotImplementedError(f"ParamSet.{name} while tracing with symbolic parameters")


def lower_symbolic(fn: Callable[[], object]) -> tuple[object, ParamTrace]:
    """Run fn() (which lowers expressions) with symbolic parameters."""
    global _PTRACE
    trace, prev = ParamTrace(), _PTRACE
    _PTRACE = trace
    try:
        return fn(), trace
    finally:
        _PTRACE = prev


# ---------------------------------------------------------------------------
# expression classes

class FunctorExpr:
    """Base expression node (functors.py:79-125)."""

    arity: int = 1

    def eval(self, args: tuple):
        raise NotImplementedError

    def lower(self, args: list):
        """Device IR node of this expression applied to argument nodes."""
        raise NotImplementedError(f"{type(self).__name__} cannot be lowered to the device")

    def __call__(self, *point):
        if len(point) != self.arity:
            raise EvaluationError(f"expression consumes {self.arity} arguments, got {len(point)}")
        out = self.eval(tuple(point))
        if np.isscalar(point[0]) and not np.isscalar(out):
            return float(np.asarray(out).reshape(()))
        return out

    def leaf_params(self) -> list[Parameter]:
        seen: set[int] = set()
        out: list[Parameter] = []
        for p in self._collect_params():
            if id(p) not in seen:
                seen.add(id(p))
                out.append(p)
        return out

    def param_set(self) -> ParamSet:
        return ParamSet(self.leaf_params())

    def _collect_params(self) -> Iterable[Parameter]:
        return ()

    def __add__(self, other): return combine("+", self, other)
    def __sub__(self, other): return combine("-", self, other)
    def __mul__(self, other): return combine("*", self, other)
    def __truediv__(self, other): return combine("/", self, other)


class GaussianShape(FunctorExpr):
    """exp(-(x-mu)^2/(2 sigma^2)) / (sigma sqrt(2 pi)) (functors.py:128-146)."""

    arity = 1

    def __init__(self, mean: Parameter, sigma: Parameter):
        self.mean = mean
        self.sigma = sigma

    def _sigma(self) -> float:
        s = self.sigma.value
        if not s > 0:
            raise EvaluationError(f"sigma must be positive, got {s}")
        return s

    def eval(self, args):
        s = self._sigma()
        z = (args[0] - self.mean.value) / s
        return np.exp(-0.5 * z * z) / (s * _SQRT_2PI)

    def lower(self, args):
        if _PTRACE is not None:
            _PTRACE.checks.append(self._sigma)
            return ("gauss", args[0], _PTRACE.leaf(self.mean), _PTRACE.leaf(self.sigma))
        return ("gauss", args[0], float(self.mean.value), float(self._sigma()))

    def _collect_params(self):
        return (self.mean, self.sigma)


class ExponentialShape(FunctorExpr):
    """exp(-x/tau), unnormalised (functors.py:149-164)."""

    arity = 1

    def __init__(self, tau: Parameter):
        self.tau = tau

    def _tau(self) -> float:
        t = self.tau.value
        if t == 0:
            raise EvaluationError("tau must be non-zero")
        return t

    def eval(self, args):
        t = self._tau()
        return np.exp(-np.asarray(args[0], dtype=float) / t)

    def lower(self, args):
        if _PTRACE is not None:
            _PTRACE.checks.append(self._tau)
            return ("expo", args[0], _PTRACE.leaf(self.tau))
        return ("expo", args[0], float(self._tau()))

    def _collect_params(self):
        return (self.tau,)


class BreitWigner(FunctorExpr):
    """Non-relativistic-in-s Breit-Wigner 1/((s - m0^2)^2 + m0^2 g0^2) of s = x.

    Device builtin for Dalitz-plane integrands (SURVEY.md 8(d) C5, K*(892)).
    """

    arity = 1

    def __init__(self, m0: Parameter, g0: Parameter):
        self.m0 = m0
        self.g0 = g0

    def eval(self, args):
        m0, g0 = self.m0.value, self.g0.value
        return 1.0 / ((np.asarray(args[0], dtype=float) - m0 * m0) ** 2 + (m0 * m0) * (g0 * g0))

    def lower(self, args):
        if _PTRACE is not None:
            return ("bw", args[0], _PTRACE.leaf(self.m0), _PTRACE.leaf(self.g0))
        return ("bw", args[0], float(self.m0.value), float(self.g0.value))

    def _collect_params(self):
        return (self.m0, self.g0)


class Constant(FunctorExpr):
    """The constant c for any point of the given arity."""

    def __init__(self, value: float, arity: int = 1):
        self.value = float(value)
        self.arity = arity

    def eval(self, args):
        return np.full(np.shape(args[0]), self.value) if np.ndim(args[0]) else self.value

    def lower(self, args):
        return ("const", self.value)


class Closure(FunctorExpr):
    """User function fn(point, params) (functors.py:167-179); traced to lower."""

    def __init__(self, fn: Callable, params: ParamSet, arity: int = 1):
        self.fn = fn
        self.params = params
        self.arity = arity

    def eval(self, args):
        return self.fn(args, self.params)

    def lower(self, args):
        if _PTRACE is not None and not _reads_only_args(self.fn):
            raise NotImplementedError("closure reads state outside its arguments")
        params = self.params if _PTRACE is None else _SymParamSet(self.params, _PTRACE)
        try:
            out = self.fn(tuple(Sym(a) for a in args), params)
        except NotImplementedError:
            raise
        except Exception as exc:  # noqa: BLE001
            raise NotImplementedError(
                f"closure could not be traced for the device ({type(exc).__name__}: {exc}); "
                "write it with + - * / ** 2 and numpy sqrt/exp/log/square/ones_like") from exc
        return Sym.wrap(out).node

    def _collect_params(self):
        return tuple(self.params)


class _BinaryOp(FunctorExpr):
    _ops = {"+": np.add, "-": np.subtract, "*": np.multiply, "/": np.divide}
    _ir = {"+": "add", "-": "sub", "*": "mul", "/": "div"}

    def __init__(self, op: str, left: FunctorExpr, right: FunctorExpr):
        if op not in self._ops:
            raise ValueError(f"unknown operator {op!r}")
        if left.arity != right.arity:
            raise ValueError(f"operand arities differ: {left.arity} vs {right.arity}")
        self.op, self.left, self.right = op, left, right
        self.arity = left.arity

    def eval(self, args):
        a = self.left.eval(args)
        b = self.right.eval(args)
        if self.op == "/":
            zero = np.asarray(b) == 0
            if np.any(zero):
                j = int(np.argmax(np.asarray(zero).ravel()))
                point = tuple(np.asarray(c).ravel()[j] if not np.isscalar(c) else c for c in args)
                raise EvaluationError(f"division by zero at point {point}")
        return self._ops[self.op](a, b)

    def lower(self, args):
        return (self._ir[self.op], self.left.lower(args), self.right.lower(args))

    def _collect_params(self):
        yield from self.left._collect_params()
        yield from self.right._collect_params()


class Composition(FunctorExpr):
    """outer(inner_1(x), ..., inner_k(x)) (functors.py:215-236)."""

    def __init__(self, outer: FunctorExpr, inners: Sequence[FunctorExpr]):
        if outer.arity != len(inners):
            raise ValueError(f"outer consumes {outer.arity} arguments, got {len(inners)} inners")
        arities = {f.arity for f in inners}
        if len(arities) != 1:
            raise ValueError(f"inner arities differ: {sorted(arities)}")
        self.outer = outer
        self.inners = tuple(inners)
        self.arity = arities.pop()

    def eval(self, args):
        return self.outer.eval(tuple(f.eval(args) for f in self.inners))

    def lower(self, args):
        return self.outer.lower([f.lower(args) for f in self.inners])

    def _collect_params(self):
        yield from self.outer._collect_params()
        for f in self.inners:
            yield from f._collect_params()


class Coordinate(FunctorExpr):
    """Projection onto component `index` (functors.py:239-249)."""

    def __init__(self, index: int, arity: int = 1):
        if not 0 <= index < arity:
            raise ValueError(f"index {index} out of range for arity {arity}")
        self.index = index
        self.arity = arity

    def eval(self, args):
        return np.asarray(args[self.index], dtype=float) + 0.0

    def lower(self, args):
        return ("add0", args[self.index])


def shape_gaussian(mean: Parameter, sigma: Parameter) -> FunctorExpr:
    if not sigma.value > 0:
        raise ValueError(f"sigma must be positive, got {sigma.value}")
    return GaussianShape(mean, sigma)


def shape_exponential(tau: Parameter) -> FunctorExpr:
    if tau.value == 0:
        raise ValueError("tau must be non-zero")
    return ExponentialShape(tau)


def breit_wigner(m0: float | Parameter, g0: float | Parameter) -> FunctorExpr:
    m = m0 if isinstance(m0, Parameter) else Parameter("bw_m0", float(m0))
    g = g0 if isinstance(g0, Parameter) else Parameter("bw_g0", float(g0))
    return BreitWigner(m, g)


def constant(value: float, arity: int = 1) -> FunctorExpr:
    return Constant(value, arity)


def wrap_closure(fn: Callable, params: ParamSet | Iterable[Parameter] = (), arity: int = 1) -> FunctorExpr:
    return Closure(fn, params if isinstance(params, ParamSet) else ParamSet(params), arity)


def combine(op: str, a: FunctorExpr, b: FunctorExpr) -> FunctorExpr:
    return _BinaryOp(op, a, b)


def compose(outer: FunctorExpr, inners: Sequence[FunctorExpr]) -> FunctorExpr:
    return Composition(outer, inners)


def coordinate(index: int, arity: int) -> FunctorExpr:
    return Coordinate(index, arity)


def identity() -> FunctorExpr:
    return Coordinate(0, 1)


# ---------------------------------------------------------------------------
# IR -> hk_program_t

_OPCODE = {"add": _lib.OP_ADD, "sub": _lib.OP_SUB, "mul": _lib.OP_MUL, "div": _lib.OP_DIV,
           "neg": _lib.OP_NEG, "sqrt": _lib.OP_SQRT, "exp": _lib.OP_EXP, "log": _lib.OP_LOG,
           "square": _lib.OP_SQUARE, "add0": _lib.OP_ADD0, "udiv": _lib.OP_UDIV}


def _children(node) -> list:
    kind = node[0]
    if kind in _BINARY:
        return [node[1], node[2]]
    if kind in _UNARY or kind in ("gauss", "expo", "bw"):
        return [node[1]]
    return []


def _is_leaf(node) -> bool:
    return node[0] in ("col", "const")


def compile_program(root, keep: Sequence = (), params: Sequence[float] | None = None):
    """Hash-consed DAG -> SSA ops in dependency order with liveness-based slots.

    Interior nodes are computed once (common subexpressions shared); leaves
    (column loads, constants) are re-issued right before each use so they
    never hold a register across the program.  ``keep`` lists further nodes
    whose values must survive to the end (multi-output programs, e.g. the
    per-component p.d.f.s next to the density); with ``keep`` the result is
    (program, slot of each kept node).  A constant ("const", ("p", k)) is the
    k-th of ``params`` (parametric programs: the structure is fixed, the
    values change per call -- see lower_density).
    """
    order: list = []                 # node per op
    args_of: list = []               # operand op indices per op
    index: dict = {}                 # interior node -> op index

    def emit(node, operands) -> int:
        order.append(node)
        args_of.append(operands)
        return len(order) - 1

    roots = [root, *keep]
    stack = [(r, False) for r in reversed(roots)]
    while stack:                     # iterative post-order over interior nodes
        node, done = stack.pop()
        if _is_leaf(node):
            continue
        if done:
            if node not in index:
                ops = []
                for ch in _children(node):
                    ops.append(emit(ch, []) if _is_leaf(ch) else index[ch])
                index[node] = emit(node, ops)
            continue
        if node in index:
            continue
        stack.append((node, True))
        for ch in reversed(_children(node)):
            stack.append((ch, False))
    root_ops = [emit(r, []) if _is_leaf(r) else index[r] for r in roots]
    pinned = set(root_ops)
    if len(order) > _lib.HK_MAX_PROGRAM:
        raise NotImplementedError(f"expression needs {len(order)} device ops "
                                  f"(limit {_lib.HK_MAX_PROGRAM})")
    last_use = {}
    for i, ops in enumerate(args_of):
        for j in ops:
            last_use[j] = i
    slot: dict = {}
    free: list[int] = list(range(_lib.HK_MAX_SLOTS - 1, -1, -1))
    prog = _lib.hk_program_t()
    prog.n_ops = len(order)
    for i, node in enumerate(order):
        src = [slot[j] for j in args_of[i]]
        for j in set(args_of[i]):    # operands whose last use is here free their slot
            if last_use.get(j) == i and j not in pinned:
                free.append(slot[j])
        if not free:
            raise NotImplementedError("expression needs more than "
                                      f"{_lib.HK_MAX_SLOTS} live device registers")
        dst = free.pop()
        slot[i] = dst
        kind = node[0]
        prog.dst[i] = dst
        prog.a[i] = src[0] if src else 0
        prog.b[i] = src[1] if len(src) > 1 else 0
        if kind == "col":
            prog.op[i] = _lib.OP_COL
            prog.a[i] = node[1]
        elif kind == "const":
            prog.op[i] = _lib.OP_CONST
            v = node[1]
            prog.cst[i] = params[v[1]] if isinstance(v, tuple) else v
        elif kind == "gauss":
            prog.op[i], prog.cst[i], prog.cst2[i] = _lib.OP_GAUSS, node[2], node[3]
        elif kind == "expo":
            prog.op[i], prog.cst[i] = _lib.OP_EXPO, node[2]
        elif kind == "bw":
            prog.op[i], prog.cst[i], prog.cst2[i] = _lib.OP_BW, node[2], node[3]
        else:
            prog.op[i] = _OPCODE[kind]
    prog.result = slot[root_ops[0]]
    if keep:
        return prog, [slot[r] for r in root_ops[1:]]
    return prog


def _param_leaf(v):
    """A builtin shape's parameter inside its op: a value, or (symbolic
    parameter tracing) already an IR leaf."""
    return v if isinstance(v, tuple) else ("const", v)


def desugar(node):
    """Builtin shape ops (gauss/expo/bw, which carry their parameters inside
    the op) rewritten as primitive ops with constant leaves, in the
    reference's operation order (functors.py:142-143, :161), so that a
    parametric program can vary those parameters per call."""
    memo: dict = {}

    def walk(n):
        key = id(n)
        if key in memo:
            return memo[key]
        kind = n[0]
        if kind in ("col", "const", "pv", "nv", "yv"):
            out = n
        elif kind == "gauss":
            a, mu, s = walk(n[1]), _param_leaf(n[2]), _param_leaf(n[3])
            z = ("udiv", ("sub", a, mu), s)
            out = ("udiv", ("exp", ("mul", ("mul", ("const", -0.5), z), z)), ("mul", s, ("const", _SQRT_2PI)))
        elif kind == "expo":
            out = ("exp", ("udiv", ("neg", walk(n[1])), _param_leaf(n[2])))
        elif kind == "bw":
            m0, g0 = _param_leaf(n[2]), _param_leaf(n[3])
            m2 = ("mul", m0, m0)
            t = ("sub", walk(n[1]), m2)
            out = ("udiv", ("const", 1.0), ("add", ("mul", t, t), ("mul", m2, ("mul", g0, g0))))
        else:
            out = (kind, *[walk(c) for c in n[1:]])
        memo[key] = out
        return out

    return walk(node)


def parametrize(roots: Sequence) -> tuple[tuple, list[float]]:
    """Lift every constant of a (desugared) IR DAG into a parameter slot:
    returns (roots with ("const", ("p", k)) leaves, [value_k]).  Shared
    sub-DAGs (same object) stay shared; the structure no longer depends on
    the values, so one compiled program serves every parameter point."""
    memo: dict = {}
    values: list[float] = []

    def walk(n):
        key = id(n)
        if key in memo:
            return memo[key]
        kind = n[0]
        if kind == "const":
            out = ("const", ("p", len(values)))
            values.append(float(n[1]))
        elif kind in ("pv", "nv", "yv"):   # symbolic parameter / norm / yield: a slot, the leaf as its source
            out = ("const", ("p", len(values)))
            values.append(n)
        elif kind == "col":
            out = n
        else:
            out = (kind, *[walk(c) for c in n[1:]])
        memo[key] = out
        return out

    return tuple(walk(r) for r in roots), values


def lower_average(expr: FunctorExpr, arg_builder, names: Sequence[str], with_root: bool = False):
    """Program computing expr(*arg_builder(columns)) per event, plus the
    argument nodes (for error messages) [and the IR root]."""
    args = trace_arg_builder(arg_builder, names)
    if len(args) != expr.arity:
        raise EvaluationError(f"expression consumes {expr.arity} arguments, got {len(args)}")
    root = expr.lower(args)
    if with_root:
        return compile_program(root), args, root
    return compile_program(root), args


def pair_mass2_node(i: int, j: int):
    """IR of m^2(daughters i+j) (1-based) exactly as tracing the reference's
    pinned builder produces it (test_phasespace.py:196-201)."""
    def comp(c):
        return ("add", ("col", 1 + 4 * (i - 1) + c), ("col", 1 + 4 * (j - 1) + c))

    e, x, y, z = (comp(c) for c in range(4))
    return ("sub", ("sub", ("sub", ("mul", e, e), ("mul", x, x)), ("mul", y, y)), ("mul", z, z))


def match_pair_integrand(root, n_daughters: int):
    """hk_pair_integrand_t if `root` is m^2_ij + 0.0 or BW(m^2_ij), else None."""
    kind, inner = None, None
    if root[0] == "add0":
        kind, inner = _lib.HK_PAIR_MASS2, root[1]
    elif root[0] == "bw":
        kind, inner = _lib.HK_PAIR_BW, root[1]
    if kind is None or inner[0] != "sub":
        return None
    for i in range(1, n_daughters + 1):
        for j in range(1, n_daughters + 1):
            if i != j and inner == pair_mass2_node(i, j):
                out = _lib.hk_pair_integrand_t()
                out.kind, out.i, out.j = kind, i - 1, j - 1
                if kind == _lib.HK_PAIR_BW:
                    out.m0, out.g0 = root[2], root[3]
                return out
    return None


def eval_node(node, cols: dict[int, float]) -> float:
    """Scalar host evaluation of an IR node (error messages only)."""
    kind = node[0]
    if kind == "col":
        return cols[node[1]]
    if kind == "const":
        return node[1]
    v = [eval_node(c, cols) for c in _children(node)]
    with np.errstate(all="ignore"):
        x = np.float64(v[0])
        if kind == "add":
            return x + v[1]
        if kind == "sub":
            return x - v[1]
        if kind == "mul":
            return x * v[1]
        if kind in ("div", "udiv"):
            return x / v[1]
        if kind == "neg":
            return -x
        if kind == "sqrt":
            return np.sqrt(x)
        if kind == "exp":
            return np.exp(x)
        if kind == "log":
            return np.log(x)
        if kind == "square":
            return x * x
        if kind == "add0":
            return x + 0.0
        if kind == "gauss":
            z = (x - node[2]) / node[3]
            return np.exp(-0.5 * z * z) / (node[3] * _SQRT_2PI)
        if kind == "expo":
            return np.exp(-x / node[2])
        if kind == "bw":
            return 1.0 / ((x - node[2] * node[2]) ** 2 + (node[2] * node[2]) * (node[3] * node[3]))
    raise ValueError(kind)


def columns_used(nodes) -> set[int]:
    out: set[int] = set()
    stack = list(nodes)
    while stack:
        n = stack.pop()
        if n[0] == "col":
            out.add(n[1])
        stack.extend(_children(n))
    return out


def map_evaluate(expr: FunctorExpr, store, arg_columns: Sequence[str], workers: int | None = 1):
    """expr over every row projection (functors.py:288-318), on the GPU."""
    if len(arg_columns) != expr.arity:
        raise ValueError(f"expression consumes {expr.arity} arguments, got {len(arg_columns)} columns")
    for name in arg_columns:
        if store.schema.dtype(name) is not np.float64:
            raise ValueError(f"column {name!r} is not real64")
    from .phasespace import _map_program  # noqa: PLC0415 -- avoid import cycle
    prog = compile_program(expr.lower([("col", i) for i in range(len(arg_columns))]))
    out = _map_program(prog, store.device_columns(arg_columns), len(store))
    out.flags.writeable = False
    return out
