"""Device compilation of user combination integrals.

The reference runs an arbitrary Python callable once per rectangle
(integrate.combine_integrate / combine_integrate_timedep / integrate_single,
integrate.py:51-171; MatrixJob's custom path, matrix.py:184-196).  Python callables cannot
run on the GPU, so this module translates the callable's source into a C expression
(Python float semantics: ``max``/``min`` as Python defines them, ``%`` with the divisor's
sign, ``x ** 2`` as one correctly rounded product, ``a if c else b``, ``and``/``or``
returning operands, ...), and ``csrc/pcf_jit.cu`` compiles it with the kernel template
through NVRTC for sm_100a.  Modules are cached per generated source.

Supported: lambdas and single-expression functions (optionally with local assignments
before the ``return``) over float arguments, using arithmetic, comparisons, conditional
expressions, the builtins ``abs``/``min``/``max``/``pow``/``float``, ``math`` functions
and constants, the matching ``numpy`` ufuncs (``np.abs``, ``np.maximum``,
``np.exp``, ...), numeric constants and numeric closure/global variables (inlined
exactly as hexadecimal literals), and calls to other such functions.  Anything else
raises :class:`errors.UnsupportedIntegrand` -- there is no CPU fallback.

Integrands made of ``+ - * /``, ``abs``, ``min``, ``max``, ``sqrt`` and constants
reproduce the reference bit for bit (IEEE operations, no FMA contraction);
transcendental functions use CUDA's libdevice (within 2 ulp of glibc).
"""

from __future__ import annotations

import ast
import builtins
import ctypes
import hashlib
import inspect
import math
import textwrap
import threading

import numpy as np

from . import _native, errors

_MATH_FUNCS = {
    "sqrt": "sqrt", "exp": "exp", "expm1": "expm1", "log": "log", "log2": "log2",
    "log10": "log10", "log1p": "log1p", "sin": "sin", "cos": "cos", "tan": "tan",
    "asin": "asin", "acos": "acos", "atan": "atan", "atan2": "atan2", "sinh": "sinh",
    "cosh": "cosh", "tanh": "tanh", "asinh": "asinh", "acosh": "acosh", "atanh": "atanh",
    "floor": "floor", "ceil": "ceil", "trunc": "trunc", "fabs": "fabs", "pow": "pow",
    "fmod": "fmod", "hypot": "hypot", "copysign": "copysign", "erf": "erf", "erfc": "erfc",
    "gamma": "tgamma", "lgamma": "lgamma", "cbrt": "cbrt", "exp2": "exp2",
}
_NP_FUNCS = {
    "abs": "fabs", "absolute": "fabs", "fabs": "fabs", "sqrt": "sqrt", "exp": "exp",
    "expm1": "expm1", "log": "log", "log2": "log2", "log10": "log10", "log1p": "log1p",
    "sin": "sin", "cos": "cos", "tan": "tan", "arcsin": "asin", "arccos": "acos",
    "arctan": "atan", "arctan2": "atan2", "sinh": "sinh", "cosh": "cosh", "tanh": "tanh",
    "floor": "floor", "ceil": "ceil", "trunc": "trunc", "power": "pow", "hypot": "hypot",
    "copysign": "copysign", "maximum": "pcf_npmax", "minimum": "pcf_npmin", "fmax": "fmax",
    "fmin": "fmin", "cbrt": "cbrt", "exp2": "exp2", "square": "pcf_sq", "fmod": "fmod",
}
def _literal(x) -> str:
    x = float(x)
    if math.isnan(x):
        return "PCF_NAN"
    if math.isinf(x):
        return "PCF_INF" if x > 0 else "(-PCF_INF)"
    return f"({x.hex()})"


class _Translator:
    """Python AST (one function) -> C source, resolving free names in the function's
    closure and globals."""

    def __init__(self, unit):
        self.unit = unit  # shared state across helper functions: emitted helpers

    def function(self, fn, cname, nargs=None):
        tree, params = _parse_function(fn)
        if nargs is not None and len(params) != nargs:
            raise errors.UnsupportedIntegrand(
                f"{_name(fn)} takes {len(params)} arguments, expected {nargs}")
        env = _environment(fn)
        local = {p: f"a_{p}" for p in params}
        body = []
        stmts = tree
        for st in stmts[:-1]:
            if not (isinstance(st, ast.Assign) and len(st.targets) == 1
                    and isinstance(st.targets[0], ast.Name)):
                raise errors.UnsupportedIntegrand(
                    f"{_name(fn)}: only `name = expression` statements before the return")
            name = st.targets[0].id
            expr = self.expr(st.value, local, env)
            cv = f"l_{name}_{len(body)}"
            body.append(f"  const double {cv} = {expr};")
            local[name] = cv
        last = stmts[-1]
        if not isinstance(last, ast.Return) or last.value is None:
            raise errors.UnsupportedIntegrand(f"{_name(fn)}: must end with `return expression`")
        body.append(f"  return {self.expr(last.value, local, env)};")
        args = ", ".join(f"double a_{p}" for p in params)
        return f"__device__ double {cname}({args}) {{\n" + "\n".join(body) + "\n}\n"

    # -- expressions
    def expr(self, node, local, env):
        e = lambda n: self.expr(n, local, env)  # noqa: E731
        if isinstance(node, ast.Constant):
            if isinstance(node.value, (bool, int, float)):
                return _literal(node.value)
            raise errors.UnsupportedIntegrand(f"constant {node.value!r}")
        if isinstance(node, ast.Name):
            if node.id in local:
                return local[node.id]
            return self.value(self.resolve(node.id, env), node.id)
        if isinstance(node, ast.Attribute):
            return self.value(self.resolve_attr(node, env), ast.unparse(node))
        if isinstance(node, ast.BinOp):
            a, b = e(node.left), e(node.right)
            op = type(node.op)
            if op is ast.Add:
                return f"({a} + {b})"
            if op is ast.Sub:
                return f"({a} - {b})"
            if op is ast.Mult:
                return f"({a} * {b})"
            if op is ast.Div:
                return f"({a} / {b})"
            if op is ast.Mod:
                return f"pcf_pymod({a}, {b})"
            if op is ast.FloorDiv:
                return f"pcf_pyfloordiv({a}, {b})"
            if op is ast.Pow:
                if isinstance(node.right, ast.Constant) and node.right.value == 2:
                    return f"pcf_sq({a})"
                if isinstance(node.right, ast.Constant) and node.right.value == 1:
                    return f"({a})"
                return f"pow({a}, {b})"
            raise errors.UnsupportedIntegrand(f"operator {op.__name__}")
        if isinstance(node, ast.UnaryOp):
            a = e(node.operand)
            if isinstance(node.op, ast.USub):
                return f"(-{a})"
            if isinstance(node.op, ast.UAdd):
                return f"(+{a})"
            if isinstance(node.op, ast.Not):
                return f"(({a}) == 0.0 ? 1.0 : 0.0)"
            raise errors.UnsupportedIntegrand(f"unary {type(node.op).__name__}")
        if isinstance(node, ast.Compare):
            ops = {ast.Lt: "<", ast.LtE: "<=", ast.Gt: ">", ast.GtE: ">=", ast.Eq: "==",
                   ast.NotEq: "!="}
            parts, left = [], e(node.left)
            for op, comp in zip(node.ops, node.comparators):
                if type(op) not in ops:
                    raise errors.UnsupportedIntegrand(f"comparison {type(op).__name__}")
                right = e(comp)
                parts.append(f"({left} {ops[type(op)]} {right})")
                left = right
            return "((" + " && ".join(parts) + ") ? 1.0 : 0.0)"
        if isinstance(node, ast.BoolOp):
            vals = [e(v) for v in node.values]
            out = vals[-1]
            for v in reversed(vals[:-1]):
                if isinstance(node.op, ast.And):  # x and y: x if x is falsy else y
                    out = f"((({v}) == 0.0) ? ({v}) : {out})"
                else:  # x or y: x if x is truthy else y
                    out = f"((({v}) != 0.0) ? ({v}) : {out})"
            return out
        if isinstance(node, ast.IfExp):
            return f"((({e(node.test)}) != 0.0) ? {e(node.body)} : {e(node.orelse)})"
        if isinstance(node, ast.Call):
            if node.keywords:
                raise errors.UnsupportedIntegrand("keyword arguments in integrand calls")
            fobj = (self.resolve(node.func.id, env) if isinstance(node.func, ast.Name)
                    else self.resolve_attr(node.func, env) if isinstance(node.func, ast.Attribute)
                    else None)
            args = [e(a) for a in node.args]
            return self.call(fobj, args, ast.unparse(node.func))
        raise errors.UnsupportedIntegrand(f"unsupported syntax: {ast.unparse(node)}")

    def resolve(self, name, env):
        if name in env:
            return env[name]
        if hasattr(builtins, name):
            return getattr(builtins, name)
        raise errors.UnsupportedIntegrand(f"unknown name {name!r}")

    def resolve_attr(self, node, env):
        if isinstance(node.value, ast.Name):
            base = self.resolve(node.value.id, env)
        elif isinstance(node.value, ast.Attribute):
            base = self.resolve_attr(node.value, env)
        else:
            raise errors.UnsupportedIntegrand(f"attribute of {ast.unparse(node.value)}")
        try:
            return getattr(base, node.attr)
        except AttributeError:
            raise errors.UnsupportedIntegrand(f"unknown attribute {ast.unparse(node)}") from None

    def value(self, obj, text):
        if isinstance(obj, (bool, int, float, np.integer, np.floating)):
            return _literal(obj)
        raise errors.UnsupportedIntegrand(f"{text!r} is not a number")

    def call(self, f, args, text):
        if f is abs or f is math.fabs:
            return self._n(f"fabs({args[0]})", args, 1, text)
        if f is float:
            return self._n(f"({args[0]})", args, 1, text)
        if f is max or f is min:
            if len(args) < 2:
                raise errors.UnsupportedIntegrand(f"{text} needs >= 2 arguments")
            fn = "pcf_pymax" if f is max else "pcf_pymin"
            out = args[0]
            for a in args[1:]:
                out = f"{fn}({out}, {a})"
            return out
        if f is pow:
            return self._n(f"pow({args[0]}, {args[1]})", args, 2, text)
        for mod, table in ((math, _MATH_FUNCS), (np, _NP_FUNCS)):
            name = getattr(f, "__name__", None)
            if name in table and getattr(mod, name, None) is f:
                cf = table[name]
                return f"{cf}({', '.join(args)})"
        if inspect.isfunction(f):
            cname = self.unit.helper(f)
            return f"{cname}({', '.join(args)})"
        raise errors.UnsupportedIntegrand(f"call of {text!r} has no device translation")

    @staticmethod
    def _n(s, args, n, text):
        if len(args) != n:
            raise errors.UnsupportedIntegrand(f"{text} takes {n} argument(s)")
        return s


class _Unit:
    """One generated translation unit: helper functions + the entry points."""

    def __init__(self):
        self.helpers = {}   # id(fn) -> (cname, source)
        self.order = []

    def helper(self, fn):
        key = id(fn)
        if key not in self.helpers:
            cname = f"pcf_fn{len(self.helpers)}_{_safe(getattr(fn, '__name__', 'f'))}"
            self.helpers[key] = (cname, None)  # recursion guard
            src = _Translator(self).function(fn, cname)
            self.helpers[key] = (cname, src)
            self.order.append(key)
        return self.helpers[key][0]

    def source(self, entries):
        return "".join(self.helpers[k][1] for k in self.order) + "".join(entries)


def _safe(s):
    return "".join(c if c.isalnum() else "_" for c in s)[:32]


def _name(fn):
    return getattr(fn, "__qualname__", repr(fn))


def _environment(fn):
    env = dict(getattr(fn, "__globals__", {}))
    code = getattr(fn, "__code__", None)
    if code is not None and fn.__closure__:
        for nm, cell in zip(code.co_freevars, fn.__closure__):
            try:
                env[nm] = cell.cell_contents
            except ValueError:
                pass
    return env


def _parse_function(fn):
    """(statements, parameter names) of a lambda or def."""
    if not inspect.isfunction(fn):
        raise errors.UnsupportedIntegrand(f"{fn!r} is not a Python function")
    code = fn.__code__
    if code.co_flags & (inspect.CO_VARARGS | inspect.CO_VARKEYWORDS) or code.co_kwonlyargcount:
        raise errors.UnsupportedIntegrand(f"{_name(fn)}: only positional arguments")
    params = list(code.co_varnames[: code.co_argcount])
    try:
        src = textwrap.dedent(inspect.getsource(fn))
    except (OSError, TypeError):
        raise errors.UnsupportedIntegrand(f"source of {_name(fn)} is unavailable") from None
    try:
        mod = ast.parse(src)
    except SyntaxError:
        # a lambda inside a larger expression: parse the enclosing lines leniently
        mod = ast.parse("(" + src.strip().rstrip(",").rstrip("\\") + ")") if src else None
    if fn.__name__ == "<lambda>":
        cands = [n for n in ast.walk(mod) if isinstance(n, ast.Lambda)
                 and [a.arg for a in n.args.args] == params]
        if len(cands) > 1:  # several lambdas on the line: match the compiled body
            target = (code.co_code, code.co_consts, code.co_names)
            match = []
            for n in cands:
                try:
                    c = compile(ast.Expression(n), "<jit>", "eval").co_consts
                    lc = next(x for x in c if inspect.iscode(x))
                    if (lc.co_code, lc.co_consts, lc.co_names) == target:
                        match.append(n)
                except (StopIteration, SyntaxError, ValueError):
                    continue
            cands = match or cands[:1]
        if not cands:
            raise errors.UnsupportedIntegrand(f"cannot locate the source of {_name(fn)}")
        return [ast.Return(value=cands[0].body)], params
    defs = [n for n in ast.walk(mod) if isinstance(n, ast.FunctionDef) and n.name == fn.__name__]
    if not defs:
        raise errors.UnsupportedIntegrand(f"cannot locate the source of {_name(fn)}")
    body = list(defs[0].body)
    if body and isinstance(body[0], ast.Expr) and isinstance(getattr(body[0], "value", None),
                                                             ast.Constant):
        body = body[1:]  # docstring
    if not body:
        raise errors.UnsupportedIntegrand(f"{_name(fn)} has an empty body")
    return body, params


class _Sym:
    """Symbolic float for tracing integrands whose source is unavailable (REPL, exec):
    arithmetic, abs and numpy ufuncs are recorded as C; Python control flow on the
    values (if/max/min/math.*) cannot be traced."""

    __array_priority__ = 1000

    def __init__(self, c):
        self.c = c

    @staticmethod
    def _c(x):
        if isinstance(x, _Sym):
            return x.c
        if isinstance(x, (bool, int, float, np.integer, np.floating)):
            return _literal(x)
        raise errors.UnsupportedIntegrand(f"cannot trace operand {x!r}")

    def _bin(self, o, fmt, rev=False):
        a, b = (self._c(o), self.c) if rev else (self.c, self._c(o))
        return _Sym(fmt.format(a, b))

    def __add__(self, o): return self._bin(o, "({} + {})")
    def __radd__(self, o): return self._bin(o, "({} + {})", True)
    def __sub__(self, o): return self._bin(o, "({} - {})")
    def __rsub__(self, o): return self._bin(o, "({} - {})", True)
    def __mul__(self, o): return self._bin(o, "({} * {})")
    def __rmul__(self, o): return self._bin(o, "({} * {})", True)
    def __truediv__(self, o): return self._bin(o, "({} / {})")
    def __rtruediv__(self, o): return self._bin(o, "({} / {})", True)
    def __mod__(self, o): return self._bin(o, "pcf_pymod({}, {})")
    def __rmod__(self, o): return self._bin(o, "pcf_pymod({}, {})", True)
    def __floordiv__(self, o): return self._bin(o, "pcf_pyfloordiv({}, {})")
    def __rfloordiv__(self, o): return self._bin(o, "pcf_pyfloordiv({}, {})", True)

    def __pow__(self, o):
        if isinstance(o, (int, float)) and o == 2:
            return _Sym(f"pcf_sq({self.c})")
        return self._bin(o, "pow({}, {})")

    def __rpow__(self, o): return self._bin(o, "pow({}, {})", True)
    def __neg__(self): return _Sym(f"(-{self.c})")
    def __pos__(self): return self
    def __abs__(self): return _Sym(f"fabs({self.c})")
    def __lt__(self, o): return self._bin(o, "(({} < {}) ? 1.0 : 0.0)")
    def __le__(self, o): return self._bin(o, "(({} <= {}) ? 1.0 : 0.0)")
    def __gt__(self, o): return self._bin(o, "(({} > {}) ? 1.0 : 0.0)")
    def __ge__(self, o): return self._bin(o, "(({} >= {}) ? 1.0 : 0.0)")

    def __bool__(self):
        raise errors.UnsupportedIntegrand(
            "the integrand branches on its arguments and its source is unavailable for "
            "translation; define it in a source file (def or lambda)")

    def __float__(self):
        raise errors.UnsupportedIntegrand(
            "the integrand converts its argument to a Python float (e.g. math.*) and its "
            "source is unavailable; use numpy ufuncs or define it in a source file")

    def __array_ufunc__(self, ufunc, method, *inputs, **kw):
        if method != "__call__" or kw or ufunc.__name__ not in _NP_FUNCS:
            raise errors.UnsupportedIntegrand(f"numpy {ufunc.__name__} cannot be traced")
        return _Sym(f"{_NP_FUNCS[ufunc.__name__]}({', '.join(self._c(x) for x in inputs)})")


def _traced(fn, cname, nargs):
    code = getattr(fn, "__code__", None)
    if code is None or code.co_argcount != nargs:
        raise errors.UnsupportedIntegrand(f"{_name(fn)}: expected {nargs} arguments")
    names = list(code.co_varnames[:nargs])
    out = fn(*[_Sym(f"a_{n}") for n in names])
    body = _Sym._c(out)
    args = ", ".join(f"double a_{n}" for n in names)
    return f"__device__ double {cname}({args}) {{\n  return {body};\n}}\n"


def _function(unit, fn, cname, nargs):
    """Translate from source; if the source is unavailable, trace with symbols."""
    if not inspect.isfunction(fn) and callable(fn):  # e.g. r=math.sqrt, h=max
        names = ["x", "y", "t"][:nargs] if nargs > 1 else ["x"]
        body = _Translator(unit).call(fn, [f"a_{n}" for n in names], repr(fn))
        args = ", ".join(f"double a_{n}" for n in names)
        return f"__device__ double {cname}({args}) {{\n  return {body};\n}}\n"
    try:
        return _Translator(unit).function(fn, cname, nargs)
    except errors.UnsupportedIntegrand as exc:
        if "source of" not in str(exc):
            raise
        return _traced(fn, cname, nargs)


def generate(h=None, H=None, r=None, u=None):
    """C definitions for the kernel template (see csrc/pcf_jit_kernels.cuh)."""
    unit = _Unit()
    entries = []
    if H is not None:
        entries.append(_function(unit, H, "pcf_H", 3))
        mode = 1
    else:
        mode = 0
        if h is not None:
            entries.append(_function(unit, h, "pcf_h", 2))
        else:
            entries.append("__device__ double pcf_h(double x, double y) { return 0.0; }\n")
    if r is not None:
        entries.append(_function(unit, r, "pcf_r", 1))
    if u is not None:
        entries.append(_function(unit, u, "pcf_u", 1))
    head = (f"#define PCF_MODE {mode}\n#define PCF_HAS_R {int(r is not None)}\n"
            f"#define PCF_HAS_U {int(u is not None)}\n"
            "#define PCF_INF __longlong_as_double(0x7ff0000000000000LL)\n"
            "#define PCF_NAN __longlong_as_double(0x7ff8000000000000LL)\n"
            "__device__ __forceinline__ double pcf_pymax(double a, double b);\n"
            "__device__ __forceinline__ double pcf_pymin(double a, double b);\n"
            "__device__ __forceinline__ double pcf_npmax(double a, double b);\n"
            "__device__ __forceinline__ double pcf_npmin(double a, double b);\n"
            "__device__ __forceinline__ double pcf_pymod(double x, double y);\n"
            "__device__ __forceinline__ double pcf_pyfloordiv(double x, double y);\n"
            "__device__ __forceinline__ double pcf_sq(double x);\n")
    return head + unit.source(entries)


class JitModule:
    """A loaded NVRTC module (one per generated source, cached)."""

    _cache = {}
    _lock = threading.Lock()

    def __init__(self, handle, defs):
        self.handle = handle
        self.defs = defs

    @classmethod
    def get(cls, defs):
        key = hashlib.sha1(defs.encode()).hexdigest()
        with cls._lock:
            mod = cls._cache.get(key)
            if mod is None:
                lib = _native.load()
                h = ctypes.c_void_p()
                log = ctypes.create_string_buffer(8192)
                rc = lib.pcf_jit_load(defs.encode(), ctypes.byref(h), log, 8192)
                if rc != 0:
                    msg = lib.pcf_last_error().decode(errors="replace")
                    if rc == 1:  # PCF_ERR_ARG: the generated code did not compile
                        raise errors.UnsupportedIntegrand(
                            f"device compilation failed: {log.value.decode(errors='replace')}"
                            f"\n--- generated ---\n{defs}")
                    raise errors.BackendUnavailable(msg)
                mod = cls(h, defs)
                cls._cache[key] = mod
            return mod


class JitTiles:
    """The tile kernels compiled for one generated integrand and record kind (cached);
    csrc/pcf_jit.cu pcf_jit_tiles_load."""

    _cache = {}
    _lock = threading.Lock()

    def __init__(self, handle, defs, f32):
        self.handle = handle
        self.defs = defs
        self.f32 = f32
        self.has_r = "#define PCF_HAS_R 1" in defs

    @classmethod
    def get(cls, defs, f32):
        key = (hashlib.sha1(defs.encode()).hexdigest(), bool(f32))
        with cls._lock:
            mod = cls._cache.get(key)
            if mod is None:
                lib = _native.load()
                h = ctypes.c_void_p()
                log = ctypes.create_string_buffer(8192)
                rc = lib.pcf_jit_tiles_load(defs.encode(), int(bool(f32)), ctypes.byref(h), log,
                                            8192)
                if rc != 0:
                    msg = lib.pcf_last_error().decode(errors="replace")
                    if rc == 1:
                        raise errors.UnsupportedIntegrand(
                            f"device compilation failed: {log.value.decode(errors='replace')}")
                    raise errors.BackendUnavailable(msg)
                mod = cls(h, defs, bool(f32))
                cls._cache[key] = mod
            return mod


def compile_only(defs):
    """NVRTC-compile without a GPU (CUBIN size); raises UnsupportedIntegrand on errors."""
    lib = _native.load()
    size = ctypes.c_int64(0)
    log = ctypes.create_string_buffer(8192)
    rc = lib.pcf_jit_cubin(defs.encode(), None, 0, ctypes.byref(size), log, 8192)
    if rc != 0:
        raise errors.UnsupportedIntegrand(
            f"device compilation failed ({lib.pcf_last_error().decode()}): "
            f"{log.value.decode(errors='replace')}")
    return size.value


def compile_tiles_only(defs, f32=False):
    """NVRTC-compile the tile kernels for a generated integrand without a GPU (CUBIN
    size); every instantiation must be exported."""
    lib = _native.load()
    size = ctypes.c_int64(0)
    log = ctypes.create_string_buffer(8192)
    rc = lib.pcf_jit_tiles_cubin(defs.encode(), int(bool(f32)), ctypes.byref(size), log, 8192)
    if rc != 0:
        raise errors.UnsupportedIntegrand(
            f"tile compilation failed ({lib.pcf_last_error().decode()}): "
            f"{log.value.decode(errors='replace')}")
    return size.value
