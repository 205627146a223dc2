"""Host-side objective DAG over the 6x6 homogenized tensor (inc/objective.hpp:19-66).

36 scalars, no kernel: this is the Python face of the reference's ``Expr`` so
users can write custom objectives and feed ``Expr.backward`` seeds to
``Homogenizer.tensor_sensitivity``. The native runner uses the C++ twin
(csrc/objective.cpp); tests check the two agree.
"""
from __future__ import annotations

import math

import numpy as np


class EvalError(RuntimeError):
    pass


class Expr:
    __slots__ = ("op", "value", "i", "j", "a", "b")

    def __init__(self, op, value=0.0, i=0, j=0, a=None, b=None):
        self.op, self.value, self.i, self.j, self.a, self.b = op, value, i, j, a, b

    # construction (src/objective.cpp:190-234: eager constant folding)
    @staticmethod
    def constant(v):
        return Expr("const", float(v))

    @staticmethod
    def entry(i, j):
        if not (0 <= i <= 5 and 0 <= j <= 5):
            raise ValueError("tensor entry index out of range")
        return Expr("entry", 0.0, i, j)

    @staticmethod
    def _wrap(x):
        return x if isinstance(x, Expr) else Expr.constant(x)

    def _bin(self, other, op, fold):
        other = Expr._wrap(other)
        if self.op == "const" and other.op == "const":
            return Expr.constant(fold(self.value, other.value))
        return Expr(op, a=self, b=other)

    def __add__(self, o):
        return self._bin(o, "add", lambda x, y: x + y)

    def __radd__(self, o):
        return Expr._wrap(o) + self

    def __sub__(self, o):
        return self._bin(o, "sub", lambda x, y: x - y)

    def __rsub__(self, o):
        return Expr._wrap(o) - self

    def __mul__(self, o):
        return self._bin(o, "mul", lambda x, y: x * y)

    def __rmul__(self, o):
        return Expr._wrap(o) * self

    def __truediv__(self, o):
        def fold(x, y):
            if y == 0.0:
                raise EvalError("division by zero in constant fold")
            return x / y
        return self._bin(o, "div", fold)

    def __rtruediv__(self, o):
        return Expr._wrap(o) / self

    def __neg__(self):
        return Expr.constant(-self.value) if self.op == "const" else Expr("neg", a=self)

    def pow(self, e):
        return Expr.constant(self.value ** e) if self.op == "const" else Expr("pow", float(e), a=self)

    def log(self):
        if self.op == "const":
            if not self.value > 0:
                raise EvalError("log of non-positive constant")
            return Expr.constant(math.log(self.value))
        return Expr("log", a=self)

    def exp(self):
        return Expr.constant(math.exp(self.value)) if self.op == "const" else Expr("exp", a=self)

    # evaluation (src/objective.cpp:70-130)
    def _ev(self, c, memo):
        k = id(self)
        if k in memo:
            return memo[k]
        op = self.op
        if op == "const":
            v = self.value
        elif op == "entry":
            v = float(c[self.i, self.j])
        elif op == "add":
            v = self.a._ev(c, memo) + self.b._ev(c, memo)
        elif op == "sub":
            v = self.a._ev(c, memo) - self.b._ev(c, memo)
        elif op == "mul":
            v = self.a._ev(c, memo) * self.b._ev(c, memo)
        elif op == "div":
            den = self.b._ev(c, memo)
            if den == 0.0:
                raise EvalError(f"division by zero at {self.str()[:120]}")
            v = self.a._ev(c, memo) / den
        elif op == "pow":
            base, e = self.a._ev(c, memo), self.value
            if base < 0.0 and e != math.floor(e):
                raise EvalError("fractional power of negative value")
            if base == 0.0 and e < 1.0 and e != 0.0:
                raise EvalError("non-positive base of power")
            v = base ** e
        elif op == "log":
            x = self.a._ev(c, memo)
            if not x > 0.0:
                raise EvalError("log of non-positive value")
            v = math.log(x)
        elif op == "exp":
            v = math.exp(self.a._ev(c, memo))
        else:  # neg
            v = -self.a._ev(c, memo)
        memo[k] = v
        return v

    def eval(self, c) -> float:
        return self._ev(np.asarray(c, dtype=np.float64).reshape(6, 6), {})

    def backward(self, seed, c) -> np.ndarray:
        """d(seed*expr)/dC, (i,j) and (j,i) separately (src/objective.cpp:132-180)."""
        c = np.asarray(c, dtype=np.float64).reshape(6, 6)
        val = {}
        self._ev(c, val)
        order, seen = [], set()

        def topo(n):
            if id(n) in seen:
                return
            seen.add(id(n))
            if n.a is not None:
                topo(n.a)
            if n.b is not None:
                topo(n.b)
            order.append(n)
        topo(self)
        adj = {id(self): float(seed)}
        g = np.zeros((6, 6))
        for n in reversed(order):
            if id(n) not in adj:
                continue
            a = adj[id(n)]
            op = n.op
            if op == "entry":
                g[n.i, n.j] += a
            elif op == "add":
                adj[id(n.a)] = adj.get(id(n.a), 0.0) + a
                adj[id(n.b)] = adj.get(id(n.b), 0.0) + a
            elif op == "sub":
                adj[id(n.a)] = adj.get(id(n.a), 0.0) + a
                adj[id(n.b)] = adj.get(id(n.b), 0.0) - a
            elif op == "mul":
                adj[id(n.a)] = adj.get(id(n.a), 0.0) + a * val[id(n.b)]
                adj[id(n.b)] = adj.get(id(n.b), 0.0) + a * val[id(n.a)]
            elif op == "div":
                bv = val[id(n.b)]
                adj[id(n.a)] = adj.get(id(n.a), 0.0) + a / bv
                adj[id(n.b)] = adj.get(id(n.b), 0.0) - a * val[id(n.a)] / (bv * bv)
            elif op == "pow":
                adj[id(n.a)] = adj.get(id(n.a), 0.0) + a * n.value * val[id(n.a)] ** (n.value - 1.0)
            elif op == "log":
                adj[id(n.a)] = adj.get(id(n.a), 0.0) + a / val[id(n.a)]
            elif op == "exp":
                adj[id(n.a)] = adj.get(id(n.a), 0.0) + a * val[id(n)]
            elif op == "neg":
                adj[id(n.a)] = adj.get(id(n.a), 0.0) - a
        return g

    def str(self) -> str:
        op = self.op
        if op == "const":
            return f"{self.value:g}"
        if op == "entry":
            return f"C({self.i},{self.j})"
        sym = {"add": "+", "sub": "-", "mul": "*", "div": "/"}
        if op in sym:
            return f"({self.a.str()}{sym[op]}{self.b.str()})"
        if op == "pow":
            return f"pow({self.a.str()},{self.value:g})"
        if op in ("log", "exp"):
            return f"{op}({self.a.str()})"
        return "-" + self.a.str()

    __str__ = str


def bulk_objective():  # src/objective.cpp:238-242
    diag = Expr.entry(0, 0) + Expr.entry(1, 1) + Expr.entry(2, 2)
    off = Expr.entry(0, 1) + Expr.entry(0, 2) + Expr.entry(1, 2)
    return -((diag + 2.0 * off) / 9.0)


def shear_objective():  # :244-246
    return -((Expr.entry(3, 3) + Expr.entry(4, 4) + Expr.entry(5, 5)) / 3.0)


def npr_relaxed(beta, it):  # :248-254
    if not (0.0 < beta < 1.0):
        raise ValueError("npr-relaxed beta must lie in (0,1)")
    off = Expr.entry(0, 1) + Expr.entry(0, 2) + Expr.entry(1, 2)
    diag = Expr.entry(0, 0) + Expr.entry(1, 1) + Expr.entry(2, 2)
    return off - (beta ** float(it)) * diag


def npr_log(eta, tau, gamma):  # :256-260
    off = Expr.entry(0, 1) + Expr.entry(1, 2) + Expr.entry(2, 0)
    diag = Expr.entry(0, 0) + Expr.entry(1, 1) + Expr.entry(2, 2)
    return (1.0 + eta * off / diag).log() + tau * diag.pow(gamma)


def poisson_ratio_report(c) -> float:  # :262-268
    c = np.asarray(c).reshape(6, 6)
    c00 = (c[0, 0] + c[1, 1] + c[2, 2]) / 3.0
    c01 = (c[0, 1] + c[0, 2] + c[1, 2]) / 3.0
    den = c00 + c01
    return 0.0 if den == 0.0 else c01 / den


class ConvergeChecker:  # inc/oc.hpp:35-61
    def __init__(self, threshold=5e-4, required=3):
        self.threshold, self.required = threshold, required
        self.reset()

    def reset(self):
        self.hits, self.prev, self.has_prev = 0, 0.0, False

    def update(self, f) -> bool:
        if self.has_prev:
            rel = abs(f - self.prev) / max(abs(self.prev), 1e-12)
            self.hits = self.hits + 1 if rel < self.threshold else 0
        self.prev, self.has_prev = f, True
        return self.hits >= self.required
