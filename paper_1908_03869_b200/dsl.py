"""Expression templates for drift/diffusion definitions (drop-in for
``sdebatch.dsl``, /root/reference/pkg/src/sdebatch/dsl.py).

Same language (dsl.py:1-27): numbers, ``t`` / ``N`` / ``i``, indexed ``y[.]``
``p[.]`` ``n[.]``, ``+ - * / ^`` (``^`` right-associative and tighter than
unary minus), ``sin cos tan exp ln sqrt abs`` and ``sum(j, body)`` over
j = 0..N-1; the same AST classes, error types, validation diagnostics,
printer and model-file format.

What differs is evaluation.  The reference walks the AST with numpy
(dsl.py:441-571); here an expression is compiled -- libsdeb200 parses the
canonical text :func:`to_source` prints, generates CUDA device functions and
builds them with NVRTC for sm_100a (include/sdeb200.h, ``sdb_model_*``) -- and
:func:`evaluate` runs on the GPU.  There is no numpy interpreter.
"""

from __future__ import annotations

import os
import re
from dataclasses import dataclass
from typing import Union

import numpy as np

__all__ = [
    "DslError", "ParseError", "ValidationError", "DomainError",
    "Num", "Var", "Index", "Neg", "BinOp", "Call", "Sum", "ExprAst",
    "EvalContext", "Diagnostic", "ModelText",
    "parse", "validate", "evaluate", "to_source", "parse_model_text", "load_model_file",
    "FUNCTIONS",
]

FUNCTIONS = ("sin", "cos", "tan", "exp", "ln", "sqrt", "abs")   # dsl.py:45-53
RESERVED = ("t", "N", "i")                                      # dsl.py:55
INDEXABLE = ("y", "p", "n")


class DslError(Exception):
    """Base class of expression-language errors (dsl.py:59-60)."""


class ParseError(DslError):
    def __init__(self, message: str, line: int, col: int):
        super().__init__("line %d, column %d: %s" % (line, col, message))
        self.line = line
        self.col = col


class ValidationError(DslError):
    def __init__(self, diagnostics):
        super().__init__("; ".join(str(d) for d in diagnostics))
        self.diagnostics = list(diagnostics)


class DomainError(DslError):
    """Evaluation error: an index out of range, or (strict mode) a non-finite
    value such as ln of a non-positive number or a division by zero."""

    def __init__(self, message: str, pos: tuple[int, int]):
        super().__init__("line %d, column %d: %s" % (pos[0], pos[1], message))
        self.pos = pos


# ---------------------------------------------------------------------------
# AST (dsl.py:85-135: same classes and fields)

@dataclass(frozen=True)
class Num:
    value: float
    pos: tuple[int, int] = (0, 0)


@dataclass(frozen=True)
class Var:
    name: str
    pos: tuple[int, int] = (0, 0)


@dataclass(frozen=True)
class Index:
    base: str
    index: "ExprAst"
    pos: tuple[int, int] = (0, 0)


@dataclass(frozen=True)
class Neg:
    operand: "ExprAst"
    pos: tuple[int, int] = (0, 0)


@dataclass(frozen=True)
class BinOp:
    op: str
    left: "ExprAst"
    right: "ExprAst"
    pos: tuple[int, int] = (0, 0)


@dataclass(frozen=True)
class Call:
    func: str
    arg: "ExprAst"
    pos: tuple[int, int] = (0, 0)


@dataclass(frozen=True)
class Sum:
    var: str
    body: "ExprAst"
    pos: tuple[int, int] = (0, 0)


ExprAst = Union[Num, Var, Index, Neg, BinOp, Call, Sum]


# ---------------------------------------------------------------------------
# lexer + Pratt parser

_LEX = re.compile(r"""
    (?P<ws>\s+)
  | (?P<num>(?:[0-9]+\.[0-9]*|\.[0-9]+|[0-9]+)(?:[eE][+-]?[0-9]+)?)
  | (?P<name>[A-Za-z_]\w*)
  | (?P<op>[-+*/^()\[\],])
""", re.VERBOSE)


def _lex(text: str):
    """[(kind, text, line, col)] ending with ('end', '', line, col)."""
    out = []
    line, line_start, k = 1, 0, 0
    while k < len(text):
        m = _LEX.match(text, k)
        col = k - line_start + 1
        if m is None:
            raise ParseError("unexpected character %r" % text[k], line, col)
        kind = m.lastgroup
        if kind != "ws":
            out.append((kind, m.group(), line, col))
        else:
            for off, ch in enumerate(m.group()):
                if ch == "\n":
                    line += 1
                    line_start = k + off + 1
        k = m.end()
    out.append(("end", "", line, len(text) - line_start + 1))
    return out


_INFIX = {"+": 10, "-": 10, "*": 20, "/": 20}


class _Pratt:
    def __init__(self, text: str):
        self.toks = _lex(text)
        self.k = 0

    def peek(self):
        return self.toks[self.k]

    def take(self):
        tok = self.toks[self.k]
        self.k += 1
        return tok

    def at_op(self, text: str) -> bool:
        kind, value, _, _ = self.peek()
        return kind == "op" and value == text

    def need(self, text: str, context: str):
        kind, value, line, col = self.peek()
        if kind == "op" and value == text:
            return self.take()
        raise ParseError("expected %r %s, found %r" % (text, context, value or "end of input"),
                         line, col)

    def expression(self, floor: int = 0) -> ExprAst:
        left = self.prefix()
        while True:
            kind, value, line, col = self.peek()
            bp = _INFIX.get(value) if kind == "op" else None
            if bp is None or bp <= floor:
                return left
            self.take()
            left = BinOp(value, left, self.expression(bp), (line, col))

    def prefix(self) -> ExprAst:
        # unary minus applies to a whole power expression: -2^2 == -(2^2)
        if self.at_op("-"):
            _, _, line, col = self.take()
            return Neg(self.prefix(), (line, col))
        base = self.primary()
        if self.at_op("^"):
            _, _, line, col = self.take()
            return BinOp("^", base, self.prefix(), (line, col))  # right-assoc, may be -x
        return base

    def primary(self) -> ExprAst:
        kind, value, line, col = self.take()
        if kind == "num":
            return Num(float(value), (line, col))
        if kind == "op" and value == "(":
            inner = self.expression()
            self.need(")", "to close parenthesis")
            return inner
        if kind != "name":
            self.k -= 1
            raise ParseError("expected a number, name or parenthesised expression, found %r"
                             % (value or "end of input"), line, col)
        if self.at_op("["):
            if value not in INDEXABLE:
                raise ParseError("only y, p and n can be indexed, not %r" % value, line, col)
            self.take()
            idx = self.expression()
            self.need("]", "to close index")
            return Index(value, idx, (line, col))
        if self.at_op("("):
            self.take()
            if value == "sum":
                ikind, ivalue, iline, icol = self.peek()
                if ikind != "name":
                    raise ParseError("sum(index, body) expects an index name first", iline, icol)
                self.take()
                self.need(",", "between sum index and body")
                body = self.expression()
                self.need(")", "to close sum")
                return Sum(ivalue, body, (line, col))
            if value not in FUNCTIONS:
                raise ParseError("unknown function %r" % value, line, col)
            arg = self.expression()
            self.need(")", "to close function call")
            return Call(value, arg, (line, col))
        return Var(value, (line, col))


def parse(source: str) -> ExprAst:
    """Expression text -> AST, or :class:`ParseError` (dsl.py:282-289)."""
    p = _Pratt(source)
    node = p.expression()
    kind, value, line, col = p.peek()
    if kind != "end":
        raise ParseError("unexpected trailing input %r" % value, line, col)
    return node


# ---------------------------------------------------------------------------
# validation (dsl.py:353-408)

@dataclass(frozen=True)
class Diagnostic:
    message: str
    line: int
    col: int

    def __str__(self):
        return "line %d, column %d: %s" % (self.line, self.col, self.message)


def _const_index(node):
    """Integer value of a variable-free index expression, else None."""
    if isinstance(node, Num):
        return int(node.value) if float(node.value).is_integer() else None
    if isinstance(node, Neg):
        v = _const_index(node.operand)
        return None if v is None else -v
    if isinstance(node, BinOp) and node.op in "+-*":
        a, b = _const_index(node.left), _const_index(node.right)
        if a is None or b is None:
            return None
        return a + b if node.op == "+" else a - b if node.op == "-" else a * b
    return None


def _index_diagnostics(node, scope, out):
    if isinstance(node, Num):
        if not float(node.value).is_integer():
            out.append(Diagnostic("non-integer constant in index expression", *node.pos))
    elif isinstance(node, Var):
        if node.name == "t":
            out.append(Diagnostic("t cannot appear in an index expression", *node.pos))
        elif node.name not in ("N", "i") and node.name not in scope:
            out.append(Diagnostic("unknown variable %r" % node.name, *node.pos))
    elif isinstance(node, Neg):
        _index_diagnostics(node.operand, scope, out)
    elif isinstance(node, BinOp):
        if node.op not in "+-*":
            out.append(Diagnostic("operator %r not allowed in index expressions" % node.op,
                                  *node.pos))
        _index_diagnostics(node.left, scope, out)
        _index_diagnostics(node.right, scope, out)
    else:
        out.append(Diagnostic("index expressions must be integer arithmetic", *node.pos))


def validate(expr: ExprAst, nequat: int, nparams: int, nnoise: int,
             role: str = "diffusion") -> list[Diagnostic]:
    """Diagnostics of ``expr`` against the model dimensions; [] = valid.
    ``role="drift"`` also rejects the noise vector."""
    if role not in ("drift", "diffusion"):
        raise ValueError("role must be 'drift' or 'diffusion'")
    dims = {"y": nequat, "p": nparams, "n": nnoise}
    out: list[Diagnostic] = []
    stack = [(expr, frozenset())]
    while stack:
        node, scope = stack.pop()
        if isinstance(node, Num):
            continue
        if isinstance(node, Var):
            if node.name not in RESERVED and node.name not in scope:
                out.append(Diagnostic("unknown variable %r" % node.name, *node.pos))
        elif isinstance(node, Index):
            if node.base == "n" and role == "drift":
                out.append(Diagnostic("noise n[...] cannot appear in a drift expression",
                                      *node.pos))
            _index_diagnostics(node.index, scope, out)
            value = _const_index(node.index)
            if value is not None and not 0 <= value < dims[node.base]:
                out.append(Diagnostic("index %d out of range for %s (length %d)"
                                      % (value, node.base, dims[node.base]), *node.pos))
        elif isinstance(node, Neg):
            stack.append((node.operand, scope))
        elif isinstance(node, BinOp):
            stack.append((node.right, scope))
            stack.append((node.left, scope))
        elif isinstance(node, Call):
            stack.append((node.arg, scope))
        elif isinstance(node, Sum):
            if node.var in scope:
                out.append(Diagnostic("nested sums reuse index %r" % node.var, *node.pos))
            elif node.var in RESERVED:
                out.append(Diagnostic("sum index %r shadows a reserved name" % node.var,
                                      *node.pos))
            stack.append((node.body, scope | {node.var}))
        else:
            raise TypeError("unknown AST node %r" % (node,))
    out.sort(key=lambda d: (d.line, d.col))
    return out


# ---------------------------------------------------------------------------
# printer (dsl.py:577-614): canonical text, round-trips through parse()

def _rank(node) -> int:
    if isinstance(node, BinOp):
        return {"+": 1, "-": 1, "*": 2, "/": 2, "^": 4}[node.op]
    return 3 if isinstance(node, Neg) else 5


def to_source(node: ExprAst) -> str:
    """AST -> expression text."""
    if isinstance(node, Num):
        return repr(float(node.value))
    if isinstance(node, Var):
        return node.name
    if isinstance(node, Index):
        return "%s[%s]" % (node.base, to_source(node.index))
    if isinstance(node, Call):
        return "%s(%s)" % (node.func, to_source(node.arg))
    if isinstance(node, Sum):
        return "sum(%s, %s)" % (node.var, to_source(node.body))
    if isinstance(node, Neg):
        inner = to_source(node.operand)
        return "-(%s)" % inner if _rank(node.operand) < 3 else "-" + inner
    if isinstance(node, BinOp):
        r = _rank(node)
        lt, rt = to_source(node.left), to_source(node.right)
        if node.op == "^":
            # right-associative: an equal-rank right operand needs no guard
            left_paren = _rank(node.left) <= r
            right_paren = _rank(node.right) < r
        else:
            left_paren = _rank(node.left) < r
            right_paren = _rank(node.right) <= r
        if left_paren:
            lt = "(%s)" % lt
        if right_paren:
            rt = "(%s)" % rt
        return "%s %s %s" % (lt, node.op, rt)
    raise TypeError("unknown AST node %r" % (node,))


def strip_positions(node):
    """The AST with every ``pos`` reset (structural comparison)."""
    if isinstance(node, Num):
        return Num(float(node.value))
    if isinstance(node, Var):
        return Var(node.name)
    if isinstance(node, Index):
        return Index(node.base, strip_positions(node.index))
    if isinstance(node, Neg):
        return Neg(strip_positions(node.operand))
    if isinstance(node, BinOp):
        return BinOp(node.op, strip_positions(node.left), strip_positions(node.right))
    if isinstance(node, Call):
        return Call(node.func, strip_positions(node.arg))
    if isinstance(node, Sum):
        return Sum(node.var, strip_positions(node.body))
    raise TypeError("unknown AST node %r" % (node,))


def as_ast(expr):
    """Our AST for ``expr``: text, one of our nodes, or a foreign AST with a
    module-level to_source (e.g. the reference's sdebatch.dsl nodes)."""
    if isinstance(expr, str):
        return parse(expr)
    if isinstance(expr, (Num, Var, Index, Neg, BinOp, Call, Sum)):
        return expr
    mod = getattr(expr.__class__, "__module__", "")
    if mod.endswith("dsl"):
        import importlib
        return parse(importlib.import_module(mod).to_source(expr))
    raise TypeError("not an expression: %r" % (expr,))


# ---------------------------------------------------------------------------
# evaluation on the device

@dataclass
class EvalContext:
    """Values an expression is evaluated against (dsl.py:416-433): ``y`` /
    ``p`` / ``n`` may carry leading batch dimensions; ``i=None`` evaluates
    every equation index and adds a trailing axis of length N."""

    t: float
    N: int
    y: np.ndarray
    p: np.ndarray
    n: np.ndarray | None = None
    i: int | None = None


def evaluate(expr: ExprAst, ctx: EvalContext, strict: bool = True):
    """Evaluate ``expr`` in double precision on the GPU (replaces the numpy
    interpreter, dsl.py:554-571).  Index errors raise :class:`DomainError`;
    in strict mode so does a non-finite result from finite inputs (ln of a
    non-positive value, division by zero); ``strict=False`` returns them."""
    from . import program
    return program.evaluate_expression(as_ast(expr), ctx, strict)


# ---------------------------------------------------------------------------
# model file format (dsl.py:620-680)

@dataclass
class ModelText:
    nequat: int
    nparams: int
    nnoise: int
    drift: str
    diffusion: str
    name: str = "model"


_HEADER = re.compile(r"(nequat|nparams|nnoise)\s*=\s*([+-]?\d+)")
_TEMPLATE = re.compile(r"(drift|diffusion)\s*:\s*(.+)")


def parse_model_text(text: str, name: str = "model") -> ModelText:
    """``nequat=`` / ``nparams=`` / ``nnoise=`` headers in any order, then
    ``drift:`` and ``diffusion:`` lines; ``#`` comments and blank lines."""
    found: dict[str, object] = {}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        m = _HEADER.fullmatch(line)
        if m:
            key, value = m.group(1), int(m.group(2))
            if key in found:
                raise ParseError("duplicate header %r" % key, lineno, 1)
        else:
            m = _TEMPLATE.fullmatch(line)
            if not m:
                raise ParseError("unrecognised model file line %r" % line, lineno, 1)
            key, value = m.group(1), m.group(2)
            if key in found:
                raise ParseError("duplicate %r template" % key, lineno, 1)
        found[key] = value
    for key in ("nequat", "nparams", "nnoise"):
        if key not in found:
            raise ParseError("missing header %r" % key, 1, 1)
    for key in ("drift", "diffusion"):
        if key not in found:
            raise ParseError("missing %r template" % key, 1, 1)
    return ModelText(nequat=found["nequat"], nparams=found["nparams"],
                     nnoise=found["nnoise"], drift=found["drift"],
                     diffusion=found["diffusion"], name=name)


def load_model_file(path) -> ModelText:
    with open(path, "r", encoding="utf-8") as handle:
        text = handle.read()
    return parse_model_text(text, name=os.path.splitext(os.path.basename(str(path)))[0])
