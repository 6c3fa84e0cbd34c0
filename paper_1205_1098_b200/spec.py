"""Kernel specs: the `.bto` half of the drop-in boundary.

The reference describes every kernel in a tiny DSL (`.bto`, grammar in
`lang.py:17-31` of the reference) and derives from it (a) the C parameter
order of the generated function -- inputs in declaration order, outputs in
declaration order, extents sorted (`cemit.py:225-241`) -- and (b) the extent
symbols M (matrix rows) / N (matrix columns), or M alone for pure-vector
kernels (`graph.py:459-501`).  A drop-in for the generated C must agree on
both, so this module re-derives them from the same text with its own code:

* `parse_kernel(text)`  -- recursive-descent parser for the `.bto` grammar;
* `infer_shapes(spec)`  -- symbolic shape check (union-find over extents)
  that names the extents the way the reference does;
* `canonical_form(spec)`-- the spec with identifiers renamed by position, used
  to recognise which hand-written CUDA sequence implements a user's text;
* `CORPUS`              -- the kernel texts this library has CUDA for.

There is no generic code generator behind this:
a spec whose canonical form is not in the table raises UnsupportedKernelError.
"""
from __future__ import annotations

from dataclasses import dataclass, field

__all__ = [
    "KernelSyntaxError", "KernelSpecError", "UnsupportedKernelError",
    "Decl", "KernelSpec", "TypedSpec", "parse_kernel", "infer_shapes",
    "canonical_form", "CORPUS", "HOT_PATH", "load_spec", "load_typed",
    "match_corpus",
]


class KernelSyntaxError(ValueError):
    """Malformed kernel text (same role as lang.py:38-45); 1-based position."""

    def __init__(self, message: str, line: int, col: int):
        super().__init__(f"{line}:{col}: {message}")
        self.line, self.col = line, col


class KernelSpecError(ValueError):
    """Well-formed text that breaks a declaration or shape rule."""


class UnsupportedKernelError(NotImplementedError):
    """The spec is valid but no hand-written sm_100a sequence implements it."""


# ---------------------------------------------------------------------------
# AST: expressions are nested tuples so specs hash and compare by value:
#   ("var", name) | ("t", expr) | (op, left, right) with op in "+-*"

@dataclass(frozen=True)
class Decl:
    kind: str                 # "scalar" | "vector" | "matrix"
    orientation: str | None   # "row" | "column"; None for scalars

    def __str__(self) -> str:
        return self.kind if self.kind == "scalar" else f"{self.kind}({self.orientation})"


@dataclass(frozen=True)
class KernelSpec:
    name: str
    inputs: tuple[tuple[str, Decl], ...]
    outputs: tuple[tuple[str, Decl], ...]
    statements: tuple[tuple[str, tuple], ...]   # (target, expr)


_PUNCT = ":,(){}=+-*'"


def _tokens(text: str):
    line, col, i, n = 1, 1, 0, len(text)
    while i < n:
        ch = text[i]
        if ch == "\n":
            line, col, i = line + 1, 1, i + 1
        elif ch.isspace():
            col, i = col + 1, i + 1
        elif ch in _PUNCT:
            yield (ch, ch, line, col)
            col, i = col + 1, i + 1
        elif ch.isalpha() or ch == "_":
            j = i
            while j < n and (text[j].isalnum() or text[j] == "_"):
                j += 1
            yield ("id", text[i:j], line, col)
            col, i = col + (j - i), j
        else:
            raise KernelSyntaxError(f"unexpected character {ch!r}", line, col)
    yield ("eof", "", line, col)


class _Reader:
    def __init__(self, text: str):
        self.toks = list(_tokens(text))
        self.at = 0

    @property
    def tok(self):
        return self.toks[self.at]

    def take(self, kind: str, what: str | None = None):
        tok = self.tok
        if tok[0] != kind:
            found = tok[1] or "end of input"
            raise KernelSyntaxError(
                f"expected {what or repr(kind)}, found {found!r}", tok[2], tok[3])
        self.at += 1
        return tok

    def word(self, text: str):
        tok = self.take("id", repr(text))
        if tok[1] != text:
            raise KernelSyntaxError(
                f"expected {text!r}, found {tok[1]!r}", tok[2], tok[3])

    # kernel ::= NAME "in" ":" decls "out" ":" decls "{" statement* "}"
    def kernel(self) -> KernelSpec:
        name = self.take("id", "kernel name")[1]
        self.word("in")
        self.take(":")
        inputs = self.decls(until_word="out")
        self.word("out")
        self.take(":")
        outputs = self.decls(until_word=None)
        self.take("{")
        body = []
        while self.tok[0] != "}":
            target = self.take("id", "assignment target")[1]
            self.take("=")
            body.append((target, self.expr()))
        self.take("}")
        if self.tok[0] != "eof":
            raise KernelSyntaxError(
                f"trailing input after kernel body: {self.tok[1]!r}",
                self.tok[2], self.tok[3])
        return KernelSpec(name, tuple(inputs), tuple(outputs), tuple(body))

    def decls(self, until_word: str | None):
        out = [self.decl()]
        while self.tok[0] == ",":
            self.at += 1
            out.append(self.decl())
        tok = self.tok
        ok = (tok[0] == "id" and tok[1] == until_word) if until_word else tok[0] == "{"
        if not ok:
            want = repr(until_word) if until_word else "'{'"
            raise KernelSyntaxError(
                f"expected ',' or {want} after declaration", tok[2], tok[3])
        return out

    def decl(self):
        name = self.take("id", "declared name")[1]
        self.take(":")
        tok = self.take("id", "type")
        if tok[1] == "scalar":
            return name, Decl("scalar", None)
        if tok[1] not in ("vector", "matrix"):
            raise KernelSyntaxError(f"unknown type {tok[1]!r}", tok[2], tok[3])
        self.take("(")
        orient = self.take("id", "'row' or 'column'")
        if orient[1] not in ("row", "column"):
            raise KernelSyntaxError(
                f"expected 'row' or 'column', found {orient[1]!r}",
                orient[2], orient[3])
        self.take(")")
        return name, Decl(tok[1], orient[1])

    # expr ::= term (("+"|"-") term)* ; term ::= factor ("*" factor)* ;
    # factor ::= primary "'"* ; both binary levels associate left
    def expr(self):
        node = self.term()
        while self.tok[0] in "+-" and self.tok[0] != "eof":
            op = self.tok[0]
            self.at += 1
            node = (op, node, self.term())
        return node

    def term(self):
        node = self.factor()
        while self.tok[0] == "*":
            self.at += 1
            node = ("*", node, self.factor())
        return node

    def factor(self):
        tok = self.tok
        if tok[0] == "(":
            self.at += 1
            node = self.expr()
            self.take(")")
        elif tok[0] == "id":
            self.at += 1
            node = ("var", tok[1])
        else:
            raise KernelSyntaxError(
                f"expected operand, found {tok[1] or 'end of input'!r}",
                tok[2], tok[3])
        while self.tok[0] == "'":
            self.at += 1
            node = ("t", node)
        return node


def _names_in(expr) -> list[str]:
    if expr[0] == "var":
        return [expr[1]]
    if expr[0] == "t":
        return _names_in(expr[1])
    return _names_in(expr[1]) + _names_in(expr[2])


def format_expr(e) -> str:
    if e[0] == "var":
        return e[1]
    if e[0] == "t":
        inner = format_expr(e[1])
        return f"{inner}'" if e[1][0] == "var" else f"({inner})'"
    return f"({format_expr(e[1])} {e[0]} {format_expr(e[2])})"


def format_kernel(spec: KernelSpec) -> str:
    """`.bto` text of a spec (fully parenthesised): `parse_kernel(format_kernel(s)) == s`, and the
    reference's parser reads it too (lang.py:337)."""
    ins = ", ".join(f"{n} : {d}" for n, d in spec.inputs)
    outs = ", ".join(f"{n} : {d}" for n, d in spec.outputs)
    body = "  ".join(f"{t} = {format_expr(e)}" for t, e in spec.statements)
    return f"{spec.name} in: {ins} out: {outs} {{ {body} }}"


def parse_kernel(text: str) -> KernelSpec:
    """Parse `.bto` text; same accept/reject behaviour as lang.py:337-344."""
    spec = _Reader(text).kernel()
    declared: dict[str, Decl] = {}
    for name, decl in spec.inputs + spec.outputs:
        if name in declared:
            raise KernelSpecError(f"{name!r} declared twice")
        declared[name] = decl
    inputs = {n for n, _ in spec.inputs}
    known, assigned = set(inputs), set()
    for target, expr in spec.statements:
        for name in _names_in(expr):
            if name not in known:
                raise KernelSpecError(
                    f"{name!r} used before it is declared or assigned")
        if target in inputs:
            raise KernelSpecError(f"cannot assign to input {target!r}")
        if target in assigned:
            raise KernelSpecError(f"{target!r} assigned more than once")
        assigned.add(target)
        known.add(target)
    for name, _ in spec.outputs:
        if name not in assigned:
            raise KernelSpecError(f"output {name!r} is never assigned")
    return spec


# ---------------------------------------------------------------------------
# Shapes.  A value is (kind, dims): kind in scalar/col/row/mat; dims are
# union-find symbols.  Mirrors the algebra interp.py:52-83 accepts.

class _Symbols:
    def __init__(self):
        self.parent: list[int] = []

    def new(self) -> int:
        self.parent.append(len(self.parent))
        return len(self.parent) - 1

    def root(self, s: int) -> int:
        while self.parent[s] != s:
            self.parent[s] = self.parent[self.parent[s]]
            s = self.parent[s]
        return s

    def same(self, a: int, b: int) -> None:
        ra, rb = self.root(a), self.root(b)
        if ra != rb:
            self.parent[max(ra, rb)] = min(ra, rb)


@dataclass(frozen=True)
class TypedSpec:
    """A spec plus what the C ABI needs: dims per declared name, extent order."""
    spec: KernelSpec
    dims: dict = field(hash=False)            # name -> tuple of extent names
    extent_names: tuple[str, ...] = ()

    @property
    def kernel_name(self) -> str:            # cemit.py:261
        return self.spec.name.lower()

    def params(self) -> tuple[tuple[str, str], ...]:
        """(logical name, class) in the generated function's order
        (cemit.py:225-241): class is 'in'/'scalar'/'out'/'scalar_out'/'extent'."""
        out = []
        for name, decl in self.spec.inputs:
            out.append((name, "scalar" if decl.kind == "scalar" else "in"))
        for name, decl in self.spec.outputs:
            out.append((name, "scalar_out" if decl.kind == "scalar" else "out"))
        out += [(e, "extent") for e in self.extent_names]
        return tuple(out)

    def shape(self, name: str, extents: dict) -> tuple[int, ...]:
        return tuple(int(extents[d]) for d in self.dims[name])


def infer_shapes(spec: KernelSpec) -> TypedSpec:
    syms = _Symbols()
    env: dict[str, tuple[str, tuple[int, ...]]] = {}
    order: list[str] = []

    def declare(name: str, decl: Decl):
        if decl.kind == "scalar":
            env[name] = ("scalar", ())
        elif decl.kind == "vector":
            env[name] = ("col" if decl.orientation == "column" else "row",
                         (syms.new(),))
        else:
            env[name] = ("mat", (syms.new(), syms.new()))
        order.append(name)

    for name, decl in spec.inputs + spec.outputs:
        declare(name, decl)
    out_names = {n for n, _ in spec.outputs}

    def value(expr):
        tag = expr[0]
        if tag == "var":
            return env[expr[1]]
        if tag == "t":
            kind, dims = value(expr[1])
            if kind == "scalar":
                raise KernelSpecError("cannot transpose a scalar")
            if kind == "mat":
                return "mat", (dims[1], dims[0])
            return ("row" if kind == "col" else "col"), dims
        (lk, ld), (rk, rd) = value(expr[1]), value(expr[2])
        if tag in "+-":
            if lk != rk:
                raise KernelSpecError(f"cannot combine {lk} and {rk} with {tag!r}")
            for a, b in zip(ld, rd):
                syms.same(a, b)
            return lk, ld
        # product
        if lk == "scalar":
            return rk, rd
        if rk == "scalar":
            return lk, ld
        if lk == "row" and rk == "col":
            syms.same(ld[0], rd[0])
            return "scalar", ()
        if lk == "col" and rk == "row":
            return "mat", (ld[0], rd[0])
        if lk == "mat" and rk == "col":
            syms.same(ld[1], rd[0])
            return "col", (ld[0],)
        raise KernelSpecError(f"cannot multiply {lk} by {rk}")

    for target, expr in spec.statements:
        kind, dims = value(expr)
        if target in out_names:
            want_kind, want_dims = env[target]
            if (kind == "scalar") != (want_kind == "scalar") or \
                    len(dims) != len(want_dims) or \
                    (len(dims) == 1 and kind != want_kind):
                raise KernelSpecError(
                    f"{target!r} declared {want_kind}, computed {kind}")
            for a, b in zip(dims, want_dims):
                syms.same(a, b)
        else:
            env[target] = (kind, dims)

    # naming scheme of graph.py:459-501: matrix rows -> M, columns -> N;
    # vector-only kernels start at M; further classes K, L, ...
    label: dict[int, str] = {}
    has_matrix = False
    for name in order:
        kind, dims = env[name]
        if kind == "mat":
            has_matrix = True
            rows, cols = syms.root(dims[0]), syms.root(dims[1])
            if rows == cols:
                raise KernelSpecError(
                    f"dimension conflict: rows and columns of {name!r} are "
                    "forced to one extent")
            label.setdefault(rows, "M")
            label.setdefault(cols, "N")
    spare = iter(["K", "L", "P", "Q"] if has_matrix else ["M", "N", "K", "L"])
    for name in order:
        for s in env[name][1]:
            if syms.root(s) not in label:
                label[syms.root(s)] = next(spare)
    dims_by_name = {name: tuple(label[syms.root(s)] for s in env[name][1])
                    for name in order}
    extents = sorted({d for dims in dims_by_name.values() for d in dims})
    return TypedSpec(spec, dims_by_name, tuple(extents))


def canonical_form(spec: KernelSpec) -> tuple:
    """Position-renamed structure: two specs that differ only in identifier
    spelling (and kernel name) get the same key; declaration order matters
    because it fixes the C argument order."""
    rename: dict[str, str] = {}
    for idx, (name, _) in enumerate(spec.inputs):
        rename[name] = f"i{idx}"
    for idx, (name, _) in enumerate(spec.outputs):
        rename[name] = f"o{idx}"

    def walk(expr):
        if expr[0] == "var":
            return ("var", rename.setdefault(expr[1], f"t{len(rename)}"))
        if expr[0] == "t":
            return ("t", walk(expr[1]))
        return (expr[0], walk(expr[1]), walk(expr[2]))

    body = []
    for target, expr in spec.statements:
        rhs = walk(expr)
        body.append((rename.setdefault(target, f"t{len(rename)}"), rhs))
    return (tuple(str(d) for _, d in spec.inputs),
            tuple(str(d) for _, d in spec.outputs), tuple(body))


# ---------------------------------------------------------------------------
# The kernels this library implements, written in the reference's DSL.  The
# statements are the standard definitions (BTO paper table 1; the reference
# ships the same ten as kernels/*.bto) and the declaration orders are the
# reference's, because those fix the C signatures in include/bto_b200.h.

CORPUS: dict[str, str] = {
    "axpydot": "AXPYDOT in: w : vector(column), v : vector(column), "
               "u : vector(column), alpha : scalar "
               "out: z : vector(column), beta : scalar "
               "{ z = w - alpha * v  beta = z' * u }",
    "bicgk": "BICGK in: A : matrix(row), p : vector(column), r : vector(column) "
             "out: q : vector(column), s : vector(column) "
             "{ q = A * p  s = A' * r }",
    "atax": "ATAX in: A : matrix(row), x : vector(column) "
            "out: y : vector(column) { y = A' * (A * x) }",
    "gesummv": "GESUMMV in: alpha : scalar, beta : scalar, A : matrix(row), "
               "B : matrix(row), x : vector(column) out: y : vector(column) "
               "{ y = alpha * A * x + beta * B * x }",
    "gemver": "GEMVER in: A : matrix(row), u1 : vector(column), "
              "v1 : vector(column), u2 : vector(column), v2 : vector(column), "
              "alpha : scalar, beta : scalar, y : vector(column), "
              "z : vector(column) "
              "out: B : matrix(row), x : vector(column), w : vector(column) "
              "{ B = A + u1 * v1' + u2 * v2'  x = beta * B' * y + z  "
              "w = alpha * B * x }",
    # the rest of TABLE_KERNELS + BATAX
    "vadd": "VADD in: w : vector(column), y : vector(column), z : vector(column) "
            "out: x : vector(column) { x = w + y + z }",
    "waxpby": "WAXPBY in: alpha : scalar, x : vector(column), beta : scalar, "
              "y : vector(column) out: w : vector(column) "
              "{ w = alpha * x + beta * y }",
    "dgemv": "DGEMV in: alpha : scalar, A : matrix(row), x : vector(column), "
             "beta : scalar, y : vector(column) out: z : vector(column) "
             "{ z = alpha * A * x + beta * y }",
    "dgemvt": "DGEMVT in: alpha : scalar, beta : scalar, A : matrix(row), "
              "y : vector(column), z : vector(column) "
              "out: x : vector(column), w : vector(column) "
              "{ x = beta * A' * y + z  w = alpha * A * x }",
    "batax": "BATAX in: x : vector(column), beta : scalar, A : matrix(row) "
             "out: y : vector(column) { y = beta * A' * (A * x) }",
}

#: the five sequences BASELINE.json's north_star names
HOT_PATH = ("axpydot", "bicgk", "atax", "gesummv", "gemver")

_typed_cache: dict[str, TypedSpec] = {}
_by_form: dict[tuple, str] = {}


def load_spec(name: str) -> KernelSpec:
    """Corpus lookup by kernel name (the reference's corpus.load_kernel)."""
    try:
        return parse_kernel(CORPUS[name.lower()])
    except KeyError:
        raise FileNotFoundError(f"no corpus kernel {name!r}") from None


def load_typed(name: str) -> TypedSpec:
    key = name.lower()
    if key not in _typed_cache:
        _typed_cache[key] = infer_shapes(load_spec(key))
    return _typed_cache[key]


def match_corpus(spec: KernelSpec) -> str:
    """Which hand-written sequence implements `spec`?  Raises if none does."""
    if not _by_form:
        for name in CORPUS:
            _by_form[canonical_form(load_spec(name))] = name
    try:
        return _by_form[canonical_form(spec)]
    except KeyError:
        raise UnsupportedKernelError(
            f"kernel {spec.name!r}: no hand-written sm_100a sequence matches "
            "this spec (generic organism-driven CUDA emission is out of scope, "
            "SURVEY.md section 8f)") from None
