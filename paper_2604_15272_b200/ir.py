"""Candidate representation consumed by the B200 backend.

The backend accepts the reference's own objects (`symfuse.graph.ConcreteGraph`,
`SymbolicGraph` + mapping dict) by duck typing, and an equivalent plain form
(`Candidate`) that can be rebuilt from the reference's canonical serialization
(`symfuse.graph.serialize`, graph.py:519-562) without importing `symfuse`.  The
GPU box carries no reference install, so tests, smoke() and bench.py use the
plain form built from committed population files.

Shape rules restate the reference's:
  * loader tile  = data extent / prod(sizes of the pdims mapped to it)
    (graph.py:353-360 dim_expr, evaluated exactly; NonIntegerError otherwise)
  * op shapes    = _sym_op_shape (graph.py:375-399)
  * saver target = extent / prod(grid sizes mapped to it) (graph.py:363-371)
"""
from __future__ import annotations

import json
import zlib
from dataclasses import dataclass, field
from fractions import Fraction
from math import prod
from typing import Iterable, Optional

from .errors import ConstraintError, DivisibilityError, NonIntegerError, ShapeError

INPUT, OUTPUT, ACCUM, MATMUL, SUM, SCALE = "input", "output", "accum", "matmul", "sum", "scale"
UNARY = ("exp", "silu", "square", "sqrt")
BINARY = ("div", "mul", "add")
KIND_CODE = {
    "input": 0, "output": 1, "matmul": 2, "exp": 3, "silu": 4, "square": 5, "sqrt": 6,
    "div": 7, "mul": 8, "add": 9, "sum": 10, "accum": 11, "scale": 12,
}


@dataclass(frozen=True)
class Tensor:
    name: str
    dims: tuple
    role: str  # "input" | "intermediate" | "output"


@dataclass(frozen=True)
class Op:
    kind: str
    inputs: tuple
    out: str
    axis: Optional[int] = None
    const: Optional[Fraction] = None


@dataclass(frozen=True)
class Program:
    name: str
    tensors: tuple
    ops: tuple
    outputs: tuple

    @property
    def inputs(self) -> tuple:
        return tuple(t.name for t in self.tensors if t.role == "input")

    def spec(self, name: str) -> Tensor:
        for t in self.tensors:
            if t.name == name:
                return t
        raise KeyError(name)

    def saver_var(self, name: str) -> str:
        # graph.py:41-47: qualified only when an output aliases an input
        return name if name not in self.inputs else f"{name}:out"

    def to_json(self) -> dict:
        return {
            "name": self.name,
            "tensors": [{"name": t.name, "dims": list(t.dims), "role": t.role} for t in self.tensors],
            "ops": [
                {"kind": o.kind, "inputs": list(o.inputs), "out": o.out,
                 **({"axis": o.axis} if o.axis is not None else {}),
                 **({"const": [o.const.numerator, o.const.denominator]} if o.const is not None else {})}
                for o in self.ops
            ],
            "outputs": list(self.outputs),
        }

    @staticmethod
    def from_json(d: dict) -> "Program":
        return Program(
            name=d["name"],
            tensors=tuple(Tensor(t["name"], tuple(t["dims"]), t["role"]) for t in d["tensors"]),
            ops=tuple(
                Op(o["kind"], tuple(o["inputs"]), o["out"], o.get("axis"),
                   Fraction(*o["const"]) if "const" in o else None)
                for o in d["ops"]
            ),
            outputs=tuple(d["outputs"]),
        )

    def shapes(self) -> dict:
        """Whole-tensor shapes of every value (numpy semantics)."""
        sh = {t.name: tuple(t.dims) for t in self.tensors if t.role == "input"}
        for o in self.ops:
            sh[o.out] = op_shape(o.kind, [sh[n] for n in o.inputs], o.axis)
        return sh


@dataclass(frozen=True)
class Node:
    idx: int
    kind: str
    inputs: tuple = ()
    tensor: Optional[str] = None
    axis: Optional[int] = None
    const: Optional[Fraction] = None


@dataclass(frozen=True)
class Block:
    grid: tuple  # grid dim names, e.g. ("x",)
    loop: str    # loop dim name, "i"
    nodes: tuple

    @property
    def pdims(self) -> tuple:
        return tuple(self.grid) + (self.loop,)

    def body(self) -> set:
        """Accumulators and their ancestors (graph.py:242-254)."""
        live: set = set()
        stack = [n.idx for n in self.nodes if n.kind == ACCUM]
        while stack:
            k = stack.pop()
            if k not in live:
                live.add(k)
                stack.extend(self.nodes[k].inputs)
        return live


@dataclass
class Candidate:
    """(template, mapping, params): one unit of evaluation."""

    program: Program
    block: Block
    mapping: frozenset  # {(var, dim, pdim)} of mapping bits that are 1
    params: dict = field(default_factory=dict)

    def on(self, var: str, dim: int, pdim: str) -> bool:
        return (var, dim, pdim) in self.mapping

    def with_params(self, params: dict) -> "Candidate":
        return Candidate(self.program, self.block, self.mapping, dict(params))

    def mapping_list(self) -> list:
        return sorted(f"{t}.{d}.{p}" for t, d, p in self.mapping)


# ---------------------------------------------------------------------------
# shape algebra (numpy semantics on concrete tiles)


def op_shape(kind: str, ins: list, axis=None) -> tuple:
    if kind in UNARY or kind in (SCALE, ACCUM, OUTPUT):
        return tuple(ins[0])
    if kind in BINARY:
        a, b = ins
        n = max(len(a), len(b))
        a = (1,) * (n - len(a)) + tuple(a)
        b = (1,) * (n - len(b)) + tuple(b)
        out = []
        for x, y in zip(a, b):
            if x == y or y == 1:
                out.append(x)
            elif x == 1:
                out.append(y)
            else:
                raise ValueError(f"operands could not be broadcast together: {a} {b}")
        return tuple(out)
    if kind == MATMUL:
        a, b = ins
        if len(a) < 2 or len(b) < 2:
            raise ValueError("matmul operands need rank >= 2")
        if a[-1] != b[-2]:
            raise ValueError(f"matmul: mismatch in its core dimension {a} @ {b}")
        batch = op_shape("add", [a[:-2], b[:-2]]) if len(a) > 2 or len(b) > 2 else ()
        return tuple(batch) + (a[-2], b[-1])
    if kind == SUM:
        (a,) = ins
        if axis is None or not 0 <= axis < len(a):
            raise ValueError(f"bad sum axis {axis} for {a}")
        return tuple(a[:axis]) + (1,) + tuple(a[axis + 1:])
    raise ShapeError(f"unknown op kind {kind}")


def _split(extent: int, factors: Iterable[int]) -> int:
    total = prod(factors)
    if extent % total:
        raise NonIntegerError(f"{extent}/{total} is not an integer")
    return extent // total


def concrete_shapes(c: Candidate) -> dict:
    """Per-node tile shapes for c.params (graph.py:339-350 + evaluate_int)."""
    prog, blk, p = c.program, c.block, c.params
    shapes: dict = {}
    for n in blk.nodes:
        if n.kind == INPUT:
            spec = prog.spec(n.tensor)
            shapes[n.idx] = tuple(
                1 if size == 1 else _split(size, [p[q] for q in blk.pdims if c.on(n.tensor, d, q)])
                for d, size in enumerate(spec.dims)
            )
        elif n.kind == OUTPUT:
            shapes[n.idx] = shapes[n.inputs[0]]
        else:
            shapes[n.idx] = _sym_shape(n, [shapes[k] for k in n.inputs])
    return shapes


def _sym_shape(n: Node, ins: list) -> tuple:
    # graph.py:375-399: broadcasting resolves a literal-1 side to the other side
    if n.kind in UNARY or n.kind in (SCALE, ACCUM):
        return ins[0]
    if n.kind in BINARY:
        a, b = ins
        if len(a) != len(b):
            raise ShapeError(f"node {n.idx}: rank mismatch")
        return tuple(y if x == 1 else x for x, y in zip(a, b))
    if n.kind == MATMUL:
        a, b = ins
        if len(a) < 2 or len(a) != len(b):
            raise ShapeError(f"node {n.idx}: matmul needs equal ranks >= 2")
        return tuple(a[:-1]) + (b[-1],)
    if n.kind == SUM:
        (a,) = ins
        if n.axis is None or not 0 <= n.axis < len(a):
            raise ShapeError(f"node {n.idx}: bad sum axis")
        return tuple(a[: n.axis]) + (1,) + tuple(a[n.axis + 1:])
    raise ShapeError(f"node {n.idx}: unknown kind {n.kind}")


def saver_target(c: Candidate, node: Node) -> tuple:
    spec = c.program.spec(node.tensor)
    var = c.program.saver_var(node.tensor)
    return tuple(
        1 if size == 1 else _split(size, [c.params[g] for g in c.block.grid if c.on(var, d, g)])
        for d, size in enumerate(spec.dims)
    )


def mapping_vars(program: Program, block: Block) -> list:
    """Flatten order of graph.py:264-285 (loaders then savers, dims, pdims)."""
    out = []
    for n in block.nodes:
        if n.kind == INPUT:
            var, pn = n.tensor, block.pdims
        elif n.kind == OUTPUT:
            var, pn = program.saver_var(n.tensor), block.grid
        else:
            continue
        for d, size in enumerate(program.spec(n.tensor).dims):
            if size == 1:
                continue
            for q in pn:
                out.append((var, d, q))
    return out


def check_linear_constraints(c: Candidate) -> bool:
    """The two linear families + saver coverage of mapping_satisfies
    (graph.py:293-320).  Recorded equalities live in the generator's
    ConstraintStore and are only checkable with the reference objects."""
    vars_ = mapping_vars(c.program, c.block)
    per_tp: dict = {}
    per_td: dict = {}
    for v in vars_:
        bit = 1 if v in c.mapping else 0
        per_tp[(v[0], v[2])] = per_tp.get((v[0], v[2]), 0) + bit
        if v[2] != c.block.loop:
            per_td[(v[0], v[1])] = per_td.get((v[0], v[1]), 0) + bit
    if any(s > 1 for s in per_tp.values()) or any(s > 1 for s in per_td.values()):
        return False
    for n in c.block.nodes:
        if n.kind != OUTPUT:
            continue
        var = c.program.saver_var(n.tensor)
        rank = len(c.program.spec(n.tensor).dims)
        for g in c.block.grid:
            if sum(1 for d in range(rank) if (var, d, g) in c.mapping) != 1:
                return False
    return True


def validate(c: Candidate, strict_mapping: bool = True) -> dict:
    """instantiate() checks (graph.py:414-441) on the plain form; returns shapes."""
    for q, v in c.params.items():
        if v < 1 or v & (v - 1):
            raise DivisibilityError(f"size of {q} must be a positive power of two, got {v}")
    for q in c.block.pdims:
        if q not in c.params:
            raise ConstraintError(f"missing size for parallel dim {q}")
    if strict_mapping and not check_linear_constraints(c):
        raise ConstraintError("mapping violates the graph's constraints")
    shapes = concrete_shapes(c)
    for idx, dims in shapes.items():
        if any(x < 1 for x in dims):
            raise DivisibilityError(f"node {idx}: shape {dims} not positive")
    for n in c.block.nodes:
        if n.kind == OUTPUT and shapes[n.idx] != saver_target(c, n):
            raise DivisibilityError(f"saver {n.tensor}: tile {shapes[n.idx]} != target {saver_target(c, n)}")
    return shapes


# ---------------------------------------------------------------------------
# canonical keys (graph.py:447-528), restated so candidate ids and the oracle's
# RNG streams (interp.py:234-235, 259, 272) match the reference byte for byte


def _payload(n: Node) -> tuple:
    return (
        n.kind,
        n.tensor or "",
        -1 if n.axis is None else n.axis,
        "" if n.const is None else f"{n.const.numerator}/{n.const.denominator}",
    )


def canonical_nodes(block: Block) -> list:
    sig: dict = {}        # surviving node -> structural signature
    rep: dict = {}        # node -> surviving representative
    first: dict = {}      # signature -> representative
    level: dict = {}
    for n in block.nodes:
        kids = tuple(rep[k] for k in n.inputs)
        s = (_payload(n), tuple(sig[k] for k in kids))
        if s in first:
            rep[n.idx] = first[s]
            continue
        rep[n.idx] = first[s] = n.idx
        sig[n.idx] = s
        level[n.idx] = 1 + max((level[k] for k in kids), default=0)
    order = sorted(first.values(), key=lambda k: (level[k], sig[k]))
    new_id = {old: i for i, old in enumerate(order)}
    out = []
    for old in order:
        n = block.nodes[old]
        out.append(Node(new_id[old], n.kind, tuple(new_id[rep[k]] for k in n.inputs), n.tensor, n.axis, n.const))
    return out


def _structure(program: Program, block: Block) -> dict:
    nodes = []
    for n in canonical_nodes(block):
        d = {"id": n.idx, "op": n.kind, "in": list(n.inputs)}
        if n.tensor is not None:
            d["tensor"] = n.tensor
        if n.axis is not None:
            d["axis"] = n.axis
        if n.const is not None:
            d["const"] = [n.const.numerator, n.const.denominator]
        nodes.append(d)
    return {"version": 1, "workload": program.name, "grid": list(block.grid), "loop": block.loop, "nodes": nodes}


def template_key(c: Candidate, with_mapping: bool = True) -> str:
    payload = _structure(c.program, c.block)
    if with_mapping:
        payload["mapping"] = c.mapping_list()
    return json.dumps(payload, sort_keys=True, separators=(",", ":"))


def serialize(c: Candidate) -> str:
    payload = _structure(c.program, c.block)
    payload["mapping"] = c.mapping_list()
    payload["params"] = {k: c.params[k] for k in sorted(c.params)}
    return json.dumps(payload, sort_keys=True, separators=(",", ":"))


def candidate_id(c: Candidate) -> int:
    return zlib.crc32(template_key(c).encode())


def from_serialized(text: str, program: Program, params: Optional[dict] = None) -> Candidate:
    """Rebuild a candidate from graph.serialize()/template_key() output."""
    d = json.loads(text)
    nodes = tuple(
        Node(x["id"], x["op"], tuple(x["in"]), x.get("tensor"), x.get("axis"),
             Fraction(*x["const"]) if "const" in x else None)
        for x in d["nodes"]
    )
    block = Block(tuple(d["grid"]), d["loop"], nodes)
    on = set()
    for s in d.get("mapping", []):
        t, dim, q = s.rsplit(".", 2)
        on.add((t, int(dim), q))
    return Candidate(program, block, frozenset(on), dict(params if params is not None else d.get("params", {})))


# ---------------------------------------------------------------------------
# adapters for the reference's objects (duck-typed; no symfuse import needed)


def program_of(obj) -> Program:
    if isinstance(obj, Program):
        return obj
    return Program(
        name=obj.name,
        tensors=tuple(Tensor(t.name, tuple(t.dims), t.role) for t in obj.tensors),
        ops=tuple(Op(o.kind, tuple(o.inputs), o.out, o.axis, o.const) for o in obj.ops),
        outputs=tuple(obj.outputs),
    )


def block_of(obj) -> Block:
    if isinstance(obj, Block):
        return obj
    return Block(
        grid=tuple(p.name for p in obj.grid),
        loop=obj.loop.name,
        nodes=tuple(Node(n.idx, n.kind, tuple(n.inputs), n.tensor, n.axis, n.const) for n in obj.nodes),
    )


def mapping_of(mapping) -> frozenset:
    if isinstance(mapping, frozenset):
        return mapping
    out = set()
    for v, bit in mapping.items():
        if bit:
            if isinstance(v, tuple):
                out.add(v)
            else:
                out.add((v.tensor, v.dim, v.pdim))
    return frozenset(out)


def candidate_of(graph, mapping=None, params=None) -> Candidate:
    """Accept a Candidate, a symfuse ConcreteGraph, or (SymbolicGraph, mapping[, params])."""
    if isinstance(graph, Candidate):
        return graph if params is None else graph.with_params(params)
    if hasattr(graph, "graph") and hasattr(graph, "params") and hasattr(graph, "mapping"):
        g = graph.graph  # ConcreteGraph (graph.py:406-411)
        return Candidate(program_of(g.program), block_of(g.block), mapping_of(graph.mapping), dict(graph.params))
    return Candidate(program_of(graph.program), block_of(graph.block), mapping_of(mapping or {}), dict(params or {}))


def program_candidate(program: Program) -> Candidate:
    """The program itself as a one-block candidate (grid 1, loop 1, whole tiles):
    run_program (interp.py:69-83) executes through the same code generator."""
    nodes = []
    where: dict = {}
    for name in program.inputs:
        where[name] = len(nodes)
        nodes.append(Node(len(nodes), INPUT, (), name))
    for o in program.ops:
        where[o.out] = len(nodes)
        nodes.append(Node(len(nodes), o.kind, tuple(where[x] for x in o.inputs), None, o.axis, o.const))
    for name in program.outputs:
        nodes.append(Node(len(nodes), OUTPUT, (where[name],), name))
    return Candidate(program, Block(("x",), "i", tuple(nodes)), frozenset(), {"x": 1, "i": 1})
