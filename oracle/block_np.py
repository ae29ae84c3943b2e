"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference interpreter.

Follows symfuse interp.py (the reference's hot path):
  run_program       interp.py:69-83    program ops on whole tensors
  run_concrete      interp.py:128-212  grid loop -> for-loop body -> epilogue -> savers
  tile bounds       interp.py:90-125   nested contiguous chunking, grid dims in grid
                                        order then the loop; unit extents never split
  body nodes        graph.py:242-254   accumulators and their ancestors
  F64 op table      interp.py:36-66    (stable two-branch silu)
  rel_err           interp.py:228-231
with a pluggable arithmetic: F64Arith (the reference's numpy semantics) or
ff_np.FFArith (finite field).  Candidates are given in the reference's
canonical serialization (graph.py:519-528) plus a program dict, so nothing here
imports symfuse or the product package.
"""
from __future__ import annotations

import itertools
import json
from fractions import Fraction

import numpy as np


class ShapeMismatch(Exception):
    """ShapeError of the reference (tile/region or divisibility)."""


class WriteConflict(Exception):
    """WriteConflictError of the reference."""


class F64Arith:
    name = "f64"

    def __call__(self, kind, args, axis=None, const_=None):
        x = args[0]
        if kind == "exp":
            return np.exp(x)
        if kind == "silu":
            out = np.empty_like(x)
            nonneg = x >= 0
            out[nonneg] = x[nonneg] / (1.0 + np.exp(-x[nonneg]))
            e = np.exp(x[~nonneg])
            out[~nonneg] = x[~nonneg] * e / (1.0 + e)
            return out
        if kind == "square":
            return x * x
        if kind == "sqrt":
            return np.sqrt(x)
        if kind == "scale":
            return float(const_) * x
        if kind == "sum":
            return x.sum(axis=axis, keepdims=True)
        if kind == "matmul":
            return np.matmul(x, args[1])
        if kind == "div":
            return x / args[1]
        if kind == "mul":
            return x * args[1]
        if kind == "add":
            return x + args[1]
        raise ValueError(f"unknown op kind {kind}")

    def accum(self, acc, val):
        return acc + val

    def zeros(self, like):
        return np.zeros_like(like)

    def cast(self, arr):
        return np.asarray(arr, dtype=np.float64)

    def fill(self, dims):
        return np.full(dims, np.nan)


def load_program(d: dict) -> dict:
    """Program dict: {name, tensors:[{name,dims,role}], ops:[{kind,inputs,out,axis?,const?}], outputs}."""
    return d


def program_inputs(prog: dict) -> list:
    return [t["name"] for t in prog["tensors"] if t["role"] == "input"]


def _dims(prog: dict, name: str) -> tuple:
    for t in prog["tensors"]:
        if t["name"] == name:
            return tuple(t["dims"])
    raise KeyError(name)


def run_program(prog: dict, inputs: dict, arith=None) -> dict:
    arith = arith or F64Arith()
    env = {}
    for name in program_inputs(prog):
        arr = arith.cast(inputs[name])
        if arr.shape != _dims(prog, name):
            raise ShapeMismatch(f"{name}: got {arr.shape}")
        env[name] = arr
    for op in prog["ops"]:
        c = Fraction(*op["const"]) if op.get("const") is not None else None
        env[op["out"]] = arith(op["kind"], [env[k] for k in op["inputs"]], op.get("axis"), c)
    return {name: env[name] for name in prog["outputs"]}


def _parse(key: str):
    d = json.loads(key)
    nodes = d["nodes"]
    on = set()
    for s in d.get("mapping", []):
        t, dim, q = s.rsplit(".", 2)
        on.add((t, int(dim), q))
    return d["grid"], d["loop"], nodes, on


def _body(nodes) -> set:
    seen = set()
    todo = [n["id"] for n in nodes if n["op"] == "accum"]
    while todo:
        k = todo.pop()
        if k in seen:
            continue
        seen.add(k)
        todo.extend(nodes[k]["in"])
    return seen


def _chunk(extent: int, splits) -> slice:
    lo, width = 0, extent
    for index, count in splits:
        if width % count:
            raise ShapeMismatch(f"extent {width} not divisible by {count}")
        width //= count
        lo += index * width
    return slice(lo, lo + width)


def _region(dims, var, pdims, on, sizes, where) -> tuple:
    """Per-dim nested chunking (interp.py:90-125); `pdims` in nesting order."""
    out = []
    for d, extent in enumerate(dims):
        cuts = [(where[q], sizes[q]) for q in pdims if extent > 1 and (var, d, q) in on]
        out.append(_chunk(extent, cuts))
    return tuple(out)


def run_concrete(prog: dict, key: str, params: dict, inputs: dict, arith=None, tile_dump=None) -> dict:
    """Execute the candidate `key` (graph.serialize()/template_key() text with a
    mapping) at `params`, block by block like the reference."""
    arith = arith or F64Arith()
    grid, loop, nodes, on = _parse(key)
    ins = program_inputs(prog)
    data = {}
    for name in ins:
        arr = arith.cast(inputs[name])
        if arr.shape != _dims(prog, name):
            raise ShapeMismatch(f"{name}: got {arr.shape}")
        data[name] = arr
    result = {name: arith.fill(_dims(prog, name)) for name in prog["outputs"]}
    owner = {name: np.zeros(_dims(prog, name), dtype=bool) for name in prog["outputs"]}
    body = _body(nodes)
    n_loop = params[loop]
    sizes = dict(params)

    def loader(n, where):
        var = n["tensor"]
        return data[var][_region(_dims(prog, var), var, list(grid) + [loop], on, sizes, where)]

    def compute(n, env):
        c = Fraction(*n["const"]) if "const" in n else None
        return arith(n["op"], [env[k] for k in n["in"]], n.get("axis"), c)

    for coords in itertools.product(*[range(params[q]) for q in grid]):
        where = dict(zip(grid, coords))
        env, acc = {}, {}
        for j in range(n_loop):
            where[loop] = j
            for n in nodes:
                if n["id"] not in body:
                    continue
                if n["op"] == "input":
                    env[n["id"]] = loader(n, where)
                elif n["op"] == "accum":
                    v = env[n["in"][0]]
                    acc[n["id"]] = arith.accum(acc[n["id"]] if n["id"] in acc else arith.zeros(v), v)
                    env[n["id"]] = acc[n["id"]]
                else:
                    env[n["id"]] = compute(n, env)
        where[loop] = max(n_loop - 1, 0)   # epilogue loaders see the last tile
        for n in nodes:
            if n["id"] in body:
                continue
            if n["op"] == "input":
                env[n["id"]] = loader(n, where)
            elif n["op"] == "output":
                name = n["tensor"]
                var = name if name not in ins else f"{name}:out"
                reg = _region(_dims(prog, name), var, list(grid), on, sizes, where)
                tile = env[n["in"][0]]
                if result[name][reg].shape != tile.shape:
                    raise ShapeMismatch(f"saver {name}: tile {tile.shape} vs region {result[name][reg].shape}")
                if owner[name][reg].any():
                    raise WriteConflict(f"{name}: block {coords} overwrote cells")
                result[name][reg] = tile
                owner[name][reg] = True
            else:
                env[n["id"]] = compute(n, env)
        if tile_dump is not None:
            tile_dump[coords] = {k: np.array(v) for k, v in env.items()}
    return result


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape or not np.isfinite(a).all():
        return float("inf")
    return float(np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b))))
