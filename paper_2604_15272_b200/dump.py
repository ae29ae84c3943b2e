"""tile_dump support for run_concrete (interp.py:132,210-211).

The reference fills `tile_dump[coords] = {node idx: tile}` after each grid
block: every node's value at the end of the block (loop-body nodes hold their
last iteration, accumulators their sum, epilogue loaders their last loop tile;
savers are not in the environment).  test_integration.py:72-85 reads it.

On the B200 the dump is produced by ONE extra kernel, generated from a dump
candidate: the same block graph with one extra saver per non-saver node, each
writing its tile into a dump tensor whose dim 0 is chunked by every grid dim in
grid order (the reference's nested saver chunking, interp.py:116-125), so block
`coords` owns rows [rank(coords) * t0, (rank(coords) + 1) * t0).  The dump
kernel runs with a physical plan that keeps every tile whole inside one CTA's
schedule (no loop split, no gsplit or cluster reductions), so each saved tile
is the block-level value, not a partial.  Outputs come from the candidate's
normal kernel.
"""
from __future__ import annotations

import itertools
from math import prod

import numpy as np

from . import ir

# plan hints of the dump kernel: whole tiles per CTA, loop iterations in order
DUMP_HINTS = {"no_loop_split": 1, "max_gsplit": 1, "max_cluster": 1, "no_tma": 1}


def dump_candidate(cand: ir.Candidate) -> tuple:
    """(dump candidate, {node idx: (dump tensor name, tile shape)})."""
    prog, blk, p = cand.program, cand.block, cand.params
    shapes = ir.concrete_shapes(cand)
    G = prod(p[g] for g in blk.grid)
    tensors = list(prog.tensors)
    outputs = list(prog.outputs)
    nodes = list(blk.nodes)
    mapping = set(cand.mapping)
    table = {}
    for n in blk.nodes:
        if n.kind == ir.OUTPUT:
            continue
        t = tuple(shapes[n.idx])
        name = f"__dump{n.idx}"
        dims = (t[0] * G,) + tuple(t[1:])
        tensors.append(ir.Tensor(name, dims, "output"))
        outputs.append(name)
        nodes.append(ir.Node(len(nodes), ir.OUTPUT, (n.idx,), name))
        if dims[0] > 1:
            for g in blk.grid:
                mapping.add((name, 0, g))
        table[n.idx] = (name, t)
    dprog = ir.Program(prog.name, tuple(tensors), prog.ops, tuple(outputs))
    dblk = ir.Block(blk.grid, blk.loop, tuple(nodes))
    return ir.Candidate(dprog, dblk, frozenset(mapping), dict(p)), table


def run_with_dump(concrete, inputs, dtype, tile_dump: dict, device=None) -> dict:
    from .interp import _execute
    from .plan import numsys_of
    cand = ir.candidate_of(concrete)
    ns = numsys_of(dtype)
    outs = _execute(cand, inputs, ns, device, None, check_missing=False)
    dc, table = dump_candidate(cand)
    res = _execute(dc, inputs, ns, device, DUMP_HINTS, check_missing=False)
    grid = cand.block.grid
    for r, coords in enumerate(itertools.product(*[range(cand.params[g]) for g in grid])):
        env = {}
        for idx, (name, t) in table.items():
            arr = res[name]
            tile = arr[r * t[0]:(r + 1) * t[0]]
            env[idx] = np.array(tile) if isinstance(tile, np.ndarray) else tile.clone()
        tile_dump[coords] = env
    return outs
