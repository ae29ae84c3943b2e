"""Batched candidate evaluation: the GPU profiler + finite-field checker over a
whole population, sharded across ranks (one process per GPU).

Replaces the reference's sequential stage-4 loop (cli.py:159-195:
random_equiv_test then tune per verified pair) with one pass over every
(template, mapping, params) triple of a workload:

  1. compile   generated kernels (NVRTC, parallel threads, persistent cubin cache)
  2. FF check  candidate vs program in GF(2^31-1) on shared device-resident inputs;
               the program's FF output is computed once per workload
  3. profile   CUDA-event timing of back-to-back launches (CUDA graph) on rotating
               input sets larger than L2, in the deployment dtype
  4. argmin    per workload; across ranks one all_reduce(MIN) of the packed key
               (latency_ns << 20 | global index) and one all_gather of records

Candidates are assigned to ranks by longest-processing-time on estimated bytes,
so the shards are balanced and every rank derives the same assignment.
"""
from __future__ import annotations

import json
import math
import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from math import prod
from typing import Optional

import numpy as np

from . import _abi, ir
from .errors import SymfuseError
from .plan import PLANS, Plan, numsys_of, torch, torch_dtype

HERE = os.path.dirname(os.path.abspath(__file__))
POP_DIR = os.path.join(HERE, "populations")
WORKLOADS = ("R", "G", "A", "Q", "L")
DTYPE_BYTES = {"f32": 4, "bf16": 2, "f64": 8}


def load_population(name: str) -> dict:
    with open(os.path.join(POP_DIR, f"{name}.json")) as fh:
        return json.load(fh)


@dataclass
class Unit:
    """One candidate of a population."""

    index: int          # global index inside the workload population
    workload: str
    pair: int           # verified (template, mapping) pair index
    cand: ir.Candidate
    est_bytes: float = 0.0


def units(pop: dict) -> list:
    prog = ir.Program.from_json(pop["program"])
    out = []
    for pi, c in enumerate(pop["candidates"]):
        base = ir.from_serialized(c["key"], prog, {})
        for params in c["space"]:
            u = Unit(len(out), pop["config"], pi, base.with_params(params))
            try:
                from .tuner import cost_stats
                s = cost_stats(u.cand)
                u.est_bytes = s["bytes_loaded"] + s["bytes_stored"]
            except SymfuseError:
                u.est_bytes = 0.0
            out.append(u)
    return out


def algorithmic_bytes(pop: dict) -> int:
    """Unique HBM traffic of the workload: every input read once, every output written once."""
    es = DTYPE_BYTES[pop["dtype"]]
    prog = pop["program"]
    ins = sum(prod(t["dims"]) for t in prog["tensors"] if t["role"] == "input")
    outs = sum(prod(t["dims"]) for t in prog["tensors"] if t["name"] in prog["outputs"])
    return (ins + outs) * es


def algorithmic_flops(pop: dict) -> int:
    prog = ir.Program.from_json(pop["program"])
    sh = prog.shapes()
    fl = 0
    for o in prog.ops:
        if o.kind == "matmul":
            a = sh[o.inputs[0]]
            fl += 2 * prod(sh[o.out]) * a[-1]
        else:
            fl += prod(sh[o.out])
    return fl


def shard(us: list, rank: int, world: int) -> list:
    """LPT assignment on estimated bytes (deterministic on every rank)."""
    if world <= 1:
        return list(us)
    order = sorted(us, key=lambda u: (-u.est_bytes, u.workload, u.index))
    load = [0.0] * world
    mine = []
    for u in order:
        r = min(range(world), key=lambda k: (load[k], k))
        load[r] += u.est_bytes + 1.0
        if r == rank:
            mine.append(u)
    return mine


def precompile(cands: list, numsys_list, device: Optional[int], threads: int = 0, hints=None) -> dict:
    """Compile (or cache-hit) plans in parallel; returns {(serialized, ns): error or None}."""
    errs = {}
    threads = threads or min(32, os.cpu_count() or 8)

    def one(arg):
        c, ns = arg
        try:
            if device is None:
                Plan(c, ns, hints, None).close()
            else:
                PLANS.get(c, ns, hints, device)
            return (ir.serialize(c), ns), None
        except Exception as exc:  # recorded, not fatal: the candidate is reported as failed
            return (ir.serialize(c), ns), f"{type(exc).__name__}: {exc}"

    work = [(c, ns) for c in cands for ns in numsys_list]
    if device is not None:
        _abi.bind_device(device)
        # module loading is cheap; compile in threads, load on this thread via PLANS
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda a: Plan(a[0], a[1], hints, None).close(), work))
        for a in work:
            k, e = one(a)
            errs[k] = e
    else:
        with ThreadPoolExecutor(threads) as ex:
            for k, e in ex.map(one, work):
                errs[k] = e
    return errs


def precompile_all(quiet: bool = False, workloads=WORKLOADS, threads: int = 8) -> None:
    """Warm the on-disk cubin cache for every committed population (no GPU needed)."""
    t0 = time.time()
    n = 0
    for w in workloads:
        pop = load_population(w)
        cs = [u.cand for u in units(pop)]
        precompile(cs, [numsys_of(pop["dtype"]), _abi.FF], None, threads)
        n += 2 * len(cs)
    if not quiet:
        print(f"precompiled {n} kernels in {time.time() - t0:.1f}s")


@dataclass
class Record:
    workload: str
    index: int
    pair: int
    params: dict
    mapping: list
    ff_ok: Optional[bool] = None
    latency_us: Optional[float] = None
    error: Optional[str] = None
    plan: dict = field(default_factory=dict)
    pruned: bool = False


class WorkloadContext:
    """Device-resident state shared by every candidate of one workload."""

    def __init__(self, pop: dict, device: int, seed: int = 0, ff: bool = True):
        from .ff import ff_fill_inputs, ff_run, ff_trial_seed
        from .tuner import workspace
        self.pop = pop
        self.name = pop["config"]
        self.device = device
        self.program = ir.Program.from_json(pop["program"])
        self.numsys = numsys_of(pop["dtype"])
        self.ws = workspace(self.program, self.numsys, device)
        self.ff_inputs = None
        self.ff_expected = None
        if ff:
            seed64 = ff_trial_seed(seed, 0x5EED0000 + WORKLOADS.index(self.name) if self.name in WORKLOADS else 0, 0)
            self.ff_inputs = ff_fill_inputs(self.program, seed64, device)
            self.ff_expected = ff_run(ir.program_candidate(self.program), self.ff_inputs, device)
        self.bytes = algorithmic_bytes(pop)
        self.best_us = None  # running best latency (prunes precise timing of losers)


def evaluate_unit(ctx: WorkloadContext, u: Unit, budget_us: float = 2000.0, max_iters: int = 200,
                  ff: bool = True, prune_factor: float = 4.0) -> Record:
    from .ff import ff_equal, ff_run
    rec = Record(u.workload, u.index, u.pair, dict(u.cand.params), u.cand.mapping_list())
    try:
        if ff:
            got = ff_run(u.cand, ctx.ff_inputs, ctx.device)
            rec.ff_ok = all(ff_equal(g, e) for g, e in zip(got, ctx.ff_expected))
        plan = PLANS.get(u.cand, ctx.numsys, None, ctx.device)
        est = plan.time(ctx.ws.sets, ctx.ws.outputs, warmup=1, iters=1)
        if ctx.best_us is not None and est > prune_factor * ctx.best_us:
            rec.latency_us = est  # clearly not the winner: one launch is enough evidence
            rec.pruned = True
        else:
            iters = int(max(5, min(max_iters, budget_us / max(est, 1.0))))
            rec.latency_us = plan.time(ctx.ws.sets, ctx.ws.outputs, warmup=2, iters=iters)
            if rec.ff_ok is not False and (ctx.best_us is None or rec.latency_us < ctx.best_us):
                ctx.best_us = rec.latency_us
        rec.plan = {k: plan.info[k] for k in ("ctas", "cluster", "smem_bytes", "free_parts", "loop_parts",
                                               "kernel_name", "summary")}
    except Exception as exc:
        rec.error = f"{type(exc).__name__}: {str(exc)[:300]}"
    return rec


def argmin(records: list) -> Optional[Record]:
    ok = [r for r in records if r.error is None and r.latency_us is not None and r.ff_ok is not False]
    if not ok:
        return None
    return min(ok, key=lambda r: (r.latency_us, r.index))


def reduce_best(best: Optional[Record], dist) -> int:
    """all_reduce(MIN) of (latency_ns << 20 | index) across ranks; returns the global winner index.
    Ties on latency resolve to the smaller population index, like tune()'s lexicographic
    (score, params) tie-break (tuner.py:221-223).  NCCL over NVLink on the GPU box; the
    same call runs on gloo (CPU tensors) in the multi-process tests."""
    t = torch()
    key = (1 << 62) if best is None else (int(round(best.latency_us * 1000)) << 20) | best.index
    if dist is None:
        return -1 if best is None else best.index
    dev = f"cuda:{t.cuda.current_device()}" if dist.get_backend() == "nccl" else "cpu"
    x = t.tensor([key], dtype=t.int64, device=dev)
    dist.all_reduce(x, op=dist.ReduceOp.MIN)
    v = int(x.item())
    return -1 if v >= (1 << 62) else (v & ((1 << 20) - 1))
