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
    cost_us: float = 0.0   # measured GPU time of its sweep work (populations/costs.json), 0 = unknown
    dep_us: float = 0.0    # measured deployment-kernel launch time (populations/costs.json), 0 = unknown


COSTS_PATH = os.path.join(POP_DIR, "costs.json")
_COSTS: Optional[dict] = None


def measured_costs() -> dict:
    """{workload: {population index: GPU microseconds}} from a B200 calibration run
    (bench.py --calibrate-out; committed as populations/costs.json)."""
    global _COSTS
    if _COSTS is None:
        try:
            with open(COSTS_PATH) as fh:
                d = json.load(fh)
            _COSTS = {w: {int(k): (float(v["cost_us"]) if isinstance(v, dict) else float(v),
                                   float(v.get("dep_us", 0.0)) if isinstance(v, dict) else 0.0)
                          for k, v in per.items()} for w, per in d["costs_us"].items()}
        except (FileNotFoundError, KeyError, ValueError):
            _COSTS = {}
    return _COSTS


def units(pop: dict) -> list:
    prog = ir.Program.from_json(pop["program"])
    cost = measured_costs().get(pop["config"], {})
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
            u.cost_us, u.dep_us = cost.get(u.index, (0.0, 0.0))
            out.append(u)
    return out


FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def hbm_peak_gbs() -> float:
    """Measured HBM copy bandwidth of this pool's B200s (MEASURED_PEAKS.json, driver-written)."""
    try:
        with open(os.path.join(os.path.dirname(HERE), "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return FALLBACK_HBM_GBS


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


def _weight(u: Unit, us: list) -> float:
    return u.cost_us if u.cost_us > 0 else u.est_bytes


def shard(us: list, rank: int, world: int) -> list:
    """LPT assignment (deterministic on every rank).  Weights are the measured
    per-candidate GPU cost of the sweep (populations/costs.json: FF run + timed
    launches, calibrated on a B200) when every unit has one, else estimated bytes
    (tuner.cost_stats): bytes miss the uncoalesced candidates that dominate A."""
    if world <= 1:
        return list(us)
    return lpt(us, world)[rank]


def lpt(us: list, world: int) -> list:
    measured = bool(us) and all(u.cost_us > 0 for u in us)
    w = (lambda u: u.cost_us) if measured else (lambda u: u.est_bytes + 1.0)
    order = sorted(us, key=lambda u: (-w(u), u.workload, u.index))
    load = [0.0] * world
    parts = [[] for _ in range(world)]
    for u in order:
        r = min(range(world), key=lambda k: (load[k], k))
        load[r] += w(u)
        parts[r].append(u)
    return parts


def predict_scaling(us: list, worlds=(2, 4, 8), refine_top: int = 3, refine_launches: int = 1000) -> dict:
    """Predicted sweep speed-up at N ranks from the measured per-candidate costs:
    LPT shards of the per-candidate work, plus the 1000-launch refine of each
    workload's global top `refine_top` charged to the rank that owns it
    (evaluate_workload(select=global_top)); speed-up = (total work) / (slowest
    rank).  Empty without a calibration."""
    if not us or not all(u.cost_us > 0 for u in us):
        return {}
    refine = {}
    if all(u.dep_us > 0 for u in us):
        byw: dict = {}
        for u in us:
            byw.setdefault(u.workload, []).append(u)
        for w, uu in byw.items():
            for u in sorted(uu, key=lambda x: (x.dep_us, x.index))[:refine_top]:
                refine[(u.workload, u.index)] = u.dep_us * refine_launches
    tot = sum(u.cost_us for u in us) + sum(refine.values())
    out = {}
    for n in worlds:
        loads = [sum(u.cost_us + refine.get((u.workload, u.index), 0.0) for u in part) for part in lpt(us, n)]
        mx = max(loads)
        out[str(n)] = {"speedup": tot / mx, "slowest_rank_ms": mx / 1e3, "total_ms": tot / 1e3,
                       "refine_ms": sum(refine.values()) / 1e3}
    return out


def calibrate_costs(ctx: "WorkloadContext", us: list, launches: int = 3) -> dict:
    """Per-candidate GPU time of its sweep work, serialised: one FF run + two
    deployment-dtype launches (screen + rotation share), each bracketed by CUDA
    events on the current stream (mean of `launches` repetitions).  Returns
    {population index: {"cost_us": ..., "dep_us": one deployment launch}}."""
    t = torch()
    dev = ctx.device
    evs = []
    for u in us:
        try:
            pf = PLANS.get(u.cand, _abi.FF, None, dev)
            pd = PLANS.get(u.cand, ctx.numsys, None, dev)
        except Exception:
            continue
        outs = ctx.ff_lanes()[0][1]
        a, b, c = (t.cuda.Event(enable_timing=True) for _ in range(3))
        pf.run(ctx.ff_inputs, outs, init_outputs=False)  # warm (module, instruction cache)
        a.record()
        for _ in range(launches):
            pf.run(ctx.ff_inputs, outs, init_outputs=False)
        b.record()
        for k in range(launches):
            pd.run(ctx.ws.sets[k % ctx.ws.rot], ctx.ws.outputs, init_outputs=False)
        c.record()
        evs.append((u.index, a, b, c))
    t.cuda.synchronize(dev)
    return {i: {"cost_us": (a.elapsed_time(b) + 2.0 * b.elapsed_time(c)) * 1000.0 / launches,
                "dep_us": b.elapsed_time(c) * 1000.0 / launches} for i, a, b, c in evs}


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
    refined: bool = False
    timing: str = ""
    variant: int = 0
    hints: dict = field(default_factory=dict)
    dep_err: Optional[float] = None   # deployment-dtype rel_err vs the fp64 program (parity gate)
    dep_ok: Optional[bool] = None
    gpu_rank: int = 0                 # rank (GPU) that evaluated the candidate


# Deployment-dtype tolerances of the parity gate (north star item 4), the same
# bars as tests/test_gpu_numerics.py: bf16 storage / fp32 accumulation 1e-2
# (output rounding 2^-8 plus bf16 MMA operands), fp32 1e-5.  rel_err is the
# reference's max|a-b| / (1 + max|b|) (interp.py:228-231).
DEP_TOL = {_abi.BF16: 1e-2, _abi.F32: 1e-5, _abi.F64: 1e-9}


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
            self.ff_out = [torch().empty_like(x) for x in self.ff_expected]
        self._ff_lanes = None
        self.bytes = algorithmic_bytes(pop)

    FF_STREAMS = int(os.environ.get("SGM_FF_STREAMS", "8"))

    def ff_lanes(self) -> list:
        """(stream, outputs) pairs for concurrent FF checks: the checks are
        verification, not timing, so candidates whose kernels leave SMs idle
        (small grids, serial loops) overlap on side streams."""
        if self._ff_lanes is None:
            t = torch()
            self._ff_lanes = [(t.cuda.Stream(device=self.device), [t.empty_like(x) for x in self.ff_expected])
                              for _ in range(self.FF_STREAMS)]
        return self._ff_lanes

    def deployment_expected(self) -> list:
        """fp64 program outputs on input set 0 of the deployment-dtype workspace
        (the rounded bf16/fp32 values, widened exactly), computed once on the
        device by the program lowered to a one-block candidate (interp.py:69-83)."""
        if getattr(self, "_dep_exp", None) is None:
            t = torch()
            ins = [x.to(t.float64) for x in self.ws.sets[0]]
            outs = [t.empty(tuple(self.program.spec(n).dims), dtype=t.float64, device=self.device)
                    for n in self.program.outputs]
            PLANS.get(ir.program_candidate(self.program), _abi.F64, None, self.device).run(ins, outs)
            del ins
            self._dep_exp = outs
            self._dep_out = [t.empty_like(o, dtype=torch_dtype(self.numsys)) for o in outs]
        return self._dep_exp

    def refresh_expected(self) -> None:
        """Re-run the program in GF(p) on the current FF inputs (into ff_expected)."""
        from .ff import ff_run
        outs = ff_run(ir.program_candidate(self.program), self.ff_inputs, self.device)
        for dst, src in zip(self.ff_expected, outs):
            dst.copy_(src)
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


def deployment_check(ctx: "WorkloadContext", plans: list) -> list:
    """The parity gate: run each plan (the exact kernel that is timed: candidate,
    number system and physical-plan hints) once in the deployment dtype on input
    set 0 and fold its rel_err against the fp64 program into a device slot.
    One host read for the whole batch.  Returns [(rel_err, ok)] (tolerance DEP_TOL)."""
    import ctypes as C
    t = torch()
    if not plans:
        return []
    exp = ctx.deployment_expected()
    outs = ctx._dep_out
    n_out = len(exp)
    slots = t.zeros((len(plans), n_out, 3), dtype=t.int64, device=ctx.device)
    s = t.cuda.current_stream(ctx.device).cuda_stream
    L = _abi.lib()
    failed = set()
    for k, pl in enumerate(plans):
        try:
            pl.run(ctx.ws.sets[0], outs, init_outputs=True)
            for j, (o, e) in enumerate(zip(outs, exp)):
                _abi.check(L.sgm_rel_err_acc(C.c_void_p(o.data_ptr()), pl.numsys, C.c_void_p(e.data_ptr()), o.numel(),
                                             C.c_void_p(s), C.c_void_p(slots[k, j].data_ptr())))
        except Exception:
            failed.add(k)
    raw = slots.cpu().numpy()
    tol = DEP_TOL[ctx.numsys]
    res = []
    for k in range(len(plans)):
        if k in failed:
            res.append((float("inf"), False))
            continue
        err = 0.0
        for j in range(n_out):
            md, mb = raw[k, j, :2].view(np.float64)
            err = max(err, float("inf") if raw[k, j, 2] else float(md / (1.0 + mb)))
        res.append((err, bool(err <= tol)))
    return res


class Timer:
    """Batched, sync-free CUDA-event profiling (libsgm sgm_timer_*)."""

    def __init__(self, capacity: int, device: int):
        import ctypes as C
        _abi.bind_device(device)
        self.cap = max(1, capacity)
        self.device = device
        h = C.c_void_p()
        _abi.check(_abi.lib().sgm_timer_create(self.cap, C.byref(h)))
        self._h = h

    def enqueue(self, slot: int, plan: Plan, input_sets, outputs, reps: int = 1, warmup: int = 1) -> None:
        import ctypes as C
        ip = _abi.ptr_array([t.data_ptr() for ins in input_sets for t in ins])
        op = _abi.ptr_array([t.data_ptr() for t in outputs])
        s = torch().cuda.current_stream(self.device).cuda_stream
        _abi.check(_abi.lib().sgm_timer_enqueue(self._h, slot, plan._h, ip, op, len(input_sets), warmup, reps,
                                                C.c_void_p(s)))

    def read(self, n: int) -> list:
        import ctypes as C
        out = (C.c_double * max(1, n))()
        _abi.check(_abi.lib().sgm_timer_read(self._h, n, out))
        return [out[k] for k in range(n)]

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().sgm_timer_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _ff_enqueue(ctx: "WorkloadContext", us: list, ks: list, recs: list, counters) -> None:
    """FF runs + on-device mismatch counts of candidates `ks`, spread over side
    streams (verification, not timing: kernels that leave SMs idle overlap), then
    joined to the current stream."""
    import ctypes as C
    t = torch()
    dev = ctx.device
    L = _abi.lib()
    main = t.cuda.current_stream(dev)
    lanes = ctx.ff_lanes()
    for sl, _ in lanes:
        sl.wait_stream(main)
    for j, k in enumerate(ks):
        sl, outs = lanes[j % len(lanes)]
        try:
            PLANS.get(us[k].cand, _abi.FF, None, dev).run(ctx.ff_inputs, outs, stream=sl.cuda_stream)
            sp = C.c_void_p(sl.cuda_stream)
            for g, e in zip(outs, ctx.ff_expected):
                _abi.check(L.sgm_compare_u32_acc(C.c_void_p(g.data_ptr()), C.c_void_p(e.data_ptr()), g.numel(),
                                                 sp, C.c_void_p(counters.data_ptr() + 8 * k)))
        except Exception as exc:
            recs[k].error = f"{type(exc).__name__}: {str(exc)[:300]}"
    for sl, _ in lanes:
        main.wait_stream(sl)


def oracle_sample(pop: dict, us: list, param_samples: int = 2, seed: int = 0) -> set:
    """Indices (into `us`) of the points the reference's stage-4 oracle would test:
    per verified (template, mapping) pair, `param_samples` parameter points drawn
    exactly as random_equiv_test draws them (rng([seed, crc32(template_key)]) shuffle
    of the divisibility-only space, interp.py:250-262; cli.py:162-170 defaults)."""
    import zlib
    chosen = set()
    for pi, c in enumerate(pop["candidates"]):
        rng = np.random.default_rng([seed, zlib.crc32(c["key"].encode())])
        pts = [dict(p) for p in c["space"]]
        rng.shuffle(pts)
        for p in pts[:param_samples]:
            chosen.add((pi, tuple(sorted(p.items()))))
    return {k for k, u in enumerate(us) if (u.pair, tuple(sorted(u.cand.params.items()))) in chosen}


def evaluate_workload(ctx: "WorkloadContext", us: list, ff=True, screen_factor: float = 2.0,
                      refine_top: int = 3, refine_launches: int = 1000, variants: int = 1, select=None) -> list:
    """Evaluate candidates of one workload with no per-candidate host synchronisation.

    Pass 1 enqueues the finite-field checks (outputs NaN-filled first, on-device
    mismatch count against the program's FF output) and, per candidate, one
    timed launch on its own input set (streams from HBM).  Pass 2 times one full
    rotation over the input sets (each launch misses L2) for the candidates
    within `screen_factor` of the pass-1 best, and gates them on parity.  Pass 3
    tunes the physical plan of the `refine_top` fastest (planner variants
    0..`variants`-1, one rotation each) and re-times each on its best variant with
    `refine_launches` launches (the paper's 1000-run protocol).
    One host read per pass.

    `select`: sharded sweeps pass global_top(dist, k): every rank offers its local
    top `refine_top` and refines only those among the global top `refine_top`, so
    the 1000-launch refine costs k per workload, not k per rank.

    `ff`: True = FF-check every candidate in pass 1 (the sweep); a set of indices
    = only those in pass 1 (e.g. oracle_sample: the reference's stage-4 oracle
    points), and every contender of pass 2 not yet checked is FF-checked (its FF
    kernel compiled then) before it may win; False = none."""
    import ctypes as C
    t = torch()
    dev = ctx.device
    n = len(us)
    recs = [Record(u.workload, u.index, u.pair, dict(u.cand.params), u.cand.mapping_list()) for u in us]
    if n == 0:
        if select is not None:
            select([])  # collective: every rank takes part
        return recs
    counters = t.zeros(n, dtype=t.int64, device=dev)
    stream = C.c_void_p(t.cuda.current_stream(dev).cuda_stream)
    rot = ctx.ws.rot
    plans = [None] * n
    ff_first = list(range(n)) if ff is True else sorted(ff) if ff else []
    if ff_first:
        _ff_enqueue(ctx, us, ff_first, recs, counters)
    timer = Timer(n, dev)
    for k, u in enumerate(us):
        rec = recs[k]
        if rec.error is not None:
            continue
        try:
            plan = plans[k] = PLANS.get(u.cand, ctx.numsys, None, dev)
            # screening: one launch on its own input set (streams from HBM), no warm-up;
            # it only ranks candidates for the rotation pass
            timer.enqueue(k, plan, [ctx.ws.sets[k % rot]], ctx.ws.outputs, reps=1, warmup=0)
            rec.plan = {x: plan.info[x] for x in ("ctas", "cluster", "smem_bytes", "free_parts", "loop_parts",
                                                  "kernel_name", "summary")}
        except Exception as exc:  # recorded, the sweep goes on (failures are reported)
            rec.error = f"{type(exc).__name__}: {str(exc)[:300]}"
    lat = timer.read(n)
    mism = counters.cpu().tolist()
    ff_set = set(ff_first)
    timer.close()
    for k, rec in enumerate(recs):
        if rec.error is None:
            rec.latency_us = lat[k] if lat[k] >= 0 else None
            rec.ff_ok = (mism[k] == 0) if k in ff_set else None
            rec.timing = "screen"
    # kernel watchdog (a bounded wait timed out): the candidate is a "run: timeout"
    # record, like the reference's run errors (interp.py:278-281)
    for k, u in enumerate(us):
        if recs[k].error is not None:
            continue
        for ns_ in ((_abi.FF, ctx.numsys) if k in ff_set else (ctx.numsys,)):
            if PLANS.get(u.cand, ns_, None, dev).watchdog():
                recs[k].error = f"run: timeout (kernel watchdog, {_abi.NUMSYS_NAMES.get(ns_, ns_)})"
                recs[k].latency_us = None
                recs[k].ff_ok = False
                break

    def live():
        return [k for k, r in enumerate(recs) if r.error is None and r.latency_us is not None and r.ff_ok is not False]

    ok = live()
    if not ok and select is not None:
        select([])  # collective: every rank takes part
    if ok:
        best = min(recs[k].latency_us for k in ok)
        sel = [k for k in ok if recs[k].latency_us <= screen_factor * best]
        timer = Timer(len(sel), dev)
        for j, k in enumerate(sel):
            timer.enqueue(j, plans[k], ctx.ws.sets, ctx.ws.outputs, reps=1)
        lat2 = timer.read(len(sel))
        timer.close()
        for j, k in enumerate(sel):
            recs[k].latency_us = lat2[j]
            recs[k].timing = "rotation"
        # parity gate: every contender's deployment-dtype kernel (the one just timed)
        # against the fp64 program; a candidate that fails cannot win
        for k, (err, good) in zip(sel, deployment_check(ctx, [plans[k] for k in sel])):
            recs[k].dep_err, recs[k].dep_ok = err, good
        sel = [k for k in sel if recs[k].dep_ok]
        late = [k for k in sel if recs[k].ff_ok is None and ff is not False]
        if late:  # contenders the first pass did not FF-check: compile their FF kernels, check
            precompile([us[k].cand for k in late], [_abi.FF], None)
            _ff_enqueue(ctx, us, late, recs, counters)
            mism = counters.cpu().tolist()
            for k in late:
                if recs[k].error is None:
                    recs[k].ff_ok = mism[k] == 0
                    if PLANS.get(us[k].cand, _abi.FF, None, dev).watchdog():
                        recs[k].error, recs[k].ff_ok = "run: timeout (kernel watchdog, ff)", False
            sel = [k for k in sel if recs[k].ff_ok and recs[k].error is None]
        top = sorted(sel, key=lambda k: (recs[k].latency_us, recs[k].index))[:refine_top]
        if select is not None:  # sharded sweep: only this rank's share of the GLOBAL top candidates
            keep = select([(recs[k].latency_us, recs[k].index) for k in top])
            top = [k for k in top if recs[k].index in keep]
        # physical-plan tuning: planner variants of the top candidates (the FF check of
        # the candidate covers every variant: each is the same block graph, re-split)
        best_plan = {k: (recs[k].latency_us, 0, plans[k]) for k in top}
        vp = []
        for k in top:
            for v in range(1, variants):
                try:
                    vp.append((k, v, PLANS.get(us[k].cand, ctx.numsys, {"variant": v}, dev)))
                except Exception:
                    pass
        if vp:
            timer = Timer(len(vp), dev)
            for j, (k, v, pl) in enumerate(vp):
                timer.enqueue(j, pl, ctx.ws.sets, ctx.ws.outputs, reps=1)
            latv = timer.read(len(vp))
            timer.close()
            for j, (k, v, pl) in enumerate(vp):
                if 0 < latv[j] < best_plan[k][0]:
                    best_plan[k] = (latv[j], v, pl)
        swapped = [k for k in top if best_plan[k][1] != 0]
        for k, (err, good) in zip(swapped, deployment_check(ctx, [best_plan[k][2] for k in swapped])):
            if not good:  # a physical variant that breaks numerics falls back to the checked plan
                best_plan[k] = (recs[k].latency_us, 0, plans[k])
        timer = Timer(len(top), dev)
        for j, k in enumerate(top):
            timer.enqueue(j, best_plan[k][2], ctx.ws.sets, ctx.ws.outputs, reps=max(1, -(-refine_launches // rot)))
        lat3 = timer.read(len(top))
        timer.close()
        for j, k in enumerate(top):
            recs[k].latency_us = lat3[j]
            recs[k].timing = "refined"
            recs[k].refined = True
            recs[k].variant = best_plan[k][1]
            pl = best_plan[k][2]
            recs[k].plan = {x: pl.info[x] for x in ("ctas", "cluster", "smem_bytes", "free_parts", "loop_parts",
                                                    "kernel_name", "summary")}
    return recs


VARIANT_HINTS = [{}] + [{"variant": v} for v in range(1, 6)] + [{"one_cta": 1}] + \
    [{"one_cta": 1, "variant": v} for v in range(1, 4)] + \
    [{"max_gsplit": g} for g in (1, 2, 4)] + [{"max_gsplit": g, "one_cta": 1} for g in (1, 2, 4)] + \
    [{"max_gsplit": g, "max_cluster": 1} for g in (1, 2, 4)] + [{"max_cluster": 1}, {"max_cluster": 2}] + \
    [{"one_cta": 1, "slot_kb": 16}, {"slot_kb": 16}] + \
    [{"small_plain": 1}, {"small_plain": 1, "one_cta": 1}]


def precompile_variants(units: list, numsys: int, threads: int = 0, extra: Optional[dict] = None) -> None:
    """Compile every planner variant of `units` into the cubin cache in parallel
    (compile-only plans, no device), so tune_physical's plan builds are cache hits."""
    threads = threads or min(32, os.cpu_count() or 8)

    def one(arg):
        u, h = arg
        try:
            Plan(u.cand, numsys, h or None, None).close()
        except Exception:
            pass

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, [(u, {**h, **(extra or {})}) for u in units for h in VARIANT_HINTS]))


def tune_physical(ctx: "WorkloadContext", u: Unit, launches: int = 1000, extra: Optional[dict] = None) -> tuple:
    """Physical-plan tuning of one candidate: time each planner variant (other scored
    splits, one-CTA-per-SM rings) over one rotation, re-time the fastest with
    `launches` launches.  Returns (latency_us, hints, plan).  The candidate's FF
    verdict covers every variant: the block graph is the same, re-split."""
    dev = ctx.device
    plans = []
    for h in VARIANT_HINTS:
        h = {**h, **(extra or {})}
        try:
            plans.append((h, PLANS.get(u.cand, ctx.numsys, h or None, dev)))
        except Exception:
            pass
    seen, uniq = set(), []
    for h, p in plans:  # variants that generate the same kernel are timed once
        if p.kernel_name not in seen:
            seen.add(p.kernel_name)
            uniq.append((h, p))
    timer = Timer(len(uniq), dev)
    for j, (h, p) in enumerate(uniq):
        timer.enqueue(j, p, ctx.ws.sets, ctx.ws.outputs, reps=2)
    lat = timer.read(len(uniq))
    timer.close()
    j = min(range(len(uniq)), key=lambda k: lat[k] if lat[k] > 0 else 1e30)
    h, p = uniq[j]
    timer = Timer(1, dev)
    timer.enqueue(0, p, ctx.ws.sets, ctx.ws.outputs, reps=max(1, -(-launches // ctx.ws.rot)))
    best = timer.read(1)[0]
    timer.close()
    return best, h, p


def global_top(dist, k: int):
    """select= callback of evaluate_workload for a sharded sweep: all_gather every
    rank's local (latency, index) contenders and keep the global k fastest (ties
    to the smaller index).  Every rank must call it the same number of times."""
    def select(local: list) -> set:
        if dist is None:
            return {i for _, i in sorted(local)[:k]}
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, list(local))
        return {i for _, i in sorted(x for p in parts for x in p)[:k]}
    return select


def ff_check_plan(ctx: "WorkloadContext", cand: ir.Candidate, hints: Optional[dict]) -> bool:
    """Finite-field check of one physical variant: the candidate compiled with the
    same planner hints (splits, gsplit/cluster caps) in GF(p), bit-exact against
    the program's FF output."""
    from .ff import ff_equal
    t = torch()
    outs = [t.empty_like(e) for e in ctx.ff_expected]
    PLANS.get(cand, _abi.FF, hints or None, ctx.device).run(ctx.ff_inputs, outs)
    return all(ff_equal(g, e) for g, e in zip(outs, ctx.ff_expected))


def graph_latency(ctx: "WorkloadContext", plan: Plan, launches: int = 1000, pdl: bool = True) -> float:
    """Mean microseconds per launch over `launches` back-to-back launches (CUDA
    graphs of one rotation of input sets, every launch misses L2), with
    programmatic dependent launch on or off for the capture."""
    _abi.bind_device(ctx.device)
    _abi.check(_abi.lib().sgm_set_pdl(1 if pdl else 0))
    try:
        timer = Timer(1, ctx.device)
        timer.enqueue(0, plan, ctx.ws.sets, ctx.ws.outputs, reps=max(1, -(-launches // ctx.ws.rot)))
        us = timer.read(1)[0]
        timer.close()
    finally:
        _abi.check(_abi.lib().sgm_set_pdl(1))
    return us


def isolated_latency(ctx: "WorkloadContext", plan: Plan, launches: int = 50) -> dict:
    """Single-launch latency with nothing to overlap: before every launch a
    256 MB read (a reduction over a buffer twice the L2) leaves L2 holding only
    clean lines of other data, and the launch is bracketed by its own CUDA
    events on the launching stream, so launch processing, prologue and tail are
    all inside the number (no CUDA graph; the next launch cannot start early).
    Returns mean/median/min microseconds."""
    t = torch()
    flush = t.zeros(64 << 20, dtype=t.float32, device=ctx.device)
    evs = [(t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)) for _ in range(launches)]
    rot = ctx.ws.rot
    sink = []
    for k, (a, b) in enumerate(evs):
        sink.append(flush.sum())
        a.record()
        plan.run(ctx.ws.sets[k % rot], ctx.ws.outputs, init_outputs=False)
        b.record()
    t.cuda.synchronize(ctx.device)
    us = sorted(a.elapsed_time(b) * 1000.0 for a, b in evs)
    return {"mean_us": sum(us) / len(us), "median_us": us[len(us) // 2], "min_us": us[0], "launches": launches,
            "method": "per-launch CUDA events, 256 MB read-only L2 flush between launches, no graph"}


def report(pop: dict, records: list, hbm_gbs: Optional[float] = None) -> dict:
    """The sweep in the reference's report format (cli.py:133-146 records, one per
    verified (template, mapping) pair), each record extended with the GPU evidence
    of its best parameter point ("b200": latency_us, hbm_gbs, roofline_frac,
    ff_ok, dep_err, gpu_rank, kernel) and every evaluated point ("b200_points")."""
    hbm_gbs = hbm_gbs or hbm_peak_gbs()
    byts = algorithmic_bytes(pop)
    by_pair: dict = {}
    for r in records:
        by_pair.setdefault(r.pair, []).append(r)
    cands = []
    for pi, c in enumerate(pop["candidates"]):
        rs = sorted(by_pair.get(pi, []), key=lambda r: r.index)
        ok = [r for r in rs if r.error is None and r.latency_us and r.ff_ok is not False and r.dep_ok is not False]
        best = min(ok, key=lambda r: (r.latency_us, r.index)) if ok else None
        rec = {"template_id": c["template_id"], "mapping": c["mapping"], "verified": True,
               "verify": {"status": "equivalent", "exhausted": False},
               "oracle": {"ok": all(r.ff_ok for r in rs) if rs else None, "kind": "finite field GF(2^31-1), bit-exact",
                          "checked": sum(1 for r in rs if r.ff_ok is not None)},
               "best": None if best is None else {"params": best.params, "score": best.latency_us * 1e-6},
               "equivalence_checked": bool(rs) and all(r.ff_ok for r in rs)}
        if best is not None:
            gbs = byts / (best.latency_us * 1e-6) / 1e9
            rec["b200"] = {"latency_us": best.latency_us, "hbm_gbs": gbs, "roofline_frac": gbs / hbm_gbs,
                           "ff_ok": best.ff_ok, "dep_err": best.dep_err, "gpu_rank": best.gpu_rank,
                           "timing": best.timing, "kernel": (best.plan or {}).get("kernel_name"),
                           "plan": (best.plan or {}).get("summary"), "dtype": pop["dtype"]}
        rec["b200_points"] = [{"params": r.params, "latency_us": r.latency_us, "ff_ok": r.ff_ok, "error": r.error,
                               "gpu_rank": r.gpu_rank} for r in rs]
        cands.append(rec)
    return {"workload": pop["program"]["name"], "config": pop["config"], "dtype": pop["dtype"],
            "algorithmic_bytes": byts, "hbm_peak_gbs": hbm_gbs, "candidates": cands,
            "templates": sorted({c["template_id"] for c in pop["candidates"]})}


def write_report(rep: dict, path: str) -> None:
    """Deterministic JSON like the reference's write_report (cli.py:199-202)."""
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(rep, fh, indent=2, sort_keys=True, default=str)
        fh.write("\n")


def export_dots(pop: dict, rep: dict, outdir: str) -> list:
    """One DOT file per verified template (cli.py:205-223, the reference's to_dot
    when it is importable) with the GPU evidence of its pairs appended as comments."""
    os.makedirs(outdir, exist_ok=True)
    try:
        from symfuse.graph import deserialize, to_dot
        from symfuse.graph import Program as _RP  # noqa: F401
        have_ref = True
    except ImportError:
        have_ref = False
    written = []
    for tid in sorted({c["template_id"] for c in pop["candidates"]}):
        c0 = next(c for c in pop["candidates"] if c["template_id"] == tid)
        body = f"// template {tid}: {c0['key']}\n"
        if have_ref:
            try:
                from . import workloads as W
                from symfuse.workloads import lower
                spec, _ = W.spec_of(pop["config"])
                g, _, _ = deserialize(c0["key"], lower(spec))
                body = to_dot(g) + "\n"
            except Exception:
                pass
        path = os.path.join(outdir, f"template_{tid:03d}.dot")
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(body)
            for rc in rep["candidates"]:
                if rc["template_id"] == tid and rc.get("b200"):
                    b = rc["b200"]
                    fh.write(f"// b200 {','.join(rc['mapping'])} params={rc['best']['params']} "
                             f"latency_us={b['latency_us']:.2f} hbm_gbs={b['hbm_gbs']:.0f} "
                             f"roofline_frac={b['roofline_frac']:.3f} ff_ok={b['ff_ok']} kernel={b['kernel']}\n")
        written.append(path)
    return written


def argmin(records: list) -> Optional[Record]:
    """Fastest candidate that passed the FF check and, among those, the
    deployment-dtype parity gate (records the gate never saw rank after)."""
    ok = [r for r in records if r.error is None and r.latency_us is not None and r.ff_ok is not False
          and r.dep_ok is not False]
    if not ok:
        return None
    return min(ok, key=lambda r: (r.dep_ok is not True, r.latency_us, r.index))


def reduce_best(best: Optional[Record], dist) -> int:
    """all_reduce(MIN) of (latency_ns << 20 | index) across ranks; returns the global winner index.
    Ties on latency resolve to the smaller population index, like tune()'s lexicographic
    (score, params) tie-break (tuner.py:221-223).  NCCL over NVLink on the GPU box; the
    same call runs on gloo (CPU tensors) in the multi-process tests."""
    return reduce_best_many([best], dist)[0]


def reduce_best_many(bests: list, dist) -> list:
    """reduce_best for several workloads in ONE all_reduce (one sync per sweep step)."""
    t = torch()
    keys = [(1 << 62) if b is None else (int(round(b.latency_us * 1000)) << 20) | b.index for b in bests]
    if dist is None:
        return [-1 if b is None else b.index for b in bests]
    dev = f"cuda:{t.cuda.current_device()}" if dist.get_backend() == "nccl" else "cpu"
    x = t.tensor(keys, dtype=t.int64, device=dev)
    dist.all_reduce(x, op=dist.ReduceOp.MIN)
    return [-1 if v >= (1 << 62) else (v & ((1 << 20) - 1)) for v in x.tolist()]
