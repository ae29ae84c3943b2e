"""Parallel CPU search + verification around the UNCHANGED reference.

`run_pipeline(spec, flags, until="verify")` (cli.py:69-157) runs template
generation, mapping enumeration and e-graph verification one after the other
in one Python thread; on QK-attention at full scale that is ~60 s, the Amdahl
term of an end-to-end optimisation run.  Here the same reference functions run
concurrently on host processes, with results identical to the sequential run:

* generation (generator.py:471-496) stays ONE depth-first search per workload,
  exactly the reference's `Generator.run`: its abstract-pruning checker
  (verifier/verify.py:51-110) saturates an e-graph incrementally under a node
  budget, so which partial graphs it prunes depends on the order of earlier
  queries; splitting the DFS across workers changes the emitted template set
  (measured on LoRA).  The workloads' searches run concurrently instead, one
  process each.
* mapping enumeration + verification (cli.py:118-149) are independent per
  template; each emitted template is streamed to a worker pool while the
  search is still running and verified there (enumerate_mappings, then
  `equivalent` per output with the pipeline's SaturationLimits).
* results come back in template order, so the report (templates, candidate
  records, verified pairs) is the sequential run_pipeline's report; only the
  wall-clock "timings" differ (tests/test_search.py).

Everything here forks: start a `SearchRun` before CUDA is initialised.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import threading
import time
from typing import Optional

_WCACHE: dict = {}  # per worker process: workload -> (program, targets, axioms, limits)


def _flags(max_ops):
    from symfuse.cli import PipelineFlags
    return PipelineFlags(until="verify", max_ops=max_ops)


def _context(name: str):
    """(spec, program, flags, k, axioms, limits) of one workload, cached per process."""
    c = _WCACHE.get(name)
    if c is None:
        from symfuse.verifier import build_axioms, encode_program
        from symfuse.verifier.engine import SaturationLimits
        from symfuse.workloads import lower
        from . import workloads as W
        spec, max_ops = W.spec_of(name)
        flags = _flags(max_ops)
        program = lower(spec)
        k = flags.grid_dims or spec.defaults.get("grid_dims", 1)
        axioms = build_axioms(k)
        limits = SaturationLimits(max_nodes=flags.sat_nodes, max_iters=flags.sat_iters,
                                  timeout_s=flags.sat_timeout_s)
        c = _WCACHE[name] = (spec, program, flags, k, axioms, limits, encode_program(program), max_ops)
    return c


def _generate_proc(name: str, q) -> None:
    """One workload's template generation: the reference's Generator.run, with
    every emitted template also sent to the parent as it appears."""
    import symfuse.generator as RG
    from symfuse.graph import template_key
    spec, program, flags, k, axioms, limits, _, max_ops = _context(name)
    t0 = time.perf_counter()
    cfg = RG.SearchConfig(max_block_ops=max_ops or spec.defaults.get("max_ops", 10), num_grid_dims=k,
                          operator_whitelist=flags.whitelist, node_budget=flags.node_budget,
                          time_budget_s=flags.time_budget_s,
                          concrete_imap=flags.ablate.get("imap") == "concrete",
                          concrete_fmap=flags.ablate.get("fmap") == "concrete",
                          concrete_omap=flags.ablate.get("omap") == "concrete")
    gen = RG.Generator(program, cfg, axioms=axioms)
    emit = gen._emit

    def streaming_emit(state):
        n0 = len(gen.out)
        emit(state)
        for j in range(n0, len(gen.out)):
            q.put(("template", name, j, gen.out[j], template_key(gen.out[j])))

    gen._emit = streaming_emit
    res = gen.run()
    st = res.stats
    q.put(("done", name, {"explored_nodes": st.explored, "pruned_by_dim": st.pruned_dim,
                          "pruned_by_expr": st.pruned_expr, "dedup_hits": st.dedup_hits,
                          "templates_emitted": st.emitted, "budget_exhausted": st.budget_exhausted},
           time.perf_counter() - t0))


def _verify_template(name: str, tid: int, g):
    """Pool task: mappings of one template + e-graph verification (cli.py:118-149)."""
    from symfuse.graph import template_key
    from symfuse.mappings import enumerate_mappings
    from symfuse.verifier import encode_graph, equivalent
    _, program, _, _, axioms, limits, targets, _ = _context(name)
    t0 = time.perf_counter()
    maps = list(enumerate_mappings(g))
    t_map = time.perf_counter() - t0
    out = []
    for mapping in maps:
        terms = encode_graph(g, mapping)
        statuses = [equivalent(terms[n], targets[n], axioms, limits=limits) for n in program.outputs]
        ok = all(s.equivalent for s in statuses)
        rec = {"template_id": tid,
               "mapping": sorted(f"{v.tensor}.{v.dim}.{v.pdim}" for v, bit in mapping.items() if bit),
               "verified": ok,
               "verify": {"status": "equivalent" if ok else "not_proven",
                          "exhausted": any(s.resource_exhausted for s in statuses)},
               "oracle": None, "best": None, "equivalence_checked": False}
        out.append((rec, template_key(g, mapping) if ok else None))
    return name, tid, out, t_map, time.perf_counter() - t0 - t_map


class SearchRun:
    """Concurrent searches of several workloads: one generator process per
    workload plus a shared verification pool.  `result(name)` blocks until that
    workload's report (the run_pipeline(until="verify") report, plus the
    template graph objects under "graphs") is complete."""

    def __init__(self, names, workers: Optional[int] = None):
        from . import workloads as W
        if W.import_reference() is None:
            raise RuntimeError("the reference (symfuse) is not importable (baseline/_ref)")
        self.names = list(names)
        self.workers = workers or os.cpu_count() or 4
        ctx = mp.get_context("fork")
        self.t0 = time.perf_counter()
        self.q = ctx.Queue()
        self.pool = ctx.Pool(max(1, self.workers - 1))
        self.procs = {n: ctx.Process(target=_generate_proc, args=(n, self.q), daemon=True) for n in self.names}
        self.state = {n: {"graphs": {}, "keys": {}, "recs": {}, "pending": 0, "done": None, "t_map": 0.0,
                          "t_ver": 0.0, "t_last": None} for n in self.names}
        self.cv = threading.Condition()
        self.error = None
        for p in self.procs.values():
            p.start()
        self.reader = threading.Thread(target=self._read, daemon=True)
        self.reader.start()

    def _read(self):
        live = len(self.names)
        try:
            while live:
                msg = self.q.get()
                if msg[0] == "template":
                    _, name, tid, g, key = msg
                    with self.cv:
                        st = self.state[name]
                        st["graphs"][tid] = g
                        st["keys"][tid] = key
                        st["pending"] += 1
                    self.pool.apply_async(_verify_template, (name, tid, g), callback=self._verified,
                                          error_callback=self._failed)
                else:
                    _, name, stats, gen_s = msg
                    with self.cv:
                        self.state[name]["done"] = (stats, gen_s, time.perf_counter() - self.t0)
                        self.cv.notify_all()
                    live -= 1
        except Exception as exc:  # pragma: no cover
            self._failed(exc)

    def _verified(self, res):
        name, tid, out, t_map, t_ver = res
        with self.cv:
            st = self.state[name]
            st["recs"][tid] = out
            st["pending"] -= 1
            st["t_map"] += t_map
            st["t_ver"] += t_ver
            st["t_last"] = time.perf_counter() - self.t0
            self.cv.notify_all()

    def _failed(self, exc):
        with self.cv:
            self.error = exc
            self.cv.notify_all()

    def result(self, name: str, timeout: float = 3600.0) -> dict:
        from . import workloads as W
        deadline = time.monotonic() + timeout
        with self.cv:
            st = self.state[name]
            while self.error is None and (st["done"] is None or st["pending"] > 0):
                if not self.cv.wait(timeout=max(0.0, deadline - time.monotonic())):
                    raise TimeoutError(f"search of {name} did not finish")
            if self.error is not None:
                raise RuntimeError(f"search worker failed: {self.error!r}")
        stats, gen_s, t_gen_end = st["done"]
        n = len(st["graphs"])
        graphs = [st["graphs"][j] for j in range(n)]
        records, vkeys = [], set()
        for j in range(n):
            for rec, vk in st["recs"][j]:
                records.append(rec)
                if vk is not None:
                    vkeys.add(vk)
        stats = dict(stats)
        stats["mapping_candidates"] = len(records)
        stats["verified_pairs"] = sum(1 for r in records if r["verified"])
        stats["unique_verified_templates"] = len(vkeys)
        done_at = max(t_gen_end, st["t_last"] or 0.0)
        spec, max_ops = W.spec_of(name)
        return {"workload": spec.name, "flags": _flags(max_ops).as_dict(),
                "templates": [{"id": j, "key": st["keys"][j]} for j in range(n)],
                "stats": stats, "candidates": records, "graphs": graphs,
                "timings": {"generate_s": gen_s, "mappings_cpu_s": st["t_map"], "verify_cpu_s": st["t_ver"],
                            "verify_tail_s": done_at - t_gen_end, "wall_s": done_at}}

    def close(self):
        self.pool.terminate()
        for p in self.procs.values():
            p.join(timeout=1)
            if p.is_alive():
                p.terminate()


def parallel_search(name: str, workers: Optional[int] = None) -> dict:
    """One workload's stages 1-3 on host processes (a SearchRun of one)."""
    run = SearchRun([name], workers)
    try:
        return run.result(name)
    finally:
        run.close()
