"""Build the full-scale candidate populations from the UNCHANGED reference search.

Runs symfuse's run_pipeline(until="verify") (stages 1-3: generate, mappings,
e-graph verification; cli.py:69-157) on each BASELINE config, then records
every verified (template, mapping) with its divisibility-only parameter space
(tuner.enumerate_param_space(budget_bytes=None), SURVEY §8a+).  This runs in
the build container (the reference is importable here); the GPU box reads the
resulting JSON.  Gated MLP at 14336 (BASELINE config 2) is not expressible
through the reference's power-of-two TensorSpec (graph.py:96-101):
its population re-uses the 16384 templates/mappings (structure is size-free)
with the parameter space enumerated by this backend's own plan layer.
The workload specs live in paper_2604_15272_b200/workloads.py (also used by
the end-to-end optimisation run, optimize.py).

Usage: python paper_2604_15272_b200/populations/make_populations.py [R G16384 A Q L]
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2604_15272_b200 import workloads as W  # noqa: E402

W.import_reference()
from symfuse.cli import PipelineFlags, run_pipeline  # noqa: E402


def build(name: str) -> dict:
    spec, max_ops = W.spec_of(name)
    t0 = time.perf_counter()
    rep = run_pipeline(spec, PipelineFlags(until="verify", max_ops=max_ops))
    return W.population_from_report(name, rep, time.perf_counter() - t0)


def main(argv) -> None:
    names = argv or ["R", "G16384", "A", "Q", "L"]
    for n in names:
        pop = build(n)
        with open(os.path.join(HERE, f"{n}.json"), "w") as fh:
            json.dump(pop, fh, indent=1)
        tot = sum(len(c["space"]) for c in pop["candidates"])
        print(f"{n}: {len(pop['candidates'])} verified pairs, {tot} candidates, search {pop['search']['wall_s']:.1f}s")
        if n == "G16384":
            g = W.derive_g14336(pop)
            with open(os.path.join(HERE, "G.json"), "w") as fh:
                json.dump(g, fh, indent=1)
            print(f"G: {len(g['candidates'])} pairs, {sum(len(c['space']) for c in g['candidates'])} candidates")


if __name__ == "__main__":
    main(sys.argv[1:])
