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

Usage: python paper_2604_15272_b200/populations/make_populations.py [R G A Q L]
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "symfuse")):
        sys.path.insert(0, p)
        break

from symfuse.cli import PipelineFlags, run_pipeline  # noqa: E402
from symfuse.graph import TensorSpec, deserialize, template_key  # noqa: E402
from symfuse.tuner import enumerate_param_space  # noqa: E402
from symfuse.workloads import BUILTINS, WorkloadOp, WorkloadSpec, lower  # noqa: E402


def lora() -> WorkloadSpec:
    # LoRA r=16 fused linear: O = X W + (X A) B  (JSON workload of primitives)
    return WorkloadSpec(
        name="lora",
        tensors=[TensorSpec("X", (8, 4096), "input"), TensorSpec("W", (4096, 4096), "input"),
                 TensorSpec("A", (4096, 16), "input"), TensorSpec("B", (16, 4096), "input"),
                 TensorSpec("O", (8, 4096), "output")],
        ops=[WorkloadOp("matmul", ("X", "W"), "Y"), WorkloadOp("matmul", ("X", "A"), "T"),
             WorkloadOp("matmul", ("T", "B"), "U"), WorkloadOp("add", ("Y", "U"), "O")],
        outputs=("O",), defaults={"grid_dims": 1, "max_ops": 9})


CONFIGS = {
    "R": dict(builtin="rmsnorm", dtype="f32", max_ops=None,
              scale={"X": (8, 4096), "W": (4096, 4096), "O": (8, 4096)},
              desc="RMSNorm+MatMul, batch 8, hidden 4096 -> 4096, fp32"),
    "G16384": dict(builtin="swiglu", dtype="bf16", max_ops=None,
                   scale={"X": (8, 4096), "Wgate": (4096, 16384), "Wup": (4096, 16384), "O": (8, 16384)},
                   desc="Gated MLP SiLU(x W1) * (x W3), batch 8, 4096 -> 16384 (power-of-two API), bf16"),
    "A": dict(builtin="attention", dtype="bf16", max_ops=11,
              scale={"Q": (2, 8, 8, 128), "Kt": (2, 8, 128, 8192), "V": (2, 8, 8192, 128), "O": (2, 8, 8, 128)},
              desc="GQA decode attention, 64 q / 8 kv heads, head_dim 128, KV 8192, batch 2, bf16"),
    "Q": dict(builtin="qk_attention", dtype="bf16", max_ops=None,
              scale={"Q": (8, 8, 4, 128), "Kt": (8, 8, 128, 8192), "V": (8, 8, 8192, 128), "O": (8, 8, 4, 128)},
              desc="QKNorm + attention, hidden 4096 (32 q / 8 kv heads), KV 8192, batch 8, bf16"),
    "L": dict(builtin=None, dtype="bf16", max_ops=None, scale=None,
              desc="LoRA rank-16 fused linear, batch 8, hidden 4096, bf16"),
}


def program_dict(p) -> dict:
    return {
        "name": p.name,
        "tensors": [{"name": t.name, "dims": list(t.dims), "role": t.role} for t in p.tensors],
        "ops": [{"kind": o.kind, "inputs": list(o.inputs), "out": o.out,
                 **({"axis": o.axis} if o.axis is not None else {}),
                 **({"const": [o.const.numerator, o.const.denominator]} if o.const is not None else {})}
                for o in p.ops],
        "outputs": list(p.outputs),
    }


def build(name: str) -> dict:
    cfg = CONFIGS[name]
    spec = lora() if cfg["builtin"] is None else BUILTINS[cfg["builtin"]]()
    if cfg["scale"]:
        spec.scale = cfg["scale"]
    t0 = time.perf_counter()
    rep = run_pipeline(spec, PipelineFlags(until="verify", max_ops=cfg["max_ops"]))
    wall = time.perf_counter() - t0
    program = lower(spec)
    cands = []
    for c in rep["candidates"]:
        if not c["verified"]:
            continue
        g, _, _ = deserialize(rep["templates"][c["template_id"]]["key"], program)
        on = set(c["mapping"])
        m = {v: (1 if f"{v.tensor}.{v.dim}.{v.pdim}" in on else 0) for v in g.mapping_vars()}
        cands.append({"template_id": c["template_id"], "mapping": c["mapping"], "key": template_key(g, m),
                      "space": enumerate_param_space(g, m, budget_bytes=None)})
    return {"config": name, "desc": cfg["desc"], "dtype": cfg["dtype"], "program": program_dict(program),
            "search": {"timings": rep["timings"], "stats": rep["stats"], "wall_s": wall,
                       "max_ops": cfg["max_ops"] or spec.defaults.get("max_ops")},
            "candidates": cands}


def derive_g14336(g16384: dict) -> dict:
    sys.path.insert(0, ROOT)
    from paper_2604_15272_b200 import ir
    from paper_2604_15272_b200.tuner import enumerate_param_space as my_space
    prog = json.loads(json.dumps(g16384["program"]))
    for t in prog["tensors"]:
        t["dims"] = [14336 if d == 16384 else d for d in t["dims"]]
    P = ir.Program.from_json(prog)
    cands = []
    for c in g16384["candidates"]:
        cand = ir.from_serialized(c["key"], P, {})
        cands.append({**c, "space": my_space(cand, budget_bytes=None)})
    return {**g16384, "config": "G", "program": prog, "candidates": cands,
            "desc": "Gated MLP SiLU(x W1) * (x W3), batch 8, 4096 -> 14336, bf16 (plan-layer extent; "
                    "templates from the 16384 search)"}


def main(argv) -> None:
    names = argv or ["R", "G16384", "A", "Q", "L"]
    for n in names:
        pop = build(n)
        with open(os.path.join(HERE, f"{n}.json"), "w") as fh:
            json.dump(pop, fh, indent=1)
        tot = sum(len(c["space"]) for c in pop["candidates"])
        print(f"{n}: {len(pop['candidates'])} verified pairs, {tot} candidates, search {pop['search']['wall_s']:.1f}s")
        if n == "G16384":
            g = derive_g14336(pop)
            with open(os.path.join(HERE, "G.json"), "w") as fh:
                json.dump(g, fh, indent=1)
            print(f"G: {len(g['candidates'])} pairs, {sum(len(c['space']) for c in g['candidates'])} candidates")


if __name__ == "__main__":
    main(sys.argv[1:])
