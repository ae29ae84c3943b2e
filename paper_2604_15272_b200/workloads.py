"""The five BASELINE workloads as reference WorkloadSpecs.

Built from the UNCHANGED reference's builtins (workloads.py:278-291) at the
configs' scale, plus LoRA as a JSON-style workload of primitives.
Gated MLP at 14336 is not expressible through the reference's power-of-two
TensorSpec (graph.py:96-101): it is searched at 16384 and its
population re-uses those templates/mappings with the parameter space
enumerated by this backend's plan layer (`derive_g14336`).
Needs the reference package importable (baseline/_ref, or /root/reference/pkg/src).
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def import_reference():
    """Make the unmodified reference (symfuse) importable; returns the module or None."""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "symfuse")):
            if p not in sys.path:
                sys.path.append(p)
            break
    try:
        import symfuse
        return symfuse
    except ImportError:
        return None


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
# the workload a config is searched as (G at 14336 is searched at 16384)
SEARCH_AS = {"R": "R", "G": "G16384", "G16384": "G16384", "A": "A", "Q": "Q", "L": "L"}


def lora():
    """LoRA r=16 fused linear: O = X W + (X A) B (a workload of primitives)."""
    from symfuse.graph import TensorSpec
    from symfuse.workloads import WorkloadOp, WorkloadSpec
    return WorkloadSpec(
        name="lora",
        tensors=[TensorSpec("X", (8, 4096), "input"), TensorSpec("W", (4096, 4096), "input"),
                 TensorSpec("A", (4096, 16), "input"), TensorSpec("B", (16, 4096), "input"),
                 TensorSpec("O", (8, 4096), "output")],
        ops=[WorkloadOp("matmul", ("X", "W"), "Y"), WorkloadOp("matmul", ("X", "A"), "T"),
             WorkloadOp("matmul", ("T", "B"), "U"), WorkloadOp("add", ("Y", "U"), "O")],
        outputs=("O",), defaults={"grid_dims": 1, "max_ops": 9})


def spec_of(name: str):
    """(WorkloadSpec at the config's scale, max_ops override) of a config name."""
    from symfuse.workloads import BUILTINS
    cfg = CONFIGS[SEARCH_AS[name]]
    spec = lora() if cfg["builtin"] is None else BUILTINS[cfg["builtin"]]()
    if cfg["scale"]:
        spec.scale = cfg["scale"]
    return spec, cfg["max_ops"]


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


def population_from_report(name: str, report: dict, wall_s: float, graphs=None) -> dict:
    """Every verified (template, mapping) of a run_pipeline(until="verify") report
    with its divisibility-only parameter space (tuner.enumerate_param_space
    budget_bytes=None, SURVEY §8a+), in the committed populations' format."""
    from symfuse.graph import deserialize, template_key
    from symfuse.tuner import enumerate_param_space
    from symfuse.workloads import lower
    cfg = CONFIGS[SEARCH_AS[name]]
    spec, max_ops = spec_of(name)
    program = lower(spec)
    cands = []
    for c in report["candidates"]:
        if not c["verified"]:
            continue
        tid = c["template_id"]
        g = graphs[tid] if graphs is not None else deserialize(report["templates"][tid]["key"], program)[0]
        on = set(c["mapping"])
        m = {v: (1 if f"{v.tensor}.{v.dim}.{v.pdim}" in on else 0) for v in g.mapping_vars()}
        cands.append({"template_id": tid, "mapping": c["mapping"], "key": template_key(g, m),
                      "space": enumerate_param_space(g, m, budget_bytes=None)})
    pop = {"config": SEARCH_AS[name], "desc": cfg["desc"], "dtype": cfg["dtype"], "program": program_dict(program),
           "search": {"timings": report["timings"], "stats": report["stats"], "wall_s": wall_s,
                      "max_ops": max_ops or spec.defaults.get("max_ops")},
           "candidates": cands}
    return derive_g14336(pop) if name == "G" else pop


def derive_g14336(g16384: dict) -> dict:
    from . import ir
    from .tuner import enumerate_param_space as my_space
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
