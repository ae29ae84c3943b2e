"""Generate the golden fixtures that pin the oracle and the B200 backend.

Runs the REFERENCE (symfuse, imported from the reference tree in the build
container; never on the GPU box) and records, per desk-scale candidate:
  * fp64 outputs of symfuse.interp.run_concrete / run_program on the inputs
    random_equiv_test would draw for trial 0 (interp.py:259,272-276);
  * finite-field outputs of the SAME reference functions with apply_op rebound
    to oracle.ff_np.FFArith (dtype=object), i.e. the reference's control flow
    with the finite-field op table -> pins oracle/block_np.py bit-exactly;
  * the reference's own random_equiv_test verdict (fp64, 3 trials x 2 params);
  * errors the reference raises (ShapeError / WriteConflictError ...).
Also records known-answer cases from the reference tests (test_interp.py).

Usage:  python tests/golden/make_golden.py   (writes desk_cases.json + desk_arrays.npz)
"""
from __future__ import annotations

import json
import os
import sys
import time
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "symfuse")):
        sys.path.insert(0, cand)
        break

import symfuse.interp as RI  # noqa: E402
from symfuse.cli import PipelineFlags, run_pipeline  # noqa: E402
from symfuse.errors import SymfuseError  # noqa: E402
from symfuse.graph import TensorSpec, deserialize, instantiate, serialize, template_key  # noqa: E402
from symfuse.mappings import enumerate_mappings  # noqa: E402
from symfuse.tuner import enumerate_param_space  # noqa: E402
from symfuse.workloads import BUILTINS, WorkloadOp, WorkloadSpec, lower  # noqa: E402

from oracle import ff_np  # noqa: E402
from paper_2604_15272_b200.ff import ff_trial_seed  # noqa: E402

MAX_OUT_ELEMS = 20000


def program_dict(p) -> dict:
    return {
        "name": p.name,
        "tensors": [{"name": t.name, "dims": list(t.dims), "role": t.role} for t in p.tensors],
        "ops": [
            {"kind": o.kind, "inputs": list(o.inputs), "out": o.out,
             **({"axis": o.axis} if o.axis is not None else {}),
             **({"const": [o.const.numerator, o.const.denominator]} if o.const is not None else {})}
            for o in p.ops
        ],
        "outputs": list(p.outputs),
    }


def lora_desk() -> WorkloadSpec:
    return WorkloadSpec(
        name="lora",
        tensors=[TensorSpec("X", (8, 256), "input"), TensorSpec("W", (256, 64), "input"),
                 TensorSpec("A", (256, 16), "input"), TensorSpec("B", (16, 64), "input"),
                 TensorSpec("O", (8, 64), "output")],
        ops=[WorkloadOp("matmul", ("X", "W"), "Y"), WorkloadOp("matmul", ("X", "A"), "T"),
             WorkloadOp("matmul", ("T", "B"), "U"), WorkloadOp("add", ("Y", "U"), "O")],
        outputs=("O",), defaults={"grid_dims": 1, "max_ops": 9})


def two_out() -> WorkloadSpec:  # test_integration.py:18-34
    return WorkloadSpec(
        name="two_out",
        tensors=[TensorSpec("X", (16, 16), "input"), TensorSpec("A", (16, 16), "output"),
                 TensorSpec("B", (16, 1), "output")],
        ops=[WorkloadOp("exp", ("X",), "A"), WorkloadOp("sum", ("X",), "B", axis=1)],
        outputs=("A", "B"), defaults={"grid_dims": 1, "max_ops": 6})


def toy2d() -> WorkloadSpec:  # test_integration.py:37-55
    return WorkloadSpec(
        name="toy2d",
        tensors=[TensorSpec("A", (32, 32), "input"), TensorSpec("B", (32, 32), "input"),
                 TensorSpec("O", (32, 32), "output")],
        ops=[WorkloadOp("add", ("A", "B"), "O")], outputs=("O",), defaults={"grid_dims": 2, "max_ops": 4})


def ff_run(fn, *args, **kw):
    """Run a reference function with its op table swapped for the FF one."""
    saved = RI.apply_op
    RI.apply_op = ff_np.FFArith()
    try:
        return fn(*args, **kw)
    finally:
        RI.apply_op = saved


def ff_to_int(a) -> np.ndarray:
    flat = [(-1 if isinstance(v, float) else int(v) % ff_np.P) for v in np.asarray(a, dtype=object).ravel()]
    return np.asarray(flat, dtype=np.int64).reshape(np.shape(a))


def main() -> None:
    t0 = time.time()
    specs = [BUILTINS[n]() for n in ("softmax_matmul", "rmsnorm", "rmsnorm_mlp", "swiglu", "attention",
                                      "qk_attention", "identity")]
    specs += [lora_desk(), two_out(), toy2d()]
    cases, arrays = [], {}
    per_workload_cap = {"softmax_matmul": 8}
    for spec in specs:
        program = lower(spec)
        rep = run_pipeline(spec, PipelineFlags(until="verify"))
        recs = rep["candidates"]
        ver = [c for c in recs if c["verified"]]
        unver = [c for c in recs if not c["verified"]]
        rng = np.random.default_rng(zlib.crc32(spec.name.encode()))
        pick_unver = [unver[i] for i in rng.choice(len(unver), size=min(6, len(unver)), replace=False)] if unver else []
        n_case = 0
        for c in ver + pick_unver:
            g, _, _ = deserialize(rep["templates"][c["template_id"]]["key"], program)
            on = set(c["mapping"])
            m = {v: (1 if f"{v.tensor}.{v.dim}.{v.pdim}" in on else 0) for v in g.mapping_vars()}
            space = enumerate_param_space(g, m, budget_bytes=None)
            if not space:
                continue
            picks = sorted({0, len(space) // 2, len(space) - 1})
            verdict = RI.random_equiv_test(g, m, program, trials=3, param_samples=2, seed=0)
            for pi in picks:
                if per_workload_cap.get(spec.name, 10**9) <= n_case:
                    break
                params = space[pi]
                cid = RI.candidate_id(g, m)
                trial_rng = np.random.default_rng([0, cid, 0])
                inputs = {nm: trial_rng.standard_normal(program.spec(nm).dims) for nm in program.inputs}
                ffin = {nm: ff_np.ff_uniform(int(np.prod(program.spec(nm).dims)), ff_trial_seed(0, cid, 0), k + 1)
                        .reshape(program.spec(nm).dims) for k, nm in enumerate(program.inputs)}
                case = {
                    "id": len(cases), "workload": spec.name, "program": program_dict(program),
                    "key": template_key(g, m), "params": params, "cid": cid, "verified": c["verified"],
                    "serialized": serialize(g, m, params),
                    "ref_verdict": {"ok": verdict.ok, "note": verdict.note, "max_rel_err": verdict.max_rel_err,
                                    "trials": verdict.trials},
                }
                try:
                    concrete = instantiate(g, m, params)
                except SymfuseError as exc:
                    case["instantiate_error"] = type(exc).__name__
                    cases.append(case)
                    continue
                out_elems = sum(int(np.prod(program.spec(nm).dims)) for nm in program.outputs)
                keep = out_elems <= MAX_OUT_ELEMS
                try:
                    got = RI.run_concrete(concrete, inputs)
                    case["f64_error"] = None
                    exp = RI.run_program(program, inputs)
                    case["f64_rel_err_vs_program"] = max(RI.rel_err(got[k], exp[k]) for k in program.outputs)
                    if keep:
                        for k in program.outputs:
                            arrays[f"c{case['id']}_f64_{k}"] = got[k]
                except SymfuseError as exc:
                    case["f64_error"] = type(exc).__name__
                except ValueError as exc:  # numpy-level failure of a force-fed mapping
                    case["f64_error"] = "ValueError"
                try:
                    ffgot = ff_run(RI.run_concrete, concrete, ffin, dtype=object)
                    ffexp = ff_run(RI.run_program, program, ffin)
                    case["ff_error"] = None
                    ok = True
                    for k in program.outputs:
                        a, b = ff_to_int(ffgot[k]), ff_to_int(ffexp[k])
                        ok = ok and bool(np.array_equal(a, b))
                        if keep:
                            arrays[f"c{case['id']}_ff_{k}"] = a.astype(np.int64)
                            arrays[f"c{case['id']}_ffprog_{k}"] = b.astype(np.int64)
                    case["ff_equal_program"] = ok
                except SymfuseError as exc:
                    case["ff_error"] = type(exc).__name__
                except ValueError:
                    case["ff_error"] = "ValueError"
                case["stored"] = keep
                cases.append(case)
                n_case += 1
        print(f"{spec.name}: {n_case} cases ({len(ver)} verified pairs), {time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(HERE, "desk_cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "symfuse 0.1.0", "cases": cases}, fh)
    np.savez_compressed(os.path.join(HERE, "desk_arrays.npz"), **arrays)
    print(f"{len(cases)} cases, {len(arrays)} arrays, {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
