"""Plug the B200 backend into an unmodified `symfuse` (the reference package).

The reference's hot path reaches its executor through module globals:
  * random_equiv_test calls `run_concrete` / `run_program` from the
    `symfuse.interp` module namespace (interp.py:277,279);
  * score_interp imports `run_concrete` from `.interp` at call time
    (tuner.py:162);
  * run_pipeline stage 4 calls `tune(..., backend=flags.backend)`
    (cli.py:182-189), whose backend switch is tuner.py:215-220.
`install()` rebinds those names, so the reference's own stage-4 loop, its
oracle and its interp-backend tuner execute on the B200 without editing the
reference; `backend="b200"` becomes a valid tune() backend (and CLI choice).
It also (a) adds "b200" to the CLI's --backend choices (cli.py:255) by wrapping
`build_parser`, (b) tunes each workload in its deployment dtype (WORKLOAD_DTYPES,
keyed by program name; BASELINE configs: RMSNorm fp32, the rest bf16), with the
B200 resource model in place of the 164 KiB budget (tuner.B200_BUDGET), and
(c) wraps `run_pipeline` / `export_dots` so every tuned record of the report
carries the GPU evidence of its best kernel (`rec["b200"]`: latency_us, hbm_gbs,
roofline_frac, ff_ok, gpu_rank, kernel, dtype; cli.py:133-146,199-223).
`uninstall()` restores the originals.  Names bound at import time elsewhere
(`symfuse.run_concrete`, `from symfuse.interp import run_concrete` in callers)
are not affected; call this module's functions directly there.
"""
from __future__ import annotations

import functools
import os

_SAVED: dict = {}

# deployment dtype per program name (BASELINE.json configs); anything else: bf16
WORKLOAD_DTYPES = {"rmsnorm": "f32", "rmsnorm_mlp": "f32", "swiglu": "bf16", "attention": "bf16",
                   "qk_attention": "bf16", "lora": "bf16", "softmax_matmul": "bf16"}
# GPU evidence of the last b200 tune per (template key, mapping) — attached to reports
_EVIDENCE: dict = {}


def dtype_of(program) -> str:
    return WORKLOAD_DTYPES.get(getattr(program, "name", ""), "bf16")


def _evidence(graph, mapping, params, score_s, dtype, device) -> dict:
    """Latency, HBM throughput against the measured peak, and an FF verdict of the
    tuned kernel (candidate vs program in GF(p), bit-exact)."""
    from . import _abi, ir
    from . import population as P
    from .ff import ff_equal, ff_fill_inputs, ff_run, ff_trial_seed
    from .plan import PLANS, numsys_of
    cand = ir.candidate_of(graph, mapping, params)
    prog = cand.program
    ns = numsys_of(dtype)
    es = {_abi.F32: 4, _abi.BF16: 2, _abi.F64: 8}[ns]
    from math import prod
    byts = (sum(prod(prog.spec(n).dims) for n in prog.inputs) + sum(prod(prog.spec(n).dims) for n in prog.outputs)) * es
    lat_us = score_s * 1e6
    dev = device if device is not None else 0
    ins = ff_fill_inputs(prog, ff_trial_seed(0, ir.candidate_id(cand), 0), dev)
    exp = ff_run(ir.program_candidate(prog), ins, dev)
    got = ff_run(cand, ins, dev)
    gbs = byts / (lat_us * 1e-6) / 1e9
    try:
        import torch.distributed as dist
        rank = dist.get_rank() if dist.is_initialized() else 0
    except Exception:  # pragma: no cover
        rank = 0
    return {"latency_us": lat_us, "hbm_gbs": gbs, "roofline_frac": gbs / P.hbm_peak_gbs(),
            "ff_ok": all(ff_equal(g, e) for g, e in zip(got, exp)), "gpu_rank": rank, "dtype": dtype,
            "kernel": PLANS.get(cand, ns, None, dev).kernel_name, "algorithmic_bytes": byts}


def install(symfuse=None, device=None, dtypes: dict | None = None):
    """Rebind the reference's executor seam to the B200 backend; returns the module."""
    if symfuse is None:
        import symfuse  # noqa: F811
    import symfuse.interp as RI
    import symfuse.tuner as RT

    from . import interp as BI
    from . import tuner as BT

    if _SAVED:
        return symfuse
    if dtypes:
        WORKLOAD_DTYPES.update(dtypes)
    _SAVED.update(run_concrete=RI.run_concrete, run_program=RI.run_program, tune=RT.tune)

    @functools.wraps(RI.run_concrete)
    def run_concrete(concrete, inputs, dtype=None, tile_dump=None):
        import numpy as np
        return BI.run_concrete(concrete, inputs, np.float64 if dtype is None else dtype, tile_dump, device=device)

    @functools.wraps(RI.run_program)
    def run_program(program, inputs):
        return BI.run_program(program, inputs, device=device)

    orig_tune = RT.tune

    @functools.wraps(orig_tune)
    def tune(graph, mapping, backend="cost", samples=16, seed=0, budget_bytes=RT.DEFAULT_BUDGET, trials=3,
             model=RT.CostModel()):
        if backend != "b200":
            return orig_tune(graph, mapping, backend, samples, seed, budget_bytes, trials, model)
        dt = dtype_of(graph.program)
        r = BT.tune(graph, mapping, backend="b200", samples=samples, seed=seed, budget_bytes=budget_bytes,
                    trials=trials, dtype=dt, device=device)
        from symfuse.graph import template_key
        _EVIDENCE[(template_key(graph), _mapping_key(mapping))] = _evidence(graph, mapping, r.params, r.score, dt,
                                                                            device)
        return RT.ProfileResult(params=r.params, score=r.score)

    RI.run_concrete = run_concrete
    RI.run_program = run_program
    RT.tune = tune
    try:
        import symfuse.cli as RC
    except ImportError:  # pragma: no cover
        return symfuse
    _SAVED.update(cli_tune=RC.tune, build_parser=RC.build_parser, run_pipeline=RC.run_pipeline,
                  export_dots=RC.export_dots)
    RC.tune = tune  # cli.py imports tune by name (stage 4, cli.py:182)
    orig_parser, orig_pipeline, orig_dots = RC.build_parser, RC.run_pipeline, RC.export_dots

    @functools.wraps(orig_parser)
    def build_parser():
        parser = orig_parser()
        for act in parser._subparsers._group_actions if parser._subparsers else []:
            for sp in act.choices.values():
                for a in sp._actions:
                    if a.dest == "backend" and a.choices is not None and "b200" not in a.choices:
                        a.choices = tuple(a.choices) + ("b200",)
        return parser

    @functools.wraps(orig_pipeline)
    def run_pipeline(spec, flags=RC.PipelineFlags()):
        report = orig_pipeline(spec, flags)
        if flags.backend == "b200":
            annotate_report(report)
        return report

    @functools.wraps(orig_dots)
    def export_dots(report, spec, flags, outdir):
        written = orig_dots(report, spec, flags, outdir)
        for path in written:
            tid = int(os.path.basename(path)[len("template_"):-len(".dot")])
            ev = [c for c in report.get("candidates", []) if c["template_id"] == tid and c.get("b200")]
            if ev:
                with open(path, "a", encoding="utf-8") as fh:
                    for c in ev:
                        b = c["b200"]
                        fh.write(f"// b200 {','.join(c['mapping'])} params={c['best']['params']} "
                                 f"latency_us={b['latency_us']:.2f} hbm_gbs={b['hbm_gbs']:.0f} "
                                 f"roofline_frac={b['roofline_frac']:.3f} ff_ok={b['ff_ok']} kernel={b['kernel']}\n")
        return written

    RC.build_parser, RC.run_pipeline, RC.export_dots = build_parser, run_pipeline, export_dots
    return symfuse


def _mapping_key(mapping) -> tuple:
    return tuple(sorted(f"{v.tensor}.{v.dim}.{v.pdim}" for v, bit in mapping.items() if bit))


def annotate_report(report: dict) -> dict:
    """Attach the GPU evidence of each tuned record (cli.py:133-146 record format)."""
    keys = {t["id"]: t["key"] for t in report.get("templates", [])}
    for rec in report.get("candidates", []):
        ev = _EVIDENCE.get((keys.get(rec["template_id"]), tuple(rec["mapping"])))
        if ev is not None and rec.get("best") and rec["best"].get("params") is not None:
            rec["b200"] = dict(ev)
    return report


def uninstall():
    if not _SAVED:
        return
    import symfuse.interp as RI
    import symfuse.tuner as RT
    RI.run_concrete = _SAVED["run_concrete"]
    RI.run_program = _SAVED["run_program"]
    RT.tune = _SAVED["tune"]
    if "cli_tune" in _SAVED:
        import symfuse.cli as RC
        RC.tune = _SAVED["cli_tune"]
        RC.build_parser = _SAVED["build_parser"]
        RC.run_pipeline = _SAVED["run_pipeline"]
        RC.export_dots = _SAVED["export_dots"]
    _SAVED.clear()
