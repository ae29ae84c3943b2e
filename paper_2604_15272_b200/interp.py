"""Drop-in replacements for the reference interpreter's public functions.

  run_concrete(concrete, inputs, dtype=np.float64, tile_dump=None)   interp.py:128-212
  run_program(program, inputs)                                       interp.py:69-83
  random_equiv_test(graph, mapping, program=None, trials=20, param_samples=3,
                    tol=1e-9, seed=0, params_list=None, budget_bytes=None)  interp.py:238-286
  rel_err, candidate_id, EquivVerdict                                interp.py:219-235

Same names, argument meaning and error behaviour; the execution happens in a
kernel generated for the candidate and compiled for sm_100a (libsgm).  Inputs
may be numpy arrays (copied to the device; results come back as numpy) or
torch CUDA tensors (zero-copy; results stay on the device).  There is no CPU
fallback: without libsgm.so or a B200 these functions raise.
"""
from __future__ import annotations

import zlib
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi, ir
from .errors import BackendUnavailable, KernelTimeout, ShapeError, SymfuseError
from .plan import PLANS, numsys_of, torch, torch_dtype

try:  # reuse the reference's verdict type when it is importable
    from symfuse.interp import EquivVerdict  # type: ignore
except ImportError:
    @dataclass
    class EquivVerdict:  # interp.py:219-225
        ok: bool
        max_rel_err: float
        trials: int
        params_tested: list = field(default_factory=list)
        note: str = ""


def device_index(device: Optional[int] = None) -> int:
    t = torch()
    if not t.cuda.is_available():
        raise BackendUnavailable("no CUDA device: the B200 backend has no CPU fallback")
    return t.cuda.current_device() if device is None else int(device)


def rel_err(a, b) -> float:
    """max|a-b| / (1 + max|b|), inf if shapes differ or a is non-finite (interp.py:228-231).
    numpy arrays are reduced on the host; CUDA tensors on the device (libsgm)."""
    if isinstance(a, np.ndarray) or isinstance(b, np.ndarray):
        a = np.asarray(a, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64)
        if a.shape != b.shape or not np.isfinite(a).all():
            return float("inf")
        return float(np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b))))
    if tuple(a.shape) != tuple(b.shape):
        return float("inf")
    t = torch()
    ns = {t.float64: _abi.F64, t.float32: _abi.F32, t.bfloat16: _abi.BF16}[a.dtype]
    if b.dtype != a.dtype:
        b = b.to(a.dtype)
    import ctypes as C
    out = C.c_double()
    _abi.bind_device(a.device.index)
    _abi.check(_abi.lib().sgm_rel_err(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), a.numel(), ns,
                                      C.c_void_p(t.cuda.current_stream(a.device).cuda_stream), C.byref(out)))
    return out.value


def candidate_id(graph, mapping=None) -> int:
    """crc32 of the canonical template key (interp.py:234-235)."""
    if hasattr(graph, "block") and hasattr(graph, "store"):
        try:
            from symfuse.graph import template_key  # type: ignore
            return zlib.crc32(template_key(graph, mapping).encode())
        except ImportError:
            pass
    return ir.candidate_id(ir.candidate_of(graph, mapping))


def _to_device(arr, ns: int, dev: int):
    t = torch()
    if hasattr(arr, "data_ptr") and getattr(arr, "is_cuda", False):
        x = arr.to(device=dev, dtype=torch_dtype(ns))
    elif ns == _abi.FF:
        x = t.from_numpy(np.ascontiguousarray(np.asarray(arr, dtype=np.int64) % ((1 << 31) - 1)).astype(np.int32))
        x = x.to(dev)
    else:
        x = t.from_numpy(np.ascontiguousarray(np.asarray(arr, dtype=np.float64))).to(dev)
        x = x.to(torch_dtype(ns))
    return x.contiguous()


def _to_host(x, ns: int):
    if ns == _abi.FF:
        return x.cpu().numpy().astype(np.int64)
    if ns == _abi.BF16:
        return x.float().cpu().numpy()
    return x.cpu().numpy()


def _execute(cand: ir.Candidate, inputs: dict, ns: int, device, hints, check_missing: bool):
    dev = device_index(device)
    prog = cand.program
    host = False
    dev_in = []
    for name in prog.inputs:
        if name not in inputs:
            if check_missing:
                raise ShapeError(f"missing input {name}")
            raise KeyError(name)
        arr = inputs[name]
        shape = tuple(getattr(arr, "shape", np.shape(arr)))
        if shape != tuple(prog.spec(name).dims):
            raise ShapeError(f"{name}: got {shape}, expected {tuple(prog.spec(name).dims)}")
        host = host or not getattr(arr, "is_cuda", False)
        dev_in.append(_to_device(arr, ns, dev))
    t = torch()
    outs = [t.empty(tuple(prog.spec(n).dims), dtype=torch_dtype(ns), device=dev) for n in prog.outputs]
    plan = PLANS.get(cand, ns, hints, dev)
    plan.run(dev_in, outs, init_outputs=True)
    if plan.watchdog():
        raise KernelTimeout(f"{plan.kernel_name}: kernel watchdog fired (a wait exceeded 2 s)")
    if host:
        return {n: _to_host(o, ns) for n, o in zip(prog.outputs, outs)}
    return dict(zip(prog.outputs, outs))


def run_concrete(concrete, inputs: dict, dtype=np.float64, tile_dump: Optional[dict] = None, *,
                 device: Optional[int] = None, hints: Optional[dict] = None) -> dict:
    """Execute one instantiated candidate on the B200 (interp.py:128-212 semantics:
    NaN-initialised outputs, ShapeError on input/tile mismatch, WriteConflictError
    on overlapping saver regions)."""
    if tile_dump is not None:
        from .dump import run_with_dump
        return run_with_dump(concrete, inputs, dtype, tile_dump, device=device)
    cand = ir.candidate_of(concrete)
    return _execute(cand, inputs, numsys_of(dtype), device, hints, check_missing=False)


def run_program(program, inputs: dict, dtype=np.float64, *, device: Optional[int] = None) -> dict:
    """The original program on whole tensors (interp.py:69-83), lowered to a
    one-block candidate and run through the same code generator."""
    prog = ir.program_of(program)
    return _execute(ir.program_candidate(prog), inputs, numsys_of(dtype), device, None, check_missing=True)


def _instantiate(graph, mapping, params):
    """instantiate() of the reference when given reference objects (it also
    checks the generator's recorded equalities); the plain-form checks otherwise."""
    if hasattr(graph, "store"):
        try:
            from symfuse.graph import instantiate  # type: ignore
            return ir.candidate_of(instantiate(graph, mapping, params))
        except ImportError:
            pass
    cand = ir.candidate_of(graph, mapping, params)
    ir.validate(cand)
    return cand


def random_equiv_test(graph, mapping, program=None, trials: int = 20, param_samples: int = 3, tol: float = 1e-9,
                      seed: int = 0, params_list=None, budget_bytes=None, *, device: Optional[int] = None):
    """fp64 random testing on the device with the reference's exact RNG streams
    (interp.py:259-276), so verdicts match the CPU interpreter's."""
    from .tuner import enumerate_param_space

    prog = ir.program_of(program if program is not None else graph.program)
    if params_list is None:
        params_list = enumerate_param_space(graph, mapping, budget_bytes=budget_bytes)
    if not params_list:
        return EquivVerdict(False, float("inf"), 0, note="empty parameter space")
    cid = candidate_id(graph, mapping)
    rng = np.random.default_rng([seed, cid])
    chosen = list(params_list)
    rng.shuffle(chosen)
    chosen = chosen[:param_samples]
    dev = device_index(device)
    t = torch()
    prog_cand = ir.program_candidate(prog)
    worst = 0.0
    for params in chosen:
        try:
            cand = _instantiate(graph, mapping, params)
        except SymfuseError as exc:
            return EquivVerdict(False, float("inf"), 0, [params], f"instantiate: {exc}")
        for trial in range(trials):
            trial_rng = np.random.default_rng([seed, cid, trial])
            host = {n: trial_rng.standard_normal(prog.spec(n).dims) for n in prog.inputs}
            dev_in = [t.from_numpy(host[n]).to(dev) for n in prog.inputs]
            expected = [t.empty(tuple(prog.spec(n).dims), dtype=t.float64, device=dev) for n in prog.outputs]
            PLANS.get(prog_cand, _abi.F64, None, dev).run(dev_in, expected)
            got = [t.empty(tuple(prog.spec(n).dims), dtype=t.float64, device=dev) for n in prog.outputs]
            try:
                cplan = PLANS.get(cand, _abi.F64, None, dev)
                cplan.run(dev_in, got)
                if cplan.watchdog():
                    raise KernelTimeout(f"{cplan.kernel_name}: kernel watchdog fired")
            except SymfuseError as exc:
                return EquivVerdict(False, float("inf"), trial, [params], f"run: {exc}")
            for g_, e_ in zip(got, expected):
                worst = max(worst, rel_err(g_, e_))
            if worst > tol:
                return EquivVerdict(False, worst, trial + 1, chosen, "mismatch")
    return EquivVerdict(True, worst, trials, chosen)
