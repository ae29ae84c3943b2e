"""Lowering of a candidate to the C-ABI descriptor, and the Plan handle.

A Plan owns one generated, compiled kernel (libsgm sgm_plan).  Buffers are
torch CUDA tensors (torch is plumbing here: allocation and streams); the
kernel itself is the NVRTC-compiled code emitted by sgm_codegen.cpp.
"""
from __future__ import annotations

import ctypes as C
import threading
from collections import OrderedDict
from fractions import Fraction
from typing import Optional

from . import _abi
from .ir import INPUT, KIND_CODE, OUTPUT, Candidate, Program

_TORCH = None


def torch():
    global _TORCH
    if _TORCH is None:
        import torch as t
        _TORCH = t
    return _TORCH


def torch_dtype(numsys: int):
    t = torch()
    return {_abi.F64: t.float64, _abi.F32: t.float32, _abi.BF16: t.bfloat16, _abi.FF: t.int32}[numsys]


def numsys_of(dtype) -> int:
    """np.float64 / 'f64' / torch.float64 ... -> number system code."""
    if isinstance(dtype, int) and dtype in _abi.NUMSYS_NAMES:
        return dtype
    s = str(getattr(dtype, "__name__", dtype)).lower().replace("torch.", "")
    if s in ("float64", "f64", "double", "<class 'numpy.float64'>"):
        return _abi.F64
    if s in ("float32", "f32", "float", "<class 'numpy.float32'>"):
        return _abi.F32
    if s in ("bfloat16", "bf16"):
        return _abi.BF16
    if s in ("ff", "finite_field", "modp", "uint32"):
        return _abi.FF
    raise ValueError(f"unsupported dtype {dtype!r}")


def build_desc(c: Candidate, numsys: int, hints: Optional[dict] = None) -> _abi.PlanDesc:
    """POD lowering (include/sgm.h sgm_plan_desc)."""
    prog: Program = c.program
    blk = c.block
    d = _abi.PlanDesc()
    d.abi_version = _abi.ABI_VERSION
    d.numsys = numsys
    ins, outs = list(prog.inputs), list(prog.outputs)
    if len(ins) > _abi.MAX_SLOTS or len(outs) > _abi.MAX_SLOTS:
        raise ValueError("too many program inputs/outputs")
    if len(blk.nodes) > _abi.MAX_NODES:
        raise ValueError("block graph has too many nodes")
    d.n_inputs, d.n_outputs = len(ins), len(outs)
    for k, name in enumerate(ins):
        dims = prog.spec(name).dims
        d.inputs[k].rank = len(dims)
        for j, v in enumerate(dims):
            d.inputs[k].dims[j] = int(v)
    for k, name in enumerate(outs):
        dims = prog.spec(name).dims
        d.outputs[k].rank = len(dims)
        for j, v in enumerate(dims):
            d.outputs[k].dims[j] = int(v)
    if not 1 <= len(blk.grid) <= _abi.MAX_GRID:
        raise ValueError("grid rank must be 1..3")
    d.n_grid = len(blk.grid)
    for g, q in enumerate(blk.grid):
        d.grid[g] = int(c.params[q])
    d.n_loop = int(c.params[blk.loop])
    d.n_nodes = len(blk.nodes)
    for k, n in enumerate(blk.nodes):
        if n.idx != k:
            raise ValueError("block nodes must be numbered 0..n-1 in order")
        nd = d.nodes[k]
        if n.kind not in KIND_CODE:
            from .errors import UnsupportedOpError
            raise UnsupportedOpError(f"unknown op kind {n.kind}")
        nd.kind = KIND_CODE[n.kind]
        nd.n_inputs = len(n.inputs)
        for j, x in enumerate(n.inputs):
            nd.inputs[j] = x
        nd.slot = -1
        nd.axis = -1 if n.axis is None else int(n.axis)
        const = n.const if n.const is not None else Fraction(1)
        nd.const_num, nd.const_den = const.numerator, const.denominator
        if n.kind == INPUT:
            nd.slot = ins.index(n.tensor)
            dims = prog.spec(n.tensor).dims
            for dd, size in enumerate(dims):
                if size <= 1:
                    continue
                mask = 0
                for g, q in enumerate(blk.grid):
                    if c.on(n.tensor, dd, q):
                        mask |= 1 << g
                nd.grid_mask[dd] = mask
                nd.loop_split[dd] = 1 if c.on(n.tensor, dd, blk.loop) else 0
        elif n.kind == OUTPUT:
            nd.slot = outs.index(n.tensor)
            var = prog.saver_var(n.tensor)
            dims = prog.spec(n.tensor).dims
            for dd, size in enumerate(dims):
                if size <= 1:
                    continue
                mask = 0
                for g, q in enumerate(blk.grid):
                    if c.on(var, dd, q):
                        mask |= 1 << g
                nd.grid_mask[dd] = mask
    h = hints or {}
    d.hints.max_cluster = int(h.get("max_cluster", 0))
    d.hints.target_ctas = int(h.get("target_ctas", 0))
    d.hints.threads = int(h.get("threads", 0))
    d.hints.smem_budget = int(h.get("smem_budget", 0))
    d.hints.no_loop_split = int(h.get("no_loop_split", 0))
    d.hints.no_hoist = int(h.get("no_hoist", 0))
    d.hints.use_tcgen05 = int(h.get("use_tcgen05", 0))
    d.hints.no_tma = int(h.get("no_tma", 0))
    d.hints.trace = int(h.get("trace", 0))
    d.hints.variant = int(h.get("variant", 0))
    d.hints.one_cta = int(h.get("one_cta", 0))
    d.hints.max_gsplit = int(h.get("max_gsplit", 0))
    d.hints.slot_kb = int(h.get("slot_kb", 0))
    d.hints.wd_test = int(h.get("wd_test", 0))
    d.hints.small_plain = int(h.get("small_plain", 0))
    d.hints.big_first = int(h.get("big_first", 0))
    d.hints.item_cost_ns = int(h.get("item_cost_ns", 0))
    d.hints.min_gsplit = int(h.get("min_gsplit", 0))
    d.hints.no_wd = int(h.get("no_wd", 0))
    d.hints.interleave = int(h.get("interleave", 0))
    d.hints.ff_tma = int(h.get("ff_tma", 0))
    d.hints.no_xcache = int(h.get("no_xcache", 0))
    d.hints.no_prefetch = int(h.get("no_prefetch", 0))
    return d


class Plan:
    """One compiled candidate kernel on one device."""

    def __init__(self, cand: Candidate, numsys: int, hints: Optional[dict] = None, device: Optional[int] = None):
        L = _abi.lib()
        self.cand = cand
        self.numsys = numsys
        self.device = device
        if device is not None:
            _abi.bind_device(device)
        self._desc = build_desc(cand, numsys, hints)
        h = C.c_void_p()
        _abi.check(L.sgm_plan_create(C.byref(self._desc), C.byref(h)))
        self._h = h
        info = _abi.PlanInfo()
        _abi.check(L.sgm_plan_info_get(h, C.byref(info)))
        self.info = {
            "logical_blocks": info.logical_blocks, "ctas": info.ctas, "cluster": info.cluster,
            "threads": info.threads, "smem_bytes": info.smem_bytes, "loop_parts": info.loop_parts,
            "free_parts": info.free_parts, "scratch_bytes": info.scratch_bytes,
            "compile_ms": info.compile_ms, "cache_hit": bool(info.cache_hit), "n_tcgen05": info.n_tcgen05,
            "kernel_name": info.kernel_name.decode(), "summary": info.plan_summary.decode(),
        }

    @property
    def kernel_name(self) -> str:
        return self.info["kernel_name"]

    def source(self) -> str:
        L = _abi.lib()
        n = C.c_size_t()
        _abi.check(L.sgm_plan_source(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _abi.check(L.sgm_plan_source(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def cubin(self) -> bytes:
        """sm_100a cubin of a compile-only plan (device=None)."""
        L = _abi.lib()
        n = C.c_size_t()
        _abi.check(L.sgm_plan_cubin(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _abi.check(L.sgm_plan_cubin(self._h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def _bind(self):
        if self.device is None:
            raise _abi.BackendUnavailable("plan compiled without a device")
        _abi.bind_device(self.device)

    def run(self, inputs, outputs, init_outputs: bool = True, stream=None) -> None:
        """inputs/outputs: torch CUDA tensors in program input/output order."""
        self._bind()
        ip = _abi.ptr_array([t.data_ptr() for t in inputs])
        op = _abi.ptr_array([t.data_ptr() for t in outputs])
        s = stream if stream is not None else torch().cuda.current_stream(self.device).cuda_stream
        _abi.check(_abi.lib().sgm_plan_run(self._h, ip, op, 1 if init_outputs else 0, C.c_void_p(s)))

    def run_host(self, host_inputs, host_outputs, stream=None) -> None:
        """numpy (C-contiguous) in/out; copies H2D/D2H inside (the e2e path)."""
        self._bind()
        ip = _abi.ptr_array([a.ctypes.data for a in host_inputs])
        op = _abi.ptr_array([a.ctypes.data for a in host_outputs])
        s = stream if stream is not None else torch().cuda.current_stream(self.device).cuda_stream
        _abi.check(_abi.lib().sgm_plan_run_host(self._h, ip, op, C.c_void_p(s)))

    def time(self, input_sets, outputs, warmup: int = 3, iters: int = 50) -> float:
        """Mean microseconds per launch over `iters` back-to-back launches,
        rotating over `input_sets` (list of input lists)."""
        self._bind()
        flat = [t.data_ptr() for ins in input_sets for t in ins]
        ip = _abi.ptr_array(flat)
        op = _abi.ptr_array([t.data_ptr() for t in outputs])
        out = C.c_double()
        s = torch().cuda.current_stream(self.device).cuda_stream
        _abi.check(_abi.lib().sgm_plan_time(self._h, ip, op, len(input_sets), warmup, iters, C.c_void_p(s),
                                            C.byref(out)))
        return out.value

    def watchdog(self, reset: bool = True, stream=None) -> bool:
        """True if a launch of this plan hit the kernel watchdog since the last reset
        (sgm_plan_watchdog; synchronises the stream)."""
        self._bind()
        s = stream if stream is not None else torch().cuda.current_stream(self.device).cuda_stream
        v = C.c_int()
        _abi.check(_abi.lib().sgm_plan_watchdog(self._h, C.c_void_p(s), 1 if reset else 0, C.byref(v)))
        return bool(v.value)

    def trace(self):
        """(launched CTAs, SGM_TRACE_N, 2) array of (time_ns, event) of the last run
        (plans created with hints={"trace": 1})."""
        import numpy as np
        n = C.c_int64()
        _abi.check(_abi.lib().sgm_plan_trace(self._h, None, 0, C.byref(n)))
        buf = np.zeros((max(1, n.value), 2), dtype=np.uint64)
        _abi.check(_abi.lib().sgm_plan_trace(self._h, buf.ctypes.data, n.value, C.byref(n)))
        return buf.reshape(-1, 512, 2)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().sgm_plan_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class PlanCache:
    """LRU of compiled plans keyed by (serialized candidate, numsys, hints, device)."""

    def __init__(self, capacity: int = 256):
        self.capacity = capacity
        self._d: "OrderedDict[tuple, Plan]" = OrderedDict()
        self._lock = threading.Lock()

    @staticmethod
    def cand_key(cand: Candidate) -> str:
        k = getattr(cand, "_plan_key", None)
        if k is None:
            from .ir import serialize
            k = serialize(cand) + "|" + repr(cand.program.to_json())
            try:
                cand._plan_key = k
            except AttributeError:
                pass
        return k

    def get(self, cand: Candidate, numsys: int, hints: Optional[dict] = None, device: Optional[int] = 0) -> Plan:
        key = (self.cand_key(cand), numsys, tuple(sorted((hints or {}).items())), device)
        with self._lock:
            p = self._d.get(key)
            if p is not None:
                self._d.move_to_end(key)
                return p
        p = Plan(cand, numsys, hints, device)
        with self._lock:
            self._d[key] = p
            while len(self._d) > self.capacity:
                _, old = self._d.popitem(last=False)
                old.close()
        return p


PLANS = PlanCache(capacity=8192)
