"""Finite-field (mod 2^31-1) equivalence checking on device.

Random-test equivalence in the reference is fp64 with a 1e-9 tolerance
(interp.py:238-286).  Here candidate and program are evaluated in GF(p),
p = 2^31-1, on uniformly random residues: exact arithmetic, so agreement is
bit-exact and a single mismatching cell refutes the candidate.  exp / silu /
sqrt are uninterpreted keyed hashes (no verifier axiom uses their identities,
verifier/axioms.py:75-355), div uses the Fermat inverse, scale uses n*d^-1.
"""
from __future__ import annotations

_M64 = (1 << 64) - 1


def _mix64(z: int) -> int:
    z &= _M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M64
    z ^= z >> 31
    return z


def ff_trial_seed(seed: int, cid: int, trial: int) -> int:
    """Seed of the FF inputs of one trial; the triple mirrors the reference's
    default_rng([seed, candidate_id, trial]) streams (interp.py:259,272)."""
    return _mix64(_mix64(seed + 0x632BE59BD9B4E019) ^ _mix64(cid + 0x8CB92BA72F3D8DD7) ^ (trial + 1))


import ctypes as _C  # noqa: E402

import numpy as np  # noqa: E402

from . import _abi, ir  # noqa: E402
from .errors import SymfuseError  # noqa: E402
from .plan import PLANS, torch  # noqa: E402


def ff_fill_inputs(program: ir.Program, seed64: int, device: int) -> list:
    """Uniform residues for every program input (salt = input index + 1);
    identical to oracle/ff_np.py:ff_uniform on the host."""
    t = torch()
    _abi.bind_device(device)
    s = _C.c_void_p(t.cuda.current_stream(device).cuda_stream)
    out = []
    for k, name in enumerate(program.inputs):
        x = t.empty(tuple(program.spec(name).dims), dtype=t.int32, device=device)
        _abi.check(_abi.lib().sgm_ff_fill(_C.c_void_p(x.data_ptr()), x.numel(), seed64 & ((1 << 64) - 1), k + 1, s))
        out.append(x)
    return out


def ff_run(cand: ir.Candidate, inputs: list, device: int, hints=None) -> list:
    t = torch()
    prog = cand.program
    outs = [t.empty(tuple(prog.spec(n).dims), dtype=t.int32, device=device) for n in prog.outputs]
    PLANS.get(cand, _abi.FF, hints, device).run(inputs, outs)
    return outs


def ff_equal(a, b) -> bool:
    t = torch()
    if tuple(a.shape) != tuple(b.shape):
        return False
    n = _C.c_int64()
    _abi.bind_device(a.device.index)
    _abi.check(_abi.lib().sgm_compare_u32(_C.c_void_p(a.data_ptr()), _C.c_void_p(b.data_ptr()), a.numel(),
                                          _C.c_void_p(t.cuda.current_stream(a.device).cuda_stream), _C.byref(n)))
    return n.value == 0


def ff_equiv_test(graph, mapping, program=None, trials: int = 2, param_samples: int = 3, seed: int = 0,
                  params_list=None, budget_bytes=None, *, device=None):
    """Finite-field counterpart of random_equiv_test (interp.py:238-286): same
    parameter sampling, same verdict type; a verdict is exact (max_rel_err 0.0
    when every output cell agrees, inf otherwise)."""
    from .interp import EquivVerdict, _instantiate, candidate_id, device_index
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
    prog_cand = ir.program_candidate(prog)
    for params in chosen:
        try:
            cand = _instantiate(graph, mapping, params)
        except SymfuseError as exc:
            return EquivVerdict(False, float("inf"), 0, [params], f"instantiate: {exc}")
        for trial in range(trials):
            ins = ff_fill_inputs(prog, ff_trial_seed(seed, cid, trial), dev)
            expected = ff_run(prog_cand, ins, dev)
            try:
                got = ff_run(cand, ins, dev)
            except SymfuseError as exc:
                return EquivVerdict(False, float("inf"), trial, [params], f"run: {exc}")
            if not all(ff_equal(g, e) for g, e in zip(got, expected)):
                return EquivVerdict(False, float("inf"), trial + 1, chosen, "mismatch")
    return EquivVerdict(True, 0.0, trials, chosen)
