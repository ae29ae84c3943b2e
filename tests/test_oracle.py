"""The oracle (oracle/) against the reference's golden fixtures (CPU only)."""
import numpy as np
import pytest

from conftest import case_inputs_f64, case_inputs_ff
from oracle import block_np, ff_np


def _stored(cases):
    return [c for c in cases if c.get("stored") and not c.get("instantiate_error")]


def test_fixture_population(desk_cases):
    assert len(desk_cases) >= 250
    assert {c["workload"] for c in desk_cases} >= {"rmsnorm", "rmsnorm_mlp", "swiglu", "attention", "qk_attention",
                                                   "softmax_matmul", "lora", "identity"}


def test_oracle_f64_matches_reference(desk_cases, desk_arrays):
    n = 0
    for c in _stored(desk_cases):
        if c.get("f64_error"):
            continue
        got = block_np.run_concrete(c["program"], c["key"], c["params"], case_inputs_f64(c))
        for name, arr in got.items():
            ref = desk_arrays[f"c{c['id']}_f64_{name}"]
            if np.isfinite(ref).all():
                assert block_np.rel_err(arr, ref) < 1e-12, (c["id"], name)
            else:  # unwritten cells / overflow must agree too
                assert np.array_equal(np.isnan(arr), np.isnan(ref))
            n += 1
    assert n >= 150


def test_oracle_ff_bit_exact_with_reference_control_flow(desk_cases, desk_arrays):
    ar = ff_np.FFArith()
    n = 0
    for c in _stored(desk_cases):
        if c.get("ff_error"):
            continue
        ins = case_inputs_ff(c)
        got = block_np.run_concrete(c["program"], c["key"], c["params"], ins, arith=ar)
        exp = block_np.run_program(c["program"], ins, arith=ar)
        for name in c["program"]["outputs"]:
            assert np.array_equal(got[name], desk_arrays[f"c{c['id']}_ff_{name}"]), (c["id"], name)
            assert np.array_equal(exp[name], desk_arrays[f"c{c['id']}_ffprog_{name}"]), (c["id"], name)
        eq = all(np.array_equal(got[k], exp[k]) for k in c["program"]["outputs"])
        assert eq == c["ff_equal_program"]
        n += 1
    assert n >= 150


def test_ff_verdict_agrees_with_fp64_oracle(desk_cases):
    for c in desk_cases:
        if "f64_rel_err_vs_program" in c and c.get("ff_equal_program") is not None:
            assert (c["f64_rel_err_vs_program"] <= 1e-9) == c["ff_equal_program"], c["id"]


def test_ff_field_laws():
    rng = np.random.default_rng(0)
    a = ff_np.ff_uniform(1000, 1, 1)
    b = ff_np.ff_uniform(1000, 2, 1)
    ar = ff_np.FFArith()
    assert np.all(ar("mul", [a, ff_np.inv(a)]) == (a != 0))
    assert np.array_equal(ar("div", [ar("mul", [a, b]), b]), a * (b != 0) % ff_np.P)
    m1 = rng.integers(0, ff_np.P, size=(3, 5))
    m2 = rng.integers(0, ff_np.P, size=(5, 4))
    exact = (m1.astype(object) @ m2.astype(object)) % ff_np.P
    assert np.array_equal(ff_np.matmul(m1, m2), exact.astype(np.int64))
    from fractions import Fraction
    s = ar("scale", [a], const_=Fraction(1, 4096))
    assert np.array_equal(ar("mul", [s, np.full_like(a, 4096)]), a)


def test_ff_uniform_range_and_determinism():
    x = ff_np.ff_uniform(4096, 123, 7)
    assert x.min() >= 0 and x.max() < ff_np.P
    assert np.array_equal(x, ff_np.ff_uniform(4096, 123, 7))
    assert not np.array_equal(x, ff_np.ff_uniform(4096, 123, 8))
