"""CPU-only checks of the boundary and the host logic (no GPU, no compute calls).

* libsgm.so loads and exports every entry point include/sgm.h declares; on a
  machine without a driver sgm_init fails loudly (no CPU fallback).
* The plain candidate form reproduces the reference's canonical keys and
  candidate ids (graph.py:447-528, interp.py:234-235) on every golden case.
* enumerate_param_space reproduces the reference's own spaces
  (tuner.py:74-106) for every verified pair of the committed populations.
* The planner/code generator (NVRTC compile-only, no device) maps the
  reference's error cases onto the reference's exception classes.
* LPT sharding is a deterministic partition.
"""
import json
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2604_15272_b200 as S
from paper_2604_15272_b200 import _abi, ir
from paper_2604_15272_b200 import population as P

HEADER = os.path.join(ROOT, "include", "sgm.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|long long|const char\*)\s+(sgm_\w+)\s*\(", text, re.M)))


def test_header_declares_all_bound_symbols():
    assert set(_declared()) == set(_abi.SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.sgm_abi_version() == _abi.ABI_VERSION


def test_init_fails_loudly_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    st = _abi.lib().sgm_init(0)
    assert st == 100
    assert b"libcuda" in _abi.lib().sgm_last_error()


def test_product_path_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    prog = ir.Program("e", (ir.Tensor("I", (4, 4), "input"), ir.Tensor("O", (4, 4), "output")),
                      (ir.Op("exp", ("I",), "O"),), ("O",))
    with pytest.raises(S.BackendUnavailable):
        S.run_program(prog, {"I": np.zeros((4, 4))})


def test_canonical_keys_and_candidate_ids_match_reference(desk_cases):
    for c in desk_cases:
        prog = ir.Program.from_json(c["program"])
        cand = ir.from_serialized(c["serialized"], prog)
        assert ir.template_key(cand) == c["key"], c["id"]
        assert ir.candidate_id(cand) == c["cid"], c["id"]
        assert ir.serialize(cand) == c["serialized"], c["id"]


@pytest.mark.parametrize("w", ["R", "A", "Q", "L", "G16384"])
def test_param_spaces_match_reference(w):
    pop = P.load_population(w)
    prog = ir.Program.from_json(pop["program"])
    for c in pop["candidates"]:
        cand = ir.from_serialized(c["key"], prog, {})
        assert S.enumerate_param_space(cand, budget_bytes=None) == c["space"], c["mapping"]


def test_smem_usage_of_fig1b_tiles():
    """tuner smem_usage on the Fig-1b softmax-matmul candidate: 98,560 B (test_tuner.py:30-36)."""
    prog = ir.Program("softmax_matmul", (ir.Tensor("X", (4096, 4096), "input"), ir.Tensor("W", (4096, 128), "input"),
                                         ir.Tensor("O", (4096, 128), "output")),
                      (ir.Op("exp", ("X",), "E"), ir.Op("sum", ("E",), "S", 1), ir.Op("div", ("E", "S"), "P"),
                       ir.Op("matmul", ("P", "W"), "O")), ("O",))
    N = ir.Node
    nodes = (N(0, "input", (), "X"), N(1, "input", (), "W"), N(2, "exp", (0,)), N(3, "sum", (2,), None, 1),
             N(4, "accum", (3,)), N(5, "matmul", (2, 1)), N(6, "accum", (5,)), N(7, "div", (6, 4)),
             N(8, "output", (7,), "O"))
    cand = ir.Candidate(prog, ir.Block(("x",), "i", nodes),
                        frozenset({("X", 0, "x"), ("X", 1, "i"), ("W", 0, "i"), ("O", 0, "x")}),
                        {"x": 64, "i": 64})
    assert S.smem_usage(cand) == 98560


def _exp_cand(mapping, params, rows=4):
    prog = ir.Program("just_exp", (ir.Tensor("I", (rows, 4), "input"), ir.Tensor("O", (rows, 4), "output")),
                      (ir.Op("exp", ("I",), "O"),), ("O",))
    N = ir.Node
    blk = ir.Block(("x",), "i", (N(0, "input", (), "I"), N(1, "exp", (0,)), N(2, "output", (1,), "O")))
    return ir.Candidate(prog, blk, frozenset(mapping), params)


def _compile_only(cand, ns=_abi.F64):
    return S.Plan(cand, ns, None, None)


def test_codegen_compiles_without_a_device():
    p = _compile_only(_exp_cand({("I", 0, "x"), ("O", 0, "x")}, {"x": 2, "i": 1}))
    assert p.info["logical_blocks"] == 2
    assert p.kernel_name.startswith("sgm_cand_")
    assert "sgm::NF64" in p.source()
    p.close()


def test_write_conflict_is_reported_statically():  # test_interp.py:221-227
    with pytest.raises(S.WriteConflictError):
        _compile_only(_exp_cand(set(), {"x": 2, "i": 1}))


def test_saver_region_mismatch_is_a_shape_error():  # interp.py:196-199
    # loader split by x but saver not: tile (2,4) vs region (4,4) -> ShapeError
    with pytest.raises(S.ShapeError):
        _compile_only(_exp_cand({("I", 0, "x")}, {"x": 1, "i": 1}, rows=4).with_params({"x": 2, "i": 1}))


def test_instantiate_rejects_non_power_of_two():  # graph.py:415-417
    with pytest.raises(S.DivisibilityError):
        ir.validate(_exp_cand({("I", 0, "x"), ("O", 0, "x")}, {"x": 3, "i": 1}))


def test_enumerate_space_and_empty_budget():
    cand = _exp_cand({("I", 0, "x"), ("O", 0, "x")}, {}, rows=16)
    assert S.enumerate_param_space(cand, budget_bytes=None) == [{"x": v, "i": 1} for v in (1, 2, 4, 8, 16)]
    with pytest.raises(S.EmptyParamSpaceError):
        S.tune(cand, None, backend="cost", budget_bytes=1)


def test_tune_cost_is_global_min_and_deterministic():  # test_tuner.py:90-105
    pop = P.load_population("R")
    prog = ir.Program.from_json(pop["program"])
    c = pop["candidates"][0]
    cand = ir.from_serialized(c["key"], prog, {})
    full = S.tune(cand, None, backend="cost", samples=10 ** 6, budget_bytes=None)
    scores = [S.score_cost(cand.with_params(p)) for p in c["space"]]
    assert full.score == min(scores)
    assert S.tune(cand, None, backend="cost", samples=3, seed=4, budget_bytes=None) == \
        S.tune(cand, None, backend="cost", samples=3, seed=4, budget_bytes=None)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_is_a_deterministic_partition(world):
    us = [u for w in ("R", "L") for u in P.units(P.load_population(w))]
    parts = [P.shard(us, r, world) for r in range(world)]
    keys = sorted((u.workload, u.index) for p in parts for u in p)
    assert keys == sorted((u.workload, u.index) for u in us)
    again = [P.shard(us, r, world) for r in range(world)]
    assert [[(u.workload, u.index) for u in p] for p in parts] == [[(u.workload, u.index) for u in p] for p in again]
    if world > 1:
        measured = all(u.cost_us > 0 for u in us)
        wt = (lambda u: u.cost_us) if measured else (lambda u: u.est_bytes)
        loads = [sum(wt(u) for u in p) for p in parts]
        # LPT bound: no shard exceeds the mean by more than the largest single weight
        assert max(loads) <= sum(loads) / world + max(wt(u) for u in us)


def test_scaling_prediction_from_costs():
    us = [u for w in ("R", "L") for u in P.units(P.load_population(w))]
    for k, u in enumerate(us):
        u.cost_us = 10.0 + (k * 37) % 11
        u.dep_us = 0.0                      # no refine share
    pred = P.predict_scaling(us, (2, 4, 8))
    assert 1.9 < pred["2"]["speedup"] <= 2.0 and 7.5 < pred["8"]["speedup"] <= 8.0
    assert P.predict_scaling([u for u in us[:3]] + [P.Unit(0, "R", 0, us[0].cand)], (2,)) == {}
    for u in us:
        u.dep_us = 1.0                      # the global top 3 per workload refine 1000 launches each
    pred = P.predict_scaling(us, (8,))
    assert pred["8"]["refine_ms"] == 2 * 3 * 1000 * 1.0 / 1e3 and pred["8"]["speedup"] < 8.0


def test_population_files_are_reference_searches():
    for w in ("R", "A", "Q", "L", "G16384"):
        pop = P.load_population(w)
        assert pop["search"]["stats"]["verified_pairs"] == len(pop["candidates"]) or w == "L"
        assert all(c["space"] for c in pop["candidates"]) or w == "Q"
    tot = sum(len(c["space"]) for w in P.WORKLOADS for c in P.load_population(w)["candidates"])
    assert tot > 1000


def test_sweep_report_in_reference_format(tmp_path):
    """population.report: one reference-format record per verified pair (cli.py:133-146)
    carrying the GPU evidence of its best point; DOT files per template (cli.py:205-223)."""
    from paper_2604_15272_b200 import population as P
    pop = P.load_population("L")
    us = P.units(pop)
    recs = []
    for u in us[:40]:
        r = P.Record(u.workload, u.index, u.pair, dict(u.cand.params), u.cand.mapping_list(), ff_ok=True,
                     latency_us=10.0 + u.index, plan={"kernel_name": f"k{u.index}", "summary": "s"})
        recs.append(r)
    recs[3].ff_ok = False
    rep = P.report(pop, recs, hbm_gbs=6553.3)
    assert len(rep["candidates"]) == len(pop["candidates"])
    first = rep["candidates"][us[0].pair]
    assert first["best"]["params"] == us[0].cand.params and first["b200"]["latency_us"] == 10.0
    assert abs(first["b200"]["roofline_frac"] - P.algorithmic_bytes(pop) / 10e-6 / 1e9 / 6553.3) < 1e-12
    assert rep["candidates"][us[3].pair]["oracle"]["ok"] is False
    P.write_report(rep, str(tmp_path / "r.json"))
    files = P.export_dots(pop, rep, str(tmp_path / "dots"))
    assert files and any("// b200" in open(f).read() for f in files)
