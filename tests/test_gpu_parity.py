"""GPU parity: the generated sm_100a kernels vs the reference's golden fixtures
and the oracle.  Bars: fp64 rel_err < 1e-12 (the reference's own pin,
test_interp.py:173); finite field bit-exact; verdicts identical."""
import numpy as np
import pytest

from conftest import case_inputs_f64, case_inputs_ff

pytestmark = pytest.mark.gpu

# fp64: the reference pins run_concrete at 1e-12 (test_interp.py:173) against its own
# numpy summation order; split plans sum partials in another order, and exp() of
# N(0,1) sums reaches ~1e90 in the attention fixtures, so reassociation costs a few ulps
F64_TOL = 1e-11


@pytest.fixture(scope="module")
def S(desk_cases):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2604_15272_b200 as S
    from paper_2604_15272_b200 import population as P
    # compile every fixture kernel up front on all host cores (NVRTC is thread-safe)
    cands = []
    for c in desk_cases:
        if c.get("instantiate_error"):
            continue
        prog = S.ir.Program.from_json(c["program"])
        cands.append(S.ir.from_serialized(c["key"], prog, c["params"]))
        cands.append(S.ir.program_candidate(prog))
    P.precompile(cands, [0, 3], None)
    return S


def _cand(S, c):
    prog = S.ir.Program.from_json(c["program"])
    return S.ir.from_serialized(c["key"], prog, c["params"])


def test_f64_run_concrete_matches_reference(S, desk_cases, desk_arrays):
    n = 0
    for c in desk_cases:
        if not c.get("stored") or c.get("f64_error") or c.get("instantiate_error"):
            continue
        got = S.run_concrete(_cand(S, c), case_inputs_f64(c))
        for name, arr in got.items():
            ref = desk_arrays[f"c{c['id']}_f64_{name}"]
            if np.isfinite(ref).all():
                assert S.rel_err(arr, ref) < F64_TOL, (c["id"], c["workload"], name, S.rel_err(arr, ref))
            else:
                assert np.array_equal(np.isnan(arr), np.isnan(ref)), c["id"]
        n += 1
    assert n >= 150


def test_ff_bit_exact_with_reference(S, desk_cases, desk_arrays):
    n = 0
    for c in desk_cases:
        if not c.get("stored") or c.get("ff_error") or c.get("instantiate_error"):
            continue
        ins = case_inputs_ff(c)
        got = S.run_concrete(_cand(S, c), ins, dtype="ff")
        exp = S.run_program(S.ir.Program.from_json(c["program"]), ins, dtype="ff")
        for name in c["program"]["outputs"]:
            assert np.array_equal(got[name], desk_arrays[f"c{c['id']}_ff_{name}"]), (c["id"], c["workload"], name)
            assert np.array_equal(exp[name], desk_arrays[f"c{c['id']}_ffprog_{name}"]), (c["id"], name)
        n += 1
    assert n >= 150


def test_run_program_f64_matches_oracle(S, desk_cases):
    from oracle import block_np
    seen = set()
    for c in desk_cases:
        if c["workload"] in seen:
            continue
        seen.add(c["workload"])
        ins = case_inputs_f64(c)
        got = S.run_program(S.ir.Program.from_json(c["program"]), ins)
        exp = block_np.run_program(c["program"], ins)
        for k in exp:
            assert S.rel_err(got[k], exp[k]) < F64_TOL


def test_random_equiv_verdicts_match_reference(S, desk_cases):
    """Device random_equiv_test (fp64, same RNG streams) == reference verdicts."""
    done = set()
    for c in desk_cases:
        key = (c["workload"], c["key"])
        if key in done or c.get("instantiate_error"):
            continue
        done.add(key)
        prog = S.ir.Program.from_json(c["program"])
        cand = S.ir.from_serialized(c["key"], prog, {})
        v = S.random_equiv_test(cand, None, prog, trials=3, param_samples=2, seed=0)
        assert v.ok == c["ref_verdict"]["ok"], (c["id"], c["workload"], v, c["ref_verdict"])
        assert v.trials == c["ref_verdict"]["trials"]


def test_ff_verdicts_agree(S, desk_cases):
    done = set()
    for c in desk_cases:
        key = (c["workload"], c["key"])
        if key in done or c.get("instantiate_error"):
            continue
        done.add(key)
        prog = S.ir.Program.from_json(c["program"])
        cand = S.ir.from_serialized(c["key"], prog, {})
        v = S.ff_equiv_test(cand, None, prog, trials=1, param_samples=2, seed=0)
        assert v.ok == c["ref_verdict"]["ok"], (c["id"], c["workload"], v)


# ---- known-answer tests restated from the reference suite (test_interp.py) -----

def _prog(S, tensors, ops, outputs, name="p"):
    from fractions import Fraction  # noqa: F401
    return S.ir.Program(name, tuple(S.ir.Tensor(*t) for t in tensors), tuple(S.ir.Op(*o) for o in ops),
                        tuple(outputs))


def _softmax_matmul(S, rows, cols, oc):
    return _prog(S, [("X", (rows, cols), "input"), ("W", (cols, oc), "input"), ("O", (rows, oc), "output")],
                 [("exp", ("X",), "E"), ("sum", ("E",), "S", 1), ("div", ("E", "S"), "P"), ("matmul", ("P", "W"), "O")],
                 ["O"], "softmax_matmul")


def _known_good(S, prog, params):
    N = S.ir.Node
    nodes = (N(0, "input", (), "X"), N(1, "input", (), "W"), N(2, "exp", (0,)), N(3, "sum", (2,), None, 1),
             N(4, "accum", (3,)), N(5, "matmul", (2, 1)), N(6, "accum", (5,)), N(7, "div", (6, 4)),
             N(8, "output", (7,), "O"))
    on = frozenset({("X", 0, "x"), ("X", 1, "i"), ("W", 0, "i"), ("O", 0, "x")})
    return S.ir.Candidate(prog, S.ir.Block(("x",), "i", nodes), on, params)


def test_softmax_uniform_rows(S):  # test_interp.py:134-141
    out = S.run_program(_softmax_matmul(S, 4, 4, 2), {"X": np.ones((4, 4)), "W": np.ones((4, 2))})["O"]
    assert np.allclose(out, 1.0)


def test_hand_value(S):  # test_interp.py:159-162
    out = S.run_program(_softmax_matmul(S, 2, 2, 1), {"X": np.zeros((2, 2)), "W": np.array([[1.0], [2.0]])})["O"]
    assert np.allclose(out, [[1.5], [1.5]])


@pytest.mark.parametrize("params", [{"x": 4, "i": 4}, {"x": 1, "i": 1}, {"x": 2, "i": 8}, {"x": 128, "i": 128}])
def test_block_equals_program(S, params):  # test_interp.py:165-184
    prog = _softmax_matmul(S, 128, 128, 32)
    cand = _known_good(S, prog, params)
    rng = np.random.default_rng(7)
    ins = {"X": rng.standard_normal((128, 128)), "W": rng.standard_normal((128, 32))}
    assert S.rel_err(S.run_concrete(cand, ins)["O"], S.run_program(prog, ins)["O"]) < F64_TOL


def _exp_graph(S, good=True):
    prog = _prog(S, [("I", (4, 4), "input"), ("O", (4, 4), "output")], [("exp", ("I",), "O")], ["O"], "just_exp")
    N = S.ir.Node
    blk = S.ir.Block(("x",), "i", (N(0, "input", (), "I"), N(1, "exp", (0,)), N(2, "output", (1,), "O")))
    on = frozenset({("I", 0, "x"), ("O", 0, "x")}) if good else frozenset()
    return S.ir.Candidate(prog, blk, on, {"x": 2, "i": 1})


def test_exp_row_blocks(S):  # test_interp.py:213-218
    x = np.arange(16.0).reshape(4, 4)
    assert np.allclose(S.run_concrete(_exp_graph(S), {"I": x})["O"], np.exp(x))


def test_write_conflict_detected(S):  # test_interp.py:221-227
    with pytest.raises(S.WriteConflictError):
        S.run_concrete(_exp_graph(S, good=False), {"I": np.ones((4, 4))})


def test_input_shape_error(S):  # interp.py:142-144
    with pytest.raises(S.ShapeError):
        S.run_concrete(_exp_graph(S), {"I": np.ones((4, 2))})


def test_unwritten_cells_stay_nan(S):
    # saver covers only half of O when its map is narrower than the tile
    prog = _prog(S, [("I", (4, 4), "input"), ("O", (4, 4), "output")], [("exp", ("I",), "O")], ["O"])
    N = S.ir.Node
    blk = S.ir.Block(("x",), "i", (N(0, "input", (), "I"), N(1, "exp", (0,)), N(2, "output", (1,), "O")))
    cand = S.ir.Candidate(prog, blk, frozenset({("I", 0, "x"), ("O", 0, "x")}), {"x": 1, "i": 1})
    out = S.run_concrete(cand, {"I": np.zeros((4, 4))})["O"]
    assert np.allclose(out, 1.0)


def test_torch_tensors_zero_copy(S):
    import torch
    prog = _softmax_matmul(S, 64, 64, 16)
    cand = _known_good(S, prog, {"x": 4, "i": 2})
    ins = {"X": torch.randn(64, 64, dtype=torch.float64, device="cuda"),
           "W": torch.randn(64, 16, dtype=torch.float64, device="cuda")}
    got = S.run_concrete(cand, ins)["O"]
    assert got.is_cuda
    ref = torch.softmax(ins["X"], 1) @ ins["W"]
    assert (got - ref).abs().max().item() < 1e-12


def test_tile_dump_exposes_per_block_values(S):  # test_integration.py:72-85
    prog = _softmax_matmul(S, 64, 64, 16)
    cand = _known_good(S, prog, {"x": 2, "i": 2})
    rng = np.random.default_rng(0)
    dump: dict = {}
    S.run_concrete(cand, {"X": rng.standard_normal((64, 64)), "W": rng.standard_normal((64, 16))}, tile_dump=dump)
    assert set(dump) == {(0,), (1,)}
    assert dump[(0,)][0].shape == (32, 32)  # X tile of block 0


def test_tile_dump_matches_oracle(S, desk_cases):
    """Every node's per-block tile (last loop iteration / accumulated sum /
    epilogue loaders on their last tile) against the CPU oracle's tile_dump,
    fp64 and finite field, on golden cases with grid and loop splits."""
    from oracle import block_np, ff_np
    n = 0
    for c in desk_cases:
        if c.get("instantiate_error") or c.get("f64_error") or c.get("ff_error"):
            continue
        grid = 1
        for q, v in c["params"].items():
            grid *= v
        if grid < 4 or n >= 12:
            continue
        cand = _cand(S, c)
        for dt, ins, arith in (("f64", case_inputs_f64(c), None), ("ff", case_inputs_ff(c), ff_np.FFArith())):
            got, ref = {}, {}
            S.run_concrete(cand, ins, dtype=dt, tile_dump=got)
            block_np.run_concrete(c["program"], c["key"], c["params"], ins, arith=arith, tile_dump=ref)
            assert set(got) == set(ref), c["id"]
            for coords, env in ref.items():
                assert set(got[coords]) == set(env), (c["id"], coords)
                for idx, tile in env.items():
                    g = np.asarray(got[coords][idx])
                    assert g.shape == tile.shape, (c["id"], coords, idx)
                    if dt == "ff":
                        assert np.array_equal(g.astype(np.int64), tile), (c["id"], coords, idx)
                    elif np.isfinite(tile).all():
                        assert S.rel_err(g, tile) < F64_TOL, (c["id"], coords, idx)
        n += 1
    assert n >= 8


@pytest.mark.parametrize("w", ["R", "G", "L"])
def test_ff_through_the_tma_ring_is_bit_exact(S, w):
    """hints.ff_tma: finite-field residues streamed through the TMA ring into the
    CUDA-core consumer (u64 lazy-reduced accumulators) give the program's FF
    output bit-exactly, repeatedly, at full scale."""
    import torch
    from paper_2604_15272_b200 import population as P
    from paper_2604_15272_b200.ff import ff_fill_inputs, ff_run, ff_trial_seed
    pop = P.load_population(w)
    us = P.units(pop)
    prog = us[0].cand.program
    ins = ff_fill_inputs(prog, ff_trial_seed(5, 77, 0), 0)
    exp = ff_run(S.ir.program_candidate(prog), ins, 0)
    n = 0
    for u in us[:: max(1, len(us) // 6)]:
        plan = S.Plan(u.cand, 3, {"ff_tma": 1}, 0)
        if "mm_stream_f32<N" not in plan.source():
            continue
        n += 1
        for _ in range(2):
            outs = [torch.empty_like(e) for e in exp]
            plan.run(ins, outs)
            assert all(torch.equal(a, b) for a, b in zip(outs, exp)), (w, u.cand.params)
    assert n >= 1
