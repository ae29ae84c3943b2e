"""Deployment-dtype numerics of generated kernels (bf16 with fp32 accumulation,
fp32) against the fp64 oracle on the same (rounded) inputs.

Tolerances (stated in DESIGN.md):
  bf16 storage / fp32 compute:  rel_err <= 1e-2   (output rounding 2^-8 + bf16 MMA operands)
  fp32:                         rel_err <= 1e-5
rel_err = max|a-b| / (1 + max|b|) as in the reference (interp.py:228-231)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"bf16": 1e-2, "f32": 1e-5}


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2604_15272_b200 as S
    return S


def _round(x, dtype):
    import torch
    t = torch.from_numpy(x)
    if dtype == "bf16":
        t = t.to(torch.bfloat16)
    elif dtype == "f32":
        t = t.to(torch.float32)
    return t.to(torch.float64).numpy()


def _gemv_program(S, M, K, N):
    T = S.ir.Tensor
    return S.ir.Program("gemv", (T("X", (M, K), "input"), T("W", (K, N), "input"), T("O", (M, N), "output")),
                        (S.ir.Op("matmul", ("X", "W"), "O"),), ("O",))


@pytest.mark.parametrize("M,K,N,x", [(8, 4096, 14336, 16), (8, 4096, 14336, 128), (2, 512, 896, 1), (8, 4096, 4096, 32),
                                     (4, 1024, 1024, 8), (1, 256, 64, 1), (16, 512, 256, 2)])
def test_streamed_matmul_bf16(S, M, K, N, x):
    """Column-split X.W: the tcgen05 GEMV (full and partial 128-column tiles)."""
    prog = _gemv_program(S, M, K, N)
    N_ = S.ir.Node
    blk = S.ir.Block(("x",), "i", (N_(0, "input", (), "X"), N_(1, "input", (), "W"), N_(2, "matmul", (0, 1)),
                                   N_(3, "output", (2,), "O")))
    cand = S.ir.Candidate(prog, blk, frozenset({("W", 1, "x"), ("O", 1, "x")}), {"x": x, "i": 1})
    rng = np.random.default_rng(M * 1000 + N)
    X = _round(rng.standard_normal((M, K)), "bf16")
    W = _round(rng.standard_normal((K, N)), "bf16")
    got = S.run_concrete(cand, {"X": X, "W": W}, dtype="bf16")["O"]
    ref = X @ W
    assert S.rel_err(got, ref) < TOL["bf16"], S.rel_err(got, ref)
    if K * N >= 4096 * 4096:  # large enough that every plan streams 128-column tiles through tcgen05
        assert S.Plan(cand, 2, None, 0).info["n_tcgen05"] == 1


@pytest.mark.parametrize("M,K,N,x", [(8, 4096, 4096, 128), (8, 4096, 4096, 1), (2, 512, 512, 16), (4, 1024, 256, 32),
                                     (8, 256, 64, 8), (1, 128, 512, 4)])
def test_streamed_matmul_f32(S, M, K, N, x):
    """Column-split X.W in fp32: the TMA-ring CUDA-core consumer (box widths 8..64)."""
    prog = _gemv_program(S, M, K, N)
    N_ = S.ir.Node
    blk = S.ir.Block(("x",), "i", (N_(0, "input", (), "X"), N_(1, "input", (), "W"), N_(2, "matmul", (0, 1)),
                                   N_(3, "output", (2,), "O")))
    cand = S.ir.Candidate(prog, blk, frozenset({("W", 1, "x"), ("O", 1, "x")}), {"x": x, "i": 1})
    rng = np.random.default_rng(M * 1000 + N + 7)
    X = _round(rng.standard_normal((M, K)), "f32")
    W = _round(rng.standard_normal((K, N)), "f32")
    got = S.run_concrete(cand, {"X": X, "W": W}, dtype="f32")["O"]
    assert S.rel_err(got, X @ W) < TOL["f32"], S.rel_err(got, X @ W)
    if K * N >= 4096 * 4096:
        assert "tma-f32" in S.Plan(cand, 1, None, 0).info["summary"]


def _population_cases(S, w, k):
    from paper_2604_15272_b200 import population as P
    pop = P.load_population(w)
    us = P.units(pop)
    step = max(1, len(us) // k)
    return pop, us[::step][:k]


@pytest.mark.parametrize("w,k", [("G", 8), ("L", 12), ("A", 12), ("Q", 8), ("R", 8)])
def test_population_candidates_deployment_dtype(S, w, k):
    from oracle import block_np
    pop, us = _population_cases(S, w, k)
    dt = pop["dtype"]
    rng = np.random.default_rng(5)
    prog = pop["program"]
    ins = {t["name"]: _round(rng.standard_normal(tuple(t["dims"])), dt) for t in prog["tensors"] if t["role"] == "input"}
    exp = block_np.run_program(prog, ins)
    for u in us:
        got = S.run_concrete(u.cand, ins, dtype=dt)
        for name in prog["outputs"]:
            err = S.rel_err(got[name], exp[name])
            assert err < TOL[dt], (w, u.index, u.cand.mapping_list(), u.cand.params, err)


def test_best_kernels_deployment_dtype(S):
    """The per-workload winners recorded in profiles/best_kernels.json (if present)."""
    import json
    import os
    from oracle import block_np
    from paper_2604_15272_b200 import population as P
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "best_kernels.json")
    if not os.path.exists(path):
        pytest.skip("no recorded winners yet")
    best = json.load(open(path))
    for w, b in best.items():
        pop = P.load_population(w)
        u = next(x for x in P.units(pop) if x.cand.mapping_list() == b["mapping"] and x.cand.params == b["params"]
                 and pop["candidates"][x.pair]["template_id"] == b.get("template", pop["candidates"][x.pair]["template_id"]))
        dt = pop["dtype"]
        rng = np.random.default_rng(11)
        prog = pop["program"]
        ins = {t["name"]: _round(rng.standard_normal(tuple(t["dims"])), dt) for t in prog["tensors"]
               if t["role"] == "input"}
        exp = block_np.run_program(prog, ins)
        hints = b.get("hints") or None
        got = S.run_concrete(u.cand, ins, dtype=dt, hints=hints)
        for name in prog["outputs"]:
            assert S.rel_err(got[name], exp[name]) < TOL[dt], w


@pytest.mark.parametrize("w,template,mapping,params", [
    ("R", 26, "O.1.x,W.1.x", {"x": 2, "i": 1}),   # RMS statistic reduced across a cluster mid-kernel
    ("G", 0, "O.1.x,Wgate.1.x,Wup.1.x", {"x": 8, "i": 1}),
    ("A", 42, "Kt.1.x,O.1.x,Q.1.x,V.1.x", {"x": 2, "i": 1}),
])
@pytest.mark.parametrize("hints", [{}, {"one_cta": 1}, {"max_cluster": 4, "max_gsplit": 1}, {"max_cluster": 1},
                                   {"variant": 2}])
def test_physical_plan_variants_deployment_dtype(S, w, template, mapping, params, hints):
    """One candidate under the physical plans the tuner picks between: two CTAs per
    SM (tcgen05, TMEM halves), one per SM, cluster reductions (one-barrier push for
    small partials, reduce-scatter for large), gsplit tail reductions."""
    from oracle import block_np
    from paper_2604_15272_b200 import population as P
    pop = P.load_population(w)
    u = next(x for x in P.units(pop) if x.cand.mapping_list() == sorted(mapping.split(",")) and x.cand.params == params
             and pop["candidates"][x.pair]["template_id"] == template)
    dt = pop["dtype"]
    rng = np.random.default_rng(13)
    prog = pop["program"]
    ins = {t["name"]: _round(rng.standard_normal(tuple(t["dims"])), dt) for t in prog["tensors"] if t["role"] == "input"}
    exp = block_np.run_program(prog, ins)
    got = S.run_concrete(u.cand, ins, dtype=dt, hints=hints)
    got2 = S.run_concrete(u.cand, ins, dtype=dt, hints=hints)  # second launch: self-resetting counters, buffer parity
    for name in prog["outputs"]:
        assert S.rel_err(got[name], exp[name]) < TOL[dt], (w, hints)
        assert np.array_equal(np.asarray(got[name]), np.asarray(got2[name])), (w, hints)


@pytest.mark.parametrize("params", [{"x": 32, "i": 1}, {"x": 2, "i": 1}, {"x": 8, "i": 1}])
@pytest.mark.parametrize("hints", [{"interleave": 1, "one_cta": 1}, {"interleave": 1, "one_cta": 1, "no_wd": 1},
                                   {"interleave": 1, "one_cta": 1, "slot_kb": 16}])
def test_interleaved_stream_deployment_dtype(S, params, hints):
    """LoRA with the big stream (X@W) split around the small chain (X@A -> T@B):
    first ring-full of W issued ahead of the chain, chain MMAs in their own TMEM
    columns, the rest of W after it; bf16 against the fp64 oracle, twice (ring
    and TMEM state carried across launches)."""
    from oracle import block_np
    from paper_2604_15272_b200 import population as P
    pop = P.load_population("L")
    u = next(x for x in P.units(pop) if x.cand.mapping_list() == ["B.1.x", "O.1.x", "W.1.x"]
             and x.cand.params == params and pop["candidates"][x.pair]["template_id"] == 4)
    assert ", false>(t" in S.Plan(u.cand, 2, hints, None).source()  # the stream really is segmented
    rng = np.random.default_rng(23)
    prog = pop["program"]
    ins = {t["name"]: _round(rng.standard_normal(tuple(t["dims"])), "bf16") for t in prog["tensors"]
           if t["role"] == "input"}
    exp = block_np.run_program(prog, ins)
    for _ in range(2):
        got = S.run_concrete(u.cand, ins, dtype="bf16", hints=hints)
        assert S.rel_err(got["O"], exp["O"]) < TOL["bf16"], (params, hints)


@pytest.mark.parametrize("params", [{"x": 32, "i": 1}, {"x": 2, "i": 1}, {"x": 8, "i": 1}])
@pytest.mark.parametrize("hints", [{"one_cta": 1}, {}, {"one_cta": 1, "slot_kb": 16, "no_wd": 1}])
def test_accumulate_into_deployment_dtype(S, params, hints):
    """LoRA's T@B issued into X@W's TMEM accumulators (accumulate-into fusion: one
    read-back gives X@W + T@B, the add becomes a copy), bf16 vs the fp64 oracle."""
    from oracle import block_np
    from paper_2604_15272_b200 import population as P
    pop = P.load_population("L")
    u = next(x for x in P.units(pop) if x.cand.mapping_list() == ["B.1.x", "O.1.x", "W.1.x"]
             and x.cand.params == params and pop["candidates"][x.pair]["template_id"] == 4)
    src = S.Plan(u.cand, 2, hints or None, None).source()
    assert ", false>(t" in src and "true, 1>(t" in src  # T@B without read-back, X@W with PRE = 1
    rng = np.random.default_rng(29)
    prog = pop["program"]
    ins = {t["name"]: _round(rng.standard_normal(tuple(t["dims"])), "bf16") for t in prog["tensors"]
           if t["role"] == "input"}
    exp = block_np.run_program(prog, ins)
    for _ in range(2):
        got = S.run_concrete(u.cand, ins, dtype="bf16", hints=hints or None)
        assert S.rel_err(got["O"], exp["O"]) < TOL["bf16"], (params, hints)
