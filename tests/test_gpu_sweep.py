"""The batched candidate sweep on the B200 (population.evaluate_workload):
on-device FF verdicts agree with per-candidate checks, mutated (wrong)
candidates are refuted, and the profiler's latencies are sane."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2604_15272_b200 as S
    return S


@pytest.mark.parametrize("w,k", [("R", 12), ("L", 16), ("A", 16)])
def test_sweep_verdicts_and_latencies(S, w, k):
    from paper_2604_15272_b200 import population as P
    pop = P.load_population(w)
    us = P.units(pop)
    us = us[:: max(1, len(us) // k)][:k]
    ctx = P.WorkloadContext(pop, 0)
    recs = P.evaluate_workload(ctx, us, refine_top=2, refine_launches=64)
    assert {r.timing for r in recs} <= {"screen", "rotation", "refined"}
    assert all(r.error is None for r in recs), [r.error for r in recs if r.error]
    assert all(r.ff_ok for r in recs)
    lat = [r.latency_us for r in recs]
    assert all(x is not None and 0.5 < x < 1e5 for x in lat), lat
    assert sum(r.refined for r in recs) == min(2, sum(r.timing in ("rotation", "refined") for r in recs))
    # the batched verdicts equal the per-candidate path
    for u, r in list(zip(us, recs))[:4]:
        one = P.evaluate_unit(ctx, u, budget_us=100.0)
        assert one.ff_ok == r.ff_ok


def test_sweep_refutes_a_wrong_candidate(S):
    """A candidate whose saver map drops a grid dim writes only some cells:
    the sweep's FF check must refute it (or the plan must raise)."""
    from paper_2604_15272_b200 import ir
    from paper_2604_15272_b200 import population as P
    pop = P.load_population("R")
    prog = ir.Program.from_json(pop["program"])
    c = pop["candidates"][0]
    good = ir.from_serialized(c["key"], prog, c["space"][3])
    # swap which operand the grid splits: W columns split but O rows split -> wrong results
    bad_map = frozenset({("W", 1, "x"), ("O", 0, "x")})
    bad = ir.Candidate(prog, good.block, bad_map, dict(good.params))
    u_good = P.Unit(0, "R", 0, good)
    u_bad = P.Unit(1, "R", 0, bad)
    ctx = P.WorkloadContext(pop, 0)
    recs = P.evaluate_workload(ctx, [u_good, u_bad], refine_top=1, refine_launches=16)
    assert recs[0].ff_ok is True
    assert recs[1].error is not None or recs[1].ff_ok is False


@pytest.mark.parametrize("w,mapping,params", [
    ("G", "O.1.x,Wgate.1.x,Wup.1.x", {"x": 16, "i": 1}),
    ("A", "Kt.3.i,O.3.x,V.2.i,V.3.x", {"x": 1, "i": 1}),
    ("Q", "Kt.1.x,O.1.x,Q.1.x,V.1.x", {"x": 8, "i": 1}),
])
@pytest.mark.parametrize("hints", [{"max_cluster": 1}, {}, {"max_cluster": 8, "no_tma": 1}])
def test_split_plans_agree_exactly_in_the_field(S, w, mapping, params, hints):
    """The same candidate under different physical plans (gsplit tail reductions
    through global memory, cluster DSMEM reductions, plain loads) gives the
    program's finite-field output bit-exactly, on repeated launches (the gsplit
    counters reset themselves)."""
    import torch
    from paper_2604_15272_b200 import population as P
    from paper_2604_15272_b200.ff import ff_fill_inputs, ff_run, ff_trial_seed
    pop = P.load_population(w)
    u = next(x for x in P.units(pop) if x.cand.mapping_list() == sorted(mapping.split(",")) and x.cand.params == params)
    prog = u.cand.program
    ins = ff_fill_inputs(prog, ff_trial_seed(3, 1, 0), 0)
    exp = ff_run(S.ir.program_candidate(prog), ins, 0)
    plan = S.Plan(u.cand, 3, hints, 0)
    for _ in range(3):
        outs = [torch.empty_like(e) for e in exp]
        plan.run(ins, outs)
        for g, e in zip(outs, exp):
            assert torch.equal(g, e), (w, hints, plan.info["summary"])


@pytest.mark.parametrize("w,mapping", [("Q", "O.3.x,V.3.x"), ("A", "Kt.2.i,O.3.x,Q.3.i,V.3.x")])
@pytest.mark.parametrize("x", [2, 16, 128])
def test_x_cache_is_exact(S, w, mapping, x):
    """x-cache: nodes independent of the grid coordinate (the attention scores when
    only V/O's head dim is split) are kept across a CTA's consecutive items and
    recomputed only when the other coordinates change.  FF bit-exact against the
    program (twice: cache state across launches), deployment dtype against the
    fp64 oracle."""
    import torch
    from oracle import block_np
    from paper_2604_15272_b200 import population as P
    from paper_2604_15272_b200.ff import ff_fill_inputs, ff_run, ff_trial_seed
    pop = P.load_population(w)
    u = next(v for v in P.units(pop) if v.cand.mapping_list() == sorted(mapping.split(","))
             and v.cand.params == {"x": x, "i": 1})
    prog = u.cand.program
    ins = ff_fill_inputs(prog, ff_trial_seed(9, x, 0), 0)
    exp = ff_run(S.ir.program_candidate(prog), ins, 0)
    plan = S.Plan(u.cand, 3, None, 0)
    assert "xc_miss" in plan.source()
    for _ in range(2):
        outs = [torch.empty_like(e) for e in exp]
        plan.run(ins, outs)
        assert all(torch.equal(a, b) for a, b in zip(outs, exp)), (w, x)
    dt = pop["dtype"]
    assert "xc_miss" in S.Plan(u.cand, 2, None, None).source()
    rng = np.random.default_rng(31)
    progd = pop["program"]
    ins_d = {t["name"]: torch.from_numpy(rng.standard_normal(tuple(t["dims"]))).bfloat16().double().numpy()
             for t in progd["tensors"] if t["role"] == "input"}
    ref = block_np.run_program(progd, ins_d)
    got = S.run_concrete(u.cand, ins_d, dtype=dt)
    assert S.rel_err(got["O"], ref["O"]) < 1e-2, (w, x)


@pytest.mark.parametrize("w,mapping,params", [
    ("A", "Kt.3.i,O.3.x,V.2.i,V.3.x", {"x": 16, "i": 2048}),
    ("A", "Kt.3.i,O.3.x,V.2.i,V.3.x", {"x": 16, "i": 4096}),
    ("A", "Kt.3.i,O.3.x,V.2.i,V.3.x", {"x": 1, "i": 8192}),
    ("L", "A.0.i,B.1.x,O.1.x,W.0.i,W.1.x,X.1.i", {"x": 256, "i": 2048}),
])
def test_loop_prefetch_is_exact(S, w, mapping, params):
    """Loop-body tiles prefetched into registers one iteration ahead (TilePf):
    FF bit-exact against the program with and without the prefetch, the
    deployment dtype against the fp64 oracle."""
    import torch
    from oracle import block_np
    from paper_2604_15272_b200 import population as P
    from paper_2604_15272_b200.ff import ff_fill_inputs, ff_run, ff_trial_seed
    pop = P.load_population(w)
    u = next(v for v in P.units(pop) if v.cand.mapping_list() == sorted(mapping.split(",")) and v.cand.params == params)
    prog = u.cand.program
    ins = ff_fill_inputs(prog, ff_trial_seed(11, 2, 0), 0)
    exp = ff_run(S.ir.program_candidate(prog), ins, 0)
    for hints in (None, {"no_prefetch": 1}):
        plan = S.Plan(u.cand, 3, hints, 0)
        src = plan.source()
        assert ("TilePf" in src or "TileStrip" in src) == (hints is None)
        if w == "A" and hints is None:
            assert "TileStrip" in src  # Kt's columns per key come from 16-byte row strips
        for _ in range(2):
            outs = [torch.empty_like(e) for e in exp]
            plan.run(ins, outs)
            assert all(torch.equal(a, b) for a, b in zip(outs, exp)), (w, params, hints)
    # the generated kernels assume 16-byte aligned bases: a misaligned one is refused
    buf = torch.empty(ins[0].numel() + 1, dtype=ins[0].dtype, device=ins[0].device)
    with pytest.raises(ValueError, match="16-byte aligned"):
        S.Plan(u.cand, 3, None, 0).run([buf[1:].view(ins[0].shape)] + list(ins[1:]), outs)
    rng = np.random.default_rng(37)
    progd = pop["program"]
    ins_d = {t["name"]: torch.from_numpy(rng.standard_normal(tuple(t["dims"]))).bfloat16().double().numpy()
             for t in progd["tensors"] if t["role"] == "input"}
    ref = block_np.run_program(progd, ins_d)
    got = S.run_concrete(u.cand, ins_d, dtype=pop["dtype"])
    assert S.rel_err(got["O"], ref["O"]) < 1e-2, (w, params)
