"""Parity at the configs' full scale (BASELINE R/G/A/Q/L shapes).

1. Finite field: the device program and split candidates of every workload are
   bit-exact against the CPU oracle (oracle/ff_np, itself pinned to the
   reference's control flow by tests/test_oracle.py) on full-size inputs, so a
   defect shared by the device program and the device candidate (e.g. in a
   K = 4096 / 8192 / 14336 contraction) cannot hide behind device-vs-device checks.
2. Deployment dtype: the top 8 of a FRESH sweep per workload (evaluate_workload
   run here, not a committed list), and the physical plan tune_physical picks
   for the best of them, against the fp64 oracle on the same rounded inputs.
   Tolerances: bf16 storage / fp32 accumulation 1e-2, fp32 1e-5.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"bf16": 1e-2, "f32": 1e-5}
WORKLOADS = ("R", "G", "A", "Q", "L")


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2604_15272_b200 as S
    return S


def _split_units(us):
    """Two split candidates per workload: the one with the most loop parts
    (a for-loop split, if any) and the one with the most grid blocks."""
    def grid(u):
        g = 1
        for q in u.cand.block.grid:
            g *= u.cand.params[q]
        return g
    loop = max(us, key=lambda u: (u.cand.params[u.cand.block.loop], grid(u), -u.index))
    wide = max(us, key=lambda u: (grid(u), -u.index))
    return [loop] if loop is wide else [loop, wide]


@pytest.mark.parametrize("w", WORKLOADS)
def test_full_scale_ff_bit_exact_vs_oracle(S, w):
    from oracle import block_np, ff_np
    from paper_2604_15272_b200 import population as P
    from paper_2604_15272_b200.ff import ff_fill_inputs, ff_run, ff_trial_seed
    pop = P.load_population(w)
    prog = S.ir.Program.from_json(pop["program"])
    dev_in = ff_fill_inputs(prog, ff_trial_seed(7, 0xF011 + WORKLOADS.index(w), 0), 0)
    host_in = {n: x.cpu().numpy().astype(np.int64) for n, x in zip(prog.inputs, dev_in)}
    exp = block_np.run_program(pop["program"], host_in, arith=ff_np.FFArith())
    got = ff_run(S.ir.program_candidate(prog), dev_in, 0)
    for n, g in zip(prog.outputs, got):
        assert np.array_equal(g.cpu().numpy().astype(np.int64), exp[n]), (w, "program", n)
    for u in _split_units(P.units(pop)):
        got = ff_run(u.cand, dev_in, 0)
        for n, g in zip(prog.outputs, got):
            assert np.array_equal(g.cpu().numpy().astype(np.int64), exp[n]), (w, u.cand.mapping_list(), u.cand.params)


def _round(x, dtype):
    import torch
    t = torch.from_numpy(x)
    t = t.to(torch.bfloat16) if dtype == "bf16" else t.to(torch.float32)
    return t.to(torch.float64).numpy()


@pytest.mark.parametrize("w", WORKLOADS)
def test_fresh_sweep_top8_deployment_dtype_vs_oracle(S, w):
    import torch
    from oracle import block_np
    from paper_2604_15272_b200 import _abi
    from paper_2604_15272_b200 import population as P
    pop = P.load_population(w)
    us = P.units(pop)
    us = us[:: max(1, len(us) // 48)]
    P.precompile([u.cand for u in us], [P.numsys_of(pop["dtype"]), _abi.FF], 0)
    ctx = P.WorkloadContext(pop, 0)
    recs = P.evaluate_workload(ctx, us, refine_top=3, refine_launches=64)
    ok = sorted((r for r in recs if r.error is None and r.latency_us and r.ff_ok), key=lambda r: (r.latency_us, r.index))
    assert len(ok) >= min(8, len(us)) // 2, [r.error for r in recs if r.error][:3]
    by_index = {u.index: u for u in us}
    dt = pop["dtype"]
    rng = np.random.default_rng(17)
    progd = pop["program"]
    ins = {t["name"]: _round(rng.standard_normal(tuple(t["dims"])), dt) for t in progd["tensors"] if t["role"] == "input"}
    exp = block_np.run_program(progd, ins)
    for r in ok[:8]:
        got = S.run_concrete(by_index[r.index].cand, ins, dtype=dt)
        for n in progd["outputs"]:
            err = S.rel_err(got[n], exp[n])
            assert err < TOL[dt], (w, r.index, r.mapping, r.params, err)
        if r.dep_ok is not None:  # the sweep's own gate agrees with the oracle
            assert r.dep_ok and r.dep_err < TOL[dt], (w, r.index, r.dep_err)
    # the physical plan the best-kernel phase would report for the winner
    win = by_index[ok[0].index]
    lat, hints, plan = P.tune_physical(ctx, win, launches=64)
    got = S.run_concrete(win.cand, ins, dtype=dt, hints=hints or None)
    for n in progd["outputs"]:
        assert S.rel_err(got[n], exp[n]) < TOL[dt], (w, hints)
    (err, good), = P.deployment_check(ctx, [plan])
    assert good and err < TOL[dt], (w, hints, err)
    assert P.ff_check_plan(ctx, win.cand, hints), (w, hints)
    torch.cuda.synchronize()
