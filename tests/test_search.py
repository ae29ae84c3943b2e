"""Parallel CPU search (search.parallel_search) around the unchanged
reference: the same templates (same order), the same mapping candidates and
the same verified pairs as the sequential run_pipeline(until="verify") that
produced the committed populations (populations/make_populations.py)."""
import pytest

from conftest import reference_symfuse


@pytest.fixture(scope="module")
def ref():
    sf = reference_symfuse()
    if sf is None:
        pytest.skip("reference not installed into baseline/_ref")
    return sf


@pytest.mark.parametrize("w", ["R", "G", "A", "L", "Q"])
def test_parallel_search_equals_sequential(ref, w):
    from paper_2604_15272_b200 import optimize
    from paper_2604_15272_b200 import population as P
    pop, st = optimize.search_workload(w, workers=4)
    com = P.load_population(w)
    assert st["matches_committed"], w
    assert st["verified_pairs"] == len(com["candidates"])
    assert st["mapping_candidates"] == com["search"]["stats"]["mapping_candidates"]
    assert st["templates"] == com["search"]["stats"]["templates_emitted"]
    assert [c["key"] for c in pop["candidates"]] == [c["key"] for c in com["candidates"]]


def test_oracle_sample_is_random_equiv_tests_draw(ref, monkeypatch):
    """The e2e-opt run FF-checks, per verified pair, exactly the parameter points the
    reference's stage-4 oracle (random_equiv_test, interp.py:250-262, cli.py:162-170
    param_samples=2) would test; execution is stubbed, only the draw is compared."""
    import numpy as np
    import symfuse.interp as RI
    from symfuse.graph import deserialize
    from symfuse.workloads import lower
    from paper_2604_15272_b200 import population as P
    from paper_2604_15272_b200 import workloads as W
    pop = P.load_population("L")
    us = P.units(pop)
    picked = P.oracle_sample(pop, us)
    spec, _ = W.spec_of("L")
    program = lower(spec)
    monkeypatch.setattr(RI, "run_concrete", lambda c, ins, *a, **k: {"O": np.zeros((8, 4096))})
    monkeypatch.setattr(RI, "run_program", lambda p, ins: {"O": np.zeros((8, 4096))})
    for pi, c in enumerate(pop["candidates"]):
        g, m, _ = deserialize(c["key"], program)
        v = RI.random_equiv_test(g, m, program, trials=1, param_samples=2)
        want = {tuple(sorted(p.items())) for p in v.params_tested}
        got = {tuple(sorted(us[k].cand.params.items())) for k in picked if us[k].pair == pi}
        assert got == want, (pi, got, want)


def test_reference_arm_cpu_sample_is_uniform_and_capped(ref):
    """bench.py's CPU arm: a uniformly random sample of the whole population per
    step (not the cheapest index-0 candidates), candidates over the cap charged
    the cap (the reported CPU throughput is an upper bound)."""
    import bench
    r = bench.cpu_eval_sample(3.0, ["R", "L"], seed=1, cap_s=2.0)
    assert r["candidates"] + r["capped"] >= 1
    assert r["kind"] in ("reference", "reference+port")
    assert "uniformly at random" in r["sample"]
    assert r["value"] == r["candidates"] / r["seconds"]


def test_both_bench_arms_name_the_same_config():
    """bench.py's GPU arm and `--impl reference` print the same `config` dict (the
    workload: population, size, data); run-dependent figures and each arm's way of
    evaluating a candidate go under `method`."""
    import bench
    src = open(bench.__file__).read()
    assert src.count('"config": arm_config(') == 2
    c = bench.arm_config(["R", "G", "A", "Q", "L"])
    assert c["candidates"] == 1421 and "R,G,A,Q,L" in c["workload"]
    assert all(not isinstance(v, float) for v in c.values())
