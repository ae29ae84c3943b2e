"""The end-to-end optimisation run (BASELINE config 5) on the B200: the unchanged
reference search on host processes, cold compile into a fresh cubin cache,
the sweep with the reference's stage-4 oracle semantics, and the argmin --
for the two quickest workloads (G at 14336, LoRA)."""
import pytest

from conftest import reference_symfuse

pytestmark = pytest.mark.gpu


def test_e2e_optimisation_run_g_and_l(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    if reference_symfuse() is None:
        pytest.skip("reference not installed into baseline/_ref")
    from paper_2604_15272_b200 import _abi, optimize
    from paper_2604_15272_b200 import population as P
    run = optimize.start_search(["G", "L"], workers=4)   # forks: before this process touches CUDA
    _abi.bind_device(0)
    _abi.check(_abi.lib().sgm_set_cache_dir(str(tmp_path).encode()))
    res = optimize.evaluate_all(run, ["G", "L"], 0, None, refine_top=2)
    assert res["candidates"] == len(P.units(P.load_population("G"))) + len(P.units(P.load_population("L")))
    for w, r in res["per_workload"].items():
        assert r["matches_committed"], w
        assert r["compile_errors"] == 0 and r["ff_mismatch"] == 0, (w, r)
        assert r["ff_checked"] >= 2, w                     # the oracle sample + contenders
        win = r["winner"]
        assert win["dep_ok"] and win["ff_ok"] and win["latency_us"] > 0, (w, win)
    assert res["cold_candidates_per_s"] > 0 and res["wall_s"] > 0
