"""The plugin seam: install() rebinds the unmodified reference's executor
(symfuse interp.py:277,279; tuner.py:162; cli.py:182) to the B200 backend."""
import numpy as np
import pytest

from conftest import reference_symfuse


@pytest.fixture()
def ref():
    sf = reference_symfuse()
    if sf is None:
        pytest.skip("reference not installed into baseline/_ref")
    from paper_2604_15272_b200 import integrate
    integrate.install(sf)
    yield sf
    integrate.uninstall()


def _softmax_case(sf, n=64, oc=16):
    from symfuse.graph import TensorSpec
    from symfuse.workloads import BUILTINS
    spec = BUILTINS["softmax_matmul"]()
    spec.scale = {"X": (n, n), "W": (n, oc), "O": (n, oc)}
    return spec


def test_install_rebinds_and_restores(ref):
    import symfuse.cli as RC
    import symfuse.interp as RI
    import symfuse.tuner as RT
    from paper_2604_15272_b200 import integrate
    assert hasattr(RI.run_concrete, "__wrapped__")
    assert RT.tune is RC.tune
    integrate.uninstall()
    assert not hasattr(RI.run_concrete, "__wrapped__")
    integrate.install(ref)


def test_reference_oracle_routes_through_backend_cpu(ref):
    """Without a GPU the reference's own random_equiv_test now fails loudly
    (BackendUnavailable), proving no silent CPU execution remains on the seam."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by test_reference_pipeline_on_b200")
    from symfuse.cli import PipelineFlags, run_pipeline
    from paper_2604_15272_b200 import BackendUnavailable
    with pytest.raises(BackendUnavailable):
        run_pipeline(_softmax_case(ref), PipelineFlags(trials=1, param_samples=1, backend="b200"))


@pytest.mark.gpu
def test_reference_pipeline_on_b200(ref):
    """The reference's unchanged run_pipeline, stage 4 on the B200: every
    verified pair passes the (device fp64) oracle and tunes with backend b200."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from symfuse.cli import PipelineFlags, run_pipeline
    rep = run_pipeline(_softmax_case(ref), PipelineFlags(trials=2, param_samples=2, backend="b200"))
    recs = [r for r in rep["candidates"] if r["verified"]]
    assert recs
    for r in recs:
        assert r["oracle"]["ok"], r
        assert r["best"]["score"] is None or r["best"]["score"] > 0


def test_cli_accepts_backend_b200(ref):
    """install() adds "b200" to the reference CLI's --backend choices (cli.py:255)."""
    import symfuse.cli as RC
    args = RC.build_parser().parse_args(["search", "--workload", "rmsnorm", "--backend", "b200"])
    assert args.backend == "b200"
    from paper_2604_15272_b200 import integrate
    integrate.uninstall()
    with pytest.raises(SystemExit):
        RC.build_parser().parse_args(["search", "--workload", "rmsnorm", "--backend", "b200"])
    integrate.install(ref)


def _qk_spec(sf):
    from symfuse.workloads import BUILTINS
    spec = BUILTINS["qk_attention"]()
    spec.scale = {"Q": (8, 8, 4, 128), "Kt": (8, 8, 128, 8192), "V": (8, 8, 8192, 128), "O": (8, 8, 4, 128)}
    return spec


def test_b200_resource_model_fills_the_q_spaces(ref):
    """under the reference's 164 KiB / 2-byte budget every verified
    QK-attention pair at full scale has an EMPTY space; the B200 resource model
    (planner feasibility, no compile, no device) keeps points for all of them."""
    from symfuse.graph import deserialize
    from symfuse.tuner import DEFAULT_BUDGET
    from symfuse.tuner import enumerate_param_space as ref_space
    from symfuse.workloads import lower
    from paper_2604_15272_b200 import population as P
    from paper_2604_15272_b200.tuner import B200_BUDGET, enumerate_param_space
    pop = P.load_population("Q")
    spec = _qk_spec(ref)
    program = lower(spec)
    for c in pop["candidates"][:8]:
        g, m, _ = deserialize(c["key"], program)
        assert ref_space(g, m, DEFAULT_BUDGET) == []
        sp = enumerate_param_space(g, m, budget_bytes=B200_BUDGET, dtype="bf16")
        assert sp and all(p in c["space"] for p in sp)


@pytest.mark.gpu
def test_reference_pipeline_q_scale_tunes_every_pair_in_bf16(ref):
    """The reference's unchanged run_pipeline on QK-attention at the Q config's
    scale with backend "b200": every verified pair passes the device oracle and
    is tuned (bf16 kernels, B200 resource model); the report carries each tuned
    kernel's GPU evidence (cli.py:133-146 records + "b200")."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from symfuse.cli import PipelineFlags, run_pipeline
    rep = run_pipeline(_qk_spec(ref), PipelineFlags(trials=1, param_samples=1, samples=4, backend="b200"))
    recs = [r for r in rep["candidates"] if r["verified"]]
    assert len(recs) == 32
    for r in recs:
        assert r["oracle"]["ok"], r
        assert r["best"]["params"] is not None, r
        ev = r["b200"]
        assert ev["dtype"] == "bf16" and ev["ff_ok"] and ev["latency_us"] > 0 and 0 < ev["roofline_frac"] < 1.2, ev
