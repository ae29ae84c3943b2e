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
