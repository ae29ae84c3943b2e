"""Shared fixtures.  GPU tests are marked `gpu` and run only on a B200 box."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libsgm.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def desk_cases():
    with open(os.path.join(GOLDEN, "desk_cases.json")) as fh:
        return json.load(fh)["cases"]


@pytest.fixture(scope="session")
def desk_arrays():
    return dict(np.load(os.path.join(GOLDEN, "desk_arrays.npz")))


def case_inputs_f64(case):
    """Trial-0 inputs of random_equiv_test (interp.py:272-276)."""
    rng = np.random.default_rng([0, case["cid"], 0])
    prog = case["program"]
    return {t["name"]: rng.standard_normal(tuple(t["dims"])) for t in prog["tensors"] if t["role"] == "input"}


def case_inputs_ff(case):
    from oracle import ff_np
    from paper_2604_15272_b200.ff import ff_trial_seed
    prog = case["program"]
    names = [t for t in prog["tensors"] if t["role"] == "input"]
    return {t["name"]: ff_np.ff_uniform(int(np.prod(t["dims"])), ff_trial_seed(0, case["cid"], 0), k + 1)
            .reshape(tuple(t["dims"])) for k, t in enumerate(names)}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_symfuse():
    """The unmodified reference package installed into baseline/_ref (travels to the
    GPU box with the snapshot); None when it was not installed."""
    if not os.path.isdir(os.path.join(REF_DIR, "symfuse")):
        return None
    if REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import symfuse
        return symfuse
    except ImportError:
        return None
