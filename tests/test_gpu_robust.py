"""Robustness of generated kernels on the B200: the per-kernel watchdog turns a
hung kernel into the reference's "run: ..." outcome (interp.py:278-281)
instead of a hung device, and the context stays usable afterwards."""
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


def _gemv(S):
    T, Op, N = S.ir.Tensor, S.ir.Op, S.ir.Node
    prog = S.ir.Program("gemv", (T("X", (8, 1024), "input"), T("W", (1024, 2048), "input"), T("O", (8, 2048), "output")),
                        (Op("matmul", ("X", "W"), "O"),), ("O",))
    blk = S.ir.Block(("x",), "i", (N(0, "input", (), "X"), N(1, "input", (), "W"), N(2, "matmul", (0, 1)),
                                   N(3, "output", (2,), "O")))
    return S.ir.Candidate(prog, blk, frozenset({("W", 1, "x"), ("O", 1, "x")}), {"x": 4, "i": 1})


def test_watchdog_turns_a_hang_into_run_timeout(S):
    import time
    from paper_2604_15272_b200.errors import KernelTimeout, SymfuseError
    cand = _gemv(S)
    rng = np.random.default_rng(0)
    ins = {"X": rng.standard_normal((8, 1024)), "W": rng.standard_normal((1024, 2048))}
    t0 = time.time()
    with pytest.raises(KernelTimeout) as ei:
        S.run_concrete(cand, ins, dtype="bf16", hints={"wd_test": 1})
    assert isinstance(ei.value, SymfuseError)   # random_equiv_test reports it as "run: ..."
    assert time.time() - t0 < 30
    # the device is still healthy: the same candidate without the fault is correct
    got = S.run_concrete(cand, ins, dtype="bf16")["O"]
    import torch
    xr = torch.from_numpy(ins["X"]).bfloat16().double().numpy()
    wr = torch.from_numpy(ins["W"]).bfloat16().double().numpy()
    assert S.rel_err(got, xr @ wr) < 1e-2
    assert not S.Plan(cand, 2, None, 0).watchdog()
