"""Plug the B200 backend into an unmodified `symfuse` (the reference package).

The reference's hot path reaches its executor through module globals:
  * random_equiv_test calls `run_concrete` / `run_program` from the
    `symfuse.interp` module namespace (interp.py:277,279);
  * score_interp imports `run_concrete` from `.interp` at call time
    (tuner.py:162);
  * run_pipeline stage 4 calls `tune(..., backend=flags.backend)`
    (cli.py:182-189), whose backend switch is tuner.py:215-220.
`install()` rebinds those names, so the reference's own stage-4 loop, its
oracle and its interp-backend tuner execute on the B200 without editing the
reference; `backend="b200"` becomes a valid tune() backend (and CLI choice).
`uninstall()` restores the originals.  Names bound at import time elsewhere
(`symfuse.run_concrete`, `from symfuse.interp import run_concrete` in callers)
are not affected; call this module's functions directly there.
"""
from __future__ import annotations

import functools

_SAVED: dict = {}


def install(symfuse=None, device=None):
    """Rebind the reference's executor seam to the B200 backend; returns the module."""
    if symfuse is None:
        import symfuse  # noqa: F811
    import symfuse.interp as RI
    import symfuse.tuner as RT

    from . import interp as BI
    from . import tuner as BT

    if _SAVED:
        return symfuse
    _SAVED.update(run_concrete=RI.run_concrete, run_program=RI.run_program, tune=RT.tune)

    @functools.wraps(RI.run_concrete)
    def run_concrete(concrete, inputs, dtype=None, tile_dump=None):
        import numpy as np
        return BI.run_concrete(concrete, inputs, np.float64 if dtype is None else dtype, tile_dump, device=device)

    @functools.wraps(RI.run_program)
    def run_program(program, inputs):
        return BI.run_program(program, inputs, device=device)

    orig_tune = RT.tune

    @functools.wraps(orig_tune)
    def tune(graph, mapping, backend="cost", samples=16, seed=0, budget_bytes=RT.DEFAULT_BUDGET, trials=3,
             model=RT.CostModel()):
        if backend != "b200":
            return orig_tune(graph, mapping, backend, samples, seed, budget_bytes, trials, model)
        r = BT.tune(graph, mapping, backend="b200", samples=samples, seed=seed, budget_bytes=budget_bytes,
                    trials=trials, device=device)
        return RT.ProfileResult(params=r.params, score=r.score)

    RI.run_concrete = run_concrete
    RI.run_program = run_program
    RT.tune = tune
    try:
        import symfuse.cli as RC
        _SAVED["cli_tune"] = RC.tune
        RC.tune = tune  # cli.py imports tune by name (stage 4, cli.py:182)
    except ImportError:  # pragma: no cover
        pass
    return symfuse


def uninstall():
    if not _SAVED:
        return
    import symfuse.interp as RI
    import symfuse.tuner as RT
    RI.run_concrete = _SAVED["run_concrete"]
    RI.run_program = _SAVED["run_program"]
    RT.tune = _SAVED["tune"]
    if "cli_tune" in _SAVED:
        import symfuse.cli as RC
        RC.tune = _SAVED["cli_tune"]
    _SAVED.clear()
