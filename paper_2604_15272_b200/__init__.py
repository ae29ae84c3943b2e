"""B200 (sm_100a) execution and evaluation backend for SIGMA sGraph candidates.

Drop-in for the reference interpreter's hot path (symfuse interp.py / tuner.py):
generated per-candidate CUDA kernels (libsgm.so, NVRTC for sm_100a), a GPU
profiler, and finite-field equivalence checking on device.
"""
from .errors import (BackendError, BackendUnavailable, ConstraintError, DivisibilityError, EmptyParamSpaceError,
                     ShapeError, SymfuseError, UnsupportedOpError, WriteConflictError)
from .ff import ff_equiv_test
from .interp import EquivVerdict, candidate_id, random_equiv_test, rel_err, run_concrete, run_program
from .ir import Candidate, Program, from_serialized, program_candidate, template_key
from .plan import Plan
from .tuner import (DEFAULT_BUDGET, CostModel, ProfileResult, cost_stats, enumerate_param_space, score_b200,
                    score_cost, smem_usage, tune)

__version__ = "0.1.0"

__all__ = [
    "run_concrete", "run_program", "random_equiv_test", "ff_equiv_test", "rel_err", "candidate_id",
    "EquivVerdict", "tune", "score_b200", "score_cost", "cost_stats", "enumerate_param_space", "smem_usage",
    "CostModel", "ProfileResult", "DEFAULT_BUDGET", "Plan", "Candidate", "Program", "from_serialized",
    "program_candidate", "template_key", "SymfuseError", "ShapeError", "DivisibilityError", "ConstraintError",
    "UnsupportedOpError", "WriteConflictError", "EmptyParamSpaceError", "BackendError", "BackendUnavailable",
]
