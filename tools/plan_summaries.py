"""Planner summaries (no compile, no device) of every population candidate in
its deployment dtype and in the finite field, for A/B comparisons of planner
changes: `python tools/plan_summaries.py out.json` (env vars such as
SGM_NO_FREE_POLICY / SGM_NO_XCACHE apply), then `--diff a.json b.json`."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_15272_b200 import _abi  # noqa: E402
from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import build_desc, numsys_of  # noqa: E402


def summaries() -> dict:
    out = {}
    for w in P.WORKLOADS:
        pop = P.load_population(w)
        d = out[w] = {}
        for u in P.units(pop):
            for ns in (numsys_of(pop["dtype"]), 3):
                info = _abi.PlanInfo()
                rc = _abi.lib().sgm_plan_feasible(C.byref(build_desc(u.cand, ns, None)), C.byref(info))
                d[f"{u.index}/{ns}"] = info.plan_summary.decode() if rc == 0 else f"infeasible {rc}"
    return out


def est(s: str) -> float:
    for tok in s.split():
        if tok.startswith("est="):
            return float(tok[4:-2])
    return float("nan")


if __name__ == "__main__":
    if sys.argv[1] == "--diff":
        a, b = (json.load(open(f)) for f in sys.argv[2:4])
        for w in a:
            ch = [(k, a[w][k], b[w][k]) for k in a[w] if a[w][k] != b[w][k]]
            print(w, len(ch), "changed of", len(a[w]))
            ch.sort(key=lambda t: est(t[2]) - est(t[1]))
            for k, x, y in ch[:8]:
                print(f"  {k}: est {est(x):.0f} -> {est(y):.0f} us")
                print("     ", x[:110]); print("     ", y[:110])
    else:
        json.dump(summaries(), open(sys.argv[1], "w"), indent=0)
