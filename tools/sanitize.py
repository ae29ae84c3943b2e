"""One generated kernel per physical-plan mode, launched twice each in the
deployment dtype and once in GF(p), for compute-sanitizer:

  compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize.py
  compute-sanitizer --tool synccheck python tools/sanitize.py
  compute-sanitizer --tool memcheck python tools/sanitize.py

Modes: gsplit tail reduction (global partials + self-resetting counters),
cluster one-barrier push (small DSMEM partials), cluster reduce-scatter +
all-gather (large partials), two TMEM-allocating CTAs per SM (paired tcgen05),
fp32 TMA ring on CUDA cores; round 2's x-cache, column strips + register
prefetch and small-tile thread counts.  Prints each plan summary and the max rel_err of
the second launch against the first (launch-to-launch determinism).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_15272_b200 import _abi  # noqa: E402
from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import Plan  # noqa: E402
from paper_2604_15272_b200.tuner import Workspace  # noqa: E402

CASES = [
    ("gsplit", "G", 0, "O.1.x,Wgate.1.x,Wup.1.x", {"x": 8, "i": 1}, {"max_cluster": 1}),
    ("cluster-push", "R", 26, "O.1.x,W.1.x", {"x": 2, "i": 1}, {"max_cluster": 4, "max_gsplit": 1}),
    ("cluster-rs-ag", "A", 42, "Kt.1.x,O.1.x,Q.1.x,V.1.x", {"x": 2, "i": 1}, {"max_cluster": 8, "max_gsplit": 1}),
    ("paired-tmem", "Q", 36, "Kt.0.x,O.0.x,Q.0.x,V.0.x", {"x": 8, "i": 1}, {}),
    ("f32-ring", "R", 26, "O.1.x,W.1.x", {"x": 2, "i": 1}, {"one_cta": 1, "max_cluster": 1}),
    # round 2 codegen: x-cache, column strips (T = 1, 2) + register prefetch, small-tile thread count
    ("x-cache", "A", 57, "Kt.2.i,O.3.x,Q.3.i,V.3.x", {"x": 16, "i": 1}, {}),
    ("strip-1", "A", 38, "Kt.3.i,O.3.x,V.2.i,V.3.x", {"x": 2, "i": 8192}, {}),
    ("strip-2", "A", 38, "Kt.3.i,O.3.x,V.2.i,V.3.x", {"x": 2, "i": 4096}, {}),
    ("small-nt", "L", 9, "A.0.i,B.1.x,O.1.x,W.0.i,W.1.x,X.1.i", {"x": 128, "i": 512}, {}),
]


def main():
    only = sys.argv[1:]
    torch.cuda.set_device(0)
    _abi.bind_device(0)
    for mode, w, tid, mapping, params, hints in CASES:
        if only and mode not in only:
            continue
        pop = P.load_population(w)
        u = next(x for x in P.units(pop) if x.cand.mapping_list() == sorted(mapping.split(","))
                 and x.cand.params == params and pop["candidates"][x.pair]["template_id"] == tid)
        for ns in (P.numsys_of(pop["dtype"]), _abi.FF):
            plan = Plan(u.cand, ns, hints or None, 0)
            ws = Workspace(u.cand.program, ns, 0, min_rot_bytes=0, max_rot=1)
            outs = [torch.empty_like(o) for o in ws.outputs]
            plan.run(ws.sets[0], ws.outputs)
            plan.run(ws.sets[0], outs)
            torch.cuda.synchronize()
            same = all(torch.equal(a, b) for a, b in zip(ws.outputs, outs))
            print(f"{mode:14s} {w} {_abi.NUMSYS_NAMES[ns]:4s} {plan.kernel_name} deterministic={same} "
                  f"watchdog={plan.watchdog()} | {plan.info['summary'][:150]}", flush=True)


if __name__ == "__main__":
    main()
