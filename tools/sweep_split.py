"""Where a workload's sweep time goes: FF checks vs timing passes.

  python tools/sweep_split.py A
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_15272_b200 import _abi  # noqa: E402
from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import PLANS  # noqa: E402


def main():
    w = sys.argv[1]
    torch.cuda.set_device(0)
    _abi.bind_device(0)
    pop = P.load_population(w)
    us = P.units(pop)
    ctx = P.WorkloadContext(pop, 0)
    P.precompile([u.cand for u in us], [ctx.numsys, _abi.FF], 0)
    P.evaluate_workload(ctx, us[:8])
    torch.cuda.synchronize()
    for ff in (True, False):
        t0 = time.time()
        P.evaluate_workload(ctx, us, ff=ff)
        torch.cuda.synchronize()
        print(f"{w}: evaluate_workload ff={ff}: {time.time() - t0:.3f} s for {len(us)} candidates")
    # FF runs alone
    t0 = time.time()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for u in us:
        try:
            PLANS.get(u.cand, _abi.FF, None, 0).run(ctx.ff_inputs, ctx.ff_out)
        except Exception:
            pass
    ev1.record()
    torch.cuda.synchronize()
    print(f"{w}: FF runs only: wall {time.time() - t0:.3f} s, GPU {ev0.elapsed_time(ev1) / 1e3:.3f} s")


if __name__ == "__main__":
    main()
