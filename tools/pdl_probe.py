"""Back-to-back launch timing of a best kernel: stream loop vs CUDA graph (run twice,
with and without SGM_NO_PDL=1, to see what programmatic dependent launch buys).

  python tools/pdl_probe.py G tools/data/best_r29.json
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from paper_2604_15272_b200 import _abi  # noqa: E402
from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import Plan  # noqa: E402
from paper_2604_15272_b200.tuner import workspace  # noqa: E402
from trace_one import pick  # noqa: E402


def main():
    w, path = sys.argv[1], sys.argv[2]
    pop, u, hints = pick(w, "best", path)
    torch.cuda.set_device(0)
    _abi.bind_device(0)
    ns = P.numsys_of(pop["dtype"])
    plan = Plan(u.cand, ns, hints or None, 0)
    ws = workspace(u.cand.program, ns, 0)
    n = 400
    for _ in range(20):
        plan.run(ws.sets[0], ws.outputs, init_outputs=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        plan.run(ws.sets[i % ws.rot], ws.outputs, init_outputs=False)
    e1.record()
    torch.cuda.synchronize()
    loop = e0.elapsed_time(e1) * 1e3 / n
    graph = plan.time(ws.sets, ws.outputs, warmup=3, iters=n)
    print(f"{w} pdl={'off' if os.environ.get('SGM_NO_PDL') else 'on'}: stream loop {loop:.2f} us/launch, "
          f"graph {graph:.2f} us/launch  {plan.info['summary'][:80]}")


if __name__ == "__main__":
    main()
