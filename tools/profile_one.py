"""Run one population candidate's generated kernel repeatedly (for ncu).

  python tools/profile_one.py G "O.1.x,Wgate.1.x,Wup.1.x" '{"x":128,"i":1}' [--iters 20] [--ff]
  python tools/profile_one.py G best    (reads gpurun_out/records.json / profiles/records_*.json)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_15272_b200 import _abi  # noqa: E402
from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import PLANS  # noqa: E402
from paper_2604_15272_b200.tuner import workspace  # noqa: E402


def main():
    w, mapping = sys.argv[1], sys.argv[2]
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 20
    pop = P.load_population(w)
    us = P.units(pop)
    if mapping == "best" and isinstance(json.load(open(sys.argv[3])), dict):  # bench --best-out file
        b = json.load(open(sys.argv[3]))[w]
        # the same mapping/params can occur under several templates: match the template too
        u = next(x for x in us if x.cand.mapping_list() == b["mapping"] and x.cand.params == b["params"]
                 and pop["candidates"][x.pair]["template_id"] == b.get("template", pop["candidates"][x.pair]["template_id"]))
        variant = b.get("hints") or {}
        if "--runner-up" in sys.argv:  # one of the next tuned kernels of the bench's best-kernel phase
            ru = b["runners_up"][int(sys.argv[sys.argv.index("--runner-up") + 1])]
            u = us[ru["index"]]
            variant = ru.get("hints") or {}
    elif mapping == "best":
        recs = json.load(open(sys.argv[3]))
        rs = [r for r in recs if r["workload"] == w and r["latency_us"] and not r.get("error")]
        r = min(rs, key=lambda r: r["latency_us"])
        u = us[r["index"]]
        variant = r.get("hints") or ({"variant": r["variant"]} if r.get("variant") else {})
    else:
        params = json.loads(sys.argv[3])
        want = sorted(mapping.split(","))
        u = next(x for x in us if x.cand.mapping_list() == want and x.cand.params == params)
        variant = {}
    if len(sys.argv) > 4 and sys.argv[4].startswith("{"):
        variant = json.loads(sys.argv[4])
    torch.cuda.set_device(0)
    _abi.bind_device(0)
    ns = _abi.FF if "--ff" in sys.argv else P.numsys_of(pop["dtype"])
    plan = PLANS.get(u.cand, ns, variant or None, 0)
    ws = workspace(u.cand.program, ns, 0)
    print(f"{w} {u.cand.mapping_list()} {u.cand.params} kernel={plan.kernel_name} {plan.info['summary']}", flush=True)
    for i in range(iters):
        plan.run(ws.sets[i % ws.rot], ws.outputs, init_outputs=False)
    torch.cuda.synchronize()
    us_ = plan.time(ws.sets, ws.outputs, warmup=3, iters=50)
    print(f"latency {us_:.2f} us  {P.algorithmic_bytes(pop) / us_ / 1e3:.0f} GB/s")
    if "--source" in sys.argv:
        print(plan.source())


if __name__ == "__main__":
    main()
