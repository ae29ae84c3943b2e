"""Timeline of one candidate kernel (plans built with hints={"trace": 1}).

  python tools/trace_one.py G "O.1.x,Wgate.1.x,Wup.1.x" '{"x":128,"i":1}' ['{"max_cluster":4}']
  python tools/trace_one.py G best <records.json>

Prints, over all CTAs of the last launch: kernel span, per-CTA busy span, and
the mean duration between consecutive compute-side events (item start, each
matmul/sum node, each flush, item end) plus the producer's stream starts
relative to item starts.  Event ids: include/sgm.h (sgm_plan_trace).
"""
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_15272_b200 import _abi  # noqa: E402
from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import Plan  # noqa: E402
from paper_2604_15272_b200.tuner import workspace  # noqa: E402


def name(ev: int) -> str:
    if ev >= 4000:
        return f"P:stream n{ev - 4000}"
    if ev >= 3000:
        return f"fl@{(ev - 3000) // 4}.{(ev - 3000) % 4}"
    if ev >= 2000:
        return f"flush@{ev - 2000}"
    if ev >= 1500:
        return f"own n{ev - 1500}"
    if ev >= 1000:
        return f"node n{ev - 1000}"
    if 600 <= ev < 700:
        return f"xT n{ev - 600}"
    return {0: "entry", 1: "start", 2: "item", 3: "P:item", 5: "item end", 6: "P:done", 7: "exit", 8: "tmem",
            9: "invariants"}.get(ev, str(ev))


def pick(w, mapping, arg):
    pop = P.load_population(w)
    us = P.units(pop)
    if mapping == "best" and isinstance(json.load(open(arg)), dict):  # bench --best-out file
        b = json.load(open(arg))[w]
        u = next(x for x in us if x.cand.mapping_list() == b["mapping"] and x.cand.params == b["params"]
                 and pop["candidates"][x.pair]["template_id"] == b.get("template", pop["candidates"][x.pair]["template_id"]))
        return pop, u, b.get("hints") or {}
    if mapping == "best":
        recs = [r for r in json.load(open(arg)) if r["workload"] == w and r.get("latency_us") and not r.get("error")]
        r = min(recs, key=lambda r: r["latency_us"])
        return pop, us[r["index"]], r.get("hints") or ({"variant": r["variant"]} if r.get("variant") else {})
    params = json.loads(arg)
    want = sorted(mapping.split(","))
    return pop, next(x for x in us if x.cand.mapping_list() == want and x.cand.params == params), 0


def main():
    w, mapping, arg = sys.argv[1:4]
    hints = json.loads(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4].startswith("{") else {}
    hints["trace"] = 1
    pop, u, variant = pick(w, mapping, arg)
    for k, v in (variant or {}).items():
        hints.setdefault(k, v)
    torch.cuda.set_device(0)
    _abi.bind_device(0)
    ns = _abi.FF if "--ff" in sys.argv else P.numsys_of(pop["dtype"])
    plan = Plan(u.cand, ns, hints, 0)
    ws = workspace(u.cand.program, ns, 0)
    for i in range(4):
        plan.run(ws.sets[i % ws.rot], ws.outputs, init_outputs=False)
    torch.cuda.synchronize()
    us_ = plan.time(ws.sets, ws.outputs, warmup=2, iters=20)
    plan.run(ws.sets[0], ws.outputs, init_outputs=False)
    tr = plan.trace()
    print(f"{w} {u.cand.mapping_list()} {u.cand.params} {plan.info['summary']}")
    print(f"timed latency {us_:.2f} us ({P.algorithmic_bytes(pop) / us_ / 1e3:.0f} GB/s)")
    t0 = min(int(x) for x in tr[:, :, 0].ravel() if x)
    comp = defaultdict(list)
    prodd = defaultdict(list)
    spans, items = [], []
    first = defaultdict(list)  # event -> absolute time of its first occurrence, per CTA
    for cta in tr:
        ev = [(int(t) - t0, int(e)) for t, e in cta[:256] if t]
        pv = [(int(t) - t0, int(e)) for t, e in cta[256:] if t]
        if not ev:
            continue
        spans.append((ev[0][0], ev[-1][0]))
        item_t = [t for t, e in ev if e == 2]
        items.append(len(item_t))
        seen = set()
        for t, e in ev + pv:
            if e not in seen:
                seen.add(e)
                first[name(e)].append(t)
        for (ta, ea), (tb, eb) in zip(ev, ev[1:]):
            comp[(name(ea), name(eb))].append(tb - ta)
        for (ta, ea), (tb, eb) in zip(pv, pv[1:]):
            prodd[(name(ea), name(eb))].append(tb - ta)
    st = np.array(spans)
    print(f"CTAs {len(spans)}  items/CTA {np.mean(items):.2f}  first start {st[:, 0].min() / 1e3:.2f} us  "
          f"last start {st[:, 0].max() / 1e3:.2f} us  last end {st[:, 1].max() / 1e3:.2f} us  "
          f"mean busy {np.mean(st[:, 1] - st[:, 0]) / 1e3:.2f} us")
    print("compute thread 0: mean us between events (count)")
    for k, v in sorted(comp.items(), key=lambda kv: -np.mean(kv[1]) * len(kv[1])):
        print(f"  {k[0]:>14} -> {k[1]:<14} {np.mean(v) / 1e3:8.3f} us  x{len(v)}")
    print("first occurrence per CTA (us from the earliest entry): min / median / max")
    for k, v in sorted(first.items(), key=lambda kv: np.median(kv[1])):
        v = np.array(v) / 1e3
        print(f"  {k:>14}  {v.min():8.2f} {np.median(v):8.2f} {v.max():8.2f}  x{len(v)}")
    print("producer lane:")
    for k, v in sorted(prodd.items(), key=lambda kv: -np.mean(kv[1]) * len(kv[1])):
        print(f"  {k[0]:>14} -> {k[1]:<14} {np.mean(v) / 1e3:8.3f} us  x{len(v)}")


if __name__ == "__main__":
    main()
