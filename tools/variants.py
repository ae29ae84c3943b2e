"""Time physical-plan variants (planner hints) of a workload's top sweep candidates.

  python tools/variants.py L [--top 6] [--hints '[{"one_cta":1},{"big_first":1}]'] [--launches 500]

Runs a screening sweep (deployment dtype, no FF) over the population, takes the
top candidates, and for each times every hint set over one rotation of input
sets x (launches / rot) (CUDA graphs, cold L2 per launch).  Prints the table
sorted by latency, with the plan summary of the best few.
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_15272_b200 import _abi  # noqa: E402
from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import PLANS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("w")
    ap.add_argument("--top", type=int, default=6)
    ap.add_argument("--hints", default=None)
    ap.add_argument("--launches", type=int, default=500)
    ap.add_argument("--cand", action="append", default=[],
                    help='explicit candidate "template|mapping,comma,list|{params json}" (skips the screening sweep)')
    args = ap.parse_args()
    torch.cuda.set_device(0)
    _abi.bind_device(0)
    pop = P.load_population(args.w)
    us = P.units(pop)
    ctx = P.WorkloadContext(pop, 0, ff=False)
    if args.cand:
        ok = []
        for spec in args.cand:
            tid, mapping, params = spec.split("|")
            params = json.loads(params)
            u = next(x for x in us if pop["candidates"][x.pair]["template_id"] == int(tid)
                     and x.cand.mapping_list() == sorted(mapping.split(",")) and x.cand.params == params)
            ok.append(P.Record(args.w, u.index, u.pair, params, u.cand.mapping_list()))
    else:
        P.precompile([u.cand for u in us], [P.numsys_of(pop["dtype"])], 0)
        recs = P.evaluate_workload(ctx, us, ff=False, refine_top=args.top, refine_launches=200)
        ok = sorted((r for r in recs if r.latency_us and r.error is None), key=lambda r: r.latency_us)[:args.top]
    if args.hints:
        hs = json.loads(args.hints)
    else:
        base = [{}, {"one_cta": 1}, {"one_cta": 1, "slot_kb": 16}, {"slot_kb": 16}]
        extra = [{}, {"small_plain": 1}, {"big_first": 1}, {"big_first": 1, "small_plain": 1}]
        hs = [dict(a, **b) for a, b in itertools.product(base, extra)]
    byi = {u.index: u for u in us}
    rows = []
    for r in ok:
        u = byi[r.index]
        for h in hs:
            try:
                pl = PLANS.get(u.cand, ctx.numsys, h or None, 0)
            except Exception as exc:
                rows.append((1e9, r.index, h, f"ERR {exc}"[:80]))
                continue
            lat = P.graph_latency(ctx, pl, args.launches)
            rows.append((lat, r.index, h, pl.info["summary"]))
    rows.sort(key=lambda x: x[0])
    byts = P.algorithmic_bytes(pop)
    for lat, idx, h, summ in rows:
        print(f"{lat:8.2f} us  {byts / (lat * 1e-6) / 1e9 / P.hbm_peak_gbs():.3f}  #{idx} {byi[idx].cand.mapping_list()} "
              f"{byi[idx].cand.params} {json.dumps(h)}")
    for lat, idx, h, summ in rows[:3]:
        print(f"--- #{idx} {json.dumps(h)}: {summ}")


if __name__ == "__main__":
    main()
