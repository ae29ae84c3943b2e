"""Generated CUDA source of one population candidate (compile-only, no GPU needed).

  python tools/dump_src.py G best gpurun_out/best.json [hints-json] > /tmp/g.cu
  python tools/dump_src.py A "O.2.x,Q.2.x" '{"x":1,"i":1}' [hints-json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import Plan  # noqa: E402
from trace_one import pick  # noqa: E402


def main():
    w, mapping, arg = sys.argv[1:4]
    hints = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
    pop, u, variant = pick(w, mapping, arg)
    for k, v in (variant or {}).items():
        hints.setdefault(k, v)
    plan = Plan(u.cand, P.numsys_of(pop["dtype"]), hints, None)
    sys.stderr.write(plan.info["summary"] + "\n")
    print(plan.source())


if __name__ == "__main__":
    main()
