"""Run one population candidate once (for compute-sanitizer / fault triage).

  python tools/run_one.py A 635 [ns] [hints-json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_15272_b200 import _abi  # noqa: E402
from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import Plan  # noqa: E402
from paper_2604_15272_b200.tuner import Workspace  # noqa: E402


def main():
    w, idx = sys.argv[1], int(sys.argv[2])
    pop = P.load_population(w)
    ns = int(sys.argv[3]) if len(sys.argv) > 3 else P.numsys_of(pop["dtype"])
    hints = json.loads(sys.argv[4]) if len(sys.argv) > 4 else None
    torch.cuda.set_device(0)
    _abi.bind_device(0)
    u = P.units(pop)[idx]
    plan = Plan(u.cand, ns, hints, 0)
    print(u.cand.mapping_list(), u.cand.params, plan.kernel_name, plan.info["summary"], flush=True)
    ws = Workspace(u.cand.program, ns, 0, min_rot_bytes=0, max_rot=1)
    plan.run(ws.sets[0], ws.outputs)
    torch.cuda.synchronize()
    print("ok", flush=True)


if __name__ == "__main__":
    main()
