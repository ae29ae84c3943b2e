"""Run population candidates one per subprocess (a device fault cannot poison the
others) against the fp64 oracle in the deployment dtype; prints one line each.

  python tools/diag_candidates.py G [index ...]      (default: every candidate)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2604_15272_b200 as S
from paper_2604_15272_b200 import population as P
from oracle import block_np
w, idx = sys.argv[1], int(sys.argv[2])
pop = P.load_population(w); u = P.units(pop)[idx]
dt = pop["dtype"]; prog = pop["program"]
rng = np.random.default_rng(5)
def rnd(x):
    t = torch.from_numpy(x)
    t = t.to(torch.bfloat16) if dt == "bf16" else t.to(torch.float32)
    return t.to(torch.float64).numpy()
ins = {t["name"]: rnd(rng.standard_normal(tuple(t["dims"]))) for t in prog["tensors"] if t["role"] == "input"}
exp = block_np.run_program(prog, ins)
plan = S.Plan(u.cand, S.plan.numsys_of(dt), None, 0)
got = S.run_concrete(u.cand, ins, dtype=dt)
torch.cuda.synchronize()
err = max(S.rel_err(got[n], exp[n]) for n in prog["outputs"])
print(json.dumps({"idx": idx, "params": u.cand.params, "map": u.cand.mapping_list(), "err": err, "plan": plan.info["summary"]}))
""" % ROOT


def main():
    w = sys.argv[1]
    from paper_2604_15272_b200 import population as P
    n = len(P.units(P.load_population(w)))
    idx = [int(x) for x in sys.argv[2:]] or list(range(n))
    for i in idx:
        r = subprocess.run([sys.executable, "-c", CHILD, w, str(i)], capture_output=True, text=True, timeout=300)
        out = r.stdout.strip().splitlines()
        print(out[-1] if r.returncode == 0 and out else f"FAIL {w} #{i} rc={r.returncode} {r.stderr.strip()[-300:]}",
              flush=True)


if __name__ == "__main__":
    main()
