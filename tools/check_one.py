"""Numerics of one population candidate under several number systems / plan hints.

  python tools/check_one.py A "Kt.2.i,O.3.x,Q.3.i,V.3.x" '{"x":2,"i":16}' '[{}, {"no_tma":1}, {"max_cluster":8}]'

For each hint set: rel_err vs the fp64 oracle of bf16 / f32 / f64 runs (inputs
rounded to the dtype), bit-exactness of the FF run vs the program, and the plan.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_15272_b200 as S  # noqa: E402
from oracle import block_np  # noqa: E402
from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.ff import ff_fill_inputs, ff_run, ff_trial_seed  # noqa: E402


def main():
    w, mapping, params = sys.argv[1], sorted(sys.argv[2].split(",")), json.loads(sys.argv[3])
    hint_sets = json.loads(sys.argv[4]) if len(sys.argv) > 4 else [{}]
    pop = P.load_population(w)
    u = next(x for x in P.units(pop) if x.cand.mapping_list() == mapping and x.cand.params == params)
    prog = pop["program"]
    rng = np.random.default_rng(5)
    raw = {t["name"]: rng.standard_normal(tuple(t["dims"])) for t in prog["tensors"] if t["role"] == "input"}
    for hints in hint_sets:
        for dt in ("bf16", "f32", "f64"):
            tt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[dt]
            ins = {k: torch.from_numpy(v).to(tt).double().numpy() for k, v in raw.items()}
            exp = block_np.run_program(prog, ins)
            try:
                plan = S.Plan(u.cand, S.plan.numsys_of(dt), hints, 0)
                got = S.interp._execute(u.cand, ins, S.plan.numsys_of(dt), 0, hints, False)
                torch.cuda.synchronize()
                err = max(S.rel_err(got[n], exp[n]) for n in prog["outputs"])
                print(f"{hints} {dt}: rel_err {err:.3e}  {plan.info['summary'][:150]}", flush=True)
            except Exception as exc:
                print(f"{hints} {dt}: ERROR {type(exc).__name__}: {str(exc)[:300]}", flush=True)
        fi = ff_fill_inputs(u.cand.program, ff_trial_seed(1, 2, 3), 0)
        fe = ff_run(S.ir.program_candidate(u.cand.program), fi, 0)
        fg = ff_run(u.cand, fi, 0, hints)
        print(f"{hints} ff: {'bit-exact' if all(torch.equal(a, b) for a, b in zip(fg, fe)) else 'MISMATCH'}", flush=True)


if __name__ == "__main__":
    main()
