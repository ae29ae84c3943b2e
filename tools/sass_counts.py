"""SASS evidence for the best kernels (no GPU needed): compile each winner of a
`bench.py --best-out` file for sm_100a, disassemble it with cuobjdump and count
the opcodes that prove the Blackwell paths (UTCHMMA = tcgen05.mma, UTCBAR =
tcgen05.commit, LDTM = tcgen05.ld, UTMALDG = TMA tensor load, SYNCS = mbarrier
ops) next to the CUDA-core ones (FFMA, HMMA = legacy mma.sync, none expected).

  python tools/sass_counts.py best.json > profiles/<tag>_sass.json
"""
import collections
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_2604_15272_b200 import population as P  # noqa: E402
from paper_2604_15272_b200.plan import Plan  # noqa: E402
from trace_one import pick  # noqa: E402

WATCH = ("UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMAPF", "SYNCS", "FFMA", "HMMA", "IMAD", "LDG", "LDS", "STS", "BAR")


def counts(cubin: bytes) -> dict:
    with tempfile.NamedTemporaryFile(suffix=".cubin") as fh:
        fh.write(cubin)
        fh.flush()
        sass = subprocess.run(["cuobjdump", "-sass", fh.name], capture_output=True, text=True).stdout
    ops = collections.Counter()
    for line in sass.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            ops[m.group(1).split(".")[0]] += 1
    return {k: ops.get(k, 0) for k in WATCH} | {"total_instructions": sum(ops.values())}


def main():
    path = sys.argv[1]
    best = json.load(open(path))
    out = {}
    for w, b in best.items():
        if "kernel" not in b:
            continue
        pop, u, hints = pick(w, "best", path)
        plan = Plan(u.cand, P.numsys_of(pop["dtype"]), hints or None, None)
        out[w] = {"kernel": plan.kernel_name, "expected_kernel": b["kernel"], "hints": hints,
                  "sass": counts(plan.cubin())}
        plan.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
