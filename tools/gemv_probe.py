"""Streaming-rate probe: a column-split X[M,K] . W[K,N] candidate timed on its own.

  python tools/gemv_probe.py bf16 8 4096 14336 16 '{"max_cluster":1}' [--trace]

Prints latency, achieved GB/s on the algorithmic bytes and the plan.  With
--trace, also the per-CTA timeline summary (see tools/trace_one.py).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2604_15272_b200 as S  # noqa: E402
from paper_2604_15272_b200 import _abi  # noqa: E402
from paper_2604_15272_b200.tuner import workspace  # noqa: E402


def main():
    dt, M, K, N, x = sys.argv[1], *map(int, sys.argv[2:6])
    hints = json.loads(sys.argv[6]) if len(sys.argv) > 6 and sys.argv[6].startswith("{") else {}
    T, Op, Nd = S.ir.Tensor, S.ir.Op, S.ir.Node
    prog = S.ir.Program("gemv", (T("X", (M, K), "input"), T("W", (K, N), "input"), T("O", (M, N), "output")),
                        (Op("matmul", ("X", "W"), "O"),), ("O",))
    blk = S.ir.Block(("x",), "i", (Nd(0, "input", (), "X"), Nd(1, "input", (), "W"), Nd(2, "matmul", (0, 1)),
                                   Nd(3, "output", (2,), "O")))
    cand = S.ir.Candidate(prog, blk, frozenset({("W", 1, "x"), ("O", 1, "x")}), {"x": x, "i": 1})
    torch.cuda.set_device(0)
    _abi.bind_device(0)
    ns = {"bf16": 2, "f32": 1}[dt]
    if "--trace" in sys.argv:
        hints["trace"] = 1
    plan = S.Plan(cand, ns, hints, 0)
    ws = workspace(prog, ns, 0)
    us = plan.time(ws.sets, ws.outputs, warmup=3, iters=200)
    es = 2 if dt == "bf16" else 4
    byts = (M * K + K * N + M * N) * es
    print(f"{dt} M={M} K={K} N={N} x={x} {hints}: {us:.2f} us  {byts / us / 1e3:.0f} GB/s  {plan.info['summary']}")


if __name__ == "__main__":
    main()
