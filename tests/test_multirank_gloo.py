"""The N>1 path of the candidate sweep on CPU: world_size 2 over gloo.

Each rank takes its LPT shard of the population (population.shard), produces
records, and the winner is reduced with the same all_reduce(MIN) of
(latency_ns << 20 | index) that bench.py issues over NCCL, plus the
all_gather of records.  The reduced winner must equal the single-process
argmin over the whole population, and the gathered records must cover every
candidate exactly once.  Latencies are synthetic (deterministic in the index),
so only the host logic is under test.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _latency(u) -> float:
    # deterministic, with ties, so the index tie-break is exercised
    return 5.0 + ((u.index * 2654435761) % 97) / 8.0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2604_15272_b200 import population as P
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for w in ("R", "L"):
            us = P.units(P.load_population(w))
            mine = P.shard(us, rank, world)
            recs = [P.Record(w, u.index, u.pair, dict(u.cand.params), u.cand.mapping_list(), ff_ok=True,
                             latency_us=_latency(u)) for u in mine]
            win = P.reduce_best(P.argmin(recs), dist)
            assert P.reduce_best_many([P.argmin(recs), None], dist) == [win, -1]
            gathered = [None] * world
            dist.all_gather_object(gathered, [r.index for r in recs])
            local = sorted((r.latency_us, r.index) for r in recs)[:3]
            top = P.global_top(dist, 3)(local)   # the sharded refine selection (evaluate_workload select=)
            res[w] = (win, sorted(i for part in gathered for i in part), sorted(top))
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_argmin_matches_single_process(world):
    from paper_2604_15272_b200 import population as P
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    assert len(out) == world
    for w in ("R", "L"):
        us = P.units(P.load_population(w))
        expect = min(us, key=lambda u: (round(_latency(u) * 1000), u.index)).index
        top3 = sorted(u.index for u in sorted(us, key=lambda u: (_latency(u), u.index))[:3])
        for r in range(world):
            win, idx, top = out[r][w]
            assert win == expect, (w, r)
            assert idx == sorted(u.index for u in us)
            assert top == top3, (w, r)
