"""Code-generator structure on the committed populations (NVRTC compile-only,
no device): which physical-plan features the planner picks for the shapes
they were built for.  Their numerics are checked on the GPU
(test_gpu_sweep.py: x-cache, loop prefetch / column strips; test_gpu_numerics.py:
accumulate-into)."""
import pytest

import paper_2604_15272_b200 as S
from paper_2604_15272_b200 import _abi
from paper_2604_15272_b200 import population as P


def _unit(w, mapping, params, template=None):
    pop = P.load_population(w)
    return next(u for u in P.units(pop) if u.cand.mapping_list() == sorted(mapping.split(","))
                and u.cand.params == params
                and (template is None or pop["candidates"][u.pair]["template_id"] == template))


def _src(u, ns, hints=None):
    p = S.Plan(u.cand, ns, hints, None)
    try:
        return p.source(), p.info["summary"]
    finally:
        p.close()


@pytest.mark.parametrize("ns", [_abi.BF16, _abi.FF])
def test_head_dim_split_scores_are_x_cached(ns):
    """Attention scores do not depend on the V/O head-dim split: kept across a
    CTA's consecutive items, recomputed only when the other coordinates change."""
    u = _unit("A", "Kt.2.i,O.3.x,Q.3.i,V.3.x", {"x": 16, "i": 1})
    src, _ = _src(u, ns)
    assert "xc_miss" in src
    assert "xc_miss" not in _src(u, ns, {"no_xcache": 1})[0]


@pytest.mark.parametrize("ns", [_abi.BF16, _abi.FF])
def test_key_per_iteration_loops_use_column_strips(ns):
    """A's one-key-per-iteration split-KV loop: the Kt column comes from 16-byte
    row strips (8 bf16 / 4 residues = that many iterations), V's row is
    prefetched one iteration ahead."""
    u = _unit("A", "Kt.3.i,O.3.x,V.2.i,V.3.x", {"x": 128, "i": 8192}, template=38)
    src, _ = _src(u, ns)
    assert "sgm::TileStrip<N, 2, 8, 128, 1," in src
    assert "sgm::TilePf<N, 2, 8, 1, 1," in src
    period = 8 if ns == _abi.BF16 else 4
    assert f"& {period - 1}) == {period - 1} && j + 1 <" in src
    plain, _ = _src(u, ns, {"no_prefetch": 1})
    assert "TileStrip" not in plain and "TilePf" not in plain


def test_small_tile_loops_run_fewer_threads():
    """L's one-k-per-iteration candidates (body tiles <= 128 elements, 1024
    iterations per part): 32 threads per CTA instead of 256."""
    u = _unit("L", "A.0.i,B.1.x,O.1.x,W.0.i,W.1.x,X.1.i", {"x": 4096, "i": 4096})
    src, summary = _src(u, _abi.BF16)
    assert " NT=32 " in summary
    assert "#define NT 32" in src


def test_lora_accumulate_into_fusion():
    """LoRA's best candidate: T@B issued into X@W's TMEM accumulators (no
    read-back of its own), X@W pre-initialised (PRE = 1), the add a copy."""
    u = _unit("L", "B.1.x,O.1.x,W.1.x", {"x": 32, "i": 1}, template=4)
    src, _ = _src(u, _abi.BF16, {"one_cta": 1, "no_wd": 1})
    assert ", false>(t" in src and "true, 1>(t" in src
    assert "sgm::tcgen05" in src or "mm_stream_tc<" in src


def test_planner_summaries_are_deterministic():
    u = _unit("Q", "O.3.x,V.3.x", {"x": 128, "i": 1}, template=37)
    a, b = _src(u, _abi.BF16), _src(u, _abi.BF16)
    assert a == b


def _res_usage(p):
    import os
    import re
    import subprocess
    import tempfile
    fd, path = tempfile.mkstemp(suffix=".cubin")
    try:
        os.write(fd, p.cubin())
        os.close(fd)
        out = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True).stdout
    finally:
        os.unlink(path)
    m = re.search(r"REG:(\d+) STACK:(\d+)", out)
    return int(m.group(1)), int(m.group(2))


def test_wide_gsplit_tail_does_not_spill():
    """A 128-way gsplit reduction tail (A's split-KV loop, finite field) reads its
    partials in batches: holding all 128 in registers spilled the whole kernel
    (255 registers + 432 B of stack, one CTA per SM)."""
    import shutil
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    u = _unit("A", "Kt.3.i,O.3.x,V.2.i,V.3.x", {"x": 2, "i": 8192}, template=38)
    p = S.Plan(u.cand, _abi.FF, None, None)
    try:
        assert "GP=128" in p.info["summary"]
        regs, stack = _res_usage(p)
    finally:
        p.close()
    assert regs < 200 and stack == 0, (regs, stack)
