"""TEST INFRASTRUCTURE ONLY — CPU oracle for the B200 backend.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker (or as the timed CPU
baseline).  The product path (paper_2604_15272_b200) never imports it; it
fails loudly when its CUDA extension is missing.

Contents
  ff_np.py     finite-field (mod 2^31-1) arithmetic in numpy, bit-identical to
               the device number system NFF (paper_2604_15272_b200/csrc/sgm_dev.cuh)
  block_np.py  CPU restatement of the reference interpreter's control flow
               (symfuse interp.py:69-212) with a pluggable arithmetic (fp64 / FF)

Pinning: tests/golden/make_golden.py runs the reference itself (symfuse,
imported from /root/reference in the build container) to produce fixtures:
fp64 outputs of interp.run_concrete / run_program, and FF outputs of the SAME
reference functions with apply_op rebound to ff_np's op table.  The oracle is
checked against those fixtures (tests/test_oracle.py).  The fp64 path is pinned
at tolerance (the reference itself is pinned only at 1e-9/1e-12);
the FF path is pinned bit-exactly.
"""
