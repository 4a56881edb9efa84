"""CPU oracle for the mixed-precision ID hot path (arXiv 2012.00706).

TEST INFRASTRUCTURE ONLY.  Plain, slow, written from PAPER.md; only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import it.  It shares no code with the CUDA path (paper_2012_00706_b200/) and
imports nothing from it.

Parity status per function:
  rounding.round_to        pinned (S:46-57 values, exhaustive fp16 midpoints, numpy/x86 conversions)
  rounding.gamma           pinned (closed form, S:65 printed form)
  qrcp.qrcp_householder    pinned (LAPACK dgeqp3 in fp64, MGS cross-check, hand example S:196,
                                   brute-force greedy pivots, planted skeleton, exact rank)
  qrcp.qrcp_mgs            pinned (S:195-196 examples, dgeqp3)
  id.coeffs_from_R         pinned (S:250-252 examples, exact-rank inputs)
  id.coeffs_lsq            pinned (numpy lstsq, exact-rank inputs)
  id.id_error              pinned (skeleton columns exact, Eckart-Young, Pythagorean identity)
  id.post_bound            parity unpinned (a derived bound; only checked to hold)
"""
