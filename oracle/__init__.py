"""CPU oracle for the GEVO-ML fitness-evaluation hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in `paper_2310_10211_b200` imports this
package; only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its
`cpu_baseline` leg and `--impl reference`) may.  It is the checker, never the
thing measured as the product.

It restates, with the same numpy calls, the reference's
  * interpreter      (pkg/src/evotir/interpreter.py:41-225)  -> oracle.interp
  * fitness protocol (pkg/src/evotir/fitness.py:338-426)     -> oracle.fitness
  * NSGA-II          (pkg/src/evotir/search.py:91-179)        -> oracle.nsga2

Parity pinned: `tests/golden/make_golden.py` (run in the build container,
where /root/reference is importable) records the reference's own outputs,
and `tests/test_oracle_golden.py` checks this restatement reproduces every
one of them bit-for-bit.
"""
