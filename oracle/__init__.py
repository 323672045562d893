"""ORACLE — test infrastructure, NOT part of the product.

Plain, slow, obviously-correct CPU implementations of what gSmart's hot path
computes (arXiv 2106.14038, /root/reference/PAPER.md).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl
reference` legs may import or execute anything here.  The product package
`paper_2106_14038_b200` never imports this package, and this package never
imports the product: they share no code (the seeded input generators live in
`synth/`, which holds none of the method's arithmetic).

Modules
  reference.py  — Python: BGP definition (brute force), tree-DP homomorphism
                  count, matrix-algebra operators of §2.1 (Eqs. 2-11),
                  degree-driven planner (§6.1.2), LSpM arrays (§6.2),
                  grouped incident-edge filter schedule (§5 Eqs. 17/21).
  bgp_oracle.c  — C: backtracking BGP matcher over sorted SPO/OPS copies
                  (the plain definition, fast enough for LUBM-100 queries).
  coracle.py    — ctypes loader for liboracle.so.

Every function states the passage it follows.  Parity status per function
is listed in DESIGN.md ("Oracle pins"); none is "parity unpinned".
"""
