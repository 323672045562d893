"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds ONLY input generation: triple sets, query graphs and the
counter-based RNG they are drawn from.  It contains none of the method's
arithmetic (no LSpM, no SpMV, no planning, no matching), so that the oracle
(`oracle/`) and the product (`paper_2106_14038_b200/`) can both consume it
without sharing any code path of the method (task rule: "only the seeded input
generators serve both, from a module of their own").

Conventions (§6.2.1 step 2): entity ids are 0-based,
predicate ids are 1-based.  A query is a `Query` (see `synth.query`).
"""
from .query import Query, var, const  # noqa: F401
