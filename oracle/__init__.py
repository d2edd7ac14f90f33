"""fp64 CPU oracle for the LOVE / KISS-GP hot path (arXiv 1803.06058).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and bench.py's
`cpu_baseline` / `--impl reference` legs may import anything from here.  The product path
(`paper_1803_06058_b200`) never imports, calls or links this package, and this package
never imports the product path: the two share no code.

Every function cites the PAPER.md passage (P:<line>, section/equation/algorithm) it
follows; readings of points the paper leaves open are SURVEY.md §8(c) A1..A25 and are
listed in DESIGN.md.  Parity status per function is in the module header of
`love_oracle.py` (every function is pinned by tests/test_oracle_pins.py).
"""
from .love_oracle import *  # noqa: F401,F403
