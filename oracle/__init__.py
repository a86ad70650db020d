"""SMP-PCA CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 reference implementation of the SMP-PCA hot path
(arXiv 1610.06656, Alg. 1 P:49-60 and Alg. 2) used to check the CUDA
path.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product path
(``paper_1610_06656_b200``) never imports it and shares no code with it.

Parity status: every function is pinned (tests/test_oracle_pins.py) except
those listed as "parity unpinned" in DESIGN.md §4 — currently none.
"""
from .oracle import *  # noqa: F401,F403
