"""NetMF+ CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 numpy/scipy restatement of PAPER.md (arxiv 2110.12782)
Alg. 2–5, Eq. 1–5, used to check the CUDA path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The product package
``paper_2110_12782_b200`` never imports it and shares no code with it.

Parity pins: every function is pinned by ``tests/test_oracle_*.py`` against
closed forms, brute force or paper invariants.  No
function here is "parity unpinned".
"""
from .netmf_oracle import *  # noqa: F401,F403
