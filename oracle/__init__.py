"""CPU fp64 oracle for the Multi-Head LatentMoE layer under Head Parallel.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path (the C-ABI library in
``paper_2602_04870_b200/`` and its Python binding) may import, call or link
anything under ``oracle/``.  The only permitted callers are ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``.

The oracle shares no code with the CUDA path: no kernels, headers, helpers,
tables or constant generators.  Its inputs come from the seeded generators in
``workloads/`` (which hold none of the method's arithmetic) or are built by the
tests themselves.

Parity status: every function in ``mhlmoe_oracle`` is pinned by a ``-m "not
gpu"`` test in ``tests/test_oracle_*.py`` ("Oracle pins").  No
function is "parity unpinned".
"""
from .mhlmoe_oracle import *  # noqa: F401,F403
