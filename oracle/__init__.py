"""CPU oracle for the IOS stage executor (arXiv 2011.01302) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this package. The product path (``paper_2011_01302_b200`` and
``libios.so``) never imports, links or executes it, and shares no code with it: the only common
dependency is ``workloads`` (seeded input generators, none of the method's arithmetic).

Plain, slow, obviously-correct NumPy in float64:

* ``tensor_ops``  O1 tensor semantics (conv, Relu-SepConv, pools, add, concat, linear).
* ``graph``       G = (V, E), shapes, groups, merge legality + explicit merged conv,
                  ``run_sequential`` / ``run_schedule`` (O2).
* ``scheduler``   Algorithm 1 literally (endings, Scheduler, GenerateStage, rebuild of Q),
                  brute force over all schedules, sequential and greedy schedules, counting (O3).

Citations: ``P:n`` = /root/reference/PAPER.md line n. Every function is pinned by a
``-m "not gpu"`` test in tests/test_oracle_*.py; the only unpinned quantity is the measured stage
latency (a measurement).
"""
from . import tensor_ops, graph, scheduler  # noqa: F401
from .graph import OracleGraph  # noqa: F401
