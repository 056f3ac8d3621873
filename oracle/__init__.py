"""ORACLE — test infrastructure only.

A plain, slow, float64 CPU implementation of SINGA's synchronous BP
TrainOneBatch step (arXiv 1603.07846, §4.1.3 Alg. 1, §5.2.1, §5.3,
§5.4.1) written from the paper and SURVEY.md §8(c).  It shares no code with the
CUDA path (``paper_1603_07846_b200/``) and imports nothing from it.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import or execute this package.
The product path never routes through it.

Parity status per function is stated in each module header; every function is
pinned by a ``-m "not gpu"`` test (tests/test_oracle_*.py) except where a header
says "parity unpinned".
"""

from . import layers, net, partition, updater  # noqa: F401
