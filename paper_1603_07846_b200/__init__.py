"""B200-native SINGA (arXiv 1603.07846) synchronous TrainOneBatch path.

The product is libsinga_b200.so (C ABI, include/singa_b200.h): hand-written
sm_100a kernels + NCCL.  ``_lib`` is the thin ctypes binding and ``net`` the
argument-marshalling helpers used by the tests and bench.py.
"""

__all__ = ["_lib", "net", "build"]
