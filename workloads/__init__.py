"""Seeded synthetic workloads (configs + input generators) shared by the oracle and the CUDA path."""
from . import configs, generate  # noqa: F401
