"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the probe's arithmetic (see synth/rng.py)."""
from . import rng, workloads  # noqa: F401
from .workloads import (PRED_DTYPE, PAIR_DTYPE, EQ, LT, LE, GT, GE, BETWEEN, NEGATE,  # noqa: F401
                        Workload, get)
