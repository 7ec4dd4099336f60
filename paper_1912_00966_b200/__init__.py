"""paper_1912_00966_b200 -- B200-native earliest-arrival-time (EAT) engine.

The hot path of arXiv 1912.00966 (topology-driven Cluster-AP relaxation) as
a C-ABI library (libeat.so: host compressor + sm_100a CUDA kernels + NCCL
edge-partition driver, include/eat.h) with a thin Python binding.
"""
from ._lib import EAT_INF, EatError  # noqa: F401
from .engine import Engine, pinned_empty  # noqa: F401
