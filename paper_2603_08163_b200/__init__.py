"""paper_2603_08163_b200 — B200-native (sm_100a) SparseLoCo outer-step hot path
(Covenant-72B, arxiv 2603.08163 §2.1).

  slc       ctypes binding of include/slc.h (libslc.so: compress / decode-aggregate / outer-update kernels)
  dist      one-process-per-GPU harness: shard payload all-gather and simulated-peer exchange over NCCL
"""
from . import slc  # noqa: F401  (fails loudly if libslc.so is missing)

__all__ = ["slc"]
