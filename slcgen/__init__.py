"""slcgen — seeded synthetic inputs for the SparseLoCo outer-step hot path.

Shared by both sides of the parity tests and by bench.py; contains no part of
the method's arithmetic (see gen.py).  Two bit-identical implementations:
  * ``generate``  — numpy, CPU (reference; used for oracle inputs and small cases)
  * ``fill_cuda`` — CUDA twin in gen_kernels.cu (libslcgen.so), for device buffers
"""
from __future__ import annotations

import ctypes
import os

from .gen import (WHAT_EF, WHAT_THETA, WHAT_THETA_LOCAL, FAMILY_NAMES, N_FAMILIES,  # noqa: F401
                  f32_to_bf16_bits, generate, generate_at, special_family)
from . import layouts  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslcgen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() first")
        lib = ctypes.CDLL(LIB_PATH)
        lib.slcgen_fill_cuda.restype = ctypes.c_int
        lib.slcgen_fill_cuda.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


def fill_cuda(out, what: int, seed: int, peer: int, G0: int, *, rowlen: int = 64,
              special_period: int = 0, warm_ef: bool = False, stream=None) -> None:
    """Fill the contiguous CUDA tensor `out` (float32, or bfloat16 for theta /
    theta_local) with global indices [G0, G0 + out.numel())."""
    import torch
    assert out.is_cuda and out.is_contiguous()
    if out.dtype == torch.bfloat16:
        bf = 1
    elif out.dtype == torch.float32:
        bf = 0
    else:
        raise TypeError(out.dtype)
    s = stream if stream is not None else torch.cuda.current_stream(out.device)
    rc = _load().slcgen_fill_cuda(what, seed, peer, G0, out.numel(), rowlen, special_period,
                                  int(bool(warm_ef)), bf, ctypes.c_void_p(out.data_ptr()),
                                  ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"slcgen_fill_cuda failed: cudaError {rc}")
