"""CPU ORACLE for the SparseLoCo outer-step hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2603_08163_b200) never imports it, and it imports nothing from the
product.  The arithmetic lives in plain C (slco.c, single-threaded, built
-O2 -ffp-contract=off -fno-fast-math); this module is ctypes marshalling.

Every function follows PAPER.md §2.1 Eq. 1 / P:88 / P:93 / P:176 /
Eq. 2; see slco.c for the step-by-step citations and DESIGN.md §3
for the readings R#1..R#26.  Parity status: Top-k, EF identity, aggregation,
outer update, chunking, record size and the printed closed forms are pinned by
tests/test_oracle.py and tests/test_oracle_pins.py (hand-worked cases for the
readings the paper leaves open: Q of R#1 per SPEC S:120, the R#13 tree, the
R#17 order and invR product, R#18 rounding); tools/oracle_mutants.py checks
that 27 plausible slips in slco.c each fail a pin.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SLCO_LIB: a mutated build of slco.c (tools/oracle_mutants.py checks that the pins catch it)
LIB_PATH = os.environ.get("SLCO_LIB") or os.path.join(_HERE, "libslco.so")
SRC = os.path.join(_HERE, "slco.c")
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]

OK, INVALID_ARGUMENT, INVALID_DATA, STALE = 0, 1, 2, 3
F32, BF16 = 0, 1


def build(force: bool = False) -> str:
    if os.environ.get("SLCO_LIB"):
        return LIB_PATH
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(_HERE, "slco.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB_PATH, SRC, "-lm"])
    return LIB_PATH


class Geom(ctypes.Structure):
    _fields_ = [("block", ctypes.c_int32), ("chunk", ctypes.c_int32), ("k", ctypes.c_int32),
                ("index_bits", ctypes.c_int32)]


def geom(block: int = 64, k: int = 64, index_bits: Optional[int] = None) -> Geom:
    C = block * block
    ib = index_bits if index_bits is not None else max(1, (C - 1).bit_length())
    return Geom(block, C, k, ib)


DEFAULT = None  # set after load

_lib = None
_P = ctypes.c_void_p


def _load():
    global _lib, DEFAULT
    if _lib is not None:
        return _lib
    build()
    L = ctypes.CDLL(LIB_PATH)
    G = ctypes.POINTER(Geom)
    i64p = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "slco_geom_check": (ctypes.c_int, [G]),
        "slco_is_blocked": (ctypes.c_int, [ctypes.c_int, i64p, G]),
        "slco_tensor_chunks": (ctypes.c_int64, [ctypes.c_int, i64p, G]),
        "slco_chunk_offsets": (ctypes.c_int, [ctypes.c_int, i64p, G, ctypes.c_int64, _P]),
        "slco_effective_k": (ctypes.c_int, [ctypes.c_int, G]),
        "slco_record_words": (ctypes.c_int, [G]),
        "slco_topk": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P]),
        "slco_tree_sum": (ctypes.c_float, [_P, ctypes.c_int, ctypes.c_int]),
        "slco_rn16": (ctypes.c_uint16, [ctypes.c_float]),
        "slco_f16_to_f32": (ctypes.c_float, [ctypes.c_uint16]),
        "slco_rnbf": (ctypes.c_uint16, [ctypes.c_float]),
        "slco_compress_chunk": (ctypes.c_int, [_P, _P, ctypes.c_int, _P, ctypes.c_int, G, ctypes.c_float, _P, _P]),
        "slco_decode_chunk": (ctypes.c_int, [_P, ctypes.c_int, G, _P, _P]),
        "slco_aggregate_chunk": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int, G, _P]),
        "slco_outer_update": (None, [_P, ctypes.c_int, _P, ctypes.c_int64, ctypes.c_float]),
        "slco_compress_tensor": (ctypes.c_int, [ctypes.c_int, i64p, _P, _P, ctypes.c_int, _P, G, ctypes.c_float,
                                                ctypes.c_int64, ctypes.c_int64, _P]),
        "slco_aggregate_tensor": (ctypes.c_int, [ctypes.c_int, i64p, _P, _P, _P, ctypes.c_int, G,
                                                 ctypes.c_int64, ctypes.c_int64, _P]),
        "slco_aggregate_update_tensor": (ctypes.c_int, [ctypes.c_int, i64p, _P, ctypes.c_int, _P, _P, _P,
                                                        ctypes.c_int, G, ctypes.c_int64, ctypes.c_int64,
                                                        ctypes.c_float]),
        "slco_index_entropy_bound": (ctypes.c_double, [ctypes.c_int, ctypes.c_int]),
        "slco_compression_ratio": (ctypes.c_double, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    DEFAULT = geom()
    return L


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _dims(shape):
    d = (ctypes.c_int64 * len(shape))(*shape)
    return len(shape), d


def _g(g):
    return ctypes.byref(g if g is not None else geom())


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.uint16:
        return BF16
    raise TypeError(f"theta arrays must be float32 or uint16 (bf16 bits), got {a.dtype}")


# ---------------------------------------------------------------- geometry
def is_blocked(shape, g=None) -> bool:
    n, d = _dims(shape)
    return bool(_load().slco_is_blocked(n, d, _g(g)))


def tensor_chunks(shape, g=None) -> int:
    n, d = _dims(shape)
    return int(_load().slco_tensor_chunks(n, d, _g(g)))


def chunk_offsets(shape, c: int, g=None) -> np.ndarray:
    g = g or geom()
    off = np.empty(g.chunk, np.int64)
    n, d = _dims(shape)
    m = _load().slco_chunk_offsets(n, d, ctypes.byref(g), c, _ptr(off))
    if m < 0:
        raise IndexError(c)
    return off[:m].copy()


def effective_k(n: int, g=None) -> int:
    return int(_load().slco_effective_k(n, _g(g)))


def record_words(g=None) -> int:
    return int(_load().slco_record_words(_g(g)))


def layout_chunks(layout, g=None):
    """Global chunk list: [(tensor_index, chunk_in_tensor, n_positions)] in layout order."""
    out = []
    for ti, (_, shape) in enumerate(layout):
        for c in range(tensor_chunks(shape, g)):
            out.append((ti, c))
    return out


# ---------------------------------------------------------------- steps
def topk(b: np.ndarray, k_eff: int) -> np.ndarray:
    b = np.ascontiguousarray(b, np.float32)
    sel = np.empty(max(k_eff, 1), np.int32)
    st = _load().slco_topk(_ptr(b), b.size, k_eff, _ptr(sel))
    if st != OK:
        raise ValueError(f"slco_topk status {st}")
    return sel[:k_eff].copy()


def tree_sum(x: np.ndarray, k: int) -> np.float32:
    x = np.ascontiguousarray(x, np.float32)
    return np.float32(_load().slco_tree_sum(_ptr(x), x.size, k))


def rn16(x: float) -> int:
    return int(_load().slco_rn16(float(x)))


def f16_to_f32(h: int) -> np.float32:
    return np.float32(_load().slco_f16_to_f32(int(h)))


def rnbf(x: float) -> int:
    return int(_load().slco_rnbf(float(x)))


def compress_chunk(a: np.ndarray, l: np.ndarray, e: np.ndarray, beta: float = 0.95, g=None):
    """Returns (status, record uint32[RW], e_new float32[n])."""
    g = g or geom()
    a = np.ascontiguousarray(a)
    l = np.ascontiguousarray(l)
    e = np.ascontiguousarray(e, np.float32)
    dt = _dtype_code(a)
    assert l.dtype == a.dtype and a.size == l.size == e.size
    rec = np.zeros(record_words(g), np.uint32)
    en = np.empty(e.size, np.float32)
    st = _load().slco_compress_chunk(_ptr(a), _ptr(l), dt, _ptr(e), e.size, ctypes.byref(g),
                                     ctypes.c_float(beta), _ptr(rec), _ptr(en))
    return st, rec, en


def decode_chunk(rec: np.ndarray, n: int, g=None):
    g = g or geom()
    rec = np.ascontiguousarray(rec, np.uint32)
    pos = np.empty(g.k, np.int32)
    dq = np.empty(g.k, np.float32)
    ke = _load().slco_decode_chunk(_ptr(rec), n, ctypes.byref(g), _ptr(pos), _ptr(dq))
    if ke < 0:
        raise ValueError("invalid record")
    return pos[:ke].copy(), dq[:ke].copy()


def _rec_ptrs(recs: Sequence[np.ndarray]):
    arrs = [np.ascontiguousarray(r, np.uint32) for r in recs]
    ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    return arrs, ptrs


def _ids_w(peer_ids, weights, R):
    ids = None if peer_ids is None else np.ascontiguousarray(peer_ids, np.uint8).reshape(R, 16)
    w = None if weights is None else np.ascontiguousarray(weights, np.float32).reshape(R)
    return ids, w, (None if ids is None else _ptr(ids)), (None if w is None else _ptr(w))


def aggregate_chunk(recs: Sequence[np.ndarray], n: int, peer_ids=None, weights=None, g=None) -> np.ndarray:
    g = g or geom()
    R = len(recs)
    arrs, ptrs = _rec_ptrs(recs)
    ids, w, pi, pw = _ids_w(peer_ids, weights, R)
    out = np.empty(n, np.float32)
    st = _load().slco_aggregate_chunk(ptrs, pi, pw, R, n, ctypes.byref(g), _ptr(out))
    if st != OK:
        raise ValueError(f"slco_aggregate_chunk status {st}")
    return out


def outer_update(theta: np.ndarray, delta: np.ndarray, alpha: float) -> np.ndarray:
    t = np.array(theta, copy=True)
    d = np.ascontiguousarray(delta, np.float32)
    assert t.size == d.size
    _load().slco_outer_update(_ptr(t), _dtype_code(t), _ptr(d), t.size, ctypes.c_float(alpha))
    return t


# ---------------------------------------------------------------- tensor level
def compress_tensor(shape, a, l, e, beta=0.95, c0=0, c1=None, g=None):
    """Compress chunks [c0, c1) of one tensor.  Returns (records uint32[c1-c0, RW], e_new)."""
    g = g or geom()
    c1 = tensor_chunks(shape, g) if c1 is None else c1
    a = np.ascontiguousarray(a).reshape(-1)
    l = np.ascontiguousarray(l).reshape(-1)
    en = np.array(e, dtype=np.float32, copy=True).reshape(-1)
    rec = np.zeros((max(c1 - c0, 0), record_words(g)), np.uint32)
    n, d = _dims(shape)
    st = _load().slco_compress_tensor(n, d, _ptr(a), _ptr(l), _dtype_code(a), _ptr(en), ctypes.byref(g),
                                      ctypes.c_float(beta), c0, c1, _ptr(rec))
    if st != OK:
        raise ValueError(f"slco_compress_tensor status {st}")
    return rec, en


def aggregate_tensor(shape, recs, peer_ids=None, weights=None, c0=0, c1=None, g=None):
    """Dense Delta for the whole tensor (positions outside [c0, c1) left 0)."""
    g = g or geom()
    c1 = tensor_chunks(shape, g) if c1 is None else c1
    R = len(recs)
    arrs, ptrs = _rec_ptrs(recs)
    ids, w, pi, pw = _ids_w(peer_ids, weights, R)
    numel = int(np.prod(shape))
    out = np.zeros(numel, np.float32)
    n, d = _dims(shape)
    st = _load().slco_aggregate_tensor(n, d, ptrs, pi, pw, R, ctypes.byref(g), c0, c1, _ptr(out))
    if st != OK:
        raise ValueError(f"slco_aggregate_tensor status {st}")
    return out


def aggregate_update_tensor(shape, theta, recs, alpha, peer_ids=None, weights=None, c0=0, c1=None, g=None):
    g = g or geom()
    c1 = tensor_chunks(shape, g) if c1 is None else c1
    R = len(recs)
    arrs, ptrs = _rec_ptrs(recs)
    ids, w, pi, pw = _ids_w(peer_ids, weights, R)
    t = np.array(theta, copy=True).reshape(-1)
    n, d = _dims(shape)
    st = _load().slco_aggregate_update_tensor(n, d, _ptr(t), _dtype_code(t), ptrs, pi, pw, R,
                                              ctypes.byref(g), c0, c1, ctypes.c_float(alpha))
    if st != OK:
        raise ValueError(f"slco_aggregate_update_tensor status {st}")
    return t


# ---------------------------------------------------------------- closed forms
def index_entropy_bound(C: int, k: int) -> float:
    return float(_load().slco_index_entropy_bound(C, k))


def compression_ratio(C: int, k: int, dense_bits: int, wire_bits_per_value: int) -> float:
    return float(_load().slco_compression_ratio(C, k, dense_bits, wire_bits_per_value))


# ---------------------------------------------------------------- median-norm (reading R#20)
def payload_norm(chunks, g=None) -> float:
    """||hatDelta_r||_2 of one peer's payload ("scaled relative to their
    median norm"), by the plain definition: decode every chunk (record,
    n_positions) and sum the squares of the decoded values.  Each value is an
    fp16 scale with a sign, so its square is exact in binary64 and math.fsum
    returns the correctly rounded sum of the exact squares; math.sqrt is
    correctly rounded.  (Reading R#20: the norm of the transmitted, decoded
    pseudo-gradient, computed per peer over the whole payload.)"""
    import math
    g = g or geom()
    sq = []
    for rec, n in chunks:
        _, dq = decode_chunk(rec, n, g)
        sq.extend(float(x) * float(x) for x in dq)
    return math.sqrt(math.fsum(sq))


def median_norm_weights(norms) -> np.ndarray:
    """Per-peer weights of the median-norm normalisation:
    m = lower median of the norms (S:283 design decision: lower median for
    even counts); a peer with norm > 0 is rescaled to norm m, w_r = m / n_r
    (binary64 division, then rounded to fp32: the weight enters Eq. 2 as an
    fp32 factor); zero norms pass through (w = 1)."""
    n = [float(x) for x in norms]
    if not n:
        raise ValueError("median_norm_weights: no peers")
    m = sorted(n)[(len(n) - 1) // 2]
    return np.array([np.float32(m / x) if x > 0 else np.float32(1.0) for x in n], np.float32)


def median_normalize(deltas):
    """SPEC S:280 median_normalize on dense deltas (test helper for the pins):
    every delta with norm > 0 rescaled to the lower-median norm."""
    import math
    norms = [math.sqrt(math.fsum(float(v) * float(v) for v in np.asarray(d, np.float64).ravel())) for d in deltas]
    m = sorted(norms)[(len(norms) - 1) // 2]
    return [np.asarray(d, np.float64) * (m / nn) if nn > 0 else np.asarray(d, np.float64) for d, nn in zip(deltas, norms)]
