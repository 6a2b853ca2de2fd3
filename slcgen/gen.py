"""Seeded synthetic-input generator (numpy reference implementation).

This module is shared by the oracle side and the CUDA side of the tests and by
bench.py.  It holds NONE of the method's arithmetic (no pseudo-gradient, no
Top-k, no quantiser, no aggregation): it only draws the synthetic inputs
theta (global params), theta_local (a peer's params after H inner steps) and
e (a peer's error-feedback buffer).

Every value is a pure function of (seed, stream, G) where G is the GLOBAL flat
index of the element in the param set (tensors concatenated in layout order, no
padding).  Any sharding of the param set therefore sees identical values, which
is what makes the sharding-invariance tests meaningful.  Only integer hashing
(splitmix64) and exact fp32 operations are used (power-of-two scalings of
24-bit integers, one rounded multiply and one rounded subtraction), so the CUDA
twin in ``gen_kernels.cu`` reproduces it bit for bit.

Value recipe (magnitudes follow PAPER.md §4.1
P:176-177, H*lr <= 30 * 1.2e-4):
  theta        = 0.02*sqrt(3) * ((u0+u1)+(u2+u3) - 2)     Irwin-Hall-4, ~N(0, 0.02^2)
  delta_target = 2^-9 * (u - 1/2) * 2^-j * 2^-s           j in 0..7 per element,
                                                           s in 0..3 per `rowlen` run
  theta_local  = theta - delta_target                      (fp32, one rounding)
  e            = 0 (cold)  or  2^-7 * (u - 1/2) * 2^-j    (warm)
Special 4096-element runs (run = G >> 12, selected with probability
1/special_period) replace the recipe with one of 8 degenerate families
(zero, constant, discrete ties, signed zeros, subnormals, spike, sparse,
equal-magnitude random signs).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

# stream ids (peer r adds r)
S_THETA = 1
S_DELTA = 1000
S_ROWSCALE = 3000
S_EF = 5000
S_SPECIAL = 7000

THETA_SCALE = np.float32(0.034641016151377546)  # 0.02*sqrt(3) rounded to fp32

WHAT_THETA = 0
WHAT_THETA_LOCAL = 1
WHAT_EF = 2

N_FAMILIES = 8
FAMILY_NAMES = ["zero", "constant", "ties", "signed_zero", "subnormal", "spike",
                "sparse", "equal_magnitude"]


def _u64(x):
    return np.asarray(x, dtype=np.uint64)


def mix64(z):
    z = _u64(z)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * M1
        z = z ^ (z >> np.uint64(27))
        z = z * M2
        z = z ^ (z >> np.uint64(31))
    return z


def stream_key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = mix64(_u64(seed) ^ GOLDEN)
        k = k + _u64(stream) * STREAM_MUL + np.uint64(1)
        return mix64(k)


def hash_at(seed: int, stream: int, G):
    """h(seed, stream, G) = mix64(key(seed, stream) + (G + 1) * GOLDEN)."""
    k = stream_key(seed, stream)
    with np.errstate(over="ignore"):
        return mix64(k + (_u64(G) + np.uint64(1)) * GOLDEN)


def _u24(h):
    # exact: 24-bit integer times 2^-24
    return (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)


def _pow2_neg(j):
    # exact 2^-j for small non-negative integer arrays
    return np.ldexp(np.float32(1.0), -j.astype(np.int32)).astype(np.float32)


def theta_values(seed, G):
    h = hash_at(seed, S_THETA, G)
    f = np.float32(2.0 ** -16)
    u = [((h >> np.uint64(16 * i)) & np.uint64(0xFFFF)).astype(np.float32) * f for i in range(4)]
    s = (u[0] + u[1]) + (u[2] + u[3])
    s = s - np.float32(2.0)
    return (s * THETA_SCALE).astype(np.float32)


def delta_target_values(seed, peer, G, rowlen):
    h = hash_at(seed, S_DELTA + peer, G)
    u = _u24(h)
    j = (h >> np.uint64(8)) & np.uint64(7)
    hs = hash_at(seed, S_ROWSCALE + peer, _u64(G) // np.uint64(rowlen))
    s = hs & np.uint64(3)
    v = (u - np.float32(0.5)) * np.float32(2.0 ** -9)
    v = v * _pow2_neg(j)
    v = v * _pow2_neg(s)
    return v.astype(np.float32)


def ef_values(seed, peer, G):
    h = hash_at(seed, S_EF + peer, G)
    u = _u24(h)
    j = (h >> np.uint64(8)) & np.uint64(7)
    v = (u - np.float32(0.5)) * np.float32(2.0 ** -7)
    return (v * _pow2_neg(j)).astype(np.float32)


def special_family(seed, G, period):
    """Family id (0..7) of the special run containing G, or -1.  Keyed on the
    seed only, so theta (shared by all peers) and every peer agree on it."""
    G = _u64(G)
    if period <= 0:
        return np.full(G.shape, -1, dtype=np.int32)
    hs = hash_at(seed, S_SPECIAL, G >> np.uint64(12))
    sel = (hs % np.uint64(period)) == np.uint64(0)
    fam = ((hs >> np.uint64(32)) % np.uint64(N_FAMILIES)).astype(np.int32)
    return np.where(sel, fam, -1).astype(np.int32)


def _special(seed, peer, G, fam, rowlen):
    """(theta, theta_local, e) for elements inside special runs of family fam.
    theta depends on (seed, G) only; theta_local and e also on the peer."""
    G = _u64(G)
    h = hash_at(seed, S_DELTA + peer, G)
    ht = hash_at(seed, S_THETA, G)
    hs = hash_at(seed, S_SPECIAL, G >> np.uint64(12))
    zero = np.zeros(G.shape, np.float32)
    th = zero.copy()
    ef = zero.copy()
    sign = np.where((h >> np.uint64(63)) == np.uint64(1), np.float32(-1.0), np.float32(1.0))
    if fam == 0:                      # all zero
        d = zero
    elif fam == 1:                    # constant +-c, one sign per run
        c = (((hs >> np.uint64(40)) & np.uint64(7)).astype(np.float32) + np.float32(1.0)) * np.float32(2.0 ** -10)
        rs = np.where(((hs >> np.uint64(20)) & np.uint64(1)) == np.uint64(1), np.float32(-1.0), np.float32(1.0))
        d = (c * rs).astype(np.float32)
    elif fam == 2:                    # discrete ties {+-1,+-2,+-3} * 2^-10
        m = ((h >> np.uint64(8)) % np.uint64(3)).astype(np.float32) + np.float32(1.0)
        d = (m * np.float32(2.0 ** -10) * sign).astype(np.float32)
    elif fam == 3:                    # signed zeros in theta, theta_local and e
        s1 = (ht >> np.uint64(1)) & np.uint64(1)
        s2 = (h >> np.uint64(2)) & np.uint64(1)
        s3 = (h >> np.uint64(3)) & np.uint64(1)
        th = np.where(s1 == 1, np.float32(-0.0), np.float32(0.0)).astype(np.float32)
        tl = np.where(s2 == 1, np.float32(-0.0), np.float32(0.0)).astype(np.float32)
        ef = np.where(s3 == 1, np.float32(-0.0), np.float32(0.0)).astype(np.float32)
        return th, tl, ef
    elif fam == 4:                    # fp32 subnormals
        mant = ((h >> np.uint64(40)) & np.uint64(0x7FFFFF)).astype(np.float32)
        d = (mant * np.float32(2.0 ** -149) * sign).astype(np.float32)
    elif fam == 5:                    # one spike x1024 on top of the normal recipe
        d = delta_target_values(seed, peer, G, rowlen)
        spike_at = (hs >> np.uint64(8)) & np.uint64(4095)
        d = np.where((G & np.uint64(4095)) == spike_at, d * np.float32(1024.0), d).astype(np.float32)
        th = theta_values(seed, G)
        return th, (th - d).astype(np.float32), ef
    elif fam == 6:                    # sparse: ~1/128 nonzero (fewer than k per chunk)
        dd = delta_target_values(seed, peer, G, rowlen)
        d = np.where((h & np.uint64(127)) == np.uint64(0), dd, np.float32(0.0)).astype(np.float32)
    else:                             # equal magnitude, random signs
        d = (np.float32(2.0 ** -10) * sign).astype(np.float32)
    # theta = 0 so that d = 0 - (0 - d) reproduces d exactly
    return th, (th - d).astype(np.float32), ef


def generate(what: int, seed: int, peer: int, G0: int, n: int, *, rowlen: int = 64,
             special_period: int = 0, warm_ef: bool = False, dtype: str = "f32") -> np.ndarray:
    """Values of `what` for global indices [G0, G0+n).  dtype 'f32' -> float32,
    'bf16' -> uint16 bit patterns (round-to-nearest-even; only theta/theta_local)."""
    return generate_at(what, seed, peer, np.arange(G0, G0 + n, dtype=np.uint64), rowlen=rowlen,
                       special_period=special_period, warm_ef=warm_ef, dtype=dtype)


def generate_at(what: int, seed: int, peer: int, G, *, rowlen: int = 64, special_period: int = 0,
                warm_ef: bool = False, dtype: str = "f32") -> np.ndarray:
    """Values of `what` at an arbitrary array of global indices G."""
    G = np.ascontiguousarray(G, dtype=np.uint64).reshape(-1)
    n = G.size
    if what == WHAT_THETA:
        out = theta_values(seed, G)
    elif what == WHAT_THETA_LOCAL:
        out = (theta_values(seed, G) - delta_target_values(seed, peer, G, rowlen)).astype(np.float32)
    elif what == WHAT_EF:
        out = ef_values(seed, peer, G) if warm_ef else np.zeros(n, np.float32)
    else:
        raise ValueError(what)
    if special_period > 0:
        fam = special_family(seed, G, special_period)
        for f in range(N_FAMILIES):
            m = fam == f
            if m.any():
                th, tl, ef = _special(seed, peer, G[m], f, rowlen)
                out[m] = (th, tl, ef)[what]
    if dtype == "bf16":
        if what == WHAT_EF:
            raise ValueError("error feedback is fp32")
        return f32_to_bf16_bits(out)
    return out


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round to nearest even (finite inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)
