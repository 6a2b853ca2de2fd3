"""CPU ORACLE for NEXT row f4 (entropy-coded indices) — TEST INFRASTRUCTURE ONLY.

PAPER.md P:91-93 (§2.1): the positions of the k values kept in a chunk of C
form a k-subset, so log2 binom(C, k) bits per chunk ((1/k) log2 binom(C, k)
bits per value, "approximately 7.36" at C = 4096, k = 64) suffice; the paper
rejects such a code for its overhead and ships 12 bits/value.  This module is
the plain definition of a code that meets the bound to within one bit per
chunk: the combinatorial number system (enumerative coding).

Reading R#28 (the paper names no specific code):
  * the ascending positions p_0 < ... < p_{k-1} of a chunk of C_eff elements
    are ranked colexicographically, rank = sum_i binom(p_i, i + 1), an integer
    in [0, binom(C_eff, k)) — a bijection between k-subsets and that range;
  * the rank is written big-endian in W = ceil(log2 binom(C_eff, k)) bits
    (W = 0 when binom = 1, i.e. k = 0 or k = C_eff);
  * decode is the greedy inverse: for i = k-1 .. 0, p_i = the largest p with
    binom(p, i + 1) <= remaining rank.
Python integers are exact, so there is no rounding anywhere.  Only tests/ may
import this module.
"""
from __future__ import annotations

import math
from typing import List, Sequence


def code_bits(C: int, k: int) -> int:
    """W = ceil(log2 binom(C, k)) bits per chunk, exact integer arithmetic."""
    if not 0 <= k <= C:
        raise ValueError("need 0 <= k <= C")
    n = math.comb(C, k)
    return (n - 1).bit_length()


def rank(positions: Sequence[int], C: int) -> int:
    """Colex rank of an ascending k-subset of range(C)."""
    prev = -1
    r = 0
    for i, p in enumerate(positions):
        if not prev < p < C:
            raise ValueError("positions must be strictly increasing and < C")
        r += math.comb(p, i + 1)
        prev = p
    return r


def unrank(r: int, C: int, k: int) -> List[int]:
    """Inverse of rank: the k-subset of range(C) with colex rank r."""
    if not 0 <= r < math.comb(C, k):
        raise ValueError("rank out of range")
    out = [0] * k
    hi = C - 1
    for i in range(k - 1, -1, -1):
        p = hi
        while math.comb(p, i + 1) > r:
            p -= 1
        out[i] = p
        r -= math.comb(p, i + 1)
        hi = p - 1
    return out


def encode(positions: Sequence[int], C: int) -> str:
    """The chunk's index field as a bit string of exactly code_bits(C, k) characters (big-endian)."""
    W = code_bits(C, len(positions))
    r = rank(positions, C)
    return format(r, "b").zfill(W) if W else ""


def decode(bits: str, C: int, k: int) -> List[int]:
    W = code_bits(C, k)
    if len(bits) != W:
        raise ValueError(f"expected {W} bits, got {len(bits)}")
    return unrank(int(bits, 2) if W else 0, C, k)


def bits_per_value(C: int, k: int) -> float:
    """Realised index cost of the code, bits per transmitted value."""
    return code_bits(C, k) / k


# ---------------------------------------------------------------- entropy-coded device records (R#28)
# An entropy-coded ("EC") record replaces the 12-bit index stream of a device
# record (R#6) with the chunk's colex rank: 15 little-endian 32-bit limbs
# (rank < binom(C_eff, k_eff) <= binom(4096, 64) < 2^472, so the top 8 of the
# 480 bits are zero), followed by the record's code words (bit 2j = sign,
# 2j+1 = bucket of slot j, as R#6) and its scale word: 15 + ceil(2k/32) + 1
# words = 80 bytes at k = 64 (116 for the fixed-width record).
EC_RANK_LIMBS = 15


def ec_record_words(k: int = 64) -> int:
    return EC_RANK_LIMBS + (2 * k + 31) // 32 + 1


def ec_from_record(rec_words, n: int, k: int = 64, ib: int = 12):
    """EC record (list of uint32) of a fixed-width record (R#6 words) of a chunk
    of n positions: decode the ascending positions with the C oracle, rank them
    (plain definition), copy the code and scale words."""
    from . import decode_chunk, geom as _geom
    import numpy as np
    g = _geom(k=k, index_bits=ib)
    rec = np.asarray(rec_words, np.uint32)
    pos, _ = decode_chunk(rec, n, g)
    r = rank([int(p) for p in pos], n)
    assert r < 1 << (32 * EC_RANK_LIMBS)
    iw = (k * ib + 31) // 32
    cw = (2 * k + 31) // 32
    limbs = [(r >> (32 * i)) & 0xFFFFFFFF for i in range(EC_RANK_LIMBS)]
    return limbs + [int(w) for w in rec[iw:iw + cw]] + [int(rec[iw + cw])]


def record_from_ec(ec_words, n: int, k_eff: int, k: int = 64, ib: int = 12):
    """Inverse: the fixed-width record (R#6 layout, unused slots zero) of an EC record."""
    ec = [int(w) for w in ec_words]
    r = sum(ec[i] << (32 * i) for i in range(EC_RANK_LIMBS))
    pos = unrank(r, n, k_eff)
    iw = (k * ib + 31) // 32
    cw = (2 * k + 31) // 32
    words = [0] * (iw + cw + 1)
    for j, p in enumerate(pos):
        b = ib * j
        for bit in range(ib):
            if (p >> bit) & 1:
                words[(b + bit) // 32] |= 1 << ((b + bit) % 32)
    words[iw:iw + cw] = ec[EC_RANK_LIMBS:EC_RANK_LIMBS + cw]
    words[iw + cw] = ec[EC_RANK_LIMBS + cw]
    return words
