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
