"""Row f4 oracle (oracle/index_coding.py): enumerative index code pinned by brute force, the
textbook colex order, the paper's printed bound and exact bit-length inequalities."""
import itertools
import math
import random

import pytest

from oracle import index_coding as ic


@pytest.mark.parametrize("C,k", [(1, 0), (1, 1), (5, 2), (8, 3), (10, 4), (12, 6), (9, 9)])
def test_bijection_and_colex_order_brute_force(C, k):
    subsets = list(itertools.combinations(range(C), k))
    # colex order (textbook): compare subsets by their largest element first
    colex = sorted(subsets, key=lambda s: tuple(reversed(s)))
    assert [ic.rank(s, C) for s in colex] == list(range(math.comb(C, k)))
    for s in subsets:
        assert tuple(ic.decode(ic.encode(s, C), C, k)) == s


def test_paper_bound_and_width(golden):
    pv = golden["paper_values"]
    C, k = pv["chunk_size_C"]["value"], pv["top_k"]["value"]
    W = ic.code_bits(C, k)
    n = math.comb(C, k)
    assert 2 ** (W - 1) < n <= 2 ** W          # W = ceil(log2 binom(C, k)) by definition
    b = pv["index_entropy_bound_bits_per_value"]
    # within one bit per chunk of the bound the paper prints ("approximately 7.36")
    assert b["value"] - b["tolerance"] <= W / k <= b["value"] + b["tolerance"] + 1 / k
    assert W == 472
    assert ic.bits_per_value(C, k) < pv["index_bits_per_value"]["value"]  # beats the shipped 12 bits/value


def test_round_trip_paper_size_and_partial_chunks():
    rng = random.Random(20260319)
    for C, k in [(4096, 64), (4096, 1), (4096, 4095), (1000, 16), (4097 - 1, 63), (64, 64), (37, 1)]:
        for _ in range(20):
            s = sorted(rng.sample(range(C), k))
            bits = ic.encode(s, C)
            assert len(bits) == ic.code_bits(C, k)
            assert ic.decode(bits, C, k) == s


def test_extremes():
    C, k = 4096, 64
    assert ic.encode(list(range(k)), C) == "0" * ic.code_bits(C, k)         # colex-first subset
    top = list(range(C - k, C))
    assert ic.rank(top, C) == math.comb(C, k) - 1                             # colex-last subset
    assert ic.encode([], C) == "" and ic.decode("", C, 0) == []
    assert ic.encode(list(range(7)), 7) == ""                                 # k = C: one subset, zero bits
    with pytest.raises(ValueError):
        ic.rank([3, 3], C)
    with pytest.raises(ValueError):
        ic.rank([5, C], C)
    with pytest.raises(ValueError):
        ic.decode("0" * 471, C, k)
