"""CPU oracle of the f2 fast checks — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SPEC S:354-362 (`fast_checks`), for PAPER.md §2.2 P:98 ("fast checks on all
participants (e.g., liveness, synchronization with the main model, etc.)"):
  liveness  fails if no submission arrived inside the round window;
  sync      fails if base-round != current round or the layout digest mismatches;
  finite    fails if any decoded value is non-finite;
  norm-sane fails if the decoded norm > 10x the median of norm_history.
Reading R#29: the median of the history is the LOWER median (the
convention of S:283, as for median-norm R#20); the norm is the exact payload
norm of oracle.payload_norm (correctly rounded); the comparison is in binary64;
an empty history, or a payload already flagged non-finite, makes no norm check.  Plain definitions: every chunk is
decoded with the C oracle's decoder, nothing is fused or reordered.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import decode_chunk, geom as _geom, payload_norm

LIVENESS, SYNC, FINITE, NORM = 1, 2, 4, 8


def lower_median(xs: Sequence[float]) -> float:
    s = sorted(float(x) for x in xs)
    return s[(len(s) - 1) // 2]


def fast_checks(chunks: Optional[Sequence], current_round: int, norm_history: Sequence[float] = (),
                base_round: Optional[int] = None, digest: Optional[bytes] = None,
                expected_digest: Optional[bytes] = None, g=None) -> int:
    """Flags (LIVENESS | SYNC | FINITE | NORM bits) of one submission.

    chunks: [(record words, chunk length)] of the peer's payload, or None when
    nothing arrived; base_round / digest: the submission's header fields (None:
    not checked)."""
    if chunks is None:
        return LIVENESS
    g = g or _geom()
    flags = 0
    if base_round is not None and base_round != current_round:
        flags |= SYNC
    if digest is not None and expected_digest is not None and bytes(digest) != bytes(expected_digest):
        flags |= SYNC
    finite = True
    for rec, n in chunks:
        _, dq = decode_chunk(rec, n, g)
        finite &= bool(np.isfinite(dq).all())
    if not finite:
        flags |= FINITE  # R#29: a non-finite payload has no norm to check
    elif len(norm_history) > 0 and payload_norm(chunks, g) > 10.0 * lower_median(norm_history):
        flags |= NORM
    return flags
