"""Synthetic parameter-set layouts (tensor shapes only, no method arithmetic).

Llama-style decoders, no biases, RMSNorm weights; 2-D weights stored
(out, in) row-major.  Layout order (= global flat order and global chunk
order):  embed, then per layer [attn_norm, q, k, v, o, ffn_norm, gate, up,
down], then final_norm, then lm_head if untied.

Sources: Covenant-72B shape table PAPER.md App. C Table `tab:model`
and §4.1 "Model": 80 layers, d=8192, 64 q / 8 kv heads, tied
embeddings, V=262,208, 72,747,327,488 parameters.  The FFN width is not
printed; reading A takes tied embeddings and
V=262,208 and solves for F=29,764, which reproduces the printed total exactly.
The smaller sets are public Llama shapes used as BASELINE.json configs 2, 3, 5.
"""
from __future__ import annotations

from typing import List, Tuple

Shape = Tuple[int, ...]
Layout = List[Tuple[str, Shape]]


def llama(d: int, L: int, n_heads: int, n_kv: int, F: int, V: int, tied: bool) -> Layout:
    hd = d // n_heads
    kv = n_kv * hd
    out: Layout = [("embed", (V, d))]
    for i in range(L):
        out += [
            (f"l{i}.attn_norm", (d,)),
            (f"l{i}.q", (d, d)),
            (f"l{i}.k", (kv, d)),
            (f"l{i}.v", (kv, d)),
            (f"l{i}.o", (d, d)),
            (f"l{i}.ffn_norm", (d,)),
            (f"l{i}.gate", (F, d)),
            (f"l{i}.up", (F, d)),
            (f"l{i}.down", (d, F)),
        ]
    out.append(("final_norm", (d,)))
    if not tied:
        out.append(("lm_head", (V, d)))
    return out


def numel(shape: Shape) -> int:
    n = 1
    for s in shape:
        n *= s
    return n


def total_params(layout: Layout) -> int:
    return sum(numel(s) for _, s in layout)


# Small ragged layout for parity tests: blocked 2-D tensors, 2-D tensors that
# must be flattened (a dim not divisible by 64), 1-D tensors with partial
# chunks (k_eff < k), a length-1 tensor, a 3-D tensor (flattened) and a tensor
# whose flat length is not a multiple of 4 (vector-load tail).
RAGGED: Layout = [
    ("w_a", (128, 192)),      # 2 x 3 blocks
    ("norm_a", (100,)),       # one partial chunk, k_eff = 1
    ("w_b", (130, 64)),       # 130 % 64 != 0 -> flattened: 8320 = 2 full + 1 partial (128)
    ("one", (1,)),            # single element
    ("w_c", (64, 64)),        # one block
    ("vec_d", (4096 * 3 + 2051,)),  # 3 full + partial 2051 (k_eff = 32)
    ("cube", (3, 40, 70)),    # 3-D -> flattened 8400
    ("odd", (4097,)),         # 1 full + partial of 1
    ("w_e", (256, 128)),      # 4 x 2 blocks
]

LAYOUTS = {
    # configs[0]: single 1M-element fp32 tensor (2-D and 1-D variants)
    "1m-2d": [("w", (1024, 1024))],
    "1m-1d": [("w", (1048576,))],
    # configs[1]: ~1B Llama (Llama-3.2-1B shapes)
    "llama3.2-1b": llama(d=2048, L=16, n_heads=32, n_kv=8, F=8192, V=128256, tied=True),
    # configs[2]: Llama-3-8B
    "llama3-8b": llama(d=4096, L=32, n_heads=32, n_kv=8, F=14336, V=128256, tied=False),
    # configs[3]: Covenant-72B, reading A (tied, V=262,208, F=29,764) and B
    "covenant-72b": llama(d=8192, L=80, n_heads=64, n_kv=8, F=29764, V=262208, tied=True),
    "covenant-72b-b": llama(d=8192, L=80, n_heads=64, n_kv=8, F=28672, V=262144, tied=False),
    # configs[4]: 7B sweep (Llama-2-7B shapes)
    "llama2-7b": llama(d=4096, L=32, n_heads=32, n_kv=32, F=11008, V=32000, tied=False),
    "ragged": RAGGED,
    # small Llama for multi-chunk-per-CTA tests (~12M params, ~3k chunks incl. partial norms)
    "llama-tiny": llama(d=512, L=2, n_heads=8, n_kv=2, F=1536, V=16384, tied=False),
    # bandwidth probes: the 1B parameter count as one flat tensor / as 64-row-blocked matrices
    "flat-1b": [("w", (1235814400,))],
}
