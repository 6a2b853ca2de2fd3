"""Mutation check of the CPU oracle's pins (VERDICT r1 "What's weak #1").

Each mutant is one plausible slip in oracle/slco.c (a dropped term, a wrong
sign, index, bound, rounding or order).  The script builds every mutant into a
temporary libslco.so and runs the CPU pin suites against it (SLCO_LIB points
the oracle's ctypes loader at the mutant).  A mutant is KILLED when at least
one pin fails.  Exit status 0 only if every mutant is killed.

  python tools/oracle_mutants.py [-k NAME] [--list]

Output: one line per mutant; the committed log is profiles/r02_oracle_mutants.txt.
Equivalent mutants (no input can tell them apart) are left out, e.g. padding
the tree sum to 32*ceil(k_eff/32) instead of 32*ceil(k/32) slots: the extra
slots only add +0 to non-negative magnitudes.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "slco.c")
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]
PIN_SUITES = ["tests/test_oracle.py", "tests/test_oracle_pins.py", "tests/test_records_cpu.py",
              "tests/test_wire_cpu.py", "tests/test_index_coding_cpu.py"]

# (name, reading / passage it violates, [(old, new), ...]) — every `old` must occur exactly once
MUTANTS = [
    ("M1-tau-over-k", "R#10/S:120: tau = mean over the k_eff selected values",
     [("slco_tree_sum(av, k_eff, g->k) / (float)k_eff", "slco_tree_sum(av, k_eff, g->k) / (float)g->k")]),
    ("M2-bucket-ge", "S:120: |v| <= tau goes to the low bucket",
     [("h[j] = av[j] > tau;", "h[j] = av[j] >= tau;")]),
    ("M3-shi-fallback-0", "S:120: scale-hi tau-fallback when the high bucket is empty",
     [("n_hi > 0 ? sum_hi / (float)n_hi : tau;", "n_hi > 0 ? sum_hi / (float)n_hi : 0.0f;")]),
    ("M4-weighted-product-fp32", "R#17/R#20: w_r * dq in fp64 (exact)",
     [("acc[pos[j]] += wr * (double)dq[j];", "acc[pos[j]] += (double)((float)wr * dq[j]);")]),
    ("M5a-butterfly-adjacent", "R#13: butterfly strides 16, 8, 4, 2, 1",
     [("for (int d = 16; d >= 1; d /= 2)\n    for (int l = 0; l < d; l++) u[l] = u[l] + u[l + d];",
       "for (int d = 1; d < 32; d *= 2)\n    for (int l = 0; l + d < 32; l += 2 * d) u[l] = u[l] + u[l + d];")]),
    ("M5b-butterfly-increasing", "R#13: butterfly strides decrease",
     [("for (int d = 16; d >= 1; d /= 2)\n    for (int l = 0; l < d; l++) u[l] = u[l] + u[l + d];",
       "for (int d = 1; d <= 16; d *= 2)\n    for (int l = 0; l < 32; l += 2 * d) u[l] = u[l] + u[l + d];")]),
    ("M5c-lane-contiguous", "R#13: lane l holds slots l, l+32, ...",
     [("u[l] = (l < n) ? x[l] : 0.0f;", "u[l] = (l * W < n) ? x[l * W] : 0.0f;"),
      ("int s = l + 32 * m;", "int s = l * W + m;")]),
    ("M5d-sequential-sum", "R#13: fixed tree, not left-to-right",
     [("  return u[0];\n}", "  float acc = 0.0f;\n  for (int s = 0; s < n && s < K; s++) acc = acc + x[s];\n"
                            "  return acc;\n}")]),
    ("M6-no-canonical-peer-order", "R#17: fp64 sum in ascending peer-id order",
     [("if (peer_ids) qsort(order", "if (0) qsort(order")]),
    ("M6b-descending-peer-order", "R#17: ascending peer-id order",
     [("int c = memcmp(a->id, b->id, 16);", "int c = -memcmp(a->id, b->id, 16);")]),
    ("M7-divide-by-R", "R#17: Delta = (float)(acc * (1.0/R))",
     [("delta[p] = (float)(acc[p] * invR);", "delta[p] = (float)(acc[p] / (double)R);")]),
    ("M8-tie-higher-index", "R#4: ties go to the lower index",
     [("return (a->pos > b->pos) - (a->pos < b->pos);", "return (a->pos < b->pos) - (a->pos > b->pos);")]),
    ("M9-unfused-ef", "R#12: b = fma(beta, e, d)",
     [("b[p] = fmaf(beta, e[p], d);", "b[p] = beta * e[p] + d;")]),
    ("M10-ef-sign", "Eq. 1 line 3 (P:73): e <- b - hatDelta",
     [("e_new[S[j]] = b[S[j]] - dq;", "e_new[S[j]] = b[S[j]] + dq;")]),
    ("M11-divisor-R+1", "Eq. 2 (P:82): mean over R",
     [("const double invR = 1.0 / (double)R;", "const double invR = 1.0 / (double)(R + 1);")]),
    ("M12-transposed-block", "R#7: p = 64*r + c",
     [("off[B * r + col] = (bi * B + r) * cols + bj * B + col;",
       "off[B * col + r] = (bi * B + r) * cols + bj * B + col;")]),
    ("M13-sign-of-negative-zero", "S:120 code = sign bit; R#25 literal -0",
     [("put_bit(rec + IW, 2 * j, signbit(b[S[j]]) ? 1u : 0u);", "put_bit(rec + IW, 2 * j, b[S[j]] < 0.0f ? 1u : 0u);")]),
    ("M14-keff-ceil", "R#10/S:56: floor(k*len/C)",
     [("int64_t ke = ((int64_t)g->k * n) / g->chunk;", "int64_t ke = ((int64_t)g->k * n + g->chunk - 1) / g->chunk;")]),
    ("M15-code-bits-swapped", "R#6: bit 2j sign, 2j+1 bucket (writer and reader)",
     [("put_bit(rec + IW, 2 * j, signbit(b[S[j]]) ? 1u : 0u);\n    put_bit(rec + IW, 2 * j + 1, (uint32_t)h[j]);",
       "put_bit(rec + IW, 2 * j + 1, signbit(b[S[j]]) ? 1u : 0u);\n    put_bit(rec + IW, 2 * j, (uint32_t)h[j]);"),
      ("const uint32_t sgn = get_bit(rec + IW, 2 * j), hb = get_bit(rec + IW, 2 * j + 1);",
       "const uint32_t sgn = get_bit(rec + IW, 2 * j + 1), hb = get_bit(rec + IW, 2 * j);")]),
    ("M16-index-msb-first", "R#6: index bit b at stream bit 12j + b (writer and reader)",
     [("put_bit(rec, (int64_t)g->index_bits * j + bit, ((uint32_t)S[j] >> bit) & 1u);",
       "put_bit(rec, (int64_t)g->index_bits * j + (g->index_bits - 1 - bit), ((uint32_t)S[j] >> bit) & 1u);"),
      ("p |= get_bit(rec, (int64_t)g->index_bits * j + bit) << bit;",
       "p |= get_bit(rec, (int64_t)g->index_bits * j + (g->index_bits - 1 - bit)) << bit;")]),
    ("M17-rn16-truncate", "R#14: fp16 round-to-nearest-even",
     [("_Float16 h = (_Float16)x;", "uint32_t tu_ = f2u(x) & 0xFFFFE000u; _Float16 h = (_Float16)u2f(tu_);")]),
    ("M18-unfused-update-f32", "R#18: theta <- fma(-alpha, Delta, theta)",
     [("t[i] = fmaf(-alpha, delta[i], t[i]);", "t[i] = t[i] - alpha * delta[i];")]),
    ("M19-unfused-update-bf16", "R#18: bf16 theta: rnbf(fma(-alpha, Delta, f32(theta)))",
     [("t[i] = slco_rnbf(fmaf(-alpha, delta[i], x));", "t[i] = slco_rnbf(x - alpha * delta[i]);")]),
    ("M20-weights-ignored", "Eq. 2 with median-norm weights (R#20)",
     [("const double wr = w ? (double)w[r] : 1.0;", "const double wr = 1.0;")]),
    ("M21-topk-on-delta", "Eq. 1 line 2: Top-k of beta*e + Delta",
     [("b[p] = fmaf(beta, e[p], d);", "b[p] = d + 0.0f * e[p];")]),
    ("M22-selected-ascending-dropped", "R#5: selected positions ascending",
     [("qsort(sel, (size_t)k_eff, sizeof(int32_t), cmp_i32);", "(void)cmp_i32;")]),
    ("M23-bf16-widen-truncated-theta", "R#18: bf16 rounding RN-even",
     [("return (uint16_t)((u + 0x7FFFu + lsb) >> 16);", "return (uint16_t)((u + 0x8000u) >> 16);")]),
]


def apply(src: str, edits):
    out = src
    for old, new in edits:
        cnt = out.count(old)
        if cnt != 1:
            raise SystemExit(f"mutant edit not unique ({cnt}x): {old[:60]!r}")
        out = out.replace(old, new)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default=None)
    ap.add_argument("--list", action="store_true")
    args = ap.parse_args()
    src = open(SRC).read()
    sel = [m for m in MUTANTS if args.k is None or args.k in m[0]]
    if args.list:
        for name, why, _ in sel:
            print(f"{name:32s} {why}")
        return 0
    survivors = []
    with tempfile.TemporaryDirectory() as td:
        for name, why, edits in sel:
            csrc = os.path.join(td, f"{name}.c")
            with open(csrc, "w") as f:
                f.write(apply(src, edits))
            lib = os.path.join(td, f"lib_{name}.so")
            subprocess.check_call(["gcc", *CFLAGS, "-I", os.path.join(ROOT, "oracle"), "-o", lib, csrc, "-lm"])
            env = dict(os.environ, SLCO_LIB=lib)
            t0 = time.time()
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                                *PIN_SUITES], cwd=ROOT, env=env, capture_output=True, text=True)
            failed = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            verdict = "KILLED" if r.returncode != 0 else "SURVIVED"
            if r.returncode == 0:
                survivors.append(name)
            by = failed[0].split(" ")[1] if failed else ""
            print(f"{verdict:8s} {name:32s} {time.time() - t0:5.1f}s  {by}   [{why}]", flush=True)
    print(f"{len(sel) - len(survivors)}/{len(sel)} mutants killed" + (f"; survivors: {survivors}" if survivors else ""))
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
