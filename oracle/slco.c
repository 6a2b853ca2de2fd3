/* slco.c — CPU ORACLE for the SparseLoCo outer-step hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see slco.h).  Written from PAPER.md §2.1:
 *   Eq. 1   Delta_r = theta - theta_r^(t,H);
 *                     hatDelta_r = Q(Top-k(beta*e_r + Delta_r));
 *                     e_r <- beta*e_r + Delta_r - hatDelta_r
 *   P:88              chunk-wise Top-k: 64x64 blocks of 2-D tensors, 4096-chunks of 1-D
 *   P:93              12 bits per transmitted index
 *   P:176             C = 4096, k = 64, beta = 0.95, alpha = 1, 2-bit values
 *   Eq. 2   Delta = (1/R) sum_r hatDelta_r;  theta <- theta - alpha*Delta
 * Readings of what the paper leaves open are DESIGN.md §3 R#1..R#26.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared.
 * Every float operation below is a single IEEE binary32 (or binary64 where
 * stated) operation, rounded to nearest even; fmaf is libm's correctly
 * rounded fused multiply-add.
 */
#include "slco.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* small helpers                                                       */
/* ------------------------------------------------------------------ */
static uint32_t f2u(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static float u2f(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }

uint16_t slco_rn16(float x) {
  /* R#14: binary16 round-to-nearest-even including subnormals; overflow -> inf */
  _Float16 h = (_Float16)x;
  uint16_t r; memcpy(&r, &h, 2); return r;
}

float slco_f16_to_f32(uint16_t bits) {
  _Float16 h; memcpy(&h, &bits, 2); return (float)h;
}

uint16_t slco_rnbf(float x) {
  uint32_t u = f2u(x);
  if (isnan(x)) return (uint16_t)((u >> 16) | 0x40); /* quiet NaN */
  uint32_t lsb = (u >> 16) & 1u;
  return (uint16_t)((u + 0x7FFFu + lsb) >> 16);
}

static float widen(const void* p, int dtype, int64_t i) {
  if (dtype == SLCO_BF16) return u2f(((uint32_t)((const uint16_t*)p)[i]) << 16);
  return ((const float*)p)[i];
}

/* ------------------------------------------------------------------ */
/* chunk geometry — P:88 "each 2D tensor is partitioned into           */
/* non-overlapping 64x64 blocks and each 1D tensor into contiguous     */
/* chunks of size 4096"; C = 4096, k = 64.                     */
/* ------------------------------------------------------------------ */
int slco_geom_check(const slco_geom* g) {
  if (!g || g->block <= 0 || g->chunk != g->block * g->block) return SLCO_INVALID_ARGUMENT;
  if (g->k < 1 || g->k > g->chunk) return SLCO_INVALID_ARGUMENT;
  if (g->index_bits < 1 || g->index_bits > 16 || (1L << g->index_bits) < g->chunk) return SLCO_INVALID_ARGUMENT;
  return SLCO_OK;
}

/* R#9: only a 2-D tensor with both dims divisible by the block side is cut
 * into blocks; anything else (1-D, 3-D, ragged 2-D) is flattened to 1-D. */
int slco_is_blocked(int ndim, const int64_t* dims, const slco_geom* g) {
  return ndim == 2 && dims[0] % g->block == 0 && dims[1] % g->block == 0;
}

static int64_t numel(int ndim, const int64_t* dims) {
  int64_t n = 1;
  for (int i = 0; i < ndim; i++) n *= dims[i];
  return n;
}

int64_t slco_tensor_chunks(int ndim, const int64_t* dims, const slco_geom* g) {
  if (slco_is_blocked(ndim, dims, g)) return (dims[0] / g->block) * (dims[1] / g->block);
  int64_t n = numel(ndim, dims);
  return (n + g->chunk - 1) / g->chunk;
}

/* R#7, R#8: blocks enumerated row-major; in-block position p = B*r + c.
 * 1-D: chunk c holds flat offsets [c*C, min(N, (c+1)*C)), p = offset - c*C. */
int slco_chunk_offsets(int ndim, const int64_t* dims, const slco_geom* g, int64_t c, int64_t* off) {
  if (c < 0 || c >= slco_tensor_chunks(ndim, dims, g)) return -1;
  if (slco_is_blocked(ndim, dims, g)) {
    const int64_t B = g->block, cols = dims[1], nb = cols / B;
    const int64_t bi = c / nb, bj = c % nb;
    for (int64_t r = 0; r < B; r++)
      for (int64_t col = 0; col < B; col++)
        off[B * r + col] = (bi * B + r) * cols + bj * B + col;
    return (int)(B * B);
  }
  const int64_t N = numel(ndim, dims);
  const int64_t start = c * g->chunk;
  int64_t n = N - start;
  if (n > g->chunk) n = g->chunk;
  for (int64_t p = 0; p < n; p++) off[p] = start + p;
  return (int)n;
}

/* R#10: partial chunk of n < C positions sends k_eff = max(1, floor(k*n/C)). */
int slco_effective_k(int n, const slco_geom* g) {
  int64_t ke = ((int64_t)g->k * n) / g->chunk;
  return ke < 1 ? 1 : (int)ke;
}

/* R#6: record = k fixed-width indices + k 2-bit codes + one
 * word of two fp16 scales, each part padded to 32-bit words. */
static int idx_words(const slco_geom* g) { return (g->k * g->index_bits + 31) / 32; }
static int code_words(const slco_geom* g) { return (2 * g->k + 31) / 32; }
int slco_record_words(const slco_geom* g) { return idx_words(g) + code_words(g) + 1; }

/* ------------------------------------------------------------------ */
/* Top-k ("Top-k", "Top-k is applied separately within each */
/* chunk").  Plain definition: sort all positions by |b| descending,   */
/* ties by position ascending (R#3, R#4), keep the first k_eff, return */
/* them in ascending position order (R#5).                             */
/* ------------------------------------------------------------------ */
typedef struct { float mag; int32_t pos; } mag_pos;

static int cmp_mag_desc(const void* x, const void* y) {
  const mag_pos* a = (const mag_pos*)x; const mag_pos* b = (const mag_pos*)y;
  if (a->mag > b->mag) return -1;
  if (a->mag < b->mag) return 1;
  return (a->pos > b->pos) - (a->pos < b->pos);
}
static int cmp_i32(const void* x, const void* y) {
  int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
  return (a > b) - (a < b);
}

int slco_topk(const float* b, int n, int k_eff, int32_t* sel) {
  if (k_eff < 0 || k_eff > n) return SLCO_INVALID_ARGUMENT;
  mag_pos* v = (mag_pos*)malloc(sizeof(mag_pos) * (size_t)(n > 0 ? n : 1));
  if (!v) return SLCO_INVALID_ARGUMENT;
  for (int p = 0; p < n; p++) {
    if (!isfinite(b[p])) { free(v); return SLCO_INVALID_DATA; }
    v[p].mag = fabsf(b[p]);  /* -0 and +0 have equal magnitude */
    v[p].pos = p;
  }
  qsort(v, (size_t)n, sizeof(mag_pos), cmp_mag_desc);
  for (int j = 0; j < k_eff; j++) sel[j] = v[j].pos;
  qsort(sel, (size_t)k_eff, sizeof(int32_t), cmp_i32);
  free(v);
  return SLCO_OK;
}

/* R#13 tree-sum T: pad x to K = 32*ceil(k/32) slots with +0; lane sums
 * u_l = x_l + x_{l+32} + ... in increasing slot order (l = 0..31); then for
 * d = 16, 8, 4, 2, 1 and l < d: u_l = u_l + u_{l+d}; result u_0. */
float slco_tree_sum(const float* x, int n, int k) {
  const int W = (k + 31) / 32;
  const int K = 32 * W;
  float u[32];
  for (int l = 0; l < 32; l++) {
    u[l] = (l < n) ? x[l] : 0.0f;
    for (int m = 1; m < W; m++) {
      int s = l + 32 * m;
      u[l] = u[l] + ((s < n && s < K) ? x[s] : 0.0f);
    }
  }
  for (int d = 16; d >= 1; d /= 2)
    for (int l = 0; l < d; l++) u[l] = u[l] + u[l + d];
  return u[0];
}

/* ------------------------------------------------------------------ */
/* record bit writer / reader (R#6)                                    */
/* index stream: slot j occupies stream bits [ib*j, ib*j+ib), stream   */
/*   bit s = bit (s%32) of word s/32, words 0..idx_words-1;            */
/* code stream: bit 2j = sign of v_j, bit 2j+1 = bucket h_j, words     */
/*   idx_words..idx_words+code_words-1;                                */
/* last word: bits 0-15 fp16 S_lo, bits 16-31 fp16 S_hi.              */
/* Slots j >= k_eff are all-zero.                                      */
/* ------------------------------------------------------------------ */
static void put_bit(uint32_t* w, int64_t s, uint32_t bit) {
  if (bit) w[s / 32] |= (1u << (s % 32));
}
static uint32_t get_bit(const uint32_t* w, int64_t s) { return (w[s / 32] >> (s % 32)) & 1u; }

/* ------------------------------------------------------------------ */
/* Eq. 1 for one chunk.                                      */
/* ------------------------------------------------------------------ */
int slco_compress_chunk(const void* a, const void* l, int dtype, const float* e, int n,
                        const slco_geom* g, float beta, uint32_t* rec, float* e_new) {
  if (slco_geom_check(g) != SLCO_OK || n < 1 || n > g->chunk) return SLCO_INVALID_ARGUMENT;
  const int k_eff = slco_effective_k(n, g);
  float* b = (float*)malloc(sizeof(float) * (size_t)n);
  int32_t* S = (int32_t*)malloc(sizeof(int32_t) * (size_t)k_eff);
  float* av = (float*)malloc(sizeof(float) * (size_t)k_eff);
  float* lo = (float*)malloc(sizeof(float) * (size_t)k_eff);
  float* hi = (float*)malloc(sizeof(float) * (size_t)k_eff);
  int* h = (int*)malloc(sizeof(int) * (size_t)k_eff);
  int st = SLCO_OK;
  if (!b || !S || !av || !lo || !hi || !h) { st = SLCO_INVALID_ARGUMENT; goto done; }

  /* step 1 — pseudo-gradient Delta = theta - theta_local (Eq. 1 line 1)
   * and EF accumulation beta*e + Delta (Eq. 1 line 2); R#12: the
   * product is fused, b = fma(beta, e, d). R#15: non-finite -> INVALID_DATA. */
  for (int p = 0; p < n; p++) {
    float av_ = widen(a, dtype, p), lv = widen(l, dtype, p);
    float d = av_ - lv;
    b[p] = fmaf(beta, e[p], d);
    if (!isfinite(av_) || !isfinite(lv) || !isfinite(e[p]) || !isfinite(b[p])) { st = SLCO_INVALID_DATA; goto done; }
  }

  /* step 2 — Top-k within the chunk */
  st = slco_topk(b, n, k_eff, S);
  if (st != SLCO_OK) goto done;

  /* steps 3-4 — Q: 2-bit quantiser ("Q is a low-bit quantizer",
   * P:176 "2-bit quantization"); R#1 sign + bucket with bucket-mean scales.
   * tau = mean |v|; bucket h = |v| > tau; scales = bucket means; fp16. */
  for (int j = 0; j < k_eff; j++) av[j] = fabsf(b[S[j]]);
  const float tau = slco_tree_sum(av, k_eff, g->k) / (float)k_eff;
  int n_hi = 0;
  for (int j = 0; j < k_eff; j++) {
    h[j] = av[j] > tau;
    n_hi += h[j];
    lo[j] = h[j] ? 0.0f : av[j];
    hi[j] = h[j] ? av[j] : 0.0f;
  }
  const int n_lo = k_eff - n_hi;
  const float sum_lo = slco_tree_sum(lo, k_eff, g->k);
  const float sum_hi = slco_tree_sum(hi, k_eff, g->k);
  const float s_lo = n_lo > 0 ? sum_lo / (float)n_lo : 0.0f;
  const float s_hi = n_hi > 0 ? sum_hi / (float)n_hi : tau;
  const uint16_t S_lo = slco_rn16(s_lo), S_hi = slco_rn16(s_hi);
  const float f_lo = slco_f16_to_f32(S_lo), f_hi = slco_f16_to_f32(S_hi);
  if (!isfinite(f_lo) || !isfinite(f_hi)) { st = SLCO_INVALID_DATA; goto done; }

  /* step 7 — record (P:93 fixed-width indices; R#6 layout) */
  const int RW = slco_record_words(g), IW = idx_words(g);
  memset(rec, 0, sizeof(uint32_t) * (size_t)RW);
  for (int j = 0; j < k_eff; j++) {
    for (int bit = 0; bit < g->index_bits; bit++)
      put_bit(rec, (int64_t)g->index_bits * j + bit, ((uint32_t)S[j] >> bit) & 1u);
    put_bit(rec + IW, 2 * j, signbit(b[S[j]]) ? 1u : 0u);
    put_bit(rec + IW, 2 * j + 1, (uint32_t)h[j]);
  }
  rec[RW - 1] = (uint32_t)S_lo | ((uint32_t)S_hi << 16);

  /* steps 5-6 — e_new = beta*e + Delta - hatDelta (Eq. 1 line 3):
   * unselected positions keep b; selected subtract their decoded value. */
  for (int p = 0; p < n; p++) e_new[p] = b[p];
  for (int j = 0; j < k_eff; j++) {
    const float mag = h[j] ? f_hi : f_lo;
    const float dq = signbit(b[S[j]]) ? -mag : mag;
    e_new[S[j]] = b[S[j]] - dq;
  }

done:
  free(b); free(S); free(av); free(lo); free(hi); free(h);
  return st;
}

/* decode: the receiving side's reading of one record (Eq. 2) */
int slco_decode_chunk(const uint32_t* rec, int n, const slco_geom* g, int32_t* pos, float* dq) {
  if (slco_geom_check(g) != SLCO_OK || n < 1 || n > g->chunk) return -1;
  const int k_eff = slco_effective_k(n, g);
  const int RW = slco_record_words(g), IW = idx_words(g);
  const float f_lo = slco_f16_to_f32((uint16_t)(rec[RW - 1] & 0xFFFFu));
  const float f_hi = slco_f16_to_f32((uint16_t)(rec[RW - 1] >> 16));
  for (int j = 0; j < k_eff; j++) {
    uint32_t p = 0;
    for (int bit = 0; bit < g->index_bits; bit++)
      p |= get_bit(rec, (int64_t)g->index_bits * j + bit) << bit;
    if ((int)p >= n) return -1;
    const uint32_t sgn = get_bit(rec + IW, 2 * j), hb = get_bit(rec + IW, 2 * j + 1);
    const float mag = hb ? f_hi : f_lo;
    pos[j] = (int32_t)p;
    dq[j] = sgn ? -mag : mag;
  }
  return k_eff;
}

/* ------------------------------------------------------------------ */
/* Eq. 2 line 1: Delta = (1/R) sum_{r in R} hatDelta_r.         */
/* R#16: R = number of aggregated records.  R#17: accumulate in fp64   */
/* in canonical peer-id order starting at +0.0, then                   */
/* Delta = (float)(acc * (1.0 / R)).                                   */
/* ------------------------------------------------------------------ */
typedef struct { const uint8_t* id; int r; } peer_ref;
static int cmp_peer(const void* x, const void* y) {
  const peer_ref* a = (const peer_ref*)x; const peer_ref* b = (const peer_ref*)y;
  int c = memcmp(a->id, b->id, 16);
  if (c) return c;
  return (a->r > b->r) - (a->r < b->r);
}

int slco_aggregate_chunk(const uint32_t* const* recs, const uint8_t* peer_ids, const float* w, int R,
                         int n, const slco_geom* g, float* delta) {
  if (R < 1 || slco_geom_check(g) != SLCO_OK || n < 1 || n > g->chunk) return SLCO_INVALID_ARGUMENT;
  peer_ref* order = (peer_ref*)malloc(sizeof(peer_ref) * (size_t)R);
  double* acc = (double*)malloc(sizeof(double) * (size_t)n);
  int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)g->k);
  float* dq = (float*)malloc(sizeof(float) * (size_t)g->k);
  int st = SLCO_OK;
  if (!order || !acc || !pos || !dq) { st = SLCO_INVALID_ARGUMENT; goto done; }
  static const uint8_t zero_id[16] = {0};
  for (int r = 0; r < R; r++) { order[r].id = peer_ids ? peer_ids + 16 * r : zero_id; order[r].r = r; }
  if (peer_ids) qsort(order, (size_t)R, sizeof(peer_ref), cmp_peer);
  for (int p = 0; p < n; p++) acc[p] = 0.0;
  for (int i = 0; i < R; i++) {
    const int r = order[i].r;
    const int ke = slco_decode_chunk(recs[r], n, g, pos, dq);
    if (ke < 0) { st = SLCO_INVALID_DATA; goto done; }
    const double wr = w ? (double)w[r] : 1.0;
    for (int j = 0; j < ke; j++) acc[pos[j]] += wr * (double)dq[j];
  }
  const double invR = 1.0 / (double)R;
  for (int p = 0; p < n; p++) delta[p] = (float)(acc[p] * invR);
done:
  free(order); free(acc); free(pos); free(dq);
  return st;
}

/* Eq. 2 line 2: theta^(t+1) = theta^(t) - alpha*Delta; R#18 fused:
 * fma(-alpha, Delta, theta); bf16 params are widened, updated, re-rounded. */
void slco_outer_update(void* theta, int dtype, const float* delta, int64_t n, float alpha) {
  for (int64_t i = 0; i < n; i++) {
    if (dtype == SLCO_BF16) {
      uint16_t* t = (uint16_t*)theta;
      float x = u2f(((uint32_t)t[i]) << 16);
      t[i] = slco_rnbf(fmaf(-alpha, delta[i], x));
    } else {
      float* t = (float*)theta;
      t[i] = fmaf(-alpha, delta[i], t[i]);
    }
  }
}

/* ------------------------------------------------------------------ */
/* tensor-level drivers                                                */
/* ------------------------------------------------------------------ */
int slco_compress_tensor(int ndim, const int64_t* dims, const void* a, const void* l, int dtype,
                         float* e_inout, const slco_geom* g, float beta, int64_t c0, int64_t c1,
                         uint32_t* rec_out) {
  if (slco_geom_check(g) != SLCO_OK) return SLCO_INVALID_ARGUMENT;
  const int RW = slco_record_words(g);
  const size_t es = dtype == SLCO_BF16 ? 2 : 4;
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)g->chunk);
  char* ga = (char*)malloc(es * (size_t)g->chunk);
  char* gl = (char*)malloc(es * (size_t)g->chunk);
  float* ge = (float*)malloc(sizeof(float) * (size_t)g->chunk);
  float* en = (float*)malloc(sizeof(float) * (size_t)g->chunk);
  int st = SLCO_OK;
  if (!off || !ga || !gl || !ge || !en) { st = SLCO_INVALID_ARGUMENT; goto done; }
  for (int64_t c = c0; c < c1; c++) {
    const int n = slco_chunk_offsets(ndim, dims, g, c, off);
    if (n < 0) { st = SLCO_INVALID_ARGUMENT; goto done; }
    for (int p = 0; p < n; p++) {
      memcpy(ga + es * p, (const char*)a + es * off[p], es);
      memcpy(gl + es * p, (const char*)l + es * off[p], es);
      ge[p] = e_inout[off[p]];
    }
    st = slco_compress_chunk(ga, gl, dtype, ge, n, g, beta, rec_out + (c - c0) * RW, en);
    if (st != SLCO_OK) goto done;
    for (int p = 0; p < n; p++) e_inout[off[p]] = en[p];
  }
done:
  free(off); free(ga); free(gl); free(ge); free(en);
  return st;
}

static int agg_range(int ndim, const int64_t* dims, const uint32_t* const* recs, const uint8_t* peer_ids,
                     const float* w, int R, const slco_geom* g, int64_t c0, int64_t c1,
                     float* delta_out, void* theta, int dtype, float alpha) {
  if (slco_geom_check(g) != SLCO_OK || R < 1) return SLCO_INVALID_ARGUMENT;
  const int RW = slco_record_words(g);
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)g->chunk);
  float* d = (float*)malloc(sizeof(float) * (size_t)g->chunk);
  const uint32_t** rp = (const uint32_t**)malloc(sizeof(void*) * (size_t)R);
  int st = SLCO_OK;
  if (!off || !d || !rp) { st = SLCO_INVALID_ARGUMENT; goto done; }
  for (int64_t c = c0; c < c1; c++) {
    const int n = slco_chunk_offsets(ndim, dims, g, c, off);
    if (n < 0) { st = SLCO_INVALID_ARGUMENT; goto done; }
    for (int r = 0; r < R; r++) rp[r] = recs[r] + (c - c0) * RW;
    st = slco_aggregate_chunk(rp, peer_ids, w, R, n, g, d);
    if (st != SLCO_OK) goto done;
    for (int p = 0; p < n; p++) {
      if (delta_out) delta_out[off[p]] = d[p];
      if (theta) {
        if (dtype == SLCO_BF16) slco_outer_update((uint16_t*)theta + off[p], dtype, d + p, 1, alpha);
        else slco_outer_update((float*)theta + off[p], dtype, d + p, 1, alpha);
      }
    }
  }
done:
  free(off); free(d); free(rp);
  return st;
}

int slco_aggregate_tensor(int ndim, const int64_t* dims, const uint32_t* const* recs,
                          const uint8_t* peer_ids, const float* w, int R, const slco_geom* g,
                          int64_t c0, int64_t c1, float* delta_out) {
  return agg_range(ndim, dims, recs, peer_ids, w, R, g, c0, c1, delta_out, NULL, 0, 0.0f);
}

int slco_aggregate_update_tensor(int ndim, const int64_t* dims, void* theta, int dtype,
                                 const uint32_t* const* recs, const uint8_t* peer_ids, const float* w,
                                 int R, const slco_geom* g, int64_t c0, int64_t c1, float alpha) {
  return agg_range(ndim, dims, recs, peer_ids, w, R, g, c0, c1, NULL, theta, dtype, alpha);
}

/* ------------------------------------------------------------------ */
/* closed forms                                                        */
/* ------------------------------------------------------------------ */
/* (1/k) log2 binom(C, k) bits per transmitted value */
double slco_index_entropy_bound(int C, int k) {
  double lb = lgamma((double)C + 1.0) - lgamma((double)k + 1.0) - lgamma((double)(C - k) + 1.0);
  return lb / log(2.0) / (double)k;
}

/* dense bits per chunk over transmitted bits per chunk */
double slco_compression_ratio(int C, int k, int dense_bits, int wire_bits_per_value) {
  return (double)dense_bits * (double)C / ((double)k * (double)wire_bits_per_value);
}
