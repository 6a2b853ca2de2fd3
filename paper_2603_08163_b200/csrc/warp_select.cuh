// warp_select.cuh — one warp selects, quantises and packs one chunk
// (Eq. 1, chunk Top-k P:88, 2-bit Q P:176), given the
// chunk's 32*NP group maxima and its dense e = b already stored.  Shared by
// the compress kernels (compress_warp.cu: warp streams its own chunk;
// compress_tma.cu: warp reads a TMA-staged chunk from shared memory).
//
//  S. T = the largest key (bits 31..14) with >= k_eff group maxima >= T
//     (bitwise search, warp reductions): >= k_eff elements have key >= T,
//     typically ~1.2 k_eff.
//  B. the groups whose max reaches T are spread over the lanes and their
//     16 values re-read from e (an L2 hit: the dense e stores carry an L2
//     evict_last hint); values with key >= T become candidates
//     key<<16 | ~pos in warp smem.
//  R. exact rank of each candidate by counting (ties: lower position first,
//     R#3, R#4); rank < k_eff -> selected; a bitmap prefix gives each its slot
//     in ascending position (R#5).  More than CAP candidates (constant / tied
//     runs): key_select (<= XCAP candidates: bitwise search for the k-th key
//     over the candidate keys in registers), else tie_select (the k-th key is
//     the smallest candidate key), else — and for a non-finite value — exact
//     radix select over the candidate groups (4 rounds of 8-bit digits).
//  Q. 2-bit quantiser + record (R#1, R#6, R#13, R#14).
//  F. EF residual of the selected positions, e = b - dequant.
//
// Position layout of a chunk: pass u, lane l owns positions 4q..4q+3 for
// q = 128u + 32v + l (v = 0..3); group (l, u) = those 16 positions.
#pragma once
#include "chunk_io.cuh"
#include "quant_pack.cuh"

namespace slc {
#ifdef SLC_PHASE_TIMING  // debug builds: per-phase SM cycles summed over warps (slc_debug_phase_cycles)
__device__ unsigned long long g_phase_cycles[8];
__device__ unsigned long long g_path_count[16];  // selection paths: candidates, tie, tie->rank, radix; then
                                                 // cycles: 4 tie_select, 5 radix rounds, 6 radix mark+fill; 7 sum G, 8 sum M (radix);
                                                 // 9 key_select calls, 10 its cycles, 11 hist_select -> key_select
#define PATH_COUNT(i) \
  do {                \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_path_count[i], 1ull); \
  } while (0)
#define PATH_ADD(i, v) \
  do {                \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_path_count[i], (unsigned long long)(v)); \
  } while (0)
#else
#define PATH_ADD(i, v) \
  do {                 \
  } while (0)
#define PATH_COUNT(i) \
  do {                \
  } while (0)
#endif
#ifdef SLC_PHASE_TIMING
#define PHASE_T0() long long _pt = clock64()
#define PHASE_MARK(i)                                                         \
  do {                                                                        \
    long long _now = clock64();                                               \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase_cycles[i], (unsigned long long)(_now - _pt)); \
    _pt = _now;                                                               \
  } while (0)
#else
#define PHASE_T0() \
  do {             \
  } while (0)
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#endif
namespace wsel {

#ifndef SLC_BR
#define SLC_BR 3  // candidate groups re-read per lane per L2 round trip (stage B)
#endif

template <int C>
struct WarpCfg {
  static constexpr int NP = C / 512;       // passes of 16 positions per lane
  static constexpr int B = (C == 1024) ? 32 : (C == 4096 ? 64 : 128);
  static constexpr int RPQ_SHIFT = (B == 32) ? 3 : (B == 64 ? 4 : 5);  // log2(B/4)
  static constexpr int BW = C / 32;         // bitmap words
};

// per-warp shared scratch; CAP = candidate capacity (larger sets take the
// fallback), KMAX = largest k the instantiation serves
// VPU = 4-position groups (quads) per unit, the span one hand-off maximum
// covers: 4 (a 16-position group (lane, u); the paper's geometry) or 1 (a quad:
// NU = 4 NP units per lane, for k close to the 32 NP groups of a chunk)
template <int C, int VPU>
struct UnitCfg {
  static constexpr int NP = C / 512;
  static constexpr int NU = NP * 4 / VPU;  // units per lane
  static constexpr int HN = 32 * NU > 256 ? 32 * NU : 256;
};

template <int C, int CAP, int KMAX, int VPU = 4>
struct WarpScratch {
  uint64_t cand[CAP];
  float candb[CAP];
  uint32_t bit[WarpCfg<C>::BW];
  union {
    struct {
      uint32_t wpre[WarpCfg<C>::BW];
      uint32_t tie[WarpCfg<C>::BW];  // tie_select / key_select: positions whose key equals the threshold
    };
    uint32_t xkey[2 * WarpCfg<C>::BW];  // stage B -> key_select: keys of candidates CAP.. (before R)
  };
  uint32_t fb[4];                // stage B -> select_fallback: G, Kmin, M, bad (kept out of registers)
  uint32_t gm[32];               // per lane: bit u = group (lane, u) may hold a selected value (max >= T)
  union {
    // the unit list of stage B (<= 32 NU entries) and the fallbacks' histograms,
    // dead once the slots below are written (R fills them, Q and F read them)
    uint32_t hist[UnitCfg<C, VPU>::HN];
    struct {
      uint32_t selpos[KMAX];
      float selval[KMAX];
      uint32_t code[KMAX];
    };
  };
  // key_select: candidates held per lane (registers), and so the largest M it serves
  static constexpr int NXK = (CAP + 2 * WarpCfg<C>::BW) / 32 < 16 ? (CAP + 2 * WarpCfg<C>::BW) / 32 : 16;
  static constexpr int XCAP = 32 * NXK;
};

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void st_f32x4_evict_last(float* ptr, float x, float y, float z, float w, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "f"(x), "f"(y), "f"(z),
               "f"(w), "l"(pol)
               : "memory");
}

__device__ __forceinline__ float absmax_nan(float m, float x) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(m), "f"(fabsf(x)));
  return r;
}

// element offset of the 4-position group q of chunk d
template <int RPQ_SHIFT>
__device__ __forceinline__ int64_t goff(const ChunkDesc& d, int q) {
  return d.ld ? d.base + (int64_t)(q >> RPQ_SHIFT) * d.ld + 4 * (q & ((1 << RPQ_SHIFT) - 1)) : d.base + 4 * (int64_t)q;
}

template <int B>
__device__ __forceinline__ int64_t pos_off(const ChunkDesc& d, int p) {
  return d.ld ? d.base + (int64_t)(p / B) * d.ld + (p % B) : d.base + p;
}

// selection state of the chunk whose selection runs during the next chunk's stream
struct Sel {
  int64_t c;  // -1: none
  ChunkDesc d;
  int len, k_eff;
  bool full, bad;
  uint32_t Tc;
  int M;  // candidates; > CAP: tie_select, then the radix fallback
  int G;  // groups re-read by stage B (their ids in ws.hist)
  uint32_t Kmin;  // smallest candidate key (>= Tc)
  QuantOut q;
};

// 0-based position of the r-th set bit of w (r < popc(w)): 5 halving steps
__device__ __forceinline__ int nth_set_bit(uint32_t w, int r) {
  int pos = 0;
#pragma unroll
  for (int sh = 16; sh; sh >>= 1) {
    const uint32_t lo = w & ((1u << sh) - 1u);
    const int c = __popc(lo);
    if (r >= c) {
      r -= c;
      w >>= sh;
      pos += sh;
    } else {
      w = lo;
    }
  }
  return pos;
}

// slots in ascending position from the selection bitmap ws.bit (n_sel bits):
// slot j (lane-strided) finds its word by binary search over the word prefix
// (the largest word whose prefix is <= j holds bit j) and its bit by
// nth_set_bit; the values are re-read from e (= b) with every lane's load in
// flight at once (a per-lane walk of its own words serialises on tied rows)
template <int C, int CAP, int KMAX, int VPU>
__device__ __forceinline__ void fill_slots(const float* ef, WarpScratch<C, CAP, KMAX, VPU>& ws, const int lane,
                                           const ChunkDesc& d, const int n_sel) {
  using K = WarpCfg<C>;
  constexpr int WPL = K::BW / 32;
  uint32_t w[WPL];
  int cw = 0;
#pragma unroll
  for (int x = 0; x < WPL; x++) { w[x] = ws.bit[WPL * lane + x]; cw += __popc(w[x]); }
  int pre = warp_excl_scan(cw);
#pragma unroll
  for (int x = 0; x < WPL; x++) { ws.wpre[WPL * lane + x] = (uint32_t)pre; pre += __popc(w[x]); }
  __syncwarp();
  for (int j = lane; j < n_sel; j += 32) {
    int lo = 0, hi = K::BW - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((int)ws.wpre[mid] <= j) lo = mid;
      else hi = mid - 1;
    }
    const int p = 32 * lo + nth_set_bit(ws.bit[lo], j - (int)ws.wpre[lo]);
    SLC_CHECK(j < KMAX, "fill_slots slot");
    ws.selpos[j] = (uint32_t)p;
    ws.selval[j] = ef[pos_off<K::B>(d, p)];
  }
}

// exact k_eff-th largest key by 4 rounds of 8-bit radix select over all positions,
// then key > K plus the first `need` positions with key == K (lower position wins)
// (a free function: as a member its `this` would pin the Compressor in local memory)
#ifndef SLC_RADIX_UB
#define SLC_RADIX_UB 1  // passes whose loads radix_fallback keeps in flight (measured: 4 spills, slower)
#endif
template <int C, int CAP, int KMAX, int VPU>
__device__ __noinline__ void radix_fallback(float* ef, WarpScratch<C, CAP, KMAX, VPU>* wsp, const int lane, const ChunkDesc d,
                                            const int len, const bool full, const int k_eff) {
  using K = WarpCfg<C>;
  constexpr int NP = K::NP;
  WarpScratch<C, CAP, KMAX, VPU>& ws = *wsp;
  // only groups whose maximum reaches T can hold a selected value (>= k_eff
  // values are >= T): the other groups are neither loaded nor counted
  const uint32_t gm = ws.gm[lane];
  constexpr int UB = NP < SLC_RADIX_UB ? NP : SLC_RADIX_UB;
  uint32_t Kth = 0;
  int need = k_eff;
#ifdef SLC_PHASE_TIMING
  long long t0 = clock64();
#endif
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) ws.hist[i] = 0u;
    __syncwarp();
    const uint32_t hi_mask = shift == 24 ? 0u : (0xFFFFFFFFu << (shift + 8));
    // UB passes' loads in flight per L2 round trip
#pragma unroll 1
    for (int u0 = 0; u0 < NP; u0 += UB) {
      float ev[UB][4][4];
      int nvs[UB][4];
      bool any = false;
#pragma unroll
      for (int b = 0; b < UB; b++) {
#pragma unroll
        for (int v = 0; v < 4; v++) {
          // unit of quad (u, v): u for 16-position groups, 4u + v for quads
          const bool act = u0 + b < NP && ((gm >> ((4 * (u0 + b) + v) / VPU)) & 1u);
          any |= act;
          const int q = 128 * (u0 + b) + 32 * v + lane;
          nvs[b][v] = act ? (full ? 4 : valid_in_group(4 * q, len)) : 0;
          load_f32x4_l2(ef, goff<K::RPQ_SHIFT>(d, q), nvs[b][v], ev[b][v]);
        }
      }
      if (!__any_sync(kFull, any)) continue;
#pragma unroll
      for (int b = 0; b < UB; b++)
#pragma unroll
        for (int v = 0; v < 4; v++)
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint32_t key = key2_of(ev[b][v][j]);
            const bool in = j < nvs[b][v] && (key & hi_mask) == (Kth & hi_mask);
            const uint32_t dg = (key >> shift) & 255u;
            // tied runs put the whole warp on one bin: one aggregated add instead
            // of 32 serialised ones
            const unsigned m = __ballot_sync(kFull, in);
            if (m) {
              const uint32_t dmin = __reduce_min_sync(kFull, in ? dg : 255u);
              const uint32_t dmax = __reduce_max_sync(kFull, in ? dg : 0u);
              if (dmin == dmax) {
                if (lane == __ffs(m) - 1) atomicAdd(&ws.hist[dg], (uint32_t)__popc(m));
              } else if (in) {
                atomicAdd(&ws.hist[dg], 1u);
              }
            }
          }
    }
    __syncwarp();
    // digit D: #(digit > D) < need <= #(digit >= D); lane l holds bins 8l..8l+7
    uint32_t h[8];
    uint32_t s8 = 0;
#pragma unroll
    for (int x = 0; x < 8; x++) { h[x] = ws.hist[8 * lane + x]; s8 += h[x]; }
    uint32_t inc = s8;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_down_sync(kFull, inc, o);
      if (lane + o < 32) inc += y;
    }
    uint32_t acc = inc - s8;  // bins in lanes above
    int found = -1;
    uint32_t found_gt = 0;
#pragma unroll
    for (int x = 7; x >= 0; x--) {
      if (found < 0 && acc < (uint32_t)need && acc + h[x] >= (uint32_t)need) { found = 8 * lane + x; found_gt = acc; }
      acc += h[x];
    }
    const int src = __ffs(__ballot_sync(kFull, found >= 0)) - 1;
    Kth |= (uint32_t)__shfl_sync(kFull, found, src) << shift;
    need -= (int)__shfl_sync(kFull, found_gt, src);
    __syncwarp();
  }
#ifdef SLC_PHASE_TIMING
  long long t1 = clock64();
  PATH_ADD(5, t1 - t0);
#endif
  int taken = 0;
#pragma unroll 1
  for (int u0 = 0; u0 < NP; u0 += UB) {
    float ev[UB][4][4];
    int nvs[UB][4];
#pragma unroll
    for (int b = 0; b < UB; b++)
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int q = 128 * (u0 + b) + 32 * v + lane;
        nvs[b][v] = (u0 + b < NP && ((gm >> ((4 * (u0 + b) + v) / VPU)) & 1u)) ? (full ? 4 : valid_in_group(4 * q, len))
                                                                                 : 0;
        load_f32x4_l2(ef, goff<K::RPQ_SHIFT>(d, q), nvs[b][v], ev[b][v]);
      }
#pragma unroll
    for (int b = 0; b < UB; b++)
#pragma unroll
      for (int v = 0; v < 4; v++) {
        // lanes hold consecutive 4-position groups: ascending position = (u, v, lane, j)
        const int q = 128 * (u0 + b) + 32 * v + lane;
        const int nv = nvs[b][v];
        uint32_t tmask = 0, m4 = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t key = key2_of(ev[b][v][j]);
          if (j < nv && key > Kth) m4 |= 1u << j;
          if (j < nv && key == Kth) tmask |= 1u << j;
        }
        const int tc = __popc(tmask);
        int o = taken + warp_excl_scan(tc);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          if ((tmask >> j) & 1u) {
            if (o < need) m4 |= 1u << j;
            o++;
          }
        }
        taken += (int)__reduce_add_sync(kFull, (unsigned)tc);
        // positions 4q..4q+3 of lanes 8i..8i+7 form bitmap word q >> 3: one store
        uint32_t wv = m4 << (4 * (lane & 7));
        wv |= __shfl_xor_sync(kFull, wv, 1);
        wv |= __shfl_xor_sync(kFull, wv, 2);
        wv |= __shfl_xor_sync(kFull, wv, 4);
        if ((lane & 7) == 0 && wv) ws.bit[q >> 3] = wv;
      }
  }
  __syncwarp();
  fill_slots<C, CAP, KMAX, VPU>(ef, ws, lane, d, k_eff);
#ifdef SLC_PHASE_TIMING
  PATH_ADD(6, clock64() - t1);
#endif
}

  // ---- T: too many candidates (degenerate chunks: zeros, constants, discrete
// ties, fewer than k nonzeros).  The candidate groups are re-read once:
// values with key > Kmin become candidates (count A), values with key ==
// Kmin go to a tie bitmap.  A < k_eff: the k_eff-th largest key IS Kmin, so
// the selection is every candidate plus the first k_eff - A tied positions
// in position order (R#4) — done here.  A >= k_eff: the answer lies among
// the A candidates (rank them if A <= CAP), else the radix fallback.
// Returns true when the selection is complete (ws.selpos / selval filled).
template <int C, int CAP, int KMAX, int VPU>
__device__ __forceinline__ bool tie_select(float* ef, WarpScratch<C, CAP, KMAX, VPU>& ws, const int lane, const Sel& s,
                                           int& M) {
using K = WarpCfg<C>;
constexpr int NU = UnitCfg<C, VPU>::NU;
{
  // Kmin: the smallest key >= Tc among the candidate groups (one more L2 pass)
  uint32_t Kc = 0xFFFFFFFFu;
  for (int gi = lane; gi < s.G; gi += 32) {
    const uint32_t id = ws.hist[gi];
    const int owner = (int)(id / NU), u = (int)(id % NU);
#pragma unroll
    for (int v = 0; v < VPU; v++) {
      const int q = 32 * (VPU * u + v) + owner;
      const int nv = s.full ? 4 : valid_in_group(4 * q, s.len);
      float x[4];
      load_f32x4_l2(ef, goff<K::RPQ_SHIFT>(s.d, q), nv, x);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint32_t key = key2_of(x[j]);
        if (j < nv && key >= s.Kmin) Kc = min(Kc, key);
      }
    }
  }
  Kc = __reduce_min_sync(kFull, Kc);
  for (int w = lane; w < K::BW; w += 32) ws.tie[w] = 0u;
  __syncwarp();
  int A = 0;
  constexpr int BR = 1;  // one group per lane in flight: the fallback keeps its register footprint small
  for (int r0 = 0; r0 < s.G; r0 += 32 * BR) {
    float vals[BR][4 * VPU];
    int owner[BR], uu[BR];
#pragma unroll
    for (int bq = 0; bq < BR; bq++) {
      const int gi = r0 + 32 * bq + lane;
      owner[bq] = 0;
      uu[bq] = 0;
      if (gi < s.G) {
        const uint32_t id = ws.hist[gi];
        owner[bq] = (int)(id / NU);
        uu[bq] = (int)(id % NU);
#pragma unroll
        for (int v = 0; v < VPU; v++) {
          const int q = 32 * (VPU * uu[bq] + v) + owner[bq];
          load_f32x4_l2(ef, goff<K::RPQ_SHIFT>(s.d, q), s.full ? 4 : valid_in_group(4 * q, s.len), &vals[bq][4 * v]);
        }
      }
    }
#pragma unroll
    for (int bq = 0; bq < BR; bq++) {
      const int gi = r0 + 32 * bq + lane;
      uint32_t cmask = 0;
      if (gi < s.G) {
#pragma unroll
        for (int v = 0; v < VPU; v++) {
          const int q = 32 * (VPU * uu[bq] + v) + owner[bq];
          const int nv = s.full ? 4 : valid_in_group(4 * q, s.len);
          uint32_t tmask = 0;
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint32_t key = key2_of(vals[bq][4 * v + j]);
            if (j < nv && key > Kc) cmask |= 1u << (4 * v + j);
            if (j < nv && key == Kc) tmask |= 1u << j;
          }
          if (tmask) atomicOr(&ws.tie[(4 * q) >> 5], tmask << ((4 * q) & 31));
        }
      }
      const int cc = __popc(cmask);
      int o = A + warp_excl_scan(cc);
      A += (int)__reduce_add_sync(kFull, (unsigned)cc);
#pragma unroll
      for (int j = 0; j < 4 * VPU; j++) {
        if ((cmask >> j) & 1u) {
          const int p = 4 * (32 * (VPU * uu[bq] + (j >> 2)) + owner[bq]) + (j & 3);
          if (o < CAP) {
            ws.cand[o] = ((uint64_t)key2_of(vals[bq][j]) << 16) | (uint64_t)(0xFFFFu - (uint32_t)p);
            ws.candb[o] = vals[bq][j];
          }
          o++;
        }
      }
    }
  }
  __syncwarp();
  if (A >= s.k_eff) {  // the k_eff-th largest key is above Kmin
    M = A <= CAP ? A : CAP + 1;
    return false;
  }
  // every candidate is selected, then the first need = k_eff - A tied positions
  for (int m = lane; m < A; m += 32) {
    const uint32_t p = 0xFFFFu - (uint32_t)(ws.cand[m] & 0xFFFFu);
    atomicOr(&ws.bit[p >> 5], 1u << (p & 31));
  }
  const int need = s.k_eff - A;
  constexpr int WPL = K::BW / 32;
  uint32_t w[WPL];
  int cw = 0;
#pragma unroll
  for (int x = 0; x < WPL; x++) { w[x] = ws.tie[WPL * lane + x]; cw += __popc(w[x]); }
  int pre = warp_excl_scan(cw);
  __syncwarp();
#pragma unroll
  for (int x = 0; x < WPL; x++) {
    uint32_t take = 0, y = w[x];
    while (y && pre < need) {
      take |= y & (0u - y);  // lowest remaining tied position of the word
      y &= y - 1;
      pre++;
    }
    if (take) atomicOr(&ws.bit[WPL * lane + x], take);
  }
  __syncwarp();
  fill_slots<C, CAP, KMAX, VPU>(ef, ws, lane, s.d, s.k_eff);
  return true;
}
}


// exact rank of the M <= CAP candidates in ws.cand (key << 16 | ~pos: ties go to
// the lower position, R#3, R#4); rank < k_eff -> selected; the selection
// bitmap's prefix gives each its slot in ascending position (R#5)
template <int C, int CAP, int KMAX, int VPU>
__device__ __forceinline__ void rank_select(WarpScratch<C, CAP, KMAX, VPU>& ws, const int lane, const int M,
                                            const int k_eff) {
  constexpr int WPL = WarpCfg<C>::BW / 32;
  const int NM = (M + 31) >> 5;
  constexpr int MM = CAP / 32;
  uint64_t mine[MM];
  int rank[MM];
#pragma unroll
  for (int m = 0; m < MM; m++) {
    mine[m] = (lane + 32 * m < M) ? ws.cand[lane + 32 * m] : ~0ull;
    rank[m] = 0;
  }
  if (NM <= 3) {
#pragma unroll 4
    for (int j = 0; j < M; j++) {
      const uint64_t x = ws.cand[j];
      rank[0] += x > mine[0];
      rank[1] += x > mine[1];
      rank[2] += x > mine[2];
    }
  } else {
    for (int j = 0; j < M; j++) {
      const uint64_t x = ws.cand[j];
#pragma unroll
      for (int m = 0; m < MM; m++) rank[m] += x > mine[m];
    }
  }
#pragma unroll
  for (int m = 0; m < MM; m++) {
    if (lane + 32 * m < M && rank[m] < k_eff) {
      const uint32_t p = 0xFFFFu - (uint32_t)(mine[m] & 0xFFFFu);
      atomicOr(&ws.bit[p >> 5], 1u << (p & 31));
    }
  }
  __syncwarp();
  {  // bitmap prefix
    uint32_t w[WPL];
    int cw = 0;
#pragma unroll
    for (int x = 0; x < WPL; x++) { w[x] = ws.bit[WPL * lane + x]; cw += __popc(w[x]); }
    int pre = warp_excl_scan(cw);
#pragma unroll
    for (int x = 0; x < WPL; x++) { ws.wpre[WPL * lane + x] = (uint32_t)pre; pre += __popc(w[x]); }
  }
  __syncwarp();
#pragma unroll
  for (int m = 0; m < MM; m++) {
    const int ci = lane + 32 * m;
    if (ci < M && rank[m] < k_eff) {
      const uint32_t p = 0xFFFFu - (uint32_t)(mine[m] & 0xFFFFu);
      const int sl = (int)ws.wpre[p >> 5] + __popc(ws.bit[p >> 5] & ((1u << (p & 31)) - 1u));
      SLC_CHECK(sl >= 0 && sl < k_eff, "rank_select slot");
      ws.selpos[sl] = p;
      ws.selval[sl] = ws.candb[ci];
    }
  }
}

// ---- more than CAP candidates, at most XCAP (a tied level crossing the top
// k, e.g. a constant run covering a few rows of a 64x64 block): stage B keeps
// the keys of candidates CAP.. in ws.xkey (wpre + tie, unused until R), so
// every candidate key is at hand.  Each lane holds its NXK keys in registers
// and the k_eff-th largest key K* is found by a bitwise search over the bits
// where Tc and the largest key differ (K* lies in [Tc, Kmax]): one register
// count + one warp reduction per bit, no atomics, no L2 traffic.  One pass
// over the candidate groups then marks key > K* (selected) and key == K*
// (tied); the first k_eff - #(key > K*) tied positions are taken in position
// order (R#3, R#4), slots in ascending position (R#5).  Values with key < Tc
// are never selected (>= k_eff values reach Tc), so the candidate groups hold
// every selected value and every tie at K*.
#ifdef SLC_KS_INLINE
#define SLC_KS_ATTR __forceinline__
#else
#define SLC_KS_ATTR __noinline__
#endif
template <int C, int CAP, int KMAX, int VPU>
__device__ SLC_KS_ATTR void key_select(float* ef, WarpScratch<C, CAP, KMAX, VPU>* wsp, const int lane, const ChunkDesc d,
                                        const int len, const int k_eff, const int G, const uint32_t Tc, const int M) {
  using K = WarpCfg<C>;
  using WS = WarpScratch<C, CAP, KMAX, VPU>;
  constexpr int NU = UnitCfg<C, VPU>::NU;
  constexpr int UPL = 4 / VPU;  // units per lane per L2 round trip of the mark pass
  constexpr int WPL = K::BW / 32;
  constexpr int NXK = WS::NXK;
  WS& ws = *wsp;
  const bool full = len == C;
  uint32_t key[NXK];
  uint32_t kmax = 0;
#pragma unroll
  for (int i = 0; i < NXK; i++) {
    const int m = lane + 32 * i;
    key[i] = m < M ? (m < CAP ? (uint32_t)(ws.cand[m] >> 16) : ws.xkey[m - CAP]) : 0u;  // 0: none (keys are odd)
    kmax = max(kmax, key[i]);
  }
  kmax = __reduce_max_sync(kFull, kmax);
  uint32_t Ks = kmax;
  const uint32_t diff = Tc ^ kmax;
  int top = 0;  // a tied top level holding >= k_eff keys (constant runs): K* = Kmax at once
#pragma unroll
  for (int i = 0; i < NXK; i++) top += key[i] == kmax;
  if (Tc < kmax && (int)__reduce_add_sync(kFull, (unsigned)top) < k_eff) {
    const int hb = 31 - __clz(diff);
    Ks = hb == 31 ? 0u : (kmax & (0xFFFFFFFFu << (hb + 1)));
#pragma unroll 1
    for (int bit = hb; bit >= 0; --bit) {
      const uint32_t Kp = Ks | (1u << bit);
      int cnt = 0;
#pragma unroll
      for (int i = 0; i < NXK; i++) cnt += key[i] >= Kp;
      if ((int)__reduce_add_sync(kFull, (unsigned)cnt) >= k_eff) Ks = Kp;
    }
  }
  int gt = 0;
#pragma unroll
  for (int i = 0; i < NXK; i++) gt += key[i] > Ks;
  const int need = k_eff - (int)__reduce_add_sync(kFull, (unsigned)gt);
  __syncwarp();  // xkey (= tie) read by every lane before it is cleared
  for (int w = lane; w < K::BW; w += 32) ws.tie[w] = 0u;
  __syncwarp();
  // mark: one pass over the candidate units (lane gi = unit list entry gi)
#pragma unroll 1
  for (int g0 = 0; g0 < G; g0 += 32 * UPL) {
    float x[UPL][VPU][4];
    int qb[UPL];
#pragma unroll
    for (int ub = 0; ub < UPL; ub++) {
      const int gi = g0 + 32 * ub + lane;
      qb[ub] = -1;
      if (gi < G) {
        const uint32_t id = ws.hist[gi];
        qb[ub] = 32 * VPU * (int)(id % NU) + (int)(id / NU);
#pragma unroll
        for (int v = 0; v < VPU; v++)
          load_f32x4_l2(ef, goff<K::RPQ_SHIFT>(d, qb[ub] + 32 * v),
                        full ? 4 : valid_in_group(4 * (qb[ub] + 32 * v), len), x[ub][v]);
      }
    }
#pragma unroll
    for (int ub = 0; ub < UPL; ub++) {
      if (qb[ub] < 0) continue;
#pragma unroll
      for (int v = 0; v < VPU; v++) {
        const int p0 = 4 * (qb[ub] + 32 * v);
        const int nv = full ? 4 : valid_in_group(p0, len);
        uint32_t mg = 0, me = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t kk = j < nv ? key2_of(x[ub][v][j]) : 0u;
          mg |= (uint32_t)(kk > Ks) << j;
          me |= (uint32_t)(kk == Ks) << j;
        }
        if (mg) atomicOr(&ws.bit[p0 >> 5], mg << (p0 & 31));
        if (me) atomicOr(&ws.tie[p0 >> 5], me << (p0 & 31));
      }
    }
  }
  __syncwarp();
  {  // the first `need` tied positions in position order
    uint32_t w[WPL];
    int cw = 0;
#pragma unroll
    for (int x = 0; x < WPL; x++) { w[x] = ws.tie[WPL * lane + x]; cw += __popc(w[x]); }
    int pre = warp_excl_scan(cw);
#pragma unroll
    for (int x = 0; x < WPL; x++) {
      uint32_t take = 0, y = w[x];
      while (y && pre < need) {
        take |= y & (0u - y);
        y &= y - 1;
        pre++;
      }
      if (take) atomicOr(&ws.bit[WPL * lane + x], take);
    }
  }
  __syncwarp();
  fill_slots<C, CAP, KMAX, VPU>(ef, ws, lane, d, k_eff);
}

// ---- more than XCAP candidates (large k against the 32*NP group maxima, so
// T is weak, or wide tied levels): one histogram pass over the candidate
// groups narrows the candidates to the bin holding the k_eff-th key.  Bins
// are 1/16 binade wide (key bits 30..19 above Tc's), 256 of them, the top one
// open-ended.  If that bin and the ones above hold at most XCAP values, a
// second pass collects their keys (as stage B does) and key_select finishes
// with T' = the bin's lower edge; otherwise false (tie_select / radix).
#ifndef SLC_HIST_BR
#define SLC_HIST_BR 1  // candidate groups per lane per L2 round trip in hist_select's counting pass
#endif
template <int C, int CAP, int KMAX, int VPU>
__device__ __noinline__ bool hist_select(float* ef, WarpScratch<C, CAP, KMAX, VPU>* wsp, const int lane, const ChunkDesc d,
                                         const int len, const int k_eff, const int G, const uint32_t Tc) {
  using K = WarpCfg<C>;
  using WS = WarpScratch<C, CAP, KMAX, VPU>;
  constexpr int NU = UnitCfg<C, VPU>::NU;
  constexpr int BR = SLC_HIST_BR * 4 / VPU;  // units per lane per L2 round trip
  static_assert(2 * CAP >= 256, "hist_select keeps its histogram in ws.cand");
  WS& ws = *wsp;
  const bool full = len == C;
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws.cand);
  const uint32_t base = Tc & ~0xFFFFFu;
  for (int i = lane; i < 256; i += 32) hist[i] = 0u;
  __syncwarp();
  // the candidate groups, BR per lane per L2 round trip; f(key, position) per valid value
  auto walk = [&](auto&& f) {
#pragma unroll 1
    for (int r0 = 0; r0 < G; r0 += 32 * BR) {
      float vals[BR][4 * VPU];
      int qb[BR];
#pragma unroll
      for (int bq = 0; bq < BR; bq++) {
        const int gi = r0 + 32 * bq + lane;
        qb[bq] = -1;
        if (gi < G) {
          const uint32_t id = ws.hist[gi];
          qb[bq] = 32 * VPU * (int)(id % NU) + (int)(id / NU);
#pragma unroll
          for (int v = 0; v < VPU; v++)
            load_f32x4_l2(ef, goff<K::RPQ_SHIFT>(d, qb[bq] + 32 * v),
                          full ? 4 : valid_in_group(4 * (qb[bq] + 32 * v), len), &vals[bq][4 * v]);
        }
      }
#pragma unroll
      for (int bq = 0; bq < BR; bq++) {
#pragma unroll
        for (int v = 0; v < VPU; v++) {
          const int p0 = 4 * (qb[bq] + 32 * v);
          const int nv = qb[bq] < 0 ? 0 : (full ? 4 : valid_in_group(p0, len));
#pragma unroll
          for (int j = 0; j < 4; j++)
            if (j < nv) f(key2_of(vals[bq][4 * v + j]), p0 + j, vals[bq][4 * v + j]);
        }
      }
    }
  };
  walk([&](uint32_t key, int, float) {
    if (key >= Tc) atomicAdd(&hist[min((key - base) >> 20, 255u)], 1u);
  });
  __syncwarp();
  // bin D: #(bin > D) < k_eff <= #(bin >= D); lane l holds bins 8l..8l+7
  uint32_t h[8];
  uint32_t s8 = 0;
#pragma unroll
  for (int x = 0; x < 8; x++) { h[x] = hist[8 * lane + x]; s8 += h[x]; }
  uint32_t inc = s8;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_down_sync(kFull, inc, o);
    if (lane + o < 32) inc += y;
  }
  uint32_t acc = inc - s8;
  int found = -1;
  uint32_t found_ge = 0;
#pragma unroll
  for (int x = 7; x >= 0; x--) {
    if (found < 0 && acc < (uint32_t)k_eff && acc + h[x] >= (uint32_t)k_eff) { found = 8 * lane + x; found_ge = acc + h[x]; }
    acc += h[x];
  }
  const int src = __ffs(__ballot_sync(kFull, found >= 0)) - 1;
  const uint32_t D = (uint32_t)__shfl_sync(kFull, found, src);
  const int M2 = (int)__shfl_sync(kFull, found_ge, src);
  if (M2 > WS::XCAP) return false;
  const uint32_t T2 = max(Tc, base + (D << 20));
  __syncwarp();  // the histogram (ws.cand) is read; the candidates overwrite it
  int M = 0;
  constexpr int UPL = 4 / VPU;
#pragma unroll 1
  for (int r0 = 0; r0 < G; r0 += 32 * UPL) {
    float vals[UPL][4 * VPU];
    int qb[UPL];
#pragma unroll
    for (int ub = 0; ub < UPL; ub++) {
      const int gi = r0 + 32 * ub + lane;
      qb[ub] = -1;
      if (gi < G) {
        const uint32_t id = ws.hist[gi];
        qb[ub] = 32 * VPU * (int)(id % NU) + (int)(id / NU);
#pragma unroll
        for (int v = 0; v < VPU; v++)
          load_f32x4_l2(ef, goff<K::RPQ_SHIFT>(d, qb[ub] + 32 * v),
                        full ? 4 : valid_in_group(4 * (qb[ub] + 32 * v), len), &vals[ub][4 * v]);
      }
    }
#pragma unroll
    for (int ub = 0; ub < UPL; ub++) {
      uint32_t cmask = 0;
      if (qb[ub] >= 0) {
#pragma unroll
        for (int v = 0; v < VPU; v++) {
          const int nv = full ? 4 : valid_in_group(4 * (qb[ub] + 32 * v), len);
#pragma unroll
          for (int j = 0; j < 4; j++)
            if (j < nv && key2_of(vals[ub][4 * v + j]) >= T2) cmask |= 1u << (4 * v + j);
        }
      }
      const int cc = __popc(cmask);
      int o = M + warp_excl_scan(cc);
      M += (int)__reduce_add_sync(kFull, (unsigned)cc);
#pragma unroll
      for (int j = 0; j < 4 * VPU; j++) {
        if ((cmask >> j) & 1u) {
          const int p = 4 * (qb[ub] + 32 * (j >> 2)) + (j & 3);
          if (o < CAP) {
            ws.cand[o] = ((uint64_t)key2_of(vals[ub][j]) << 16) | (uint64_t)(0xFFFFu - (uint32_t)p);
            ws.candb[o] = vals[ub][j];
          } else if (o < WS::XCAP) {
            ws.xkey[o - CAP] = key2_of(vals[ub][j]);
          }
          o++;
        }
      }
    }
  }
  __syncwarp();
  SLC_CHECK(M == M2, "hist_select candidates");
  key_select<C, CAP, KMAX, VPU>(ef, wsp, lane, d, len, k_eff, G, T2, M);
  return true;
}

// every selection that the candidate path cannot finish (a free, non-inlined
// function: the common path keeps its registers).  Returns 0 when ws.selpos /
// selval are complete, else the number of candidates left in ws.cand (<= CAP)
// for the exact-rank path.
template <int C, int CAP, int KMAX, int VPU>
__device__ __noinline__ int select_fallback(float* ef, WarpScratch<C, CAP, KMAX, VPU>* wsp, const int lane,
                                            const ChunkDesc d, const int len, const int k_eff) {
  Sel s;
  s.d = d;
  s.len = len;
  s.full = len == C;
  s.k_eff = k_eff;
  s.G = (int)wsp->fb[0];
  s.Kmin = wsp->fb[1];
  int M = (int)wsp->fb[2];
  const int M0 = M;
  (void)M0;
  const bool bad = wsp->fb[3] != 0;
  if (!bad && s.G <= UnitCfg<C, VPU>::HN && M <= WarpScratch<C, CAP, KMAX, VPU>::XCAP) {
#ifdef SLC_PHASE_TIMING
    const long long t0 = clock64();
#endif
    key_select<C, CAP, KMAX, VPU>(ef, wsp, lane, d, len, k_eff, s.G, s.Kmin, M);
#ifdef SLC_PHASE_TIMING
    PATH_ADD(10, clock64() - t0);
#endif
    PATH_COUNT(9);
    return 0;
  }
  if (!bad && s.G <= UnitCfg<C, VPU>::HN && hist_select<C, CAP, KMAX, VPU>(ef, wsp, lane, d, len, k_eff, s.G, s.Kmin)) {
    PATH_COUNT(11);
    return 0;
  }
  if (!bad && s.G <= UnitCfg<C, VPU>::HN) {
#ifdef SLC_PHASE_TIMING
    const long long t0 = clock64();
#endif
    const bool done = tie_select<C, CAP, KMAX, VPU>(ef, *wsp, lane, s, M);
#ifdef SLC_PHASE_TIMING
    PATH_ADD(4, clock64() - t0);
#endif
    if (done) {
      PATH_COUNT(1);
      return 0;
    }
    if (M <= CAP) {  // the k_eff-th largest key is above the tie: rank the candidates above it
      PATH_COUNT(2);
      rank_select<C, CAP, KMAX, VPU>(*wsp, lane, M, k_eff);
      return 0;
    }
  }
  PATH_COUNT(3);
  PATH_ADD(7, s.G);
  PATH_ADD(8, M0);
  radix_fallback<C, CAP, KMAX, VPU>(ef, wsp, lane, d, len, len == C, k_eff);
  return 0;
}

// DEFER: a chunk that leaves the candidate path (M > CAP or non-finite) is
// appended to a.defer and finished by compress_fallback_kernel (its selection
// code then stays out of the streaming kernel: registers, i-cache)
template <int C, bool BF16, int KC, int IBC, int CAP, int KMAX, int VPU = 4, bool DEFER = false>
struct Compressor {
  using K = WarpCfg<C>;
  static constexpr int NP = K::NP;
  static constexpr int NU = UnitCfg<C, VPU>::NU;  // hand-off maxima (units) per lane
  // fields of CompressArgs held by value (a reference to the kernel's param
  // struct would force the struct into local memory)
  float* ef;
  uint32_t* records;
  uint32_t* err;
  const uint64_t* rec_extra;
  int n_extra;
  uint32_t* defer;
  int64_t defer_cap;
  int defer_info;
  Geom g;
  int64_t n_elems, n_chunks;
  WarpScratch<C, CAP, KMAX, VPU>& ws;
  int lane;
  int k;

  __device__ __forceinline__ Compressor(const CompressArgs& a, WarpScratch<C, CAP, KMAX, VPU>& ws_, int lane_, int k_)
      : ef(a.ef),
        records(a.records),
        err(a.err),
        rec_extra(a.rec_extra),
        n_extra(a.n_extra),
        defer(a.defer),
        defer_cap(a.defer_cap),
        defer_info(a.defer_info),
        g(a.g),
        n_elems(a.n_elems),
        n_chunks(a.n_chunks),
        ws(ws_),
        lane(lane_),
        k(k_) {}

  // ---- S ---------------------------------------------------------------------------
  __device__ __forceinline__ void stage_S(Sel& s, const uint32_t (&gk)[NU]) {
    uint32_t gmaxk = 0;
#pragma unroll
    for (int u = 0; u < NU; u++) gmaxk = max(gmaxk, gk[u]);
    s.bad = __reduce_max_sync(kFull, gmaxk) >= 0xFF000001u;  // |b| = inf or NaN somewhere
    if (s.bad && lane == 0) atomicOr(err, kErrNonFinite);
    uint32_t T = 0;
#pragma unroll 1
    for (int bit = 31; bit >= 14; --bit) {
      const uint32_t Tp = T | (1u << bit);
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < NU; u++) cnt += gk[u] >= Tp;
      if ((int)__reduce_add_sync(kFull, (unsigned)cnt) >= s.k_eff) T = Tp;
    }
    // quads hand over keys rounded down to 16 bits: T's low 16 bits are
    // cleared so that "unit key >= Tc" still keeps every unit holding a key >= Tc
    s.Tc = max(VPU == 1 ? T & 0xFFFF0000u : T, 1u);
  }

  // ---- B ---------------------------------------------------------------------------
  // this lane's candidate groups: bit u = group (lane, u) has max key >= Tc
  __device__ __forceinline__ uint32_t group_mask(const Sel& s, const uint32_t (&gk)[NU]) const {
    uint32_t gmask = 0;
#pragma unroll
    for (int u = 0; u < NU; u++) gmask |= (uint32_t)(gk[u] >= s.Tc) << u;
    return gmask;
  }

  __device__ __forceinline__ void stage_B(Sel& s, const uint32_t gmask) {
    __syncwarp();  // e of chunk s.c (written by all lanes) is read back by other lanes
    const int gcnt = __popc(gmask);
    const int gbase = warp_excl_scan(gcnt);
    const int G = (int)__reduce_add_sync(kFull, (unsigned)gcnt);
    int M = 0;
    if (!s.bad) {
      {
        int o = gbase;
        uint32_t mm = gmask;
        while (mm) {
          const int u = __ffs(mm) - 1;
          mm &= mm - 1;
          ws.hist[o++] = (uint32_t)(lane * NU + u);
        }
      }
      __syncwarp();
      // up to BR groups per lane are re-read at once: one L2 round trip, not BR
      constexpr int BR = SLC_BR * 4 / VPU;  // the same loads in flight for either unit size
      for (int r0 = 0; r0 < G; r0 += 32 * BR) {
        float vals[BR][4 * VPU];
        int owner[BR], uu[BR];
#pragma unroll
        for (int bq = 0; bq < BR; bq++) {
          const int gi = r0 + 32 * bq + lane;
          owner[bq] = 0;
          uu[bq] = 0;
          if (gi < G) {
            const uint32_t id = ws.hist[gi];
            owner[bq] = (int)(id / NU);
            uu[bq] = (int)(id % NU);
#pragma unroll
            for (int v = 0; v < VPU; v++) {
              const int q = 32 * (VPU * uu[bq] + v) + owner[bq];
              (DEFER ? load_f32x4 : load_f32x4_l2)(ef, goff<K::RPQ_SHIFT>(s.d, q), s.full ? 4 : valid_in_group(4 * q, s.len),
                         &vals[bq][4 * v]);
            }
          }
        }
        // one warp scan per round: the lane's candidates of all BR units
        uint32_t cmask[BR];
        int cc = 0;
#pragma unroll
        for (int bq = 0; bq < BR; bq++) {
          const int gi = r0 + 32 * bq + lane;
          cmask[bq] = 0;
          if (gi < G) {
#pragma unroll
            for (int v = 0; v < VPU; v++) {
              const int nv = s.full ? 4 : valid_in_group(4 * (32 * (VPU * uu[bq] + v) + owner[bq]), s.len);
#pragma unroll
              for (int j = 0; j < 4; j++)
                if (j < nv && key2_of(vals[bq][4 * v + j]) >= s.Tc) cmask[bq] |= 1u << (4 * v + j);
            }
          }
          cc += __popc(cmask[bq]);
        }
        int o = M + warp_excl_scan(cc);
        M += (int)__reduce_add_sync(kFull, (unsigned)cc);
#pragma unroll
        for (int bq = 0; bq < BR; bq++) {
#pragma unroll
          for (int j = 0; j < 4 * VPU; j++) {
            if ((cmask[bq] >> j) & 1u) {
              const int p = 4 * (32 * (VPU * uu[bq] + (j >> 2)) + owner[bq]) + (j & 3);
              if (o < CAP) {
                ws.cand[o] = ((uint64_t)key2_of(vals[bq][j]) << 16) | (uint64_t)(0xFFFFu - (uint32_t)p);
                ws.candb[o] = vals[bq][j];
              } else if (o < WarpScratch<C, CAP, KMAX, VPU>::XCAP) {
                ws.xkey[o - CAP] = key2_of(vals[bq][j]);
              }
              o++;
            }
          }
        }
      }
    } else {
      M = CAP + 1;
    }
    s.M = M;
    ws.gm[lane] = s.bad ? 0xFFFFFFFFu : gmask;
    if (lane == 0) {
      ws.fb[0] = (uint32_t)G;
      ws.fb[1] = s.Tc;
      ws.fb[2] = (uint32_t)M;
      ws.fb[3] = s.bad ? 1u : 0u;
    }
    for (int w = lane; w < K::BW; w += 32) ws.bit[w] = 0u;
    __syncwarp();
  }

  // ---- R: exact selection -> slots ---------------------------------------------------
  __device__ __forceinline__ void bitmap_prefix() {
    constexpr int WPL = K::BW / 32;
    uint32_t w[WPL];
    int cw = 0;
#pragma unroll
    for (int x = 0; x < WPL; x++) { w[x] = ws.bit[WPL * lane + x]; cw += __popc(w[x]); }
    int pre = warp_excl_scan(cw);
#pragma unroll
    for (int x = 0; x < WPL; x++) { ws.wpre[WPL * lane + x] = (uint32_t)pre; pre += __popc(w[x]); }
  }

  // false: the chunk was deferred (DEFER), Q and F are the fallback kernel's.
  // Deferral entry i: defer[kDeferHdr + i] = chunk; info i (defer_info words
  // at defer + kDeferHdr + defer_cap) = Tc (0: non-finite chunk), then word u = the
  // ballot of group (lane, u) being a candidate group.
  __device__ __forceinline__ bool stage_R(const Sel& s, const uint32_t gmask) {
    if (s.M <= CAP) {
      PATH_COUNT(0);
      rank_select<C, CAP, KMAX, VPU>(ws, lane, s.M, s.k_eff);
    } else if (DEFER) {
      uint32_t i = 0;
      if (lane == 0) i = atomicAdd(&defer[0], 1u);
      i = __shfl_sync(kFull, i, 0);
      uint32_t* info = defer + kDeferHdr + defer_cap + (int64_t)i * defer_info;
#pragma unroll
      for (int u = 0; u < NU; u++) {
        const uint32_t wu = __ballot_sync(kFull, (gmask >> u) & 1u);
        if (lane == u) info[1 + u] = wu;
      }
      if (lane == 0) {
        info[0] = s.bad ? 0u : s.Tc;
        defer[kDeferHdr + i] = (uint32_t)s.c;
      }
      return false;
    } else {
      select_fallback<C, CAP, KMAX, VPU>(ef, &ws, lane, s.d, s.len, s.k_eff);
    }
    __syncwarp();
    return true;
  }

  // ---- Q, F ----------------------------------------------------------------------------
  __device__ __forceinline__ void stage_Q(Sel& s) {
    SLC_CHECK(s.c >= 0 && s.c < n_chunks, "stage_Q chunk");
    SLC_CHECK(s.k_eff >= 1 && s.k_eff <= KMAX, "stage_Q k_eff");
    s.q = warp_quantize_pack<KC, IBC>(ws.selpos, ws.selval, ws.code, k, s.k_eff, g,
                                      records + s.c * g.rec_words, err, rec_extra, n_extra,
                                      s.c * g.rec_words);
  }

  __device__ __forceinline__ void stage_F(const Sel& s) {
    for (int j = lane; j < s.k_eff; j += 32) {
      const int p = (int)ws.selpos[j];
      const float bb = ws.selval[j];
      SLC_CHECK(p >= 0 && p < s.len, "stage_F position");
      SLC_CHECK(pos_off<K::B>(s.d, p) < n_elems, "stage_F offset");
      const float mag = fabsf(bb) > s.q.tau ? s.q.fhi : s.q.flo;
      ef[pos_off<K::B>(s.d, p)] = __fsub_rn(bb, signbit(bb) ? -mag : mag);
    }
    __syncwarp();
  }

  // all stages, in order, for the chunk in s (whose dense e = b is stored)
  __device__ __forceinline__ void select(Sel& s, const uint32_t (&gk)[NU]) {
    PHASE_T0();
    stage_S(s, gk);
    PHASE_MARK(1);
    const uint32_t gmask = group_mask(s, gk);
    stage_B(s, gmask);
    PHASE_MARK(2);
    if (!stage_R(s, gmask)) return;
    PHASE_MARK(3);
    stage_Q(s);
    PHASE_MARK(4);
    stage_F(s);
    PHASE_MARK(5);
  }

  // a chunk the streaming kernel deferred: T and the candidate groups from its
  // deferral info (S is not redone, e is not re-streamed)
  __device__ __forceinline__ void select_deferred(Sel& s, const uint32_t* info) {
    PHASE_T0();
    const uint32_t Tc = info[0];
    s.bad = Tc == 0u;
    s.Tc = s.bad ? 1u : Tc;
    uint32_t gmask = 0;
#pragma unroll
    for (int u = 0; u < NU; u++) gmask |= ((info[1 + u] >> lane) & 1u) << u;
    if (s.bad) gmask = NU == 32 ? 0xFFFFFFFFu : (1u << NU) - 1u;
    stage_B(s, gmask);
    PHASE_MARK(2);
    stage_R(s, gmask);
    PHASE_MARK(3);
    stage_Q(s);
    PHASE_MARK(4);
    stage_F(s);
    PHASE_MARK(5);
  }
};


}  // namespace wsel
}  // namespace slc
