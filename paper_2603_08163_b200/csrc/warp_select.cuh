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
//     in ascending position (R#5).  More than CAP candidates (constant / zero /
//     tied chunks) or a non-finite value: exact radix select over all
//     positions (4 rounds of 8-bit digits).
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
template <int C, int CAP, int KMAX>
struct WarpScratch {
  uint64_t cand[CAP];
  float candb[CAP];
  uint32_t bit[WarpCfg<C>::BW];
  uint32_t wpre[WarpCfg<C>::BW];
  uint32_t hist[256];  // fallback histogram; also the group list of stage B (<= 32*NP <= 256 groups)
  uint32_t selpos[KMAX];
  float selval[KMAX];
  uint32_t code[KMAX];
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
  int M;  // candidates; > CAP: fallback
  QuantOut q;
};

// exact k_eff-th largest key by 4 rounds of 8-bit radix select over all positions,
// then key > K plus the first `need` positions with key == K (lower position wins)
// (a free function: as a member its `this` would pin the Compressor in local memory)
template <int C, int CAP, int KMAX>
__device__ __noinline__ void radix_fallback(float* ef, WarpScratch<C, CAP, KMAX>* wsp, const int lane, const ChunkDesc d,
                                            const int len, const bool full, const int k_eff) {
  using K = WarpCfg<C>;
  constexpr int NP = K::NP;
  WarpScratch<C, CAP, KMAX>& ws = *wsp;
  uint32_t Kth = 0;
  int need = k_eff;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) ws.hist[i] = 0u;
    __syncwarp();
    const uint32_t hi_mask = shift == 24 ? 0u : (0xFFFFFFFFu << (shift + 8));
#pragma unroll 1
    for (int u = 0; u < NP; u++) {
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int q = 128 * u + 32 * v + lane;
        const int nv = full ? 4 : valid_in_group(4 * q, len);
        float ev[4];
        load_f32x4(ef, goff<K::RPQ_SHIFT>(d, q), nv, ev);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t key = key2_of(ev[j]);
          if (j < nv && (key & hi_mask) == (Kth & hi_mask)) atomicAdd(&ws.hist[(key >> shift) & 255u], 1u);
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
  int taken = 0;
#pragma unroll 1
  for (int u = 0; u < NP; u++) {
#pragma unroll
    for (int v = 0; v < 4; v++) {
      // lanes hold consecutive 4-position groups: ascending position = (u, v, lane, j)
      const int q = 128 * u + 32 * v + lane;
      const int nv = full ? 4 : valid_in_group(4 * q, len);
      float ev[4];
      load_f32x4(ef, goff<K::RPQ_SHIFT>(d, q), nv, ev);
      uint32_t tmask = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint32_t key = key2_of(ev[j]);
        if (j < nv && key > Kth) atomicOr(&ws.bit[(4 * q + j) >> 5], 1u << ((4 * q + j) & 31));
        if (j < nv && key == Kth) tmask |= 1u << j;
      }
      const int tc = __popc(tmask);
      int o = taken + warp_excl_scan(tc);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        if ((tmask >> j) & 1u) {
          if (o < need) atomicOr(&ws.bit[(4 * q + j) >> 5], 1u << ((4 * q + j) & 31));
          o++;
        }
      }
      taken += (int)__reduce_add_sync(kFull, (unsigned)tc);
    }
  }
  __syncwarp();
  // slots in ascending position; values re-read from e (= b, written by the stream)
  constexpr int WPL = K::BW / 32;
  uint32_t w[WPL];
  int cw = 0;
#pragma unroll
  for (int x = 0; x < WPL; x++) { w[x] = ws.bit[WPL * lane + x]; cw += __popc(w[x]); }
  int pre = warp_excl_scan(cw);
#pragma unroll
  for (int x = 0; x < WPL; x++) {
    uint32_t y = w[x];
    while (y) {
      const int bp = __ffs(y) - 1;
      y &= y - 1;
      const int p = 32 * (WPL * lane + x) + bp;
      if (pre < KMAX) {
        ws.selpos[pre] = (uint32_t)p;
        ws.selval[pre] = ef[pos_off<K::B>(d, p)];
      }
      pre++;
    }
  }
}

template <int C, bool BF16, int KC, int IBC, int CAP, int KMAX>
struct Compressor {
  using K = WarpCfg<C>;
  static constexpr int NP = K::NP;
  // fields of CompressArgs held by value (a reference to the kernel's param
  // struct would force the struct into local memory)
  float* ef;
  uint32_t* records;
  uint32_t* err;
  const uint64_t* rec_extra;
  int n_extra;
  Geom g;
  int64_t n_elems, n_chunks;
  WarpScratch<C, CAP, KMAX>& ws;
  int lane;
  int k;

  __device__ __forceinline__ Compressor(const CompressArgs& a, WarpScratch<C, CAP, KMAX>& ws_, int lane_, int k_)
      : ef(a.ef),
        records(a.records),
        err(a.err),
        rec_extra(a.rec_extra),
        n_extra(a.n_extra),
        g(a.g),
        n_elems(a.n_elems),
        n_chunks(a.n_chunks),
        ws(ws_),
        lane(lane_),
        k(k_) {}

  // ---- S ---------------------------------------------------------------------------
  __device__ __forceinline__ void stage_S(Sel& s, const uint32_t (&gk)[NP]) {
    uint32_t gmaxk = 0;
#pragma unroll
    for (int u = 0; u < NP; u++) gmaxk = max(gmaxk, gk[u]);
    s.bad = __reduce_max_sync(kFull, gmaxk) >= 0xFF000001u;  // |b| = inf or NaN somewhere
    if (s.bad && lane == 0) atomicOr(err, kErrNonFinite);
    uint32_t T = 0;
#pragma unroll 1
    for (int bit = 31; bit >= 14; --bit) {
      const uint32_t Tp = T | (1u << bit);
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < NP; u++) cnt += gk[u] >= Tp;
      if ((int)__reduce_add_sync(kFull, (unsigned)cnt) >= s.k_eff) T = Tp;
    }
    s.Tc = max(T, 1u);
  }

  // ---- B ---------------------------------------------------------------------------
  __device__ __forceinline__ void stage_B(Sel& s, const uint32_t (&gk)[NP]) {
    __syncwarp();  // e of chunk s.c (written by all lanes) is read back by other lanes
    uint32_t gmask = 0;
#pragma unroll
    for (int u = 0; u < NP; u++) gmask |= (uint32_t)(gk[u] >= s.Tc) << u;
    const int gcnt = __popc(gmask);
    const int gbase = warp_excl_scan(gcnt);
    const int G = (int)__reduce_add_sync(kFull, (unsigned)gcnt);
    int M = 0;
    if (!s.bad && G <= 256) {
      {
        int o = gbase;
        uint32_t mm = gmask;
        while (mm) {
          const int u = __ffs(mm) - 1;
          mm &= mm - 1;
          ws.hist[o++] = (uint32_t)(lane * NP + u);
        }
      }
      __syncwarp();
      // up to BR groups per lane are re-read at once: one L2 round trip, not BR
      constexpr int BR = SLC_BR;
      for (int r0 = 0; r0 < G; r0 += 32 * BR) {
        float vals[BR][16];
        int owner[BR], uu[BR];
#pragma unroll
        for (int bq = 0; bq < BR; bq++) {
          const int gi = r0 + 32 * bq + lane;
          owner[bq] = 0;
          uu[bq] = 0;
          if (gi < G) {
            const uint32_t id = ws.hist[gi];
            owner[bq] = (int)(id / NP);
            uu[bq] = (int)(id % NP);
#pragma unroll
            for (int v = 0; v < 4; v++) {
              const int q = 128 * uu[bq] + 32 * v + owner[bq];
              load_f32x4(ef, goff<K::RPQ_SHIFT>(s.d, q), s.full ? 4 : valid_in_group(4 * q, s.len),
                         &vals[bq][4 * v]);
            }
          }
        }
#pragma unroll
        for (int bq = 0; bq < BR; bq++) {
          const int gi = r0 + 32 * bq + lane;
          uint32_t cmask = 0;
          if (gi < G) {
#pragma unroll
            for (int v = 0; v < 4; v++) {
              const int nv = s.full ? 4 : valid_in_group(4 * (128 * uu[bq] + 32 * v + owner[bq]), s.len);
#pragma unroll
              for (int j = 0; j < 4; j++)
                if (j < nv && key2_of(vals[bq][4 * v + j]) >= s.Tc) cmask |= 1u << (4 * v + j);
            }
          }
          const int cc = __popc(cmask);
          int o = M + warp_excl_scan(cc);
          M += (int)__reduce_add_sync(kFull, (unsigned)cc);
#pragma unroll
          for (int j = 0; j < 16; j++) {
            if ((cmask >> j) & 1u) {
              const int p = 4 * (128 * uu[bq] + 32 * (j >> 2) + owner[bq]) + (j & 3);
              if (o < CAP) {
                ws.cand[o] = ((uint64_t)key2_of(vals[bq][j]) << 16) | (uint64_t)(0xFFFFu - (uint32_t)p);
                ws.candb[o] = vals[bq][j];
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

  __device__ __forceinline__ void stage_R(const Sel& s) {
    const int M = s.M;
    if (M <= CAP) {
      // lane owns candidates lane + 32m; each broadcast candidate is compared with the owned ones
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
        if (lane + 32 * m < M && rank[m] < s.k_eff) {
          const uint32_t p = 0xFFFFu - (uint32_t)(mine[m] & 0xFFFFu);
          atomicOr(&ws.bit[p >> 5], 1u << (p & 31));
        }
      }
      __syncwarp();
      bitmap_prefix();
      __syncwarp();
#pragma unroll
      for (int m = 0; m < MM; m++) {
        const int ci = lane + 32 * m;
        if (ci < M && rank[m] < s.k_eff) {
          const uint32_t p = 0xFFFFu - (uint32_t)(mine[m] & 0xFFFFu);
          const int sl = (int)ws.wpre[p >> 5] + __popc(ws.bit[p >> 5] & ((1u << (p & 31)) - 1u));
          SLC_CHECK(sl >= 0 && sl < s.k_eff && p < (uint32_t)s.len, "stage_R slot");
          ws.selpos[sl] = p;
          ws.selval[sl] = ws.candb[ci];
        }
      }
    } else {
      radix_fallback<C, CAP, KMAX>(ef, &ws, lane, s.d, s.len, s.full, s.k_eff);
    }
    __syncwarp();
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
  __device__ __forceinline__ void select(Sel& s, const uint32_t (&gk)[NP]) {
    PHASE_T0();
    stage_S(s, gk);
    PHASE_MARK(1);
    stage_B(s, gk);
    PHASE_MARK(2);
    stage_R(s);
    PHASE_MARK(3);
    stage_Q(s);
    PHASE_MARK(4);
    stage_F(s);
    PHASE_MARK(5);
  }
};


}  // namespace wsel
}  // namespace slc
