// compress_warp.cu — slc_compress, one WARP per chunk (Eq. 1 of PAPER.md,
// P:68-75; chunking P:88; C, k P:176).
//
// Every warp is an independent chunk worker: CTAs of 8 warps, ~24 warps per SM,
// warp w of the grid walks chunks w, w+W, w+2W, ...  There is no block-level
// synchronisation anywhere — all coordination is __syncwarp / shuffles /
// warp reductions — so the SM always has warps ready to issue, and the many
// warps streaming their inputs keep ~100 KB per SM of loads in flight.
//
// Per chunk (C = 32 * 16 * NP positions; NP passes of 16 positions per lane):
//  A. stream: pass u, lane l owns positions 4q..4q+3 for q = 128u + 32v + l
//     (v = 0..3) — every 128-bit load of a warp covers two whole 256-byte
//     rows of a 64x64 block (or 512 contiguous bytes of a flat chunk).
//     d = theta - theta_local, b = fma(beta, e, d) (R#12); e <- b is stored
//     densely at once (the k selected positions are corrected in step Q);
//     the lane keeps the max |b| of each pass: NP*32 group maxima of 16.
//  S. T = the largest key (bits 31..14) with >= k_eff group maxima >= T, by
//     bitwise search with warp reductions: at least k_eff elements have
//     key >= T, and typically only ~1.2 k_eff do.
//  B. the groups whose max reaches T (~k_eff of them) are spread over the
//     lanes and their 16 values re-read from e (just written: an L2 hit);
//     values with key >= T become candidates key<<16 | ~pos in warp smem.
//  R. exact rank of each candidate by counting (ties: lower position first,
//     R#3, R#4); rank < k_eff -> selected.  More than kCap candidates
//     (constant / zero / heavily tied chunks) or a non-finite value take an
//     exact radix-select fallback over all positions (4 rounds of 8-bit
//     digits, warp-smem histogram).
//  P. selection bitmap -> slots in ascending position (R#5).
//  Q. 2-bit quantiser + record (R#1, R#6, R#13, R#14); selected positions'
//     EF residual e = b - dequant.
#include "chunk_io.cuh"
#include "quant_pack.cuh"

namespace slc {
namespace {

constexpr int kWarps = 8;  // warps per CTA
#ifndef SLC_PFN
#define SLC_PFN 0  // passes of the NEXT chunk prefetched into L2 when a warp leaves its streaming pass
#endif
#ifndef SLC_A2
#define SLC_A2 0   // 1: phase A issues the loads of two passes before consuming them
#endif
#ifndef SLC_MINB
#define SLC_MINB 3  // CTAs per SM the register budget is sized for
#endif

template <int C>
struct WarpCfg {
  static constexpr int NP = C / 512;       // passes of 16 positions per lane
  static constexpr int B = (C == 1024) ? 32 : (C == 4096 ? 64 : 128);
  static constexpr int RPQ_SHIFT = (B == 32) ? 3 : (B == 64 ? 4 : 5);  // log2(B/4)
  static constexpr int BW = C / 32;         // bitmap words
  static constexpr int CAP = 256;           // candidate capacity
};

// per-warp shared scratch
template <int C>
struct WarpScratch {
  uint64_t cand[WarpCfg<C>::CAP];
  float candb[WarpCfg<C>::CAP];
  uint32_t bit[WarpCfg<C>::BW];
  uint32_t wpre[WarpCfg<C>::BW];
  uint32_t hist[256];                     // fallback histogram; also the group list in step B
  uint32_t selpos[kMaxK];
  float selval[kMaxK];
  uint32_t code[kMaxK];
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

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

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

__device__ __forceinline__ int64_t pos_off(const ChunkDesc& d, int p, int B) {
  return d.ld ? d.base + (int64_t)(p / B) * d.ld + (p % B) : d.base + p;
}

template <int C, bool BF16, int KC, int IBC>
__global__ void __launch_bounds__(kWarps * 32, SLC_MINB) compress_warp_kernel(const CompressArgs a) {
  using K = WarpCfg<C>;
  constexpr int NP = K::NP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpScratch<C>& ws = reinterpret_cast<WarpScratch<C>*>(smem_raw)[warp];
  const int64_t W = (int64_t)gridDim.x * kWarps;
  const int k = KC ? KC : a.g.k;
  const uint64_t pol_last = l2_policy_evict_last();

  for (int64_t c = (int64_t)blockIdx.x * kWarps + warp; c < a.n_chunks; c += W) {
    const ChunkDesc d = a.chunks[c];
    const int len = d.len;
    const bool full = len == C;
    const int k_eff = full ? k : max(1, (k * len) / C);

    // ---- A. stream inputs, b, dense e <- b, group maxima -------------------------
    // All loads of a pass (12 x 128-bit per lane; PB passes with SLC_A2) are
    // issued before any store: e may alias nothing here, but the compiler
    // cannot know that, so the order is spelled out.
    uint32_t gk[NP];
    constexpr int PB = SLC_A2 ? 2 : 1;
#pragma unroll
    for (int u0 = 0; u0 < NP; u0 += PB) {
      float av[PB][16], lv[PB][16], ev[PB][16];
      if (full) {
#pragma unroll
        for (int h = 0; h < PB; h++)
#pragma unroll
          for (int v = 0; v < 4; v++) {
            const int64_t off = goff<K::RPQ_SHIFT>(d, 128 * (u0 + h) + 32 * v + lane);
            load_param4<BF16>(a.theta, off, 4, &av[h][4 * v]);
            load_param4<BF16>(a.theta_local, off, 4, &lv[h][4 * v]);
            load_f32x4(a.ef, off, 4, &ev[h][4 * v]);
          }
      } else {
#pragma unroll
        for (int h = 0; h < PB; h++)
#pragma unroll
          for (int v = 0; v < 4; v++) {
            const int q = 128 * (u0 + h) + 32 * v + lane;
            const int64_t off = goff<K::RPQ_SHIFT>(d, q);
            const int nv = valid_in_group(4 * q, len);
            load_param4<BF16>(a.theta, off, nv, &av[h][4 * v]);
            load_param4<BF16>(a.theta_local, off, nv, &lv[h][4 * v]);
            load_f32x4(a.ef, off, nv, &ev[h][4 * v]);
          }
      }
#pragma unroll
      for (int h = 0; h < PB; h++) {
        float gm = 0.0f;
#pragma unroll
        for (int x = 0; x < 16; x++) {
          av[h][x] = __fmaf_rn(a.beta, ev[h][x], __fsub_rn(av[h][x], lv[h][x]));  // b
          gm = absmax_nan(gm, av[h][x]);  // missing positions hold b = 0: never above a valid max
        }
        int nvalid = 4 * 4;
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const int q = 128 * (u0 + h) + 32 * v + lane;
          const int64_t off = goff<K::RPQ_SHIFT>(d, q);
          const float* b = &av[h][4 * v];
          // e <- b, kept L2-resident (evict_last) until the candidate groups are re-read below
          if (full) {
            st_f32x4_evict_last(a.ef + off, b[0], b[1], b[2], b[3], pol_last);
          } else {
            const int nv = valid_in_group(4 * q, len);
            nvalid -= 4 - nv;
            store_f32x4(a.ef, off, nv, b);
          }
        }
        gk[u0 + h] = nvalid ? key2_of(gm) : 0u;
      }
    }

#ifdef SLC_STREAM_ONLY  // bandwidth probe: the streaming pass alone (tools/, never shipped)
    if (lane == 0 && gk[0] == 0x12345u) a.records[c] = gk[1];
    continue;
#endif
#if SLC_PFN > 0
    if (c + W < a.n_chunks) {  // the next chunk's first passes travel to L2 while this warp selects
      const ChunkDesc dn = a.chunks[c + W];
      if (dn.len == C) {
#pragma unroll
        for (int u = 0; u < SLC_PFN; u++)
#pragma unroll
          for (int v = 0; v < 4; v++) {
            const int64_t off = goff<K::RPQ_SHIFT>(dn, 128 * u + 32 * v + lane);
            prefetch_l2(static_cast<const char*>(a.theta) + off * (BF16 ? 2 : 4));
            prefetch_l2(static_cast<const char*>(a.theta_local) + off * (BF16 ? 2 : 4));
            prefetch_l2(a.ef + off);
          }
      }
    }
#endif
    // ---- S. lower bound T ----------------------------------------------------------
    uint32_t gmaxk = 0;
#pragma unroll
    for (int u = 0; u < NP; u++) gmaxk = max(gmaxk, gk[u]);
    const bool bad = __reduce_max_sync(kFull, gmaxk) >= 0xFF000001u;  // |b| = inf or NaN somewhere
    if (bad && lane == 0) atomicOr(a.err, kErrNonFinite);
    uint32_t T = 0;
#pragma unroll
    for (int bit = 31; bit >= 14; --bit) {
      const uint32_t Tp = T | (1u << bit);
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < NP; u++) cnt += gk[u] >= Tp;
      if ((int)__reduce_add_sync(kFull, (unsigned)cnt) >= k_eff) T = Tp;
    }
    const uint32_t Tc = max(T, 1u);
    __syncwarp();  // e written above is read back by other lanes below

    // ---- B. candidates from the groups that reach T ------------------------------
    uint32_t gmask = 0;
#pragma unroll
    for (int u = 0; u < NP; u++) gmask |= (uint32_t)(gk[u] >= Tc) << u;
    const int gcnt = __popc(gmask);
    const int gbase = warp_excl_scan(gcnt);
    const int G = (int)__reduce_add_sync(kFull, (unsigned)gcnt);
    int M = 0;
    if (!bad && G <= 256) {
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
      for (int r = 0; r < G; r += 32) {
        const int gi = r + lane;
        uint32_t cmask = 0;
        int owner = 0, u = 0;
        float vals[16];
        if (gi < G) {
          const uint32_t id = ws.hist[gi];
          owner = (int)(id / NP);
          u = (int)(id % NP);
#pragma unroll
          for (int v = 0; v < 4; v++) {
            const int q = 128 * u + 32 * v + owner;
            const int64_t off = goff<K::RPQ_SHIFT>(d, q);
            const int nv = full ? 4 : valid_in_group(4 * q, len);
            float ev[4];
            load_f32x4(a.ef, off, nv, ev);
#pragma unroll
            for (int j = 0; j < 4; j++) {
              vals[4 * v + j] = ev[j];
              if (j < nv && key2_of(ev[j]) >= Tc) cmask |= 1u << (4 * v + j);
            }
          }
        }
        const int cc = __popc(cmask);
        const int cb = M + warp_excl_scan(cc);
        M += (int)__reduce_add_sync(kFull, (unsigned)cc);
        int o = cb;
#pragma unroll
        for (int j = 0; j < 16; j++) {
          if ((cmask >> j) & 1u) {
            const int p = 4 * (128 * u + 32 * (j >> 2) + owner) + (j & 3);
            if (o < K::CAP) {
              ws.cand[o] = ((uint64_t)key2_of(vals[j]) << 16) | (uint64_t)(0xFFFFu - (uint32_t)p);
              ws.candb[o] = vals[j];
            }
            o++;
          }
        }
      }
    } else {
      M = K::CAP + 1;
    }
    for (int w = lane; w < K::BW; w += 32) ws.bit[w] = 0u;
    __syncwarp();

    // ---- R. exact selection -> bitmap ----------------------------------------------
    if (M <= K::CAP) {
      // lane owns candidates lane + 32m; each broadcast candidate is compared with all owned ones
      const int NM = (M + 31) >> 5;
      uint64_t mine[K::CAP / 32];
      int rank[K::CAP / 32];
#pragma unroll
      for (int m = 0; m < K::CAP / 32; m++) {
        mine[m] = (m < NM && lane + 32 * m < M) ? ws.cand[lane + 32 * m] : ~0ull;
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
          for (int m = 0; m < K::CAP / 32; m++) rank[m] += x > mine[m];
        }
      }
#pragma unroll
      for (int m = 0; m < K::CAP / 32; m++) {
        const int ci = lane + 32 * m;
        if (m < NM && ci < M && rank[m] < k_eff) {
          const uint32_t p = 0xFFFFu - (uint32_t)(mine[m] & 0xFFFFu);
          atomicOr(&ws.bit[p >> 5], 1u << (p & 31));
        }
      }
      __syncwarp();
      // ---- P. slot = selected positions below p (bitmap prefix) ----------------------------
      {
        constexpr int WPL = K::BW / 32;
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
      for (int m = 0; m < K::CAP / 32; m++) {
        const int ci = lane + 32 * m;
        if (m < NM && ci < M && rank[m] < k_eff) {
          const uint32_t p = 0xFFFFu - (uint32_t)(mine[m] & 0xFFFFu);
          const int sl = (int)ws.wpre[p >> 5] + __popc(ws.bit[p >> 5] & ((1u << (p & 31)) - 1u));
          ws.selpos[sl] = p;
          ws.selval[sl] = ws.candb[ci];
        }
      }
    } else {
      // ---- fallback: exact k_eff-th largest key by 4 rounds of 8-bit radix select ----
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
            load_f32x4(a.ef, goff<K::RPQ_SHIFT>(d, q), nv, ev);
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
        // suffix sum of lanes above
        uint32_t above = 0;
        {
          uint32_t inc = s8;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_down_sync(kFull, inc, o);
            if (lane + o < 32) inc += y;
          }
          above = inc - s8;  // sum of bins in lanes > lane
        }
        int found = -1;
        uint32_t found_gt = 0;
        uint32_t acc = above;
#pragma unroll
        for (int x = 7; x >= 0; x--) {
          if (found < 0 && acc < (uint32_t)need && acc + h[x] >= (uint32_t)need) { found = 8 * lane + x; found_gt = acc; }
          acc += h[x];
        }
        const unsigned who = __ballot_sync(kFull, found >= 0);
        const int src = __ffs(who) - 1;
        const int D = __shfl_sync(kFull, found, src);
        const uint32_t gt = __shfl_sync(kFull, found_gt, src);
        Kth |= (uint32_t)D << shift;
        need -= (int)gt;
        __syncwarp();
      }
      // select key > Kth, and the first `need` positions with key == Kth (lower position wins)
      int taken = 0;
#pragma unroll 1
      for (int u = 0; u < NP; u++) {
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const int q = 128 * u + 32 * v + lane;
          const int nv = full ? 4 : valid_in_group(4 * q, len);
          float ev[4];
          load_f32x4(a.ef, goff<K::RPQ_SHIFT>(d, q), nv, ev);
          // lanes hold consecutive 4-position groups in position order: q = base + lane
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint32_t key = key2_of(ev[j]);
            const bool gtk = j < nv && key > Kth;
            if (gtk) atomicOr(&ws.bit[(4 * q + j) >> 5], 1u << ((4 * q + j) & 31));
          }
          // ties in ascending position within this (u, v) row of 128 positions
          uint32_t tmask = 0;
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint32_t key = key2_of(ev[j]);
            if (j < nv && key == Kth) tmask |= 1u << j;
          }
          const int tc = __popc(tmask);
          const int before = taken + warp_excl_scan(tc);
          int o = before;
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
      // slots in ascending position; values re-read from e (b, written in step A)
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
          if (pre < kMaxK) {
            ws.selpos[pre] = (uint32_t)p;
            ws.selval[pre] = a.ef[pos_off(d, p, K::B)];
          }
          pre++;
        }
      }
    }
    __syncwarp();

    // ---- Q. quantise, record, EF residual of the selected positions ---------------------
    const QuantOut qo = warp_quantize_pack<KC, IBC>(ws.selpos, ws.selval, ws.code, k, k_eff, a.g,
                                                    a.records + c * a.g.rec_words, a.err);
    for (int j = lane; j < k_eff; j += 32) {
      const int p = (int)ws.selpos[j];
      const float bb = ws.selval[j];
      const float mag = fabsf(bb) > qo.tau ? qo.fhi : qo.flo;
      a.ef[pos_off(d, p, K::B)] = __fsub_rn(bb, signbit(bb) ? -mag : mag);
    }
    __syncwarp();
  }
}

template <int C, bool BF16, int KC, int IBC>
cudaError_t launch_warp_t(const CompressArgs& a, cudaStream_t s) {
  constexpr size_t smem = sizeof(WarpScratch<C>) * kWarps;
  auto kern = compress_warp_kernel<C, BF16, KC, IBC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sms * per_sm;
  const int64_t need = (a.n_chunks + kWarps - 1) / kWarps;
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, kWarps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int C, bool BF16>
cudaError_t launch_warp_c(const CompressArgs& a, cudaStream_t s) {
  if (C == 4096 && a.g.k == 64 && a.g.ib == 12) return launch_warp_t<C, BF16, 64, 12>(a, s);
  return launch_warp_t<C, BF16, 0, 0>(a, s);
}

}  // namespace

cudaError_t launch_compress_warp(const CompressArgs& a, int bf16, cudaStream_t s) {
  if (a.n_chunks == 0) return cudaSuccess;
  switch (a.g.C) {
    case 1024: return bf16 ? launch_warp_c<1024, true>(a, s) : launch_warp_c<1024, false>(a, s);
    case 4096: return bf16 ? launch_warp_c<4096, true>(a, s) : launch_warp_c<4096, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace slc
