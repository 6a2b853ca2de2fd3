// compress_tma.cu — slc_compress for the paper's geometry (C = 4096 as 64x64
// blocks / 4096-chunks, k = 64, 12-bit indices):
// a TMA producer warp feeds warp-per-chunk consumers through a shared-memory
// stage ring.  Eq. 1.
//
// CTA = 1 producer warp + NC consumer warps, one CTA per SM.  CTA b owns the
// chunks b, b+G, b+2G, ... (local index i); a consumer that becomes free
// claims the next i (so stages are drained in order by whichever warp is idle).
//  producer (one lane): for chunk i, wait until stage i % S is empty, arm its
//    mbarrier with the chunk's byte count and issue three TMA copies — a 2-D
//    tensor-map copy of the 64x64 block (theta, theta_local, e) for a
//    blocked chunk, a 1-D bulk copy of 16 KB (x3) for a flat chunk; a
//    partial chunk is only signalled (its consumer reads global memory).
//    S stages of 48 KB (fp32) keep ~100+ KB per SM of HBM reads in flight
//    with no registers or LSU work spent on them.
//  consumer warp: claim chunk i, wait for its stage, read theta,
//    theta_local, e from shared memory (LDS.128, conflict-free), b =
//    fma(beta, e, theta - theta_local) (R#12), store e <- b densely to HBM
//    (L2 evict_last), keep the 256 group maxima, release the stage, then run
//    the selection / quantise / pack / EF-fix-up stages of warp_select.cuh.
// The stage is held only for the short read; the long selection runs
// after the release, so the producer keeps streaming while consumers select.
#include <cuda.h>

#include "ptx.cuh"
#include "warp_select.cuh"

namespace slc {
namespace {

using namespace wsel;

constexpr int kC = 4096;
#ifndef SLC_TMA_NC
#define SLC_TMA_NC 12
#endif
#ifndef SLC_TMA_S
#define SLC_TMA_S 3
#endif
constexpr int kNC = SLC_TMA_NC;  // consumer warps
constexpr int kCapT = 128;       // candidate capacity (k = 64)
constexpr int kKmaxT = 64;

template <bool BF16>
struct TmaCfg {
  static constexpr int PB = BF16 ? 2 : 4;
  static constexpr int S = BF16 ? SLC_TMA_S + 2 : SLC_TMA_S;  // stages
  static constexpr size_t arr_theta = 0;
  static constexpr size_t arr_tl = (size_t)kC * PB;
  static constexpr size_t arr_e = 2 * (size_t)kC * PB;
  static constexpr size_t stage_bytes = (size_t)kC * (2 * PB + 4);
  using Scratch = WarpScratch<kC, kCapT, kKmaxT>;
  static constexpr size_t off_scratch = S * stage_bytes;
  static constexpr size_t off_bar = off_scratch + kNC * sizeof(Scratch);
  static constexpr size_t off_rel = off_bar + 2 * S * sizeof(uint64_t);
  static constexpr size_t bytes = off_rel + (S + 1) * sizeof(int);  // rel[S], next claim
};

__device__ __forceinline__ void tma_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(ptx::smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(ptx::smem_u32(bar))
      : "memory");
}

template <bool BF16>
__global__ void __launch_bounds__(32 * (kNC + 1), 1) compress_tma_kernel(const CompressArgs a) {
  using T = TmaCfg<BF16>;
  constexpr int S = T::S;
  constexpr int NP = WarpCfg<kC>::NP;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + T::off_bar);
  uint64_t* empty = full + S;
  // releases per stage so far: an mbarrier parity wait is only valid within one
  // phase, and with NC > S consumers a consumer could otherwise start waiting
  // on a stage several uses ahead — it first waits until the stage's previous
  // use has been released
  volatile int* rel = reinterpret_cast<volatile int*>(smem + T::off_rel);
  int* next_claim = const_cast<int*>(rel) + S;  // consumers claim chunks in order as they become free
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t G = gridDim.x, n = a.n_chunks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      rel[s] = 0;
    }
    *next_claim = 0;
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ======================= producer =======================
    if (lane != 0) return;
    const CUtensorMap* maps = static_cast<const CUtensorMap*>(a.tmaps);
    for (int64_t i = 0;; ++i) {
      const int64_t c = (int64_t)blockIdx.x + i * G;
      if (c >= n) break;
      const int s = (int)(i % S);
      const int64_t use = i / S;
      if (use > 0) ptx::mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
      const ChunkDesc d = a.chunks[c];
      unsigned char* st = smem + s * T::stage_bytes;
      SLC_CHECK(d.tmap < 0 || 3 * d.tmap + 2 < a.n_tmaps, "producer tmap index");
      SLC_CHECK(d.base >= 0 && d.base + (d.ld ? 63LL * d.ld + 64 : (int64_t)d.len) <= a.n_elems, "producer chunk range");
      if (d.len != kC) {
        ptx::mbar_arrive(&full[s]);  // partial chunk: read from global by the consumer
      } else {
        ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)T::stage_bytes);
        if (d.tmap >= 0) {
          const CUtensorMap* m = maps + 3 * d.tmap;
          tma_2d(st + T::arr_theta, m + 0, d.tx, d.ty, &full[s]);
          tma_2d(st + T::arr_tl, m + 1, d.tx, d.ty, &full[s]);
          tma_2d(st + T::arr_e, m + 2, d.tx, d.ty, &full[s]);
        } else {
          ptx::bulk_g2s(st + T::arr_theta, static_cast<const char*>(a.theta) + d.base * T::PB, kC * T::PB, &full[s]);
          ptx::bulk_g2s(st + T::arr_tl, static_cast<const char*>(a.theta_local) + d.base * T::PB, kC * T::PB,
                        &full[s]);
          ptx::bulk_g2s(st + T::arr_e, a.ef + d.base, kC * 4, &full[s]);
        }
      }
    }
    return;
  }

  // ======================= consumers =======================
  const int cw = warp - 1;
  auto& scratch = reinterpret_cast<typename T::Scratch*>(smem + T::off_scratch)[cw];
  Compressor<kC, BF16, 64, 12, kCapT, kKmaxT> cp(a, scratch, lane, 64);
  const uint64_t pol_last = l2_policy_evict_last();

  (void)cw;
  for (;;) {
    int claim = 0;
    if (lane == 0) claim = atomicAdd(next_claim, 1);
    const int64_t i = __shfl_sync(kFull, claim, 0);
    const int64_t c = (int64_t)blockIdx.x + i * G;
    if (c >= n) break;
    const int s = (int)(i % S);
    Sel sel;
    sel.c = c;
    sel.d = a.chunks[c];
    sel.len = sel.d.len;
    sel.full = sel.len == kC;
    sel.k_eff = sel.full ? 64 : max(1, (64 * sel.len) / kC);
    const ChunkDesc& d = sel.d;
    const unsigned char* st = smem + s * T::stage_bytes;
    const int use = (int)(i / S);
    while (rel[s] < use) __nanosleep(64);
    ptx::mbar_wait(&full[s], (uint32_t)(use & 1));
    SLC_CHECK(d.base >= 0 && d.base + (d.ld ? 63LL * d.ld + 64 : (int64_t)d.len) <= a.n_elems, "consumer chunk range");

    uint32_t gk[NP];
#pragma unroll
    for (int u = 0; u < NP; u++) {
      float av[16], lv[16], ev[16];
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int q = 128 * u + 32 * v + lane;
        const int p0 = 4 * q;
        if (sel.full) {
          if (BF16) {
            const uint2 ua = *reinterpret_cast<const uint2*>(st + T::arr_theta + 2 * p0);
            const uint2 ul = *reinterpret_cast<const uint2*>(st + T::arr_tl + 2 * p0);
            av[4 * v + 0] = bf16_bits_to_f32(ua.x & 0xFFFFu); av[4 * v + 1] = bf16_bits_to_f32(ua.x >> 16);
            av[4 * v + 2] = bf16_bits_to_f32(ua.y & 0xFFFFu); av[4 * v + 3] = bf16_bits_to_f32(ua.y >> 16);
            lv[4 * v + 0] = bf16_bits_to_f32(ul.x & 0xFFFFu); lv[4 * v + 1] = bf16_bits_to_f32(ul.x >> 16);
            lv[4 * v + 2] = bf16_bits_to_f32(ul.y & 0xFFFFu); lv[4 * v + 3] = bf16_bits_to_f32(ul.y >> 16);
          } else {
            const float4 fa = *reinterpret_cast<const float4*>(st + T::arr_theta + 4 * p0);
            const float4 fl = *reinterpret_cast<const float4*>(st + T::arr_tl + 4 * p0);
            av[4 * v + 0] = fa.x; av[4 * v + 1] = fa.y; av[4 * v + 2] = fa.z; av[4 * v + 3] = fa.w;
            lv[4 * v + 0] = fl.x; lv[4 * v + 1] = fl.y; lv[4 * v + 2] = fl.z; lv[4 * v + 3] = fl.w;
          }
          const float4 fe = *reinterpret_cast<const float4*>(st + T::arr_e + 4 * p0);
          ev[4 * v + 0] = fe.x; ev[4 * v + 1] = fe.y; ev[4 * v + 2] = fe.z; ev[4 * v + 3] = fe.w;
        } else {
          const int64_t off = goff<4>(d, q);
          const int nv = valid_in_group(p0, sel.len);
          load_param4<BF16>(a.theta, off, nv, &av[4 * v]);
          load_param4<BF16>(a.theta_local, off, nv, &lv[4 * v]);
          load_f32x4(a.ef, off, nv, &ev[4 * v]);
        }
      }
      float gm = 0.0f;
#pragma unroll
      for (int x = 0; x < 16; x++) {
        av[x] = __fmaf_rn(a.beta, ev[x], __fsub_rn(av[x], lv[x]));  // b
        gm = absmax_nan(gm, av[x]);  // missing positions hold b = 0: never above a valid max
      }
      int nvalid = 16;
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int q = 128 * u + 32 * v + lane;
        const int64_t off = goff<4>(d, q);
        if (sel.full) {
#ifndef SLC_DBG_NOSTORE
          st_f32x4_evict_last(a.ef + off, av[4 * v], av[4 * v + 1], av[4 * v + 2], av[4 * v + 3], pol_last);
#endif
        } else {
          const int nv = valid_in_group(4 * q, sel.len);
          nvalid -= 4 - nv;
          store_f32x4(a.ef, off, nv, &av[4 * v]);
        }
      }
      gk[u] = nvalid ? key2_of(gm) : 0u;
    }
    __syncwarp();
    if (lane == 0) {  // stage read: the producer may refill it
      ptx::mbar_arrive(&empty[s]);
      atomicAdd((int*)&rel[s], 1);
    }
#ifdef SLC_DBG_B
    if (lane == 0 && c < 2)
      printf("consumer chunk %lld a.ef=%p a.records=%p a.n_elems=%lld cp.ef=%p cp.n_elems=%lld\n", (long long)c,
             (void*)a.ef, (void*)a.records, (long long)a.n_elems, (void*)cp.ef, (long long)cp.n_elems);
#endif
#ifndef SLC_DBG_NOSELECT
    cp.select(sel, gk);
#endif
  }
}

template <bool BF16>
cudaError_t launch_tma(const CompressArgs& a, cudaStream_t s) {
  using T = TmaCfg<BF16>;
  constexpr size_t smem = T::bytes;
  auto kern = compress_tma_kernel<BF16>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  int64_t grid = sms;
  if (grid > a.n_chunks) grid = a.n_chunks;
  kern<<<(unsigned)grid, 32 * (kNC + 1), smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool compress_tma_supported(const Geom& g) {
  // Off by default: measured slower than compress_warp.cu on B200 (the 48 KB
  // stage ring caps the bytes in flight per SM at ~3 chunks).
#ifdef SLC_USE_TMA
  return g.C == kC && g.B == 64 && g.k == 64 && g.ib == 12;
#else
  (void)g;
  return false;
#endif
}

cudaError_t launch_compress_tma(const CompressArgs& a, int bf16, cudaStream_t s) {
  if (a.n_chunks == 0) return cudaSuccess;
  if (!compress_tma_supported(a.g)) return cudaErrorInvalidValue;
  return bf16 ? launch_tma<true>(a, s) : launch_tma<false>(a, s);
}

}  // namespace slc
