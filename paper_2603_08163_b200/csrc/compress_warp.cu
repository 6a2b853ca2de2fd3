// compress_warp.cu — slc_compress, one WARP per chunk, reading its chunk
// straight from global memory (Eq. 1 of PAPER.md).  Used for
// C = 1024 and as the general path; the paper's C = 4096 runs the TMA-fed
// kernel of compress_tma.cu.
//
// CTAs of 8 independent warps, no block-level synchronisation.  Warp w walks
// chunks w, w+W, ...: it streams the chunk in NP passes (all 12 128-bit loads
// of a pass issued before any store), forms b = fma(beta, e, theta -
// theta_local) (R#12), stores e <- b densely (L2 evict_last), keeps the 32*NP
// group maxima, then runs the selection stages of warp_select.cuh.
#include "warp_select.cuh"

namespace slc {
namespace {

using namespace wsel;

constexpr int kWarps = 8;  // warps per CTA
constexpr int kCap = 256;

template <int C, bool BF16, int KC, int IBC>
__global__ void __launch_bounds__(kWarps * 32, 2) compress_warp_kernel(const CompressArgs a) {
  using K = WarpCfg<C>;
  constexpr int NP = K::NP;
  using Scratch = WarpScratch<C, kCap, kMaxK>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Compressor<C, BF16, KC, IBC, kCap, kMaxK> cp(a, reinterpret_cast<Scratch*>(smem_raw)[warp], lane,
                                                KC ? KC : a.g.k);
  const int64_t W = (int64_t)gridDim.x * kWarps;
  const uint64_t pol_last = l2_policy_evict_last();

  for (int64_t c = (int64_t)blockIdx.x * kWarps + warp; c < a.n_chunks; c += W) {
    Sel s;
    s.c = c;
    s.d = a.chunks[c];
    s.len = s.d.len;
    s.full = s.len == C;
    s.k_eff = s.full ? cp.k : max(1, (cp.k * s.len) / C);
    const ChunkDesc& d = s.d;
    uint32_t gk[NP];
#pragma unroll
    for (int u = 0; u < NP; u++) {
      float av[16], lv[16], ev[16];
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int q = 128 * u + 32 * v + lane;
        const int64_t off = goff<K::RPQ_SHIFT>(d, q);
        const int nv = s.full ? 4 : valid_in_group(4 * q, s.len);
        load_param4<BF16>(a.theta, off, nv, &av[4 * v]);
        load_param4<BF16>(a.theta_local, off, nv, &lv[4 * v]);
        load_f32x4(a.ef, off, nv, &ev[4 * v]);
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
        const int64_t off = goff<K::RPQ_SHIFT>(d, q);
        if (s.full) {
          st_f32x4_evict_last(a.ef + off, av[4 * v], av[4 * v + 1], av[4 * v + 2], av[4 * v + 3], pol_last);
        } else {
          const int nv = valid_in_group(4 * q, s.len);
          nvalid -= 4 - nv;
          store_f32x4(a.ef, off, nv, &av[4 * v]);
        }
      }
      gk[u] = nvalid ? key2_of(gm) : 0u;
    }
    cp.select(s, gk);
  }
}

template <int C, bool BF16, int KC, int IBC>
cudaError_t launch_warp_t(const CompressArgs& a, cudaStream_t s) {
  constexpr size_t smem = sizeof(WarpScratch<C, kCap, kMaxK>) * kWarps;
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
