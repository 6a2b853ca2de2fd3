// compress_warp.cu — slc_compress, one WARP per chunk (Eq. 1 of PAPER.md,
// P:68-75; chunk Top-k P:88; C, k P:176).
//
// CTAs of WPC independent warps, no block-level synchronisation.  Warp w walks
// chunks w, w+W, ...  Each warp streams its inputs through its own cp.async
// ring of D pass buffers in shared memory (a pass = 16 positions per lane =
// 512 positions, 6 KB of theta / theta_local / e in fp32): the ring always
// holds the next D passes in flight — including the next chunk's first passes
// while the warp runs the selection of the current one — with no registers
// tied up in loads.  Each lane copies (cp.async, 16 B) and later reads back
// only its own groups, so the ring needs no intra-warp synchronisation.
//
// Per pass: b = fma(beta, e, theta - theta_local) (R#12); e <- b stored at once
// (L2 evict_last: re-read by stage B); the lane keeps each 16-position group's
// max |b|.  Then the selection / quantise / pack / EF-fix-up stages of
// warp_select.cuh.
#include "warp_select.cuh"

namespace slc {
namespace {

using namespace wsel;

#ifndef SLC_RING_D
#define SLC_RING_D 2  // passes in flight per warp
#endif

__device__ __forceinline__ void cp_async_n(void* dst, const void* src, int bytes, int src_bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int C, bool BF16>
struct Ring {
  static constexpr int PB = BF16 ? 2 : 4;
  static constexpr int off_tl = 512 * PB;
  static constexpr int off_e = 1024 * PB;
  static constexpr int pass_bytes = 512 * (2 * PB + 4);
};

template <int C, bool BF16, int KC, int IBC, int CAP, int KMAX, int D>
struct WarpSmem {
  unsigned char ring[D][Ring<C, BF16>::pass_bytes];
  WarpScratch<C, CAP, KMAX> scratch;
};

// issue pass u of chunk d into buf (lane's 4 groups of theta, theta_local, e)
template <int C, bool BF16>
__device__ __forceinline__ void issue_pass(const CompressArgs& a, const ChunkDesc& d, int u, unsigned char* buf,
                                           int lane) {
  using RG = Ring<C, BF16>;
  constexpr int PB = RG::PB;
  const bool full = d.len == C;
#pragma unroll
  for (int v = 0; v < 4; v++) {
    const int q = 128 * u + 32 * v + lane;
    const int nv = full ? 4 : valid_in_group(4 * q, d.len);
    if (nv == 0) continue;
    const int64_t off = goff<WarpCfg<C>::RPQ_SHIFT>(d, q);
    const int slot = v * 32 + lane;
    cp_async_n(buf + slot * 4 * PB, static_cast<const char*>(a.theta) + off * PB, 4 * PB, nv * PB);
    cp_async_n(buf + RG::off_tl + slot * 4 * PB, static_cast<const char*>(a.theta_local) + off * PB, 4 * PB,
               nv * PB);
    cp_async_n(buf + RG::off_e + slot * 16, a.ef + off, 16, nv * 4);
  }
}

template <int C, bool BF16, int KC, int IBC, int CAP, int KMAX, int D, int WPC>
__global__ void __launch_bounds__(WPC * 32, 3) compress_warp_kernel(const CompressArgs a) {
  using K = WarpCfg<C>;
  using RG = Ring<C, BF16>;
  constexpr int NP = K::NP;
  using Smem = WarpSmem<C, BF16, KC, IBC, CAP, KMAX, D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Smem& sm = reinterpret_cast<Smem*>(smem_raw)[warp];
  Compressor<C, BF16, KC, IBC, CAP, KMAX> cp(a, sm.scratch, lane, KC ? KC : a.g.k);
  const int64_t W = (int64_t)gridDim.x * WPC;
  const int64_t first = (int64_t)blockIdx.x * WPC + warp;
  const int64_t n = a.n_chunks;
  const uint64_t pol_last = l2_policy_evict_last();

  // issue cursor: (chunk ic, pass iu), D passes ahead of the consumer
  int64_t ic = first;
  int iu = 0;
  ChunkDesc di;
  di.base = 0; di.ld = 0; di.len = C;
  if (ic < n) di = a.chunks[ic];
  int slot_i = 0;
  auto issue_next = [&]() {
    if (ic < n) issue_pass<C, BF16>(a, di, iu, sm.ring[slot_i], lane);
    cp_async_commit();  // an empty group past the end keeps the wait_group accounting uniform
    slot_i = slot_i + 1 == D ? 0 : slot_i + 1;
    if (++iu == NP) {
      iu = 0;
      ic += W;
      if (ic < n) di = a.chunks[ic];
    }
  };
#pragma unroll
  for (int j = 0; j < D; j++) issue_next();

  int slot_c = 0;
  for (int64_t c = first; c < n; c += W) {
    Sel s;
    s.c = c;
    s.d = a.chunks[c];
    s.len = s.d.len;
    s.full = s.len == C;
    s.k_eff = s.full ? cp.k : max(1, (cp.k * s.len) / C);
    const ChunkDesc& d = s.d;
    PHASE_T0();
    uint32_t gk[NP];
#pragma unroll
    for (int u = 0; u < NP; u++) {
      cp_async_wait<D - 1>();  // this lane's copies of pass u have landed
      const unsigned char* buf = sm.ring[slot_c];
      float gm = 0.0f;
      int nvalid = 0;
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int q = 128 * u + 32 * v + lane;
        const int nv = s.full ? 4 : valid_in_group(4 * q, s.len);
        const int sl = v * 32 + lane;
        float av[4], lv[4];
        if (BF16) {
          const uint2 ua = *reinterpret_cast<const uint2*>(buf + sl * 8);
          const uint2 ul = *reinterpret_cast<const uint2*>(buf + RG::off_tl + sl * 8);
          av[0] = bf16_bits_to_f32(ua.x & 0xFFFFu); av[1] = bf16_bits_to_f32(ua.x >> 16);
          av[2] = bf16_bits_to_f32(ua.y & 0xFFFFu); av[3] = bf16_bits_to_f32(ua.y >> 16);
          lv[0] = bf16_bits_to_f32(ul.x & 0xFFFFu); lv[1] = bf16_bits_to_f32(ul.x >> 16);
          lv[2] = bf16_bits_to_f32(ul.y & 0xFFFFu); lv[3] = bf16_bits_to_f32(ul.y >> 16);
        } else {
          const float4 fa = *reinterpret_cast<const float4*>(buf + sl * 16);
          const float4 fl = *reinterpret_cast<const float4*>(buf + RG::off_tl + sl * 16);
          av[0] = fa.x; av[1] = fa.y; av[2] = fa.z; av[3] = fa.w;
          lv[0] = fl.x; lv[1] = fl.y; lv[2] = fl.z; lv[3] = fl.w;
        }
        const float4 fe = *reinterpret_cast<const float4*>(buf + RG::off_e + sl * 16);
        const float ev[4] = {fe.x, fe.y, fe.z, fe.w};
        float b[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          b[j] = __fmaf_rn(a.beta, ev[j], __fsub_rn(av[j], lv[j]));
          if (j < nv) gm = absmax_nan(gm, b[j]);  // missing positions excluded
        }
        nvalid += nv;
        const int64_t off = goff<K::RPQ_SHIFT>(d, q);
        if (nv == 4) st_f32x4_evict_last(a.ef + off, b[0], b[1], b[2], b[3], pol_last);
        else store_f32x4(a.ef, off, nv, b);
      }
      gk[u] = nvalid ? key2_of(gm) : 0u;
      // this lane is done with the slot: refill it with the pass D ahead (the next
      // chunk's first passes are issued while this chunk is selected)
      issue_next();
      slot_c = slot_c + 1 == D ? 0 : slot_c + 1;
    }
    PHASE_MARK(0);
    cp.select(s, gk);
  }
  cp_async_wait<0>();
}

template <int C, bool BF16, int KC, int IBC, int CAP, int KMAX, int D, int WPC>
cudaError_t launch_warp_t(const CompressArgs& a, cudaStream_t s) {
  using Smem = WarpSmem<C, BF16, KC, IBC, CAP, KMAX, D>;
  constexpr size_t smem = sizeof(Smem) * WPC;
  auto kern = compress_warp_kernel<C, BF16, KC, IBC, CAP, KMAX, D, WPC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPC * 32, smem)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sms * per_sm;
  const int64_t need = (a.n_chunks + WPC - 1) / WPC;
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, WPC * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int C, bool BF16>
cudaError_t launch_warp_c(const CompressArgs& a, cudaStream_t s) {
  if (C == 4096 && a.g.k == 64 && a.g.ib == 12)  // the paper's geometry: small scratch, more warps per SM
    return launch_warp_t<C, BF16, 64, 12, 128, 64, SLC_RING_D, 4>(a, s);
  return launch_warp_t<C, BF16, 0, 0, 256, kMaxK, SLC_RING_D, 4>(a, s);
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

#ifdef SLC_PHASE_TIMING
extern "C" int slc_debug_phase_cycles(unsigned long long* out8, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, g_phase_cycles, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return (int)e;
}
#endif
}  // namespace slc
