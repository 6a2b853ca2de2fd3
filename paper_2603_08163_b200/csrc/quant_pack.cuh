// quant_pack.cuh — pieces shared by the compress kernels: Top-k key, block
// counting, and the single-warp quantiser + record packer.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "slc_internal.cuh"

namespace slc {

constexpr unsigned kFull = 0xFFFFFFFFu;

// key(b) = |b| bits + 1 (order-preserving for finite b; 0 = missing position)
__device__ __forceinline__ uint32_t key_of(float b) { return (__float_as_uint(b) & 0x7FFFFFFFu) + 1u; }
// key2(b) = |b| bits << 1 | 1 — same order, one instruction (LEA); 0 = missing
__device__ __forceinline__ uint32_t key2_of(float b) { return (__float_as_uint(b) << 1) | 1u; }

// xor butterfly of __fadd_rn: lane l < d adds u_{l+d} exactly as the oracle's
// tree (R#13); the partner lane computes the same commutative sum, so every
// lane ends with the oracle's u_0.
__device__ __forceinline__ float warp_tree_sum(float u) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) u = __fadd_rn(u, __shfl_xor_sync(kFull, u, d));
  return u;
}

// sum over the NT threads of named barrier BAR
template <int NT, int BAR>
__device__ __forceinline__ int block_sum_named(int v, int* s_w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = __reduce_add_sync(kFull, v);
  if (lane == 0) s_w[warp] = v;
  asm volatile("barrier.cta.sync.aligned %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
  int tot = 0;
#pragma unroll
  for (int i = 0; i < NT / 32; i++) tot += s_w[i];
  asm volatile("barrier.cta.sync.aligned %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
  return tot;
}

template <int NT>
__device__ __forceinline__ int block_sum(int v, int* s_w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = __reduce_add_sync(kFull, v);
  if (lane == 0) s_w[warp] = v;
  __syncthreads();
  int tot = 0;
#pragma unroll
  for (int i = 0; i < NT / 32; i++) tot += s_w[i];
  __syncthreads();
  return tot;
}

__device__ __forceinline__ int warp_excl_scan(int c) {
  const int lane = threadIdx.x & 31;
  int inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  return inc - c;
}

struct QuantOut {
  float tau, flo, fhi;
};

// One full warp.  selpos/selval hold the k_eff selected positions / values in
// ascending position order.  Computes the 2-bit quantiser of R#1 with the
// fixed-order sums of R#13 and fp16 scales (R#14), writes the record (R#6) and
// returns tau and the decoded scales.  selcode is scratch (k entries).
// KC / IBC > 0 fix k / index_bits at compile time (the paper's 64 / 12),
// which unrolls the slot loops and turns the packing divisions into shifts.
template <int KC = 0, int IBC = 0>
__device__ __forceinline__ QuantOut warp_quantize_pack(const uint32_t* selpos, const float* selval,
                                                       uint32_t* selcode, int k_rt, int k_eff, const Geom& g,
                                                       uint32_t* rec, uint32_t* err, const uint64_t* extra = nullptr,
                                                       int n_extra = 0, int64_t rec_word = 0) {
  const int lane = threadIdx.x & 31;
  const int k = KC ? KC : k_rt;
  const int W = (k + 31) >> 5;
  float u = 0.0f;
  for (int m = 0; m < W; m++) {
    const int j = lane + 32 * m;
    u = __fadd_rn(u, j < k_eff ? fabsf(selval[j]) : 0.0f);
  }
  const float tau = __fdiv_rn(warp_tree_sum(u), (float)k_eff);
  float ulo = 0.0f, uhi = 0.0f;
  int nhi = 0;
  for (int m = 0; m < W; m++) {
    const int j = lane + 32 * m;
    if (j < k_eff) {
      const float v = selval[j];
      const float av = fabsf(v);
      const bool h = av > tau;
      ulo = __fadd_rn(ulo, h ? 0.0f : av);
      uhi = __fadd_rn(uhi, h ? av : 0.0f);
      nhi += h;
      selcode[j] = (signbit(v) ? 1u : 0u) | (h ? 2u : 0u);
    }
  }
  const float sum_lo = warp_tree_sum(ulo), sum_hi = warp_tree_sum(uhi);
  nhi = __reduce_add_sync(kFull, nhi);
  const int nlo = k_eff - nhi;
  const float s_lo = nlo > 0 ? __fdiv_rn(sum_lo, (float)nlo) : 0.0f;
  const float s_hi = nhi > 0 ? __fdiv_rn(sum_hi, (float)nhi) : tau;
  const __half hlo = __float2half_rn(s_lo), hhi = __float2half_rn(s_hi);
  QuantOut q;
  q.tau = tau;
  q.flo = __half2float(hlo);
  q.fhi = __half2float(hhi);
  if (lane == 0 && (isinf(q.flo) || isinf(q.fhi))) atomicOr(err, kErrScaleOverflow);
  const uint32_t scale_word = (uint32_t)__half_as_ushort(hlo) | ((uint32_t)__half_as_ushort(hhi) << 16);
  __syncwarp();
  const int ib = IBC ? IBC : g.ib;
  const int IW = (KC && IBC) ? (KC * IBC + 31) / 32 : g.idx_words;
  const int CW = KC ? (2 * KC + 31) / 32 : g.code_words;
  const int RW = IW + CW + 1;
  for (int wi = lane; wi < RW; wi += 32) {
    uint32_t word = 0;
    if (wi < IW) {
      const int b0 = 32 * wi;
      const int j0 = b0 / ib, j1 = min((b0 + 31) / ib, k_eff - 1);
      for (int j = j0; j <= j1; j++) {
        const int sh = ib * j - b0;
        const uint32_t pv = selpos[j];
        word |= sh >= 0 ? (pv << sh) : (pv >> (-sh));
      }
    } else if (wi < IW + CW) {
      const int j0 = 16 * (wi - IW);
      for (int j = j0; j < min(j0 + 16, k_eff); j++) word |= selcode[j] << (2 * (j - j0));
    } else {
      word = scale_word;
    }
    rec[wi] = word;
    // the same record pushed to every extra destination (slc_compress_multi:
    // e.g. each rank's peer message over NVLink — the a8 all-gather folded
    // into the compress kernel)
    for (int e = 0; e < n_extra; e++) reinterpret_cast<uint32_t*>(__ldg(extra + e))[rec_word + wi] = word;
  }
  return q;
}

}  // namespace slc
