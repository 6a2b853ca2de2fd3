// aggregate.cu — decode / aggregate / outer-update kernels: Eq. 2 of PAPER.md
// per chunk.
//
// One CTA of C/16 threads per chunk, 16 positions per thread (same mapping and
// 128-bit accesses as compress).  Modes:
//   kAggOnly       slc_decode_aggregate: Delta -> dense fp32 agg
//   kUpdateFromAgg slc_outer_update(agg != NULL): theta <- fma(-alpha, agg, theta)
//   kFused         slc_outer_update(agg == NULL): decode + aggregate + update in
//                  one pass; Delta never leaves shared memory, so HBM sees the R
//                  records and one read + one write of theta per element.
// Aggregation (R#17): with unit weights every decoded value is an fp16 scale
// with a sign, i.e. an integer multiple of 2^-24 below 2^16, so the sum is
// accumulated EXACTLY as a 64-bit fixed-point integer (units of 2^-24) with
// shared-memory atomics — order-free, so bit-identical to the oracle's fp64
// sum in any peer order.  Delta = (float)((double)acc * 2^-24 * (1.0/R)), the
// same two roundings as the oracle.  With weights (median-norm) the sum
// is fp64 in canonical peer order, one warp walking the peers sequentially.
#include <cuda_fp16.h>

#include "chunk_io.cuh"

namespace slc {
namespace {

// fp16 bit pattern (non-negative scale) -> integer multiple of 2^-24
__device__ __forceinline__ long long f16_fixed24(uint32_t h) {
  const uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
  return e == 0 ? (long long)m : (long long)(1024u + m) << (e - 1);
}

__device__ __forceinline__ uint32_t rec_index(const uint32_t* rec, int j, int ib) {
  const int bit = ib * j;
  const int w = bit >> 5, sh = bit & 31;
  uint64_t two = rec[w];
  if (sh + ib > 32) two |= (uint64_t)rec[w + 1] << 32;
  return (uint32_t)(two >> sh) & ((1u << ib) - 1u);
}

// records of the chunk are staged in shared memory when they fit
constexpr int kRecSmemWords = 8192;  // 32 KB

template <int C, bool BF16>
__global__ void __launch_bounds__(C / 16) aggregate_kernel(const AggArgs a) {
  using K = ChunkCfg<C>;
  constexpr int NT = K::NT;
  constexpr int RPQ_SHIFT = (K::RPQ == 8) ? 3 : (K::RPQ == 16 ? 4 : 5);
  extern __shared__ __align__(16) unsigned char smem[];
  long long* acc = reinterpret_cast<long long*>(smem);  // exact path
  double* accd = reinterpret_cast<double*>(smem);       // weighted path
  uint32_t* srec = reinterpret_cast<uint32_t*>(smem + sizeof(long long) * C);

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t chunk = blockIdx.x;
  const ChunkDesc d = a.chunks[chunk];
  const int len = d.len;
  const int mode = a.mode;

  float th[16], dl[16];
  int64_t off[4];
  int nvs[4];
#pragma unroll
  for (int v = 0; v < 4; v++) {
    const int q = v * NT + t;
    off[v] = group_offset(d, q, RPQ_SHIFT);
    nvs[v] = valid_in_group(4 * q, len);
  }
#ifdef SLC_AGG_THETA_FIRST
  // theta (and agg) first: their HBM latency overlaps the decode below
#pragma unroll
  for (int v = 0; v < 4; v++) {
    if (mode != kAggOnly) load_param4<BF16>(a.theta, off[v], nvs[v], &th[4 * v]);
    if (mode == kUpdateFromAgg) load_f32x4(a.agg, off[v], nvs[v], &dl[4 * v]);
  }
#else
  if (mode == kUpdateFromAgg) {
#pragma unroll
    for (int v = 0; v < 4; v++) {
      load_param4<BF16>(a.theta, off[v], nvs[v], &th[4 * v]);
      load_f32x4(a.agg, off[v], nvs[v], &dl[4 * v]);
    }
  }
#endif

#ifdef SLC_STREAM_ONLY  // bandwidth probe: theta read + write only (tools/, never shipped)
  if (mode == kFused) {
#pragma unroll
    for (int v = 0; v < 4; v++) store_param4<BF16>(a.theta, off[v], nvs[v], &th[4 * v]);
    return;
  }
#endif
  if (mode != kUpdateFromAgg) {
    const int k_eff = max(1, (a.g.k * len) / C);
    const int RW = a.g.rec_words, IW = a.g.idx_words, ib = a.g.ib;
    const bool staged = a.R * RW <= kRecSmemWords;
    if (staged) {
      for (int r = warp; r < a.R; r += NT / 32) {
        const uint32_t* rec = a.rec[r] + chunk * RW;
        for (int w = lane; w < RW; w += 32) srec[r * RW + w] = __ldcs(rec + w);
      }
    }
    for (int i = t; i < C / 2; i += NT) reinterpret_cast<longlong2*>(acc)[i] = make_longlong2(0, 0);
    __syncthreads();
    bool bad = false;
    if (!a.weighted) {
      const int total = a.R * k_eff;
      for (int s = t; s < total; s += NT) {
        const int r = k_eff == 64 ? (s >> 6) : s / k_eff;
        const int j = s - r * k_eff;
        const uint32_t* rec = staged ? srec + r * RW : a.rec[r] + chunk * RW;
        const uint32_t p = rec_index(rec, j, ib);
        const uint32_t code = (rec[IW + (j >> 4)] >> (2 * (j & 15))) & 3u;
        const uint32_t sw = rec[RW - 1];
        const uint32_t h = (code & 2u) ? (sw >> 16) : (sw & 0xFFFFu);
        if ((int)p >= len || ((h >> 10) & 0x1Fu) == 0x1Fu) { bad = true; continue; }
        long long v = f16_fixed24(h);
        if (code & 1u) v = -v;
        atomicAdd(reinterpret_cast<unsigned long long*>(&acc[p]), (unsigned long long)v);
      }
    } else if (t < 32) {
      for (int i = 0; i < a.R; i++) {  // canonical peer order (host-sorted)
        const uint32_t* rec = staged ? srec + i * RW : a.rec[i] + chunk * RW;
        const double w = (double)a.w[i];
        const uint32_t sw = rec[RW - 1];
        for (int j = t; j < k_eff; j += 32) {
          const uint32_t p = rec_index(rec, j, ib);
          const uint32_t code = (rec[IW + (j >> 4)] >> (2 * (j & 15))) & 3u;
          const uint32_t h = (code & 2u) ? (sw >> 16) : (sw & 0xFFFFu);
          if ((int)p >= len || ((h >> 10) & 0x1Fu) == 0x1Fu) { bad = true; continue; }
          float dq = __half2float(__ushort_as_half((unsigned short)h));
          if (code & 1u) dq = -dq;
          accd[p] = __dadd_rn(accd[p], __dmul_rn(w, (double)dq));
        }
        __syncwarp();
      }
    }
    if (bad) atomicOr(a.err, kErrNonFinite);
    __syncthreads();
    const double invR = a.invR;
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const int p0 = 4 * (v * NT + t);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const double x = a.weighted ? accd[p0 + j] : __dmul_rn((double)acc[p0 + j], 0x1p-24);
        dl[4 * v + j] = __double2float_rn(__dmul_rn(x, invR));
      }
    }
  }

#ifndef SLC_AGG_THETA_FIRST
  if (mode == kFused) {
#pragma unroll
    for (int v = 0; v < 4; v++) load_param4<BF16>(a.theta, off[v], nvs[v], &th[4 * v]);
  }
#endif
  const float alpha = a.alpha;
#pragma unroll
  for (int v = 0; v < 4; v++) {
    if (nvs[v] == 0) continue;
    if (mode == kAggOnly) {
      store_f32x4(a.agg, off[v], nvs[v], &dl[4 * v]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) th[4 * v + j] = __fmaf_rn(-alpha, dl[4 * v + j], th[4 * v + j]);
      store_param4<BF16>(a.theta, off[v], nvs[v], &th[4 * v]);
    }
  }
}

template <int C, bool BF16>
cudaError_t launch_one(const AggArgs& a, cudaStream_t s) {
  size_t smem = 0;
  if (a.mode != kUpdateFromAgg) {
    smem = sizeof(long long) * C;
    if ((size_t)a.R * a.g.rec_words <= (size_t)kRecSmemWords) smem += sizeof(uint32_t) * a.R * a.g.rec_words;
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(aggregate_kernel<C, BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (a.n_chunks > 0x7FFFFFFFll) return cudaErrorInvalidValue;
  aggregate_kernel<C, BF16><<<(unsigned)a.n_chunks, ChunkCfg<C>::NT, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_aggregate(const AggArgs& a, int bf16, cudaStream_t s) {
  if (a.n_chunks == 0) return cudaSuccess;
  switch (a.g.C) {
    case 1024: return bf16 ? launch_one<1024, true>(a, s) : launch_one<1024, false>(a, s);
    case 4096: return bf16 ? launch_one<4096, true>(a, s) : launch_one<4096, false>(a, s);
    case 16384: return bf16 ? launch_one<16384, true>(a, s) : launch_one<16384, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace slc
