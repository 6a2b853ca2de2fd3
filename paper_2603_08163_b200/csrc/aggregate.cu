// aggregate.cu — decode / aggregate / outer-update kernels: Eq. 2 of PAPER.md
// per chunk.
//
// One CTA of C/16 threads per chunk, 16 positions per thread (same mapping and
// 128-bit accesses as the compress kernels).  Modes:
//   kAggOnly       slc_decode_aggregate: Delta -> dense fp32 agg
//   kUpdateFromAgg slc_outer_update(agg != NULL): theta <- fma(-alpha, agg, theta)
//   kFused         slc_outer_update(agg == NULL): decode + aggregate + update in
//                  one pass; Delta never leaves shared memory, so HBM sees the R
//                  records and one read + one write of theta per element.
//
// Aggregation (R#17).  With unit weights every decoded value is an fp16 scale
// with a sign: an integer multiple of 2^-24 below 2^40 units.  The sum is
// accumulated EXACTLY in fixed point: the value is split as hi*2^20 + lo
// (lo < 2^20) and the two halves go to two 32-bit shared-memory counters with
// native ATOMS.ADD (a 64-bit shared atomic add is a CAS loop on sm_100a); with
// R <= 256 neither half can overflow.  The exact sum is order-free, hence
// bit-identical to the oracle's fp64 sum in any peer order; then
// Delta = (float)((double)acc * 2^-24 * (1.0/R)), the oracle's two roundings.
// With weights (median-norm) the sum is fp64 in canonical peer order:
// one warp walks the peers sequentially (no atomics, deterministic).
#include <cuda_fp16.h>

#include <cstring>

#include "chunk_io.cuh"

namespace slc {
namespace {

// fp16 bit pattern (non-negative scale) -> integer multiple of 2^-24
__device__ __forceinline__ long long f16_fixed24(uint32_t h) {
  const uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
  return e == 0 ? (long long)m : (long long)(1024u + m) << (e - 1);
}

// ib-bit index of slot j from the record's index stream (needs rec[w + 1] readable)
__device__ __forceinline__ uint32_t rec_index(const uint32_t* rec, int j, int ib) {
  const int bit = ib * j;
  const int w = bit >> 5, sh = bit & 31;
  return __funnelshift_r(rec[w], rec[w + 1], sh) & ((1u << ib) - 1u);
}

// records of the chunk are staged in shared memory when they fit
constexpr int kRecSmemWords = 8192;  // 32 KB
constexpr int kMaxTable = 256;

template <int C>
struct AggSmem {
  static constexpr size_t off_acc = 0;                                  // int2[C] or double[C]
  static constexpr size_t off_tab = sizeof(int2) * C;                   // int4[R]: lo/hi split of S_lo, S_hi
  static constexpr size_t off_rec = off_tab + sizeof(int4) * kMaxTable;  // u32[R * RW + 1]
  static size_t bytes(int R, int RW, bool staged) {
    return off_rec + (staged ? sizeof(uint32_t) * ((size_t)R * RW + 1) : 0);
  }
};

template <int C, bool BF16>
__global__ void __launch_bounds__(C / 16) aggregate_kernel(const AggArgs a) {
  using K = ChunkCfg<C>;
  using S = AggSmem<C>;
  constexpr int NT = K::NT;
  constexpr int RPQ_SHIFT = (K::RPQ == 8) ? 3 : (K::RPQ == 16 ? 4 : 5);
  extern __shared__ __align__(16) unsigned char smem[];
  int2* acc = reinterpret_cast<int2*>(smem + S::off_acc);        // exact path: (lo, hi) halves
  double* accd = reinterpret_cast<double*>(smem + S::off_acc);   // weighted path
  int4* tab = reinterpret_cast<int4*>(smem + S::off_tab);
  uint32_t* srec = reinterpret_cast<uint32_t*>(smem + S::off_rec);

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t chunk = blockIdx.x;
  const ChunkDesc d = a.chunks[chunk];
  const int len = d.len;
  const int mode = a.mode;

  float th[16], dl[16];
  if (mode == kUpdateFromAgg) {
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const int q = v * NT + t;
      const int64_t off = group_offset(d, q, RPQ_SHIFT);
      const int nv = valid_in_group(4 * q, len);
      load_param4<BF16>(a.theta, off, nv, &th[4 * v]);
      load_f32x4(a.agg, off, nv, &dl[4 * v]);
    }
  } else {
    const int k_eff = max(1, (a.g.k * len) / C);
    const int RW = a.g.rec_words, IW = a.g.idx_words, ib = a.g.ib;
    const bool staged = a.R * RW <= kRecSmemWords;
    if (staged) {
      for (int r = warp; r < a.R; r += NT / 32) {
        const uint32_t* rec = a.rec[r] + chunk * RW;
        for (int w = lane; w < RW; w += 32) srec[r * RW + w] = __ldcs(rec + w);
      }
      if (t == 0) srec[a.R * RW] = 0u;  // rec_index may read one word past the last record
    }
    bool bad = false;
    if (!a.weighted) {
      for (int r = t; r < a.R; r += NT) {  // per record: fixed-point split of its two scales
        const uint32_t sw = __ldg(a.rec[r] + chunk * RW + RW - 1);
        int4 e4;
        const uint32_t h0 = sw & 0xFFFFu, h1 = sw >> 16;
        bad |= ((h0 >> 10) & 0x1Fu) == 0x1Fu || ((h1 >> 10) & 0x1Fu) == 0x1Fu;  // inf / NaN scale
        const long long f0 = f16_fixed24(h0), f1 = f16_fixed24(h1);
        e4.x = (int)(f0 & 0xFFFFF); e4.y = (int)(f0 >> 20);
        e4.z = (int)(f1 & 0xFFFFF); e4.w = (int)(f1 >> 20);
        tab[r] = e4;
      }
      for (int i = t; i < C / 2; i += NT) reinterpret_cast<int4*>(acc)[i] = make_int4(0, 0, 0, 0);
    } else {
      for (int i = t; i < C / 2; i += NT) reinterpret_cast<longlong2*>(accd)[i] = make_longlong2(0, 0);
    }
    __syncthreads();
    if (!a.weighted) {
      const int total = a.R * k_eff;
      for (int s = t; s < total; s += NT) {
        const int r = k_eff == 64 ? (s >> 6) : s / k_eff;
        const int j = s - r * k_eff;
        const uint32_t* rec = staged ? srec + r * RW : a.rec[r] + chunk * RW;
        const uint32_t p = rec_index(rec, j, ib);
        const uint32_t code = (rec[IW + (j >> 4)] >> (2 * (j & 15))) & 3u;
        const int4 e4 = tab[r];
        int lo = (code & 2u) ? e4.z : e4.x;
        int hi = (code & 2u) ? e4.w : e4.y;
        if (code & 1u) { lo = -lo; hi = -hi; }
        if ((int)p >= len) { bad = true; continue; }
        atomicAdd(&acc[p].x, lo);
        atomicAdd(&acc[p].y, hi);
      }
    } else if (t < 32) {
      for (int i = 0; i < a.R; i++) {  // canonical peer order (host-sorted)
        const uint32_t* rec = staged ? srec + i * RW : a.rec[i] + chunk * RW;
        const double w = peer_weight(a, i);
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
      if (a.weighted) {
#pragma unroll
        for (int j = 0; j < 4; j++) dl[4 * v + j] = __double2float_rn(__dmul_rn(accd[p0 + j], invR));
      } else {
        const int4 q0 = reinterpret_cast<const int4*>(acc)[(p0 >> 1)];
        const int4 q1 = reinterpret_cast<const int4*>(acc)[(p0 >> 1) + 1];
        const int lo[4] = {q0.x, q0.z, q1.x, q1.z};
        const int hi[4] = {q0.y, q0.w, q1.y, q1.w};
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const long long s = (long long)hi[j] * (1ll << 20) + (long long)lo[j];
          // exact: |s| < 2^53; untouched positions give +0 as in the oracle
          dl[4 * v + j] = s == 0 ? 0.0f : __double2float_rn(__dmul_rn(__dmul_rn((double)s, 0x1p-24), invR));
        }
      }
    }
    if (mode == kFused) {
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int q = v * NT + t;
        load_param4<BF16>(a.theta, group_offset(d, q, RPQ_SHIFT), valid_in_group(4 * q, len), &th[4 * v]);
      }
    }
  }

  const float alpha = a.alpha;
#pragma unroll
  for (int v = 0; v < 4; v++) {
    const int q = v * NT + t;
    const int nv = valid_in_group(4 * q, len);
    if (nv == 0) continue;
    const int64_t off = group_offset(d, q, RPQ_SHIFT);
    if (mode == kAggOnly) {
      store_f32x4(a.agg, off, nv, &dl[4 * v]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) th[4 * v + j] = __fmaf_rn(-alpha, dl[4 * v + j], th[4 * v + j]);
      store_param4<BF16>(a.theta, off, nv, &th[4 * v]);
    }
  }
}

template <int C, bool BF16>
cudaError_t launch_one(const AggArgs& a, cudaStream_t s) {
  size_t smem = 0;
  if (a.mode != kUpdateFromAgg) {
    if (a.R > kMaxTable) return cudaErrorInvalidValue;
    const bool staged = (size_t)a.R * a.g.rec_words <= (size_t)kRecSmemWords;
    smem = AggSmem<C>::bytes(a.R, a.g.rec_words, staged);
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
  // decode / fused update: the persistent pipelined kernel (aggregate_pipe.cu)
  // by default, else this file's one-CTA-per-chunk kernel.  SLC_OPT_AGG_KERNEL
  // (slc_plan_set_option) pins one of them, or the TMA-tile kernel
  // (aggregate_batch.cu: fused update only, paper geometry; measured slower than
  // the pipelined one on B200) — the parity tests run all of them.
  if (a.mode != kUpdateFromAgg) {
    if (a.variant == 1 && aggregate_batch_supported(a)) return launch_aggregate_batch(a, bf16, s);
    if (a.variant != 3 && aggregate_pipe_supported(a) && !(bf16 && a.mode == kAggOnly))
      return launch_aggregate_pipe(a, bf16, s);
  }
  switch (a.g.C) {
    case 1024: return bf16 ? launch_one<1024, true>(a, s) : launch_one<1024, false>(a, s);
    case 4096: return bf16 ? launch_one<4096, true>(a, s) : launch_one<4096, false>(a, s);
    case 16384: return bf16 ? launch_one<16384, true>(a, s) : launch_one<16384, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace slc
