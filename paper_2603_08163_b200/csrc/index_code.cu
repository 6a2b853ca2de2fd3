// index_code.cu — NEXT row f4: enumerative (colex) rank of each chunk's index
// set, the code that meets P:92's bound log2 binom(C, k) bits per chunk to
// within one bit (reading R#28): rank = sum_i binom(p_i, i + 1) over the
// ascending positions p_0 < ... < p_{k_eff-1} of the chunk's record.
//
// Paper geometry only (C = 4096, k <= 64, 12-bit indices): every binomial
// binom(p, j), p < 4096, j <= 64, is < 2^472 = 15 32-bit limbs.
//  * binom_table_kernel: one CTA of k threads builds the table T[p][j-1] =
//    binom(p, j) row by row with Pascal's rule in multi-precision (4096 rows,
//    a barrier between rows), entries padded to 64 B; built once per plan
//    (16.8 MB of HBM, L2-resident).
//  * index_rank_kernel: one warp per chunk; lane l adds the table entries (four
//    16-B loads each; 15 scalar loads made the kernel L1-bound) of
//    positions l and l + 32 into per-limb 64-bit sums, a xor butterfly sums
//    the lanes, lane 0 propagates the carries and writes 16 limbs.
#include <algorithm>

#include "slc_internal.cuh"

namespace slc {
namespace {

// table loads: read-only cached (__ldg) by default; -DSLC_IC_LOAD=__ldcg (L2 only)
// measured slower: 0.484 vs 0.444 ms on Llama-3.2-1B (the table rows of hot
// low positions do hit in L1)
#ifndef SLC_IC_LOAD
#define SLC_IC_LOAD __ldg
#endif
constexpr int kL = 15;  // limbs of a binomial
constexpr int kS = 16;  // table stride in limbs (64 B: four 16-B loads per entry; limb 15 = 0)

__global__ void __launch_bounds__(64) binom_table_kernel(uint32_t* T, int C, int K) {
  const int j = threadIdx.x + 1;  // binom(p, j)
  for (int p = 0; p < C; p++) {
    uint32_t* out = T + ((int64_t)p * K + (j - 1)) * kS;
    if (j <= K) {
      if (p == 0) {
        for (int l = 0; l < kS; l++) out[l] = 0u;  // binom(0, j) = 0 for j >= 1
      } else {
        const uint32_t* b = T + ((int64_t)(p - 1) * K + (j - 1)) * kS;               // binom(p-1, j)
        const uint32_t* a = j >= 2 ? T + ((int64_t)(p - 1) * K + (j - 2)) * kS : nullptr;  // binom(p-1, j-1)
        uint64_t carry = 0;
        for (int l = 0; l < kL; l++) {
          const uint64_t s = (uint64_t)b[l] + (a ? a[l] : (l == 0 ? 1u : 0u)) + carry;
          out[l] = (uint32_t)s;
          carry = s >> 32;
        }
        out[kL] = 0u;
      }
    }
    __syncthreads();
  }
}

// -DSLC_IC_MINB=3 (80 regs, small spill) measured 0.453 ms vs 0.444 ms without a minimum
#ifdef SLC_IC_MINB
__global__ void __launch_bounds__(256, SLC_IC_MINB) index_rank_kernel(
#else
__global__ void __launch_bounds__(256) index_rank_kernel(
#endif
    const ChunkDesc* chunks, int64_t n_chunks, const uint32_t* rec, const uint32_t* T, uint32_t* ranks, Geom g) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < n_chunks; c += warps) {
    const int ke = max(1, (g.k * __ldg(&chunks[c].len)) / g.C);
    const uint32_t* r = rec + c * g.rec_words;
    uint64_t acc[kL];
#pragma unroll
    for (int l = 0; l < kL; l++) acc[l] = 0;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int i = lane + 32 * h;
      if (i < ke) {
        const int bit = g.ib * i;
        const uint32_t p =
            __funnelshift_r(__ldg(r + (bit >> 5)), __ldg(r + (bit >> 5) + 1), bit & 31) & ((1u << g.ib) - 1u);
        const uint4* t = reinterpret_cast<const uint4*>(T + ((int64_t)p * g.k + i) * kS);  // binom(p, i + 1)
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const uint4 v = SLC_IC_LOAD(t + q);
          acc[4 * q] += v.x;
          acc[4 * q + 1] += v.y;
          acc[4 * q + 2] += v.z;
          if (4 * q + 3 < kL) acc[4 * q + 3] += v.w;
        }
      }
    }
#pragma unroll
    for (int l = 0; l < kL; l++)
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[l] += __shfl_xor_sync(0xffffffffu, acc[l], o);
    if (lane == 0) {
      uint64_t carry = 0;
      uint32_t* out = ranks + c * 16;
#pragma unroll
      for (int l = 0; l < kL; l++) {
        const uint64_t s = acc[l] + carry;
        out[l] = (uint32_t)s;
        carry = s >> 32;
      }
      out[kL] = (uint32_t)carry;
    }
  }
}

}  // namespace

bool index_rank_supported(const Geom& g) { return g.C == 4096 && g.k >= 1 && g.k <= 64 && g.ib == 12; }

cudaError_t build_binom_table(uint32_t* T, const Geom& g, cudaStream_t s) {
  binom_table_kernel<<<1, 64, 0, s>>>(T, g.C, g.k);
  return cudaGetLastError();
}

size_t binom_table_bytes(const Geom& g) { return (size_t)g.C * g.k * kS * sizeof(uint32_t); }

cudaError_t launch_index_rank(const ChunkDesc* chunks, int64_t n_chunks, const uint32_t* rec, const uint32_t* T,
                              uint32_t* ranks, const Geom& g, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (n_chunks + 7) / 8;
  const int grid = (int)std::min<int64_t>(need, (int64_t)sms * 8);
  index_rank_kernel<<<grid, 256, 0, s>>>(chunks, n_chunks, rec, T, ranks, g);
  return cudaGetLastError();
}

}  // namespace slc
