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

// ---- entropy-coded (EC) records (R#28): 15 rank limbs + the record's code
// words + its scale word; ec_words = 15 + code_words + 1 (20 = 80 B at k = 64)

// one warp per chunk: the colex rank as in index_rank_kernel, written with the
// record's code and scale words into the EC record
__global__ void __launch_bounds__(256) index_encode_kernel(const ChunkDesc* chunks, int64_t n_chunks,
                                                           const uint32_t* rec, const uint32_t* T, uint32_t* ec,
                                                           Geom g) {
  const int lane = threadIdx.x & 31;
  const int ecw = kL + g.code_words + 1;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < n_chunks; c += warps) {
    const int ke = max(1, (g.k * __ldg(&chunks[c].len)) / g.C);
    const uint32_t* r = rec + c * g.rec_words;
    uint32_t* out = ec + c * ecw;
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
          const uint4 v = __ldg(t + q);
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
#pragma unroll
      for (int l = 0; l < kL; l++) {
        const uint64_t s = acc[l] + carry;
        out[l] = (uint32_t)s;
        carry = s >> 32;
      }
    }
    for (int w = lane; w < g.code_words + 1; w += 32) out[kL + w] = __ldg(r + g.idx_words + w);
  }
}

// C(p, j) <= r for the table entry of (p, j) and the 15-limb r (most significant limb first)
__device__ __forceinline__ bool binom_le(const uint32_t* T, int K, int p, int j, const uint32_t (&r)[kL]) {
  const uint4* t = reinterpret_cast<const uint4*>(T + ((int64_t)p * K + (j - 1)) * kS);
#pragma unroll
  for (int q = 3; q >= 0; q--) {
    const uint4 v = __ldg(t + q);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 3; e >= 0; e--) {
      const int l = 4 * q + e;
      if (l >= kL) continue;
      if (w[e] != r[l]) return w[e] < r[l];
    }
  }
  return true;  // equal
}

// one warp per chunk: greedy colex unranking (R#28), p_i = the largest p with
// binom(p, i + 1) <= the remaining rank, for i = k_eff - 1 .. 0; each step is a
// 32-way search (every lane tests one candidate, a ballot keeps the largest
// that fits), then binom(p_i, i + 1) is subtracted (every lane keeps all 15
// limbs).  The positions are packed back into the R#6 index stream; a rank
// that does not reduce to 0 (not a valid code) latches INVALID_DATA.
__global__ void __launch_bounds__(256) index_decode_kernel(const ChunkDesc* chunks, int64_t n_chunks,
                                                           const uint32_t* ec, const uint32_t* T, uint32_t* rec,
                                                           uint32_t* err, Geom g) {
  __shared__ uint16_t spos[8][64];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int ecw = kL + g.code_words + 1;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  bool bad = false;
  for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; c < n_chunks; c += warps) {
    const int len = __ldg(&chunks[c].len);
    const int ke = max(1, (g.k * len) / g.C);
    const uint32_t* e = ec + c * ecw;
    uint32_t r[kL];
#pragma unroll
    for (int l = 0; l < kL; l++) r[l] = __ldg(e + l);
    int hi = len - 1;
    for (int i = ke - 1; i >= 0; i--) {
      const int j = i + 1;
      int lo = i;  // binom(i, i + 1) = 0 <= r: the answer lies in [lo, hi]
      while (hi > lo) {
        const int step = (hi - lo + 32) >> 5;  // ceil((hi - lo + 1) / 32)
        const int cand = lo + lane * step;
        const bool le = cand <= hi && binom_le(T, g.k, cand, j, r);
        const unsigned b = __ballot_sync(0xffffffffu, le) | 1u;
        const int top = 31 - __clz(b);
        lo += top * step;
        hi = min(hi, lo + step - 1);
      }
      // r -= binom(lo, j)
      const uint4* t = reinterpret_cast<const uint4*>(T + ((int64_t)lo * g.k + (j - 1)) * kS);
      uint64_t borrow = 0;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const uint4 v = __ldg(t + q);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int x = 0; x < 4; x++) {
          const int l = 4 * q + x;
          if (l >= kL) continue;
          const uint64_t d = (uint64_t)r[l] - w[x] - borrow;
          r[l] = (uint32_t)d;
          borrow = (d >> 63) & 1u;
        }
      }
      bad |= borrow != 0;
      if (lane == 0) spos[wib][i] = (uint16_t)lo;
      hi = lo - 1;
    }
    uint32_t rest = 0;
#pragma unroll
    for (int l = 0; l < kL; l++) rest |= r[l];
    bad |= rest != 0;
    __syncwarp();
    // pack: word w of the index stream holds the bits [32w, 32w + 32) of the slots' 12-bit fields
    uint32_t* out = rec + c * g.rec_words;
    for (int w = lane; w < g.idx_words; w += 32) {
      uint32_t word = 0;
      const int b0 = 32 * w;
      const int j0 = b0 / g.ib, j1 = min((b0 + 31) / g.ib, ke - 1);
      for (int jj = j0; jj <= j1; jj++) {
        const int sh = g.ib * jj - b0;
        const uint32_t pv = spos[wib][jj];
        word |= sh >= 0 ? (pv << sh) : (pv >> (-sh));
      }
      out[w] = word;
    }
    for (int w = lane; w < g.code_words + 1; w += 32) out[g.idx_words + w] = __ldg(e + kL + w);
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, kErrNonFinite);
}

}  // namespace

int ec_record_words(const Geom& g) { return kL + g.code_words + 1; }

cudaError_t launch_index_encode(const ChunkDesc* chunks, int64_t n_chunks, const uint32_t* rec, const uint32_t* T,
                                uint32_t* ec, const Geom& g, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((n_chunks + 7) / 8, (int64_t)sms * 8);
  index_encode_kernel<<<grid, 256, 0, s>>>(chunks, n_chunks, rec, T, ec, g);
  return cudaGetLastError();
}

cudaError_t launch_index_decode(const ChunkDesc* chunks, int64_t n_chunks, const uint32_t* ec, const uint32_t* T,
                                uint32_t* rec, uint32_t* err, const Geom& g, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((n_chunks + 7) / 8, (int64_t)sms * 8);
  index_decode_kernel<<<grid, 256, 0, s>>>(chunks, n_chunks, ec, T, rec, err, g);
  return cudaGetLastError();
}

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
