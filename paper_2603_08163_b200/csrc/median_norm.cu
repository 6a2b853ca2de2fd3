// median_norm.cu — median-norm normalisation of the peers' contributions
// (§2.2: "Pseudo-gradient contributions are scaled relative to
// their median norm so that no single participant can dominate"; reading R#20:
// every nonzero contribution rescaled to the lower-median norm).
//
// Step 1, slc_payload_sqnorm: ||hatDelta_r||^2 over this shard's chunks, from
// the records alone.  A record's values are k_eff signed fp16 scales, n_lo of
// them S_lo and n_hi = popc(bucket bits) of them S_hi, so the chunk adds
// n_lo*F_lo^2 + n_hi*F_hi^2 in units of 2^-48 (F = scale as an integer
// multiple of 2^-24, F < 2^40).  The sum is EXACT in unsigned 128-bit integer
// arithmetic (< 2^111 for any shard), hence independent of summation order,
// of the grid and of the sharding.  Each warp's 128-bit partial is split into
// four 32-bit limbs added to four 64-bit counters per peer (un-carried limb
// sums; they stay exact when summed again across ranks, e.g. by an int64 NCCL
// all-reduce).
//
// Step 2, slc_median_norm_weights (one CTA): limbs -> exact 128-bit sum ->
// correctly rounded binary64 -> * 2^-48 -> sqrt (IEEE) = ||hatDelta_r||; lower
// median m; w_r = (float)(m / n_r) for n_r > 0, else 1.  Weights stay on the
// device and feed the weighted fused update (slc_outer_update_wdev).
#include <algorithm>

#include "slc_internal.cuh"

namespace slc {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ unsigned long long f16_fixed24u(uint32_t h) {
  const uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
  return e == 0 ? (unsigned long long)m : (unsigned long long)(1024u + m) << (e - 1);
}

__device__ __forceinline__ u128 shfl_down_u128(u128 v, int d) {
  const unsigned long long lo = __shfl_down_sync(0xFFFFFFFFu, (unsigned long long)v, d);
  const unsigned long long hi = __shfl_down_sync(0xFFFFFFFFu, (unsigned long long)(v >> 64), d);
  return ((u128)hi << 64) | lo;
}

// grid (x, R): peer r = blockIdx.y; threads stride over the shard's chunks
__global__ void __launch_bounds__(256) payload_sqnorm_kernel(const AggArgs a, unsigned long long* out) {
  const int r = blockIdx.y;
  const uint32_t* recs = a.rec[r];
  const int RW = a.g.rec_words, IW = a.g.idx_words, CW = a.g.code_words;
  const int C = a.g.C;
  u128 acc = 0;
  bool bad = false;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < a.n_chunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int len = __ldg(&a.chunks[c].len);
    const int k_eff = max(1, (a.g.k * len) / C);
    const uint32_t* rec = recs + c * RW;
    int n_hi = 0;
    for (int w = 0; w < CW; w++) n_hi += __popc(__ldg(rec + IW + w) & 0xAAAAAAAAu);  // bucket bits (2j+1)
    const uint32_t sw = __ldg(rec + RW - 1);
    const uint32_t h0 = sw & 0xFFFFu, h1 = sw >> 16;
    bad |= ((h0 >> 10) & 0x1Fu) == 0x1Fu || ((h1 >> 10) & 0x1Fu) == 0x1Fu || n_hi > k_eff;
    const unsigned long long f0 = f16_fixed24u(h0), f1 = f16_fixed24u(h1);
    acc += (u128)(unsigned)(k_eff - n_hi) * ((u128)f0 * f0) + (u128)(unsigned)n_hi * ((u128)f1 * f1);
  }
  for (int d = 16; d > 0; d >>= 1) acc += shfl_down_u128(acc, d);
  if ((threadIdx.x & 31) == 0 && acc != 0) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const unsigned long long limb = (unsigned long long)(uint32_t)(acc >> (32 * i));
      if (limb) atomicAdd(out + 4 * r + i, limb);
    }
  }
  if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.err, kErrNonFinite);
}

// correctly rounded u128 -> binary64
__device__ __forceinline__ double u128_to_double_rn(u128 v) {
  const unsigned long long hi = (unsigned long long)(v >> 64);
  if (hi == 0) return __ull2double_rn((unsigned long long)v);
  const int L = 128 - __clzll(hi);  // bit length, > 64
  const int s = L - 64;
  unsigned long long top = (unsigned long long)(v >> s);
  const u128 rest = v & (((u128)1 << s) - 1);
  if (rest != 0) top |= 1ull;  // sticky below the rounding position
  return __dmul_rn(__ull2double_rn(top), __longlong_as_double((long long)(1023 + s) << 52));  // exact scaling
}

__global__ void __launch_bounds__(kMaxPeers) median_weights_kernel(const unsigned long long* limbs, int R,
                                                                   float* w, double* norms_out) {
  __shared__ double nrm[kMaxPeers];
  __shared__ double med;
  const int r = threadIdx.x;
  double x = 0.0;
  if (r < R) {
    u128 v = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) v += (u128)limbs[4 * r + i] << (32 * i);
    // sum * 2^-48 is exact in binary64 (power-of-two scaling, no underflow for nonzero sums)
    x = __dsqrt_rn(__dmul_rn(u128_to_double_rn(v), 0x1p-48));
    nrm[r] = x;
  }
  __syncthreads();
  if (r < R) {
    int rank = 0;  // position in (value, index) order; the lower median has rank (R-1)/2
    for (int i = 0; i < R; i++) rank += (nrm[i] < x) || (nrm[i] == x && i < r);
    if (rank == (R - 1) / 2) med = x;
  }
  __syncthreads();
  if (r < R) {
    w[r] = x > 0.0 ? __double2float_rn(__ddiv_rn(med, x)) : 1.0f;
    if (norms_out) norms_out[r] = x;
  }
}

// fast checks: per peer, flags |= finite (a decoded value is
// non-finite: a used bucket's scale is Inf / NaN) and norm-sane (the payload
// norm, from the rank-summed limbs, exceeds `thresh` = 10 x the lower median of
// the norm history); host-side flags (liveness, sync) come in `hflags`.
struct FastCheckArgs {
  uint32_t hflags[kMaxPeers];
  double thresh;             // +inf: no norm check
  const unsigned long long* limbs;  // NULL: no norm check
};

__global__ void __launch_bounds__(256) fast_checks_kernel(const AggArgs a, const FastCheckArgs f, uint32_t* flags) {
  const int r = blockIdx.y;
  if (f.hflags[r] & SLC_CHECK_LIVENESS) {  // no submission: nothing to scan
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags + r, f.hflags[r]);
    return;
  }
  const uint32_t* recs = a.rec[r];
  const int RW = a.g.rec_words, IW = a.g.idx_words, CW = a.g.code_words;
  bool nonfin = false;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < a.n_chunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int len = __ldg(&a.chunks[c].len);
    const int k_eff = max(1, (a.g.k * len) / a.g.C);
    const uint32_t* rec = recs + c * RW;
    int n_hi = 0;
    for (int w = 0; w < CW; w++) n_hi += __popc(__ldg(rec + IW + w) & 0xAAAAAAAAu);
    const uint32_t sw = __ldg(rec + RW - 1);
    const bool lo_bad = ((sw >> 10) & 0x1Fu) == 0x1Fu, hi_bad = ((sw >> 26) & 0x1Fu) == 0x1Fu;
    nonfin |= (lo_bad && n_hi < k_eff) || (hi_bad && n_hi > 0);
  }
  uint32_t fl = __any_sync(0xFFFFFFFFu, nonfin) ? SLC_CHECK_FINITE : 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) fl |= f.hflags[r];
  if ((threadIdx.x & 31) == 0 && fl) atomicOr(flags + r, fl);
}

// second launch, one thread per peer: the norm of every finite, present payload
__global__ void fast_norm_kernel(const FastCheckArgs f, int R, uint32_t* flags) {
  const int r = threadIdx.x;
  if (r >= R || !f.limbs || (flags[r] & (SLC_CHECK_LIVENESS | SLC_CHECK_FINITE))) return;
  u128 v = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) v += (u128)f.limbs[4 * r + i] << (32 * i);
  const double x = __dsqrt_rn(__dmul_rn(u128_to_double_rn(v), 0x1p-48));
  if (x > f.thresh) flags[r] |= SLC_CHECK_NORM;
}

}  // namespace

cudaError_t launch_fast_checks(const AggArgs& a, const uint32_t* hflags, double thresh,
                               const unsigned long long* limbs, uint32_t* flags, cudaStream_t s) {
  FastCheckArgs f;
  for (int r = 0; r < kMaxPeers; r++) f.hflags[r] = r < a.R ? hflags[r] : 0u;
  f.thresh = thresh;
  f.limbs = limbs;
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(uint32_t) * a.R, s);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  const int64_t want = std::max<int64_t>(1, (a.n_chunks + 255) / 256);
  const int gx = (int)std::min<int64_t>(want, std::max<int64_t>(1, (int64_t)4 * sms / a.R + 1));
  fast_checks_kernel<<<dim3(gx, a.R), 256, 0, s>>>(a, f, flags);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (limbs) fast_norm_kernel<<<1, kMaxPeers, 0, s>>>(f, a.R, flags);
  return cudaGetLastError();
}

cudaError_t launch_payload_sqnorm(const AggArgs& a, unsigned long long* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long) * 4 * a.R, s);
  if (e != cudaSuccess || a.n_chunks == 0) return e;
  int dev = 0, sms = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  const int64_t want = (a.n_chunks + 255) / 256;
  const int gx = (int)std::min<int64_t>(want, std::max<int64_t>(1, (int64_t)4 * sms / a.R + 1));
  payload_sqnorm_kernel<<<dim3(gx, a.R), 256, 0, s>>>(a, out);
  return cudaGetLastError();
}

cudaError_t launch_median_weights(const unsigned long long* limbs, int R, float* w, double* norms,
                                  cudaStream_t s) {
  median_weights_kernel<<<1, kMaxPeers, 0, s>>>(limbs, R, w, norms);
  return cudaGetLastError();
}

}  // namespace slc
