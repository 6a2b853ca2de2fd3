// compress.cu — slc_compress kernel: Eq. 1 of PAPER.md per chunk.
//
// One CTA of C/16 threads per chunk; every element lives in registers (16 per
// thread) from load to EF store, so HBM sees exactly one read of theta,
// theta_local and e and one write of e per element plus the chunk record.
//
//  1. load (128-bit, coalesced), d = theta - theta_local, b = fma(beta, e, d)   (R#12)
//     key(b) = (|b| bits) + 1 (0 marks a missing position of a partial chunk)
//  2. Top-k, exact, ties to the lower position (R#3-R#5):
//     a. lower bound T: largest T with #{threads whose max key >= T} >= k_eff,
//        found bit by bit (bits 30..16) with __syncthreads_count — at least
//        k_eff elements have key >= T;
//     b. candidates (key >= T, typically ~1.2 k_eff) compacted to smem as
//        64-bit (key << 16 | ~pos) so a larger value = larger |b|, then lower p;
//     c. exact rank of each candidate by counting; rank < k_eff -> selected
//        bit in a C-bit smem bitmap.  If the candidate set overflows (ties,
//        zero / constant chunks) a fallback finds the k_eff-th largest key by
//        bitwise block counting over all elements and resolves ties at that
//        key by position order.
//  3. warp 0: bitmap -> slots in ascending position order; 2-bit quantiser Q
//     (R#1) with the fixed-order tree sums of R#13 (xor butterfly == the
//     oracle's tree on every lane); fp16 scales (R#14); record words (R#6).
//  4. all threads: e <- b - dequant (selected) or b, 128-bit stores.
#include <cuda_fp16.h>

#include "chunk_io.cuh"
#include "quant_pack.cuh"

namespace slc {
namespace {

template <int C>
struct CompressSmem {
  static constexpr int NT = ChunkCfg<C>::NT;
  static constexpr int BW = ChunkCfg<C>::BW;
  static constexpr int MAXC = NT;
  static constexpr size_t off_cand = sizeof(float) * C;
  static constexpr size_t off_bit = off_cand + sizeof(uint64_t) * MAXC;
  static constexpr size_t off_tie = off_bit + sizeof(uint32_t) * BW;
  static constexpr size_t off_selpos = off_tie + sizeof(uint32_t) * BW;
  static constexpr size_t off_selval = off_selpos + sizeof(uint32_t) * kMaxK;
  static constexpr size_t off_code = off_selval + sizeof(float) * kMaxK;
  static constexpr size_t bytes = off_code + sizeof(uint32_t) * kMaxK;
};

template <int C, bool BF16>
__global__ void __launch_bounds__(C / 16) compress_kernel(const CompressArgs a) {
  using K = ChunkCfg<C>;
  using S = CompressSmem<C>;
  constexpr int NT = K::NT;
  constexpr int RPQ_SHIFT = (K::RPQ == 8) ? 3 : (K::RPQ == 16 ? 4 : 5);
  extern __shared__ __align__(16) unsigned char smem[];
  float* sb = reinterpret_cast<float*>(smem);
  uint64_t* scand = reinterpret_cast<uint64_t*>(smem + S::off_cand);
  uint32_t* sbit = reinterpret_cast<uint32_t*>(smem + S::off_bit);
  uint32_t* stie = reinterpret_cast<uint32_t*>(smem + S::off_tie);
  uint32_t* selpos = reinterpret_cast<uint32_t*>(smem + S::off_selpos);
  float* selval = reinterpret_cast<float*>(smem + S::off_selval);
  uint32_t* selcode = reinterpret_cast<uint32_t*>(smem + S::off_code);
  __shared__ int s_ncand;
  __shared__ float s_tau, s_flo, s_fhi;
  __shared__ int s_w[32];

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t chunk = blockIdx.x;
  const ChunkDesc d = a.chunks[chunk];
  const int len = d.len;
  const int k = a.g.k;
  const int k_eff = max(1, (k * len) / C);

  if (t == 0) s_ncand = 0;
  for (int i = t; i < K::BW; i += NT) { sbit[i] = 0u; stie[i] = 0u; }

  // ---- 1. load, pseudo-gradient, EF accumulation -------------------------
  float b[16];
  uint32_t lm = 0;
  bool bad = false;
#pragma unroll
  for (int v = 0; v < 4; v++) {
    const int q = v * NT + t;
    const int p0 = 4 * q;
    const int n = valid_in_group(p0, len);
    const int64_t off = group_offset(d, q, RPQ_SHIFT);
    float av[4], lv[4], ev[4];
    load_param4<BF16>(a.theta, off, n, av);
    load_param4<BF16>(a.theta_local, off, n, lv);
    load_f32x4(a.ef, off, n, ev);
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const float dd = __fsub_rn(av[j], lv[j]);
      const float bb = __fmaf_rn(a.beta, ev[j], dd);
      b[4 * v + j] = bb;
      const uint32_t key = (j < n) ? key_of(bb) : 0u;
      bad |= key > 0x7F800000u;
      lm = max(lm, key);
    }
    *reinterpret_cast<float4*>(sb + p0) = make_float4(b[4 * v], b[4 * v + 1], b[4 * v + 2], b[4 * v + 3]);
  }
  if (bad) atomicOr(a.err, kErrNonFinite);

  // ---- 2a. lower bound on the k_eff-th largest key ----------------------
  uint32_t T = 0;
#pragma unroll 1
  for (int bit = 30; bit >= 16; --bit) {
    const uint32_t Tp = T | (1u << bit);
    if (__syncthreads_count(lm >= Tp) >= k_eff) T = Tp;
  }
  const uint32_t Tc = max(T, 1u);

  // ---- 2b. candidate compaction ------------------------------------------
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const int p = 4 * ((i >> 2) * NT + t) + (i & 3);
    cnt += (p < len && key_of(b[i]) >= Tc);
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  int wbase = 0;
  if (lane == 31) wbase = atomicAdd(&s_ncand, incl);
  wbase = __shfl_sync(kFull, wbase, 31);
  int slot = wbase + incl - cnt;
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const int p = 4 * ((i >> 2) * NT + t) + (i & 3);
    const uint32_t key = key_of(b[i]);
    if (p < len && key >= Tc) {
      if (slot < S::MAXC) scand[slot] = ((uint64_t)key << 16) | (uint64_t)(0xFFFFu - (uint32_t)p);
      slot++;
    }
  }
  __syncthreads();
  const int M = s_ncand;

  // ---- 2c. exact selection -------------------------------------------------
  if (M <= S::MAXC) {
    if (t < M) {
      const uint64_t me = scand[t];
      int rank = 0;
#pragma unroll 4
      for (int j = 0; j < M; j++) rank += (scand[j] > me);
      if (rank < k_eff) {
        const uint32_t p = 0xFFFFu - (uint32_t)(me & 0xFFFFu);
        atomicOr(&sbit[p >> 5], 1u << (p & 31));
      }
    }
  } else {
    // fallback: K = k_eff-th largest key with multiplicity
    uint32_t Kth = 0;
#pragma unroll 1
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t Tp = Kth | (1u << bit);
      int c = 0;
#pragma unroll
      for (int i = 0; i < 16; i++) {
        const int p = 4 * ((i >> 2) * NT + t) + (i & 3);
        c += (p < len && key_of(b[i]) >= Tp);
      }
      if (block_sum<NT>(c, s_w) >= k_eff) Kth = Tp;
    }
    int gt = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) {
      const int p = 4 * ((i >> 2) * NT + t) + (i & 3);
      if (p < len) {
        const uint32_t key = key_of(b[i]);
        if (key > Kth) { atomicOr(&sbit[p >> 5], 1u << (p & 31)); gt++; }
        else if (key == Kth) atomicOr(&stie[p >> 5], 1u << (p & 31));
      }
    }
    const int need = k_eff - block_sum<NT>(gt, s_w);  // block_sum also orders the bitmap writes
    if (warp == 0) {
      constexpr int WPL = K::BW / 32;
      uint32_t w[WPL];
      int c = 0;
#pragma unroll
      for (int i = 0; i < WPL; i++) { w[i] = stie[lane * WPL + i]; c += __popc(w[i]); }
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
      }
      int before = inc - c;
#pragma unroll
      for (int i = 0; i < WPL; i++) {
        uint32_t keep = 0, x = w[i];
        while (x && before < need) {
          const uint32_t lowbit = x & (0u - x);
          keep |= lowbit;
          x ^= lowbit;
          before++;
        }
        if (keep) atomicOr(&sbit[lane * WPL + i], keep);
      }
    }
  }
  __syncthreads();

  // ---- 3. slots, quantiser, record (warp 0) --------------------------------
  if (warp == 0) {
    constexpr int WPL = K::BW / 32;
    uint32_t w[WPL];
    int c = 0;
#pragma unroll
    for (int i = 0; i < WPL; i++) { w[i] = sbit[lane * WPL + i]; c += __popc(w[i]); }
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    int s = inc - c;
#pragma unroll
    for (int i = 0; i < WPL; i++) {
      uint32_t x = w[i];
      while (x) {
        const int bitpos = __ffs(x) - 1;
        x &= x - 1;
        const int p = (lane * WPL + i) * 32 + bitpos;
        if (s < kMaxK) { selpos[s] = (uint32_t)p; selval[s] = sb[p]; }
        s++;
      }
    }
    __syncwarp();
    const QuantOut qo = warp_quantize_pack(selpos, selval, selcode, k, k_eff, a.g,
                                           a.records + chunk * a.g.rec_words, a.err, a.rec_extra, a.n_extra,
                                           chunk * a.g.rec_words);
    if (lane == 0) { s_tau = qo.tau; s_flo = qo.flo; s_fhi = qo.fhi; }
  }
  __syncthreads();

  // ---- 4. EF residual --------------------------------------------------
  const float tau = s_tau, flo = s_flo, fhi = s_fhi;
#pragma unroll
  for (int v = 0; v < 4; v++) {
    const int q = v * NT + t;
    const int p0 = 4 * q;
    const int n = valid_in_group(p0, len);
    const uint32_t bits = (sbit[p0 >> 5] >> (p0 & 31)) & 0xFu;
    float en[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const float bb = b[4 * v + j];
      float e_new = bb;
      if ((bits >> j) & 1u) {
        const float mag = fabsf(bb) > tau ? fhi : flo;
        e_new = __fsub_rn(bb, signbit(bb) ? -mag : mag);
      }
      en[j] = e_new;
    }
    store_f32x4(a.ef, group_offset(d, q, RPQ_SHIFT), n, en);
  }
}

template <int C, bool BF16>
cudaError_t launch_one(const CompressArgs& a, cudaStream_t s) {
  constexpr size_t smem = CompressSmem<C>::bytes;
  if (smem > 48 * 1024) {  // per device context; cheap, so set on every launch
    cudaError_t e = cudaFuncSetAttribute(compress_kernel<C, BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (a.n_chunks > 0x7FFFFFFFll) return cudaErrorInvalidValue;
  compress_kernel<C, BF16><<<(unsigned)a.n_chunks, ChunkCfg<C>::NT, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool compress_supported(int C) { return C == 1024 || C == 4096 || C == 16384; }

cudaError_t launch_compress(const CompressArgs& a, int bf16, cudaStream_t s) {
  if (a.n_chunks == 0) return cudaSuccess;
  switch (a.g.C) {
    case 1024:
    case 4096:
#ifdef SLC_NO_WS
      return launch_compress_warp(a, bf16, s);
#else
      return launch_compress_ws(a, bf16, s);
#endif
    case 16384: return bf16 ? launch_one<16384, true>(a, s) : launch_one<16384, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace slc
