// compress_pipe.cu — slc_compress for the paper's geometry (C = 4096, 64x64
// blocks): persistent, warp-specialised, cp.async double-buffered.
//
// CTA = 8 compute warps + 1 quantiser warp; 2 CTAs per SM (~106 KB smem each).
// CTA b walks chunks b, b+G, b+2G, ...
//
//  compute warps, chunk i (stage s = i & 1):
//   1. wait the stage's mbarrier; smem -> registers (LDS.128), d = theta -
//      theta_local, b = fma(beta, e, d) (R#12); e <- b stored densely
//      at once (selected positions are corrected by the quantiser warp);
//   2. lower bound T on the k-th largest key: the largest T with at least k of
//      the 256 thread maxima >= T (bits 30..16, one barrier.red.popc each).  After
//      the first round every thread is done with stage s, so each thread
//      issues its 12 x 16-byte cp.async of chunk i+2 into it and arrives on the
//      stage mbarrier with cp.async.mbarrier.arrive.noinc — loads are spread
//      over all 256 threads, ~96 KB in flight per SM, no registers held;
//   3. candidates key >= T (typically ~1.2 k) -> smem as key<<16 | ~pos;
//   4. exact rank by counting -> 4096-bit selection bitmap (fallback when more
//      than 256 candidates: exact k-th key by bitwise block counting, ties to
//      the lower position);
//   5. bitmap word prefix; 6. each selected value lands at its slot (ascending
//      position) in hand-off buffer i & 1 -> named-barrier arrive.
//  quantiser warp, chunk i: named-barrier sync on the hand-off buffer; 2-bit
//   quantiser + record (R#1, R#6, R#13, R#14); EF of the selected positions
//   e = b - dequant; release the buffer.  It runs concurrently with the
//   compute warps' next chunk, so its serial latency is off the critical path.
#include "chunk_io.cuh"
#include "ptx.cuh"
#include "quant_pack.cuh"

namespace slc {
namespace {

constexpr int kC = 4096;
constexpr int kNT = 256;                // compute threads
constexpr int kThreads = kNT + 32;      // + quantiser warp
constexpr int kMaxCand = 256;
enum : int { kBarCompute = 1, kBarReady0 = 2, kBarFree0 = 4 };

template <bool BF16>
struct PipeSmem {
  static constexpr int PB = BF16 ? 2 : 4;
  static constexpr size_t arr_theta = 0;
  static constexpr size_t arr_tl = (size_t)kC * PB;
  static constexpr size_t arr_e = 2 * (size_t)kC * PB;
  static constexpr size_t stage_bytes = (size_t)kC * (2 * PB + 4);
  static constexpr size_t off_cand = 2 * stage_bytes;                 // u64[256]
  static constexpr size_t off_candb = off_cand + 8 * kMaxCand;         // f32[256]
  static constexpr size_t off_bit = off_candb + 4 * kMaxCand;          // u32[128]
  static constexpr size_t off_tie = off_bit + 4 * (kC / 32);           // u32[128]
  static constexpr size_t off_wpre = off_tie + 4 * (kC / 32);          // u32[128]
  static constexpr size_t off_selpos = off_wpre + 4 * (kC / 32);       // u32[2][kMaxK]
  static constexpr size_t off_selval = off_selpos + 8 * kMaxK;         // f32[2][kMaxK]
  static constexpr size_t off_code = off_selval + 8 * kMaxK;           // u32[kMaxK]
  static constexpr size_t off_bar = off_code + 4 * kMaxK;              // u64[2]
  static constexpr size_t bytes = off_bar + 16;
};

// all 256 compute threads: cp.async chunk c into `stage`, then arrive on `bar`
template <bool BF16>
__device__ __forceinline__ void prefetch_chunk(const CompressArgs& a, int64_t c, unsigned char* stage, uint64_t* bar,
                                               int t) {
  using S = PipeSmem<BF16>;
  const ChunkDesc d = a.chunks[c];
  if (d.len == kC) {
    const unsigned char* th = static_cast<const unsigned char*>(a.theta);
    const unsigned char* tl = static_cast<const unsigned char*>(a.theta_local);
    const unsigned char* ef = reinterpret_cast<const unsigned char*>(a.ef);
    // fp32 pieces: positions 4(t + 256u), u = 0..3 — the consumer's groups
    const int64_t g0 = group_offset(d, t, 4);
    const int64_t gs = d.ld ? 16 * (int64_t)d.ld : 4 * kNT;
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int p = 4 * (u * kNT + t);
      const int64_t g = g0 + u * gs;
      ptx::cp_async16(stage + S::arr_e + (size_t)p * 4, ef + g * 4);
      if (!BF16) {
        ptx::cp_async16(stage + S::arr_theta + (size_t)p * 4, th + g * 4);
        ptx::cp_async16(stage + S::arr_tl + (size_t)p * 4, tl + g * 4);
      }
    }
    if (BF16) {  // bf16 pieces of 8 elements: positions 8(t + 256u), u = 0..1
      const int64_t h0 = d.ld ? d.base + (int64_t)(t >> 3) * d.ld + 8 * (t & 7) : d.base + 8 * t;
      const int64_t hs = d.ld ? 32 * (int64_t)d.ld : 8 * kNT;
#pragma unroll
      for (int u = 0; u < 2; u++) {
        const int p = 8 * (u * kNT + t);
        const int64_t g = h0 + u * hs;
        ptx::cp_async16(stage + S::arr_theta + (size_t)p * 2, th + g * 2);
        ptx::cp_async16(stage + S::arr_tl + (size_t)p * 2, tl + g * 2);
      }
    }
  }
  ptx::cp_async_arrive_noinc(bar);  // partial chunk: consumers read global memory directly
}

template <bool BF16, int KC, int IBC>
__global__ void __launch_bounds__(kThreads, 2) compress_pipe_kernel(const CompressArgs a) {
  using S = PipeSmem<BF16>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* scand = reinterpret_cast<uint64_t*>(smem + S::off_cand);
  float* candb = reinterpret_cast<float*>(smem + S::off_candb);
  uint32_t* sbit = reinterpret_cast<uint32_t*>(smem + S::off_bit);
  uint32_t* stie = reinterpret_cast<uint32_t*>(smem + S::off_tie);
  uint32_t* wpre = reinterpret_cast<uint32_t*>(smem + S::off_wpre);
  uint32_t* selpos = reinterpret_cast<uint32_t*>(smem + S::off_selpos);
  float* selval = reinterpret_cast<float*>(smem + S::off_selval);
  uint32_t* selcode = reinterpret_cast<uint32_t*>(smem + S::off_code);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::off_bar);
  __shared__ int s_ncand;
  __shared__ uint32_t s_T;
  __shared__ int s_w[kNT / 32];
  __shared__ __align__(16) uint32_t slm[kNT];

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t G = gridDim.x, n = a.n_chunks;
  const int k = KC ? KC : a.g.k;

  if (t == 0) {
    ptx::mbar_init(&bars[0], kNT);
    ptx::mbar_init(&bars[1], kNT);
    ptx::fence_mbar_init();
  }
  if (t < kC / 32) { sbit[t] = 0u; stie[t] = 0u; }
  if (t == 0) s_ncand = 0;
  __syncthreads();

  if (warp == kNT / 32) {
    // ======================= quantiser warp =======================
    ptx::named_arrive<kBarFree0>(kThreads);
    ptx::named_arrive<kBarFree0 + 1>(kThreads);
    for (int64_t i = 0;; ++i) {
      const int64_t c = (int64_t)blockIdx.x + i * G;
      if (c >= n) break;
      const int buf = (int)(i & 1);
      const ChunkDesc d = a.chunks[c];
      const int k_eff = d.len == kC ? k : max(1, (k * d.len) / kC);
      if (buf) ptx::named_sync<kBarReady0 + 1>(kThreads);
      else ptx::named_sync<kBarReady0>(kThreads);
      const uint32_t* sp = selpos + buf * kMaxK;
      const float* sv = selval + buf * kMaxK;
      const QuantOut qo =
          warp_quantize_pack<KC, IBC>(sp, sv, selcode, k, k_eff, a.g, a.records + c * a.g.rec_words, a.err);
      for (int j = lane; j < k_eff; j += 32) {
        const int p = (int)sp[j];
        const float bb = sv[j];
        const float mag = fabsf(bb) > qo.tau ? qo.fhi : qo.flo;
        const int64_t addr = d.ld ? d.base + (int64_t)(p >> 6) * d.ld + (p & 63) : d.base + p;
        a.ef[addr] = __fsub_rn(bb, signbit(bb) ? -mag : mag);
      }
      __syncwarp();
      if (c + 2 * G < n) {
        if (buf) ptx::named_arrive<kBarFree0 + 1>(kThreads);
        else ptx::named_arrive<kBarFree0>(kThreads);
      }
    }
    return;
  }

  // ======================= compute warps =======================
  if ((int64_t)blockIdx.x < n) prefetch_chunk<BF16>(a, blockIdx.x, smem, &bars[0], t);
  if ((int64_t)blockIdx.x + G < n) prefetch_chunk<BF16>(a, blockIdx.x + G, smem + S::stage_bytes, &bars[1], t);

  for (int64_t i = 0;; ++i) {
    const int64_t c = (int64_t)blockIdx.x + i * G;
    if (c >= n) break;
    const int s = (int)(i & 1);
    const uint32_t par = (uint32_t)((i >> 1) & 1);
    unsigned char* stage = smem + s * S::stage_bytes;
    const ChunkDesc d = a.chunks[c];
    const int len = d.len;
    const bool full = len == kC;
    const int k_eff = full ? k : max(1, (k * len) / kC);

    // ---- 1. inputs -> b; dense e <- b -------------------------------------------
    // key2(b) = |b| bits << 1 | 1: order-preserving on |b|, 0 marks a missing position
    ptx::mbar_wait(&bars[s], par);
    float b[16];
    uint32_t lm = 0;
    if (full) {
      const int64_t off0 = group_offset(d, t, 4);
      const int64_t vstride = d.ld ? 16 * (int64_t)d.ld : 4 * kNT;  // element step between groups v
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int p0 = 4 * (v * kNT + t);
        float av[4], lv[4];
        if (BF16) {
          const uint2 ua = *reinterpret_cast<const uint2*>(stage + S::arr_theta + 2 * p0);
          const uint2 ul = *reinterpret_cast<const uint2*>(stage + S::arr_tl + 2 * p0);
          av[0] = bf16_bits_to_f32(ua.x & 0xFFFFu); av[1] = bf16_bits_to_f32(ua.x >> 16);
          av[2] = bf16_bits_to_f32(ua.y & 0xFFFFu); av[3] = bf16_bits_to_f32(ua.y >> 16);
          lv[0] = bf16_bits_to_f32(ul.x & 0xFFFFu); lv[1] = bf16_bits_to_f32(ul.x >> 16);
          lv[2] = bf16_bits_to_f32(ul.y & 0xFFFFu); lv[3] = bf16_bits_to_f32(ul.y >> 16);
        } else {
          const float4 fa = *reinterpret_cast<const float4*>(stage + S::arr_theta + 4 * p0);
          const float4 fl = *reinterpret_cast<const float4*>(stage + S::arr_tl + 4 * p0);
          av[0] = fa.x; av[1] = fa.y; av[2] = fa.z; av[3] = fa.w;
          lv[0] = fl.x; lv[1] = fl.y; lv[2] = fl.z; lv[3] = fl.w;
        }
        const float4 fe = *reinterpret_cast<const float4*>(stage + S::arr_e + 4 * p0);
        const float ev[4] = {fe.x, fe.y, fe.z, fe.w};
#pragma unroll
        for (int j = 0; j < 4; j++) b[4 * v + j] = __fmaf_rn(a.beta, ev[j], __fsub_rn(av[j], lv[j]));
        *reinterpret_cast<float4*>(a.ef + off0 + v * vstride) =
            make_float4(b[4 * v], b[4 * v + 1], b[4 * v + 2], b[4 * v + 3]);
      }
#pragma unroll
      for (int j = 0; j < 16; j += 2) lm = max(lm, max(key2_of(b[j]), key2_of(b[j + 1])));
    } else {
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int q = v * kNT + t;
        const int p0 = 4 * q;
        const int64_t off = group_offset(d, q, 4);
        const int nv = valid_in_group(p0, len);
        float av[4], lv[4], ev[4];
        load_param4<BF16>(a.theta, off, nv, av);
        load_param4<BF16>(a.theta_local, off, nv, lv);
        load_f32x4(a.ef, off, nv, ev);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          b[4 * v + j] = __fmaf_rn(a.beta, ev[j], __fsub_rn(av[j], lv[j]));
          if (j < nv) lm = max(lm, key2_of(b[4 * v + j]));
        }
        store_f32x4(a.ef, off, nv, &b[4 * v]);
      }
    }
    if (lm >= 0xFF000001u) atomicOr(a.err, kErrNonFinite);  // |b| = inf or NaN (max key wins)
    slm[t] = lm;

    // ---- 2. lower bound T from the thread maxima; refill the stage ---------------
    ptx::named_sync<kBarCompute>(kNT);  // every thread is done with stage s
    if (c + 2 * G < n) prefetch_chunk<BF16>(a, c + 2 * G, stage, &bars[s], t);
    if (t >= kNT - kC / 32) { sbit[t - (kNT - kC / 32)] = 0u; stie[t - (kNT - kC / 32)] = 0u; }
    if (t == 32) s_ncand = 0;
    if (warp == 0) {
      // largest T (bits 31..17) with >= k_eff of the 256 thread maxima >= T
      const uint4 m0 = *reinterpret_cast<const uint4*>(slm + 8 * lane);
      const uint4 m1 = *reinterpret_cast<const uint4*>(slm + 8 * lane + 4);
      uint32_t T = 0;
#pragma unroll
      for (int bit = 31; bit >= 17; --bit) {
        const uint32_t Tp = T | (1u << bit);
        const int c8 = (m0.x >= Tp) + (m0.y >= Tp) + (m0.z >= Tp) + (m0.w >= Tp) + (m1.x >= Tp) + (m1.y >= Tp) +
                       (m1.z >= Tp) + (m1.w >= Tp);
        if (__reduce_add_sync(kFull, c8) >= k_eff) T = Tp;
      }
      if (lane == 0) s_T = T;
    }
    ptx::named_sync<kBarCompute>(kNT);
    const uint32_t Tc = max(s_T, 1u);

    // ---- 3. candidates -----------------------------------------------------------------
    uint32_t mask = 0;
#pragma unroll
    for (int j = 0; j < 16; j++) mask |= (uint32_t)(key2_of(b[j]) >= Tc) << j;
    if (!full) {  // missing positions of a partial chunk are never candidates
#pragma unroll
      for (int j = 0; j < 16; j++)
        if (4 * ((j >> 2) * kNT + t) + (j & 3) >= len) mask &= ~(1u << j);
    }
    const int cnt = __popc(mask);
    const int incl = warp_excl_scan(cnt) + cnt;
    int wbase = 0;
    if (lane == 31) wbase = atomicAdd(&s_ncand, incl);
    wbase = __shfl_sync(kFull, wbase, 31);
    int slot = wbase + incl - cnt;
#pragma unroll
    for (int j = 0; j < 16; j++) {
      if (__ballot_sync(kFull, (mask >> j) & 1u)) {  // warp-uniform skip: candidates are sparse
        if ((mask >> j) & 1u) {
          const int p = 4 * ((j >> 2) * kNT + t) + (j & 3);
          if (slot < kMaxCand) {
            scand[slot] = ((uint64_t)key2_of(b[j]) << 16) | (uint64_t)(0xFFFFu - (uint32_t)p);
            candb[slot] = b[j];
          }
          slot++;
        }
      }
    }
    ptx::named_sync<kBarCompute>(kNT);
    const int M = s_ncand;

    // ---- 4. exact selection -> bitmap --------------------------------------------------
    int my_p = -1;
    float my_b = 0.0f;
    if (M <= kMaxCand) {
      if (t < M) {
        const uint64_t me = scand[t];
        int rank = 0;
#pragma unroll 8
        for (int j = 0; j < M; j++) rank += (scand[j] > me);
        if (rank < k_eff) {
          my_p = (int)(0xFFFFu - (uint32_t)(me & 0xFFFFu));
          my_b = candb[t];
          atomicOr(&sbit[my_p >> 5], 1u << (my_p & 31));
        }
      }
    } else {
      uint32_t Kth = 0;
#pragma unroll 1
      for (int bit = 31; bit >= 0; --bit) {
        const uint32_t Tp = Kth | (1u << bit);
        int cc = 0;
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const int p = 4 * ((j >> 2) * kNT + t) + (j & 3);
          cc += (p < len && key2_of(b[j]) >= Tp);
        }
        if (block_sum_named<kNT, kBarCompute>(cc, s_w) >= k_eff) Kth = Tp;
      }
      int gt = 0;
#pragma unroll
      for (int j = 0; j < 16; j++) {
        const int p = 4 * ((j >> 2) * kNT + t) + (j & 3);
        if (p < len) {
          const uint32_t key = key2_of(b[j]);
          if (key > Kth) { atomicOr(&sbit[p >> 5], 1u << (p & 31)); gt++; }
          else if (key == Kth) atomicOr(&stie[p >> 5], 1u << (p & 31));
        }
      }
      const int need = k_eff - block_sum_named<kNT, kBarCompute>(gt, s_w);
      if (warp == 0) {
        uint32_t w[4];
        int cw = 0;
#pragma unroll
        for (int x = 0; x < 4; x++) { w[x] = stie[4 * lane + x]; cw += __popc(w[x]); }
        int before = warp_excl_scan(cw);
#pragma unroll
        for (int x = 0; x < 4; x++) {
          uint32_t keep = 0, y = w[x];
          while (y && before < need) {
            const uint32_t lowbit = y & (0u - y);
            keep |= lowbit;
            y ^= lowbit;
            before++;
          }
          if (keep) atomicOr(&sbit[4 * lane + x], keep);
        }
      }
    }
    ptx::named_sync<kBarCompute>(kNT);

    // ---- 5. bitmap word prefix -----------------------------------------------------------
    if (warp == 0) {
      uint32_t w[4];
      int cw = 0;
#pragma unroll
      for (int x = 0; x < 4; x++) { w[x] = sbit[4 * lane + x]; cw += __popc(w[x]); }
      int pre = warp_excl_scan(cw);
#pragma unroll
      for (int x = 0; x < 4; x++) { wpre[4 * lane + x] = (uint32_t)pre; pre += __popc(w[x]); }
    }
    // hand-off buffer i & 1 must have been released by the quantiser (chunk i-2)
    const int buf = (int)(i & 1);
    if (buf) ptx::named_sync<kBarFree0 + 1>(kThreads);
    else ptx::named_sync<kBarFree0>(kThreads);
    ptx::named_sync<kBarCompute>(kNT);

    // ---- 6. selected values to their slots, hand off --------------------------------------
    uint32_t* sp = selpos + buf * kMaxK;
    float* sv = selval + buf * kMaxK;
    if (M <= kMaxCand) {
      if (my_p >= 0) {
        const int sl = (int)wpre[my_p >> 5] + __popc(sbit[my_p >> 5] & ((1u << (my_p & 31)) - 1u));
        sp[sl] = (uint32_t)my_p;
        sv[sl] = my_b;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; j++) {
        const int p = 4 * ((j >> 2) * kNT + t) + (j & 3);
        if (p < len && ((sbit[p >> 5] >> (p & 31)) & 1u)) {
          const int sl = (int)wpre[p >> 5] + __popc(sbit[p >> 5] & ((1u << (p & 31)) - 1u));
          sp[sl] = (uint32_t)p;
          sv[sl] = b[j];
        }
      }
    }
    __threadfence_block();  // slots + the dense e stores of step 1 before the quantiser's fix-ups
    if (buf) ptx::named_arrive<kBarReady0 + 1>(kThreads);
    else ptx::named_arrive<kBarReady0>(kThreads);
  }
}

template <bool BF16, int KC, int IBC>
cudaError_t launch_pipe_t(const CompressArgs& a, cudaStream_t s) {
  constexpr size_t smem = PipeSmem<BF16>::bytes;
  auto kern = compress_pipe_kernel<BF16, KC, IBC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > a.n_chunks) grid = a.n_chunks;
  kern<<<(unsigned)grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <bool BF16>
cudaError_t launch_pipe(const CompressArgs& a, cudaStream_t s) {
  if (a.g.k == 64 && a.g.ib == 12) return launch_pipe_t<BF16, 64, 12>(a, s);  // the paper's geometry
  return launch_pipe_t<BF16, 0, 0>(a, s);
}

}  // namespace

cudaError_t launch_compress_pipe(const CompressArgs& a, int bf16, cudaStream_t s) {
  if (a.n_chunks == 0) return cudaSuccess;
  if (a.g.C != kC) return cudaErrorInvalidValue;
  return bf16 ? launch_pipe<true>(a, s) : launch_pipe<false>(a, s);
}

}  // namespace slc
