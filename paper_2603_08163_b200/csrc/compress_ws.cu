// compress_ws.cu — slc_compress with warp-specialised CTAs (Eq. 1 of PAPER.md,
// P:68-75; chunk Top-k P:88; C, k P:176).
//
// One persistent CTA per SM, two kinds of warps:
//   NSW stream warps   read theta / theta_local / e through a per-warp cp.async
//                      ring (D passes of 512 positions in flight), compute
//                      b = fma(beta, e, theta - theta_local) (R#12), store e <- b
//                      at once (L2 evict_last) and hand the chunk's 32*NP group
//                      maxima to the selectors through a shared-memory slot.
//   NSEL select warps  take a slot and run S / B / R / Q / F of warp_select.cuh
//                      (candidate groups re-read from L2, rank, quantise, pack,
//                      EF fix-ups).
// The stream warps keep a fixed number of bytes in flight whatever the
// selectors are doing, and the selectors' latency-bound work (L2 round trips,
// warp reductions) overlaps the stream instead of alternating with it.
//
// Hand-off: NS slots, each with a `full` and an `empty` mbarrier (32 arrivals:
// every lane of the producing / consuming warp).  Chunk j of the CTA (global
// chunk blockIdx.x + j*gridDim.x) goes through slot j % NS; stream warp j % NSW
// produces it, select warp j % NSEL consumes it.  A producer only waits for its
// slot to be empty right before writing the maxima, after the whole stream of
// the chunk.  The release/acquire mbarrier pair also orders the producer's
// global e stores before the selector's re-reads (same CTA).
#include <type_traits>

#include "ptx.cuh"
#include "warp_select.cuh"

namespace slc {
namespace {

using namespace wsel;

#ifndef SLC_WS_NSW
#define SLC_WS_NSW 4
#endif
#ifndef SLC_WS_NSEL
#define SLC_WS_NSEL 12
#endif
#ifndef SLC_WS_D
#define SLC_WS_D 3
#endif
#ifndef SLC_WS_CAPG
#define SLC_WS_CAPG 256  // candidate capacity of the any-geometry instantiation (k != 64)
#endif
#ifndef SLC_WS_CAP64
#define SLC_WS_CAP64 128  // candidate capacity of the paper's geometry (C 4096, k 64)
#endif
#ifndef SLC_WS_XS
#define SLC_WS_XS 0  // hand-off slots beyond one per warp
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

template <bool BF16>
struct PassBuf {
  static constexpr int PB = BF16 ? 2 : 4;
  static constexpr int off_tl = 512 * PB;
  static constexpr int off_e = 1024 * PB;
  static constexpr int bytes = 512 * (2 * PB + 4);
};

// hand-off slot: one maximum key per unit and lane; 16-position groups keep
// the full key, quads (VPU = 1, 4x as many) its upper 16 bits (T stays a
// lower bound: a truncated maximum never exceeds the true one)
template <int C, int VPU>
struct SlotCfg {
  using T = typename std::conditional<VPU == 1, uint16_t, uint32_t>::type;
  static constexpr int words = 32 * UnitCfg<C, VPU>::NU;
};

template <int C, bool BF16, int CAP, int KMAX, int VPU, int NSW, int NSEL, int D, int NS>
struct WsSmem {
  uint64_t full[NS];
  uint64_t empty[NS];
  typename SlotCfg<C, VPU>::T gk[NS][SlotCfg<C, VPU>::words];
  unsigned char ring[NSW][D][PassBuf<BF16>::bytes];
  WarpScratch<C, CAP, KMAX, VPU> scratch[NSEL];
};

// Per-lane addressing of a FULL chunk: group q = 128u + 32v + lane sits at
// element lb + (4u + v) * sv (blocked: 32 groups = 32/RPQ rows; flat: 128
// elements).  Lane pointers are formed once per chunk; in-chunk byte offsets
// are 32-bit (launch_ws_t requires 248 * max_ld < 2^32).
template <int C, bool BF16>
struct LaneAddr {
  static constexpr int PB = BF16 ? 2 : 4;
  const char* th;
  const char* tl;
  char* e;
  uint32_t sv;  // elements per step of (4u + v)
  __device__ __forceinline__ void init(const CompressArgs& a, const ChunkDesc& d, int lane) {
    constexpr int RS = WarpCfg<C>::RPQ_SHIFT;
    int64_t lb;
    if (d.ld) {
      lb = d.base + (int64_t)(lane >> RS) * d.ld + 4 * (lane & ((1 << RS) - 1));
      sv = (uint32_t)(32 >> RS) * (uint32_t)d.ld;
    } else {
      lb = d.base + 4 * lane;
      sv = 128;
    }
    th = static_cast<const char*>(a.theta) + lb * PB;
    tl = static_cast<const char*>(a.theta_local) + lb * PB;
    e = reinterpret_cast<char*>(a.ef) + lb * 4;
  }
  __device__ __forceinline__ uint32_t step(int u, int v) const { return (uint32_t)(4 * u + v) * sv; }
};

// issue pass u of chunk d (this lane's 4 groups of theta, theta_local, e)
template <int C, bool BF16>
__device__ __forceinline__ void issue_pass(const CompressArgs& a, const ChunkDesc& d, const LaneAddr<C, BF16>& la, int u,
                                           unsigned char* buf, int lane) {
  using PBuf = PassBuf<BF16>;
  constexpr int PB = PBuf::PB;
  const char* th = static_cast<const char*>(a.theta);
  const char* tl = static_cast<const char*>(a.theta_local);
  if (d.len == C) {
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const uint32_t st = la.step(u, v);
      const int slot = v * 32 + lane;
      cp_async_n(buf + slot * 4 * PB, la.th + st * PB, 4 * PB, 4 * PB);
      cp_async_n(buf + PBuf::off_tl + slot * 4 * PB, la.tl + st * PB, 4 * PB, 4 * PB);
      cp_async_n(buf + PBuf::off_e + slot * 16, la.e + st * 4, 16, 16);
    }
    return;
  }
#pragma unroll
  for (int v = 0; v < 4; v++) {
    const int q = 128 * u + 32 * v + lane;
    const int nv = valid_in_group(4 * q, d.len);
    if (nv == 0) continue;
    const int64_t off = goff<WarpCfg<C>::RPQ_SHIFT>(d, q);
    const int slot = v * 32 + lane;
    cp_async_n(buf + slot * 4 * PB, th + off * PB, 4 * PB, nv * PB);
    cp_async_n(buf + PBuf::off_tl + slot * 4 * PB, tl + off * PB, 4 * PB, nv * PB);
    cp_async_n(buf + PBuf::off_e + slot * 16, a.ef + off, 16, nv * 4);
  }
}

// b of this lane's 4 groups of the pass in buf; returns max |b| (NaN-propagating)
// over the valid positions, stores e <- b
// (qdst: quad hand-off — qdst[32 * (4u + v)] = 1 + the upper 16 bits of the
// quad's maximum key (saturating), 0 for a quad with no valid position)
template <bool BF16, bool FULL, int RPQ_SHIFT, class Addr>
__device__ __forceinline__ float consume_pass(const unsigned char* buf, float beta, float* ef, const Addr& la,
                                              const ChunkDesc& d, int u, int lane, uint64_t pol, int& nvalid,
                                              uint16_t* qdst = nullptr) {
  using PBuf = PassBuf<BF16>;
  float gm = 0.0f;
#pragma unroll
  for (int v = 0; v < 4; v++) {
    const int q = 128 * u + 32 * v + lane;
    const int nv = FULL ? 4 : valid_in_group(4 * q, d.len);
    const int sl = v * 32 + lane;
    float av[4], lv[4];
    if (BF16) {
      const uint2 ua = *reinterpret_cast<const uint2*>(buf + sl * 8);
      const uint2 ul = *reinterpret_cast<const uint2*>(buf + PBuf::off_tl + sl * 8);
      av[0] = bf16_bits_to_f32(ua.x & 0xFFFFu); av[1] = bf16_bits_to_f32(ua.x >> 16);
      av[2] = bf16_bits_to_f32(ua.y & 0xFFFFu); av[3] = bf16_bits_to_f32(ua.y >> 16);
      lv[0] = bf16_bits_to_f32(ul.x & 0xFFFFu); lv[1] = bf16_bits_to_f32(ul.x >> 16);
      lv[2] = bf16_bits_to_f32(ul.y & 0xFFFFu); lv[3] = bf16_bits_to_f32(ul.y >> 16);
    } else {
      const float4 fa = *reinterpret_cast<const float4*>(buf + sl * 16);
      const float4 fl = *reinterpret_cast<const float4*>(buf + PBuf::off_tl + sl * 16);
      av[0] = fa.x; av[1] = fa.y; av[2] = fa.z; av[3] = fa.w;
      lv[0] = fl.x; lv[1] = fl.y; lv[2] = fl.z; lv[3] = fl.w;
    }
    const float4 fe = *reinterpret_cast<const float4*>(buf + PBuf::off_e + sl * 16);
    const float ev[4] = {fe.x, fe.y, fe.z, fe.w};
    float b[4];
    float qm = 0.0f;
#pragma unroll
    for (int jj = 0; jj < 4; jj++) {
      b[jj] = __fmaf_rn(beta, ev[jj], __fsub_rn(av[jj], lv[jj]));
      if (FULL || jj < nv) qm = absmax_nan(qm, b[jj]);  // missing positions excluded
    }
    gm = absmax_nan(gm, qm);
    if (qdst) qdst[32 * (4 * u + v)] = (FULL || nv) ? (uint16_t)min((key2_of(qm) >> 16) + 1u, 0xFFFFu) : (uint16_t)0;
    if (FULL) {
      st_f32x4_evict_last(reinterpret_cast<float*>(la.e + la.step(u, v) * 4), b[0], b[1], b[2], b[3], pol);
    } else {
      nvalid += nv;
      const int64_t off = goff<RPQ_SHIFT>(d, q);
      if (nv == 4) st_f32x4_evict_last(ef + off, b[0], b[1], b[2], b[3], pol);
      else store_f32x4(ef, off, nv, b);
    }
  }
  return gm;
}

template <int C, bool BF16, int VPU, int NSW, int D, int NS, class Smem>
__device__ __forceinline__ void stream_warp(const CompressArgs& a, Smem& sm, int sw, int lane) {
  using PBuf = PassBuf<BF16>;
  constexpr int NP = WarpCfg<C>::NP;
  constexpr int RPQ_SHIFT = WarpCfg<C>::RPQ_SHIFT;
  const int64_t G = gridDim.x, n = a.n_chunks;
  unsigned char(*ring)[PBuf::bytes] = sm.ring[sw];
  const uint64_t pol_last = l2_policy_evict_last();
  const float beta = a.beta;
  float* ef = a.ef;

  // issue cursor: (chunk index ji of this CTA, pass iu), D passes ahead of the consumer
  int64_t ji = sw;
  int iu = 0;
  ChunkDesc di;
  di.base = 0; di.ld = 0; di.len = C;
  LaneAddr<C, BF16> lai;
  bool live_i = blockIdx.x + ji * G < n;
  if (live_i) di = a.chunks[blockIdx.x + ji * G];
  lai.init(a, di, lane);
  int slot_i = 0;
  auto issue_next = [&]() {
    if (live_i) issue_pass<C, BF16>(a, di, lai, iu, ring[slot_i], lane);
    cp_async_commit();  // empty groups past the end keep the wait_group accounting uniform
    slot_i = slot_i + 1 == D ? 0 : slot_i + 1;
    if (++iu == NP) {
      iu = 0;
      ji += NSW;
      live_i = blockIdx.x + ji * G < n;
      if (live_i) {
        di = a.chunks[blockIdx.x + ji * G];
        lai.init(a, di, lane);
      }
    }
  };
#pragma unroll
  for (int j = 0; j < D; j++) issue_next();

  int slot_c = 0;
  for (int64_t j = sw;; j += NSW) {
    const int64_t c = blockIdx.x + j * G;
    if (c >= n) break;
    const ChunkDesc d = a.chunks[c];
    LaneAddr<C, BF16> la;
    la.init(a, d, lane);
    PHASE_T0();
    const int slot = (int)(j % NS);
    const int64_t use = j / NS;
    if (VPU == 1) {
      // quads: each pass writes its 4 keys straight into the slot, so the slot
      // is claimed before the chunk's first pass (it was freed when the chunk
      // NS back started its selection)
      if (use > 0) ptx::mbar_wait(&sm.empty[slot], (uint32_t)((use - 1) & 1));
      uint16_t* qdst = reinterpret_cast<uint16_t*>(&sm.gk[slot][lane]);
#pragma unroll 1
      for (int u = 0; u < NP; u++) {
        cp_async_wait<D - 1>();
        int nv = 0;
        if (d.len == C)
          consume_pass<BF16, true, RPQ_SHIFT>(ring[slot_c], beta, ef, la, d, u, lane, pol_last, nv, qdst);
        else
          consume_pass<BF16, false, RPQ_SHIFT>(ring[slot_c], beta, ef, la, d, u, lane, pol_last, nv, qdst);
        issue_next();
        slot_c = slot_c + 1 == D ? 0 : slot_c + 1;
      }
      PHASE_MARK(0);
      ptx::mbar_arrive(&sm.full[slot]);  // release: e stores and keys of this lane
      continue;
    }
    uint32_t gk[NP];
    // passes not unrolled (instruction-cache footprint: the select warps run
    // other code on the same SM); gk[u] written by predicated moves so the
    // array stays in registers
    if (d.len == C) {
#pragma unroll 1
      for (int u = 0; u < NP; u++) {
        cp_async_wait<D - 1>();  // this lane's copies of pass u have landed
        int nv = 0;
        const uint32_t key =
            key2_of(consume_pass<BF16, true, RPQ_SHIFT>(ring[slot_c], beta, ef, la, d, u, lane, pol_last, nv));
#pragma unroll
        for (int x = 0; x < NP; x++) gk[x] = x == u ? key : gk[x];
        issue_next();  // refill the slot with the pass D ahead (possibly the next chunk's)
        slot_c = slot_c + 1 == D ? 0 : slot_c + 1;
      }
    } else {
#pragma unroll 1
      for (int u = 0; u < NP; u++) {
        cp_async_wait<D - 1>();
        int nv = 0;
        const float gm = consume_pass<BF16, false, RPQ_SHIFT>(ring[slot_c], beta, ef, la, d, u, lane, pol_last, nv);
        const uint32_t key = nv ? key2_of(gm) : 0u;
#pragma unroll
        for (int x = 0; x < NP; x++) gk[x] = x == u ? key : gk[x];
        issue_next();
        slot_c = slot_c + 1 == D ? 0 : slot_c + 1;
      }
    }
    // hand the maxima over: wait for the slot's previous chunk to be taken
    PHASE_MARK(0);
    if (use > 0) ptx::mbar_wait(&sm.empty[slot], (uint32_t)((use - 1) & 1));
    PHASE_MARK(6);
#pragma unroll
    for (int u = 0; u < NP; u++) sm.gk[slot][32 * u + lane] = gk[u];
    ptx::mbar_arrive(&sm.full[slot]);  // release: e stores and maxima of this lane
  }
  cp_async_wait<0>();
}

template <int C, bool BF16, int KC, int IBC, int CAP, int KMAX, int VPU, int NSEL, int NS, class Smem>
__device__ __forceinline__ void select_warp(const CompressArgs& a, Smem& sm, int sel, int lane) {
  constexpr int NU = UnitCfg<C, VPU>::NU;
  Compressor<C, BF16, KC, IBC, CAP, KMAX, VPU, true> cp(a, sm.scratch[sel], lane, KC ? KC : a.g.k);
  const int64_t G = gridDim.x, n = a.n_chunks;
  for (int64_t j = sel;; j += NSEL) {
    const int64_t c = blockIdx.x + j * G;
    if (c >= n) break;
    const int slot = (int)(j % NS);
    PHASE_T0();
    ptx::mbar_wait(&sm.full[slot], (uint32_t)((j / NS) & 1));
    PHASE_MARK(7);
    uint32_t gk[NU];
#pragma unroll
    for (int u = 0; u < NU; u++) {
      // quads: the key rounded down to 16 bits (| 1: a zero quad keeps the key
      // of 0, as a 16-position group does); 0 = no valid position
      const uint32_t h = sm.gk[slot][32 * u + lane];
      gk[u] = VPU == 1 ? (h ? ((h - 1u) << 16) | 1u : 0u) : h;
    }
    ptx::mbar_arrive(&sm.empty[slot]);
    Sel s;
    s.c = c;
    s.d = a.chunks[c];
    s.len = s.d.len;
    s.full = s.len == C;
    s.k_eff = s.full ? cp.k : max(1, (cp.k * s.len) / C);
    cp.select(s, gk);
  }
}

template <int C, bool BF16, int KC, int IBC, int CAP, int KMAX, int VPU, int NSW, int NSEL, int D, int NS>
__global__ void __launch_bounds__((NSW + NSEL) * 32, 1) compress_ws_kernel(const CompressArgs a) {
  using Smem = WsSmem<C, BF16, CAP, KMAX, VPU, NSW, NSEL, D, NS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < NS) {
    ptx::mbar_init(&sm.full[threadIdx.x], 32);
    ptx::mbar_init(&sm.empty[threadIdx.x], 32);
  }
  ptx::fence_mbar_init();
  __syncthreads();
  if (warp < NSW)
    stream_warp<C, BF16, VPU, NSW, D, NS>(a, sm, warp, lane);
  else
    select_warp<C, BF16, KC, IBC, CAP, KMAX, VPU, NSEL, NS>(a, sm, warp - NSW, lane);
}

// The chunks compress_ws_kernel deferred (more than CAP candidates: tied
// levels, constant or sparse runs; or a non-finite value): one warp per chunk
// takes T and the candidate groups from the deferral info, re-reads those
// groups of e = b (stored by the stream) and runs the selection with its
// fallback chain (key_select / tie_select / radix, warp_select.cuh), then Q
// and F.  Warp-strided over the list; the last block to finish zeroes the
// list header for the next launch.
constexpr int kFbWarps = 4;

// L2 prefetch of a full chunk's e (the warp's next deferred chunk, so its
// HBM latency hides behind the current one; partial chunks are not prefetched)
template <int C>
__device__ __forceinline__ void prefetch_chunk_l2(const float* ef, const ChunkDesc& d, int lane) {
  if (d.len != C) return;
  constexpr int B = WarpCfg<C>::B;
  constexpr int LPR = B * 4 / 128;  // 128-byte lines per block row
  constexpr int LINES = C * 4 / 128;
#pragma unroll
  for (int t = lane; t < LINES; t += 32) {
    const float* p = d.ld ? ef + d.base + (int64_t)(t / LPR) * d.ld + 32 * (t % LPR) : ef + d.base + 32 * (int64_t)t;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
}
#ifndef SLC_FB_MINB
#define SLC_FB_MINB 4  // fallback blocks per SM (register cap 65536 / (32 * kFbWarps * SLC_FB_MINB))
#endif
template <int C, bool BF16, int KC, int IBC, int CAP, int KMAX, int VPU>
__global__ void __launch_bounds__(kFbWarps * 32, SLC_FB_MINB) compress_fallback_kernel(const CompressArgs a) {
  __shared__ WarpScratch<C, CAP, KMAX, VPU> scratch[kFbWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Compressor<C, BF16, KC, IBC, CAP, KMAX, VPU, false> cp(a, scratch[warp], lane, KC ? KC : a.g.k);
  const uint32_t n = *reinterpret_cast<volatile uint32_t*>(&a.defer[0]);
  const uint32_t* list = a.defer + kDeferHdr;
  // entries are taken one at a time from a shared counter (a tied chunk's
  // selection costs several times a plain one), the next one as soon as the
  // current one starts, so its e can be prefetched into L2 meanwhile
  auto take = [&]() {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(&a.defer[2], 1u);
    return __shfl_sync(kFull, i, 0);
  };
  uint32_t i = take();
  while (i < n) {
    const uint32_t next = take();
    if (next < n) prefetch_chunk_l2<C>(a.ef, a.chunks[list[next]], lane);
    Sel s;
    s.c = list[i];
    s.d = a.chunks[s.c];
    s.len = s.d.len;
    s.full = s.len == C;
    s.k_eff = s.full ? cp.k : max(1, (cp.k * s.len) / C);
    cp.select_deferred(s, list + a.defer_cap + (int64_t)i * a.defer_info);
    i = next;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.defer[1], 1u) == gridDim.x - 1) {
      a.defer[0] = 0u;
      a.defer[1] = 0u;
      a.defer[2] = 0u;
      __threadfence();
    }
  }
}

template <int C, bool BF16, int KC, int IBC, int CAP, int KMAX, int VPU>
cudaError_t launch_ws_t(const CompressArgs& a, cudaStream_t s) {
  if (a.max_ld >= (1 << 24)) return launch_compress_warp(a, BF16, s);  // in-chunk offsets need > 32 bits
  constexpr int NSW = SLC_WS_NSW, NSEL = SLC_WS_NSEL, D = SLC_WS_D, NS = NSW + NSEL + SLC_WS_XS;
  using Smem = WsSmem<C, BF16, CAP, KMAX, VPU, NSW, NSEL, D, NS>;
  constexpr size_t smem = sizeof(Smem);
  static_assert(smem <= 227 * 1024, "compress_ws shared memory");
  auto kern = compress_ws_kernel<C, BF16, KC, IBC, CAP, KMAX, VPU, NSW, NSEL, D, NS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  int64_t grid = sms;
  if (grid > a.n_chunks) grid = a.n_chunks;
  kern<<<(unsigned)grid, (NSW + NSEL) * 32, smem, s>>>(a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  compress_fallback_kernel<C, BF16, KC, IBC, CAP, KMAX, VPU><<<(unsigned)(SLC_FB_MINB * sms), kFbWarps * 32, 0, s>>>(a);
  return cudaGetLastError();
}

template <int C, bool BF16>
cudaError_t launch_ws_c(const CompressArgs& a, cudaStream_t s) {
  if (C == 4096 && a.g.k == 64 && a.g.ib == 12)  // the paper's geometry
    return launch_ws_t<C, BF16, 64, 12, SLC_WS_CAP64, 64, 4>(a, s);
  if (ws_vpu(a.g) == 1) return launch_ws_t<C, BF16, 0, 0, SLC_WS_CAPG, kMaxK, 1>(a, s);
  return launch_ws_t<C, BF16, 0, 0, SLC_WS_CAPG, kMaxK, 4>(a, s);
}

}  // namespace

cudaError_t launch_compress_ws(const CompressArgs& a, int bf16, cudaStream_t s) {
  if (a.n_chunks == 0) return cudaSuccess;
  switch (a.g.C) {
    case 1024: return bf16 ? launch_ws_c<1024, true>(a, s) : launch_ws_c<1024, false>(a, s);
    case 4096: return bf16 ? launch_ws_c<4096, true>(a, s) : launch_ws_c<4096, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

#ifdef SLC_PHASE_TIMING
extern "C" int slc_debug_phase_cycles_ws(unsigned long long* out8, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, g_phase_cycles, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
    cudaMemcpyToSymbol(g_path_count, z, sizeof(z));
    cudaMemcpyToSymbol(g_path_count, z, sizeof(z), sizeof(z));
  }
  return (int)e;
}
extern "C" int slc_debug_path_count_ws(unsigned long long* out8) {
  return (int)cudaMemcpyFromSymbol(out8, g_path_count, sizeof(unsigned long long) * 16);
}
#endif
}  // namespace slc
