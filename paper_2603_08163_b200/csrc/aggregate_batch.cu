// aggregate_batch.cu — fused decode / aggregate / outer update for the paper's
// geometry (C = 4096, k = 64, 12-bit indices): Eq. 2 of PAPER.md
// with the arithmetic of R#17 / R#18 (the same sums and roundings as
// aggregate.cu / aggregate_pipe.cu).  Built from what the R = 20 profiles of
// aggregate_pipe.cu showed: 5.1 k warp instructions per chunk, 55 %
// issue-active, and a theta stream that cannot keep enough bytes in flight
// from registers (measured alone: 3.4 ms fp32 / 2.9 ms bf16 for 8B/4, where
// HBM allows 2.6 / 1.4).
//
//  * theta never passes through registers: the TMA engine loads each chunk's
//    64x64 block (2-D tensor map per blocked segment) or 4096-run (1-D bulk
//    copy) into a shared-memory tile, D chunks ahead, and stores the tile back
//    after the update (bulk async groups) — the stream runs while the warps
//    decode;
//  * theta changes only where Delta != 0 (fma(-alpha, +0, x) == x for every
//    x), so the update is applied in the tile at the touched positions only,
//    by the entry that owns each position: no dense pass, no Delta array;
//  * every CTA takes batches of NB consecutive chunks, dealt round-robin; a
//    batch's R records are contiguous per peer, so ONE bulk copy per peer
//    stages them (with the NB chunk descriptors);
//  * warp 0 turns the batch's 2*R*NB fp16 scales into per-(chunk, record)
//    VALUE tables — the four signed, pre-shifted integers a 2-bit code can
//    select — and picks each chunk's accumulator (FAST / PAIR / W below), so
//    the scatter is: decode index, decode code, one table load, one atomic;
//  * two CTA barriers per chunk: scatter | convert+update; the accumulator is
//    read back AND re-zeroed by one atomic exchange per entry (exactly one
//    entry of each touched position sees the sum).
//
// Accumulators (exact, so order-free, R#17):
//  FAST  unit weights, the chunk's nonzero scales within 2^(20 - ceil(log2 R)):
//        F >> sh per entry (F = scale * 2^24), an int32 sum per position;
//  PAIR  unit weights otherwise (F split hi * 2^20 + lo), or weights whose exact
//        products w_r * S_b (35 bits, M * 2^E) span <= 2^(17 - ceil(log2 R)):
//        (lo, hi) int32 pair per position;
//  W     weights otherwise: fp64 in canonical peer order, one warp.
// Delta = (float)(X * invR), X the exact sum as a double (X * 2^e exact): the
// oracle's (float)(acc * (1.0 / R)); for R a power of two (invR exact) the
// FAST conversion is I2F + an exact power-of-two FMUL.  decode_aggregate
// (dense Delta out) stays on aggregate_pipe.cu.
#include <cuda_fp16.h>

#include <algorithm>

#include "chunk_io.cuh"
#include "ptx.cuh"

#ifdef SLC_BATCH_TIMING  // debug builds: per-phase SM cycles summed over warps (slc_debug_batch_cycles)
namespace slc {
__device__ unsigned long long g_batch_cycles[8];
}
#define BT0() long long _bt = clock64()
#define BTM(i)                        \
  do {                                \
    long long _n = clock64();         \
    B.tcy[i] += (unsigned long long)(_n - _bt); \
    _bt = _n;                         \
  } while (0)
#else
#define BT0() \
  do {        \
  } while (0)
#define BTM(i) \
  do {         \
  } while (0)
#endif

namespace slc {
namespace {

#ifndef SLC_BATCH_NT
#define SLC_BATCH_NT 256  // threads per CTA (measured: 512 with 2 CTAs per SM is slower)
#endif
constexpr int kC = 4096, kK = 64, kIB = 12, kRW = 29, kNT = SLC_BATCH_NT;
constexpr int kNW = kNT / 32;
constexpr int kMinBlocks = kNT >= 512 ? 2 : 3;
constexpr int kMaxR = 64;

enum : int { kFast = 0, kPair = 1, kSeqW = 2 };
constexpr int kBadV = (int)0x80000000;  // table sentinel: non-finite scale (never a valid value)

// shared-memory layout, computed on the host and passed as a kernel parameter
// (device code reads the offsets from the constant bank instead of recomputing them)
struct BatchLayout {
  int R, NB, SP;  // SP: bytes per peer in a stage (16-B multiple)
  int NTILE, D;   // theta tiles, chunks loaded ahead (D <= NTILE - 2)
  int tile_bytes;
  uint32_t off_spos, off_tab, off_tab1, off_meta, off_bar, off_tbar, off_stage, stage_bytes, off_tile, total;
  void init(int R_, int NB_, int NTILE_, int pb) {
    R = R_;
    NB = NB_;
    NTILE = NTILE_;
    D = NTILE_ - 2;
    tile_bytes = kC * pb;
    SP = (116 * NB + 24 + 15) & ~15;
    off_spos = 16384;                                         // acc: int[C] / int2[C/2] / double[C/2]
    off_tab = off_spos + (((uint32_t)R * kK * 2 + 15) & ~15u);  // u16 entry positions
    off_tab1 = off_tab + (uint32_t)NB * R * 32;               // PAIR: int2[NB][R][4] value tables
    off_meta = off_tab1 + (uint32_t)NB * R * 16;              // FAST: int[NB][R][4]
    off_bar = off_meta + (uint32_t)NB * 16;                   // per chunk: mode, L, cf (double)
    off_tbar = off_bar + 16;                                  // 2 stage mbarriers
    off_stage = (off_tbar + 8 * NTILE + 127) & ~127u;         // NTILE tile mbarriers
    stage_bytes = ((uint32_t)R * SP + (uint32_t)NB * 32 + 127) & ~127u;  // records + descriptors
    off_tile = off_stage + 2 * stage_bytes;                   // 128-B aligned (TMA destination)
    total = off_tile + (uint32_t)NTILE * tile_bytes;
  }
};

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// a CUtensorMap (128 B, 64-B aligned) without the driver header
struct alignas(64) CUtensorMapLike {
  unsigned long long v[16];
};

struct Meta {
  int mode;
  int L;      // PAIR: bits of the lo half
  double cf;  // exact power of two: X = (sum) * cf
};

__device__ __forceinline__ long long f16_fixed24(uint32_t h) {
  const uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
  return e == 0 ? (long long)m : (long long)(1024u + m) << (e - 1);
}

// exact int32 -> double with one DADD (the FP64 pipe) instead of I2F.F64 (measured on
// B200: 10.9 vs 7.3 conversions per SM clock for the whole chain)
__device__ __forceinline__ double i2d_exact(int v) {
  return __hiloint2double(0x43300000, (int)((unsigned)v ^ 0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}

__device__ __forceinline__ uint32_t rec_index(const uint32_t* rec, int j) {
  const int bit = kIB * j;
  const int w = bit >> 5, sh = bit & 31;
  return __funnelshift_r(rec[w], rec[w + 1], sh) & 0xFFFu;
}

struct Desc {
  int64_t base;
  int32_t ld, len;
};

__device__ __forceinline__ Desc read_desc(const unsigned char* p) {
  const int4 v = *reinterpret_cast<const int4*>(p);
  Desc d;
  d.base = (int64_t)(((uint64_t)(uint32_t)v.y << 32) | (uint32_t)v.x);
  d.ld = v.z;
  d.len = v.w;
  return d;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          ptx::smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(ptx::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* tmap, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap), "r"(x),
               "r"(y), "r"(ptx::smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(ptx::smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ptx::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <bool BF16, bool POW2R>
struct Batch {
  const AggArgs& a;
  const BatchLayout& lay;
  unsigned char* sm;
  int* acc32;
  uint16_t* spos;
  int2* tab;   // PAIR value tables
  int* tab1;   // FAST value tables
  Meta* meta;
  uint64_t* bar;
  int64_t q0, G;   // this CTA's batches: q0, q0 + G, q0 + 2G, ... (batch q = chunks [q*NB, q*NB + NB))
  int64_t nbat;    // batches of this CTA
  int64_t bi;      // current batch
  int jj, nb;      // chunk within the batch, chunks in the batch
  int64_t j;       // chunk sequence number of this CTA (tile ring position)
  Desc dcur;       // current chunk
  unsigned char* tiles;
  uint64_t* tbar;
  // the TMA side (thread 0 only): chunk sequence number of the next load, and
  // that chunk's descriptor, fetched one load ahead (its latency off the path)
  int64_t jload, bload;
  int jjload;
  int4 pf0, pf1;
  int t, lane, warp;
  bool bad;
#ifdef SLC_BATCH_TIMING
  unsigned long long tcy[8];
#endif

  __device__ __forceinline__ int64_t first_chunk(int64_t bi) const { return (q0 + bi * G) * lay.NB; }
  __device__ __forceinline__ int chunks_in(int64_t bi) const { return (int)min64(lay.NB, a.n_chunks - first_chunk(bi)); }
  __device__ __forceinline__ unsigned char* stage(int s) const { return sm + lay.off_stage + s * lay.stage_bytes; }
  __device__ __forceinline__ unsigned char* stage_desc(int s, int jj) const {
    return stage(s) + lay.R * lay.SP + 32 * jj;
  }
  // words of record (jj, r) in stage s; o0w = (116 * c0 / 4) & 3 words of alignment slop
  __device__ __forceinline__ const uint32_t* rec_of(int s, int o0w, int jj, int r) const {
    return reinterpret_cast<const uint32_t*>(stage(s) + r * lay.SP) + o0w + kRW * jj;
  }

  // ---- stage batch bi's records and descriptors (all threads): 16-B cp.async
  // pieces of each peer's window [w0, floor16(b1)) and 4-B pieces of the rest
  // (never past the peers' buffers); every thread then arrives on the stage
  // barrier when its copies have landed.  (One TMA bulk copy per peer was
  // measured slower: ~25 small TMA ops per batch queue up behind / in front of
  // the theta tile loads and stores.)
  __device__ __forceinline__ void issue(int64_t bi) {
    const int64_t c0 = first_chunk(bi);
    const int nb = chunks_in(bi);
    const int s = (int)(bi & 1);
    const int64_t b0 = 116 * c0, b1 = 116 * (c0 + nb);
    const int64_t w0 = b0 & ~(int64_t)15;
    const int P16 = (int)(((b1 & ~(int64_t)15) - w0) >> 4);
    const int P4 = (int)((b1 & 15) >> 2);
    const int P = P16 + P4;
    unsigned char* st = stage(s);
    for (int i = t; i < a.R * P; i += kNT) {
      const int r = i / P, q = i - r * P;
      const char* src = reinterpret_cast<const char*>(a.rec[r]) + w0;
      unsigned char* dst = st + r * lay.SP;
      if (q < P16) {
        cp_async16(dst + 16 * q, src + 16 * q);
      } else {
        const int o = 16 * P16 + 4 * (q - P16);
        cp_async4(dst + o, src + o);
      }
    }
    for (int i = t; i < 2 * nb; i += kNT)
      cp_async16(st + lay.R * lay.SP + 16 * i, reinterpret_cast<const char*>(a.chunks + c0) + 16 * i);
    ptx::cp_async_arrive_noinc(&bar[s]);
  }

  __device__ __forceinline__ void wait_stage(int64_t bi) {
    ptx::mbar_wait(&bar[bi & 1], (uint32_t)((bi >> 1) & 1));
  }

  // ---- warp 0 after wait_stage: per chunk of batch bi, lane r takes record r:
  // the chunk's exponent range (two warp reductions) picks its accumulator and
  // shift (every lane computes the same), then each lane writes its record's
  // value table; lane 0 the chunk's Meta
  __device__ void build_tables(int64_t bi) {
    const int64_t c0 = first_chunk(bi);
    const int nb = chunks_in(bi);
    const int s = (int)(bi & 1);
    const int o0w = (int)((29 * c0) & 3);
    const int R = a.R;
    const int rbits = R > 1 ? 32 - __clz(R - 1) : 0;
    for (int jj = 0; jj < nb; jj++) {
      // the exponents (unweighted: fp16 exponent fields of nonzero finite
      // scales, e = 0 counted as 1; weighted: E of the exact products M * 2^E)
      int mn = 0x7FFFFFFF, mx = (int)0x80000000;
      for (int r = lane; r < R; r += 32) {
        const uint32_t sw = rec_of(s, o0w, jj, r)[kRW - 1];
#pragma unroll
        for (int b = 0; b < 2; b++) {
          const uint32_t h = (sw >> (16 * b)) & 0xFFFFu;
          const int e = (int)((h >> 10) & 0x1Fu);
          if (!a.weighted) {
            if ((h & 0x7FFFu) != 0 && e < 31) { mn = min(mn, max(1, e)); mx = max(mx, max(1, e)); }
          } else {
            const double d = __dmul_rn(peer_weight(a, r), (double)__half2float(__ushort_as_half((unsigned short)h)));
            if (!isfinite(d) || e == 31) {
              mn = -(1 << 20);  // -> sequential path (which latches the error)
              mx = 1 << 20;
            } else if (d != 0.0) {
              const unsigned long long db = (unsigned long long)__double_as_longlong(d);
              const unsigned long long M = ((db & 0xFFFFFFFFFFFFFull) | (1ull << 52)) >> 18;
              const int E = (int)((db >> 52) & 0x7FF) - 1075 + 18;
              if (M & ~((1ull << 35) - 1)) { mn = -(1 << 20); mx = 1 << 20; }
              mn = min(mn, E);
              mx = max(mx, E);
            }
          }
        }
      }
      const int lo = __reduce_min_sync(0xFFFFFFFFu, mn);
      const int hi = __reduce_max_sync(0xFFFFFFFFu, mx);
      int md, sh;
      if (!a.weighted) {
        if (lo > hi || hi - lo + 11 + rbits <= 31) { md = kFast; sh = lo > hi ? 0 : lo - 1; }
        else { md = kPair; sh = 0; }
      } else {
        if (lo > hi) { md = kPair; sh = 0; }
        else if (hi - lo + 35 + rbits <= 52) { md = kPair; sh = lo; }
        else { md = kSeqW; sh = 0; }
      }
      if (lane == 0) {
        Meta mt;
        mt.mode = md;
        mt.L = a.weighted ? 31 - rbits : 20;
        // exact powers of two, built from their bits
        const int ce = !a.weighted ? (md == kFast ? sh - 24 : -24) : sh;
        mt.cf = __longlong_as_double((long long)(1023 + ce) << 52);
        meta[jj] = mt;
      }
      if (md == kSeqW) continue;
      for (int r = lane; r < R; r += 32) {
        const uint32_t sw = rec_of(s, o0w, jj, r)[kRW - 1];
        int2* T = tab + (jj * R + r) * 4;
        int* T1 = tab1 + (jj * R + r) * 4;
#pragma unroll
        for (int b = 0; b < 2; b++) {  // b = bucket bit; code = 2*b + sign
          const uint32_t h = (sw >> (16 * b)) & 0xFFFFu;
          const bool nonfin = ((h >> 10) & 0x1Fu) == 0x1Fu;
          if (!a.weighted) {
            const long long F = f16_fixed24(h);
            if (md == kFast) {
              const int v = (int)(F >> sh);
              T1[2 * b] = nonfin ? kBadV : v;
              T1[2 * b + 1] = nonfin ? kBadV : -v;
            } else {
              const int l = (int)(F & 0xFFFFF), u = (int)(F >> 20);
              T[2 * b] = make_int2(l, nonfin ? kBadV : u);
              T[2 * b + 1] = make_int2(-l, nonfin ? kBadV : -u);
            }
          } else {
            const float wf = (float)peer_weight(a, r);
            const double d = __dmul_rn((double)wf, (double)__half2float(__ushort_as_half((unsigned short)h)));
            unsigned long long V = 0;
            if (d != 0.0) {
              const unsigned long long db = (unsigned long long)__double_as_longlong(d);
              const unsigned long long M = ((db & 0xFFFFFFFFFFFFFull) | (1ull << 52)) >> 18;
              const int E = (int)((db >> 52) & 0x7FF) - 1075 + 18;
              V = M << (E - sh);  // < 2^(52 - rbits)
            }
            const int L = 31 - rbits;
            int l = (int)(V & ((1ull << L) - 1)), u = (int)(V >> L);
            if (wf < 0.0f) { l = -l; u = -u; }
            T[2 * b] = make_int2(l, u);
            T[2 * b + 1] = make_int2(-l, -u);
          }
        }
      }
    }
  }

  // FAST chunks in one pass over the whole chunk; PAIR / W chunks in two passes
  // hf = 0, 1 over the position halves [2048 hf, 2048 hf + 2048), so that every
  // accumulator fits 16 KB (int[4096] / int2[2048] / double[2048])
  __device__ __forceinline__ void scatter(int s, int o0w, int jj, int len, const Meta& m, int hf) {
    const int R = a.R;
    const int k_eff = len == kC ? kK : max(1, (kK * len) / kC);
    if (m.mode == kSeqW) {
      if (warp == 0) {
        double* accd = reinterpret_cast<double*>(acc32);
        for (int r = 0; r < R; r++) {  // canonical peer order (host-sorted)
          const uint32_t* rec = rec_of(s, o0w, jj, r);
          const double w = peer_weight(a, r);
          const uint32_t sw = rec[kRW - 1];
          for (int j = lane; j < k_eff; j += 32) {
            uint32_t p = rec_index(rec, j);
            const uint32_t code = (rec[24 + (j >> 4)] >> (2 * (j & 15))) & 3u;
            const uint32_t h = (code & 2u) ? (sw >> 16) : (sw & 0xFFFFu);
            if ((int)p >= len || ((h >> 10) & 0x1Fu) == 0x1Fu) {
              bad = true;
              spos[r * k_eff + j] = 0;
              continue;
            }
            spos[r * k_eff + j] = (uint16_t)p;
            if ((int)(p >> 11) != hf) continue;
            float dq = __half2float(__ushort_as_half((unsigned short)h));
            if (code & 1u) dq = -dq;
            accd[p & 2047u] = __dadd_rn(accd[p & 2047u], __dmul_rn(w, (double)dq));
          }
          __syncwarp();
        }
      }
      return;
    }
    const int* T1 = tab1 + jj * R * 4;                                // FAST: int per (r, code)
    const int2* T2 = tab + jj * R * 4;                                // PAIR: (lo, hi) per (r, code)
    if (k_eff == kK) {
      // full chunk: unit u = (record r = u/2, half h = u%2): 32 consecutive
      // slots with lane-constant bit offsets; units spread evenly over the warps
      const int wl = (kIB * lane) >> 5, shl = (kIB * lane) & 31;
      const int cw = 24 + (lane >> 4), csh = 2 * (lane & 15);
      const uint32_t* rec0 = rec_of(s, o0w, jj, 0);
      const int spw = lay.SP >> 2;  // words per peer in a stage
      if (m.mode == kFast) {
        // warp w: half h = w % 2 of records r = w/2, w/2 + 4, ... (units spread
        // evenly); lane-constant word offsets, pointers stepped per record
        const int h = warp & 1;
        const int r0 = warp >> 1;
        constexpr int RS = kNW / 2;  // records per warp step
        const uint32_t* rp = rec0 + r0 * spw;
        const uint32_t* rend = rec0 + R * spw;
        const int io = 12 * h + wl, co = cw + 2 * h;
        const int* tp = T1 + 4 * r0;
        uint16_t* sp = spos + 64 * r0 + 32 * h + lane;
        int vmin = 0;
        for (; rp < rend; rp += RS * spw, tp += 4 * RS, sp += 64 * RS) {
          const uint32_t p = __funnelshift_r(rp[io], rp[io + 1], shl) & 0xFFFu;
          const uint32_t code = (rp[co] >> csh) & 3u;
          const int v = tp[code];
          vmin = min(vmin, v);
          *sp = (uint16_t)p;
          atomicAdd(&acc32[p], v);
        }
        bad |= vmin == kBadV;  // kBadV = INT_MIN: no valid value is smaller
      } else {
        for (int u = warp; u < 2 * R; u += kNT / 32) {
          const int r = u >> 1, h = u & 1;
          const uint32_t* rec = rec0 + r * spw;
          const uint32_t p = __funnelshift_r(rec[12 * h + wl], rec[12 * h + wl + 1], shl) & 0xFFFu;
          const uint32_t code = (rec[cw + 2 * h] >> csh) & 3u;
          const int2 v = T2[4 * r + code];
          bad |= v.y == kBadV;
          spos[64 * r + 32 * h + lane] = (uint16_t)p;
          if ((int)(p >> 11) == hf) {
            const uint32_t q = p & 2047u;
            atomicAdd(&acc32[2 * q], v.x);
            atomicAdd(&acc32[2 * q + 1], v.y);
          }
        }
      }
    } else {
      const int total = R * k_eff;
      for (int e = t; e < total; e += kNT) {
        const int r = e / k_eff, j = e - r * k_eff;
        const uint32_t* rec = rec_of(s, o0w, jj, r);
        uint32_t p = rec_index(rec, j);
        const uint32_t code = (rec[24 + (j >> 4)] >> (2 * (j & 15))) & 3u;
        const bool inr = (int)p < len;
        bad |= !inr;
        if (!inr) p = 0;
        spos[e] = (uint16_t)p;
        if (m.mode == kFast) {
          const int v = T1[4 * r + code];
          bad |= v == kBadV;
          if (inr) atomicAdd(&acc32[p], v);
        } else {
          const int2 v = T2[4 * r + code];
          bad |= v.y == kBadV;
          if (inr && (int)(p >> 11) == hf) {
            const uint32_t q = p & 2047u;
            atomicAdd(&acc32[2 * q], v.x);
            atomicAdd(&acc32[2 * q + 1], v.y);
          }
        }
      }
    }
  }

  // theta <- fma(-alpha, Delta, theta) at tile position p (R#18; bf16: widened, updated, re-rounded)
  __device__ __forceinline__ void update_at(unsigned char* tile, int p, float d, float alpha) const {
    if (BF16) {
      uint16_t* t16 = reinterpret_cast<uint16_t*>(tile) + p;
      *t16 = f32_to_bf16_rn_bits(__fmaf_rn(-alpha, d, bf16_bits_to_f32(*t16)));
    } else {
      float* t32 = reinterpret_cast<float*>(tile) + p;
      *t32 = __fmaf_rn(-alpha, d, *t32);
    }
  }

  // ---- pass 2: every touched position: the accumulator is read back and
  // re-zeroed by an exchange (exactly one entry of each position sees the sum),
  // Delta = (float)(X * invR), and theta is updated in the tile.  Untouched
  // positions keep theta: fma(-alpha, +0, x) == x.  Threads [t0, kNT) take the
  // entries (warp 0 sits out while it builds the next batch's tables).
  __device__ __forceinline__ void convert_update(int len, const Meta& m, int t0, unsigned char* tile, int hf) {
    const int k_eff = len == kC ? kK : max(1, (kK * len) / kC);
    const int total = a.R * k_eff;
    const int tt = t - t0, NTc = kNT - t0;
    if (tt < 0) return;
    const double invR = a.invR;
    const float alpha = a.alpha;
    if (m.mode == kFast) {
      const double cfi = m.cf * invR;  // exact: cf is a power of two
      if (POW2R) {
        const float cfif = (float)cfi;  // exact power of two: I2F (one rounding), then an exact scaling
        for (int e = tt; e < total; e += NTc) {
          const int p = spos[e];
          const int v = atomicExch(&acc32[p], 0);
          if (v != 0) update_at(tile, p, __fmul_rn(__int2float_rn(v), cfif), alpha);
        }
      } else {
        for (int e = tt; e < total; e += NTc) {
          const int p = spos[e];
          const int v = atomicExch(&acc32[p], 0);
          if (v != 0) update_at(tile, p, __double2float_rn(__dmul_rn(i2d_exact(v), cfi)), alpha);
        }
      }
    } else {
      unsigned long long* acc64 = reinterpret_cast<unsigned long long*>(acc32);
      const double twoL = ldexp(1.0, m.L);
      for (int e = tt; e < total; e += NTc) {
        const int p = spos[e];
        if ((p >> 11) != hf) continue;
        const unsigned long long u = atomicExch(&acc64[p & 2047], 0ull);
        if (u == 0ull) continue;
        double X;
        if (m.mode == kSeqW) {
          X = __longlong_as_double((long long)u);
        } else {
          const int lo = (int)(uint32_t)u, hi = (int)(uint32_t)(u >> 32);
          X = __dmul_rn(__fma_rn((double)hi, twoL, (double)lo), m.cf);  // exact
        }
        update_at(tile, p, __double2float_rn(__dmul_rn(X, invR)), alpha);
      }
    }
  }

  __device__ __forceinline__ void wait_tile(int64_t jseq) {
    ptx::mbar_wait(&tbar[jseq % lay.NTILE], (uint32_t)((jseq / lay.NTILE) & 1));
  }

  // ---- the theta stream (thread 0): tile j % NTILE holds chunk j of this CTA
  __device__ __forceinline__ unsigned char* tile_of(int64_t jseq) const {
    return tiles + (int)(jseq % lay.NTILE) * lay.tile_bytes;
  }
  // load the chunk at sequence position jload (batch bload, index jjload) and advance
  __device__ __forceinline__ void fetch_desc() {
    if (bload >= nbat) return;
    const int4* q = reinterpret_cast<const int4*>(a.chunks + first_chunk(bload) + jjload);
    pf0 = __ldg(q);
    pf1 = __ldg(q + 1);
  }
  __device__ __forceinline__ void load_next_tile() {
    if (bload >= nbat) return;
    ChunkDesc d;
    d.base = (int64_t)(((uint64_t)(uint32_t)pf0.y << 32) | (uint32_t)pf0.x);
    d.ld = pf0.z;
    d.len = pf0.w;
    d.tmap = pf1.x;
    d.tx = pf1.y;
    d.ty = pf1.z;
    const int k = (int)(jload % lay.NTILE);
    unsigned char* dst = tiles + k * lay.tile_bytes;
    uint64_t* tb = &tbar[k];
    constexpr int PB = BF16 ? 2 : 4;
    if (d.tmap >= 0) {
      ptx::mbar_arrive_expect_tx(tb, (uint32_t)lay.tile_bytes);
      tma_load_2d(dst, static_cast<const CUtensorMapLike*>(a.tmaps) + d.tmap, d.tx, d.ty, tb);
    } else {
      const uint32_t full16 = ((uint32_t)d.len * PB) & ~15u;
      tail_in(d.base, d.len, dst);  // generic stores, disjoint from the bulk copy's bytes
      if (full16) {
        ptx::mbar_arrive_expect_tx(tb, full16);
        ptx::bulk_g2s(dst, static_cast<const char*>(a.theta) + d.base * PB, full16, tb);
      } else {
        ptx::mbar_arrive(tb);
      }
    }
    jload++;
    if (++jjload == chunks_in(bload)) {
      bload++;
      jjload = 0;
    }
    fetch_desc();
  }
  // flat chunks whose byte length is not a multiple of 16: the last < 16 bytes by hand
  __device__ __forceinline__ void tail_in(int64_t base, int len, unsigned char* tile) const {
    constexpr int PB = BF16 ? 2 : 4;
    const int bytes = len * PB, full16 = bytes & ~15;
    const char* src = static_cast<const char*>(a.theta) + base * PB;
    for (int b = full16; b < bytes; b += PB) {
      if (BF16) *reinterpret_cast<uint16_t*>(tile + b) = *reinterpret_cast<const uint16_t*>(src + b);
      else *reinterpret_cast<uint32_t*>(tile + b) = *reinterpret_cast<const uint32_t*>(src + b);
    }
  }
  __device__ __forceinline__ void store_tile(const Desc& d, int tmap, int tx, int ty, const unsigned char* tile) const {
    constexpr int PB = BF16 ? 2 : 4;
    char* dst = static_cast<char*>(a.theta) + d.base * PB;
    if (tmap >= 0) {
      tma_store_2d(static_cast<const CUtensorMapLike*>(a.tmaps) + tmap, tx, ty, tile);
    } else {
      const int bytes = d.len * PB, full16 = bytes & ~15;
      if (full16) bulk_s2g(dst, tile, (uint32_t)full16);
      for (int b = full16; b < bytes; b += PB) {
        if (BF16) *reinterpret_cast<uint16_t*>(dst + b) = *reinterpret_cast<const uint16_t*>(tile + b);
        else *reinterpret_cast<uint32_t*>(dst + b) = *reinterpret_cast<const uint32_t*>(tile + b);
      }
    }
    bulk_commit();
  }
};

template <bool BF16, bool POW2R>
__device__ __forceinline__ bool batch_step(Batch<BF16, POW2R>& B) {
  BT0();
  const int s = (int)(B.bi & 1);
  const int64_t c0 = B.first_chunk(B.bi);
  const int o0w = (int)((29 * c0) & 3);
  const int jj = B.jj;
  const bool last_in_batch = jj + 1 == B.nb;
  const bool has_next = !last_in_batch || B.bi + 1 < B.nbat;
#ifndef SLC_BATCH_DECODE_ONLY  // tuning builds: no theta traffic
  if (B.t == 0) {
    // tile (j + D) % NTILE last held chunk j + D - NTILE <= j - 2, whose store
    // group is the second most recent: its shared-memory reads must be done
    bulk_wait_read<1>();
    B.load_next_tile();
  }
#endif
  // the current chunk's descriptor (stage of the current batch) and the
  // separate per-tile fields the TMA store needs (tmap, block coordinates)
  const unsigned char* dp = B.stage_desc(s, jj);
  const Desc d = read_desc(dp);
  const int4 dtm = *reinterpret_cast<const int4*>(dp + 16);  // tmap, tx, ty, pad
  const Meta m = B.meta[jj];
  unsigned char* tile = B.tile_of(B.j);
  BTM(0);
  const bool build = last_in_batch && B.bi + 1 < B.nbat;
  const int nh = m.mode == kFast ? 1 : 2;
  for (int hf = 0; hf < nh; hf++) {
#ifndef SLC_BATCH_STREAM_ONLY  // tuning builds: the theta stream alone
    B.scatter(s, o0w, jj, d.len, m, hf);
#endif
    BTM(1);
    __syncthreads();  // B1: scatter complete
    BTM(2);
    if (hf == nh - 1) {
      // this batch's stage is no longer read: refill it two batches ahead; warp 0
      // builds the next batch's tables (tab / meta are not read again before B2)
      if (last_in_batch && B.bi + 2 < B.nbat) B.issue(B.bi + 2);
#ifndef SLC_BATCH_STREAM_ONLY
      if (build && B.warp == 0) {
        B.wait_stage(B.bi + 1);
        B.build_tables(B.bi + 1);
      }
#else
      if (build) B.wait_stage(B.bi + 1);
#endif
      BTM(3);
    }
#ifndef SLC_BATCH_DECODE_ONLY
    if (hf == 0) B.wait_tile(B.j);
#endif
#if !defined(SLC_BATCH_NO_DECODE) && !defined(SLC_BATCH_STREAM_ONLY)
    B.convert_update(d.len, m, (hf == nh - 1 && build) ? 32 : 0, tile, hf);
#endif
    ptx::fence_proxy_async_smem();  // the tile writes, visible to the TMA store
    BTM(4);
    __syncthreads();  // B2: tile updated (and the next batch's tables built)
    BTM(5);
  }
#ifndef SLC_BATCH_DECODE_ONLY
  if (B.t == 0) B.store_tile(d, dtm.x, dtm.y, dtm.z, tile);
#endif
  BTM(6);
  if (!has_next) return false;
  B.j++;
  if (last_in_batch) {
    B.bi++;
    B.jj = 0;
    B.nb = B.chunks_in(B.bi);
  } else {
    B.jj = jj + 1;
  }
  return true;
}

template <bool BF16, bool POW2R>
__global__ void __launch_bounds__(kNT, kMinBlocks) agg_batch_kernel(const AggArgs a, const BatchLayout lay) {
  extern __shared__ __align__(128) unsigned char smem[];
  Batch<BF16, POW2R> B{a, lay};
  B.sm = smem;
  B.acc32 = reinterpret_cast<int*>(smem);
  B.spos = reinterpret_cast<uint16_t*>(smem + lay.off_spos);
  B.tab = reinterpret_cast<int2*>(smem + lay.off_tab);
  B.tab1 = reinterpret_cast<int*>(smem + lay.off_tab1);
  B.meta = reinterpret_cast<Meta*>(smem + lay.off_meta);
  B.bar = reinterpret_cast<uint64_t*>(smem + lay.off_bar);
  B.tbar = reinterpret_cast<uint64_t*>(smem + lay.off_tbar);
  B.tiles = smem + lay.off_tile;
  B.t = threadIdx.x;
  B.lane = threadIdx.x & 31;
  B.warp = threadIdx.x >> 5;
  B.bad = false;
#ifdef SLC_BATCH_TIMING
  for (int i = 0; i < 8; i++) B.tcy[i] = 0;
#endif
  // batches of NB consecutive chunks, dealt round-robin: concurrently running
  // CTAs work on neighbouring blocks (DRAM page locality of the theta rows)
  B.G = gridDim.x;
  B.q0 = blockIdx.x;
  const int64_t nq = (a.n_chunks + lay.NB - 1) / lay.NB;
  if (B.q0 >= nq) return;
  B.nbat = (nq - B.q0 + B.G - 1) / B.G;
  const int t = B.t;

  for (int i = t; i < 16384 / 16; i += kNT) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
  if (t == 0) {
    ptx::mbar_init(&B.bar[0], kNT);  // every thread's cp.async pieces
    ptx::mbar_init(&B.bar[1], kNT);
    for (int k = 0; k < lay.NTILE; k++) ptx::mbar_init(&B.tbar[k], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  B.issue(0);
  if (B.nbat > 1) B.issue(1);
  if (t == 0) {  // theta tiles of the first D chunks
    B.jload = 0;
    B.bload = 0;
    B.jjload = 0;
    B.fetch_desc();
#ifndef SLC_BATCH_DECODE_ONLY
    for (int i = 0; i < lay.D; i++) {
      B.load_next_tile();
      bulk_commit();  // (empty) store groups keep wait_group accounting uniform
    }
#endif
  }
  if (B.warp == 0) {
    B.wait_stage(0);
    B.build_tables(0);
  }
  __syncthreads();
  B.wait_stage(0);
  B.bi = 0;
  B.jj = 0;
  B.j = 0;
  B.nb = B.chunks_in(0);
  while (batch_step(B)) {
  }
  if (t == 0) bulk_wait_all();  // every tile store has landed before the CTA exits
  if (B.bad) atomicOr(a.err, kErrNonFinite);
#ifdef SLC_BATCH_TIMING
  if (B.lane == 0)
    for (int i = 0; i < 8; i++) atomicAdd(&g_batch_cycles[i], B.tcy[i]);
#endif
}

int pick_nb(int R) {
#ifdef SLC_BATCH_NB  // tuning builds
  if (SLC_BATCH_NB * 116 * R <= 40000) return SLC_BATCH_NB;
#endif
  return R <= 8 ? 4 : (R <= 12 ? 2 : 1);
}

// theta tiles: as many as fit 3 CTAs per SM (228 KB per SM, 1 KB reserved per
// CTA), at least 3 (one load in flight); else 2 CTAs per SM
int pick_ntile(int R, int NB, int pb, int& ctas) {
  BatchLayout l;
  l.init(R, NB, 0, pb);
  const int tb = kC * pb;
  for (ctas = kMinBlocks; ctas >= 1; ctas--) {
    const int budget = 233472 / ctas - 1024 - 128;
    const int nt = (budget - (int)l.total) / tb;
    if (nt >= 3) return std::min(nt, 16);
  }
  ctas = 1;
  return 3;
}

template <bool BF16, bool POW2R>
cudaError_t launch_t(const AggArgs& a, cudaStream_t s) {
  const int NB = pick_nb(a.R);
  const int pb = BF16 ? 2 : 4;
  int ctas = 0;
  BatchLayout lay;
  lay.init(a.R, NB, pick_ntile(a.R, NB, pb, ctas), pb);
  auto kern = agg_batch_kernel<BF16, POW2R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.total);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNT, lay.total)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = min64((a.n_chunks + NB - 1) / NB, (int64_t)sms * per_sm);
  if (a.grid_cap > 0) grid = min64(grid, a.grid_cap);
  kern<<<(unsigned)grid, kNT, lay.total, s>>>(a, lay);
  return cudaGetLastError();
}

}  // namespace

bool aggregate_batch_supported(const AggArgs& a) {
  if (!(a.g.C == kC && a.g.k == kK && a.g.ib == kIB && a.R <= kMaxR && a.rec_al16 && a.mode == kFused && a.tmaps_ok))
    return false;
  BatchLayout lay;
  lay.init(a.R, pick_nb(a.R), 3, 4);
  return lay.total <= 200 * 1024;
}

cudaError_t launch_aggregate_batch(const AggArgs& a, int bf16, cudaStream_t s) {
  if (a.n_chunks == 0) return cudaSuccess;
  const bool p2 = (a.R & (a.R - 1)) == 0;
  if (bf16) return p2 ? launch_t<true, true>(a, s) : launch_t<true, false>(a, s);
  return p2 ? launch_t<false, true>(a, s) : launch_t<false, false>(a, s);
}

#ifdef SLC_BATCH_TIMING
extern "C" int slc_debug_batch_cycles(unsigned long long* out8, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, g_batch_cycles, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_batch_cycles, z, sizeof(z));
  }
  return (int)e;
}
#endif
}  // namespace slc
