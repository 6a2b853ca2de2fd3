// aggregate_pipe.cu — persistent, software-pipelined decode / aggregate (/ outer
// update) kernel: Eq. 2 of PAPER.md, the same arithmetic as
// aggregate.cu (R#17, R#18) with the HBM latency hidden.
//
// The one-CTA-per-chunk kernel (aggregate.cu) runs its phases back to back —
// records in, scatter, theta in, theta out — so theta's HBM round trip is
// exposed once per chunk, and it converts all C accumulator entries although
// at most R*k of them were touched (ncu: 4.6 TB/s, 67 % issue-active).  Here a
// CTA of C/16 threads walks chunks c = blockIdx.x + i*gridDim.x and, while it
// works on chunk i, already has chunk i+1's theta loads (registers) and records
// (cp.async into the other shared-memory buffer) in flight; descriptors are
// loaded three chunks ahead, so no load waits on another.  Per thread: 16
// positions in 4 groups of 4 (chunk_io.cuh mapping), theta double-buffered in
// registers (2 x 16 fp32).
//
// Per chunk, with E = R * k_eff entries:
//   pass 1  every entry -> exact fixed-point accumulator acc[p] (shared
//           atomics), its position remembered in spos[]
//   pass 2  every entry: Delta[p] = (float)(acc[p] * 2^-24 * (1/R)) -> dlt[p];
//           untouched dlt stay +0
//   pass 3  dense: theta <- fma(-alpha, dlt, theta), dlt re-zeroed; acc
//           re-zeroed at the E touched positions only
// Accumulation is exact (R#17): each fp16 scale is an integer multiple of
// 2^-24.  When the chunk's nonzero scales span a small enough exponent range
// (always, on real pseudo-gradients) the sum of R of them fits one int32 after
// a common exact right shift — one shared atomic per entry, read back and
// re-zeroed by one atomicExch; otherwise the value is split hi*2^20 + lo over
// two int32 arrays as in aggregate.cu.  Either way the exact sum times the
// exact 2^(sh-24) * invR is one fp64 rounding, then one fp32 rounding: the
// oracle's (float)(acc * invR).  fma(-alpha, +0, theta) == theta for every
// theta, so the dense pass needs no special case.  Weighted mode (median-norm
// weights): fp64 in canonical peer order, one warp walking the peers.
#include <cuda_fp16.h>

#include <algorithm>

#include "chunk_io.cuh"

namespace slc {
namespace {

__device__ __forceinline__ long long f16_fixed24(uint32_t h) {
  const uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
  return e == 0 ? (long long)m : (long long)(1024u + m) << (e - 1);
}

__device__ __forceinline__ uint32_t rec_index(const uint32_t* rec, int j, int ib) {
  const int bit = ib * j;
  const int w = bit >> 5, sh = bit & 31;
  return __funnelshift_r(rec[w], rec[w + 1], sh) & ((1u << ib) - 1u);
}

__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// words of one record buffer (all R records of a chunk + 1 pad word), 16-B multiple
__host__ __device__ inline int rec_buf_words(int R, int RW) { return ((R * RW + 1) + 3) & ~3; }

template <int C>
struct PipeSmem {
  static constexpr size_t off_acc = 0;                 // int2[C] / double[C]
  static constexpr size_t off_dlt = sizeof(int2) * C;  // float[C]: Delta
  static constexpr size_t off_pos = off_dlt + sizeof(float) * C;  // u16[R * k]: entry positions
  __host__ __device__ static size_t off_rec(int R, int k) {
    return off_pos + ((sizeof(uint16_t) * R * k + 15) & ~size_t(15));
  }
  __host__ __device__ static size_t off_desc(int R, int k, int RW) {
    return off_rec(R, k) + 2 * sizeof(uint32_t) * rec_buf_words(R, RW);
  }
  // per-record scale table int4[R] and the chunk's scale-exponent range int2[2] (by buffer)
  __host__ __device__ static size_t off_tab(int R, int k, int RW) { return off_desc(R, k, RW) + 4 * 16; }
  __host__ __device__ static size_t off_erange(int R, int k, int RW) { return off_tab(R, k, RW) + 16 * R; }
  __host__ __device__ static size_t bytes(int R, int k, int RW) { return off_erange(R, k, RW) + 16; }
};

#ifndef SLC_AGG_UNROLL
#define SLC_AGG_UNROLL 1  // unroll of the per-entry loops (independent iterations in flight)
#endif
#define SLC_PRAGMA(x) _Pragma(#x)
#define SLC_UNROLL(n) SLC_PRAGMA(unroll n)

#ifndef SLC_AGG_MINB
#define SLC_AGG_MINB 3  // CTAs per SM the register budget is sized for (C = 4096)
#endif
#ifndef SLC_AGG_MINB_BF16
#define SLC_AGG_MINB_BF16 4  // the same with bf16 theta (half the theta registers: 64 suffice)
#endif

#ifndef SLC_AGG_THETA_NOW
#define SLC_AGG_THETA_NOW 0  // 1: theta loaded at the start of its own step (single register buffer)
#endif
#ifndef SLC_AGG_GPT
#define SLC_AGG_GPT 4  // 4-position groups per thread (C/(4*GPT) threads per CTA)
#endif
#ifndef SLC_AGG_WTAB
#define SLC_AGG_WTAB 1  // WFAST: per-record summand table instead of per-entry shifts
#endif
#ifndef SLC_AGG_FUSE_MUL
#define SLC_AGG_FUSE_MUL 64  // fuse when R * k_eff >= C / SLC_AGG_FUSE_MUL (measured: 64 beats 8 at R = 2-4, ties elsewhere)
#endif
#ifndef SLC_AGG_FUSE2
#define SLC_AGG_FUSE2 1  // FAST chunks: Delta converted in the dense pass (no pass 2, one barrier less)
#endif

template <int C>
struct PipeCfg {
  static constexpr int GPT = SLC_AGG_GPT;
  static constexpr int NT = C / (4 * GPT);
  static constexpr int MIN_BLOCKS = GPT == 4 ? ((C == 4096) ? SLC_AGG_MINB : 4 * SLC_AGG_MINB)
                                            : ((C == 4096) ? 4 : 16);
  static constexpr int MIN_BLOCKS_BF16 = (GPT == 4 && C == 4096) ? SLC_AGG_MINB_BF16 : MIN_BLOCKS;
  static constexpr int RPQ = ChunkCfg<C>::RPQ;  // 4-element groups per block row
  static constexpr int RPQ_SHIFT = (RPQ == 8) ? 3 : (RPQ == 16 ? 4 : 5);
};

// the 16 bytes of a chunk descriptor the update needs
struct Desc {
  int64_t base;
  int32_t ld, len;
};

__device__ __forceinline__ Desc unpack_desc(const int4 v) {
  Desc d;
  d.base = (int64_t)(((uint64_t)(uint32_t)v.y << 32) | (uint32_t)v.x);
  d.ld = v.z;
  d.len = v.w;
  return d;
}

// element offset of thread t's group v is o + v * step (full chunks)
template <int C>
__device__ __forceinline__ void full_addr(const Desc& d, int t, int64_t& o, int64_t& step) {
  using K = PipeCfg<C>;
  if (d.ld) {
    o = d.base + (int64_t)(t >> K::RPQ_SHIFT) * d.ld + 4 * (t & (K::RPQ - 1));
    step = (int64_t)(K::NT / K::RPQ) * d.ld;
  } else {
    o = d.base + 4 * t;
    step = 4 * K::NT;
  }
}

__device__ __forceinline__ int64_t generic_offset(const Desc& d, int q, int rpq_shift) {
  return d.ld ? d.base + (int64_t)(q >> rpq_shift) * d.ld + 4 * (q & ((1 << rpq_shift) - 1))
              : d.base + 4 * (int64_t)q;
}

template <int C, bool BF16>
__device__ __forceinline__ void load_theta(const void* theta, const Desc& d, int t, float th[4 * SLC_AGG_GPT]) {
  using K = PipeCfg<C>;
  if (d.len == C) {
    int64_t o, step;
    full_addr<C>(d, t, o, step);
#pragma unroll
    for (int v = 0; v < K::GPT; v++) load_param4<BF16>(theta, o + v * step, 4, &th[4 * v]);
  } else {
#pragma unroll
    for (int v = 0; v < K::GPT; v++) {
      const int q = v * K::NT + t;
      load_param4<BF16>(theta, generic_offset(d, q, K::RPQ_SHIFT), valid_in_group(4 * q, d.len), &th[4 * v]);
    }
  }
}

// Slot of record r in a shared-memory record buffer: SR words (32 for the
// compile-time layout, else RW).  Default layout (KC = 64, RW = 29 words =
// 116 B): record r is copied in 8 parts q — eight 16-B pieces of the
// 16-B-aligned 128-B window holding it ("wide"; the record then starts
// o = (29c) & 3 words into the slot) when every record buffer is 16-B aligned
// and the window stays inside the buffer (not the last chunk), else 4-B words
// w with w % 8 == (q + 5) % 8.  Part 7 holds the scale word (word 28); it is
// copied by thread r (mod NT), the other parts by threads R + 7r + q, so the
// scale tables are built by the first R threads (one warp at R <= 32) right
// after their own cp.async wait, without a barrier.
template <int KC>
__device__ __forceinline__ bool wide_window(const AggArgs& a, int64_t c) {
  return KC == 64 && a.rec_al16 && c + 1 < a.n_chunks;
}

template <int NT, int KC>
__device__ __forceinline__ void issue_records(const AggArgs& a, int64_t c, uint32_t* srec, int t, int RW) {
  if (KC == 64) {
    if (wide_window<KC>(a, c)) {
      const int64_t wstart = (c * RW * 4) & ~(int64_t)15;
      for (int i = t; i < a.R * 8; i += NT) {
        const int r = i < a.R ? i : (i - a.R) / 7, q = i < a.R ? 7 : (i - a.R) % 7;
        cp_async16(srec + r * 32 + q * 4, reinterpret_cast<const char*>(a.rec[r]) + wstart + 16 * q);
      }
    } else {
      for (int i = t; i < a.R * 8; i += NT) {
        const int r = i < a.R ? i : (i - a.R) / 7, q = i < a.R ? 7 : (i - a.R) % 7;
        const uint32_t* rec = a.rec[r] + c * RW;
        for (int w = (q + 5) & 7; w < RW; w += 8) cp_async4(srec + r * 32 + w, rec + w);
      }
    }
  } else {
    const int lane = t & 31, warp = t >> 5;
    for (int r = warp; r < a.R; r += NT / 32) {
      const uint32_t* rec = a.rec[r] + c * RW;
      for (int w = lane; w < RW; w += 32) cp_async4(srec + r * RW + w, rec + w);
    }
  }
}

// KC = 64: the default geometry (k = 64, 12-bit indices) with compile-time
// record layout; KC = 0: any geometry, read from the arguments
template <int C, bool BF16, int MODE, int KC>
struct Pipe {
  using K = PipeCfg<C>;
  static constexpr int NT = K::NT;

  const AggArgs& a;
  int2* acc;
  double* accd;
  float* dlt;
  uint16_t* spos;
  uint32_t* srec0;
  int bufw;
  int t;
  int64_t n, G;
  int64_t c;
  int4* ring;  // descriptors (first 16 B) of chunks c, c+G, c+2G, c+3G: slot = step & 3
  int4* tab;   // per record: F(S_lo) lo/hi words, F(S_hi) lo/hi words; bit 31 of a hi word = non-finite
  int2* erange;  // [buf]: min / max fp16 exponent field of the chunk's nonzero finite scales
  int it;      // step counter
  int buf;
  bool bad;

  // one chunk: `cur` holds chunk c's theta, `nxt` receives chunk c+G's
  __device__ __forceinline__ bool step(float (&cur)[4 * K::GPT], float (&nxt)[4 * K::GPT]) {
    const int RWc = KC ? (KC * 12 + 31) / 32 + (2 * KC + 31) / 32 + 1 : a.g.rec_words;
    const int64_t cn = c + G;
    const bool has_next = cn < n;
    // descriptors travel through shared memory by cp.async, three chunks ahead:
    // a register load would be consumed (uniform-register move) at once
#if SLC_AGG_THETA_NOW
    // theta of THIS chunk, loaded at the start of its step: its HBM latency hides
    // behind the chunk's own decode (passes 1-2), one register buffer suffices
    if (MODE == kFused) load_theta<C, BF16>(a.theta, unpack_desc(ring[it & 3]), t, cur);
    if (has_next) issue_records<NT, KC>(a, cn, srec0 + (buf ^ 1) * bufw, t, RWc);
#else
    if (has_next) {
      if (MODE == kFused) load_theta<C, BF16>(a.theta, unpack_desc(ring[(it + 1) & 3]), t, nxt);
      issue_records<NT, KC>(a, cn, srec0 + (buf ^ 1) * bufw, t, RWc);
    }
#endif
    if (t == 0 && cn + 2 * G < n) cp_async16(&ring[(it + 3) & 3], a.chunks + cn + 2 * G);
    cp_async_commit();
    const Desc d0 = unpack_desc(ring[it & 3]);

    const int SR = KC ? 32 : RWc;  // slot words
    const uint32_t* srec = srec0 + buf * bufw + (wide_window<KC>(a, c) ? (int)((29 * c) & 3) : 0);
    const int len = d0.len;
    const int kk = KC ? KC : a.g.k;
    const int ib = KC ? 12 : a.g.ib;
    const int IW = KC ? (KC * 12 + 31) / 32 : a.g.idx_words;
    const int RW = RWc;
    const int k_eff = max(1, (kk * len) / C);
    const int total = a.R * k_eff;
    cp_async_wait1();
    const bool owner = KC ? t < a.R : (t & 31) == (RW - 1) % 32;
    if (a.weighted && owner) {
      // weighted: the exact products w_r * S_b (35 significant bits) as M * 2^E,
      // M < 2^35; hi word = M >> 32 | (E + 1024) << 8 | sign(w) << 30
      int emin = 0x7FFFFFFF, emax = (int)0x80000000;
      for (int r = KC ? t : (t >> 5); r < a.R; r += KC ? NT : NT / 32) {
        const uint32_t sw = srec[r * SR + RW - 1];
        const float wf = (float)peer_weight(a, r);
        uint32_t fw[4];
#pragma unroll
        for (int b = 0; b < 2; b++) {
          const uint32_t h = (sw >> (16 * b)) & 0xFFFFu;
          const double d = __dmul_rn((double)wf, (double)__half2float(__ushort_as_half((unsigned short)h)));
          const unsigned long long db = (unsigned long long)__double_as_longlong(d);
          const int ed = (int)((db >> 52) & 0x7FF);
          unsigned long long M = 0;
          int E = 0;
          if (!isfinite(d) || ((h >> 10) & 0x1Fu) == 0x1Fu) {
            emax = 1 << 20;  // non-finite: this chunk takes the sequential path
          } else if (d != 0.0) {
            // |d| = (2^52 + frac) * 2^(ed - 1075) for normal d (products are never fp64-subnormal)
            M = ((db & 0xFFFFFFFFFFFFFull) | (1ull << 52)) >> 18;
            E = ed - 1075 + 18;
            if (M & ~((1ull << 35) - 1)) emax = 1 << 20;  // not a 35-bit product: sequential path
            emin = min(emin, E);
            emax = max(emax, E);
          }
          fw[2 * b] = (uint32_t)M;
          fw[2 * b + 1] = (uint32_t)(M >> 32) | ((uint32_t)(E + 1024) & 0xFFFu) << 8 | (wf < 0.0f ? 1u << 30 : 0u);
        }
        tab[r] = make_int4((int)fw[0], (int)fw[1], (int)fw[2], (int)fw[3]);
      }
      if (emin <= emax) {
        atomicMin(&erange[buf].x, emin);
        atomicMax(&erange[buf].y, emax);
      }
    }
    if (!a.weighted && owner) {
      // this thread copied the scale word of records r (issue_records), so it
      // may read them without a barrier: F = fp16 scale as a multiple of 2^-24
      int emin = 31, emax = 0;
      for (int r = KC ? t : (t >> 5); r < a.R; r += KC ? NT : NT / 32) {
        const uint32_t sw = srec[r * SR + RW - 1];
        uint32_t fw[4];
#pragma unroll
        for (int b = 0; b < 2; b++) {
          const uint32_t h = (sw >> (16 * b)) & 0xFFFFu;
          const int e = (int)((h >> 10) & 0x1Fu);
          const unsigned long long f = (unsigned long long)f16_fixed24(h);
          fw[2 * b] = (uint32_t)f;
          fw[2 * b + 1] = (uint32_t)(f >> 32) | (e == 31 ? 0x80000000u : 0u);
          if ((h & 0x7FFFu) != 0 && e < 31) {
            emin = min(emin, max(1, e));
            emax = max(emax, max(1, e));
          }
          if (e == 31) emax = 1 << 20;  // a non-finite scale: the chunk takes WIDE, which checks every entry
        }
        tab[r] = make_int4((int)fw[0], (int)fw[1], (int)fw[2], (int)fw[3]);
      }
      if (emin <= emax) {
        atomicMin(&erange[buf].x, emin);
        atomicMax(&erange[buf].y, emax);
      }
    }
    __syncthreads();  // chunk c's records and scale table visible; previous chunk's passes done

    // Per chunk, one of three accumulators (CTA-uniform choice):
    //  FAST  unit weights and every nonzero scale of the chunk within a
    //        2^(20 - ceil(log2 R)) range: each decoded value F * 2^-24 is
    //        F >> sh exactly (sh = min exponent - 1), and any sum of R of them
    //        fits an int32: one native atomic per entry, read back and
    //        re-zeroed by atomicExch
    //  WIDE  unit weights otherwise: the R#17 hi*2^20 + lo split over two int32
    //        arrays (acc, acc + C)
    //  WFAST weights, and the chunk's exact products w_r * S_b within a
    //        2^(17 - ceil(log2 R)) range: every partial sum of the oracle's
    //        fp64 canonical-order sum is then exact, so the order-free exact
    //        fixed-point sum (M << (E - Emin), split over two int32 arrays) is
    //        bitwise the same
    //  W     weights otherwise: fp64 in canonical peer order (one warp)
    int mode;  // 0 FAST, 1 WIDE, 2 W, 3 WFAST
    int sh = 0;
    const int rbits = a.R > 1 ? 32 - __clz(a.R - 1) : 0;  // ceil(log2 R)
    const int Lw = 31 - rbits;                            // WFAST lo/hi split
    if (a.weighted) {
      const int2 er = erange[buf];
      if (er.x > er.y) {
        mode = 3;  // every product is zero
        sh = 0;
      } else if (er.y - er.x + 35 + rbits <= 52) {
        mode = 3;
        sh = er.x;
      } else {
        mode = 2;
      }
    } else {
      const int2 er = erange[buf];
      if (er.x > er.y || er.y - er.x + 11 + rbits <= 31) {
        mode = 0;
        sh = er.x > er.y ? 0 : er.x - 1;
      } else {
        mode = 1;
      }
    }
    int* acc32 = reinterpret_cast<int*>(acc);
    const bool wtab = SLC_AGG_WTAB && mode == 3;  // CTA-uniform
    if (wtab) {
      // WFAST: each record's two signed summands (M << (E - Emin), split
      // lo / hi at Lw bits, the weight's sign applied) once per record here
      // instead of once per entry; then one barrier
      for (int r = t; r < a.R; r += NT) {
        const int4 tb = tab[r];
        const uint32_t fw[4] = {(uint32_t)tb.x, (uint32_t)tb.y, (uint32_t)tb.z, (uint32_t)tb.w};
        int out[4];
#pragma unroll
        for (int b = 0; b < 2; b++) {
          const uint32_t flo = fw[2 * b], fhi = fw[2 * b + 1];
          const unsigned long long M = ((unsigned long long)(fhi & 0xFFu) << 32) | flo;
          const int E = (int)((fhi >> 8) & 0xFFFu) - 1024;
          const unsigned long long v = M ? M << (E - sh) : 0ull;  // < 2^(52 - rbits)
          int lo = (int)(v & ((1ull << Lw) - 1)), hi = (int)(v >> Lw);
          if ((fhi >> 30) & 1u) { lo = -lo; hi = -hi; }
          out[2 * b] = lo;
          out[2 * b + 1] = hi;
        }
        tab[r] = make_int4(out[0], out[1], out[2], out[3]);
      }
      __syncthreads();
    }
    // FAST chunks with at least C/64 entries convert Delta in the dense pass
    // (C conversions there beat pass 2's per-entry work + barrier only when
    // enough positions are touched; CTA-uniform)
    const bool fuse = SLC_AGG_FUSE2 && mode == 0 && SLC_AGG_FUSE_MUL * total >= C;

    if (mode == 0 && k_eff == kk && (kk & 31) == 0) {
      // pass 1, FAST, full chunk: warp w takes 32-slot units (record r, slots
      // 32h..32h+31) with lane-constant bit offsets
      const int KW = kk >> 5, lane = t & 31;
      const int wl = (ib * lane) >> 5, shl = (ib * lane) & 31;
      const int cw = IW + (lane >> 4), csh = 2 * (lane & 15);
      const uint32_t imask = (1u << ib) - 1u;
      const bool check_p = (1 << ib) > len;
      SLC_UNROLL(SLC_AGG_UNROLL)
      for (int u = t >> 5; u < a.R * KW; u += NT / 32) {
        const int r = u / KW;
        const int h = u - r * KW;
        const uint32_t* rec = srec + r * SR;
        uint32_t p = __funnelshift_r(rec[ib * h + wl], rec[ib * h + wl + 1], shl) & imask;
        const uint32_t code = (rec[cw + 2 * h] >> csh) & 3u;
        const int4 tb = tab[r];
        const bool hb = (code & 2u) != 0;
        const uint32_t flo = (uint32_t)(hb ? tb.z : tb.x), fhi = (uint32_t)(hb ? tb.w : tb.y);
        int v = (int)__funnelshift_r(flo, fhi, sh);  // F >> sh, exact (FAST chunks have finite scales)
        if (check_p && (int)p >= len) {
          p = 0;
          v = 0;
          bad = true;
        }
        if (code & 1u) v = -v;
        if (!fuse) spos[r * kk + 32 * h + lane] = (uint16_t)p;
        atomicAdd(&acc32[p], v);
      }
    } else if (mode != 2) {
      // pass 1: every entry into the exact accumulator; remember its position.
      // Full chunks: warp w takes 32-slot units (record r, slots 32h..32h+31)
      // with lane-constant bit offsets; partial chunks walk entries.
      const bool full = k_eff == kk && (k_eff & 31) == 0;
      const int KW = k_eff >> 5, lane = t & 31;
      const int wl = (ib * lane) >> 5, shl = (ib * lane) & 31;
      const uint32_t imask = (1u << ib) - 1u;
      const bool check_p = (1 << ib) > len;
      const int n_iter = full ? a.R * KW : total;
      for (int u = full ? (t >> 5) : t; u < n_iter; u += full ? NT / 32 : NT) {
        int r, s;
        uint32_t p, code;
        if (full) {
          r = KW == 2 ? (u >> 1) : u / KW;
          const int h = u - r * KW;
          const uint32_t* rec = srec + r * SR;
          p = __funnelshift_r(rec[ib * h + wl], rec[ib * h + wl + 1], shl) & imask;
          code = (rec[IW + 2 * h + (lane >> 4)] >> (2 * (lane & 15))) & 3u;
          s = r * k_eff + 32 * h + lane;
        } else {
          s = u;
          r = s / k_eff;
          const int j = s - r * k_eff;
          const uint32_t* rec = srec + r * SR;
          p = rec_index(rec, j, ib);
          code = (rec[IW + (j >> 4)] >> (2 * (j & 15))) & 3u;
        }
        const int4 tb = tab[r];
        const uint32_t flo = (uint32_t)((code & 2u) ? tb.z : tb.x);
        const uint32_t fhi = (uint32_t)((code & 2u) ? tb.w : tb.y);
        const bool ok = (wtab || !(fhi >> 31)) && !(check_p && (int)p >= len);
        bad |= !ok;
        if (!ok) p = 0;
        spos[s] = (uint16_t)p;
        if (mode == 0) {
          int v = ok ? (int)__funnelshift_r(flo, fhi, sh) : 0;  // F >> sh, exact
          if (code & 1u) v = -v;
          atomicAdd(&acc32[p], v);
        } else if (wtab) {
          int lo = ok ? (int)flo : 0, hi = ok ? (int)fhi : 0;
          if (code & 1u) { lo = -lo; hi = -hi; }
          atomicAdd(&acc32[p], lo);
          atomicAdd(&acc32[C + p], hi);
        } else if (mode == 3) {
          const unsigned long long M = ((unsigned long long)(fhi & 0xFFu) << 32) | flo;
          const int E = (int)((fhi >> 8) & 0xFFFu) - 1024;
          const unsigned long long v = (ok && M) ? M << (E - sh) : 0ull;  // < 2^(52 - rbits)
          int lo = (int)(v & ((1ull << Lw) - 1)), hi = (int)(v >> Lw);
          if (((code & 1u) != 0) != (((fhi >> 30) & 1u) != 0)) { lo = -lo; hi = -hi; }
          atomicAdd(&acc32[p], lo);
          atomicAdd(&acc32[C + p], hi);
        } else {
          int lo = ok ? (int)(flo & 0xFFFFFu) : 0, hi = ok ? (int)__funnelshift_r(flo, fhi, 20) : 0;
          if (code & 1u) { lo = -lo; hi = -hi; }
          atomicAdd(&acc32[p], lo);
          atomicAdd(&acc32[C + p], hi);
        }
      }
    } else {
      for (int s = t; s < total; s += NT) {
        const int r = k_eff == 64 ? (s >> 6) : s / k_eff;
        const uint32_t p = rec_index(srec + r * SR, s - r * k_eff, ib);
        spos[s] = (int)p < len ? (uint16_t)p : (uint16_t)0;
      }
      if (t < 32) {
        for (int i = 0; i < a.R; i++) {  // canonical peer order (host-sorted)
          const uint32_t* rec = srec + i * SR;
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
    }
    __syncthreads();  // scatter complete
    if (t == 0) erange[buf] = make_int2(0x7FFFFFFF, (int)0x80000000);  // read by every thread before the barrier above

    // pass 2: Delta only at touched positions; untouched dlt stay +0.  The
    // oracle's Delta = (float)(acc * invR) with acc = V * 2^(sh-24) exactly,
    // and 2^(sh-24) * invR is exact, so one fp64 product and one fp32 rounding.
    const double invR = a.invR;
    // FAST: 2^(sh-24) * invR, exact
    const double cs = __dmul_rn(invR, __longlong_as_double((long long)(1023 + sh - 24) << 52));
    if (fuse) {
      // FAST with the conversion folded into the dense pass: no pass 2, no
      // barrier, no entry positions — the dense pass reads the int32 sums
    } else if (mode == 0) {
      SLC_UNROLL(SLC_AGG_UNROLL)
      for (int s = t; s < total; s += NT) {
        const int p = spos[s];
        const int v = atomicExch(&acc32[p], 0);  // exactly one entry of p sees the sum
        if (v != 0) dlt[p] = __double2float_rn(__dmul_rn((double)v, cs));
      }
    } else if (mode == 1) {
      const double c24 = invR * 0x1p-24;
      for (int s = t; s < total; s += NT) {
        const int p = spos[s];
        // exact: hi*2^20 + lo (|.| < 2^53) is representable; duplicates write the same value
        const double sd = __fma_rn((double)acc32[C + p], 0x1p20, (double)acc32[p]);
        dlt[p] = sd == 0.0 ? 0.0f : __double2float_rn(__dmul_rn(sd, c24));
      }
    } else if (mode == 3) {
      // acc = (hi * 2^Lw + lo) * 2^Emin exactly (|.| < 2^52 before the exact scaling)
      const double ce = __longlong_as_double((long long)(1023 + sh) << 52);
      const double cl = __longlong_as_double((long long)(1023 + Lw) << 52);
      for (int s = t; s < total; s += NT) {
        const int p = spos[s];
        const double sd = __fma_rn((double)acc32[C + p], cl, (double)acc32[p]);
        dlt[p] = sd == 0.0 ? 0.0f : __double2float_rn(__dmul_rn(__dmul_rn(sd, ce), invR));
      }
    } else {
      for (int s = t; s < total; s += NT) {
        const int p = spos[s];
        dlt[p] = __double2float_rn(__dmul_rn(accd[p], invR));
      }
    }
    if (!fuse) __syncthreads();  // Delta complete

    // pass 3: dense, untouched positions hold +0 (fused FAST: Delta of each
    // nonzero sum here, RN32(RN64(V * cs)) as in pass 2; the sums re-zeroed)
    const float alpha = a.alpha;
    auto delta4 = [&](int qq, float (&dl)[4]) {
      if (fuse) {
        int4* a4 = reinterpret_cast<int4*>(acc32) + qq;
        const int4 av = *a4;
        *a4 = make_int4(0, 0, 0, 0);
        const int vv[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
        // a zero sum gives +0 (cs > 0), as the untouched dlt of pass 2 does
        for (int j = 0; j < 4; j++) dl[j] = __double2float_rn(__dmul_rn((double)vv[j], cs));
      } else {
        float4* d4 = reinterpret_cast<float4*>(dlt) + qq;
        const float4 dv = *d4;
        *d4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        dl[0] = dv.x; dl[1] = dv.y; dl[2] = dv.z; dl[3] = dv.w;
      }
    };
    if (len == C) {
      int64_t o, stp;
      full_addr<C>(d0, t, o, stp);
#pragma unroll
      for (int v = 0; v < K::GPT; v++) {
        float dl[4];
        delta4(v * NT + t, dl);
        if (MODE == kAggOnly) {
          store_f32x4(a.agg, o + v * stp, 4, dl);
        } else {
          float th[4];
#pragma unroll
          for (int j = 0; j < 4; j++) th[j] = __fmaf_rn(-alpha, dl[j], cur[4 * v + j]);
          store_param4<BF16>(a.theta, o + v * stp, 4, th);
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < K::GPT; v++) {
        const int q = v * NT + t;
        float dl[4];
        delta4(q, dl);
        const int nv = valid_in_group(4 * q, len);
        if (nv == 0) continue;
        const int64_t off = generic_offset(d0, q, K::RPQ_SHIFT);
        if (MODE == kAggOnly) {
          store_f32x4(a.agg, off, nv, dl);
        } else {
          float th[4];
#pragma unroll
          for (int j = 0; j < 4; j++) th[j] = __fmaf_rn(-alpha, dl[j], cur[4 * v + j]);
          store_param4<BF16>(a.theta, off, nv, th);
        }
      }
    }
    // WIDE / W: the accumulator is re-zeroed where it was touched (the next
    // scatter follows a barrier); FAST re-zeroed it in pass 2
    if (mode == 1 || mode == 3) {
      for (int s = t; s < total; s += NT) {
        const int p = spos[s];
        acc32[p] = 0;
        acc32[C + p] = 0;
      }
    } else if (mode == 2) {
      for (int s = t; s < total; s += NT) accd[spos[s]] = 0.0;
    }

    c = cn;
    it++;
    buf ^= 1;
    return has_next;
  }
};

template <int C, bool BF16, int MODE, int KC>
__global__ void __launch_bounds__(PipeCfg<C>::NT, BF16 ? PipeCfg<C>::MIN_BLOCKS_BF16 : PipeCfg<C>::MIN_BLOCKS)
    agg_pipe_kernel(const AggArgs a) {
  using S = PipeSmem<C>;
  constexpr int NT = PipeCfg<C>::NT;
  extern __shared__ __align__(16) unsigned char smem[];
  const int t = threadIdx.x;
  Pipe<C, BF16, MODE, KC> P{a};
  P.acc = reinterpret_cast<int2*>(smem + S::off_acc);
  P.accd = reinterpret_cast<double*>(smem + S::off_acc);
  P.dlt = reinterpret_cast<float*>(smem + S::off_dlt);
  P.spos = reinterpret_cast<uint16_t*>(smem + S::off_pos);
  const int SR = KC ? 32 : a.g.rec_words;
  P.srec0 = reinterpret_cast<uint32_t*>(smem + S::off_rec(a.R, a.g.k));
  P.bufw = rec_buf_words(a.R, SR);
  P.t = t;
  P.n = a.n_chunks;
  P.G = gridDim.x;
  P.c = blockIdx.x;
  P.buf = 0;
  P.it = 0;
  P.bad = false;
  P.ring = reinterpret_cast<int4*>(smem + S::off_desc(a.R, a.g.k, SR));
  P.tab = reinterpret_cast<int4*>(smem + S::off_tab(a.R, a.g.k, SR));
  P.erange = reinterpret_cast<int2*>(smem + S::off_erange(a.R, a.g.k, SR));
  if (P.c >= P.n) return;

  for (int i = t; i < C / 2; i += NT) reinterpret_cast<int4*>(P.acc)[i] = make_int4(0, 0, 0, 0);
  for (int i = t; i < C / 4; i += NT) reinterpret_cast<float4*>(P.dlt)[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (t < 2) P.srec0[t * P.bufw + a.R * SR] = 0u;  // rec_index may read one word past the last record

  if (t < 2) P.erange[t] = make_int2(0x7FFFFFFF, (int)0x80000000);
  if (t < 3 && P.c + t * P.G < P.n) P.ring[t] = __ldg(reinterpret_cast<const int4*>(a.chunks + P.c + t * P.G));
  __syncthreads();
  float thA[4 * PipeCfg<C>::GPT];
#if !SLC_AGG_THETA_NOW
  float thB[4 * PipeCfg<C>::GPT];
#endif
#if !SLC_AGG_THETA_NOW
  if (MODE == kFused) load_theta<C, BF16>(a.theta, unpack_desc(P.ring[0]), t, thA);
#endif
  issue_records<NT, KC>(a, P.c, P.srec0, t, a.g.rec_words);
  cp_async_commit();

#if SLC_AGG_THETA_NOW
  for (;;)
    if (!P.step(thA, thA)) break;
#else
  for (;;) {
    if (!P.step(thA, thB)) break;
    if (!P.step(thB, thA)) break;
  }
#endif
  if (P.bad) atomicOr(a.err, kErrNonFinite);
}

template <int C, bool BF16, int MODE>
cudaError_t launch_pipe(const AggArgs& a, cudaStream_t s) {
  if (a.R > kMaxPeers) return cudaErrorInvalidValue;
  const bool fixed = a.g.k == 64 && a.g.ib == 12;
  auto kern = fixed ? agg_pipe_kernel<C, BF16, MODE, 64> : agg_pipe_kernel<C, BF16, MODE, 0>;
  const size_t smem = PipeSmem<C>::bytes(a.R, a.g.k, fixed ? 32 : a.g.rec_words);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PipeCfg<C>::NT, smem)) != cudaSuccess)
    return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = std::min<int64_t>(a.n_chunks, (int64_t)sms * per_sm);
  // SLC_OPT_AGG_GRID_CAP: every CTA walks many chunks (pipeline hand-offs under test)
  if (a.grid_cap > 0) grid = std::min<int64_t>(grid, a.grid_cap);
  kern<<<(unsigned)grid, PipeCfg<C>::NT, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool aggregate_pipe_supported(const AggArgs& a) {
  if (a.g.C != 1024 && a.g.C != 4096) return false;
  const int SR = (a.g.k == 64 && a.g.ib == 12) ? 32 : a.g.rec_words;
  const size_t smem = a.g.C == 1024 ? PipeSmem<1024>::bytes(a.R, a.g.k, SR) : PipeSmem<4096>::bytes(a.R, a.g.k, SR);
  return smem <= 200 * 1024;  // leaves room for 1 CTA per SM with any driver reservation
}

cudaError_t launch_aggregate_pipe(const AggArgs& a, int bf16, cudaStream_t s) {
  if (a.n_chunks == 0) return cudaSuccess;
  if (a.mode != kFused && a.mode != kAggOnly) return cudaErrorInvalidValue;
  const bool fused = a.mode == kFused;
  switch (a.g.C) {
    case 1024:
      if (fused) return bf16 ? launch_pipe<1024, true, kFused>(a, s) : launch_pipe<1024, false, kFused>(a, s);
      return launch_pipe<1024, false, kAggOnly>(a, s);
    case 4096:
      if (fused) return bf16 ? launch_pipe<4096, true, kFused>(a, s) : launch_pipe<4096, false, kFused>(a, s);
      return launch_pipe<4096, false, kAggOnly>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace slc
