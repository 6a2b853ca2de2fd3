// slc_internal.cuh — shared declarations of libslc (host plan + CUDA kernels).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include <vector>

#include "../../include/slc.h"

namespace slc {

constexpr int kMaxPeers = 256;
constexpr int kMaxK = 256;

// One chunk of the shard: dense position p of the chunk lives at shard element
//   base + (p / B) * ld + (p % B)   (blocked, ld = tensor cols)
//   base + p                        (flat,    ld = 0)
// len = number of positions (C, or less for the last chunk of a flat tensor).
// Blocked chunks also carry their TMA coordinates: tensor map triple `tmap`
// (theta, theta_local, e of the chunk's segment) and the block's (col, row).
struct __align__(16) ChunkDesc {
  int64_t base;
  int32_t ld;
  int32_t len;
  int32_t tmap;  // -1: flat chunk
  int32_t tx, ty;
  int32_t pad;
};
static_assert(sizeof(ChunkDesc) == 32, "ChunkDesc must be 32 bytes");

// Error bits latched on the device.
enum : uint32_t { kErrNonFinite = 1u, kErrScaleOverflow = 2u };

struct Geom {
  int B, C, k, ib;
  int idx_words, code_words, rec_words;
};

#ifdef SLC_CHECKED  // debug builds: bounds-checked kernels
#define SLC_CHECK(cond, what)                                                                          \
  do {                                                                                                 \
    if (!(cond)) {                                                                                     \
      printf("SLC_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x);                                                                             \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define SLC_CHECK(cond, what) \
  do {                        \
  } while (0)
#endif

struct CompressArgs {
  int64_t n_elems;    // shard buffer length (bounds checks in debug builds)
  int32_t n_tmaps;
  const void* tmaps;  // CUtensorMap[3 * blocked segments] (theta, theta_local, e), device memory
  const ChunkDesc* chunks;
  int64_t n_chunks;
  const void* theta;
  const void* theta_local;
  float* ef;
  uint32_t* records;
  uint32_t* err;
  float beta;
  int64_t max_ld;  // largest row length of a blocked chunk (32-bit in-chunk offsets if small)
  Geom g;
  // slc_compress_multi: n_extra more record buffers (device array of pointers,
  // e.g. NVLink peer memory) receive the same records at the same offsets
  const uint64_t* rec_extra;
  int n_extra;
  // compress_ws: chunks whose selection leaves the candidate path (more than
  // CAP candidates, or a non-finite value) are deferred to a second kernel.
  // defer[0] = count, defer[1] = fallback blocks done, defer[2] = next entry
  // to take (all zero between launches), defer[kDeferHdr ..] = defer_cap
  // chunk indices (relative to chunks), then defer_cap entries of kDeferInfo
  // words (warp_select.cuh stage_R).
  uint32_t* defer;
  int64_t defer_cap;
  int32_t defer_info;  // words per deferral info entry (defer_info_words)
};
constexpr int kMaxRecOut = 16;
constexpr int kDeferHdr = 4;
// compress_ws hand-off unit: quads (VPU = 1) when k exceeds a quarter of the
// 32 NP 16-position groups of a chunk (their maxima then give a weak T),
// else the groups (VPU = 4; the paper's C = 4096, k = 64)
inline int ws_vpu(const Geom& g) { return (g.C == 1024 || g.C == 4096) && 4 * g.k > 32 * (g.C / 512) ? 1 : 4; }
// deferral info entry: T, then one unit-mask ballot word per unit of a lane
inline int defer_info_words(const Geom& g) { return 1 + (g.C / 512) * 4 / ws_vpu(g); }
inline int64_t defer_words(const Geom& g, int64_t n_chunks) {
  return kDeferHdr + n_chunks * (1 + (int64_t)defer_info_words(g));
}

enum AggMode : int { kAggOnly = 0, kUpdateFromAgg = 1, kFused = 2 };

struct AggArgs {
  const ChunkDesc* chunks;
  int64_t n_chunks;
  const uint32_t* rec[kMaxPeers];  // per peer: this shard's records
  float w[kMaxPeers];              // per peer weight (weighted mode only)
  const float* wdev;               // weighted mode: device weights in the caller's peer order, or NULL (use w)
  int16_t worder[kMaxPeers];       // canonical position i -> caller's peer index (for wdev)
  int R;
  int rec_al16;  // every rec[r] is 16-byte aligned (enables 16-B record copies)
  int weighted;
  int mode;
  float alpha;
  double invR;
  float* agg;     // kAggOnly: out; kUpdateFromAgg: in
  void* theta;    // kUpdateFromAgg / kFused: in-out
  uint32_t* err;
  Geom g;
  int variant;       // SLC_OPT_AGG_KERNEL: 0 auto, 1 batched, 2 pipelined, 3 one CTA per chunk
  int64_t grid_cap;  // SLC_OPT_AGG_GRID_CAP: > 0 caps the persistent kernels' grid (test aid)
  const void* tmaps;  // fused update: CUtensorMap per blocked segment over theta (ChunkDesc.tmap)
  int tmaps_ok;       // tmaps valid for this call's theta (always 1 without blocked segments)
};

// f2 wire format (wire.cu)
struct WireArgs {
  const ChunkDesc* chunks;
  int64_t n_chunks;
  const int64_t* wire_off;  // per chunk: byte offset of its encoding from the shard's first chunk
  const uint32_t* rec;      // encode: records in
  uint8_t* wire;            // encode: bytes out
  const uint8_t* wire_in;   // decode: bytes in
  uint32_t* rec_out;        // decode: records out
  uint32_t* err;
  Geom g;
};
cudaError_t launch_wire(const WireArgs& a, bool encode, cudaStream_t s);

// row f4 (index_code.cu): colex rank of each chunk's index set (R#28)
bool index_rank_supported(const Geom& g);
size_t binom_table_bytes(const Geom& g);
cudaError_t build_binom_table(uint32_t* T, const Geom& g, cudaStream_t s);
cudaError_t launch_index_rank(const ChunkDesc* chunks, int64_t n_chunks, const uint32_t* rec, const uint32_t* T,
                              uint32_t* ranks, const Geom& g, cudaStream_t s);
// entropy-coded records (R#28): rank limbs + code words + scale word
int ec_record_words(const Geom& g);
cudaError_t launch_index_encode(const ChunkDesc* chunks, int64_t n_chunks, const uint32_t* rec, const uint32_t* T,
                                uint32_t* ec, const Geom& g, cudaStream_t s);
cudaError_t launch_index_decode(const ChunkDesc* chunks, int64_t n_chunks, const uint32_t* ec, const uint32_t* T,
                                uint32_t* rec, uint32_t* err, const Geom& g, cudaStream_t s);

// launchers (return cudaGetLastError())
cudaError_t launch_compress(const CompressArgs& a, int param_bf16, cudaStream_t s);
// one CTA per chunk, any compiled C (reference kernel for the pipelined one)
// one warp per chunk, no block-level synchronisation (C = 1024, 4096)
cudaError_t launch_compress_warp(const CompressArgs& a, int param_bf16, cudaStream_t s);
// persistent warp-specialised CTAs: stream warps + select warps (C = 1024, 4096)
cudaError_t launch_compress_ws(const CompressArgs& a, int param_bf16, cudaStream_t s);
// TMA producer warp + warp-per-chunk consumers (C = 4096, k = 64, 12-bit indices)
cudaError_t launch_compress_tma(const CompressArgs& a, int param_bf16, cudaStream_t s);
bool compress_tma_supported(const Geom& g);
cudaError_t launch_aggregate(const AggArgs& a, int param_bf16, cudaStream_t s);
// persistent software-pipelined decode / fused update (C = 1024, 4096)
cudaError_t launch_aggregate_pipe(const AggArgs& a, int param_bf16, cudaStream_t s);
bool aggregate_pipe_supported(const AggArgs& a);
// contiguous chunk ranges, bulk-copied record batches, value tables (C = 4096, k = 64, 12-bit, R <= 64)
cudaError_t launch_aggregate_batch(const AggArgs& a, int param_bf16, cudaStream_t s);
bool aggregate_batch_supported(const AggArgs& a);
// median-norm: exact per-peer squared norms as 4 un-carried 32-bit limbs per peer; weights
cudaError_t launch_payload_sqnorm(const AggArgs& a, unsigned long long* out, cudaStream_t s);
cudaError_t launch_median_weights(const unsigned long long* limbs, int R, float* w, double* norms, cudaStream_t s);
// f2 fast checks: finite / norm-sane per peer on the device, host flags ORed in
cudaError_t launch_fast_checks(const AggArgs& a, const uint32_t* hflags, double thresh,
                               const unsigned long long* limbs, uint32_t* flags, cudaStream_t s);

#ifdef __CUDACC__
// weight of canonical peer i (weighted mode)
__device__ __forceinline__ double peer_weight(const AggArgs& a, int i) {
  return (double)(a.wdev ? __ldg(a.wdev + a.worder[i]) : a.w[i]);
}
#endif
bool compress_supported(int C);
// a8 / a9 over NVLink peer memory: copy up to kMaxPeers byte ranges in one kernel
cudaError_t launch_peer_copy(const void* const* src, void* const* dst, const int64_t* bytes, int n, void* dev_scratch,
                             cudaStream_t s);
size_t peer_copy_scratch_bytes();

}  // namespace slc
