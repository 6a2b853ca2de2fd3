// plan.cpp — host side of libslc: geometry validation, FSDP-style shard
// partition (R#11), per-chunk table, payload-header checks, error
// latch and the C-ABI entry points declared in include/slc.h.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "slc_internal.cuh"

using slc::ChunkDesc;

struct slc_plan {
  slc_geometry geom;
  slc::Geom g;
  slc_dtype dtype;
  int device;
  int rank, nranks;
  std::vector<slc_tensor> layout;
  std::vector<slc_segment> segs;
  int64_t total_elems = 0, total_chunks = 0, first_chunk = 0, n_chunks = 0, shard_elems = 0;
  int64_t max_ld = 0;  // largest row length of a blocked segment
  ChunkDesc* d_chunks = nullptr;
  uint32_t* d_err = nullptr;
  // TMA: one (theta, theta_local, e) tensor-map triple per blocked segment,
  // encoded for the buffers of the last slc_compress call
  std::vector<int> blk_segs;  // index into segs
  std::vector<CUtensorMap> h_tmaps;
  CUtensorMap* d_tmaps = nullptr;
  const void* tmap_ptrs[3] = {nullptr, nullptr, nullptr};
  // fused outer update: one tensor map per blocked segment over theta (tiles in / out)
  std::vector<CUtensorMap> h_utmaps;
  CUtensorMap* d_utmaps = nullptr;
  const void* utmap_ptr = nullptr;
  slc_status latched = SLC_OK;
  uint8_t digest[32];
  // f2 wire format: per-chunk byte offsets of the shard's encodings, their
  // total, and the offset of the shard's first encoding in the message body
  int64_t* d_wire_off = nullptr;
  int64_t wire_bytes = 0, wire_offset = 0;
  // f4 index code: binomial table binom(p, j), built by slc_plan_set_option(SLC_OPT_INDEX_CODE)
  uint32_t* d_binom = nullptr;
  // slc_compress_multi: device array of the extra record destinations
  uint64_t* d_rec_extra = nullptr;
  int n_extra_next = 0;
  void* d_pc_scratch = nullptr;  // slc_peer_copy's segment table
  uint32_t* d_defer = nullptr;   // compress: deferred-chunk list (count, blocks done, chunk ids)
  // slc_plan_set_option
  int agg_variant = 0;
  int64_t agg_grid_cap = 0;
  // stream of the most recent compute call (slc_get_status(synchronize) waits on it)
  cudaStream_t last_stream = nullptr;
};

namespace {

int64_t numel(const slc_tensor& t) {
  int64_t n = 1;
  for (int i = 0; i < t.ndim; i++) n *= t.dims[i];
  return n;
}

bool blocked(const slc_tensor& t, int B) { return t.ndim == 2 && t.dims[0] % B == 0 && t.dims[1] % B == 0; }

int64_t tensor_chunks(const slc_tensor& t, const slc_geometry& g) {
  if (blocked(t, g.block)) return (t.dims[0] / g.block) * (t.dims[1] / g.block);
  return (numel(t) + g.chunk - 1) / g.chunk;
}

slc_status check_geom(const slc_geometry* g) {
  if (!g) return SLC_ERR_INVALID_ARGUMENT;
  if (g->block <= 0 || g->block > 1024 || g->chunk != g->block * g->block) return SLC_ERR_INVALID_ARGUMENT;
  if (g->k < 1 || g->k > g->chunk || g->k > slc::kMaxK) return SLC_ERR_INVALID_ARGUMENT;
  if (g->index_bits < 1 || g->index_bits > 16 || (1L << g->index_bits) < g->chunk) return SLC_ERR_INVALID_ARGUMENT;
  return SLC_OK;
}

slc::Geom make_geom(const slc_geometry& g) {
  slc::Geom r;
  r.B = g.block;
  r.C = g.chunk;
  r.k = g.k;
  r.ib = g.index_bits;
  r.idx_words = (g.k * g.index_bits + 31) / 32;
  r.code_words = (2 * g.k + 31) / 32;
  r.rec_words = r.idx_words + r.code_words + 1;
  return r;
}

uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31;
  return z;
}

void digest_of(const slc_geometry& g, const slc_tensor* lay, int n, uint8_t out[32]) {
  uint64_t h[4] = {0x5EED0001ull, 0x5EED0002ull, 0x5EED0003ull, 0x5EED0004ull};
  auto feed = [&](uint64_t v) {
    for (int i = 0; i < 4; i++) h[i] = mix64(h[i] ^ (v + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1)));
  };
  feed((uint64_t)g.block); feed((uint64_t)g.chunk); feed((uint64_t)g.k); feed((uint64_t)g.index_bits);
  feed((uint64_t)n);
  for (int t = 0; t < n; t++) {
    feed((uint64_t)lay[t].ndim);
    for (int d = 0; d < lay[t].ndim; d++) feed((uint64_t)lay[t].dims[d]);
  }
  for (int i = 0; i < 4; i++)
    for (int b = 0; b < 8; b++) out[8 * i + b] = (uint8_t)(h[i] >> (8 * b));
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Partition (R#11): cut points are element positions in the global flat order
// that fall on unit boundaries (unit = block-row of a blocked tensor, chunk of
// a flat tensor), each the boundary nearest to g*total/nranks.
std::vector<int64_t> cut_points(const std::vector<slc_tensor>& lay, const slc_geometry& g, int nranks,
                                int64_t total) {
  std::vector<int64_t> cuts(nranks + 1, 0);
  cuts[nranks] = total;
  for (int r = 1; r < nranks; r++) {
    const long double target = (long double)total * r / nranks;
    int64_t best = 0;
    long double best_d = -1;
    int64_t off = 0;
    for (const auto& t : lay) {
      const int64_t n = numel(t);
      if (target >= off && target <= off + n) {
        int64_t unit = blocked(t, g.block) ? (int64_t)g.block * t.dims[1] : (int64_t)g.chunk;
        int64_t i = (int64_t)((target - off) / unit);
        for (int64_t cand_i : {i, i + 1}) {
          int64_t pos = off + std::min(cand_i * unit, n);
          long double d = pos > target ? pos - target : target - pos;
          if (best_d < 0 || d < best_d) { best_d = d; best = pos; }
        }
      }
      off += n;
    }
    cuts[r] = best;
  }
  for (int r = 1; r <= nranks; r++) cuts[r] = std::max(cuts[r], cuts[r - 1]);
  return cuts;
}

slc_status header_checks(const slc_plan* p, const slc_payload_hdr* h, int R, std::vector<int>& order) {
  order.resize(R);
  for (int r = 0; r < R; r++) order[r] = r;
  if (!h) return SLC_OK;
  for (int r = 0; r < R; r++) {
    if (std::memcmp(h[r].magic, "SLC1", 4) != 0 || h[r].version != 1) return SLC_ERR_INVALID_ARGUMENT;
    if (h[r].first_chunk != p->first_chunk || h[r].n_chunks != p->n_chunks) return SLC_ERR_INVALID_ARGUMENT;
    if (std::memcmp(&h[r].geom, &p->geom, sizeof(slc_geometry)) != 0) return SLC_ERR_STALE;
    if (std::memcmp(h[r].layout_digest, p->digest, 32) != 0) return SLC_ERR_STALE;
    if (h[r].base_round != h[0].base_round) return SLC_ERR_STALE;
  }
  std::sort(order.begin(), order.end(),
            [&](int a, int b) { return std::memcmp(h[a].peer_id, h[b].peer_id, 16) < 0; });
  for (int i = 1; i < R; i++)
    if (std::memcmp(h[order[i - 1]].peer_id, h[order[i]].peer_id, 16) == 0) return SLC_ERR_INVALID_ARGUMENT;
  return SLC_OK;
}

slc_status prep_agg(slc_plan* p, const slc_payload_hdr* hdrs, const void* const* recs, int R, const float* w,
                    slc::AggArgs& a) {
  if (R < 1 || R > slc::kMaxPeers || !recs) return SLC_ERR_INVALID_ARGUMENT;
  std::vector<int> order;
  slc_status st = header_checks(p, hdrs, R, order);
  if (st != SLC_OK) return st;
  std::memset(&a, 0, sizeof(a));
  a.chunks = p->d_chunks;
  a.n_chunks = p->n_chunks;
  a.R = R;
  a.weighted = w != nullptr;
  a.invR = 1.0 / (double)R;
  a.rec_al16 = 1;
  a.err = p->d_err;
  a.g = p->g;
  a.variant = p->agg_variant;
  a.grid_cap = p->agg_grid_cap;
  for (int i = 0; i < R; i++) {
    const int r = order[i];  // canonical order (matters only when weighted)
    if (!recs[r] && p->n_chunks > 0) return SLC_ERR_INVALID_ARGUMENT;
    if (((uintptr_t)recs[r]) & 3u) return SLC_ERR_INVALID_ARGUMENT;
    a.rec[i] = static_cast<const uint32_t*>(recs[r]);
    if (((uintptr_t)recs[r]) & 15u) a.rec_al16 = 0;
    a.w[i] = w ? w[r] : 1.0f;
    a.worder[i] = (int16_t)r;
  }
  return SLC_OK;
}

slc_status cuda_status(cudaError_t e, slc_plan* p) {
  if (e == cudaSuccess) return SLC_OK;
  p->latched = SLC_ERR_CUDA;
  if (std::getenv("SLC_DEBUG")) std::fprintf(stderr, "libslc: CUDA error %d: %s\n", (int)e, cudaGetErrorString(e));
  return SLC_ERR_CUDA;
}

bool aligned16(const void* q) { return (((uintptr_t)q) & 15u) == 0; }

cudaStream_t use_stream(slc_plan* p, void* stream) {
  p->last_stream = static_cast<cudaStream_t>(stream);
  return p->last_stream;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// (re)encode the 64x64-box tensor maps of every blocked segment for these buffers
cudaError_t ensure_tmaps(slc_plan* p, const void* theta, const void* theta_local, const float* ef,
                         cudaStream_t stream) {
  if (p->blk_segs.empty()) return cudaSuccess;
  if (p->tmap_ptrs[0] == theta && p->tmap_ptrs[1] == theta_local && p->tmap_ptrs[2] == ef) return cudaSuccess;
  PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const int B = p->geom.block;
  const int pb = p->dtype == SLC_BF16 ? 2 : 4;
  const void* bufs[3] = {theta, theta_local, ef};
  for (size_t i = 0; i < p->blk_segs.size(); i++) {
    const slc_segment& s = p->segs[p->blk_segs[i]];
    for (int a = 0; a < 3; a++) {
      const int esz = a < 2 ? pb : 4;
      const CUtensorMapDataType dt = esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
      char* base = (char*)bufs[a] + (size_t)s.shard_offset * esz;
      const cuuint64_t dims[2] = {(cuuint64_t)s.cols, (cuuint64_t)s.rows};
      const cuuint64_t strides[1] = {(cuuint64_t)s.cols * esz};
      const cuuint32_t box[2] = {(cuuint32_t)B, (cuuint32_t)B};
      const cuuint32_t estr[2] = {1, 1};
      CUresult r = enc(&p->h_tmaps[3 * i + a], dt, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
  }
  cudaError_t e = cudaMemcpyAsync(p->d_tmaps, p->h_tmaps.data(), p->h_tmaps.size() * sizeof(CUtensorMap),
                                  cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return e;
  p->tmap_ptrs[0] = theta;
  p->tmap_ptrs[1] = theta_local;
  p->tmap_ptrs[2] = ef;
  return cudaSuccess;
}

// (re)encode the 64x64-box tensor maps over theta of every blocked segment
// (the fused update's tile loads / stores); cached per theta pointer
cudaError_t ensure_update_tmaps(slc_plan* p, const void* theta, cudaStream_t stream) {
  if (p->blk_segs.empty() || p->utmap_ptr == theta) return cudaSuccess;
  PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const int B = p->geom.block;
  const int esz = p->dtype == SLC_BF16 ? 2 : 4;
  const CUtensorMapDataType dt = esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  for (size_t i = 0; i < p->blk_segs.size(); i++) {
    const slc_segment& s = p->segs[p->blk_segs[i]];
    char* base = (char*)theta + (size_t)s.shard_offset * esz;
    const cuuint64_t dims[2] = {(cuuint64_t)s.cols, (cuuint64_t)s.rows};
    const cuuint64_t strides[1] = {(cuuint64_t)s.cols * esz};
    const cuuint32_t box[2] = {(cuuint32_t)B, (cuuint32_t)B};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&p->h_utmaps[i], dt, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaMemcpyAsync(p->d_utmaps, p->h_utmaps.data(), p->h_utmaps.size() * sizeof(CUtensorMap),
                                  cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return e;
  p->utmap_ptr = theta;
  return cudaSuccess;
}

// the fused update's theta tensor maps for this call (falls back to the other
// kernels, tmaps_ok = 0, if they cannot be encoded)
void set_update_tmaps(slc_plan* p, const void* theta, cudaStream_t stream, slc::AggArgs& a) {
  if (p->blk_segs.empty()) {
    a.tmaps = nullptr;
    a.tmaps_ok = 1;
    return;
  }
  const bool ok = ((uintptr_t)theta & 15u) == 0 && ensure_update_tmaps(p, theta, stream) == cudaSuccess;
  if (!ok) cudaGetLastError();
  a.tmaps = p->d_utmaps;
  a.tmaps_ok = ok ? 1 : 0;
}

}  // namespace

extern "C" {

int64_t slc_record_bytes(const slc_geometry* g) {
  if (check_geom(g) != SLC_OK) return -1;
  return 4 * (int64_t)make_geom(*g).rec_words;
}

slc_status slc_layout_digest(const slc_geometry* g, const slc_tensor* lay, int32_t n, uint8_t out[32]) {
  if (check_geom(g) != SLC_OK || !lay || n < 1 || !out) return SLC_ERR_INVALID_ARGUMENT;
  digest_of(*g, lay, n, out);
  return SLC_OK;
}

slc_status slc_plan_create(const slc_geometry* geom, const slc_tensor* layout, int32_t n_tensors, int32_t rank,
                           int32_t nranks, slc_dtype dtype, int32_t device, slc_plan** out) {
  if (!out) return SLC_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  slc_status st = check_geom(geom);
  if (st != SLC_OK) return st;
  if (!layout || n_tensors < 1 || nranks < 1 || rank < 0 || rank >= nranks) return SLC_ERR_INVALID_ARGUMENT;
  if (dtype != SLC_F32 && dtype != SLC_BF16) return SLC_ERR_INVALID_ARGUMENT;
  if (!slc::compress_supported(geom->chunk)) return SLC_ERR_UNSUPPORTED;
  for (int t = 0; t < n_tensors; t++) {
    if (layout[t].ndim < 1 || layout[t].ndim > 4) return SLC_ERR_INVALID_ARGUMENT;
    for (int d = 0; d < layout[t].ndim; d++)
      if (layout[t].dims[d] < 1) return SLC_ERR_INVALID_ARGUMENT;
    if (blocked(layout[t], geom->block) && layout[t].dims[1] > INT32_MAX) return SLC_ERR_INVALID_ARGUMENT;
  }

  slc_plan* p = new (std::nothrow) slc_plan();
  if (!p) return SLC_ERR_INVALID_ARGUMENT;
  p->geom = *geom;
  p->g = make_geom(*geom);
  p->dtype = dtype;
  p->device = device;
  p->rank = rank;
  p->nranks = nranks;
  p->layout.assign(layout, layout + n_tensors);
  digest_of(*geom, layout, n_tensors, p->digest);

  for (const auto& t : p->layout) {
    p->total_elems += numel(t);
    p->total_chunks += tensor_chunks(t, *geom);
  }
  const std::vector<int64_t> cuts = cut_points(p->layout, *geom, nranks, p->total_elems);
  const int64_t lo = cuts[rank], hi = cuts[rank + 1];

  // segments of [lo, hi) and the chunk table
  std::vector<ChunkDesc> table;
  int64_t off = 0, chunk0 = 0, shard_off = 0;
  bool first_set = false;
  for (int ti = 0; ti < n_tensors; ti++) {
    const slc_tensor& t = p->layout[ti];
    const int64_t n = numel(t), nc = tensor_chunks(t, *geom);
    const int64_t b = std::max(lo, off), e = std::min(hi, off + n);
    if (b < e) {
      slc_segment s;
      std::memset(&s, 0, sizeof(s));
      s.tensor = ti;
      s.blocked = blocked(t, geom->block);
      s.tensor_begin = b - off;
      s.n_elems = e - b;
      s.shard_offset = (shard_off + 63) / 64 * 64;
      const int64_t B = geom->block, C = geom->chunk;
      if (s.blocked) {
        const int64_t cols = t.dims[1], nb = cols / B;
        const int64_t r0 = s.tensor_begin / cols, r1 = (s.tensor_begin + s.n_elems) / cols;
        s.rows = r1 - r0;
        s.cols = cols;
        p->max_ld = std::max(p->max_ld, cols);
        s.first_chunk = chunk0 + (r0 / B) * nb;
        s.n_chunks = (s.rows / B) * nb;
        for (int64_t bi = 0; bi < s.rows / B; bi++)
          for (int64_t bj = 0; bj < nb; bj++)
            table.push_back(ChunkDesc{s.shard_offset + bi * B * cols + bj * B, (int32_t)cols, (int32_t)C,
                                      (int32_t)p->blk_segs.size(), (int32_t)(bj * B), (int32_t)(bi * B), 0});
      } else {
        s.rows = s.n_elems;
        s.cols = 1;
        const int64_t c_first = s.tensor_begin / C;
        s.first_chunk = chunk0 + c_first;
        s.n_chunks = (s.n_elems + C - 1) / C;
        for (int64_t c = 0; c < s.n_chunks; c++) {
          const int64_t len = std::min(C, s.n_elems - c * C);
          table.push_back(ChunkDesc{s.shard_offset + c * C, 0, (int32_t)len, -1, 0, 0, 0});
        }
      }
      if (!first_set) { p->first_chunk = s.first_chunk; first_set = true; }
      shard_off = s.shard_offset + s.n_elems;
      if (s.blocked) p->blk_segs.push_back((int)p->segs.size());
      p->segs.push_back(s);
    }
    off += n;
    chunk0 += nc;
  }
  if (!first_set) {  // empty shard: first_chunk = chunks before lo
    int64_t c = 0, o = 0;
    for (const auto& t : p->layout) {
      if (o >= lo) break;
      c += tensor_chunks(t, *geom);
      o += numel(t);
    }
    p->first_chunk = c;
  }
  p->n_chunks = (int64_t)table.size();
  p->shard_elems = shard_off;
  // wire encodings: 6 + ceil(k_eff*ib/8) + ceil(2 k_eff/8) bytes per chunk
  auto wire_size = [&](int64_t len) {
    const int64_t ke = std::max<int64_t>(1, (int64_t)geom->k * len / geom->chunk);
    return 6 + (ke * geom->index_bits + 7) / 8 + (2 * ke + 7) / 8;
  };
  std::vector<int64_t> wire_off(table.size());
  for (size_t i = 0; i < table.size(); i++) {
    wire_off[i] = p->wire_bytes;
    p->wire_bytes += wire_size(table[i].len);
  }
  {
    int64_t c = 0;  // global chunks before first_chunk, tensor by tensor
    for (const auto& t : p->layout) {
      const int64_t nc = tensor_chunks(t, *geom);
      if (c >= p->first_chunk) break;
      const int64_t take = std::min(nc, p->first_chunk - c);
      if (blocked(t, geom->block)) {
        p->wire_offset += take * wire_size(geom->chunk);
      } else {
        const int64_t n = numel(t);
        for (int64_t q = 0; q < take; q++) p->wire_offset += wire_size(std::min<int64_t>(geom->chunk, n - q * geom->chunk));
      }
      c += take;
    }
  }

  if (device < 0) {  // host-only plan: geometry / partition queries, no compute
    *out = p;
    return SLC_OK;
  }
  DeviceGuard guard(device);
  cudaError_t ce = cudaMalloc(&p->d_err, sizeof(uint32_t));
  if (ce == cudaSuccess) ce = cudaMemset(p->d_err, 0, sizeof(uint32_t));
  if (ce == cudaSuccess && !p->blk_segs.empty()) {
    p->h_tmaps.resize(3 * p->blk_segs.size());
    ce = cudaMalloc(&p->d_tmaps, p->h_tmaps.size() * sizeof(CUtensorMap));
    p->h_utmaps.resize(p->blk_segs.size());
    if (ce == cudaSuccess) ce = cudaMalloc(&p->d_utmaps, p->h_utmaps.size() * sizeof(CUtensorMap));
  }
  if (ce == cudaSuccess && !table.empty()) {
    ce = cudaMalloc(&p->d_chunks, table.size() * sizeof(ChunkDesc));
    if (ce == cudaSuccess)
      ce = cudaMemcpy(p->d_chunks, table.data(), table.size() * sizeof(ChunkDesc), cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMalloc(&p->d_wire_off, wire_off.size() * sizeof(int64_t));
    if (ce == cudaSuccess) ce = cudaMalloc(&p->d_rec_extra, slc::kMaxRecOut * sizeof(uint64_t));
    if (ce == cudaSuccess) ce = cudaMalloc(&p->d_pc_scratch, slc::peer_copy_scratch_bytes());
    if (ce == cudaSuccess) ce = cudaMalloc(&p->d_defer, slc::defer_words(p->g, (int64_t)table.size()) * sizeof(uint32_t));
    if (ce == cudaSuccess) ce = cudaMemset(p->d_defer, 0, slc::kDeferHdr * sizeof(uint32_t));
    if (ce == cudaSuccess)
      ce = cudaMemcpy(p->d_wire_off, wire_off.data(), wire_off.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  }
  if (ce != cudaSuccess) {
    if (p->d_wire_off) cudaFree(p->d_wire_off);
    if (p->d_rec_extra) cudaFree(p->d_rec_extra);
    if (p->d_pc_scratch) cudaFree(p->d_pc_scratch);
    if (p->d_defer) cudaFree(p->d_defer);
    if (p->d_err) cudaFree(p->d_err);
    if (p->d_chunks) cudaFree(p->d_chunks);
    if (p->d_tmaps) cudaFree(p->d_tmaps);
    if (p->d_utmaps) cudaFree(p->d_utmaps);
    delete p;
    cudaGetLastError();
    return SLC_ERR_CUDA;
  }
  *out = p;
  return SLC_OK;
}

slc_status slc_plan_info_get(const slc_plan* p, slc_plan_info* o) {
  if (!p || !o) return SLC_ERR_INVALID_ARGUMENT;
  o->total_elems = p->total_elems;
  o->total_chunks = p->total_chunks;
  o->first_chunk = p->first_chunk;
  o->n_chunks = p->n_chunks;
  o->shard_elems = p->shard_elems;
  o->record_bytes = 4 * (int64_t)p->g.rec_words;
  o->payload_bytes = o->record_bytes * p->n_chunks;
  o->n_segments = (int32_t)p->segs.size();
  o->rank = p->rank;
  o->nranks = p->nranks;
  return SLC_OK;
}

slc_status slc_plan_segment(const slc_plan* p, int32_t i, slc_segment* o) {
  if (!p || !o || i < 0 || i >= (int32_t)p->segs.size()) return SLC_ERR_INVALID_ARGUMENT;
  *o = p->segs[i];
  return SLC_OK;
}

slc_status slc_compress(slc_plan* p, const void* theta, const void* theta_local, float* ef, float beta,
                        void* records, void* stream) {
  if (!p) return SLC_ERR_INVALID_ARGUMENT;
  return slc_compress_range(p, 0, p->n_chunks, theta, theta_local, ef, beta, records, stream);
}

slc_status slc_compress_multi(slc_plan* p, const void* theta, const void* theta_local, float* ef, float beta,
                              void* const* records_out, int32_t n_out, void* stream) {
  if (!p || p->device < 0 || !records_out || n_out < 1 || n_out > slc::kMaxRecOut) return SLC_ERR_INVALID_ARGUMENT;
  uint64_t h[slc::kMaxRecOut];
  for (int i = 1; i < n_out; i++) {
    if (!records_out[i] || (((uintptr_t)records_out[i]) & 3u)) return SLC_ERR_INVALID_ARGUMENT;
    h[i - 1] = (uint64_t)(uintptr_t)records_out[i];
  }
  if (n_out > 1 && p->n_chunks > 0) {
    DeviceGuard guard(p->device);
    // stream-ordered: the kernel below reads the pointers after this copy
    cudaError_t e = cudaMemcpyAsync(p->d_rec_extra, h, sizeof(uint64_t) * (n_out - 1), cudaMemcpyHostToDevice,
                                    static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_status(e, p);
  }
  p->n_extra_next = n_out - 1;
  const slc_status st = slc_compress_range(p, 0, p->n_chunks, theta, theta_local, ef, beta, records_out[0], stream);
  p->n_extra_next = 0;
  return st;
}

slc_status slc_compress_range(slc_plan* p, int64_t c0, int64_t nc, const void* theta, const void* theta_local,
                              float* ef, float beta, void* records, void* stream) {
  if (!p || p->device < 0) return SLC_ERR_INVALID_ARGUMENT;
  if (c0 < 0 || nc < 0 || c0 > p->n_chunks || nc > p->n_chunks - c0) return SLC_ERR_INVALID_ARGUMENT;
  if (nc == 0) return SLC_OK;
  if (!theta || !theta_local || !ef || !records) return SLC_ERR_INVALID_ARGUMENT;
  if (!aligned16(theta) || !aligned16(theta_local) || !aligned16(ef) || (((uintptr_t)records) & 3u))
    return SLC_ERR_INVALID_ARGUMENT;
  slc::CompressArgs a;
  a.n_elems = p->shard_elems;
  a.n_tmaps = (int32_t)p->h_tmaps.size();
  a.tmaps = p->d_tmaps;
  a.chunks = p->d_chunks + c0;
  a.n_chunks = nc;
  a.theta = theta;
  a.theta_local = theta_local;
  a.ef = ef;
  a.records = static_cast<uint32_t*>(records) + c0 * p->g.rec_words;
  a.err = p->d_err;
  a.beta = beta;
  a.max_ld = p->max_ld;
  a.g = p->g;
  a.rec_extra = p->d_rec_extra;
  a.n_extra = p->n_extra_next;
  a.defer = p->d_defer;
  a.defer_cap = p->n_chunks;
  a.defer_info = slc::defer_info_words(p->g);
  DeviceGuard guard(p->device);
  cudaStream_t st = use_stream(p, stream);
#ifdef SLC_USE_TMA  // measured history: the TMA-fed ring (compress_tma.cu) is slower than compress_ws
  if (slc::compress_tma_supported(p->g)) {
    cudaError_t e = ensure_tmaps(p, theta, theta_local, ef, st);
    if (e != cudaSuccess) return cuda_status(e, p);
    return cuda_status(slc::launch_compress_tma(a, p->dtype == SLC_BF16, st), p);
  }
#endif
  return cuda_status(slc::launch_compress(a, p->dtype == SLC_BF16, st), p);
}

slc_status slc_decode_aggregate(slc_plan* p, const slc_payload_hdr* hdrs, const void* const* recs, int32_t R,
                                const float* w, float* agg, void* stream) {
  if (!p || p->device < 0) return SLC_ERR_INVALID_ARGUMENT;
  slc::AggArgs a;
  slc_status st = prep_agg(p, hdrs, recs, R, w, a);
  if (st != SLC_OK) return st;
  if (p->n_chunks == 0) return SLC_OK;
  if (!agg || !aligned16(agg)) return SLC_ERR_INVALID_ARGUMENT;
  a.mode = slc::kAggOnly;
  a.agg = agg;
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_aggregate(a, p->dtype == SLC_BF16, use_stream(p, stream)), p);
}

slc_status slc_outer_update(slc_plan* p, void* theta, const float* agg, const slc_payload_hdr* hdrs,
                            const void* const* recs, int32_t R, const float* w, float alpha, void* stream) {
  if (!p || p->device < 0) return SLC_ERR_INVALID_ARGUMENT;
  slc::AggArgs a;
  if (agg) {
    std::memset(&a, 0, sizeof(a));
    a.chunks = p->d_chunks;
    a.n_chunks = p->n_chunks;
    a.g = p->g;
    a.err = p->d_err;
    a.mode = slc::kUpdateFromAgg;
    a.agg = const_cast<float*>(agg);
    if (p->n_chunks > 0 && !aligned16(agg)) return SLC_ERR_INVALID_ARGUMENT;
  } else {
    slc_status st = prep_agg(p, hdrs, recs, R, w, a);
    if (st != SLC_OK) return st;
    a.mode = slc::kFused;
  }
  if (p->n_chunks == 0) return SLC_OK;
  if (!theta || !aligned16(theta)) return SLC_ERR_INVALID_ARGUMENT;
  a.alpha = alpha;
  a.theta = theta;
  DeviceGuard guard(p->device);
  cudaStream_t cs = use_stream(p, stream);
  if (a.mode == slc::kFused) set_update_tmaps(p, theta, cs, a);
  return cuda_status(slc::launch_aggregate(a, p->dtype == SLC_BF16, cs), p);
}

slc_status slc_decode_aggregate_wdev(slc_plan* p, const slc_payload_hdr* hdrs, const void* const* recs, int32_t R,
                                     const float* w_dev, float* agg, void* stream) {
  if (!p || p->device < 0 || !w_dev) return SLC_ERR_INVALID_ARGUMENT;
  slc::AggArgs a;
  slc_status st = prep_agg(p, hdrs, recs, R, nullptr, a);
  if (st != SLC_OK) return st;
  if (p->n_chunks == 0) return SLC_OK;
  if (!agg || !aligned16(agg)) return SLC_ERR_INVALID_ARGUMENT;
  a.weighted = 1;
  a.wdev = w_dev;
  a.mode = slc::kAggOnly;
  a.agg = agg;
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_aggregate(a, p->dtype == SLC_BF16, use_stream(p, stream)), p);
}

slc_status slc_outer_update_wdev(slc_plan* p, void* theta, const slc_payload_hdr* hdrs, const void* const* recs,
                                 int32_t R, const float* w_dev, float alpha, void* stream) {
  if (!p || p->device < 0 || !w_dev) return SLC_ERR_INVALID_ARGUMENT;
  slc::AggArgs a;
  slc_status st = prep_agg(p, hdrs, recs, R, nullptr, a);
  if (st != SLC_OK) return st;
  if (p->n_chunks == 0) return SLC_OK;
  if (!theta || !aligned16(theta)) return SLC_ERR_INVALID_ARGUMENT;
  a.weighted = 1;
  a.wdev = w_dev;
  a.mode = slc::kFused;
  a.alpha = alpha;
  a.theta = theta;
  DeviceGuard guard(p->device);
  cudaStream_t cs = use_stream(p, stream);
  set_update_tmaps(p, theta, cs, a);
  return cuda_status(slc::launch_aggregate(a, p->dtype == SLC_BF16, cs), p);
}

slc_status slc_payload_sqnorm(slc_plan* p, const slc_payload_hdr* hdrs, const void* const* recs, int32_t R,
                              uint64_t* sqnorm_dev, void* stream) {
  if (!p || p->device < 0 || !sqnorm_dev || (((uintptr_t)sqnorm_dev) & 7u)) return SLC_ERR_INVALID_ARGUMENT;
  slc::AggArgs a;
  slc_status st = prep_agg(p, hdrs, recs, R, nullptr, a);
  if (st != SLC_OK) return st;
  // caller's peer order (not canonical): limbs of peer r go to sqnorm_dev[4r..4r+3]
  for (int r = 0; r < R; r++) a.rec[r] = static_cast<const uint32_t*>(recs[r]);
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_payload_sqnorm(a, reinterpret_cast<unsigned long long*>(sqnorm_dev),
                                                use_stream(p, stream)),
                     p);
}

slc_status slc_median_norm_weights(slc_plan* p, int32_t R, const uint64_t* sqnorm_dev, float* weights_dev,
                                   double* norms_dev, void* stream) {
  if (!p || p->device < 0 || R < 1 || R > slc::kMaxPeers || !sqnorm_dev || !weights_dev)
    return SLC_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_median_weights(reinterpret_cast<const unsigned long long*>(sqnorm_dev), R,
                                                weights_dev, norms_dev, use_stream(p, stream)),
                     p);
}

slc_status slc_peer_copy(slc_plan* p, const void* const* src, void* const* dst, const int64_t* bytes, int32_t n,
                         void* stream) {
  if (!p || p->device < 0 || n < 0 || n > slc::kMaxPeers || (n > 0 && (!src || !dst || !bytes)))
    return SLC_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < n; i++)
    if (bytes[i] < 0 || (bytes[i] > 0 && (!src[i] || !dst[i]))) return SLC_ERR_INVALID_ARGUMENT;
  if (!p->d_pc_scratch) return SLC_OK;  // plan without device tables: nothing to copy into (n_chunks == 0)
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_peer_copy(src, dst, bytes, n, p->d_pc_scratch, use_stream(p, stream)), p);
}

slc_status slc_fast_checks(slc_plan* p, const slc_payload_hdr* hdrs, const void* const* recs, int32_t R,
                           uint64_t current_round, const uint64_t* sqnorm_dev, const double* hist, int32_t n_hist,
                           uint32_t* flags_dev, void* stream) {
  if (!p || p->device < 0 || R < 1 || R > slc::kMaxPeers || !recs || !flags_dev || (((uintptr_t)flags_dev) & 3u))
    return SLC_ERR_INVALID_ARGUMENT;
  if (n_hist < 0 || (n_hist > 0 && !hist)) return SLC_ERR_INVALID_ARGUMENT;
  slc::AggArgs a;
  std::memset(&a, 0, sizeof(a));
  a.chunks = p->d_chunks;
  a.n_chunks = p->n_chunks;
  a.R = R;
  a.err = p->d_err;
  a.g = p->g;
  std::vector<uint32_t> hf(R, 0u);
  for (int r = 0; r < R; r++) {
    a.rec[r] = static_cast<const uint32_t*>(recs[r]);
    if (!recs[r]) {
      hf[r] |= SLC_CHECK_LIVENESS;
      continue;
    }
    if ((((uintptr_t)recs[r]) & 3u)) return SLC_ERR_INVALID_ARGUMENT;
    if (hdrs && (hdrs[r].base_round != current_round || std::memcmp(hdrs[r].layout_digest, p->digest, 32) != 0))
      hf[r] |= SLC_CHECK_SYNC;
  }
  double thresh = __builtin_inf();
  if (sqnorm_dev && n_hist > 0) {  // R#29: 10 x the lower median of the history
    std::vector<double> h(hist, hist + n_hist);
    std::sort(h.begin(), h.end());
    thresh = 10.0 * h[(n_hist - 1) / 2];
  }
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_fast_checks(a, hf.data(), thresh,
                                             reinterpret_cast<const unsigned long long*>(sqnorm_dev), flags_dev,
                                             use_stream(p, stream)),
                     p);
}

slc_status slc_wire_layout(const slc_plan* p, int64_t* body_bytes, int64_t* body_offset) {
  if (!p || !body_bytes || !body_offset) return SLC_ERR_INVALID_ARGUMENT;
  *body_bytes = p->wire_bytes;
  *body_offset = p->wire_offset;
  return SLC_OK;
}

static slc::WireArgs wire_args(slc_plan* p) {
  slc::WireArgs a;
  std::memset(&a, 0, sizeof(a));
  a.chunks = p->d_chunks;
  a.n_chunks = p->n_chunks;
  a.wire_off = p->d_wire_off;
  a.err = p->d_err;
  a.g = p->g;
  return a;
}

slc_status slc_wire_encode(slc_plan* p, const void* records, void* wire, void* stream) {
  if (!p || p->device < 0) return SLC_ERR_INVALID_ARGUMENT;
  if (p->n_chunks == 0) return SLC_OK;
  if (!records || !wire || (((uintptr_t)records) & 3u)) return SLC_ERR_INVALID_ARGUMENT;
  slc::WireArgs a = wire_args(p);
  a.rec = static_cast<const uint32_t*>(records);
  a.wire = static_cast<uint8_t*>(wire);
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_wire(a, true, use_stream(p, stream)), p);
}

slc_status slc_wire_decode(slc_plan* p, const void* wire, int64_t nbytes, void* records, void* stream) {
  if (!p || p->device < 0) return SLC_ERR_INVALID_ARGUMENT;
  if (nbytes < p->wire_bytes) return SLC_ERR_FORMAT;  // truncated body: nothing is read
  if (p->n_chunks == 0) return SLC_OK;
  if (!records || !wire || (((uintptr_t)records) & 3u)) return SLC_ERR_INVALID_ARGUMENT;
  slc::WireArgs a = wire_args(p);
  a.wire_in = static_cast<const uint8_t*>(wire);
  a.rec_out = static_cast<uint32_t*>(records);
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_wire(a, false, use_stream(p, stream)), p);
}

slc_status slc_index_rank(slc_plan* p, const void* records, uint32_t* ranks, void* stream) {
  if (!p || p->device < 0) return SLC_ERR_INVALID_ARGUMENT;
  if (!slc::index_rank_supported(p->g)) return SLC_ERR_UNSUPPORTED;
  if (p->n_chunks == 0) return SLC_OK;
  if (!p->d_binom) return SLC_ERR_INVALID_ARGUMENT;  // slc_plan_set_option(SLC_OPT_INDEX_CODE, 1) first
  if (!records || !ranks || (((uintptr_t)records) & 3u) || (((uintptr_t)ranks) & 3u))
    return SLC_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_index_rank(p->d_chunks, p->n_chunks, static_cast<const uint32_t*>(records),
                                            p->d_binom, ranks, p->g, use_stream(p, stream)),
                     p);
}

int64_t slc_ec_record_bytes(const slc_geometry* geom) {
  if (check_geom(geom) != SLC_OK) return -1;
  const slc::Geom g = make_geom(*geom);
  if (!slc::index_rank_supported(g)) return -1;
  return 4 * (int64_t)slc::ec_record_words(g);
}

slc_status slc_index_encode(slc_plan* p, const void* records, void* ec, void* stream) {
  if (!p || p->device < 0) return SLC_ERR_INVALID_ARGUMENT;
  if (!slc::index_rank_supported(p->g)) return SLC_ERR_UNSUPPORTED;
  if (p->n_chunks == 0) return SLC_OK;
  if (!p->d_binom) return SLC_ERR_INVALID_ARGUMENT;  // slc_plan_set_option(SLC_OPT_INDEX_CODE, 1) first
  if (!records || !ec || (((uintptr_t)records) & 3u) || (((uintptr_t)ec) & 3u)) return SLC_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_index_encode(p->d_chunks, p->n_chunks, static_cast<const uint32_t*>(records),
                                              p->d_binom, static_cast<uint32_t*>(ec), p->g, use_stream(p, stream)),
                     p);
}

slc_status slc_index_decode(slc_plan* p, const void* ec, void* records, void* stream) {
  if (!p || p->device < 0) return SLC_ERR_INVALID_ARGUMENT;
  if (!slc::index_rank_supported(p->g)) return SLC_ERR_UNSUPPORTED;
  if (p->n_chunks == 0) return SLC_OK;
  if (!p->d_binom) return SLC_ERR_INVALID_ARGUMENT;
  if (!records || !ec || (((uintptr_t)records) & 3u) || (((uintptr_t)ec) & 3u)) return SLC_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(p->device);
  return cuda_status(slc::launch_index_decode(p->d_chunks, p->n_chunks, static_cast<const uint32_t*>(ec),
                                              p->d_binom, static_cast<uint32_t*>(records), p->d_err, p->g,
                                              use_stream(p, stream)),
                     p);
}

slc_status slc_plan_set_option(slc_plan* p, int32_t option, int64_t value) {
  if (!p) return SLC_ERR_INVALID_ARGUMENT;
  switch (option) {
    case SLC_OPT_AGG_KERNEL:
      if (value < 0 || value > 3) return SLC_ERR_INVALID_ARGUMENT;
      p->agg_variant = (int)value;
      return SLC_OK;
    case SLC_OPT_AGG_GRID_CAP:
      if (value < 0) return SLC_ERR_INVALID_ARGUMENT;
      p->agg_grid_cap = value;
      return SLC_OK;
    case SLC_OPT_INDEX_CODE: {
      if (value != 0 && value != 1) return SLC_ERR_INVALID_ARGUMENT;
      if (p->device < 0) return SLC_ERR_INVALID_ARGUMENT;
      DeviceGuard guard(p->device);
      if (value == 0) {
        if (p->d_binom) cudaFree(p->d_binom);
        p->d_binom = nullptr;
        return SLC_OK;
      }
      if (!slc::index_rank_supported(p->g)) return SLC_ERR_UNSUPPORTED;
      if (p->d_binom) return SLC_OK;
      uint32_t* T = nullptr;
      cudaError_t e = cudaMalloc(&T, slc::binom_table_bytes(p->g));
      if (e == cudaSuccess) e = slc::build_binom_table(T, p->g, nullptr);
      if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
      if (e != cudaSuccess) {
        if (T) cudaFree(T);
        cudaGetLastError();
        return SLC_ERR_CUDA;
      }
      p->d_binom = T;
      return SLC_OK;
    }
  }
  return SLC_ERR_INVALID_ARGUMENT;
}

static void put_be(uint8_t* o, uint64_t v, int n) {
  for (int i = 0; i < n; i++) o[i] = (uint8_t)(v >> (8 * (n - 1 - i)));
}
static uint64_t get_be(const uint8_t* o, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; i++) v = (v << 8) | o[i];
  return v;
}

slc_status slc_wire_header_write(const slc_payload_hdr* h, int64_t total_chunks, uint8_t out[65]) {
  if (!h || !out || total_chunks < 0 || total_chunks > 0xFFFFFFFFll) return SLC_ERR_INVALID_ARGUMENT;
  std::memcpy(out, "SLC1", 4);
  out[4] = 1;
  put_be(out + 5, h->base_round, 8);
  std::memcpy(out + 13, h->peer_id, 16);
  std::memcpy(out + 29, h->layout_digest, 32);
  put_be(out + 61, (uint64_t)total_chunks, 4);
  return SLC_OK;
}

slc_status slc_wire_header_read(const uint8_t* in, int64_t nbytes, slc_payload_hdr* h, int64_t* total_chunks) {
  if (!in || !h || !total_chunks) return SLC_ERR_INVALID_ARGUMENT;
  if (nbytes < 65 || std::memcmp(in, "SLC1", 4) != 0 || in[4] != 1) return SLC_ERR_FORMAT;
  std::memset(h, 0, sizeof(*h));
  std::memcpy(h->magic, "SLC1", 4);
  h->version = 1;
  h->base_round = get_be(in + 5, 8);
  std::memcpy(h->peer_id, in + 13, 16);
  std::memcpy(h->layout_digest, in + 29, 32);
  *total_chunks = (int64_t)get_be(in + 61, 4);
  return SLC_OK;
}

slc_status slc_get_status(slc_plan* p, int32_t synchronize) {
  if (!p) return SLC_ERR_INVALID_ARGUMENT;
  slc_status st = p->latched;
  p->latched = SLC_OK;
  if (synchronize && p->device >= 0) {
    // read and clear the device error word on the stream of the plan's last
    // call (stream order puts it after that call's kernels), then wait for it
    DeviceGuard guard(p->device);
    uint32_t err = 0;
    cudaStream_t s = p->last_stream;
    cudaError_t ce = cudaMemcpyAsync(&err, p->d_err, sizeof(err), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(p->d_err, 0, sizeof(uint32_t), s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return SLC_ERR_CUDA;
    if (err && st == SLC_OK) st = SLC_ERR_INVALID_DATA;
  }
  return st;
}

void slc_plan_destroy(slc_plan* p) {
  if (!p) return;
  if (p->device >= 0) {
    DeviceGuard guard(p->device);
    if (p->d_chunks) cudaFree(p->d_chunks);
    if (p->d_err) cudaFree(p->d_err);
    if (p->d_tmaps) cudaFree(p->d_tmaps);
    if (p->d_utmaps) cudaFree(p->d_utmaps);
    if (p->d_wire_off) cudaFree(p->d_wire_off);
    if (p->d_rec_extra) cudaFree(p->d_rec_extra);
    if (p->d_pc_scratch) cudaFree(p->d_pc_scratch);
    if (p->d_defer) cudaFree(p->d_defer);
    if (p->d_binom) cudaFree(p->d_binom);
  }
  delete p;
}

const char* slc_status_string(slc_status s) {
  switch (s) {
    case SLC_OK: return "ok";
    case SLC_ERR_INVALID_ARGUMENT: return "invalid argument";
    case SLC_ERR_INVALID_DATA: return "invalid data (non-finite input or fp16 scale overflow)";
    case SLC_ERR_STALE: return "stale submission (base round / layout digest / geometry mismatch)";
    case SLC_ERR_CUDA: return "CUDA runtime error";
    case SLC_ERR_UNSUPPORTED: return "unsupported geometry";
    case SLC_ERR_FORMAT: return "format error";
  }
  return "unknown status";
}

}  // extern "C"
