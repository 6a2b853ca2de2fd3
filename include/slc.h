/* slc.h — C ABI of the B200 (sm_100a) SparseLoCo outer-step hot path.
 *
 * Implements, per FSDP shard of one peer, §2.1 (arxiv 2603.08163):
 *   Eq. 1  Delta_r = theta - theta_r^(t,H);
 *                    hatDelta_r = Q(Top-k(beta*e_r + Delta_r));
 *                    e_r <- beta*e_r + Delta_r - hatDelta_r          -> slc_compress
 *   Eq. 2  Delta = (1/R) sum_r hatDelta_r                   -> slc_decode_aggregate
 *                    theta <- theta - alpha*Delta                     -> slc_outer_update
 * with the chunk-wise Top-k of P:88 (64x64 blocks of 2-D tensors, 4096-chunks
 * of 1-D tensors), C = 4096, k = 64, beta = 0.95, alpha = 1 (0.65 P:180),
 * 2-bit values and 12-bit fixed-width indices.  Points the
 * paper leaves open follow DESIGN.md §3 (readings R#1..R#25).
 *
 * General conventions
 *  - Every buffer argument named *_dev is a CUDA DEVICE pointer on the plan's
 *    device, owned by the caller (the library never frees or retains it).
 *    Arguments named *_host are host pointers read before the call returns.
 *  - Compute calls are asynchronous on `stream` (a cudaStream_t passed as
 *    void*, NULL = legacy default stream), allocate nothing and never
 *    synchronize.  One plan must not be used on two streams concurrently.
 *    The plan remembers the stream of its most recent call (for
 *    slc_get_status); that stream must outlive the call to slc_get_status.
 *  - Argument / header errors are detected on the host and returned
 *    synchronously; nothing is launched then.  Data errors found on the device
 *    (a non-finite theta, theta_local, e or beta*e + Delta; an fp16 scale that
 *    overflows) are LATCHED in the plan and reported by slc_get_status(); the
 *    outputs of the offending call are then unspecified.
 *  - Allocations are made only by slc_plan_create (device chunk table, wire
 *    offsets, error word, and the compress deferral list: 4 + n_chunks * (2 +
 *    units per lane) 32-bit words, 40 B per chunk at the paper's geometry —
 *    chunks whose selection leaves the candidate path are finished by a second
 *    kernel of the same call) and by slc_plan_set_option(SLC_OPT_INDEX_CODE)
 *    (the f4 binomial table); slc_plan_destroy releases them.
 */
#ifndef SLC_H
#define SLC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SLC_OK = 0,
  SLC_ERR_INVALID_ARGUMENT = 1, /* bad pointer / size / geometry / header field      */
  SLC_ERR_INVALID_DATA = 2,     /* non-finite input or fp16 scale overflow (latched)  */
  SLC_ERR_STALE = 3,            /* peer headers disagree: base_round, layout digest, geometry */
  SLC_ERR_CUDA = 4,             /* a CUDA runtime call failed                         */
  SLC_ERR_UNSUPPORTED = 5,      /* geometry without a compiled kernel                 */
  SLC_ERR_FORMAT = 6            /* wire bytes: bad magic / version, truncated  */
} slc_status;

typedef enum { SLC_F32 = 0, SLC_BF16 = 1 } slc_dtype; /* dtype of theta / theta_local; e is fp32 */

/* Chunk geometry.  Default {64, 4096, 64, 12}.
 * Requires chunk == block*block, 1 <= k <= 256, k <= chunk,
 * 2^index_bits >= chunk, index_bits <= 16.  Compiled chunk sizes: 1024, 4096, 16384. */
typedef struct {
  int32_t block;      /* side of a square 2-D chunk                  */
  int32_t chunk;      /* C, positions per chunk                      */
  int32_t k;          /* values sent per full chunk                  */
  int32_t index_bits; /* bits per transmitted in-chunk index         */
} slc_geometry;

/* One tensor of the GLOBAL parameter layout (row-major, up to 4 dims).  A
 * 2-D tensor whose dims are both multiples of `block` is cut into blocks in
 * row-major block order, in-block position p = block*row + col (R#7, R#8);
 * every other tensor is flattened and cut into C-element chunks, the last one
 * possibly partial with k_eff = max(1, floor(k*len/C)) (R#9, R#10). */
typedef struct {
  int32_t ndim;
  int64_t dims[4];
} slc_tensor;

/* What a plan covers (filled by slc_plan_info). */
typedef struct {
  int64_t total_elems;   /* parameters in the whole layout                       */
  int64_t total_chunks;  /* chunks in the whole layout (global chunk order)      */
  int64_t first_chunk;   /* global index of this shard's first chunk             */
  int64_t n_chunks;      /* chunks in this shard                                 */
  int64_t shard_elems;   /* length of this shard's dense buffers, in elements    */
  int64_t record_bytes;  /* bytes per chunk record (116 at the default geometry) */
  int64_t payload_bytes; /* n_chunks * record_bytes                              */
  int32_t n_segments;    /* tensor slices held by this shard                     */
  int32_t rank, nranks;
} slc_plan_info;

/* One tensor slice held by a shard (slc_plan_segment).  The shard's dense
 * buffers (theta, theta_local, e, Delta) are the concatenation of its
 * segments, each starting at a 64-element (256-byte) aligned shard offset;
 * the padding between segments is never read or written by the library. */
typedef struct {
  int32_t tensor;        /* index into the layout                                        */
  int32_t blocked;       /* 1: rows x cols slice cut into blocks; 0: flat chunks          */
  int64_t tensor_begin;  /* first element of the slice in the tensor's row-major order    */
  int64_t n_elems;       /* elements in the slice (contiguous in that order)              */
  int64_t shard_offset;  /* element offset of the slice in the shard buffers              */
  int64_t rows, cols;    /* blocked: slice shape; flat: rows = n_elems, cols = 1          */
  int64_t first_chunk;   /* global chunk index of the slice's first chunk                 */
  int64_t n_chunks;
} slc_segment;

/* Host-side header of one peer's payload slice (SPEC S:99-104 CompressedDelta,
 * its base-round / peer-id / layout-digest fields).  Optional: pass NULL to
 * skip the checks. */
typedef struct {
  char magic[4];             /* "SLC1"                                        */
  uint32_t version;          /* 1                                             */
  slc_geometry geom;
  uint64_t base_round;       /* outer round the payload was built on          */
  uint8_t peer_id[16];       /* canonical aggregation order = ascending id    */
  uint8_t layout_digest[32]; /* slc_layout_digest of the global layout        */
  int64_t first_chunk;       /* global chunk range of the records described   */
  int64_t n_chunks;
} slc_payload_hdr;

typedef struct slc_plan slc_plan;

/* Build the plan of shard `rank` of `nranks` (R#11): the global chunk sequence
 * (tensors in layout order, chunks in row-major block order) is cut into
 * nranks contiguous ranges balanced by element count, cutting blocked tensors
 * only at block-row boundaries ("compression can be performed independently on
 * each shard"; EF sharded like the inner state).  Uploads the
 * shard's chunk table to `device`.  Returns INVALID_ARGUMENT for a bad
 * layout / rank, UNSUPPORTED for a geometry without a kernel, CUDA on a failed
 * allocation.  *out is NULL on failure. */
slc_status slc_plan_create(const slc_geometry* geom_host, const slc_tensor* layout_host, int32_t n_tensors,
                           int32_t rank, int32_t nranks, slc_dtype param_dtype, int32_t device,
                           slc_plan** out);
slc_status slc_plan_info_get(const slc_plan* plan, slc_plan_info* out_host);
slc_status slc_plan_segment(const slc_plan* plan, int32_t i, slc_segment* out_host);
/* bytes of one chunk record: 4*(ceil(k*index_bits/32) + ceil(2k/32) + 1); -1 on a bad geometry */
int64_t slc_record_bytes(const slc_geometry* geom_host);
/* 32-byte digest of (geometry, layout); non-cryptographic (splitmix64 lanes) */
slc_status slc_layout_digest(const slc_geometry* geom_host, const slc_tensor* layout_host, int32_t n_tensors,
                             uint8_t out_host[32]);

/* Eq. 1 on the plan's shard, all chunks:
 *   theta_dev        [shard_elems] param_dtype — theta^(t), the synchronized anchor (read)
 *   theta_local_dev  [shard_elems] param_dtype — theta_r^(t,H) after H inner steps (read)
 *   ef_dev           [shard_elems] fp32        — e_r^(t) in, e_r^(t+1) out (in place)
 *   beta             EF decay (0.95)
 *   records_dev      [n_chunks * record_bytes] — hatDelta_r of the shard, chunk c of the
 *                    shard at byte c*record_bytes, 4-byte aligned (R#6 layout)
 * Per chunk: d = theta - theta_local; b = fma(beta, e, d) (R#12); the k_eff
 * positions of largest |b|, ties to the lower position (R#3, R#4), ascending
 * (R#5); 2-bit sign+bucket code with two fp16 bucket-mean scales (R#1, R#13,
 * R#14); e <- b - dequant (selected) or b (others).  16-byte aligned dense
 * buffers required.  Latches INVALID_DATA on a non-finite value or an fp16
 * overflow. */
slc_status slc_compress(slc_plan* plan, const void* theta_dev, const void* theta_local_dev, float* ef_dev,
                        float beta, void* records_dev, void* stream);

/* slc_compress that writes the shard's records to n_out buffers at once:
 * records_out_host[0] (the caller's own, as records_dev of slc_compress) and
 * records_out_host[1..n_out-1], device pointers valid on the plan's device —
 * typically NVLink peer mappings of every other rank's peer-message buffer at
 * this shard's offset (CUDA IPC / symmetric memory), so the intra-box payload
 * all-gather of row a8 is folded into the compress
 * kernel: each 116-B record is stored to every destination as it is packed,
 * and no separate collective runs.  The caller synchronises the ranks after
 * the call (e.g. a device-side barrier) before reading a gathered message.
 * 1 <= n_out <= 16; 4-byte aligned destinations. */
slc_status slc_compress_multi(slc_plan* plan, const void* theta_dev, const void* theta_local_dev, float* ef_dev,
                              float beta, void* const* records_out_host, int32_t n_out, void* stream);

/* Rows a8 / a9 over NVLink peer memory: copy n byte ranges (src_host[i] ->
 * dst_host[i], bytes_host[i] bytes; device pointers valid on the plan's device,
 * either side may be a peer mapping of another GPU's buffer) with one kernel
 * in which every SM pulls 32 KB at a time, so all links stream at once — the
 * simulated-peer exchange pulls each rank's slice of every peer message from
 * its owner this way.  16-B aligned ranges take the vector path.  The caller
 * orders it against the peers (device barrier).  0 <= n <= 256. */
slc_status slc_peer_copy(slc_plan* plan, const void* const* src_host, void* const* dst_host,
                         const int64_t* bytes_host, int32_t n, void* stream);

/* slc_compress restricted to the shard-local chunks [chunk_begin, chunk_begin + n_chunks)
 * (same buffers and meaning as slc_compress: full-shard theta / theta_local / ef
 * base pointers, records_dev the full shard record buffer, chunk c at byte
 * c*record_bytes).  Only those chunks' elements and records are read or
 * written, so the EF of the other chunks may be absent from device memory —
 * the piecewise swap of NEXT row f3 (EF swapped in for compression
 * and out again, overlapped).  Results are bitwise those of slc_compress for
 * those chunks (chunks are independent).  INVALID_ARGUMENT for a range
 * outside [0, n_chunks]; n_chunks == 0 is a no-op. */
slc_status slc_compress_range(slc_plan* plan, int64_t chunk_begin, int64_t n_chunks, const void* theta_dev,
                              const void* theta_local_dev, float* ef_dev, float beta, void* records_dev,
                              void* stream);

/* Eq. 2 line 1: agg_dev[shard_elems] (fp32, padding untouched) <-
 * (1/R) sum_r w_r * decode(records_dev_host[r]) over the shard's chunks.
 *   hdrs_host          R headers or NULL (then no checks, given order is canonical)
 *   records_dev_host   host array of R device pointers, each to this shard's
 *                      n_chunks records of one peer (same layout as slc_compress)
 *   R                  1 <= R <= 256 (own payload counts as one peer, R#16)
 *   weights_host       R floats or NULL (= all 1).  With NULL the sum is exact
 *                      (fixed-point, order-free, R#17); otherwise fp64 in
 *                      ascending peer-id order (median-norm weights).
 * Header checks: magic/version/chunk range -> INVALID_ARGUMENT; differing
 * geometry, base_round or layout_digest -> STALE; duplicate peer ids ->
 * INVALID_ARGUMENT.  Records are device records as slc_compress writes them:
 * an index >= the chunk length or a non-finite used scale latches
 * INVALID_DATA, but indices are not re-checked for being strictly increasing
 * (a repeated index could overflow the exact int32 accumulator) — records
 * from untrusted peers enter through slc_wire_decode, which rejects them
 * (S:144). */
slc_status slc_decode_aggregate(slc_plan* plan, const slc_payload_hdr* hdrs_host,
                                const void* const* records_dev_host, int32_t R, const float* weights_host,
                                float* agg_dev, void* stream);

/* Eq. 2 line 2: theta <- fma(-alpha, Delta, theta) (R#18) over the shard.
 *   theta_dev  [shard_elems] param_dtype, in place
 *   agg_dev    dense fp32 Delta from slc_decode_aggregate, or NULL: then the
 *              fused kernel decodes and aggregates hdrs/records/R/weights (same
 *              meaning as above) per chunk and never materialises Delta.
 *   alpha      outer learning rate (1, later 0.65) */
slc_status slc_outer_update(slc_plan* plan, void* theta_dev, const float* agg_dev,
                            const slc_payload_hdr* hdrs_host, const void* const* records_dev_host, int32_t R,
                            const float* weights_host, float alpha, void* stream);

/* Median-norm normalisation ("Pseudo-gradient contributions are scaled
 * relative to their median norm so that no single participant can dominate";
 * reading R#20: every nonzero contribution rescaled to the
 * lower-median norm; zero contributions pass through).  Three calls, no host
 * synchronisation:
 *
 * 1. slc_payload_sqnorm: ||hatDelta_r||^2 of each peer's payload restricted to
 *    this plan's shard, computed from the records alone and EXACT: an integer
 *    in units of 2^-48, returned as four un-carried 32-bit limbs per peer,
 *      sqnorm_dev[4r + i] (uint64, device, caller's peer order r = 0..R-1),
 *      value = sum_i sqnorm_dev[4r + i] * 2^(32 i).
 *    Limbs of several shards add exactly (an int64 sum, e.g. an NCCL
 *    all-reduce over the ranks), so the result is independent of the sharding.
 *    hdrs/records/R as for slc_decode_aggregate.  The call zeroes sqnorm_dev
 *    first.  Latches INVALID_DATA on a non-finite scale.
 * 2. slc_median_norm_weights: from the (summed) limbs, n_r = sqrt(RN64(value *
 *    2^-48)) (IEEE), m = lower median of the n_r, weights_dev[r] =
 *    RN32(m / n_r) for n_r > 0 else 1 (fp32, device, caller's order);
 *    norms_dev[r] = n_r (fp64, device) unless NULL.  1 <= R <= 256.
 * 3. slc_decode_aggregate_wdev / slc_outer_update_wdev: as slc_decode_aggregate /
 *    slc_outer_update (fused) with weights read from weights_dev (device, the
 *    caller's peer order) — fp64 sum in ascending peer-id order. */
slc_status slc_payload_sqnorm(slc_plan* plan, const slc_payload_hdr* hdrs_host, const void* const* records_dev_host,
                              int32_t R, uint64_t* sqnorm_dev, void* stream);
slc_status slc_median_norm_weights(slc_plan* plan, int32_t R, const uint64_t* sqnorm_dev, float* weights_dev,
                                   double* norms_dev, void* stream);
slc_status slc_decode_aggregate_wdev(slc_plan* plan, const slc_payload_hdr* hdrs_host,
                                     const void* const* records_dev_host, int32_t R, const float* weights_dev,
                                     float* agg_dev, void* stream);
slc_status slc_outer_update_wdev(slc_plan* plan, void* theta_dev, const slc_payload_hdr* hdrs_host,
                                 const void* const* records_dev_host, int32_t R, const float* weights_dev,
                                 float alpha, void* stream);

/* NEXT row f2: SPEC's SLC1 wire format (the paper fixes no byte
 * layout, P:93 fixes 12 bits per index).  A message is the 65-byte header
 * (magic "SLC1", version 1, base-round u64, peer-id 16 B, layout-digest 32 B,
 * chunk count u32; big-endian) followed by one encoding per chunk in global
 * chunk order: count u16 (= k_eff), scale-lo and scale-hi (fp16 bits, u16),
 * the k_eff indices as index_bits-bit big-endian fields concatenated and
 * zero-padded to a byte, the k_eff 2-bit symbols (sign*2 + bucket, reading
 * R#27) packed likewise.  A shard's encodings are one contiguous byte range.
 *
 * slc_wire_layout: this shard's encodings take body_bytes bytes starting
 *   body_offset bytes after the header.
 * slc_wire_encode: records_dev (this shard's records, slc_compress layout) ->
 *   wire_dev[body_bytes] (device).  Asynchronous on stream.
 * slc_wire_decode: wire_dev[nbytes] -> records_dev; nbytes < body_bytes (a
 *   truncated body) returns SLC_ERR_FORMAT and reads nothing; else
 *   the first body_bytes bytes are decoded, validating every chunk
 *   (count == k_eff, indices strictly increasing and < the chunk length, zero
 *   padding, scales finite, >= 0, lo <= hi); a violation latches
 *   SLC_ERR_INVALID_DATA (reported by slc_get_status) and zeroes that record.
 * slc_wire_header_write / _read: host-side header (65 bytes).  _read returns
 *   SLC_ERR_FORMAT on a short buffer, bad magic or version; it fills magic,
 *   version, base_round, peer_id, layout_digest (geometry and chunk range are
 *   not on the wire: the caller's plan supplies them). */
/* Fast checks on every peer's submission ("fast checks
 * on all participants (e.g., liveness, synchronization with the main model,
 * etc.)"; reading R#29).  flags_dev[r] (uint32, device) <- OR of
 *   SLC_CHECK_LIVENESS  records_dev_host[r] == NULL (no submission this round);
 *   SLC_CHECK_SYNC      hdrs_host given and hdrs[r].base_round != current_round
 *                       or hdrs[r].layout_digest != the plan's digest;
 *   SLC_CHECK_FINITE    a decoded value is non-finite (a used bucket's fp16
 *                       scale is Inf / NaN), scanned on the device;
 *   SLC_CHECK_NORM      sqnorm_dev given (slc_payload_sqnorm limbs, summed over
 *                       the ranks for a sharded job) and the payload norm
 *                       sqrt(RN64(sum * 2^-48)) > 10 * m, m the lower median of
 *                       norm_history_host[0..n_hist) (fp64, compared in fp64;
 *                       n_hist == 0: no norm check).
 * Unlike slc_decode_aggregate, a peer's header mismatch is reported, not
 * returned: the round goes on without the flagged peers.  Returns
 * INVALID_ARGUMENT for R outside [1, 256] or a misaligned flags_dev. */
enum { SLC_CHECK_LIVENESS = 1, SLC_CHECK_SYNC = 2, SLC_CHECK_FINITE = 4, SLC_CHECK_NORM = 8 };
slc_status slc_fast_checks(slc_plan* plan, const slc_payload_hdr* hdrs_host, const void* const* records_dev_host,
                           int32_t R, uint64_t current_round, const uint64_t* sqnorm_dev,
                           const double* norm_history_host, int32_t n_hist, uint32_t* flags_dev, void* stream);

slc_status slc_wire_layout(const slc_plan* plan, int64_t* body_bytes_host, int64_t* body_offset_host);
slc_status slc_wire_encode(slc_plan* plan, const void* records_dev, void* wire_dev, void* stream);
slc_status slc_wire_decode(slc_plan* plan, const void* wire_dev, int64_t nbytes, void* records_dev, void* stream);
slc_status slc_wire_header_write(const slc_payload_hdr* hdr_host, int64_t total_chunks, uint8_t out_host[65]);
slc_status slc_wire_header_read(const uint8_t* in_host, int64_t nbytes, slc_payload_hdr* hdr_host,
                                int64_t* total_chunks_host);

/* NEXT row f4 (reading R#28): the enumerative index code.  For every
 * chunk c of the shard, ranks_dev[16c .. 16c+15] (uint32, little-endian limbs,
 * limb 0 least significant) <- sum_i binom(p_i, i + 1) over the k_eff ascending
 * positions of record c (records_dev as written by slc_compress) — the colex
 * rank, < binom(C_eff, k_eff), so ceil(log2 binom(C_eff, k_eff)) bits carry it
 * (472 at C = 4096, k = 64; 7.375 bits/value against the 7.36 of P:93).
 * Paper geometry only (C = 4096, k <= 64, 12-bit indices): UNSUPPORTED
 * otherwise.  Needs the plan's binomial table: slc_plan_set_option(plan,
 * SLC_OPT_INDEX_CODE, 1) first (INVALID_ARGUMENT otherwise).  4-byte aligned
 * buffers; INVALID_ARGUMENT otherwise. */
slc_status slc_index_rank(slc_plan* plan, const void* records_dev, uint32_t* ranks_dev, void* stream);

/* Entropy-coded ("EC") records (row f4, reading R#28): the 12-bit index stream
 * of each record replaced by its colex rank.  EC record of chunk c at byte
 * c*ec_record_bytes, little-endian u32 words: 0..14 the rank (limb 0 least
 * significant; < binom(C_eff, k_eff) < 2^472), then the record's code words
 * (R#6: bit 2j sign, 2j+1 bucket of slot j) and its scale word (S_lo | S_hi<<16).
 * 80 bytes at C = 4096, k = 64 against 116 (ratio 16384/80 = 204.8x dense fp32).
 * slc_ec_record_bytes: that size; -1 off the paper geometry (C = 4096, k <= 64,
 *   12-bit indices).
 * slc_index_encode: records_dev (slc_compress layout) -> ec_dev.
 * slc_index_decode: ec_dev -> records_dev (R#6 layout, unused slots zero) by
 *   greedy colex unranking (p_i = the largest p with binom(p, i+1) <= the
 *   remaining rank, i = k_eff-1 .. 0); a rank that is not a valid code
 *   (>= binom(C_eff, k_eff)) latches INVALID_DATA.
 * Both need the plan's binomial table (SLC_OPT_INDEX_CODE); UNSUPPORTED off the
 * paper geometry; 4-byte aligned buffers. */
int64_t slc_ec_record_bytes(const slc_geometry* geom_host);
slc_status slc_index_encode(slc_plan* plan, const void* records_dev, void* ec_dev, void* stream);
slc_status slc_index_decode(slc_plan* plan, const void* ec_dev, void* records_dev, void* stream);

/* Plan options (configuration calls: synchronous, may allocate).
 *  SLC_OPT_AGG_KERNEL    which decode / fused-update implementation runs:
 *                        0 auto (default: the persistent pipelined kernel
 *                        where it applies, else one CTA per chunk), 1 the
 *                        TMA-tile kernel (fused update, C = 4096, k = 64,
 *                        12-bit indices, R <= 64, 16-B aligned records; else
 *                        as 0), 2 pipelined, 3 one CTA per chunk.  Results are
 *                        bitwise identical; the parity tests run all of them.
 *  SLC_OPT_AGG_GRID_CAP  > 0: at most this many CTAs for the persistent decode
 *                        kernels (every CTA then walks many chunks; test aid).
 *  SLC_OPT_INDEX_CODE    1: build the f4 binomial table (C(p, j), p < 4096,
 *                        j <= 64; 16.8 MB on the plan's device, synchronously);
 *                        0: free it.  UNSUPPORTED off the paper geometry.
 * INVALID_ARGUMENT for an unknown option or value. */
typedef enum { SLC_OPT_AGG_KERNEL = 1, SLC_OPT_AGG_GRID_CAP = 2, SLC_OPT_INDEX_CODE = 3 } slc_option;
slc_status slc_plan_set_option(slc_plan* plan, int32_t option, int64_t value);

/* Latched status of the plan, cleared by the call.  synchronize != 0: the
 * device error word is read and cleared on the stream of the plan's most
 * recent call, which is then synchronized (not the whole device);
 * synchronize == 0: only what was latched on the host (argument-time and
 * launch errors). */
slc_status slc_get_status(slc_plan* plan, int32_t synchronize);
void slc_plan_destroy(slc_plan* plan);
const char* slc_status_string(slc_status s);

#ifdef __cplusplus
}
#endif
#endif /* SLC_H */
