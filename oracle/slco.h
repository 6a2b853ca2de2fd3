/* slco.h — CPU ORACLE for the SparseLoCo outer-step hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2603_08163_b200/, libslc.so) never links, includes or
 * calls anything here, and this tree includes nothing from the product.
 *
 * Plain, slow, single-threaded C, compiled -O2 -ffp-contract=off
 * -fno-fast-math (no FMA contraction, no FTZ/DAZ).  Each function cites the
 * passage of /root/reference/PAPER.md (P:line) it follows; readings of points
 * the paper leaves open are the numbered ones in DESIGN.md §3 ("R#n").
 *
 * Parity pins: tests/test_oracle.py, tests/test_oracle_pins.py.  Q (R#1) is
 * not defined by the paper; it is pinned to SPEC S:120's reading by
 * hand-worked cases (tests/golden/oracle_pins.json).
 */
#ifndef SLCO_H
#define SLCO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SLCO_OK = 0, SLCO_INVALID_ARGUMENT = 1, SLCO_INVALID_DATA = 2, SLCO_STALE = 3 };
enum { SLCO_F32 = 0, SLCO_BF16 = 1 };

typedef struct {
  int32_t block;      /* side of the square 2-D chunk, 64            */
  int32_t chunk;      /* positions per chunk C = block^2, 4096  */
  int32_t k;          /* Top-k per full chunk, 64                    */
  int32_t index_bits; /* bits per transmitted index, 12               */
} slco_geom;

/* ---- chunk geometry (partial chunks R#10, flattening R#9) ---- */
int     slco_geom_check(const slco_geom* g);
int     slco_is_blocked(int ndim, const int64_t* dims, const slco_geom* g);
int64_t slco_tensor_chunks(int ndim, const int64_t* dims, const slco_geom* g);
/* flat in-tensor offsets of positions p = 0..n-1 of chunk c; returns n (or -1) */
int     slco_chunk_offsets(int ndim, const int64_t* dims, const slco_geom* g, int64_t c, int64_t* off);
int     slco_effective_k(int n, const slco_geom* g);
int     slco_record_words(const slco_geom* g);

/* ---- per-step functions ---- */
/* Top-k of one chunk buffer b[0..n): the k_eff positions of largest |b|, ties
 * to the lower position, returned ascending (R#3-R#5). */
int      slco_topk(const float* b, int n, int k_eff, int32_t* sel);
/* fixed-order fp32 sum T(x[0..n)) used by the quantiser (R#13) */
float    slco_tree_sum(const float* x, int n, int k);
uint16_t slco_rn16(float x);           /* fp32 -> binary16, RN-even (R#14) */
float    slco_f16_to_f32(uint16_t h);
uint16_t slco_rnbf(float x);           /* fp32 -> bfloat16, RN-even */

/* Eq. 1 for one chunk: b = beta*e + (a - l); Top-k; Q; record;
 * e_new = b - decode(record).  a, l are fp32 or bf16 (dtype); e fp32.
 * Q is the 2-bit sign+bucket quantiser of R#1 (pinned by hand-worked cases). */
int slco_compress_chunk(const void* a, const void* l, int dtype, const float* e, int n,
                        const slco_geom* g, float beta, uint32_t* rec, float* e_new);
/* decode one record: positions and dequantised values; returns k_eff */
int slco_decode_chunk(const uint32_t* rec, int n, const slco_geom* g, int32_t* pos, float* dq);
/* Eq. 2 first line: delta[p] = (1/R) sum_r w_r * dq_r[p], fp64 in
 * peer-id order (R#16, R#17).  peer_ids: R*16 bytes or NULL; w: R or NULL. */
int slco_aggregate_chunk(const uint32_t* const* recs, const uint8_t* peer_ids, const float* w, int R,
                         int n, const slco_geom* g, float* delta);
/* Eq. 2 second line: theta <- theta - alpha*delta (R#18) */
void slco_outer_update(void* theta, int dtype, const float* delta, int64_t n, float alpha);

/* ---- tensor-level drivers over a chunk range [c0, c1) of one tensor ---- */
int slco_compress_tensor(int ndim, const int64_t* dims, const void* a, const void* l, int dtype,
                         float* e_inout, const slco_geom* g, float beta, int64_t c0, int64_t c1,
                         uint32_t* rec_out);
/* recs[r] points at the record of chunk c0 of peer r (records of c0..c1-1 contiguous) */
int slco_aggregate_tensor(int ndim, const int64_t* dims, const uint32_t* const* recs,
                          const uint8_t* peer_ids, const float* w, int R, const slco_geom* g,
                          int64_t c0, int64_t c1, float* delta_out /* dense, whole tensor */);
int slco_aggregate_update_tensor(int ndim, const int64_t* dims, void* theta, int dtype,
                                 const uint32_t* const* recs, const uint8_t* peer_ids, const float* w,
                                 int R, const slco_geom* g, int64_t c0, int64_t c1, float alpha);

/* ---- closed forms printed in the paper ---- */
double slco_index_entropy_bound(int C, int k);
double slco_compression_ratio(int C, int k, int dense_bits, int wire_bits_per_value);

#ifdef __cplusplus
}
#endif
#endif
