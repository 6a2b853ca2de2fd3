// wire.cu — NEXT row f2: the SLC1 wire format of SPEC S:137-145 ("the paper
// does not fix a byte layout") for the chunks of a shard, converted on the GPU
// from / to the device record layout (R#6).
//
// Per chunk, big-endian: count (2 B) = k_eff, scale-lo (2 B fp16),
// scale-hi (2 B fp16), the k_eff indices as ib-bit big-endian fields
// concatenated and zero-padded to a byte ("12 bits/value"), the
// k_eff 2-bit code symbols (sign*2 + bucket, R#27) packed the same way.
// Chunk c's encoding starts at wire_off[c] (bytes from the shard's first
// chunk; the plan's prefix sums over k_eff).
//
// One warp per chunk: the record (or the chunk's bytes) is staged in a
// per-warp shared-memory slice, lanes extract slots j = lane + 32m, then each
// lane writes output bytes / words b = lane + 32m independently.  Decoding
// validates every CompressedChunk invariant of S:92-95 (count == k_eff, indices
// strictly increasing and < chunk length, zero padding bits, scales finite,
// >= 0 and lo <= hi) and latches INVALID_DATA otherwise.
#include "slc_internal.cuh"

namespace slc {
namespace {

constexpr int kWarps = 8;  // warps per CTA
constexpr int kMaxRecWords = (256 * 16 + 31) / 32 + (2 * 256 + 31) / 32 + 1;
constexpr int kMaxWireBytes = 6 + (256 * 16 + 7) / 8 + (2 * 256 + 7) / 8;

struct WarpSmem {
  uint32_t w[kMaxRecWords + 1];
  uint16_t idx[256 + 2];
  uint8_t code[256 + 4];
  uint8_t bytes[kMaxWireBytes + 8];
};

__device__ __forceinline__ int k_eff_of(const WireArgs& a, int64_t c) {
  return max(1, (a.g.k * __ldg(&a.chunks[c].len)) / a.g.C);
}

__global__ void __launch_bounds__(32 * kWarps) wire_encode_kernel(const WireArgs a) {
  __shared__ WarpSmem sm[kWarps];
  WarpSmem& S = sm[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int RW = a.g.rec_words, IW = a.g.idx_words, ib = a.g.ib;
  for (int64_t c = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); c < a.n_chunks;
       c += (int64_t)gridDim.x * kWarps) {
    const int ke = k_eff_of(a, c);
    const uint32_t* rec = a.rec + c * RW;
    for (int w = lane; w < RW; w += 32) S.w[w] = __ldg(rec + w);
    if (lane == 0) S.w[RW] = 0u;
    __syncwarp();
    for (int j = lane; j < ke + 2; j += 32) {
      uint32_t p = 0, code = 0;
      if (j < ke) {
        const int bit = ib * j;
        p = __funnelshift_r(S.w[bit >> 5], S.w[(bit >> 5) + 1], bit & 31) & ((1u << ib) - 1u);
        const uint32_t cb = S.w[IW + (j >> 4)] >> (2 * (j & 15));
        code = ((cb & 1u) << 1) | ((cb >> 1) & 1u);  // sign*2 + bucket
      }
      S.idx[j] = (uint16_t)p;
      if (j < ke + 2) S.code[j] = (uint8_t)code;
    }
    for (int j = ke + 2 + lane; j < ke + 4; j += 32) S.code[j] = 0;
    __syncwarp();
    const int nbi = (ke * ib + 7) / 8, nbc = (2 * ke + 7) / 8;
    const int size = 6 + nbi + nbc;
    uint8_t* out = a.wire + __ldg(&a.wire_off[c]);
    const uint32_t sw = S.w[RW - 1];
    for (int b = lane; b < size; b += 32) {
      uint32_t v;
      if (b < 6) {
        const uint32_t f = b < 2 ? (uint32_t)ke : (b < 4 ? (sw & 0xFFFFu) : (sw >> 16));
        v = (b & 1) ? (f & 0xFFu) : (f >> 8);
      } else if (b < 6 + nbi) {
        const int bb = b - 6;
        const int j0 = (8 * bb) / ib, off = 8 * bb - j0 * ib;  // off < ib, off + 8 <= 2 ib
        const uint32_t win = ((uint32_t)S.idx[j0] << ib) | (uint32_t)S.idx[j0 + 1];
        v = (win >> (2 * ib - off - 8)) & 0xFFu;
      } else {
        const int bb = b - 6 - nbi;
        v = ((uint32_t)S.code[4 * bb] << 6) | ((uint32_t)S.code[4 * bb + 1] << 4) |
            ((uint32_t)S.code[4 * bb + 2] << 2) | (uint32_t)S.code[4 * bb + 3];
      }
      out[b] = (uint8_t)v;
    }
    __syncwarp();
  }
}

__device__ __forceinline__ bool f16_finite_nonneg(uint32_t h) { return (h >> 15) == 0 && ((h >> 10) & 0x1Fu) != 0x1Fu; }

__global__ void __launch_bounds__(32 * kWarps) wire_decode_kernel(const WireArgs a) {
  __shared__ WarpSmem sm[kWarps];
  WarpSmem& S = sm[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int RW = a.g.rec_words, IW = a.g.idx_words, CW = a.g.code_words, ib = a.g.ib;
  bool bad = false;
  for (int64_t c = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); c < a.n_chunks;
       c += (int64_t)gridDim.x * kWarps) {
    const int ke = k_eff_of(a, c);
    const int len = __ldg(&a.chunks[c].len);
    const int nbi = (ke * ib + 7) / 8, nbc = (2 * ke + 7) / 8;
    const int size = 6 + nbi + nbc;
    const uint8_t* in = a.wire_in + __ldg(&a.wire_off[c]);
    for (int b = lane; b < size; b += 32) S.bytes[b] = __ldg(in + b);
    if (lane < 4) S.bytes[size + lane] = 0;
    __syncwarp();
    const uint32_t cnt = ((uint32_t)S.bytes[0] << 8) | S.bytes[1];
    const uint32_t lo = ((uint32_t)S.bytes[2] << 8) | S.bytes[3];
    const uint32_t hi = ((uint32_t)S.bytes[4] << 8) | S.bytes[5];
    bool ok = cnt == (uint32_t)ke && f16_finite_nonneg(lo) && f16_finite_nonneg(hi) && lo <= hi;
    // slots: big-endian ib-bit fields / 2-bit symbols
    for (int j = lane; j < ke; j += 32) {
      const int bit = ib * j;
      const int byte = bit >> 3;
      const uint32_t win = ((uint32_t)S.bytes[6 + byte] << 16) | ((uint32_t)S.bytes[6 + byte + 1] << 8) |
                           (uint32_t)S.bytes[6 + byte + 2];
      const uint32_t p = (win >> (24 - (bit & 7) - ib)) & ((1u << ib) - 1u);
      S.idx[j] = (uint16_t)p;
      S.code[j] = (uint8_t)((S.bytes[6 + nbi + (j >> 2)] >> (6 - 2 * (j & 3))) & 3u);
      ok &= (int)p < len;
    }
    // zero padding bits at the end of both sections
    if (lane == 0) {
      const int pi = 8 * nbi - ib * ke, pc = 8 * nbc - 2 * ke;
      if (pi) ok &= (S.bytes[6 + nbi - 1] & ((1u << pi) - 1u)) == 0;
      if (pc) ok &= (S.bytes[6 + nbi + nbc - 1] & ((1u << pc) - 1u)) == 0;
    }
    __syncwarp();
    for (int j = lane + 1; j < ke; j += 32) ok &= S.idx[j] > S.idx[j - 1];
    ok = __all_sync(0xFFFFFFFFu, ok);
    bad |= !ok;
    // record words (R#6): little-endian index stream, code stream bit 2j = sign / 2j+1 = bucket, scales
    uint32_t* rec = a.rec_out + c * RW;
    for (int w = lane; w < RW; w += 32) {
      uint32_t v = 0;
      if (!ok) {
        v = 0;
      } else if (w < IW) {
        const int b0 = 32 * w;
        const int j0 = b0 / ib, j1 = min(ke - 1, (b0 + 31) / ib);
        unsigned long long acc = 0;
        for (int j = j0; j <= j1; j++) {
          const int sh = ib * j - b0;  // may be negative for the slot straddling the word start
          const unsigned long long pj = S.idx[j];
          acc |= sh >= 0 ? (pj << sh) : (pj >> (-sh));
        }
        v = (uint32_t)acc;
      } else if (w < IW + CW) {
        const int j0 = 16 * (w - IW);
        for (int t = 0; t < 16 && j0 + t < ke; t++) {
          const uint32_t cd = S.code[j0 + t];
          v |= ((cd >> 1) & 1u) << (2 * t) | (cd & 1u) << (2 * t + 1);
        }
      } else {
        v = lo | (hi << 16);
      }
      rec[w] = v;
    }
    __syncwarp();
  }
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(a.err, kErrNonFinite);
}

}  // namespace

cudaError_t launch_wire(const WireArgs& a, bool encode, cudaStream_t s) {
  if (a.n_chunks == 0) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  const int64_t want = (a.n_chunks + kWarps - 1) / kWarps;
  const int grid = (int)(want < 8LL * sms ? want : 8LL * sms);
  if (encode)
    wire_encode_kernel<<<grid, 32 * kWarps, 0, s>>>(a);
  else
    wire_decode_kernel<<<grid, 32 * kWarps, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace slc
