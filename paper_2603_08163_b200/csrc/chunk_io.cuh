// chunk_io.cuh — element addressing and vectorised loads/stores of one chunk.
//
// Thread t of a C/16-thread CTA owns 4 groups of 4 consecutive in-chunk
// positions: group v covers p = 4q .. 4q+3 with q = v*NT + t.  For a blocked
// chunk (ld > 0) position p = B*row + col lives at base + row*ld + col, so
// every group is 4 contiguous elements (16 B fp32 / 8 B bf16) and one warp's
// group covers 512 B (fp32) of whole 256-B block rows: fully coalesced
// 128-bit loads.  Flat chunks are contiguous.  Only the last chunk of a flat
// tensor can be partial (len < C); its tail group is loaded element by element.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "slc_internal.cuh"

namespace slc {

template <int C>
struct ChunkCfg {
  static constexpr int NT = C / 16;  // threads per CTA, 16 elements per thread
  static constexpr int B = (C == 1024) ? 32 : (C == 4096 ? 64 : 128);
  static constexpr int RPQ = B / 4;  // 4-element groups per block row
  static constexpr int BW = C / 32;  // bitmap words
  static_assert(B * B == C, "chunk must be a square block");
};

__device__ __forceinline__ int64_t group_offset(const ChunkDesc& d, int q, int rpq_shift) {
  return d.ld ? d.base + (int64_t)(q >> rpq_shift) * d.ld + 4 * (q & ((1 << rpq_shift) - 1))
              : d.base + 4 * (int64_t)q;
}

__device__ __forceinline__ float bf16_bits_to_f32(uint32_t h) { return __uint_as_float(h << 16); }

// Load 4 consecutive param values (fp32 or bf16) as fp32; n = valid count (0..4).
template <bool BF16>
__device__ __forceinline__ void load_param4(const void* base, int64_t off, int n, float v[4]) {
  if (BF16) {
    const uint16_t* p = static_cast<const uint16_t*>(base) + off;
    if (n == 4) {
      uint2 u = __ldcs(reinterpret_cast<const uint2*>(p));
      v[0] = bf16_bits_to_f32(u.x & 0xFFFFu);
      v[1] = bf16_bits_to_f32(u.x >> 16);
      v[2] = bf16_bits_to_f32(u.y & 0xFFFFu);
      v[3] = bf16_bits_to_f32(u.y >> 16);
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) v[j] = j < n ? bf16_bits_to_f32(p[j]) : 0.0f;
    }
  } else {
    const float* p = static_cast<const float*>(base) + off;
    if (n == 4) {
      float4 u = __ldcs(reinterpret_cast<const float4*>(p));
      v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) v[j] = j < n ? p[j] : 0.0f;
    }
  }
}

__device__ __forceinline__ void load_f32x4(const float* base, int64_t off, int n, float v[4]) {
  const float* p = base + off;
  if (n == 4) {
    float4 u = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; j++) v[j] = j < n ? p[j] : 0.0f;
  }
}

// the same through L2 with the normal eviction policy (ld.global.cg): the
// selection fallbacks re-read a chunk's candidate groups several times
__device__ __forceinline__ void load_f32x4_l2(const float* base, int64_t off, int n, float v[4]) {
  const float* p = base + off;
  if (n == 4) {
    float4 u = __ldcg(reinterpret_cast<const float4*>(p));
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; j++) v[j] = j < n ? __ldcg(p + j) : 0.0f;
  }
}

__device__ __forceinline__ void store_f32x4(float* base, int64_t off, int n, const float v[4]) {
  float* p = base + off;
  if (n == 4) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  } else {
#pragma unroll
    for (int j = 0; j < 4; j++)
      if (j < n) p[j] = v[j];
  }
}

__device__ __forceinline__ uint16_t f32_to_bf16_rn_bits(float x) {
  __nv_bfloat16 h = __float2bfloat16_rn(x);
  return *reinterpret_cast<uint16_t*>(&h);
}

template <bool BF16>
__device__ __forceinline__ void store_param4(void* base, int64_t off, int n, const float v[4]) {
  if (BF16) {
    uint16_t* p = static_cast<uint16_t*>(base) + off;
    if (n == 4) {
      uint2 u;
      // two values per packed convert (each rounded to nearest even, as one at a time)
      const __nv_bfloat162 lo = __floats2bfloat162_rn(v[0], v[1]), hi = __floats2bfloat162_rn(v[2], v[3]);
      u.x = *reinterpret_cast<const uint32_t*>(&lo);
      u.y = *reinterpret_cast<const uint32_t*>(&hi);
      __stcs(reinterpret_cast<uint2*>(p), u);
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++)
        if (j < n) p[j] = f32_to_bf16_rn_bits(v[j]);
    }
  } else {
    store_f32x4(static_cast<float*>(base), off, n, v);
  }
}

__device__ __forceinline__ int valid_in_group(int p0, int len) {
  const int r = len - p0;
  return r >= 4 ? 4 : (r > 0 ? r : 0);
}

}  // namespace slc
