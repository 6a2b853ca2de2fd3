// CUDA twin of slcgen/gen.py — seeded synthetic-input generator.
//
// Holds none of the method's arithmetic: it only draws theta, theta_local and
// the error-feedback buffer e as pure functions of (seed, stream, G), G the
// global flat element index.  Bit-identical to the numpy reference (integer
// splitmix64 hashing + exact fp32 operations; compiled without fast-math, no
// FTZ, and every fp32 op written as an explicit _rn intrinsic so no FMA
// contraction can change a rounding).  Used by tests and bench.py to fill
// device buffers at sizes numpy cannot reach quickly.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace {

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t STREAM_MUL = 0xD1B54A32D192ED03ull;
constexpr uint64_t M1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t M2 = 0x94D049BB133111EBull;
constexpr int S_THETA = 1, S_DELTA = 1000, S_ROWSCALE = 3000, S_EF = 5000, S_SPECIAL = 7000;
constexpr uint32_t THETA_SCALE_BITS = 0x3d0de3bdu;  // fp32(0.02*sqrt(3))

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= M1; z ^= z >> 27; z *= M2; z ^= z >> 31;
  return z;
}
__host__ __device__ inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed ^ GOLDEN) + stream * STREAM_MUL + 1ull);
}
__device__ inline uint64_t hat(uint64_t key, uint64_t G) { return mix64(key + (G + 1ull) * GOLDEN); }
__device__ inline float pow2neg(uint32_t j) { return __int_as_float((int)((127u - j) << 23)); }
__device__ inline float u24(uint64_t h) { return __fmul_rn((float)(uint32_t)(h >> 40), 5.9604644775390625e-08f); }

struct Keys {
  uint64_t theta, delta, rowscale, ef, special;
};

__device__ float theta_at(const Keys& k, uint64_t G) {
  uint64_t h = hat(k.theta, G);
  const float f = 1.52587890625e-05f;  // 2^-16
  float u0 = __fmul_rn((float)(uint32_t)(h & 0xFFFF), f);
  float u1 = __fmul_rn((float)(uint32_t)((h >> 16) & 0xFFFF), f);
  float u2 = __fmul_rn((float)(uint32_t)((h >> 32) & 0xFFFF), f);
  float u3 = __fmul_rn((float)(uint32_t)((h >> 48) & 0xFFFF), f);
  float s = __fadd_rn(__fadd_rn(u0, u1), __fadd_rn(u2, u3));
  s = __fsub_rn(s, 2.0f);
  return __fmul_rn(s, __int_as_float((int)THETA_SCALE_BITS));
}

__device__ float delta_at(const Keys& k, uint64_t G, uint64_t rowlen) {
  uint64_t h = hat(k.delta, G);
  float u = u24(h);
  uint32_t j = (uint32_t)((h >> 8) & 7);
  uint64_t hs = hat(k.rowscale, G / rowlen);
  uint32_t s = (uint32_t)(hs & 3);
  float v = __fmul_rn(__fsub_rn(u, 0.5f), 0.001953125f);  // 2^-9
  v = __fmul_rn(v, pow2neg(j));
  v = __fmul_rn(v, pow2neg(s));
  return v;
}

__device__ float ef_at(const Keys& k, uint64_t G) {
  uint64_t h = hat(k.ef, G);
  float u = u24(h);
  uint32_t j = (uint32_t)((h >> 8) & 7);
  float v = __fmul_rn(__fsub_rn(u, 0.5f), 0.0078125f);  // 2^-7
  return __fmul_rn(v, pow2neg(j));
}

// out[0]=theta, out[1]=theta_local, out[2]=e for an element of special family fam
__device__ void special_at(const Keys& k, uint64_t G, int fam, uint64_t rowlen, float out[3]) {
  uint64_t h = hat(k.delta, G);
  uint64_t ht = hat(k.theta, G);
  uint64_t hs = hat(k.special, G >> 12);
  float th = 0.0f, ef = 0.0f, d = 0.0f;
  float sign = (h >> 63) ? -1.0f : 1.0f;
  switch (fam) {
    case 0: d = 0.0f; break;
    case 1: {
      float c = __fmul_rn(__fadd_rn((float)(uint32_t)((hs >> 40) & 7), 1.0f), 0.0009765625f);
      float rs = ((hs >> 20) & 1) ? -1.0f : 1.0f;
      d = __fmul_rn(c, rs);
    } break;
    case 2: {
      float m = __fadd_rn((float)(uint32_t)((h >> 8) % 3), 1.0f);
      d = __fmul_rn(__fmul_rn(m, 0.0009765625f), sign);
    } break;
    case 3: {
      out[0] = ((ht >> 1) & 1) ? -0.0f : 0.0f;
      out[1] = ((h >> 2) & 1) ? -0.0f : 0.0f;
      out[2] = ((h >> 3) & 1) ? -0.0f : 0.0f;
      return;
    }
    case 4: {
      float mant = (float)(uint32_t)((h >> 40) & 0x7FFFFF);
      d = __fmul_rn(__fmul_rn(mant, __int_as_float(1)), sign);  // 2^-149
    } break;
    case 5: {
      d = delta_at(k, G, rowlen);
      uint64_t spike_at = (hs >> 8) & 4095;
      if ((G & 4095) == spike_at) d = __fmul_rn(d, 1024.0f);
      th = theta_at(k, G);
      out[0] = th; out[1] = __fsub_rn(th, d); out[2] = ef;
      return;
    }
    case 6: {
      float dd = delta_at(k, G, rowlen);
      d = ((h & 127) == 0) ? dd : 0.0f;
    } break;
    default: d = __fmul_rn(0.0009765625f, sign); break;
  }
  out[0] = th; out[1] = __fsub_rn(th, d); out[2] = ef;
}

__device__ inline uint16_t bf16_bits_rn(float x) {
  uint32_t b = __float_as_uint(x);
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

__global__ void fill_kernel(int what, Keys k, uint64_t G0, uint64_t n, uint64_t rowlen,
                            uint64_t period, int warm_ef, int out_bf16, void* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t G = G0 + i;
    float v;
    int fam = -1;
    if (period > 0) {
      uint64_t hs = hat(k.special, G >> 12);
      if (hs % period == 0) fam = (int)((hs >> 32) % 8);
    }
    if (fam >= 0) {
      float o[3];
      special_at(k, G, fam, rowlen, o);
      v = o[what];
    } else if (what == 0) {
      v = theta_at(k, G);
    } else if (what == 1) {
      v = __fsub_rn(theta_at(k, G), delta_at(k, G, rowlen));
    } else {
      v = warm_ef ? ef_at(k, G) : 0.0f;
    }
    if (out_bf16) static_cast<uint16_t*>(out)[i] = bf16_bits_rn(v);
    else static_cast<float*>(out)[i] = v;
  }
}

}  // namespace

extern "C" {

// Fill out[0..n) with the values of `what` (0 theta, 1 theta_local, 2 e) for
// global indices [G0, G0+n) of peer `peer`.  out is a device pointer (fp32, or
// bf16 bit patterns when out_bf16).  Returns a cudaError_t value.
int slcgen_fill_cuda(int what, uint64_t seed, int peer, uint64_t G0, uint64_t n, int rowlen,
                     int special_period, int warm_ef, int out_bf16, void* out, void* stream) {
  if (what < 0 || what > 2 || rowlen <= 0 || (out_bf16 && what == 2)) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  Keys k;
  k.theta = stream_key(seed, S_THETA);
  k.delta = stream_key(seed, (uint64_t)(S_DELTA + peer));
  k.rowscale = stream_key(seed, (uint64_t)(S_ROWSCALE + peer));
  k.ef = stream_key(seed, (uint64_t)(S_EF + peer));
  k.special = stream_key(seed, S_SPECIAL);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (n + 255) / 256;
  uint64_t cap = (uint64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      what, k, G0, n, (uint64_t)rowlen, (uint64_t)(special_period > 0 ? special_period : 0), warm_ef,
      out_bf16, out);
  return (int)cudaGetLastError();
}

}  // extern "C"
