// Throughput (thread-ops per SM clock) of the conversions the decode needs:
// Delta = RN32(RN64(v * c)), v int32, c fp64.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double i2d_magic(int v) {  // exact int32 -> double via one DADD
  return __hiloint2double(0x43300000, (int)((unsigned)v ^ 0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}
__device__ __forceinline__ float d2f_int(double x) {  // RN-even double -> float, normal results only
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  const unsigned long long t = u + 0x0FFFFFFFull + ((u >> 29) & 1ull);
  const unsigned long long m = t >> 29;  // sign | exp11 | mant23 (rounded, carries into the exponent)
  const unsigned int e = (unsigned int)(m >> 23) & 0x7FFu;
  const unsigned int f = ((unsigned int)(m >> 34) << 31) | ((e - 896u) << 23) | ((unsigned int)m & 0x7FFFFFu);
  return __uint_as_float(f);
}

template <int K>
__global__ void chain(const int* in, float* out, double c, int iters) {
  int v = in[threadIdx.x & 31] + threadIdx.x + 1000;
  float acc = 0.f;
#pragma unroll 8
  for (int i = 0; i < iters; i++) {
    const int w = v + i;
    float r;
    if (K == 0) r = __double2float_rn(__dmul_rn((double)w, c));
    if (K == 1) r = __double2float_rn(__dmul_rn(i2d_magic(w), c));
    if (K == 2) r = d2f_int(__dmul_rn(i2d_magic(w), c));
    if (K == 3) r = __fmul_rn(__int2float_rn(w), (float)c);
    if (K == 4) r = (float)__double_as_longlong(__dmul_rn(__longlong_as_double((long long)w), c));
    acc += r;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void check(float* bad, double c) {
  int w = blockIdx.x * blockDim.x + threadIdx.x - (1 << 29);
  for (int k = 0; k < 64; k++, w += 104729 * 97) {
    float a = __double2float_rn(__dmul_rn((double)w, c));
    float b = d2f_int(__dmul_rn(i2d_magic(w), c));
    if (w != 0 && __float_as_uint(a) != __float_as_uint(b)) atomicAdd(bad, 1.0f);
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int* in; float* out;
  cudaMalloc(&in, 128); cudaMemset(in, 0, 128);
  cudaMalloc(&out, (size_t)sms * 8 * 1024 * 4);
  const int blocks = sms * 4, threads = 512, iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads * iters;
    printf("%-40s %8.3f ms  %7.1f per clk per SM\n", name, ms, ops / (ms * 1e-3) / (clk * 1e3) / sms);
  };
  const double c = 0.05 * 0x1p-10;
  run("I2F.F64 + DMUL + F2F.F32.F64", [&] { chain<0><<<blocks, threads>>>(in, out, c, iters); });
  run("magic DADD + DMUL + F2F.F32.F64", [&] { chain<1><<<blocks, threads>>>(in, out, c, iters); });
  run("magic DADD + DMUL + integer RN", [&] { chain<2><<<blocks, threads>>>(in, out, c, iters); });
  run("I2F + FMUL (fp32, pow2 R)", [&] { chain<3><<<blocks, threads>>>(in, out, c, iters); });
  run("DMUL only", [&] { chain<4><<<blocks, threads>>>(in, out, c, iters); });
  float* bad; cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  for (double cc : {0.05, 1.0 / 3, 1.0 / 49, 1.0 / 20 * 0x1p-20, 1.0 / 7 * 0x1p-30}) check<<<4096, 256>>>(bad, cc);
  float hb; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("integer-RN mismatches vs F2F: %.0f (of %d)\n", hb, 5 * 4096 * 256 * 64);
  return 0;
}
