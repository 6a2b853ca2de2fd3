// Streaming read-modify-write of 16 KB tiles through shared memory with 1-D bulk
// copies (TMA engine): how many bytes in flight does B200 need?  Each CTA walks
// tiles t = blockIdx + i*grid; a ring of NT tiles, loads D ahead; the update is
// x += 1 by all threads (or nothing); store back with bulk S2G.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(su(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}
__device__ __forceinline__ void s2g(void* d, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(su(s)), "r"(n) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

template <int NT, int D, bool STORE, bool TOUCH>
__global__ void stream(float* x, long ntiles) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  float* tiles = reinterpret_cast<float*>(sm + 128);
  const long G = gridDim.x;
  const long my = (ntiles - blockIdx.x + G - 1) / G;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NT; k++) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto tile = [&](long i) { return tiles + (i % NT) * 4096; };
  if (threadIdx.x == 0)
    for (long i = 0; i < D && i < my; i++) {
      expect(&bar[i % NT], 16384);
      g2s(tile(i), x + (blockIdx.x + i * G) * 4096, 16384, &bar[i % NT]);
      commit();
    }
  for (long i = 0; i < my; i++) {
    if (threadIdx.x == 0 && i + D < my) {
      if (STORE) wait_read<NT - D - 1>();
      const long k = i + D;
      expect(&bar[k % NT], 16384);
      g2s(tile(k), x + (blockIdx.x + k * G) * 4096, 16384, &bar[k % NT]);
    }
    while (!try_wait(&bar[i % NT], (uint32_t)((i / NT) & 1))) {}
    if (TOUCH) {
      float* t = tile(i);
      for (int j = threadIdx.x; j < 4096; j += blockDim.x) t[j] += 1.0f;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (STORE) s2g(x + (blockIdx.x + i * G) * 4096, tile(i), 16384);
      commit();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long ntiles = 2L * 1024 * 1024 * 1024 / 16384;  // 8 GB of fp32
  float* x; cudaMalloc(&x, ntiles * 16384); cudaMemset(x, 0, ntiles * 16384);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern, int nt, int ctas_per_sm, bool store) {
    size_t smem = 128 + (size_t)nt * 16384;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int grid = sms * ctas_per_sm;
    kern<<<grid, 256, smem>>>(x, ntiles);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    kern<<<grid, 256, smem>>>(x, ntiles);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)ntiles * 16384 * (store ? 2 : 1);
    printf("%-44s %7.3f ms %7.0f GB/s  (%s)\n", name, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run("load only  NT=4 D=3  1 CTA/SM", stream<4, 3, false, false>, 4, 1, false);
  run("load only  NT=8 D=7  1 CTA/SM", stream<8, 7, false, false>, 8, 1, false);
  run("load only  NT=4 D=3  2 CTA/SM", stream<4, 3, false, false>, 4, 2, false);
  run("rmw NT=4 D=2 2 CTA/SM", stream<4, 2, true, true>, 4, 2, true);
  run("rmw NT=6 D=4 2 CTA/SM", stream<6, 4, true, true>, 6, 2, true);
  run("rmw NT=8 D=6 1 CTA/SM", stream<8, 6, true, true>, 8, 1, true);
  run("rmw NT=12 D=10 1 CTA/SM", stream<12, 10, true, true>, 12, 1, true);
  run("rmw NT=4 D=2 3 CTA/SM", stream<4, 2, true, true>, 4, 3, true);
  run("copy-only(no touch) NT=6 D=4 2 CTA/SM", stream<6, 4, true, false>, 6, 2, true);
  return 0;
}
