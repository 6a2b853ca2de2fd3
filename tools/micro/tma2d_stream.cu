// 2-D tensor-map TMA streaming of 64x64 blocks of a row-major (rows x cols)
// matrix (the theta blocks of the fused update): RMW through shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(su(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void ld2d(void* d, const void* m, int x, int y, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(su(d)), "l"(m), "r"(x), "r"(y), "r"(su(b)) : "memory");
}
__device__ __forceinline__ void st2d(const void* m, int x, int y, const void* s) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(x), "r"(y), "r"(su(s)) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

template <int NT, int D, int EB, int MAPMODE>
__global__ void stream2d(const CUtensorMap* gmap, const __grid_constant__ CUtensorMap pmap, long nblk, int bcols) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  unsigned char* tiles = sm + 128;
  const int TB = 4096 * EB;
  const void* map = MAPMODE == 0 ? (const void*)gmap : (const void*)&pmap;
  const long G = gridDim.x;
  const long my = (nblk - blockIdx.x + G - 1) / G;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NT; k++) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto blk = [&](long i, int& x, int& y) { long q = blockIdx.x + i * G; x = (int)(q % bcols) * 64; y = (int)(q / bcols) * 64; };
  if (threadIdx.x == 0)
    for (long i = 0; i < D && i < my; i++) {
      int x, y; blk(i, x, y);
      expect(&bar[i % NT], TB); ld2d(tiles + (i % NT) * TB, map, x, y, &bar[i % NT]); commit();
    }
  for (long i = 0; i < my; i++) {
    if (threadIdx.x == 0 && i + D < my) {
      wait_read<NT - D - 1>();
      const long k = i + D; int x, y; blk(k, x, y);
      expect(&bar[k % NT], TB); ld2d(tiles + (k % NT) * TB, map, x, y, &bar[k % NT]);
    }
    while (!try_wait(&bar[i % NT], (uint32_t)((i / NT) & 1))) {}
    unsigned char* t = tiles + (i % NT) * TB;
    for (int j = threadIdx.x; j < TB / 4; j += blockDim.x) reinterpret_cast<uint32_t*>(t)[j] += 1u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) { int x, y; blk(i, x, y); st2d(map, x, y, t); commit(); }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  const long rows = 4096 * 8, cols = 8192;  // 256 M elements
  void* x; cudaMalloc(&x, rows * cols * 4); cudaMemset(x, 0, rows * cols * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  CUtensorMap* dmap; cudaMalloc(&dmap, sizeof(CUtensorMap));
  for (int eb : {4, 2}) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t str[1] = {(cuuint64_t)cols * eb};
    const cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    CUresult r = enc(&m, eb == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", r); return 1; }
    cudaMemcpy(dmap, &m, sizeof(m), cudaMemcpyHostToDevice);
    const long nblk = (rows / 64) * (cols / 64);
    auto run = [&](const char* name, auto kern, int nt, int cpsm) {
      size_t smem = 128 + (size_t)nt * 4096 * eb;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<sms * cpsm, 256, smem>>>(dmap, m, nblk, (int)(cols / 64)); cudaDeviceSynchronize();
      cudaEventRecord(a); kern<<<sms * cpsm, 256, smem>>>(dmap, m, nblk, (int)(cols / 64)); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("eb=%d %-36s %7.3f ms %7.0f GB/s (%s)\n", eb, name, ms, 2.0 * rows * cols * eb / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    if (eb == 4) {
      run("gmem map NT=4 D=2 2/SM", stream2d<4, 2, 4, 0>, 4, 2);
      run("param map NT=4 D=2 2/SM", stream2d<4, 2, 4, 1>, 4, 2);
      run("gmem map NT=6 D=4 2/SM", stream2d<6, 4, 4, 0>, 6, 2);
      run("gmem map NT=12 D=10 1/SM", stream2d<12, 10, 4, 0>, 12, 1);
    } else {
      run("gmem map NT=8 D=6 2/SM", stream2d<8, 6, 2, 0>, 8, 2);
      run("param map NT=8 D=6 2/SM", stream2d<8, 6, 2, 1>, 8, 2);
      run("gmem map NT=4 D=2 2/SM", stream2d<4, 2, 2, 0>, 4, 2);
    }
  }
  return 0;
}
