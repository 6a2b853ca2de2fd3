// peer_copy.cu — rows a8 / a9 over NVLink peer memory: one kernel copies a
// list of byte ranges whose sources (or destinations) are peer mappings of
// other GPUs' buffers (CUDA IPC / symmetric memory).  Every SM pulls: 16-B
// vector loads, 8 per thread in flight (32 KB per CTA), so all NVLink links
// of the GPU stream at once; no copy-engine queue, no NCCL protocol.
#include <algorithm>

#include "slc_internal.cuh"

namespace slc {
namespace {

constexpr int kPcThreads = 256, kPcUnroll = 8;
constexpr int64_t kPcTile = (int64_t)kPcThreads * kPcUnroll * 16;  // 32 KB per CTA step

struct PcSeg {
  const char* src;
  char* dst;
  int64_t bytes;
  int64_t tile0;  // first global tile index of this segment
};

__global__ void __launch_bounds__(kPcThreads) peer_copy_kernel(const PcSeg* segs, int nseg, int64_t ntiles) {
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // segment of this tile (few segments: linear scan)
    int s = 0;
    while (s + 1 < nseg && segs[s + 1].tile0 <= tile) s++;
    const PcSeg g = segs[s];
    const int64_t base = (tile - g.tile0) * kPcTile;
    const int64_t n = min(kPcTile, g.bytes - base);
    if ((n & 15) == 0 && ((uintptr_t)(g.src + base) & 15) == 0 && ((uintptr_t)(g.dst + base) & 15) == 0) {
      uint4 v[kPcUnroll];
#pragma unroll
      for (int u = 0; u < kPcUnroll; u++) {
        const int64_t o = ((int64_t)u * kPcThreads + threadIdx.x) * 16;
        if (o < n) v[u] = *reinterpret_cast<const uint4*>(g.src + base + o);
      }
#pragma unroll
      for (int u = 0; u < kPcUnroll; u++) {
        const int64_t o = ((int64_t)u * kPcThreads + threadIdx.x) * 16;
        if (o < n) *reinterpret_cast<uint4*>(g.dst + base + o) = v[u];
      }
    } else {
      for (int64_t o = threadIdx.x; o < n; o += kPcThreads) g.dst[base + o] = g.src[base + o];
    }
  }
}

}  // namespace

cudaError_t launch_peer_copy(const void* const* src, void* const* dst, const int64_t* bytes, int n, void* dev_scratch,
                             cudaStream_t s) {
  PcSeg h[kMaxPeers];
  int64_t t = 0;
  int m = 0;
  for (int i = 0; i < n; i++) {
    if (bytes[i] <= 0) continue;
    h[m].src = static_cast<const char*>(src[i]);
    h[m].dst = static_cast<char*>(dst[i]);
    h[m].bytes = bytes[i];
    h[m].tile0 = t;
    t += (bytes[i] + kPcTile - 1) / kPcTile;
    m++;
  }
  if (m == 0) return cudaSuccess;
  cudaError_t e = cudaMemcpyAsync(dev_scratch, h, sizeof(PcSeg) * m, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(t, (int64_t)sms * 8);
  peer_copy_kernel<<<grid, kPcThreads, 0, s>>>(static_cast<const PcSeg*>(dev_scratch), m, t);
  return cudaGetLastError();
}

size_t peer_copy_scratch_bytes() { return sizeof(PcSeg) * kMaxPeers; }

}  // namespace slc
