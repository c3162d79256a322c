// NVLink peer-write microbenchmark (profiling aid, not product code): GPU 0 writes
// 109 MB of 256-byte rows (gathered from random local rows) into GPU 1's memory,
//   A: 16 lanes x float4 stores per row (what x_owner_gather does)
//   B: rows staged in shared memory, written with cp.async.bulk (TMA) 8 KB at a time
//   C: cudaMemcpyPeerAsync of the same bytes (copy engines, contiguous)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/p2p_bench tools/p2p_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void wr_plain(const float4* __restrict__ src, const uint32_t* __restrict__ idx,
                         float4* __restrict__ dst, uint32_t n) {
  const uint32_t lane = threadIdx.x & 15;
  const uint64_t groups = (uint64_t)gridDim.x * blockDim.x / 16;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 16; r < n; r += groups)
    dst[r * 16 + lane] = src[(uint64_t)idx[r] * 16 + lane];
}

// 32 rows (8 KB) per chunk; warp w of the block gathers 4 rows, then one thread issues a
// bulk copy of the chunk to the peer.
__global__ void __launch_bounds__(256) wr_bulk(const float4* __restrict__ src,
                                               const uint32_t* __restrict__ idx,
                                               float4* __restrict__ dst, uint32_t n) {
  __shared__ __align__(128) float4 buf[2][32 * 16];
  const uint32_t lane = threadIdx.x & 15, grp = threadIdx.x >> 4;  // 16 groups
  int b = 0;
  for (uint64_t c = blockIdx.x; c * 32 < n; c += gridDim.x, b ^= 1) {
    const uint64_t r0 = c * 32;
    // make sure the bulk copy that used this buffer two chunks ago has read it
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    for (int k = 0; k < 2; ++k) {
      const uint64_t r = r0 + grp * 2 + k;
      if (r < n) buf[b][(grp * 2 + k) * 16 + lane] = src[(uint64_t)idx[r] * 16 + lane];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t rows = (uint32_t)((n - r0) < 32 ? (n - r0) : 32);
      const uint32_t s = (uint32_t)__cvta_generic_to_shared(&buf[b][0]);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   :: "l"(dst + r0 * 16), "r"(s), "r"(rows * 256) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int n_dev = 0;
  CK(cudaGetDeviceCount(&n_dev));
  if (n_dev < 2) { printf("need 2 GPUs\n"); return 0; }
  const uint32_t n = 425984, rows_total = 100000000 / 64;  // 1.56M source rows
  CK(cudaSetDevice(1));
  float4* peer;
  CK(cudaMalloc(&peer, (size_t)n * 256));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  float4 *src, *loc;
  uint32_t* idx;
  CK(cudaMalloc(&src, (size_t)rows_total * 256));
  CK(cudaMalloc(&loc, (size_t)n * 256));
  CK(cudaMalloc(&idx, n * 4));
  uint32_t* h = (uint32_t*)malloc(n * 4);
  uint64_t x = 88172645463325252ull;
  for (uint32_t i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = x % rows_total; }
  CK(cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
    printf("%-28s %8.1f us  %7.1f GB/s  (%s)\n", name, ms * 1000, n * 256.0 / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  run("plain stores -> local", [&] { wr_plain<<<148 * 16, 256>>>(src, idx, loc, n); });
  run("plain stores -> peer", [&] { wr_plain<<<148 * 16, 256>>>(src, idx, peer, n); });
  run("bulk (TMA) -> local", [&] { wr_bulk<<<148 * 4, 256>>>(src, idx, loc, n); });
  run("bulk (TMA) -> peer", [&] { wr_bulk<<<148 * 4, 256>>>(src, idx, peer, n); });
  run("bulk (TMA) -> peer g8", [&] { wr_bulk<<<148 * 8, 256>>>(src, idx, peer, n); });
  run("memcpyPeer contiguous", [&] { cudaMemcpyPeerAsync(peer, 1, loc, 0, (size_t)n * 256); });
  return 0;
}
