// Memory-system ceilings on this B200 for the access patterns of the hot path
// (profiling aid, not product code). Reports GB/s for:
//   copy      : streaming read+write of 1 GiB (the MEASURED_PEAKS pattern)
//   rmw512    : random 512-byte row read-modify-write (update kernel pattern)
//   gather256 : random 256-byte row read + sequential 256-byte write (pool pattern)
//   read512   : random 512-byte row read only
// Rows: 100M x 512 B table (51.2 GB), 425,984 random rows per launch.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o microbench tools/microbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// 32 lanes per 512-byte row: lane l moves float4 l.
__global__ void rmw512_kernel(float4* __restrict__ rows, const uint32_t* __restrict__ idx,
                              size_t n) {
  const int lane = threadIdx.x & 31;
  for (size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((size_t)gridDim.x * blockDim.x) >> 5) {
    float4* r = rows + (size_t)idx[w] * 32;
    float4 v = r[lane];
    v.x += 1.0f;
    r[lane] = v;
  }
}

__global__ void read512_kernel(const float4* __restrict__ rows, const uint32_t* __restrict__ idx,
                               size_t n, float* sink) {
  const int lane = threadIdx.x & 31;
  float acc = 0;
  for (size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((size_t)gridDim.x * blockDim.x) >> 5) {
    float4 v = rows[(size_t)idx[w] * 32 + lane];
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.0f) *sink = acc;
}

// 16 lanes per 256-byte half row (the w part), written densely to out.
__global__ void gather256_kernel(const float4* __restrict__ rows,
                                 const uint32_t* __restrict__ idx, size_t n,
                                 float4* __restrict__ out) {
  const int lane = threadIdx.x & 15;
  for (size_t g = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 4; g < n;
       g += ((size_t)gridDim.x * blockDim.x) >> 4) {
    float4 v = rows[(size_t)idx[g] * 32 + lane];
    out[g * 16 + lane] = v;
  }
}

int main() {
  const size_t R = 100000000, N = 425984;
  float4 *rows, *a, *b, *out;
  uint32_t* idx;
  float* sink;
  cudaMalloc(&rows, R * 512);
  cudaMalloc(&a, 1ull << 30);
  cudaMalloc(&b, 1ull << 30);
  cudaMalloc(&out, N * 256);
  cudaMalloc(&idx, 8 * N * 4);
  cudaMalloc(&sink, 4);
  cudaMemset(rows, 0, R * 512);
  std::vector<uint32_t> h(8 * N);
  uint64_t x = 7;
  for (auto& v : h) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    v = (uint32_t)((x >> 33) % R);
  }
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](auto fn, int reps) {
    fn(0);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) fn(r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
  };
  int sms = 148;
  for (int bpsm : {4, 8, 16, 32}) {
    float ms = time([&](int) { copy_kernel<<<sms * bpsm, 256>>>(a, b, (1ull << 30) / 16); }, 10);
    printf("copy      blocks/SM=%2d  %8.1f us  %7.1f GB/s\n", bpsm, ms * 1e3, 2.0 * (1 << 30) / ms / 1e6);
  }
  for (int bpsm : {4, 8, 16, 32, 64}) {
    float ms = time([&](int r) { rmw512_kernel<<<sms * bpsm, 256>>>(rows, idx + (r % 8) * N, N); }, 16);
    printf("rmw512    blocks/SM=%2d  %8.1f us  %7.1f GB/s\n", bpsm, ms * 1e3, 2.0 * N * 512 / ms / 1e6);
  }
  for (int bpsm : {4, 8, 16, 32, 64}) {
    float ms = time([&](int r) { read512_kernel<<<sms * bpsm, 256>>>(rows, idx + (r % 8) * N, N, sink); }, 16);
    printf("read512   blocks/SM=%2d  %8.1f us  %7.1f GB/s\n", bpsm, ms * 1e3, 1.0 * N * 512 / ms / 1e6);
  }
  for (int bpsm : {4, 8, 16, 32, 64}) {
    float ms = time([&](int r) { gather256_kernel<<<sms * bpsm, 256>>>(rows, idx + (r % 8) * N, N, out); }, 16);
    printf("gather256 blocks/SM=%2d  %8.1f us  %7.1f GB/s\n", bpsm, ms * 1e3, 2.0 * N * 256 / ms / 1e6);
  }
  return 0;
}
