// Cost breakdown of the update pattern on B200 (profiling aid, not product code).
// One warp per random 512-byte row [w 64 | acc 64], 425,984 rows per launch, adding
// the update kernel's ingredients one at a time:
//   v1 row RMW only                          v2 + sequential 256 B gradient read
//   v3 + 8 B version word RMW (random)       v4 + Adagrad math (IEEE div/sqrt)
//   v5 = v4 with two rows in flight per warp
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench2 tools/microbench2.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

template <int kVariant, int kRows>
__global__ void __launch_bounds__(256) upd(float4* __restrict__ rows, uint2* __restrict__ vt,
                                           const uint32_t* __restrict__ idx,
                                           const float4* __restrict__ grads, size_t n) {
  const int lane = threadIdx.x & 31;
  const int q = lane & 15;
  const size_t warps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t w0 = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5; w0 < n;
       w0 += warps * kRows) {
    float4 x[kRows], g[kRows];
    uint32_t s[kRows];
    uint2 v[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      size_t w = w0 + r * warps;
      s[r] = w < n ? idx[w] : 0;
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      size_t w = w0 + r * warps;
      if (w >= n) continue;
      x[r] = rows[(size_t)s[r] * 32 + lane];
      if (kVariant >= 2) g[r] = __ldcs(grads + w * 16 + q);
      if (kVariant >= 3 && lane == 0) v[r] = vt[s[r]];
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      size_t w = w0 + r * warps;
      if (w >= n) continue;
      float4 y = x[r];
      if (kVariant >= 4) {
        float c[4] = {g[r].x, g[r].y, g[r].z, g[r].w};
        float vv[4] = {y.x, y.y, y.z, y.w};
        float an[4];
        for (int k = 0; k < 4; ++k) an[k] = __fadd_rn(vv[k], __fmul_rn(c[k], c[k]));
        for (int k = 0; k < 4; ++k) an[k] = __shfl_down_sync(0xffffffffu, an[k], 16);
        if (lane >= 16) {
          for (int k = 0; k < 4; ++k) vv[k] = __fadd_rn(vv[k], __fmul_rn(c[k], c[k]));
        } else {
          for (int k = 0; k < 4; ++k)
            vv[k] = __fsub_rn(vv[k], __fdiv_rn(__fmul_rn(0.05f, c[k]),
                                                __fadd_rn(__fsqrt_rn(an[k]), 1e-10f)));
        }
        y = make_float4(vv[0], vv[1], vv[2], vv[3]);
      } else if (kVariant >= 2) {
        y.x += g[r].x;
      } else {
        y.x += 1.0f;
      }
      rows[(size_t)s[r] * 32 + lane] = y;
      if (kVariant >= 3 && lane == 0) vt[s[r]] = make_uint2(v[r].x + 1, v[r].y);
    }
  }
}

int main() {
  const size_t R = 100000000, N = 425984;
  float4 *rows, *grads;
  uint2* vt;
  uint32_t* idx;
  cudaMalloc(&rows, R * 512);
  cudaMalloc(&vt, R * 8);
  cudaMalloc(&grads, 8 * N * 256);
  cudaMalloc(&idx, 8 * N * 4);
  cudaMemset(rows, 0, R * 512);
  cudaMemset(vt, 0, R * 8);
  cudaMemset(grads, 0, 8 * N * 256);
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
  auto time = [&](auto kern, int bpsm) {
    kern<<<148 * bpsm, 256>>>(rows, vt, idx, grads, N);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 16; ++r)
      kern<<<148 * bpsm, 256>>>(rows, vt, idx + (r % 8) * N, grads + (r % 8) * N * 16, N);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 16 * 1e3;
  };
  for (int bpsm : {8, 16, 32}) {
    printf("bpsm=%2d v1 rmw %.1f us | v2 +grad %.1f | v3 +vt %.1f | v4 +adagrad %.1f | v5 2rows %.1f\n",
           bpsm, time(upd<1, 1>, bpsm), time(upd<2, 1>, bpsm), time(upd<3, 1>, bpsm),
           time(upd<4, 1>, bpsm), time(upd<4, 2>, bpsm));
  }
  // the same rows visited in ascending slot order (each batch's index list sorted): DRAM
  // page / TLB locality of a slot-ordered update
  for (int b = 0; b < 8; ++b) std::sort(h.begin() + b * N, h.begin() + (b + 1) * N);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  for (int bpsm : {8, 16}) {
    printf("sorted bpsm=%2d v1 rmw %.1f us | v2 +grad %.1f | v4 +adagrad %.1f | v5 2rows %.1f\n",
           bpsm, time(upd<1, 1>, bpsm), time(upd<2, 1>, bpsm), time(upd<4, 1>, bpsm),
           time(upd<4, 2>, bpsm));
  }
  return 0;
}
