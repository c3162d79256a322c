// The reference's lossy value codec on the device (codec.hpp:
// 30-103, 208-261): each block of `block_len` floats (one embedding row on the wire,
// embedding_worker.hpp:48-85) is scaled by kappa / ||block||_inf (1.0 for an all-zero
// block) and rounded to IEEE binary16, round-to-nearest-even with subnormals
// (float_to_half_bits); decompression widens (half_bits_to_float) and divides by the
// scale. Every operation is the reference's single rounded float operation, so the
// payload and the round trip are bit-identical to compress_values / decompress_values.
//
// One warp per block: a shuffle max-reduction of |v|, then the lanes convert their
// elements. cvt.rn.f16.f32 is exactly float_to_half_bits for every finite input (and
// non-finite inputs are rejected, as the reference does).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "table.cuh"
#include "table_impl.h"

namespace hps {

namespace {

__global__ void compress_kernel(const float* __restrict__ v, uint64_t rows, uint32_t len,
                                float kappa, float* __restrict__ scales,
                                uint16_t* __restrict__ payload, unsigned int* bad) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += warps) {
    const float* x = v + r * len;
    float m = 0.0f;
    bool nonfinite = false;
    for (uint32_t i = lane; i < len; i += 32) {
      const float a = x[i];
      nonfinite |= !isfinite(a);
      m = fmaxf(m, fabsf(a));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (__any_sync(0xffffffffu, nonfinite)) {
      if (lane == 0) atomicExch(bad, 1u);  // compress_values: non-finite input
      continue;
    }
    const float scale = m == 0.0f ? 1.0f : __fdiv_rn(kappa, m);
    if (lane == 0) scales[r] = scale;
    uint16_t* out = payload + r * len;
    for (uint32_t i = lane; i < len; i += 32)
      out[i] = m == 0.0f ? 0u : __half_as_ushort(__float2half_rn(__fmul_rn(x[i], scale)));
  }
}

__global__ void decompress_kernel(const float* __restrict__ scales,
                                  const uint16_t* __restrict__ payload, uint64_t rows,
                                  uint32_t len, float* __restrict__ out, unsigned int* bad) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += warps) {
    const float scale = scales[r];
    if (!(scale > 0.0f) || !isfinite(scale)) {  // decompress_values: bad scale
      if (lane == 0) atomicExch(bad, 1u);
      continue;
    }
    const uint16_t* p = payload + r * len;
    float* o = out + r * len;
    for (uint32_t i = lane; i < len; i += 32) {
      const float w = __half2float(__ushort_as_half(p[i]));
      if (!isfinite(w)) atomicExch(bad, 2u);  // non-finite payload value
      o[i] = __fdiv_rn(w, scale);
    }
  }
}

uint32_t codec_grid(uint64_t rows) {
  return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(rows, 8), 148ull * 32)));
}

}  // namespace

void compress_values(const float* v, uint64_t rows, uint32_t len, float kappa, float* scales,
                     uint16_t* payload, cudaStream_t st) {
  if (!(kappa > 0.0f)) throw Error(HPS_E_PRECONDITION, "compress_values: kappa must be positive");
  if (!rows || !len) return;
  StagePool pool;
  Stager stg(pool);
  const float* d_v = static_cast<const float*>(stg.in(v, rows * len * sizeof(float), st));
  float* d_s = static_cast<float*>(stg.out(scales, rows * sizeof(float)));
  uint16_t* d_p = static_cast<uint16_t*>(stg.out(payload, rows * len * sizeof(uint16_t)));
  unsigned int* d_bad = nullptr;
  HPS_CUDA(cudaMallocAsync(&d_bad, sizeof(unsigned int), st));
  HPS_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned int), st));
  launch(compress_kernel, codec_grid(rows), 256, 0, st, d_v, rows, len, kappa, d_s, d_p, d_bad);
  HPS_LAUNCH_CHECK();
  unsigned int bad = 0;
  HPS_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaFreeAsync(d_bad, st));
  stg.finish(st);
  HPS_CUDA(cudaStreamSynchronize(st));
  if (bad) throw Error(HPS_E_PRECONDITION, "compress_values: non-finite input");
}

void decompress_values(const float* scales, const uint16_t* payload, uint64_t rows, uint32_t len,
                       float* out, cudaStream_t st) {
  if (!rows || !len) return;
  StagePool pool;
  Stager stg(pool);
  const float* d_s = static_cast<const float*>(stg.in(scales, rows * sizeof(float), st));
  const uint16_t* d_p =
      static_cast<const uint16_t*>(stg.in(payload, rows * len * sizeof(uint16_t), st));
  float* d_o = static_cast<float*>(stg.out(out, rows * len * sizeof(float)));
  unsigned int* d_bad = nullptr;
  HPS_CUDA(cudaMallocAsync(&d_bad, sizeof(unsigned int), st));
  HPS_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned int), st));
  launch(decompress_kernel, codec_grid(rows), 256, 0, st, d_s, d_p, rows, len, d_o, d_bad);
  HPS_LAUNCH_CHECK();
  unsigned int bad = 0;
  HPS_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaFreeAsync(d_bad, st));
  stg.finish(st);
  HPS_CUDA(cudaStreamSynchronize(st));
  if (bad == 1) throw Error(HPS_E_PROTOCOL, "decompress_values: bad scale");
  if (bad) throw Error(HPS_E_PROTOCOL, "decompress_values: non-finite payload value");
}

}  // namespace hps
