// Row-group helpers shared by the row-moving kernels (pool, update, gather).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "table.cuh"

namespace hps {

template <typename T>
__device__ __forceinline__ T ld_volatile(const T* p) {
  return *const_cast<const volatile T*>(p);
}

__device__ __forceinline__ bool slot_ok(const DevTable& t, uint32_t s) { return s < t.capacity; }

template <int V>
__device__ __forceinline__ void load_vec(const float* p, float (&v)[V]) {
  if constexpr (V == 4) {
    float4 x = *reinterpret_cast<const float4*>(p);
    v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
  } else if constexpr (V == 2) {
    float2 x = *reinterpret_cast<const float2*>(p);
    v[0] = x.x, v[1] = x.y;
  } else {
    v[0] = *p;
  }
}

// Streaming (evict-first) load for data read exactly once.
template <int V>
__device__ __forceinline__ void load_vec_cs(const float* p, float (&v)[V]) {
  if constexpr (V == 4) {
    float4 x = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
  } else if constexpr (V == 2) {
    float2 x = __ldcs(reinterpret_cast<const float2*>(p));
    v[0] = x.x, v[1] = x.y;
  } else {
    v[0] = __ldcs(p);
  }
}

// Load with an L2 evict_last policy: data read again by a later kernel of the same step.
template <int V, int kPct = 100>
__device__ __forceinline__ void load_vec_keep(const float* p, float (&v)[V]) {
  if constexpr (V == 4) {
    asm volatile(
        "{.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_last.L2::evict_first.b64 pol, %5;\n\t"
        "ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], pol;}"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
        : "l"(p), "f"(kPct / 100.0f));
  } else {
    load_vec<V>(p, v);
  }
}

template <int V>
__device__ __forceinline__ void store_vec(float* p, const float (&v)[V]) {
  if constexpr (V == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

// Streaming store for outputs nobody in this step reads again.
template <int V>
__device__ __forceinline__ void store_vec_cs(float* p, const float (&v)[V]) {
  if constexpr (V == 4) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  } else if constexpr (V == 2) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(v[0], v[1]));
  } else {
    __stcs(p, v[0]);
  }
}

// Row-group geometry: L lanes x V floats cover kSpan = L*V dims per chunk; a row of D
// dims takes ceil(D / kSpan) chunks (1 on the specialised paths). kGuard enables the
// d < D bounds check of the generic path.
template <int V, int L, bool kGuard>
struct Geo {
  static constexpr int kSpan = V * L;
  __device__ static int lane() { return threadIdx.x % L; }
  __device__ static uint64_t group() {
    return (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / L;
  }
  __device__ static uint64_t groups() { return static_cast<uint64_t>(gridDim.x) * blockDim.x / L; }
};

// Dispatch on embedding dim: 128-bit row groups where D allows, else the generic
// one-float-per-lane path (any D).
#define HPS_DISPATCH_DIM(D, ...)                                                              \
  do {                                                                                        \
    switch (D) {                                                                              \
      case 1: { constexpr int V = 1, L = 1; constexpr bool G = false; __VA_ARGS__; } break;   \
      case 2: { constexpr int V = 2, L = 1; constexpr bool G = false; __VA_ARGS__; } break;   \
      case 4: { constexpr int V = 4, L = 1; constexpr bool G = false; __VA_ARGS__; } break;   \
      case 8: { constexpr int V = 4, L = 2; constexpr bool G = false; __VA_ARGS__; } break;   \
      case 16: { constexpr int V = 4, L = 4; constexpr bool G = false; __VA_ARGS__; } break;  \
      case 32: { constexpr int V = 4, L = 8; constexpr bool G = false; __VA_ARGS__; } break;  \
      case 64: { constexpr int V = 4, L = 16; constexpr bool G = false; __VA_ARGS__; } break; \
      case 128: { constexpr int V = 4, L = 32; constexpr bool G = false; __VA_ARGS__; } break; \
      default: { constexpr int V = 1, L = 32; constexpr bool G = true; __VA_ARGS__; } break;  \
    }                                                                                         \
  } while (0)

}  // namespace hps
