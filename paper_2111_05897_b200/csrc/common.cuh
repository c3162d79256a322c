// Shared device helpers for the embedding hot path (sm_100a).
//
// Bit-exactness rules: every float/double operation that
// the reference performs as a separately-rounded C++ expression is written with
// an explicit round-to-nearest intrinsic (__fadd_rn, __fmul_rn, __dadd_rn, ...),
// which nvcc never contracts into an FMA. The library is also built with
// --fmad=false as a second guard.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../include/hps_c.h"

namespace hps {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;  // core.hpp:32
constexpr uint64_t kMul1 = 0xbf58476d1ce4e5b9ULL;   // core.hpp:33
constexpr uint64_t kMul2 = 0x94d049bb133111ebULL;   // core.hpp:34
constexpr uint64_t kEmptyKey = ~0ull;              // hash-table empty marker
constexpr uint32_t kPending = 0xffffffffu;          // slot not yet published
constexpr uint32_t kInvalidSlot = 0xfffffffeu;      // insert failed (capacity)
constexpr uint32_t kNoStep = 0xffffffffu;           // PsShard::kNoStep embedding_ps.hpp:61
constexpr uint32_t kTagRing = 16;                   // PsShard::kTagRing embedding_ps.hpp:60
constexpr float kAdagradEps = 1e-10f;               // embedding_ps.hpp:39
constexpr uint64_t kTableHashSalt = 0x6a09e667f3bcc909ULL;

// Thrown inside the library, mapped to hps_status at the C boundary.
struct Error : std::runtime_error {
  hps_status code;
  Error(hps_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define HPS_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess)                                                               \
      throw ::hps::Error(HPS_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// Every kernel launch of the library is counted (hps_launch_count), so a caller can
// prove how many of these kernels ran inside a timed region.
inline std::atomic<unsigned long long> g_launches{0};

#define HPS_LAUNCH_CHECK_N(k)                                      \
  do {                                                             \
    ::hps::g_launches.fetch_add((k), std::memory_order_relaxed);   \
    HPS_CUDA(cudaGetLastError());                                  \
  } while (0)
#define HPS_LAUNCH_CHECK() HPS_LAUNCH_CHECK_N(1)

// Programmatic dependent launch (PDL). Every kernel of the library starts with
// pdl_entry(): griddepcontrol.wait (the previous grid of the stream has completed and
// its writes are visible -- so nothing a kernel reads can race its predecessor, and by
// induction any earlier kernel), then griddepcontrol.launch_dependents (the next grid
// may be scheduled now). launch() issues kernels with the programmatic-serialization
// attribute, so the next kernel's launch and block rasterisation overlap this one's
// tail instead of following its completion; a step is ~15 short dependent kernels,
// most of them a few microseconds (measured 0.2753 -> 0.2693 ms per C2 step with PDL,
// profiles/r1_pdl_ab.txt). Outside a PDL launch both instructions are no-ops.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   cudaStream_t st, Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HPS_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += kGamma;
  x ^= x >> 30;
  x *= kMul1;
  x ^= x >> 27;
  x *= kMul2;
  x ^= x >> 31;
  return x;
}

// route_shard, core.hpp:145-150.
__host__ __device__ __forceinline__ uint32_t route_shard(uint64_t id, uint32_t shard_count) {
  return static_cast<uint32_t>(mix64(id) % shard_count);
}

// Lazy-init element d of a fresh row (embedding_ps.hpp:424-428): the d-th draw of
// Rng(seed) is mix64(seed + d*gamma) (core.hpp:53-57); uniform01 takes the top 53
// bits (:60); uniform(lo, hi) = lo + (hi - lo) * u (:63), evaluated in double with
// each operation rounded, then narrowed to float. Random access into the stream
// lets every lane initialise its own dimension.
__device__ __forceinline__ float init_value(uint64_t seed, uint32_t d, double lo, double span) {
  uint64_t r = mix64(seed + static_cast<uint64_t>(d) * kGamma);
  double u = __dmul_rn(static_cast<double>(r >> 11), 0x1.0p-53);
  return __double2float_rn(__dadd_rn(lo, __dmul_rn(span, u)));
}

__host__ __device__ __forceinline__ uint32_t ceil_div(uint64_t a, uint64_t b) {
  return static_cast<uint32_t>((a + b - 1) / b);
}

inline int bits_for(uint64_t max_value) {  // bits needed to represent [0, max_value]
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b;
}

}  // namespace hps
