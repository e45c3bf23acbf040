// Shared device/host helpers for the hb200 rank-reveal path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "hb.h"

namespace hb {

// Error carrying an hb_status; converted to a status code at the C ABI (abi.cpp).
struct Error : std::runtime_error {
  hb_status status;
  Error(hb_status s, const std::string& what) : std::runtime_error(what), status(s) {}
};

#define HB_CUDA(x)                                                                           \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      throw ::hb::Error(e_ == cudaErrorMemoryAllocation ? HB_ENOMEM : HB_ECUDA,              \
                        std::string(#x) + ": " + cudaGetErrorString(e_) + " @" __FILE__ ":" + \
                            std::to_string(__LINE__));                                       \
  } while (0)

// Raise (never lower) a kernel's dynamic shared-memory limit on the current device.  Host threads
// (hb_sweep workers, concurrent sub-streams) launch the same kernels with different sizes: an
// attribute lowered between another thread's set and launch fails that launch ("too many resources
// requested" / "invalid argument").  Monotonic updates under one lock make that impossible.
inline void ensure_dyn_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;
  int dev = 0;
  HB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[{dev, kern}];
  if (c >= bytes) return;
  HB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  c = bytes;
}

// every kernel launch site of the library passes through here: the counter backs the
// "gpu_launches" figure of bench.py (hb_stats.launches)
inline std::atomic<unsigned long long>& launch_counter() {
  static std::atomic<unsigned long long> n{0};
  return n;
}
#define HB_LAUNCH_CHECK()                                         \
  do {                                                            \
    ::hb::launch_counter().fetch_add(1, std::memory_order_relaxed); \
    HB_CUDA(cudaGetLastError());                                  \
  } while (0)

#define HB_REQUIRE(cond, st, msg) \
  do {                            \
    if (!(cond)) throw ::hb::Error(st, msg); \
  } while (0)

constexpr int kSketchRows = 128;  // ℓ: sketch rows (block size cap + oversampling)
constexpr int kBlockMax = 120;    // largest pivot block b (multiple of 8, ℓ - b >= 8)

__host__ __device__ inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
__host__ __device__ inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------------------------
// Grid-wide barrier for cooperative (co-resident) launches.  State = {count, generation}; the
// count self-resets, the generation grows monotonically, so no reset between launches is needed
// as long as every launch uses the same gridDim for a given state slot.
// ---------------------------------------------------------------------------------------------
struct GridBarrier {
  unsigned int* count;
  unsigned int* gen;
};

__device__ __forceinline__ void grid_sync(GridBarrier b) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = b.gen;
    const unsigned int my_gen = *vgen;
    __threadfence();
    const unsigned int nb = gridDim.x * gridDim.y * gridDim.z;
    const unsigned int arrived = atomicAdd(b.count, 1u);
    if (arrived == nb - 1) {
      *b.count = 0;
      __threadfence();
      atomicAdd(b.gen, 1u);
    } else {
      while (*vgen == my_gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; result valid in all threads. smem must hold >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += smem[w];  // fixed order: deterministic
  return t;
}

// Sum of n values base[h*stride] (h < n) over the whole block, fixed order (deterministic).
__device__ __forceinline__ double block_sum_strided(const double* base, int n, int64_t stride,
                                                    double* smem) {
  double v = 0.0;
  for (int h = threadIdx.x; h < n; h += blockDim.x) v += base[(int64_t)h * stride];
  return block_sum(v, smem);
}

// Warp-wide sum of n values base[h*stride]; result in every lane, fixed order.
__device__ __forceinline__ double warp_sum_strided(const double* base, int n, int64_t stride) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  for (int h = lane; h < n; h += 32) v += base[(int64_t)h * stride];
  return warp_sum(v);
}

}  // namespace hb
