// Shared device/host helpers for the hb200 rank-reveal path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "hb.h"

namespace hb {

// HB_HOSTTRACE=1 (diagnostics): per host thread, time blocked in stream syncs and in launch calls
struct HostTrace {
  double sync_s = 0.0, max_sync_s = 0.0, launch_s = 0.0, max_launch_s = 0.0;
  long n_sync = 0;
  double max_call_s = 0.0, max_gap_s = 0.0, last_end = 0.0;
  const char* max_call_at = "";
  const char* max_gap_at = "";
};
inline HostTrace& host_trace() {
  thread_local HostTrace t;
  return t;
}
inline bool host_trace_enabled() {
  static const bool on = getenv("HB_HOSTTRACE") != nullptr;
  return on;
}
inline double host_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
// every HB_CUDA call: the longest call and the longest host gap before a call (label = call site)
inline void host_trace_call(double t0, const char* at) {
  HostTrace& h = host_trace();
  const double t1 = host_now();
  if (t1 - t0 > h.max_call_s) {
    h.max_call_s = t1 - t0;
    h.max_call_at = at;
  }
  if (h.last_end > 0.0 && t0 - h.last_end > h.max_gap_s) {
    h.max_gap_s = t0 - h.last_end;
    h.max_gap_at = at;
  }
  h.last_end = t1;
}
struct TraceSync {  // scope guard: time inside counts as a host wait for the device
  double t0;
  bool launch;
  explicit TraceSync(bool is_launch = false) : t0(host_trace_enabled() ? host_now() : 0.0), launch(is_launch) {}
  ~TraceSync() {
    if (!host_trace_enabled()) return;
    const double d = host_now() - t0;
    HostTrace& h = host_trace();
    if (launch) {
      h.launch_s += d;
      h.max_launch_s = std::max(h.max_launch_s, d);
    } else {
      h.sync_s += d;
      h.max_sync_s = std::max(h.max_sync_s, d);
      h.n_sync++;
    }
  }
};
// Error carrying an hb_status; converted to a status code at the C ABI (abi.cpp).
struct Error : std::runtime_error {
  hb_status status;
  Error(hb_status s, const std::string& what) : std::runtime_error(what), status(s) {}
};

#define HB_STR2(x) #x
#define HB_STR(x) HB_STR2(x)
#define HB_CUDA(x)                                                                           \
  do {                                                                                       \
    const double ht0_ = ::hb::host_trace_enabled() ? ::hb::host_now() : 0.0;                  \
    cudaError_t e_ = (x);                                                                    \
    if (ht0_ != 0.0) ::hb::host_trace_call(ht0_, __FILE__ ":" HB_STR(__LINE__));             \
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
// HB_SYNC_DEBUG=1: wait for every launch (device-wide, 10 s watchdog) and name the launch site
// that did not finish — hang triage without a debugger.
void debug_sync_after_launch(const char* file, int line);
inline bool sync_debug_enabled() {
  static const bool on = getenv("HB_SYNC_DEBUG") != nullptr;
  return on;
}

#define HB_LAUNCH_CHECK()                                         \
  do {                                                            \
    ::hb::launch_counter().fetch_add(1, std::memory_order_relaxed); \
    HB_CUDA(cudaGetLastError());                                  \
    if (::hb::sync_debug_enabled()) ::hb::debug_sync_after_launch(__FILE__, __LINE__); \
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

// Per-launch barrier handle: thread 0 of every CTA reads the generation once at kernel start (it
// cannot advance before every CTA has arrived at the first barrier), so each barrier costs one
// acq_rel atomic arrival plus acquire polling — no extra generation read per barrier.
// (Same release/acquire pattern as CUTLASS's GenericBarrier.)
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// acq_rel: the LAST arriver never polls `gen`, so its arrival must itself acquire the other
// CTAs' writes (and drop stale L1 lines) — with a release-only arrival it read stale partials
// and left the grid with diverging barrier counts (observed hang).
__device__ __forceinline__ unsigned int atom_add_acq_rel_gpu(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

struct GridSync {
  unsigned int* count;
  unsigned int* gen;
  unsigned int g;  // generation seen by thread 0
  __device__ __forceinline__ explicit GridSync(GridBarrier b) : count(b.count), gen(b.gen), g(0) {
    if (threadIdx.x == 0) g = ld_acquire_gpu(gen);
  }
  __device__ __forceinline__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int nb = gridDim.x * gridDim.y * gridDim.z;
      if (atom_add_acq_rel_gpu(count, 1u) == nb - 1) {
        *count = 0;  // ordered before the generation bump by the release below
        st_release_gpu(gen, g + 1);
      } else {
        unsigned int seen, spins = 0;
        while ((seen = ld_acquire_gpu(gen)) == g) {
          if (++spins == (1u << 26)) {
            printf("[hb barrier] block %d of %d stuck: gen %u count %u\n", blockIdx.x, nb, seen,
                   *(volatile unsigned int*)count);
            __trap();
          }
        }
        if (seen != g + 1)
          printf("[hb barrier] block %d: generation jumped %u -> %u\n", blockIdx.x, g, seen);
      }
      ++g;
    }
    __syncthreads();
  }
};

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
