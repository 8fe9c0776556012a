// common.cuh — shared internals of libspmv.so (product side only).
// Error model: internal C++ code throws SpmvError; every extern "C" entry
// point in api.cu catches it and returns the status code (include/spmv.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/spmv.h"

namespace spmv {

struct SpmvError {
  spmv_status_t status;
  std::string msg;
};

// NVTX range for the duration of a scope (host-side phases: create, features,
// convert, tune, the plan's exchange) so an nsys timeline shows the pipeline
// and the overlap of the interior SpMV with the exchange. Header-only NVTX3:
// a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

[[noreturn]] inline void fail(spmv_status_t s, const std::string& m) { throw SpmvError{s, m}; }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      fail(SPMV_ERR_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e));
    }
    fail(SPMV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define CK(call) ::spmv::cuda_check((call), #call)

// Every kernel launch of the library goes through LAUNCH so the process-wide
// launch counter (spmv_launch_count) is exact.
extern std::atomic<uint64_t> g_launches;
#define LAUNCH(kern, grid, block, smem, stream, ...)                                  \
  do {                                                                                \
    kern<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                         \
    ::spmv::g_launches.fetch_add(1, std::memory_order_relaxed);                       \
    ::spmv::cuda_check(cudaGetLastError(), #kern);                                    \
  } while (0)

// Launch through the runtime API; a failed launch is cleared from the
// runtime's last-error slot so it cannot poison the next LAUNCH check.
inline void launch_checked(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaLaunchKernel(fn, grid, block, args, smem, s);
  if (e != cudaSuccess) cudaGetLastError();
  cuda_check(e, "cudaLaunchKernel");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Stream-ordered device allocation from the device's default pool (release
// threshold raised once per device so repeated create/destroy reuses memory).
void* dalloc(size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);

template <class T>
T* dalloc_n(int64_t n, cudaStream_t s) {
  return static_cast<T*>(dalloc((size_t)(n > 0 ? n : 1) * sizeof(T), s));
}

// Stream-ordered scratch buffers released when the scope ends (also on throw).
struct Scratch {
  cudaStream_t s;
  void* p[16] = {};
  int n = 0;
  explicit Scratch(cudaStream_t st) : s(st) {}
  template <class T>
  T* get(int64_t count) {
    T* q = dalloc_n<T>(count, s);
    p[n++] = q;
    return q;
  }
  void keep(void* q) {  // ownership moved elsewhere
    for (int i = 0; i < n; ++i)
      if (p[i] == q) p[i] = nullptr;
  }
  ~Scratch() {
    for (int i = 0; i < n; ++i)
      if (p[i]) dfree(p[i], s);
  }
};

inline unsigned grid_for(int64_t n, int block, int64_t cap = 148LL * 32) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------- device helpers

// L2 cache policies (createpolicy; both fold into the load's uniform
// descriptor, so they cost no instruction in the loop).
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Streaming loads of the matrix arrays: read once per SpMV, so do not allocate
// in L1 and mark evict-first in L2 (x stays resident instead).
#define SPMV_LD_STREAM(T, SUF, CONS)                                                                   \
  __device__ __forceinline__ T ld_stream(const T* p) {                                                  \
    T r;                                                                                                \
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint." SUF " %0, [%1], %2;" : "=" CONS(r) : "l"(p),     \
        "l"(l2_evict_first()));                                                                         \
    return r;                                                                                           \
  }
SPMV_LD_STREAM(int, "b32", "r")
SPMV_LD_STREAM(float, "f32", "f")
SPMV_LD_STREAM(double, "f64", "d")
#undef SPMV_LD_STREAM
__device__ __forceinline__ int2 ld_stream(const int2* p) {
  int2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.b32 {%0,%1}, [%2], %3;"
      : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ float2 ld_stream(const float2* p) {
  float2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
      : "=f"(r.x), "=f"(r.y) : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
      : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(l2_evict_first()));
  return r;
}

// 256-bit streaming loads (sm_100: one LDG.256 per lane, the L2 evict-first
// priority as an instruction qualifier — no policy register to move into a
// uniform register per load). p must be 32-byte aligned.
__device__ __forceinline__ void ld_stream256(const int* p, int (&o)[8]) {
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7])
      : "l"(p));
}
__device__ __forceinline__ void ld_stream256(const float* p, float (&o)[8]) {
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]), "=f"(o[6]), "=f"(o[7])
      : "l"(p));
}
__device__ __forceinline__ void ld_stream256(const double* p, double (&o)[4]) {
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
      : "l"(p));
}
// W (a multiple of the 256-bit width) consecutive values of one lane.
template <int W>
__device__ __forceinline__ void ld_stream256_w(const int* p, int (&o)[W]) {
#pragma unroll
  for (int q = 0; q < W; q += 8) ld_stream256(p + q, *reinterpret_cast<int(*)[8]>(&o[q]));
}
template <int W>
__device__ __forceinline__ void ld_stream256_w(const float* p, float (&o)[W]) {
#pragma unroll
  for (int q = 0; q < W; q += 8) ld_stream256(p + q, *reinterpret_cast<float(*)[8]>(&o[q]));
}
template <int W>
__device__ __forceinline__ void ld_stream256_w(const double* p, double (&o)[W]) {
#pragma unroll
  for (int q = 0; q < W; q += 4) ld_stream256(p + q, *reinterpret_cast<double(*)[4]>(&o[q]));
}

// Gathers of x: read-only path, keep in L1, evict-last in L2 (x is reused by
// every row that touches the column; the matrix stream is evicted first).
__device__ __forceinline__ double ld_x(const double* p) {
  double r;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(l2_evict_last()));
  return r;
}
__device__ __forceinline__ float ld_x(const float* p) {
  float r;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(l2_evict_last()));
  return r;
}

template <class T>
__device__ __forceinline__ double widen(T v) {
  return (double)v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace spmv
