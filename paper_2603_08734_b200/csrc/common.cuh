// Shared helpers for the RSH-SpMM sm_100a library (librsh.so).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>
#include "rsh.h"

namespace rsh {

enum Status : int { kOk = 0, kInvalid = 1, kFormat = 2, kCuda = 3 };

// thread-local message behind rsh_last_error()
int fail(int status, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* where);

#define RSH_CUDA(x)                                              \
  do {                                                           \
    cudaError_t _e = (x);                                        \
    if (_e != cudaSuccess) return ::rsh::cuda_fail(_e, #x);      \
  } while (0)
// every kernel launch is followed by RSH_LAUNCHED, which also bumps the process-wide launch
// counter behind rsh_launch_count() (diagnostic: the bench reports launches per timed region)
void count_launch();
#define RSH_LAUNCHED(name)                                       \
  do {                                                           \
    ::rsh::count_launch();                                       \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::rsh::cuda_fail(_e, name);    \
  } while (0)
#define RSH_OK(x)                                                \
  do {                                                           \
    int _s = (x);                                                \
    if (_s != ::rsh::kOk) return _s;                             \
  } while (0)

constexpr int kThreads = 256;

inline unsigned grid_1d(int64_t work, int threads = kThreads) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 0x7fffffffLL) g = 0x7fffffffLL;
  return (unsigned)g;
}

// Bump allocator over a caller-owned device workspace.  Layouts are computed twice: once with
// base == nullptr to size the workspace, once with the real pointer.
struct Carve {
  char* base;
  size_t used = 0;
  explicit Carve(void* b) : base((char*)b) {}
  template <class T>
  T* take(size_t n) {
    used = (used + 255) & ~size_t(255);
    T* p = base ? (T*)(base + used) : nullptr;
    used += n * sizeof(T);
    return p;
  }
};

int sm_count();

// -------------------------------------------------------------------------------------------
// device helpers
// -------------------------------------------------------------------------------------------

// largest r in [0, n_rows) with rp[r] <= p  (the CSR row owning position p)
__device__ __forceinline__ int64_t row_of(const int64_t* __restrict__ rp, int64_t n_rows, int64_t p) {
  int64_t lo = 0, hi = n_rows - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(rp + mid) <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// first i in sorted a[0, n) with a[i] >= x
__device__ __forceinline__ int64_t lower_bound(const int32_t* __restrict__ a, int64_t n, int32_t x) {
  int64_t lo = 0;
  while (n > 0) {
    int64_t half = n >> 1;
    if (__ldg(a + lo + half) < x) { lo += half + 1; n -= half + 1; } else { n = half; }
  }
  return lo;
}

__device__ __forceinline__ bool row_has(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                        int64_t r, int32_t c) {
  int64_t s = __ldg(rp + r), e = __ldg(rp + r + 1);
  int64_t k = lower_bound(ci + s, e - s, c);
  return k < e - s && __ldg(ci + s + k) == c;
}

}  // namespace rsh
