// C-ABI plumbing for librsh.so: status codes, thread-local error text, device queries.
#include "common.cuh"
#include <cstdarg>
#include <cstdio>
#include <atomic>

namespace rsh {

static thread_local char g_err[512] = "";

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(kCuda, "CUDA error %d (%s) at %s", (int)e, cudaGetErrorString(e), where);
}

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 1;
}

}  // namespace rsh

extern "C" {

const char* rsh_last_error(void) { return rsh::g_err; }

int rsh_abi_version(void) { return 1; }

// kernels this process has launched through the library so far (all threads, all devices)
unsigned long long rsh_launch_count(void) { return rsh::g_launches.load(std::memory_order_relaxed); }

// 0 ok; sets *major/*minor to the compute capability of the current device
int rsh_device_info(int32_t* major, int32_t* minor, int32_t* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return rsh::cuda_fail(e, "cudaGetDevice");
  cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev);
  *sms = rsh::sm_count();
  return rsh::kOk;
}

}  // extern "C"
