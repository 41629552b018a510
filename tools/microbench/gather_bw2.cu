// Gather-bandwidth roof, second pass: is ~6.8 TB/s (L2-resident random 512-B rows) a fabric
// limit or a latency limit of the first probe?  Varies rows in flight per warp, occupancy, L1
// policy, row width, and an asynchronous cp.async.cg variant with a deep per-warp smem ring.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int RIF, bool NOALLOC>
__global__ void __launch_bounds__(256) ldg_gather(const float4* __restrict__ B, const int* __restrict__ idx, long n_idx,
                                                  int row_f4, float* out) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (gridDim.x * (long)blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (long base = warp * RIF; base < n_idx; base += nwarps * RIF) {
    int r[RIF];
#pragma unroll
    for (int k = 0; k < RIF; ++k) r[k] = (base + k < n_idx) ? __ldg(idx + base + k) : 0;
    float4 v[RIF];
#pragma unroll
    for (int k = 0; k < RIF; ++k) {
      const float4* p = B + (long)r[k] * row_f4 + lane;
      if (NOALLOC)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[k].x), "=f"(v[k].y), "=f"(v[k].z), "=f"(v[k].w) : "l"(p));
      else
        v[k] = __ldg(p);
    }
#pragma unroll
    for (int k = 0; k < RIF; ++k) { acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w; }
  }
  if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
}

// each warp streams rows through a private smem ring with cp.async.cg, DEPTH rows in flight
template <int DEPTH>
__global__ void __launch_bounds__(128) cpasync_gather(const char* __restrict__ B, const int* __restrict__ idx, long n_idx,
                                                      int row_bytes, float* out) {
  extern __shared__ __align__(16) char ring[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (gridDim.x * (long)blockDim.x) >> 5;
  char* my = ring + wib * DEPTH * 512;
  float acc = 0;
  long i = warp;
  int issued = 0;
  for (; i < n_idx; i += nwarps) {
    int r = __ldg(idx + i);
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(my + (issued % DEPTH) * 512 + lane * 16);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(B + (long)r * row_bytes + lane * 16) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    ++issued;
    if (issued >= DEPTH) {
      asm volatile("cp.async.wait_group %0;" :: "n"(DEPTH - 1) : "memory");
      acc += ((float*)(my + (issued % DEPTH) * 512))[lane];
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const int row_bytes = 512, row_f4 = row_bytes / 16;
  const long big_rows = (2L << 30) / row_bytes;
  char* B; CK(cudaMalloc(&B, big_rows * row_bytes)); CK(cudaMemset(B, 0, big_rows * row_bytes));
  const long n_idx = 16L << 20;
  int* idx; CK(cudaMalloc(&idx, n_idx * 4));
  float* out; CK(cudaMalloc(&out, 4));
  std::vector<int> h(n_idx);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::mt19937_64 rng(1);
  auto timeit = [&](auto launch) {
    float best = 1e9, ms;
    for (int it = 0; it < 4; ++it) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); best = fminf(best, ms);
    }
    return best;
  };
  for (long fmb : {64L, 2048L}) {
    long rows = fmb * (1L << 20) / row_bytes;
    for (long i = 0; i < n_idx; ++i) h[i] = (int)(rng() % rows);
    CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
    double gb = n_idx * (double)row_bytes / 1e9;
    printf("footprint %ld MB\n", fmb);
    for (int occ : {4, 8}) {
      float t8 = timeit([&] { ldg_gather<8, false><<<148 * occ, 256>>>((float4*)B, idx, n_idx, row_f4, out); });
      float t16 = timeit([&] { ldg_gather<16, false><<<148 * occ, 256>>>((float4*)B, idx, n_idx, row_f4, out); });
      float t16n = timeit([&] { ldg_gather<16, true><<<148 * occ, 256>>>((float4*)B, idx, n_idx, row_f4, out); });
      float t32 = timeit([&] { ldg_gather<32, false><<<148 * occ, 256>>>((float4*)B, idx, n_idx, row_f4, out); });
      printf("  ldg occ %d: 8 rows/warp %.0f GB/s | 16 %.0f | 16 no_allocate %.0f | 32 %.0f\n", occ, gb / t8 * 1e3,
             gb / t16 * 1e3, gb / t16n * 1e3, gb / t32 * 1e3);
    }
    for (int ctas : {4, 8, 12}) {
      const int D = 16;
      size_t sm = 4 * D * 512;
      CK(cudaFuncSetAttribute(cpasync_gather<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      float t = timeit([&] { cpasync_gather<D><<<148 * ctas, 128, sm>>>(B, idx, n_idx, row_bytes, out); });
      printf("  cp.async.cg ring depth %d, %d CTAs x 4 warps / SM: %.0f GB/s\n", D, ctas, gb / t * 1e3);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
