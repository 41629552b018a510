// Does a 1-D TMA bulk copy (cp.async.bulk, one 512-B B row per instruction, completion on an
// mbarrier) add gather bandwidth on top of L1-allocating LDG.128?  The LDG path looks capped by
// the bytes an SM can keep in flight through L1 (~64 KB); bulk copies land in shared memory
// without L1 miss tracking.  Random 512-B rows, L2-resident (64 MB) and HBM (2 GB) footprints.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_gather bulk_gather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void mbar_init(uint64_t* m, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}"
               ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, int bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                 "r"((uint32_t)__cvta_generic_to_shared(m)) : "memory");
}

// warps [0, n_bulk) stream rows with bulk copies through an S-stage smem ring; the others gather
// with LDG.128, R rows in flight.  Each warp takes every nwarps-th index.
template <int S, int R>
__global__ void __launch_bounds__(256) mixed(const char* __restrict__ B, const int* __restrict__ idx, long n_idx,
                                             int n_bulk, float* out) {
  extern __shared__ __align__(128) char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  if (wib < n_bulk) {
    char* ring = smem + wib * (S * 512 + S * 8);
    uint64_t* bar = reinterpret_cast<uint64_t*>(ring + S * 512);
    if (lane == 0)
      for (int s = 0; s < S; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    long i = gw;
    int issued = 0;
    // prologue
    for (int s = 0; s < S && i + (long)s * nw < n_idx; ++s) {
      if (lane == 0) {
        mbar_expect(bar + s, 512);
        bulk_copy(ring + s * 512, B + (long)__ldg(idx + i + (long)s * nw) * 512, 512, bar + s);
      }
      ++issued;
    }
    long next = i + (long)S * nw;
    for (int k = 0; k < issued || next < n_idx; ++k) {
      const int s = k % S;
      if (k >= issued) break;
      mbar_wait(bar + s, (uint32_t)((k / S) & 1));
      acc += reinterpret_cast<const float4*>(ring + s * 512)[lane].x;
      __syncwarp();
      if (next < n_idx) {
        if (lane == 0) {
          mbar_expect(bar + s, 512);
          bulk_copy(ring + s * 512, B + (long)__ldg(idx + next) * 512, 512, bar + s);
        }
        ++issued;
        next += nw;
      }
    }
  } else {
    // same index partition as the bulk warps: warp gw takes gw, gw + nw, gw + 2 nw, ...
    for (long base = gw; base < n_idx; base += nw * R) {
      int r[R];
#pragma unroll
      for (int k = 0; k < R; ++k) r[k] = (base + k * nw < n_idx) ? __ldg(idx + base + k * nw) : 0;
      float4 v[R];
#pragma unroll
      for (int k = 0; k < R; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(B + (long)r[k] * 512) + lane);
#pragma unroll
      for (int k = 0; k < R; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const long big_rows = (2L << 30) / 512;
  char* B; CK(cudaMalloc(&B, big_rows * 512)); CK(cudaMemset(B, 0, big_rows * 512));
  const long n_idx = 16L << 20;
  int* idx; CK(cudaMalloc(&idx, n_idx * 4));
  float* out; CK(cudaMalloc(&out, 4));
  std::vector<int> h(n_idx);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::mt19937_64 rng(1);
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (long foot : {64L << 20, 2L << 30}) {
    const long rows = foot / 512;
    for (long i = 0; i < n_idx; ++i) h[i] = (int)(rng() % rows);
    CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
    printf("footprint %ld MB\n", foot >> 20);
    auto run = [&](auto kern, int ctas, int n_bulk, int S, const char* name) {
      const int smem = n_bulk * (S * 512 + S * 8);
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem > 0 ? smem : 0));
      float best = 1e9, ms;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        kern<<<sms * ctas, 256, smem>>>(B, idx, n_idx, n_bulk, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        cudaEventElapsedTime(&ms, e0, e1);
        best = fminf(best, ms);
      }
      printf("  %-44s ctas/SM %d bulk warps/CTA %d: %7.0f GB/s\n", name, ctas, n_bulk, n_idx * 512.0 / best / 1e6);
    };
    run(mixed<16, 8>, 4, 0, 16, "LDG only, 8 rows/warp");
    run(mixed<16, 16>, 4, 0, 16, "LDG only, 16 rows/warp");
    run(mixed<8, 8>, 2, 8, 8, "bulk only, 8 stages/warp");
    run(mixed<16, 8>, 1, 8, 16, "bulk only, 16 stages/warp");
    run(mixed<16, 8>, 2, 4, 16, "bulk only, 16 stages/warp, 4 warps");
    run(mixed<8, 8>, 3, 8, 8, "bulk only, 8 stages/warp");
    run(mixed<8, 8>, 4, 4, 8, "mixed: 4 bulk (8 stages) + 4 LDG (8 rows)");
    run(mixed<8, 16>, 4, 4, 8, "mixed: 4 bulk (8 stages) + 4 LDG (16 rows)");
    run(mixed<16, 8>, 3, 4, 16, "mixed: 4 bulk (16 stages) + 4 LDG (8 rows)");
    run(mixed<8, 8>, 4, 2, 8, "mixed: 2 bulk (8 stages) + 6 LDG (8 rows)");
  }
  return 0;
}
