// Day-1 microbenchmark: how fast can 148 SMs pull random 512-B B-rows out of L2 / HBM?
// (a) LDG.128 warp gather into registers, (b) cp.async.bulk (TMA engine, UBLKCP) gather into a
// shared-memory ring with mbarrier completion.  Answers SURVEY.md §7.3(1): the L2->SM gather roof.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void ldg_gather(const float4* __restrict__ B, const int* __restrict__ idx, long n_idx, int row_f4, float* out) {
  int lane = threadIdx.x & 31;
  long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  long nwarps = (gridDim.x * (long)blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  // each warp handles rows i = warp*8 + k*nwarps*8 ... in groups of 8 for MLP
  for (long base = warp * 8; base < n_idx; base += nwarps * 8) {
    int r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = (base + k < n_idx) ? __ldg(idx + base + k) : 0;
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      for (int f = lane; f < row_f4; f += 32) v[k] = __ldg(B + (long)r[k] * row_f4 + f);
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w; }
  }
  if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(bar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" :: "r"(a), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* g, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

// one producer thread per CTA, one consumer warp; STAGES x 8 rows in flight
template <int STAGES>
__global__ void bulk_gather(const char* __restrict__ B, const int* __restrict__ idx, long n_idx, int row_bytes, float* out) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  long groups = (n_idx + 7) / 8;
  float acc = 0;
  if (warp == 0 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (long g = blockIdx.x; g < groups; g += gridDim.x) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], 8 * row_bytes);
      for (int k = 0; k < 8; ++k) {
        long i = g * 8 + k; int r = i < n_idx ? idx[i] : 0;
        bulk_g2s(smem + (s * 8 + k) * row_bytes, B + (long)r * row_bytes, row_bytes, &full[s]);
      }
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    int s = 0; uint32_t ph = 0;
    for (long g = blockIdx.x; g < groups; g += gridDim.x) {
      mbar_wait(&full[s], ph);
      acc += ((float*)(smem + s * 8 * row_bytes))[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void stream_read(const float4* __restrict__ a, long n, float* out) {
  float4 acc = make_float4(0,0,0,0);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    float4 v = __ldg(a + i); acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
  if (acc.x == 12345.f) out[0] = acc.y;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int l2; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  printf("device %s SMs %d L2 %d MB smem/block optin %zu KB clock %d MHz\n", p.name, p.multiProcessorCount, l2 >> 20, p.sharedMemPerBlockOptin >> 10, p.clockRate / 1000);
  const int row_bytes = 512, row_f4 = row_bytes / 16;
  const long big_rows = (4L << 30) / row_bytes;  // 4 GB table
  char* B; CK(cudaMalloc(&B, big_rows * row_bytes)); CK(cudaMemset(B, 0, big_rows * row_bytes));
  const long n_idx = 16L << 20;  // 16M gathers = 8 GB
  int* idx; CK(cudaMalloc(&idx, n_idx * 4));
  float* out; CK(cudaMalloc(&out, 4));
  std::vector<int> h(n_idx);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // stream read baseline
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0); stream_read<<<148 * 8, 256>>>((float4*)B, big_rows * row_f4, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("stream read 4GB: %.3f ms = %.1f GB/s\n", ms, 4.0 * (1 << 30) / ms / 1e6);
  long footprints_mb[] = {16, 48, 96, 128, 256, 1024, 4096};
  std::mt19937_64 rng(1);
  for (long fmb : footprints_mb) {
    long rows = fmb * (1L << 20) / row_bytes;
    for (long i = 0; i < n_idx; ++i) h[i] = (int)(rng() % rows);
    CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
    double gb = n_idx * (double)row_bytes / 1e9;
    for (int occ : {4, 8, 16}) {
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0); ldg_gather<<<148 * occ, 256>>>((float4*)B, idx, n_idx, row_f4, out); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); best = fminf(best, ms);
      }
      printf("footprint %5ld MB ldg  occ %2d: %.3f ms = %.1f GB/s gathered\n", fmb, occ, best, gb / best * 1e3);
    }
    const int ST = 24;
    size_t sm = ST * 8 * row_bytes;
    CK(cudaFuncSetAttribute(bulk_gather<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (int ctas : {1, 2}) {
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0); bulk_gather<ST><<<148 * ctas, 64, sm>>>(B, idx, n_idx, row_bytes, out); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); best = fminf(best, ms);
      }
      printf("footprint %5ld MB bulk ctas/SM %d (%d KB smem): %.3f ms = %.1f GB/s gathered\n", fmb, ctas, (int)(sm >> 10), best, gb / best * 1e3);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
