// Do the LSU (LDG.128) and the TMA (tile::gather4) gather paths add up?  One kernel, two warp roles
// per CTA gathering random 512-B B rows side by side: W_L warps with LDG (R rows in flight per warp)
// and W_T warps with TMA gather4 of full rows into a shared-memory ring (D batches of 32 rows per
// warp, 8 issuing lanes).  Each role consumes what it fetched.  Compared with each role alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dual_gather_bin dual_gather.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int RB = 512;  // row bytes

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g4(const CUtensorMap* map, uint32_t dst, uint32_t bar, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
      ::"r"(dst), "l"((uint64_t)map), "r"(bar), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}

template <int R>
__device__ void ldg_role(const char* __restrict__ B, const int* __restrict__ idx, long n, long w, long nw, float* out) {
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (long base = w * R; base < n; base += nw * R) {
    int r[R];
#pragma unroll
    for (int k = 0; k < R; ++k) r[k] = base + k < n ? __ldg(idx + base + k) : 0;
    uint4 v[R];
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = __ldg(reinterpret_cast<const uint4*>(B + (long)r[k] * RB) + lane);
#pragma unroll
    for (int k = 0; k < R; ++k) acc += __int_as_float(v[k].x) + __int_as_float(v[k].w);
  }
  if (acc == 12345.f) out[0] = acc;
}

__device__ void tma_role(const CUtensorMap* map, const int* __restrict__ idx, long n, long w, long nw, int D, uint8_t* ring,
                         uint64_t* bars, float* out) {
  const int lane = threadIdx.x & 31;
  constexpr int BATCH = 32 * RB;
  const long nb = (n + 31) / 32;
  float acc = 0.f;
  auto issue = [&](long b, int d, int myrow) {
    if (lane == 0) mbar_expect(bars + d, BATCH);
    __syncwarp();
    const int r0 = __shfl_sync(0xffffffffu, myrow, (lane & 7) * 4 + 0);
    const int r1 = __shfl_sync(0xffffffffu, myrow, (lane & 7) * 4 + 1);
    const int r2 = __shfl_sync(0xffffffffu, myrow, (lane & 7) * 4 + 2);
    const int r3 = __shfl_sync(0xffffffffu, myrow, (lane & 7) * 4 + 3);
    if (lane < 8) g4(map, su32(ring + (size_t)d * BATCH + lane * 4 * RB), su32(bars + d), r0, r1, r2, r3);
  };
  for (int d = 0; d < D; ++d) {
    const long b = w + (long)d * nw;
    const long i = b * 32 + lane;
    if (b < nb) issue(b, d, i < n ? __ldg(idx + i) : 0);
  }
  uint32_t phase = 0;
  for (long k = 0; w + k * nw < nb; ++k) {
    const int d = (int)(k % D);
    if (k > 0 && d == 0) phase ^= 1;
    const long bnext = w + (k + D) * nw;
    const long inext = bnext * 32 + lane;
    const int rnext = (bnext < nb && inext < n) ? __ldg(idx + inext) : 0;
    mbar_wait(bars + d, phase);
    const uint8_t* s = ring + (size_t)d * BATCH;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(s + q * RB + lane * 16);
      acc += __int_as_float(v.x) + __int_as_float(v.w);
    }
    __syncwarp();
    if (bnext < nb) issue(bnext, d, rnext);
  }
  if (acc == 12345.f) out[0] = acc;
}

// warps [0, WL) LDG, [WL, WL + WT) TMA; nL / nT rows for each role (separate index arrays)
template <int R>
__global__ void k_dual(const char* B, const __grid_constant__ CUtensorMap map, const int* idxL, long nL,
                       const int* idxT, long nT, int WL, int WT, int D, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WT * D * 32 * RB);
  if (warp >= WL && lane == 0)
    for (int d = 0; d < D; ++d) mbar_init(bars + (warp - WL) * 8 + d, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (warp < WL) {
    ldg_role<R>(B, idxL, nL, blockIdx.x * (long)WL + warp, (long)gridDim.x * WL, out);
  } else {
    const int tw = warp - WL;
    tma_role(&map, idxT, nT, blockIdx.x * (long)WT + tw, (long)gridDim.x * WT, D, smem + (size_t)tw * D * 32 * RB,
             bars + tw * 8, out);
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long big = 2L << 30;
  char* B;
  CK(cudaMalloc(&B, big));
  CK(cudaMemset(B, 0, big));
  const long n = 16L << 20;
  int *idxL, *idxT;
  CK(cudaMalloc(&idxL, n * 4));
  CK(cudaMalloc(&idxT, n * 4));
  float* out;
  CK(cudaMalloc(&out, 4));
  std::vector<int> h(n);
  std::mt19937_64 rng(7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (long foot : {64L << 20, 256L << 20, 2L << 30}) {
    const long rows = foot / RB;
    for (long i = 0; i < n; ++i) h[i] = (int)(rng() % rows);
    CK(cudaMemcpy(idxL, h.data(), n * 4, cudaMemcpyHostToDevice));
    for (long i = 0; i < n; ++i) h[i] = (int)(rng() % rows);
    CK(cudaMemcpy(idxT, h.data(), n * 4, cudaMemcpyHostToDevice));
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)(RB / 4), (cuuint64_t)(big / RB)};
    cuuint64_t strides[1] = {(cuuint64_t)RB};
    cuuint32_t box[2] = {(cuuint32_t)(RB / 4), 1}, estr[2] = {1, 1};
    if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    printf("footprint %ld MB\n", foot >> 20);
    auto run = [&](int WL, int WT, int D, int ctas, long nl, long nt, const char* name) {
      const size_t smem = (size_t)WT * D * 32 * RB + 8 * 8 * 8 + 2048;
      if (smem > 227 * 1024) return;
      auto kern = k_dual<8>;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, (WL + WT) * 32, smem));
      if (occ < ctas) { printf("  %-28s: occupancy %d < %d\n", name, occ, ctas); return; }
      float best = 1e9, ms;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        kern<<<sms * ctas, (WL + WT) * 32, smem>>>(B, map, idxL, nl, idxT, nt, WL, WT, D, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        cudaEventElapsedTime(&ms, e0, e1);
        if (it) best = fminf(best, ms);
      }
      printf("  %-28s ctas/SM %d LDG warps %2d TMA warps %2d D %d: %8.0f GB/s\n", name, ctas, WL, WT, D,
             (double)(nl + nt) * RB / best / 1e6);
    };
    run(8, 0, 1, 4, n, 0, "LDG only (R8)");
    run(8, 0, 1, 2, n, 0, "LDG only (R8)");
    run(0, 4, 3, 1, 0, n, "TMA only");
    run(0, 6, 2, 1, 0, n, "TMA only");
    // both: split the rows in proportion to each role's solo rate (about 6:4)
    run(8, 4, 3, 1, n * 6 / 10, n * 4 / 10, "LDG + TMA");
    run(16, 4, 3, 1, n * 6 / 10, n * 4 / 10, "LDG + TMA");
    run(16, 6, 2, 1, n * 6 / 10, n * 4 / 10, "LDG + TMA");
    run(24, 4, 2, 1, n * 7 / 10, n * 3 / 10, "LDG + TMA");
    run(16, 2, 3, 2, n * 6 / 10, n * 4 / 10, "LDG + TMA");
    fflush(stdout);
  }
  return 0;
}
