// TMA gather4 roof: random 512-B B rows (128 fp32) gathered into shared memory by
// cp.async.bulk.tensor.2d.tile::gather4 (4 rows x 128 B per instruction), one issuing lane per
// CTA, an mbarrier ring of S stages of 8 rows (4 KB, the RSH window block), a consumer warp that
// releases stages.  Compared against the LDG gather roof of gather_bw2.cu.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" :: "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gather4(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int r0, int r1, int r2, int r3,
                                        uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;"
      :: "r"(smem_u32(dst)), "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "l"(policy)
      : "memory");
}

template <int S>
__global__ void __launch_bounds__(64) tma_gather(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx,
                                                 long n_blocks, float* out, int evict_last) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S], empty[S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint64_t policy;
  if (evict_last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
  float acc = 0.f;
  if (warp == 0) {
    long j = 0;
    for (long base = blockIdx.x * 4L; base < n_blocks; base += gridDim.x * 4L) {
      // 4 blocks x 8 rows: lane l holds row index l of the batch
      const long i = base * 8 + lane;
      const int r = i < n_blocks * 8 ? __ldg(idx + i) : 0;
      for (int b = 0; b < 4 && base + b < n_blocks; ++b, ++j) {
        const int s = (int)(j % S);
        const uint32_t ph = (uint32_t)((j / S) & 1);
        int rr[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) rr[k] = __shfl_sync(0xffffffffu, r, b * 8 + k);
        if (lane == 0) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect(&full[s], 4096);
          uint8_t* dst = ring + s * 4096;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            gather4(&map, &full[s], dst + 0 * 2048 + a * 512, a * 32, rr[0], rr[1], rr[2], rr[3], policy);
            gather4(&map, &full[s], dst + 1 * 2048 + a * 512, a * 32, rr[4], rr[5], rr[6], rr[7], policy);
          }
        }
        __syncwarp();
      }
    }
  } else {
    long j = 0;
    for (long base = blockIdx.x * 4L; base < n_blocks; base += gridDim.x * 4L)
      for (int b = 0; b < 4 && base + b < n_blocks; ++b, ++j) {
        const int s = (int)(j % S);
        mbar_wait(&full[s], (uint32_t)((j / S) & 1));
        acc += ((float*)(ring + s * 4096))[lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
  }
  if (acc == 12345.f) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  const long big_rows = (2L << 30) / 512;
  float* B; CK(cudaMalloc(&B, big_rows * 512)); CK(cudaMemset(B, 0, big_rows * 512));
  const long n_blocks = 2L << 20;  // 16M rows gathered
  int* idx; CK(cudaMalloc(&idx, n_blocks * 8 * 4));
  float* out; CK(cudaMalloc(&out, 4));
  std::vector<int> h(n_blocks * 8);
  std::mt19937_64 rng(1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (long fmb : {64L, 2048L}) {
    long rows = fmb * (1L << 20) / 512;
    for (auto& x : h) x = (int)(rng() % rows);
    CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CUtensorMap map;
    cuuint64_t dims[2] = {128, (cuuint64_t)big_rows};
    cuuint64_t strides[1] = {512};
    cuuint32_t box[2] = {32, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
    double gb = n_blocks * 4096.0 / 1e9;
    printf("footprint %ld MB\n", fmb);
    for (int ev : {0, 1})
      for (int ctas : {1, 2, 4}) {
        constexpr int S = 24;
        size_t sm = S * 4096 + 1024;
        CK(cudaFuncSetAttribute(tma_gather<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        float best = 1e9, ms;
        for (int it = 0; it < 4; ++it) {
          cudaEventRecord(e0);
          tma_gather<S><<<148 * ctas, 64, sm>>>(map, idx, n_blocks, out, ev);
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          cudaEventElapsedTime(&ms, e0, e1);
          best = fminf(best, ms);
        }
        printf("  gather4, %d CTA/SM x %d stages, evict_%s: %.0f GB/s\n", ctas, S, ev ? "last" : "normal", gb / best * 1e3);
      }
  }
  CK(cudaGetLastError());
  return 0;
}
