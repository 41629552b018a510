// Gather-bandwidth plateau curves on B200: random B rows (512 B or 256 B) gathered by all 148
// SMs through four paths, sweeping the bytes each SM keeps in flight until throughput plateaus.
//
//   ldg    LDG.128 into registers (L1-allocating or L1::no_allocate), R rows in flight per warp
//   cpa    cp.async 16 B per lane into a shared-memory ring (LDGSTS), D batches of 32 rows/warp
//   bulk   cp.async.bulk (UBLKCP) one row per lane -> 32 copies issued by one warp instruction,
//          one mbarrier per 32-row batch, D batches in flight per warp
//   g4     cp.async.bulk.tensor.2d.tile::gather4 (UTMALDG): 4 rows per instruction, issued by 8
//          lanes per warp; box 128 B wide with SWIZZLE_128B_ATOM_32B (the tf32 MMA operand
//          layout) or the full row with SWIZZLE_NONE
//
// Every row is consumed (the warp reads it from registers / shared memory and sums it) so the
// numbers include the consumer's shared-memory reads.  Indices are prefetched one batch ahead
// (no dependent index load on the issue path -- the flaw of round 1's bulk_gather.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_plateau gather_plateau.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src),
               "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void g4(const CUtensorMap* map, uint32_t dst, uint32_t bar, int x, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
      ::"r"(dst), "l"((uint64_t)map), "r"(bar), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}

// ---- LDG: R rows in flight per warp (each lane 16 B of each row; RB = row bytes) ------------------
template <int R, int RB, bool kNoL1>
__global__ void __launch_bounds__(256) k_ldg(const char* __restrict__ B, const int* __restrict__ idx, long n, float* out) {
  constexpr int LPR = RB / 16;  // lanes per row
  constexpr int RPI = 32 / LPR; // rows per warp instruction
  const int lane = threadIdx.x & 31;
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
  float acc = 0.f;
  const long per = (long)R * RPI;
  for (long base = gw * per; base < n; base += nw * per) {
    int r[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const long i = base + (long)k * RPI + lane / LPR;
      r[k] = i < n ? __ldg(idx + i) : 0;
    }
    uint4 v[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const char* p = B + (long)r[k] * RB + (lane % LPR) * 16;
      if (kNoL1)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(p));
      else
        v[k] = __ldg(reinterpret_cast<const uint4*>(p));
    }
#pragma unroll
    for (int k = 0; k < R; ++k) acc += __int_as_float(v[k].x) + __int_as_float(v[k].y) + __int_as_float(v[k].z) + __int_as_float(v[k].w);
  }
  if (acc == 12345.f) out[0] = acc;
}

// ---- shared-memory rings: D batches of 32 rows per warp ---------------------------------------
// MODE 0: cp.async 16 B per lane per row (LDGSTS); MODE 1: cp.async.bulk one row per lane;
// MODE 2: gather4 with 128-B boxes (SWIZZLE_128B_ATOM_32B); MODE 3: gather4 with full-row boxes.
template <int MODE, int RB>
__global__ void __launch_bounds__(512) k_ring(const char* __restrict__ B, const __grid_constant__ CUtensorMap map,
                                              const int* __restrict__ idx, long n, int D, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  constexpr int BATCH = 32 * RB;
  uint8_t* ring = smem + (size_t)w * D * BATCH;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nwb * D * BATCH) + w * 16;
  if (lane == 0)
    for (int d = 0; d < D; ++d) mbar_init(bars + d, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
  const long nb = (n + 31) / 32;  // batches
  float acc = 0.f;
  auto issue = [&](long bt, int d, int myrow) {
    const uint32_t dst = su32(ring + (size_t)d * BATCH);
    const uint32_t bar = su32(bars + d);
    if constexpr (MODE == 0) {
      // lane = (row within an instruction, 16-B chunk): every row of the batch, row-major slots
      constexpr int LPR = RB / 16, RPI = 32 / LPR;
#pragma unroll 4
      for (int k = 0; k < 32 / RPI; ++k) {
        const int rr = k * RPI + lane / LPR;
        const int rk = __shfl_sync(0xffffffffu, myrow, rr);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + rr * RB + (lane % LPR) * 16),
                     "l"(B + (long)rk * RB + (lane % LPR) * 16) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    } else if constexpr (MODE == 1) {
      if (lane == 0) mbar_expect(bars + d, BATCH);
      __syncwarp();
      bulk(dst + lane * RB, B + (long)myrow * RB, RB, bar);
    } else {
      if (lane == 0) mbar_expect(bars + d, BATCH);
      __syncwarp();
      const int r0 = __shfl_sync(0xffffffffu, myrow, (lane & 7) * 4 + 0);
      const int r1 = __shfl_sync(0xffffffffu, myrow, (lane & 7) * 4 + 1);
      const int r2 = __shfl_sync(0xffffffffu, myrow, (lane & 7) * 4 + 2);
      const int r3 = __shfl_sync(0xffffffffu, myrow, (lane & 7) * 4 + 3);
      if (lane < 8) {
        if constexpr (MODE == 2) {
          // quad q = lane: atoms of 4 rows x 128 B, one per 128-B column chunk
#pragma unroll
          for (int c = 0; c < RB / 128; ++c)
            g4(&map, dst + (lane * (RB / 128) + c) * 512, bar, c * 32, r0, r1, r2, r3);
        } else {
          g4(&map, dst + lane * 4 * RB, bar, 0, r0, r1, r2, r3);
        }
      }
    }
  };
  long bt = gw;
  int rows[8];  // prefetched row index of this lane for batches in flight (D <= 8)
  int issued = 0;
  for (int d = 0; d < D; ++d) {
    const long b = bt + (long)d * nw;
    const long i = b * 32 + lane;
    rows[d] = (b < nb && i < n) ? __ldg(idx + i) : 0;
  }
  for (int d = 0; d < D; ++d)
    if (bt + (long)d * nw < nb) { issue(bt + (long)d * nw, d, rows[d]); ++issued; }
  uint32_t phase = 0;
  for (long k = 0; bt + k * nw < nb; ++k) {
    const int d = (int)(k % D);
    if (k > 0 && d == 0) phase ^= 1;
    // prefetch the index this slot will need next
    const long bnext = bt + (k + D) * nw;
    const long inext = bnext * 32 + lane;
    const int rnext = (bnext < nb && inext < n) ? __ldg(idx + inext) : 0;
    if constexpr (MODE == 0) {
      // groups complete in order: the oldest is this one
      switch (D) {  // the oldest group is this slot's
        case 1: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
      }
      __syncwarp();
    } else {
      mbar_wait(bars + d, phase);
    }
    const uint8_t* s = ring + (size_t)d * BATCH;
#pragma unroll 8
    for (int q = 0; q < 32 * RB / 512; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(s + q * 512 + lane * 16);
      acc += __int_as_float(v.x) + __int_as_float(v.w);
    }
    __syncwarp();
    if (bnext < nb) issue(bnext, d, rnext);
    else if (MODE == 0) asm volatile("cp.async.commit_group;" ::: "memory");  // keep one group per slot
  }
  if (acc == 12345.f) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long big = 2L << 30;
  char* B;
  CK(cudaMalloc(&B, big));
  CK(cudaMemset(B, 0, big));
  const long n = 16L << 20;  // rows gathered per launch
  int* idx;
  CK(cudaMalloc(&idx, n * 4));
  float* out;
  CK(cudaMalloc(&out, 4));
  std::vector<int> h(n);
  std::mt19937_64 rng(7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int RB : {512, 256}) {
    for (long foot : {64L << 20, 2L << 30}) {
      const long rows = foot / RB;
      for (long i = 0; i < n; ++i) h[i] = (int)(rng() % rows);
      CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
      CUtensorMap m_sw, m_none;
      {
        cuuint64_t dims[2] = {(cuuint64_t)(RB / 4), (cuuint64_t)(big / RB)};
        cuuint64_t strides[1] = {(cuuint64_t)RB};
        cuuint32_t box[2] = {32, 1}, estr[2] = {1, 1};
        if (encode(&m_sw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          printf("encode sw failed\n");
          return 1;
        }
        cuuint32_t box2[2] = {(cuuint32_t)(RB / 4), 1};
        if (encode(&m_none, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, strides, box2, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          printf("encode none failed\n");
          return 1;
        }
      }
      printf("row %d B, footprint %ld MB\n", RB, foot >> 20);
      auto timeit = [&](auto launch) {
        float best = 1e9, ms;
        for (int it = 0; it < 4; ++it) {
          cudaEventRecord(e0);
          launch();
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          CK(cudaGetLastError());
          cudaEventElapsedTime(&ms, e0, e1);
          if (it) best = fminf(best, ms);
        }
        return n * (double)RB / best / 1e6;  // GB/s
      };
      // LDG sweep
      auto ldg = [&](auto kern, int ctas, const char* name) {
        double g = timeit([&] { kern<<<sms * ctas, 256>>>(B, idx, n, out); });
        printf("  ldg %-18s ctas/SM %d: %8.0f GB/s\n", name, ctas, g);
      };
      if (RB == 512) {
        for (int c : {2, 4, 8}) {
          ldg(k_ldg<4, 512, false>, c, "R4");
          ldg(k_ldg<8, 512, false>, c, "R8");
          ldg(k_ldg<16, 512, false>, c, "R16");
          ldg(k_ldg<8, 512, true>, c, "R8 no_allocate");
          ldg(k_ldg<16, 512, true>, c, "R16 no_allocate");
        }
      } else {
        for (int c : {2, 4, 8}) {
          ldg(k_ldg<4, 256, false>, c, "R4");
          ldg(k_ldg<8, 256, false>, c, "R8");
          ldg(k_ldg<16, 256, false>, c, "R16");
          ldg(k_ldg<16, 256, true>, c, "R16 no_allocate");
        }
      }
      // ring sweeps: bytes in flight per SM = ctas * warps * D * 32 * RB
      auto ring = [&](auto kern, const CUtensorMap& m, int mode, int ctas, int warps, int D) {
        const size_t smem = (size_t)warps * D * 32 * RB + warps * 16 * 8 + 1024;
        if (smem > 227 * 1024) return;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem));
        if (occ < ctas) return;
        double g = timeit([&] { kern<<<sms * ctas, warps * 32, smem>>>(B, m, idx, n, D, out); });
        static const char* names[] = {"cp.async 16B", "bulk row/lane", "gather4 128B sw32", "gather4 row none"};
        printf("  %-18s ctas/SM %d warps %2d D %d: in flight %4ld KB/SM  %8.0f GB/s\n", names[mode], ctas, warps, D,
               (long)ctas * warps * D * 32 * RB / 1024, g);
      };
      const int cfg[][3] = {{1, 4, 1}, {1, 8, 1}, {1, 8, 2}, {1, 12, 1}, {1, 16, 1}, {2, 8, 1}, {2, 6, 1},
                            {3, 4, 1}, {1, 4, 4}, {1, 8, 3}, {1, 12, 2}, {2, 4, 2}, {4, 4, 1}, {1, 16, 2}};
      for (auto& c : cfg) {
        if (RB == 512) {
          ring(k_ring<0, 512>, m_none, 0, c[0], c[1], c[2]);
          ring(k_ring<1, 512>, m_none, 1, c[0], c[1], c[2]);
          ring(k_ring<2, 512>, m_sw, 2, c[0], c[1], c[2]);
          ring(k_ring<3, 512>, m_none, 3, c[0], c[1], c[2]);
        } else {
          ring(k_ring<0, 256>, m_none, 0, c[0], c[1], c[2]);
          ring(k_ring<1, 256>, m_none, 1, c[0], c[1], c[2]);
          ring(k_ring<2, 256>, m_sw, 2, c[0], c[1], c[2]);
          ring(k_ring<3, 256>, m_none, 3, c[0], c[1], c[2]);
        }
      }
      fflush(stdout);
    }
  }
  return 0;
}
