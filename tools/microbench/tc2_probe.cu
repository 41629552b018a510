// Tensor-core window path v2 probe: validates, against a CPU reference, the three layout facts the
// TMA-staged window kernel (csrc/spmm_tc.cu) relies on.
//
//   1. TMA tile::gather4 of 4 B rows (128-B box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B for fp32,
//      CU_TENSOR_MAP_SWIZZLE_128B for bf16) lands the rows in exactly the MN-major swizzled
//      operand layout the UMMA smem descriptor describes (tf32: layout 1 "128B_BASE32B", atoms of
//      4 K-rows x 128 B; bf16: layout 2 "128B", atoms of 8 K-rows x 128 B).
//   2. M = 64 (N = 64 features): where the 64 rows of D land among the 128 TMEM lanes.
//   3. bf16 with K = 16: two 8-column blocks of one window in one MMA.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc2_probe_bin tc2_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g4(const CUtensorMap* map, uint32_t dst, uint32_t bar, int x, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
      ::"r"(dst), "l"((uint64_t)map), "r"(bar), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

// KIND 0: tf32, F features (64 or 128), K = 8.  KIND 1: bf16, F = 128 (or 256 cols of 2 B... F
// features), K = 16 (rows 0-7 block 0, rows 8-15 block 1).
template <int KIND, int F>
__global__ void probe(const __grid_constant__ CUtensorMap map, const int* rows, const float* Blk, float* Dout) {
  constexpr int KB = KIND == 0 ? 8 : 16;          // K rows
  constexpr int EB = KIND == 0 ? 4 : 2;
  constexpr int PER_ATOM = 128 / EB;              // features per 128-B box
  constexpr int NMA = F / PER_ATOM;               // MN atoms
  constexpr int KG = KIND == 0 ? 4 : 8;           // K rows per swizzle atom
  constexpr int ATOM = KG * 128;                  // bytes per atom
  constexpr uint32_t LBO = ATOM;                  // MN atom stride
  constexpr uint32_t SBO = ATOM * NMA;            // K group stride
  constexpr int M = F < 128 ? 64 : 128;
  __shared__ __align__(1024) uint8_t sA[KB * F * EB + 1024];
  __shared__ __align__(1024) uint8_t sB[8 * KB * 4];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (int)sizeof(sA) / 4; i += blockDim.x) ((uint32_t*)sA)[i] = 0xFFFFFFFFu;  // poison
  // fragment operand: K-major, no swizzle: core matrix 8 rows x 16 B, K chunks at +128 (LBO), N groups +256 (SBO)
  for (int idx = tid; idx < 8 * KB; idx += blockDim.x) {
    const int i = idx / KB, k = idx % KB;
    const int per16 = 16 / EB, kc = k / per16, kk = k % per16;
    const int off = kc * 128 + i * 16 + kk * EB;
    if (KIND == 0) *(float*)(sB + off) = Blk[i * KB + k];
    else *(__nv_bfloat16*)(sB + off) = __float2bfloat16(Blk[i * KB + k]);
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    mbar_expect(bar, KB * F * EB);
    // quad q of K rows (4 rows) x MN atom ma -> atom base + (q % (KG/4)) * 512
    for (int q = 0; q < KB / 4; ++q)
      for (int ma = 0; ma < NMA; ++ma) {
        const int kg = (q * 4) / KG, qin = (q * 4) % KG;
        const uint32_t dst = su32(sA) + kg * SBO + ma * LBO + qin * 128;
        g4(&map, dst, su32(bar), ma * PER_ATOM, rows[q * 4], rows[q * 4 + 1], rows[q * 4 + 2], rows[q * 4 + 3]);
      }
    mbar_wait(bar, 0);
    const uint32_t fmt = KIND == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 15) | (1u << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t ad = desc(su32(sA), LBO, SBO, KIND == 0 ? 1u : 2u);
    const uint64_t bd = desc(su32(sB), 128, 256, 0);
    if (KIND == 0)
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
    else
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar + 1)) : "memory");
  }
  __syncwarp();
  mbar_wait(bar + 1, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    uint32_t r[8];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) Dout[(warp * 32 + lane) * 8 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn encode;

static float tf32_trunc(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x; }
static float bf16_rn(float x) { return __bfloat162float(__float2bfloat16(x)); }

template <int KIND, int F>
void run(const char* name) {
  constexpr int KB = KIND == 0 ? 8 : 16;
  constexpr int EB = KIND == 0 ? 4 : 2;
  const int nrows = 5000, ld = F;  // B: nrows x F
  std::mt19937 rng(11);
  std::uniform_real_distribution<float> U(-1, 1);
  std::vector<float> Bh((size_t)nrows * ld);
  for (auto& x : Bh) x = U(rng);
  std::vector<int> rows(KB);
  for (auto& r : rows) r = (int)(rng() % nrows);
  std::vector<float> Blk(8 * KB);
  for (auto& x : Blk) x = (rng() % 3 == 0) ? U(rng) : 0.f;
  void* dB;
  size_t bytes = (size_t)nrows * ld * EB;
  CK(cudaMalloc(&dB, bytes));
  if (KIND == 0) {
    CK(cudaMemcpy(dB, Bh.data(), bytes, cudaMemcpyHostToDevice));
  } else {
    std::vector<__nv_bfloat16> hb(Bh.size());
    for (size_t i = 0; i < Bh.size(); ++i) hb[i] = __float2bfloat16(Bh[i]);
    CK(cudaMemcpy(dB, hb.data(), bytes, cudaMemcpyHostToDevice));
  }
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)F, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * EB};
  cuuint32_t box[2] = {(cuuint32_t)(128 / EB), 1}, estr[2] = {1, 1};
  CUresult cr = encode(&map, KIND == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, dims, strides,
                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       KIND == 0 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { printf("%s: encode failed %d\n", name, (int)cr); return; }
  int* drows; float *dBlk, *dD;
  CK(cudaMalloc(&drows, KB * 4)); CK(cudaMalloc(&dBlk, Blk.size() * 4)); CK(cudaMalloc(&dD, 128 * 8 * 4));
  CK(cudaMemcpy(drows, rows.data(), KB * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dBlk, Blk.data(), Blk.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, 128 * 8 * 4));
  probe<KIND, F><<<1, 128>>>(map, drows, dBlk, dD);
  CK(cudaDeviceSynchronize());
  std::vector<float> D(128 * 8);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  // reference with quantised operands (tf32 truncation as the hardware does for smem fp32)
  const int M = F < 128 ? 64 : 128;
  std::vector<double> ref((size_t)F * 8);
  double max_ref = 0;
  for (int f = 0; f < F; ++f)
    for (int i = 0; i < 8; ++i) {
      double s = 0;
      for (int k = 0; k < KB; ++k) {
        float g = Bh[(size_t)rows[k] * ld + f];
        float a = KIND == 0 ? tf32_trunc(g) : bf16_rn(g);
        float b = KIND == 0 ? tf32_trunc(Blk[i * KB + k]) : bf16_rn(Blk[i * KB + k]);
        s += (double)a * b;
      }
      ref[(size_t)f * 8 + i] = s;
      max_ref = fmax(max_ref, fabs(s));
    }
  // identity lane mapping check (f -> lane f) and, failing that, search where each row landed
  double max_err = 0;
  for (int f = 0; f < M; ++f)
    for (int i = 0; i < 8; ++i) max_err = fmax(max_err, fabs(ref[(size_t)f * 8 + i] - D[f * 8 + i]));
  printf("%s F=%d M=%d: identity lane map max|D-ref| = %.3e (max|ref| %.3f)\n", name, F, M, max_err, max_ref);
  if (max_err > 1e-4) {
    printf("  searching: row f -> lane\n  ");
    int found = 0;
    for (int f = 0; f < M; ++f) {
      int hit = -1;
      for (int l = 0; l < 128 && hit < 0; ++l) {
        double e = 0;
        for (int i = 0; i < 8; ++i) e = fmax(e, fabs(ref[(size_t)f * 8 + i] - D[l * 8 + i]));
        if (e < 1e-4) hit = l;
      }
      printf("%d:%d ", f, hit);
      found += hit >= 0;
    }
    printf("\n  rows located: %d of %d\n", found, M);
  }
  cudaFree(dB); cudaFree(drows); cudaFree(dBlk); cudaFree(dD);
}

int main() {
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  run<0, 128>("tf32");
  run<0, 64>("tf32");
  run<1, 128>("bf16");
  run<1, 64>("bf16");
  return 0;
}
