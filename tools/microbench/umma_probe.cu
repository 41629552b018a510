// UMMA probe: validates the smem descriptor layouts the tensor-core window kernel relies on and
// measures tiny-N tcgen05.mma throughput.
//   D[f, i] (TMEM, M=128 lanes = features, N=8 columns = window rows)
//     = sum_k G[k][f] * Blk[i][k]       (A = gathered rows, MN-major SW128; B = block, K-major)
// kind::tf32 (K=8) and kind::f16 with bf16 operands (K=16).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128_mn(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;              // version = 1 (sm100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" :: "r"(smem_u32(bar)), "r"(phase));
}

template <int KIND>  // 0 = tf32, 1 = bf16
__global__ void probe(const float* G, const float* Blk, float* D, int reps, long long* cycles, int rot) {
  // G: [KB][128] fp32 (KB = 8 tf32 / 16 bf16 gathered rows); Blk: [8][KB] fp32 (dense block rows)
  constexpr int KB = KIND == 0 ? 8 : 16;
  constexpr int EB = KIND == 0 ? 4 : 2;
  __shared__ __align__(1024) uint8_t sA[KB * 128 * EB];   // atoms of 1 KB: 128 B (MN) x 8 rows (K)
  __shared__ __align__(1024) uint8_t sB[8 * KB * EB];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // fill A: element (f, k) -> atom (k / 8 along K group, f / (128/EB) along MN), row k%8, chunk
  const int per_atom_f = 128 / EB;              // features per 128 B
  const int n_mn_atoms = 128 / per_atom_f;      // 4 (tf32) or 2 (bf16)
  for (int idx = tid; idx < KB * 128; idx += blockDim.x) {
    int k = idx / 128, f = idx % 128;
    int ma = f / per_atom_f, fi = f % per_atom_f;
    int byte = fi * EB;
    int chunk = byte >> 4, within = byte & 15;
    int off;
    if (KIND == 0) {  // SWIZZLE_128B_BASE32B: atom = 4 K-rows x 128 B, 32-B granules XOR row
      int kg = k / 4, kr = k % 4;
      off = kg * 2048 + ma * 512 + kr * 128 + ((((chunk >> 1) ^ kr)) << 5) + ((chunk & 1) << 4) + within;
    } else {          // SWIZZLE_128B: atom = 8 K-rows x 128 B, 16-B chunks XOR row
      int kg = k / 8, kr = k % 8;
      off = kg * 2048 + ma * 1024 + kr * 128 + ((chunk ^ kr) << 4) + within;
    }
    if (KIND == 0) *(float*)(sA + off) = G[k * 128 + f];
    else *(__nv_bfloat16*)(sA + off) = __float2bfloat16(G[k * 128 + f]);
  }
  // fill B: K-major, no swizzle: core matrix = 8 rows x 16 B; k-chunk kc at + kc*128
  for (int idx = tid; idx < 8 * KB; idx += blockDim.x) {
    int i = idx / KB, k = idx % KB;
    int per16 = 16 / EB;
    int kc = k / per16, kk = k % per16;
    int off = kc * 128 + i * 16 + kk * EB;
    if (KIND == 0) *(float*)(sB + off) = Blk[i * KB + k];
    else *(__nv_bfloat16*)(sB + off) = __float2bfloat16(Blk[i * KB + k]);
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tmem_base;
  // descriptors
  uint32_t idesc = (1u << 4) | ((KIND == 0 ? 2u : 1u) << 7) | ((KIND == 0 ? 2u : 1u) << 10) | (1u << 15) | (0u << 16) |
                   ((8u >> 3) << 17) | ((128u >> 4) << 24);
  uint64_t adesc = KIND == 0 ? (desc_none(smem_u32(sA), 512, 2048) | ((uint64_t)1 << 61))
                             : desc_sw128_mn(smem_u32(sA), 1024, 2048);
  uint64_t bdesc = desc_none(smem_u32(sB), 128, 256);
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      uint32_t acc = r >= rot;
      uint32_t dcol = tmem + (uint32_t)((r % rot) * 8);
      if (KIND == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                     :: "r"(dcol), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                     :: "r"(dcol), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    mbar_wait(&bar, 0);
    t1 = clock64();
    cycles[0] = t1 - t0;
  }
  __syncthreads();
  if (tid != 0) mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w reads lanes 32w..32w+31, 8 columns
  if (warp < 4) {
    uint32_t r[8];
    uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int f = warp * 32 + lane;
    for (int i = 0; i < 8; ++i) D[f * 8 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
}

static float tf32_trunc(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x; }
static float bf16_rn(float x) { return __bfloat162float(__float2bfloat16(x)); }

template <int KIND>
void run(const char* name) {
  constexpr int KB = KIND == 0 ? 8 : 16;
  std::mt19937 rng(7);
  std::uniform_real_distribution<float> U(-1, 1);
  std::vector<float> G(KB * 128), Blk(8 * KB), D(128 * 8);
  for (auto& x : G) x = U(rng);
  for (auto& x : Blk) x = (rng() % 3 == 0) ? U(rng) : 0.f;
  // special rows probing rounding: G[0][0] = 1 + 3*2^-12, Blk[0][0] = 1, rest of row/col 0 zero
  for (int k = 0; k < KB; ++k) G[k * 128 + 0] = 0.f;
  for (int k = 0; k < KB; ++k) Blk[0 * KB + k] = 0.f;
  G[0] = 1.0f + 3.0f / 4096.0f; Blk[0] = 1.0f;
  float *dG, *dB, *dD; long long* dc;
  CK(cudaMalloc(&dG, G.size() * 4)); CK(cudaMalloc(&dB, Blk.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4)); CK(cudaMalloc(&dc, 8));
  CK(cudaMemcpy(dG, G.data(), G.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Blk.data(), Blk.size() * 4, cudaMemcpyHostToDevice));
  probe<KIND><<<1, 128>>>(dG, dB, dD, 1, dc, 1);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double max_err = 0, max_ref = 0, max_err_tr = 0;
  for (int f = 0; f < 128; ++f)
    for (int i = 0; i < 8; ++i) {
      double ref = 0, ref_q = 0;
      for (int k = 0; k < KB; ++k) {
        ref += (double)G[k * 128 + f] * Blk[i * KB + k];
        float a = KIND == 0 ? tf32_trunc(G[k * 128 + f]) : bf16_rn(G[k * 128 + f]);
        float b = KIND == 0 ? tf32_trunc(Blk[i * KB + k]) : bf16_rn(Blk[i * KB + k]);
        ref_q += (double)a * b;
      }
      max_err = fmax(max_err, fabs(ref - D[f * 8 + i]));
      max_err_tr = fmax(max_err_tr, fabs(ref_q - D[f * 8 + i]));
      max_ref = fmax(max_ref, fabs(ref));
    }
  printf("%s layout check: max|D-ref| %.3e (vs quantized-operand ref %.3e), max|ref| %.3f, D[0][0]=%.9f (1+3/4096 -> trunc 1.0, RN %.9f)\n",
         name, max_err, max_err_tr, max_ref, D[0], 1.0 + 1.0 / 1024);
  for (int rot : {1, 4, 16, 64}) {
    int reps = 8192;
    probe<KIND><<<1, 128>>>(dG, dB, dD, reps, dc, rot);
    CK(cudaDeviceSynchronize());
    long long c; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
    printf("%s throughput: %d MMAs (M=128,N=8,K=%d) over %d accumulators in %lld cycles = %.2f cyc/MMA\n", name, reps, KB, rot, c, (double)c / reps);
  }
}

int main() {
  run<0>("tf32");
  run<1>("bf16");
  return 0;
}
