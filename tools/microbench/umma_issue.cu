// Issue-cost model of tiny tcgen05.mma (M=128, N=8, K=8 tf32, SS operands), the shape the RSH
// window kernel issues once per 8x8 block.  Variants: plain back-to-back, rotating accumulators,
// a commit per MMA, an mbarrier try_wait per MMA, and several issuing warps in one CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" :: "r"(smem_u32(bar)), "r"(phase));
}

// mode: 0 same acc, 1 rotate 64 accs, 2 rotate + commit each, 3 rotate + try_wait each (completed bar),
//       4 rotate + commit every 4
__global__ void issue(int mode, int reps, int issuers, long long* out) {
  __shared__ __align__(1024) uint8_t sA[4096 * 8];
  __shared__ __align__(1024) uint8_t sB[256 * 8];
  __shared__ uint64_t bar[8], done_bar, ready;
  __shared__ uint32_t tmem_base;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 4096 * 8 / 4; i += blockDim.x) ((float*)sA)[i] = 0.5f;
  for (int i = tid; i < 256 * 8 / 4; i += blockDim.x) ((float*)sB)[i] = 0.25f;
  asm volatile("fence.proxy.async.shared::cta;");
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    mbar_init(&done_bar, issuers);
    mbar_init(&ready, 1);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&ready)));  // completes phase 0
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 17) | (8u << 24);
  long long t0 = clock64();
  if (warp < issuers && lane == 0) {
    uint32_t acc_col = warp * (64 / issuers) * 8;
    const uint32_t col_lo = acc_col, col_hi = acc_col + (64 / issuers) * 8;
    int my = reps / issuers;
    for (int r = 0; r < my; ++r) {
      int s = r & 7;
      uint64_t a = desc(smem_u32(sA + s * 4096), 512, 2048, 1);
      uint64_t b = desc(smem_u32(sB + s * 256), 128, 256, 0);
      uint32_t d = mode == 0 ? tmem : tmem + acc_col;
      if (mode == 3) mbar_wait(&ready, 0);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                   :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(1u));
      if (mode == 2 || (mode == 4 && (r & 3) == 3))
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar[s])));
      acc_col += 8;
      if (acc_col == col_hi) acc_col = col_lo;
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&done_bar)));
  }
  if (tid == 0) {
    mbar_wait(&done_bar, 0);
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
}

int main() {
  long long* d;
  CK(cudaMalloc(&d, 8));
  const char* names[] = {"same accumulator", "rotate 64 accs", "rotate + commit each", "rotate + try_wait each",
                         "rotate + commit every 4"};
  for (int mode = 0; mode < 5; ++mode)
    for (int iss : {1, 2, 4, 8}) {
      if (mode == 0 && iss > 1) continue;
      int reps = 8192;
      issue<<<1, 256>>>(mode, reps, iss, d);
      CK(cudaDeviceSynchronize());
      long long c;
      CK(cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost));
      printf("%-26s issuers %d: %.1f cycles per MMA (M=128 N=8 K=8 tf32)\n", names[mode], iss, (double)c / reps);
    }
  // many CTAs: chip-level rate with one CTA per SM
  long long* dd;
  CK(cudaMalloc(&dd, 148 * 8));
  return 0;
}
