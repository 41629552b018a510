// Tensor-core window path (north-star subsystem (2)) inside the persistent hybrid launch (4).
//
// Per step (one 8x8 bitmap block for TF32, two blocks of the same window for BF16/FP16 -- the
// reference's fragments, execute.py:65-89,171-182):
//   D[f, i] += sum_k G[k][f] * F[i][k]      one tcgen05.mma per M tile; M = features (128, or 64
//                                           when N <= 64), N = 8 window rows, K = 8 (tf32) / 16
// Operand A = G, the step's gathered B rows, staged into shared memory by the TMA
//             (cp.async.bulk.tensor tile::gather4: four B rows x 128 B per instruction) straight
//             into the MN-major 128-byte-swizzled canonical layout (tf32: SWIZZLE_128B_ATOM_32B /
//             descriptor layout 1, bf16/fp16: SWIZZLE_128B / layout 2; validated by
//             tools/microbench/tc2_probe.cu).  Padding slots (a col_id slot whose bitmap column is
//             empty) get row coordinate -1: out of bounds, so the TMA writes zeros.
// Operand B = F, the block's fragment in the MMA's K-major smem image, decoded once per format at
//             schedule time (rsh_tc_fragments: values rounded to tf32 with cvt.rna, or to bf16 /
//             fp16) and fetched with one cp.async.bulk per super-stage.
// D         = fp32 accumulator in TMEM, 8 columns per M tile per work unit.
//
// Warp roles per CTA (one CTA per SM, persistent, cost-balanced contiguous unit ranges):
//   warps 0-7      epilogue, two groups of four (one warp per TMEM lane quadrant); group e drains
//                  the units ua = e (mod 2) of the CTA in order, two at a time (their tcgen05.ld
//                  share one wait) -> streaming C stores, or chunk partials + the ordered ticket
//                  reduction for multi-unit windows
//   next P warps   MMA issuers, one per pipeline (an elected lane issues; tiny MMAs need several
//                  issuing warps per SM to keep the tensor pipe fed)
//   next P warps   producers, one per pipeline: a super-stage is up to R consecutive blocks of one
//                  unit; the producer waits for it to be free, posts expect_tx, bulk-copies the
//                  fragments, and lane j issues block j's gather4s.  Block metadata is loaded one
//                  32-block batch ahead, unit descriptors 32 units at a time.  Afterwards the
//                  producers take the residual / zero-row units (CUDA cores) from a global counter.
// Pipeline p owns the units ua = p (mod P) of the CTA's range and a ring of SSP super-stages,
// consumed strictly in order.
//
// Measured on config 3 (stencil, N = 64, 18 nonzeros per block): the pipeline mechanics alone
// (no gathers, MMAs or stores; flags bits 0, 2, 5, 6) cost ~0.42 ms, the TMA gathers of 128-B
// boxes ~10 cycles each per SM (~0.4 ms for 12.3 M gather4s) -- DESIGN.md section 3.3.
#include <cuda.h>
#include <mutex>
#include "sched.cuh"

namespace rsh {
template <class AccT>
int launch_fixup(const SpmmArgs& a, cudaStream_t st);  // spmm_cc.cu
namespace tc {

constexpr int kEpiGroups = 2;
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kTmemCols = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a protocol bug traps (the launch fails with an error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (uint32_t n = 0; !mbar_try(bar, parity); ++n)
    if (n == (1u << 28)) __trap();
}

#ifdef RSH_TC_PROFILE
// development build only: per-warp cycle counters [warp slot][0 total, 1 wait empty, 2 wait full,
// 3 wait tempty, 4 wait tfull, 5 super-stages / units]
__device__ unsigned long long g_tc_prof[148 * 40][8];
#define PROF_WAIT(slot, stmt)                                      \
  do {                                                             \
    const long long _t = clock64();                                \
    stmt;                                                          \
    prof[slot] += clock64() - _t;                                  \
  } while (0)
#else
#define PROF_WAIT(slot, stmt) stmt
#endif

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

__device__ __forceinline__ void gather4(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int x, int r0, int r1, int r2,
                                        int r3, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(dst),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// Compile-time geometry of one (operand type, N) instantiation.
template <class BT, int NF>
struct Geo {
  static constexpr int EB = (int)sizeof(BT);
  static constexpr int KB = 32 / EB;                 // K rows per MMA (8 tf32, 16 half)
  static constexpr int BPS = KB / 8;                 // bitmap blocks per MMA step
  static constexpr int M = NF >= 128 ? 128 : 64;     // MMA M (features per tile)
  static constexpr int MT = NF >= 128 ? NF / 128 : 1;
  static constexpr int PER_ATOM = 128 / EB;          // features per 128-B swizzle row
  static constexpr int NMA = M * EB / 128;           // MN atoms per tile
  static constexpr int NRA = NF / PER_ATOM;          // MN atoms holding real features (all tiles)
  static constexpr int KGR = EB == 4 ? 4 : 8;        // K rows per swizzle atom
  static constexpr uint32_t LBO = KGR * 128;         // MN atom stride
  static constexpr uint32_t SBO = LBO * NMA;         // K group stride
  static constexpr int TILE = KB * M * EB;           // A bytes per tile per step
  static constexpr int ABYTES = MT * TILE;           // A bytes per step
  static constexpr uint32_t TXB = 8 * NF * EB;       // gathered bytes per block
  static constexpr uint32_t FB = 8 * 8 * EB;         // fragment bytes per block (256 tf32, 128 half)
  static constexpr uint32_t layout = EB == 4 ? 1u : 2u;
  static constexpr uint32_t fmt = EB == 4 ? 2u : (std::is_same<BT, __nv_bfloat16>::value ? 1u : 0u);
  static constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 15) | (1u << 17) |
                                    ((uint32_t)(M >> 4) << 24);
  static constexpr int NACC0 = kTmemCols / (8 * MT);
  static constexpr int NACC = NACC0 < 64 ? NACC0 : 64;
  static constexpr int VEC = NF / 32;                // CUDA-core features per lane (residual units)
  static_assert(NF % PER_ATOM == 0, "unsupported N for this operand type");
  static_assert(ABYTES % 1024 == 0, "stage A regions stay 1024-B aligned");
};

// shared-memory carve-up: [A super-stages][fragment super-stages][barriers][misc]
template <class G, int S, int R>
struct Smem {
  static constexpr int STEPS = R / G::BPS;  // MMA steps per super-stage
  static constexpr size_t A = 0;
  static constexpr size_t F = A + (size_t)S * STEPS * G::ABYTES;
  static constexpr size_t BAR = F + (size_t)S * R * G::FB;
  static constexpr size_t MISC = BAR + (size_t)(2 * S + 2 * G::NACC) * 8;
  static constexpr size_t BYTES = MISC + 64 + 1024;  // + alignment slack
};

// first unit index u in [0, nu] with unit_cost[u] >= target
__device__ __forceinline__ int64_t cost_bound(const int64_t* __restrict__ cost, int64_t nu, int64_t target) {
  int64_t lo = 0, hi = nu;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cost[mid] < target) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// P pipelines x SSP super-stages of R blocks each.  A super-stage holds up to R consecutive blocks
// of one work unit: their gathered B rows (operand A of R / BPS MMA steps) and their fragments.
template <class BT, int NF, int P, int SSP, int R, int kLsu>
__global__ void __launch_bounds__((kEpiWarps + 2 * P) * 32, 1)
    k_spmm_tc(SpmmArgs a, const uint8_t* __restrict__ frags, const __grid_constant__ CUtensorMap bmap) {
  using G = Geo<BT, NF>;
  constexpr int S = P * SSP;
  using L = Smem<G, S, R>;
  static_assert(32 % R == 0 && R % G::BPS == 0, "super-stages tile the 32-block metadata batches");
  constexpr int kMma0 = kEpiWarps, kProd0 = kEpiWarps + P;
  check_workspace(a);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem + L::A;
  uint8_t* sF = smem + L::F;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + G::NACC;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L::MISC);  // [0] tmem base, [2 + e] ticket

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef RSH_TC_PROFILE
  unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();
#endif

  // zero the A stages once: feature atoms no gather writes (fp32 N = 32 under an M = 64 MMA) stay
  // zero for the whole launch
  for (int i = threadIdx.x * 16; i < (int)L::F; i += blockDim.x * 16) *(uint4*)(sA + i) = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      // the producer's arrive.expect_tx (+ gather and fragment bytes); LSU-staged super-stages
      // add one cp.async.mbarrier.arrive.noinc per producer lane
      mbar_init(full + s, (s % SSP) >= SSP - kLsu ? 33 : 1);
      mbar_init(empty + s, 1);  // tcgen05.commit after the super-stage's MMAs
    }
    for (int s = 0; s < G::NACC; ++s) {
      mbar_init(tfull + s, 1);
      mbar_init(tempty + s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMma0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(misc)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = misc[0];

  // this CTA's contiguous, cost-balanced range of window units
  const int64_t nwu = a.s.header[1];
  const int64_t total = a.s.unit_cost[nwu];
  const int64_t NG = gridDim.x;
  const int64_t u0 = cost_bound(a.s.unit_cost, nwu, (total * (int64_t)blockIdx.x) / NG);
  const int64_t u1 =
      blockIdx.x + 1 == NG ? nwu : cost_bound(a.s.unit_cost, nwu, (total * ((int64_t)blockIdx.x + 1)) / NG);

  if (warp >= kProd0) {
    // ------------------------------------------------------------------ producers
    const int p = warp - kProd0;
    uint64_t pol_b, pol_a;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_b));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_a));
    const bool no_gather = a.flags & 1;  // perf-probe knob (results invalid)
    // block metadata of a 32-block batch, lane l <-> block z0 + l (coalesced), loaded one batch
    // ahead; padding slots (no bit in the column) get the out-of-bounds row -1 when the batch is
    // used, which the TMA fills with zeros
    struct Meta {
      unsigned long long bm;
      int4 c0, c1;
    };
    auto load_meta = [&](int32_t z0, int nb, Meta& m) {
      const int64_t blk = (int64_t)z0 + lane;
      m.bm = 0ull;
      m.c0 = make_int4(-1, -1, -1, -1);
      m.c1 = m.c0;
      if (lane < nb) {
        m.bm = ldg_hint64(a.bitmaps + blk, pol_a);
        m.c0 = make_int4_u(ldg_hint(reinterpret_cast<const int4*>(a.col_id + blk * 8), pol_a));
        m.c1 = make_int4_u(ldg_hint(reinterpret_cast<const int4*>(a.col_id + blk * 8) + 1, pol_a));
      }
      if (lane == 0 && nb > 0)  // the batch's fragments, on their way to L2 while this one runs
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(frags + (size_t)z0 * G::FB),
                     "r"((uint32_t)(((nb + 1) & ~1) * G::FB)) : "memory");
    };
    auto pad = [&](const Meta& m, int4& c0, int4& c1) {
      unsigned long long x = m.bm | (m.bm >> 32);
      x |= x >> 16;
      x |= x >> 8;
      const uint32_t cm = (uint32_t)x & 0xffu;
      c0.x = (cm & 1u) ? m.c0.x : -1;
      c0.y = (cm & 2u) ? m.c0.y : -1;
      c0.z = (cm & 4u) ? m.c0.z : -1;
      c0.w = (cm & 8u) ? m.c0.w : -1;
      c1.x = (cm & 16u) ? m.c1.x : -1;
      c1.y = (cm & 32u) ? m.c1.y : -1;
      c1.z = (cm & 64u) ? m.c1.z : -1;
      c1.w = (cm & 128u) ? m.c1.w : -1;
    };
    int64_t q = 0;  // super-stages issued by this pipeline
    // units ua = p + P l of this pipeline, 32 at a time: lane l holds unit l's block range
    for (int64_t ub = p; u0 + ub < u1; ub += 32 * P) {
      const int64_t ul = ub + (int64_t)P * lane;
      const bool uv = u0 + ul < u1;
      const int4 unl = uv ? a.s.units[u0 + ul] : make_int4(0, 0, 0, 0);
      const int nu = __popc(__ballot_sync(0xffffffffu, uv));
      // batches (unit k, offset z0) in order; the next batch's metadata is loaded while the
      // current one is issued
      int k = 0;
      int32_t z = __shfl_sync(0xffffffffu, unl.z, 0), w = __shfl_sync(0xffffffffu, unl.w, 0);
      while (k < nu && z >= w) {  // empty units
        ++k;
        z = __shfl_sync(0xffffffffu, unl.z, k & 31);
        w = __shfl_sync(0xffffffffu, unl.w, k & 31);
      }
      Meta cur;
      int nb = w - z < 32 ? w - z : 32;
      if (k < nu) load_meta(z, nb, cur);
      while (k < nu) {
        // position of the next batch
        int kn = k;
        int32_t zn = z + 32, wn = w;
        while (kn < nu && zn >= wn) {
          ++kn;
          if (kn < nu) {
            zn = __shfl_sync(0xffffffffu, unl.z, kn & 31);
            wn = __shfl_sync(0xffffffffu, unl.w, kn & 31);
          }
        }
        Meta nxt;
        const int nbn = wn - zn < 32 ? wn - zn : 32;
        if (kn < nu) load_meta(zn, nbn, nxt);
        int4 c0, c1;
        pad(cur, c0, c1);
        for (int k0 = 0; k0 < nb; k0 += R, ++q) {
          const int nblk = nb - k0 < R ? nb - k0 : R;
          const int nfb = (nblk + G::BPS - 1) / G::BPS * G::BPS;  // blocks of whole steps
          const int ss = p * SSP + (int)(q % SSP);
          PROF_WAIT(1, mbar_wait(empty + ss, (uint32_t)(((q / SSP) & 1) ^ 1)));
          uint8_t* stA = sA + (size_t)ss * L::STEPS * G::ABYTES;
          // staging engine of this super-stage: the TMA (gather4) or, for the last kLsu of each
          // pipeline's SSP super-stages, the LSU (16-byte cp.async per lane): the two engines run
          // side by side
          const bool lsu = (ss % SSP) >= SSP - kLsu;
          if (lane == 0) {
            const bool no_frag = a.flags & 64;  // perf-probe knobs: no fragment copy / a fixed one
            mbar_expect_tx(full + ss, ((no_gather || lsu) ? 0u : nfb * G::TXB) + (no_frag ? 0u : nfb * G::FB));
            if (!no_frag)
              asm volatile(
                  "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                  ::"r"(smem_u32(sF + (size_t)ss * R * G::FB)),
                  "l"(frags + ((a.flags & 128) ? (size_t)0 : (size_t)(z + k0) * G::FB)), "r"(nfb * G::FB),
                  "r"(smem_u32(full + ss)), "l"(pol_a)
                  : "memory");
          }
          __syncwarp();
          if (lsu) {
            // block j of the super-stage, row r, 16-byte chunk cc of the row's real features: one
            // cp.async per lane per chunk into the swizzled operand image (padding rows: zero
            // fill); completion reaches the full barrier through cp.async.mbarrier.arrive.noinc
            constexpr int CPR = NF * G::EB / 16;  // chunks per row
            constexpr int CPB = 8 * CPR;          // chunks per block
            const char* Bb = reinterpret_cast<const char*>(a.B);
            const int64_t rowb = a.ldb * G::EB;
            for (int j = 0; j < nfb; ++j) {
              const int src = (k0 + j) & 31;
              int col8[8];
              col8[0] = __shfl_sync(0xffffffffu, c0.x, src);
              col8[1] = __shfl_sync(0xffffffffu, c0.y, src);
              col8[2] = __shfl_sync(0xffffffffu, c0.z, src);
              col8[3] = __shfl_sync(0xffffffffu, c0.w, src);
              col8[4] = __shfl_sync(0xffffffffu, c1.x, src);
              col8[5] = __shfl_sync(0xffffffffu, c1.y, src);
              col8[6] = __shfl_sync(0xffffffffu, c1.z, src);
              col8[7] = __shfl_sync(0xffffffffu, c1.w, src);
              const int step = j / G::BPS, b = j % G::BPS;
              uint8_t* stS = stA + step * G::ABYTES;
            // rows covered by one warp instruction: 32 / CPR (CPR >= 32: one row, warp-uniform)
            constexpr int RPI = CPR >= 32 ? 1 : 32 / CPR;
#pragma unroll
              for (int it = 0; it < (CPB + 31) / 32; ++it) {
                const int c = lane + 32 * it;
                if (CPB % 32 == 0 || c < CPB) {
                  const int r = c / CPR, cc = c % CPR;
                  const int fb = cc * 16, ga = fb >> 7, ci = (fb & 127) >> 4;
                  const int t = ga / G::NMA, ma = ga % G::NMA;
                  const int kk = 8 * b + r, kg = kk / G::KGR, kr = kk % G::KGR;
                  const int within = G::EB == 4 ? kr * 128 + ((((ci >> 1) ^ kr)) << 5) + ((ci & 1) << 4)
                                                : kr * 128 + ((ci ^ kr) << 4);
                  // this instruction's rows are r0 .. r0 + RPI - 1 (r0 compile-time): RPI - 1 selects
                  const int r0 = CPR >= 32 ? (32 * it) / CPR : (32 * it) / CPR;
                  int col = col8[r0 & 7];
#pragma unroll
                  for (int q8 = 1; q8 < RPI; ++q8)
                    if (r == r0 + q8) col = col8[(r0 + q8) & 7];
                  const uint32_t dst = smem_u32(stS + t * G::TILE) + kg * G::SBO + ma * G::LBO + within;
                  const char* srcp = Bb + (col >= 0 ? (int64_t)col * rowb + fb : 0);
                  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst),
                               "l"(srcp), "r"(col >= 0 ? 16 : 0), "l"(pol_b)
                               : "memory");
                }
              }
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + ss)) : "memory");
          } else {
            // lanes k0 .. k0 + nfb - 1 gather their own block's rows (lanes past nblk: the missing
            // half of a bf16 step, rows -1): K quad qd (rows 4qd..4qd+3) x real MN atom ga; block j
            // of the super-stage is K group (j % BPS) of step j / BPS
            const int j = lane - k0;
            if (j >= 0 && j < nfb && !no_gather) {
              const int step = j / G::BPS, b = j % G::BPS;
#pragma unroll
              for (int qd = 0; qd < 2; ++qd) {
                const int4 cc = qd ? c1 : c0;
                const int kr0 = 8 * b + 4 * qd, kg = kr0 / G::KGR, qin = kr0 % G::KGR;
#pragma unroll
                for (int ga = 0; ga < G::NRA; ++ga) {
                  const int t = ga / G::NMA, ma = ga % G::NMA;
                  const uint32_t dst = smem_u32(stA + step * G::ABYTES + t * G::TILE) + kg * G::SBO + ma * G::LBO +
                                       qin * 128;
                  gather4(&bmap, dst, full + ss, ga * G::PER_ATOM, cc.x, cc.y, cc.z, cc.w, pol_b);
                }
              }
            }
          }
        }
        k = kn;
        z = zn;
        w = wn;
        nb = nbn;
        cur = nxt;
      }
    }

    // residual and zero-row units (CUDA cores), fetched dynamically across the grid
    const int64_t nunits = a.s.header[2];
    for (;;) {
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(a.s.counters, 1u);
      t = __shfl_sync(0xffffffffu, t, 0);
      const int64_t u = nwu + t;
      if (u >= nunits) break;
      const int4 un = a.s.units[u];
      if ((un.x & 3) == kUnitResidual) residual_rows<G::VEC, BT, float>(a, un.y, un.z, 1);
      else zero_rows<G::VEC>(a, un.y, un.z);
    }
    __syncwarp();
    if (lane == 0) {
      const uint32_t producers = gridDim.x * P;
      if (atomicAdd(a.s.counters + 1, 1u) == producers - 1) {
        a.s.counters[0] = 0;
        a.s.counters[1] = 0;
      }
    }
  } else if (warp >= kMma0) {
    // ------------------------------------------------------------------ MMA issuers
    const int p = warp - kMma0;
    int64_t q = 0;
    const bool no_mma = a.flags & 4;  // perf-probe knob (results invalid)
    const uint64_t adesc0 = umma_desc(smem_u32(sA), G::LBO, G::SBO, G::layout);
    const uint64_t bdesc0 = umma_desc(smem_u32(sF), 128, 256, 0);
    for (int64_t ub = p; u0 + ub < u1; ub += 32 * P) {
      // the block ranges of this pipeline's next 32 units, one per lane
      const int64_t ul = ub + (int64_t)P * lane;
      const bool uv = u0 + ul < u1;
      const int4 unl = uv ? a.s.units[u0 + ul] : make_int4(0, 0, 0, 0);
      const int nu = __popc(__ballot_sync(0xffffffffu, uv));
      for (int k = 0; k < nu; ++k) {
        const int64_t ua = ub + (int64_t)P * k;
        const int32_t uz = __shfl_sync(0xffffffffu, unl.z, k), uw = __shfl_sync(0xffffffffu, unl.w, k);
        if (lane == 0) {
          const int slot = (int)(ua % G::NACC);
          PROF_WAIT(3, mbar_wait(tempty + slot, (uint32_t)(((ua / G::NACC) & 1) ^ 1)));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (uz == uw) {
            mbar_arrive(tfull + slot);
          } else {
            bool first = true;
            for (int32_t z0 = uz; z0 < uw; z0 += 32) {
              const int nb = uw - z0 < 32 ? uw - z0 : 32;
              for (int k0 = 0; k0 < nb; k0 += R, ++q) {
                const int nblk = nb - k0 < R ? nb - k0 : R;
                const int nsteps = (nblk + G::BPS - 1) / G::BPS;
                const int ss = p * SSP + (int)(q % SSP);
                PROF_WAIT(2, mbar_wait(full + ss, (uint32_t)((q / SSP) & 1)));
                // LSU-staged rows are generic-proxy writes: order them before the MMA's
                // async-proxy reads (consumer-side proxy fence after the barrier's acquire)
                if ((ss % SSP) >= SSP - kLsu) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                // descriptors: the 14-bit start-address field (bytes >> 4) of the stage-0 descriptors
                // plus the stage / step / tile offset (shared memory < 256 KB: no carry out)
                const uint64_t abase = adesc0 + (uint64_t)(((uint32_t)ss * (L::STEPS * G::ABYTES)) >> 4);
                const uint64_t bbase = bdesc0 + (uint64_t)(((uint32_t)ss * (R * G::FB)) >> 4);
                const uint32_t dbase = tmem + (uint32_t)(slot * G::MT * 8);
                for (int st = 0; st < nsteps; ++st) {
                  const uint64_t bdesc = bbase + (uint64_t)(((uint32_t)st * (G::BPS * G::FB)) >> 4);
                  const uint32_t acc = first ? 0u : 1u;
#pragma unroll
                  for (int t = 0; t < G::MT; ++t) {
                    const uint64_t adesc = abase + (uint64_t)(((uint32_t)st * G::ABYTES + t * G::TILE) >> 4);
                    const uint32_t d = dbase + (uint32_t)(t * 8);
                    if (no_mma) continue;
                    if constexpr (G::EB == 4)
                      asm volatile("{\n.reg .pred pp;\nsetp.ne.b32 pp, %4, 0;\n"
                                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, pp;\n}" ::"r"(d),
                                   "l"(adesc), "l"(bdesc), "r"(G::idesc), "r"(acc));
                    else
                      asm volatile("{\n.reg .pred pp;\nsetp.ne.b32 pp, %4, 0;\n"
                                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pp;\n}" ::"r"(d),
                                   "l"(adesc), "l"(bdesc), "r"(G::idesc), "r"(acc));
                  }
                  first = false;
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                   smem_u32(empty + ss))
                               : "memory");
              }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               smem_u32(tfull + slot))
                           : "memory");
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (2 groups x 4 warps)
    const int e = warp >> 2, qd = warp & 3;
    // feature of this lane in tile t: M = 128 -> lane quadrant qd holds features 32 qd + lane;
    // M = 64 -> D row f sits in TMEM lane (f % 16) + 32 (f / 16) (tools/microbench/tc2_probe.cu)
    const int fl = G::M == 128 ? qd * 32 + lane : qd * 16 + lane;
    const bool lane_ok = G::M == 128 ? true : (lane < 16 && fl < NF);
    constexpr int U = G::MT == 1 ? 2 : 1;  // units drained per round (their TMEM loads share one wait)
    for (int64_t ub = e; u0 + ub < u1; ub += 32 * kEpiGroups) {
      // the next 32 units of this group, one per lane: descriptor, first row, partial slot, chunks
      const int64_t ul = ub + (int64_t)kEpiGroups * lane;
      const bool uv = u0 + ul < u1;
      const int4 unl = uv ? a.s.units[u0 + ul] : make_int4(0, 0, 0, 0);
      const int32_t gl = unl.y;
      const int64_t ridl = uv ? (int64_t)a.s.grp_rid[gl] : 0;
      const int32_t psl = uv ? a.s.grp_slot[gl] : -1;
      const int32_t nchl = (uv && psl >= 0) ? a.s.grp_nch[gl] : 0;
      const int nu = __popc(__ballot_sync(0xffffffffu, uv));
      for (int k0 = 0; k0 < nu; k0 += U) {
        float r[U][G::MT][8];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
          const int ku = k0 + uu;
          if (ku >= nu) break;
          const int64_t ua = ub + (int64_t)kEpiGroups * ku;
          const int slot = (int)(ua % G::NACC);
          const bool has = __shfl_sync(0xffffffffu, unl.z, ku) != __shfl_sync(0xffffffffu, unl.w, ku);
          PROF_WAIT(4, mbar_wait(tfull + slot, (uint32_t)((ua / G::NACC) & 1)));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int t = 0; t < G::MT; ++t) {
            if (has && !(a.flags & 32)) {  // bit 5: perf-probe knob, no TMEM loads / stores
              const uint32_t taddr = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)((slot * G::MT + t) * 8);
              uint32_t v[8];
              asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                           : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                             "=r"(v[7])
                           : "r"(taddr));
#pragma unroll
              for (int i = 0; i < 8; ++i) r[uu][t][i] = __uint_as_float(v[i]);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) r[uu][t][i] = 0.f;
            }
          }
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int uu = 0; uu < U; ++uu)
            if (k0 + uu < nu) mbar_arrive(tempty + (int)((ub + (int64_t)kEpiGroups * (k0 + uu)) % G::NACC));
        }
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
          const int ku = k0 + uu;
          if (ku >= nu) break;
          const int32_t g = __shfl_sync(0xffffffffu, gl, ku);
          const int32_t k = __shfl_sync(0xffffffffu, unl.x, ku) >> 2;
          const int64_t rid = __shfl_sync(0xffffffffu, ridl, ku);
          const int32_t pslot = __shfl_sync(0xffffffffu, psl, ku);
          const int32_t nch = __shfl_sync(0xffffffffu, nchl, ku);
          const int64_t avail = a.window_size < a.n_rows - rid ? a.window_size : a.n_rows - rid;
          if (pslot < 0) {
            if (lane_ok && !(a.flags & 32)) {
              float* c0 = a.C + rid * a.ldc + fl;
              if (avail >= 8) {
#pragma unroll
                for (int t = 0; t < G::MT; ++t)
#pragma unroll
                  for (int i = 0; i < 8; ++i) __stcs(c0 + i * a.ldc + t * 128, r[uu][t][i]);
              } else {
#pragma unroll
                for (int t = 0; t < G::MT; ++t)
#pragma unroll
                  for (int i = 0; i < 8; ++i)
                    if (i < avail) __stcs(c0 + i * a.ldc + t * 128, r[uu][t][i]);
              }
            }
            continue;
          }
          float* part = reinterpret_cast<float*>(a.partials) + ((int64_t)(pslot + k) * 8) * a.N;
          if (lane_ok) {
#pragma unroll
            for (int t = 0; t < G::MT; ++t)
#pragma unroll
              for (int i = 0; i < 8; ++i) __stcg(part + (int64_t)i * a.N + t * 128 + fl, r[uu][t][i]);
          }
          // one thread publishes for the group (bar.sync orders the others' stores before its
          // fence) and, if it took the last ticket, acquires for all; windows with more than
          // kTicketMax chunks are left to the fixup kernels
          if (nch > kTicketMax) continue;
          asm volatile("bar.sync %0, 128;" ::"r"(1 + e) : "memory");
          if (qd == 0 && lane == 0) {
            __threadfence();
            const uint32_t tk = atomicAdd(a.s.ticket + g, 1u);
            if ((int32_t)tk == nch - 1) __threadfence();
            misc[2 + e] = tk;
          }
          asm volatile("bar.sync %0, 128;" ::"r"(1 + e) : "memory");
          if ((int32_t)misc[2 + e] == nch - 1) {
            if (lane_ok) {
              for (int t = 0; t < G::MT; ++t) {
                const int64_t f = t * 128 + fl;
                for (int i = 0; i < avail; ++i) {
                  // partials summed in chunk order; loads issued 8 chunks ahead of the adds
                  const float* part0 = reinterpret_cast<const float*>(a.partials) + (int64_t)i * a.N + f;
                  const int64_t cstride = (int64_t)8 * a.N;
                  float sum = 0.f;
                  int kk = 0;
                  for (; kk + 8 <= nch; kk += 8) {
                    float buf[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) buf[u] = __ldcg(part0 + (int64_t)(pslot + kk + u) * cstride);
#pragma unroll
                    for (int u = 0; u < 8; ++u) sum += buf[u];
                  }
                  for (; kk < nch; ++kk) sum += __ldcg(part0 + (int64_t)(pslot + kk) * cstride);
                  __stcs(a.C + (rid + i) * a.ldc + f, sum);
                }
              }
            }
            if (qd == 0 && lane == 0) a.s.ticket[g] = 0;
          }
          asm volatile("bar.sync %0, 128;" ::"r"(1 + e) : "memory");
        }
      }
    }
  }

#ifdef RSH_TC_PROFILE
  if (lane == 0) {
    prof[0] = clock64() - t_start;
    const int slot = blockIdx.x * 40 + warp;
    if (slot < 148 * 40)
      for (int i = 0; i < 8; ++i) atomicAdd(&g_tc_prof[slot][i], prof[i]);
  }
#endif
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kMma0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// ---- schedule-time fragments -------------------------------------------------------------
// Every block's 8x8 fragment decoded once per (format, operand type) into the exact shared-memory
// image the MMA reads (K-major, no swizzle: row i at 16 i, K chunk kc at 128 kc): tf32 -> 256 B
// per block (values rounded with cvt.rna); bf16 / fp16 -> 128 B per block (round to nearest), two
// consecutive blocks forming the K = 16 operand of one step.  Value of bit pos = values[vstart +
// popc(bits below pos)] (tile.py:123-131 order).  Two zero blocks of padding follow the last.
template <class BT>
__global__ void k_fragments(const unsigned long long* __restrict__ bitmaps, const int32_t* __restrict__ vstart,
                            const float* __restrict__ values, int64_t n_blocks, uint8_t* out) {
  constexpr int EB = (int)sizeof(BT);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t blk = tid >> 6;
  const int pos = (int)(tid & 63);
  if (blk >= n_blocks + 2) return;
  float v = 0.f;
  if (blk < n_blocks) {
    const unsigned long long bm = __ldg(bitmaps + blk);
    if ((bm >> pos) & 1ull) v = __ldg(values + __ldg(vstart + blk) + __popcll(bm & ((1ull << pos) - 1ull)));
  }
  const int i = pos >> 3, c = pos & 7;
  uint8_t* o = out + blk * (64 * EB);
  if constexpr (EB == 4) {
    *(uint32_t*)(o + (c >> 2) * 128 + i * 16 + (c & 3) * 4) = to_tf32(v);
  } else if constexpr (std::is_same<BT, __nv_bfloat16>::value) {
    *(__nv_bfloat16*)(o + i * 16 + c * 2) = __float2bfloat16_rn(v);
  } else {
    *(__half*)(o + i * 16 + c * 2) = __float2half_rn(v);
  }
}

// ---- host side ---------------------------------------------------------------------------

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiled)p;
  });
  return fn;
}

// B as a 2-D tensor [b_rows, N] (row stride ldb elements), boxes of one row x 128 bytes, swizzled
// into the MMA operand layout, out-of-bounds rows read as zeros
template <class BT>
int make_bmap(CUtensorMap* map, const void* B, int64_t b_rows, int64_t ldb, int N) {
  EncodeTiled enc = encode_fn();
  if (!enc) return fail(kCuda, "rsh_spmm_tc: cuTensorMapEncodeTiled is unavailable");
  constexpr int EB = (int)sizeof(BT);
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)(b_rows > 0 ? b_rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(ldb * EB)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / EB), 1}, estr[2] = {1, 1};
  const CUtensorMapDataType dt = EB == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                         : (std::is_same<BT, __nv_bfloat16>::value ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                                                    : CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  CUresult r = enc(map, dt, 2, const_cast<void*>(B), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   EB == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(kInvalid, "rsh_spmm_tc: tensor map encode failed (%d)", (int)r);
  return kOk;
}

template <class BT, int NF, int P, int SSP, int R, int LSU>
int launch(const SpmmArgs& a, const uint8_t* frags, const void* B, int64_t b_rows, cudaStream_t st) {
  using G = Geo<BT, NF>;
  using L = Smem<G, P * SSP, R>;
  static_assert(L::BYTES <= 227 * 1024, "shared memory budget");
  CUtensorMap map;
  RSH_OK(make_bmap<BT>(&map, B, b_rows, a.ldb, NF));
  auto kern = k_spmm_tc<BT, NF, P, SSP, R, LSU>;
  // opt in to the dynamic shared memory once (thread-safe static init)
  static const cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
  RSH_CUDA(attr);
  kern<<<sm_count(), (kEpiWarps + 2 * P) * 32, L::BYTES, st>>>(a, frags, map);
  RSH_LAUNCHED("k_spmm_tc");
  return launch_fixup<float>(a, st);
}

// pipelines x super-stages x blocks per super-stage (~200 KB of shared memory) and how many of a
// pipeline's super-stages the LSU stages (measured: N <= 64 runs best on the TMA alone -- config 3
// 0.84 vs 0.93 ms half-and-half -- while wider rows gain from the second engine, config 2 1.52 vs
// 1.68 ms; profiles/r02_tc_kernel_evolution.txt)
template <class BT>
int dispatch_n(const SpmmArgs& a, const uint8_t* frags, const void* B, int64_t b_rows, int N, cudaStream_t st) {
  if constexpr (sizeof(BT) == 4) {
    switch (N) {
      case 32: return launch<BT, 32, 10, 2, 4, 0>(a, frags, B, b_rows, st);
      case 64: return launch<BT, 64, 10, 2, 4, 0>(a, frags, B, b_rows, st);
      case 128: return launch<BT, 128, 8, 2, 2, 1>(a, frags, B, b_rows, st);
      case 256: return launch<BT, 256, 6, 2, 2, 1>(a, frags, B, b_rows, st);
    }
  } else {
    switch (N) {
      case 64: return launch<BT, 64, 8, 2, 8, 0>(a, frags, B, b_rows, st);
      case 128: return launch<BT, 128, 8, 2, 4, 1>(a, frags, B, b_rows, st);
      case 256: return launch<BT, 256, 6, 2, 4, 1>(a, frags, B, b_rows, st);
    }
  }
  return fail(kInvalid, "rsh_spmm_tc: unsupported N %d", N);
}

}  // namespace tc
}  // namespace rsh

using namespace rsh;

extern "C" {

#ifdef RSH_TC_PROFILE
int rsh_tc_profile_read(unsigned long long* host_out) {
  RSH_CUDA(cudaMemcpyFromSymbol(host_out, tc::g_tc_prof, sizeof(tc::g_tc_prof)));
  static unsigned long long zeros[148 * 40][8];
  RSH_CUDA(cudaMemcpyToSymbol(tc::g_tc_prof, zeros, sizeof(zeros)));
  return kOk;
}
#endif

size_t rsh_tc_fragment_bytes(int64_t n_blocks, int32_t b_dtype) {
  return (size_t)(n_blocks + 2) * (b_dtype == 0 ? 256 : 128);
}

// Schedule-time fragments for rsh_spmm_tc (the decoded 8x8 blocks in the MMA operand layout).
int rsh_tc_fragments(int64_t n_rows, int64_t n_entries, const uint64_t* bitmaps, const float* tc_values, int64_t n_blocks,
                     int64_t n_res, int32_t b_dtype, const void* sched, size_t sched_bytes, void* out, size_t out_bytes,
                     cudaStream_t st) {
  if (b_dtype < 0 || b_dtype > 2) return fail(kInvalid, "rsh_tc_fragments: bad b_dtype");
  Sched s;
  const size_t need = sched_layout(const_cast<void*>(sched), n_rows, n_entries, n_blocks, n_res, &s);
  if (!sched || sched_bytes < need) return fail(kInvalid, "rsh_tc_fragments: schedule buffer too small");
  if (!out || out_bytes < rsh_tc_fragment_bytes(n_blocks, b_dtype) || ((uintptr_t)out & 15))
    return fail(kInvalid, "rsh_tc_fragments: output smaller than rsh_tc_fragment_bytes() or misaligned");
  const int64_t work = (n_blocks + 2) * 64;
  const auto bm = (const unsigned long long*)bitmaps;
  if (b_dtype == 0) tc::k_fragments<float><<<grid_1d(work), kThreads, 0, st>>>(bm, s.vstart, tc_values, n_blocks, (uint8_t*)out);
  else if (b_dtype == 1)
    tc::k_fragments<__nv_bfloat16><<<grid_1d(work), kThreads, 0, st>>>(bm, s.vstart, tc_values, n_blocks, (uint8_t*)out);
  else tc::k_fragments<__half><<<grid_1d(work), kThreads, 0, st>>>(bm, s.vstart, tc_values, n_blocks, (uint8_t*)out);
  RSH_LAUNCHED("k_fragments");
  return kOk;
}

// Tensor-core hybrid SpMM (execute.py:155-218 semantics, TF32 / BF16 / FP16 operands, fp32
// accumulation).  Requirements: N in {32, 64, 128, 256} for fp32 B, {64, 128, 256} for half B;
// f32 accumulation; 16-byte aligned B rows; fragments from rsh_tc_fragments for this b_dtype.
int rsh_spmm_tc(int64_t n_rows, int32_t window_size, int64_t n_entries, const uint64_t* bitmaps,
                const int32_t* col_id, const void* fragments, size_t fragment_bytes, int64_t n_blocks,
                const int32_t* res_row_id, const int64_t* res_offset, const int32_t* res_col_id, const float* res_values,
                int64_t n_res, const void* B, int64_t b_rows, int64_t ldb, int32_t b_dtype, int64_t N, float* C,
                int64_t ldc, int32_t flags, void* sched, size_t sched_bytes, void* partials, size_t partial_bytes,
                cudaStream_t st) {
  if (b_dtype < 0 || b_dtype > 2) return fail(kInvalid, "rsh_spmm_tc: bad b_dtype");
  const bool ok_n = b_dtype == 0 ? (N == 32 || N == 64 || N == 128 || N == 256) : (N == 64 || N == 128 || N == 256);
  if (!ok_n)
    return fail(kInvalid, "rsh_spmm_tc: N must be in {32, 64, 128, 256} (fp32) or {64, 128, 256} (bf16/fp16), got %lld",
                (long long)N);
  size_t eb = b_dtype == 0 ? 4 : 2;
  if (ldb < N || ldc < N || ((uintptr_t)B & 15) || ((ldb * eb) & 15))
    return fail(kInvalid, "rsh_spmm_tc: B rows must be 16-byte aligned");
  if (b_rows < 0 || b_rows > 0x7fffffffLL) return fail(kInvalid, "rsh_spmm_tc: B row count out of range");
  if (!fragments || fragment_bytes < rsh_tc_fragment_bytes(n_blocks, b_dtype) || ((uintptr_t)fragments & 15))
    return fail(kInvalid, "rsh_spmm_tc: fragments missing or smaller than rsh_tc_fragment_bytes() for this dtype");
  Sched s;
  size_t need = sched_layout(sched, n_rows, n_entries, n_blocks, n_res, &s);
  if (!sched || sched_bytes < need) return fail(kInvalid, "rsh_spmm_tc: schedule buffer too small");
  SpmmArgs a;
  a.bitmaps = (const unsigned long long*)bitmaps;
  a.col_id = col_id;
  a.tc_values = nullptr;
  a.res_row = res_row_id;
  a.res_off = res_offset;
  a.res_col = res_col_id;
  a.res_val = res_values;
  a.B = B;
  a.ldb = ldb;
  a.C = C;
  a.ldc = ldc;
  a.n_rows = n_rows;
  a.N = (int32_t)N;
  a.window_size = window_size;
  a.s = s;
  RSH_OK(bind_workspace(a, partials, partial_bytes, n_entries, sizeof(float)));
  a.flags = flags;
  const auto* fr = (const uint8_t*)fragments;
  if (b_dtype == 0) return tc::dispatch_n<float>(a, fr, B, b_rows, (int)N, st);
  if (b_dtype == 1) return tc::dispatch_n<__nv_bfloat16>(a, fr, B, b_rows, (int)N, st);
  return tc::dispatch_n<__half>(a, fr, B, b_rows, (int)N, st);
}

}  // extern "C"
