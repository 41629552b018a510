// Tensor-core window path (north-star subsystem (2)) inside the persistent hybrid launch (4).
//
// Per 8-row window block (the reference's 8x8 bitmap fragment, execute.py:65-89,171-182):
//   D[f, i] += sum_k B[col_k][f] * Ablk[i][k]      one tcgen05.mma, M = 128 features,
//                                                  N = 8 window rows, K = 8 (tf32) / 16 (bf16)
// Operand A  = the 8 gathered B rows, MN-major, 128-byte swizzled canonical layout, staged into
//              shared memory by cp.async (16-byte, L1-allocating: hot B rows hit in L1) with
//              zero-fill for padding slots (a col_id slot whose bitmap column is empty);
// Operand B  = the decoded bitmap block (popc-rank scatter), K-major, rounded to tf32 (cvt.rna);
// D          = fp32 accumulator in TMEM (8 columns per window, up to 64 windows in flight).
//
// Warp roles per CTA (one CTA per SM, persistent, cost-balanced contiguous unit ranges):
//   warps 0-3   epilogue: tcgen05.ld -> registers -> streaming C stores (or chunk partials +
//               ordered ticket reduction for windows longer than one unit)
//   warps 4-7   MMA issuers, one per pipeline / SM sub-partition (+ TMEM allocation)
//   warps 8-15  producers, 2 per pipeline: block metadata, LDG gather into registers, swizzled
//               STS into the stage, decode, mbarrier signalling;
//               afterwards they take the residual / zero-row units (CUDA-core path) from a
//               global counter.
// Units ua = w (mod 4) of the CTA's range form pipeline w with its own stage ring, consumed
// strictly in order; the epilogue drains accumulators in unit order.
#include "sched.cuh"

namespace rsh {
template <class AccT>
int launch_fixup(const SpmmArgs& a, cudaStream_t st);  // spmm_cc.cu
namespace tc {

constexpr int kPipes = 4;        // independent producer -> MMA pipelines per CTA
constexpr int kProdPerPipe = 2;  // producer warps per pipeline
constexpr int kEpiWarps = 4;
constexpr int kMmaWarp0 = 4;
constexpr int kMmaWarps = kPipes;
constexpr int kProd0 = kMmaWarp0 + kMmaWarps;
constexpr int kProdWarps = kPipes * kProdPerPipe;
constexpr int kThreadsTC = (kProd0 + kProdWarps) * 32;
constexpr int kTileBytes = 4096;  // A operand bytes per 128-feature tile per block
constexpr int kBopBytes = 256;    // decoded block (8 rows x 32 B)
constexpr int kTmemCols = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
    if (n == (1u << 26)) __trap();
}

// Optional per-CTA role timing (flags bit 4): cycle counters, read back with rsh_tc_profile().
constexpr int kProfSlots = 16;
__device__ unsigned long long g_tc_prof[1024][kProfSlots];

struct Prof {
  bool on;
  unsigned long long v[kProfSlots];
  __device__ void flush(int cta, int lo, int hi) {
    if (!on) return;
    for (int i = lo; i < hi; ++i)
      if (v[i]) atomicAdd(&g_tc_prof[cta & 1023][i], v[i]);
  }
};
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, Prof& p, int slot) {
  if (!p.on) {
    mbar_wait(bar, parity);
    return;
  }
  const long long t = clock64();
  mbar_wait(bar, parity);
  p.v[slot] += clock64() - t;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

// Operand A (gathered rows) smem layouts, MN-major, one 4 KB tile per 128 features:
//   tf32: SWIZZLE_128B_BASE32B (layout 1) atoms of 4 K-rows x 128 B with 32-B granules XOR'd by
//         the row; 4 MN atoms (LBO 512 B) x 2 K groups (SBO 2048 B) for K = 8
//   bf16/f16: SWIZZLE_128B (layout 2) atoms of 8 K-rows x 128 B with 16-B chunks XOR'd by the
//         row; 2 MN atoms (LBO 1024 B) x 2 K groups (SBO 2048 B) for K = 16, the second all zero
// (validated by tools/microbench/umma_probe.cu against a CPU reference)
template <class BT>
struct Kind;
template <>
struct Kind<float> {  // kind::tf32
  static constexpr uint32_t fmt = 2;
  static constexpr int eb = 4;
  static constexpr uint32_t layout = 1, lbo = 512, sbo = 2048;
};
template <>
struct Kind<__nv_bfloat16> {  // kind::f16 with bf16 operands, K = 16 (upper 8 zero)
  static constexpr uint32_t fmt = 1;
  static constexpr int eb = 2;
  static constexpr uint32_t layout = 2, lbo = 1024, sbo = 2048;
};
template <>
struct Kind<__half> {
  static constexpr uint32_t fmt = 0;
  static constexpr int eb = 2;
  static constexpr uint32_t layout = 2, lbo = 1024, sbo = 2048;
};

// byte offset inside a 4 KB A tile of 16-B chunk ci (0..7) of MN atom ma for gathered row k
template <int EB>
__device__ __forceinline__ uint32_t a_offset(int ma, int k, int ci) {
  if constexpr (EB == 4) {
    const int kg = k >> 2, kr = k & 3;
    return kg * 2048 + ma * 512 + kr * 128 + ((((ci >> 1) ^ kr)) << 5) + ((ci & 1) << 4);
  } else {
    return ma * 1024 + k * 128 + ((ci ^ k) << 4);
  }
}

template <class BT>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (Kind<BT>::eb == 4)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

template <bool kL1>
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint32_t src_bytes) {
  if constexpr (kL1)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
  else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// first unit index u in [0, nu] with unit_cost[u] >= target
__device__ __forceinline__ int64_t cost_bound(const int64_t* __restrict__ cost, int64_t nu, int64_t target) {
  int64_t lo = 0, hi = nu;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cost[mid] < target) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <class BT, int MT, int STAGES, bool kL1>
__global__ void __launch_bounds__(kThreadsTC, 1) k_spmm_tc(SpmmArgs a) {
  constexpr int EB = Kind<BT>::eb;
  constexpr int NACC = kTmemCols / (8 * MT) < 64 ? kTmemCols / (8 * MT) : 64;
  constexpr int kVec = 4 * MT;  // per-lane features (N = 128 MT) for the CUDA-core tail units
  constexpr int SP = STAGES / kPipes;  // stages per pipeline
  static_assert(STAGES % kPipes == 0, "stages split evenly across pipelines");
  static_assert(SP >= 2, "at least double buffering per pipeline");
  check_workspace(a);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                                   // STAGES * MT * 4 KB
  uint8_t* sB = sA + STAGES * MT * kTileBytes;          // STAGES * 256 B decoded blocks
  uint64_t* full = (uint64_t*)(sB + STAGES * kBopBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + NACC;
  uint32_t* misc = (uint32_t*)(tempty + NACC);         // [0] tmem base, [1] ticket broadcast

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // zero operand memory once: padding never leaks stale data, bf16 K-half stays zero
  for (int i = threadIdx.x * 16; i < STAGES * (MT * kTileBytes + kBopBytes); i += kThreadsTC * 16)
    *(uint4*)(smem + i) = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int s = 0; s < NACC; ++s) {
      mbar_init(tfull + s, 1);
      mbar_init(tempty + s, kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp0) {
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
  const int64_t G = gridDim.x;
  const int64_t u0 = cost_bound(a.s.unit_cost, nwu, (total * (int64_t)blockIdx.x) / G);
  const int64_t u1 = blockIdx.x + 1 == G ? nwu : cost_bound(a.s.unit_cost, nwu, (total * ((int64_t)blockIdx.x + 1)) / G);
  Prof prof;
  prof.on = (a.flags & 16) != 0;
#pragma unroll
  for (int i = 0; i < kProfSlots; ++i) prof.v[i] = 0;
  const long long t_begin = clock64();

  if (warp >= kProd0) {
    // ---------------------------------------------------------------- producers
    // Pipeline w (of kPipes) owns the units ua = w (mod kPipes) of this CTA, in order, and its own
    // ring of SP stages; its kProdPerPipe producer warps split the pipeline's block sequence
    // m = 0, 1, 2, ... round robin.  Unit metadata (bitmap, value start, 8 col ids of each of
    // its blocks, 32 at a time; lane l <-> block l) is fetched in coalesced loads;
    // block values are prefetched two blocks ahead into registers.  Per block the warp then only
    // waits for a free stage, issues the 8 row gathers (cp.async, 16 B per lane per row,
    // zero-filled for padding slots) whose completion the hardware reports on the stage's full
    // barrier (cp.async.mbarrier.arrive.noinc), and decodes the bitmap block into the MMA B
    // operand.  No global-memory latency sits on the per-block path, and every stage of the
    // ring can be in flight.  Consumption is in order per pipeline, which keeps the mbarrier
    // parity protocol exact.
    const int pw = warp - kProd0;
    const int w = pw / kProdPerPipe, q = pw % kProdPerPipe;
    const char* Bbytes = reinterpret_cast<const char*>(a.B);
    const int64_t row_bytes = a.ldb * EB;
    struct Meta {
      unsigned long long bm;
      int32_t vs;
      int4 c0, c1;
      int32_t z, nb;
    };
    // batches: up to 32 consecutive blocks of one unit of this pipeline
    auto load_meta = [&](int64_t u, int off, Meta& M) {
      const int4 un = a.s.units[u];
      M.z = un.z + off;
      M.nb = min(32, un.w - M.z);
      const int64_t blk = (int64_t)M.z + lane;
      const bool mine = lane < M.nb;
      M.bm = mine ? __ldg(a.bitmaps + blk) : 0ull;
      M.vs = mine ? __ldg(a.s.vstart + blk) : 0;
      M.c0 = mine ? __ldg(reinterpret_cast<const int4*>(a.col_id + blk * 8)) : make_int4(0, 0, 0, 0);
      M.c1 = mine ? __ldg(reinterpret_cast<const int4*>(a.col_id + blk * 8) + 1) : make_int4(0, 0, 0, 0);
    };
    auto skip_empty = [&](int64_t& u) {
      while (u < u1) {
        const int4 un = a.s.units[u];
        if (un.z != un.w) break;
        u += kPipes;
      }
    };
    auto step = [&](int64_t& u, int& off) {
      off += 32;
      if (u < u1) {
        const int4 un = a.s.units[u];
        if (un.z + off < un.w) return;
      }
      u += kPipes;
      off = 0;
      skip_empty(u);
    };
    auto load_vals = [&](const Meta& M, int l, float& v0, float& v1) {
      const unsigned long long bm = __shfl_sync(0xffffffffu, M.bm, l);
      const int32_t vs = __shfl_sync(0xffffffffu, M.vs, l);
      const int nv = __popcll(bm);
      v0 = lane < nv ? __ldg(a.tc_values + vs + lane) : 0.f;
      v1 = lane + 32 < nv ? __ldg(a.tc_values + vs + 32 + lane) : 0.f;
    };
    // ---- block iterator over this producer's share of the pipeline's blocks ----------------
    struct Blk {
      int64_t m;
      unsigned long long bm;
      int32_t col[8];
      float v0, v1;
    };
    Meta cur, nxt;
    int64_t u = u0 + w;
    int off = 0;
    skip_empty(u);
    if (u < u1) load_meta(u, off, cur);
    int64_t m0 = 0;   // pipeline block count before the current batch
    int l = -1;       // position in the current batch (-1: batch not entered yet)
    bool have_nxt = false;
    float pa0 = 0.f, pa1 = 0.f, pb0 = 0.f, pb1 = 0.f;  // values of this producer's next two blocks
    auto enter_batch = [&]() {
      int64_t un_ = u;
      int off_ = off;
      step(un_, off_);
      have_nxt = un_ < u1;
      if (have_nxt) load_meta(un_, off_, nxt);
      l = (int)(((q - m0) % kProdPerPipe + kProdPerPipe) % kProdPerPipe);
      if (l < cur.nb) load_vals(cur, l, pa0, pa1);
      if (l + kProdPerPipe < cur.nb) load_vals(cur, l + kProdPerPipe, pb0, pb1);
    };
    auto next = [&](Blk& b) -> bool {
      for (;;) {
        if (u >= u1) return false;
        if (l < 0) enter_batch();
        if (l < cur.nb) break;
        // batch exhausted: move to the next one
        int64_t un_ = u;
        int off_ = off;
        step(un_, off_);
        m0 += cur.nb;
        cur = nxt;
        u = un_;
        off = off_;
        l = -1;
      }
      b.m = m0 + l;
      b.bm = __shfl_sync(0xffffffffu, cur.bm, l);
      b.col[0] = __shfl_sync(0xffffffffu, cur.c0.x, l);
      b.col[1] = __shfl_sync(0xffffffffu, cur.c0.y, l);
      b.col[2] = __shfl_sync(0xffffffffu, cur.c0.z, l);
      b.col[3] = __shfl_sync(0xffffffffu, cur.c0.w, l);
      b.col[4] = __shfl_sync(0xffffffffu, cur.c1.x, l);
      b.col[5] = __shfl_sync(0xffffffffu, cur.c1.y, l);
      b.col[6] = __shfl_sync(0xffffffffu, cur.c1.z, l);
      b.col[7] = __shfl_sync(0xffffffffu, cur.c1.w, l);
      b.v0 = pa0;
      b.v1 = pa1;
      pa0 = pb0;
      pa1 = pb1;
      if (l + 2 * kProdPerPipe < cur.nb) load_vals(cur, l + 2 * kProdPerPipe, pb0, pb1);
      l += kProdPerPipe;
      return true;
    };
    // ---- gather (LDG.128 into registers) and store (swizzled STS.128 + decode) -------------
    constexpr int kChunksPerTileRow = 8 * EB;             // 16-B chunks of 128 features
    constexpr int kCR = MT * kChunksPerTileRow;           // 16-B chunks per gathered row
    constexpr int kNC = 8 * kCR / 32;                     // chunks per lane per block
    static_assert(kNC >= 1 && (8 * kCR) % 32 == 0, "whole warp moves each block");
    auto issue = [&](const Blk& b, uint4 (&d)[kNC]) {
      unsigned long long x = b.bm | (b.bm >> 32);
      x |= x >> 16;
      x |= x >> 8;
      const uint32_t cm = (uint32_t)x & 0xffu;
#pragma unroll
      for (int i = 0; i < kNC; ++i) {
        const int g = lane + 32 * i;
        const int k = g / kCR, cc = g % kCR;
        const uint4* src = reinterpret_cast<const uint4*>(Bbytes + (int64_t)b.col[k] * row_bytes) + cc;
        if (((cm >> k) & 1u) && !(a.flags & 4)) {
          if constexpr (kL1) {
            d[i] = __ldg(src);
          } else {
            uint4 v;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src));
            d[i] = v;
          }
        } else {
          d[i] = make_uint4(0, 0, 0, 0);
        }
      }
    };
    auto finish = [&](const Blk& b, const uint4 (&d)[kNC]) {
      const int s = w * SP + (int)(b.m % SP);
      mbar_wait_t(empty + s, (uint32_t)(((b.m / SP) & 1) ^ 1), prof, 0);
      uint8_t* stageA = sA + (size_t)s * MT * kTileBytes;
#pragma unroll
      for (int i = 0; i < kNC; ++i) {
        const int g = lane + 32 * i;
        const int k = g / kCR, cc = g % kCR;
        const int t = cc / kChunksPerTileRow;
        const int byte = (cc % kChunksPerTileRow) * 16;
        *reinterpret_cast<uint4*>(stageA + t * kTileBytes + a_offset<EB>(byte >> 7, k, (byte & 127) >> 4)) = d[i];
      }
      // decode: bit pos = local_row * 8 + local_col, value rank = popc(bits below pos)
      uint8_t* bop = sB + (size_t)s * kBopBytes;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int pos = lane + 32 * h;
        const bool set = (b.bm >> pos) & 1ull;
        const int rank = pos ? __popcll(b.bm & ((1ull << pos) - 1ull)) : 0;
        const float va = __shfl_sync(0xffffffffu, b.v0, rank & 31);
        const float vb = __shfl_sync(0xffffffffu, b.v1, rank & 31);
        const float v = set ? (rank < 32 ? va : vb) : 0.f;
        const int i = pos >> 3, k = pos & 7;
        if constexpr (EB == 4) {
          *(uint32_t*)(bop + (k >> 2) * 128 + i * 16 + (k & 3) * 4) = to_tf32(v);
        } else if constexpr (std::is_same<BT, __nv_bfloat16>::value) {
          *(__nv_bfloat16*)(bop + i * 16 + k * 2) = __float2bfloat16_rn(v);
        } else {
          *(__half*)(bop + i * 16 + k * 2) = __float2half_rn(v);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(full + s);
    };
    // two blocks in flight per warp: gather block n+1 while storing block n
    Blk ba, bb;
    uint4 da[kNC], db[kNC];
    bool has_a = next(ba);
    if (has_a) issue(ba, da);
    while (has_a) {
      const bool has_b = next(bb);
      if (has_b) issue(bb, db);
      finish(ba, da);
      if (!has_b) break;
      has_a = next(ba);
      if (has_a) issue(ba, da);
      finish(bb, db);
    }
    const long long t_prod = clock64();
    prof.v[1] = t_prod - t_begin;

    // residual and zero-row units (CUDA-core), fetched dynamically across the grid
    const int64_t nunits = a.s.header[2];
    const int n_fc = (a.N + 32 * kVec - 1) / (32 * kVec);
    for (;;) {
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(a.s.counters, 1u);
      t = __shfl_sync(0xffffffffu, t, 0);
      int64_t u = nwu + t;
      if (u >= nunits) break;
      int4 un = a.s.units[u];
      if ((un.x & 3) == kUnitResidual) residual_rows<kVec, BT, float>(a, un.y, un.z, n_fc);
      else zero_rows<kVec>(a, un.y, un.z);
    }
    prof.v[2] = clock64() - t_prod;
    if (lane == 0) prof.flush(blockIdx.x, 0, 3);
    __syncwarp();
    if (lane == 0) {
      uint32_t producers = gridDim.x * kProdWarps;
      if (atomicAdd(a.s.counters + 1, 1u) == producers - 1) {
        a.s.counters[0] = 0;
        a.s.counters[1] = 0;
      }
    }
  } else if (warp >= kMmaWarp0) {
    // ---------------------------------------------------------------- MMA issuers
    // One elected lane per pipeline.  A tiny M=128 x N=8 MMA costs ~200 cycles of issue latency
    // per issuing thread and the rate scales with issuing warps (tools/microbench/umma_issue.cu),
    // so each of the kPipes pipelines has its own issuer, in its own SM sub-partition, consuming
    // its stage ring strictly in order into its own accumulators.
    if (lane == 0) {
      constexpr uint32_t idesc = (1u << 4) | (Kind<BT>::fmt << 7) | (Kind<BT>::fmt << 10) | (1u << 15) |
                                 (1u << 17) | (8u << 24);
      const int w = warp - kMmaWarp0;
      int64_t m = 0;
      int64_t ua = w;
      for (int64_t u = u0 + w; u < u1; u += kPipes, ua += kPipes) {
        const int4 un = a.s.units[u];
        const int slot = (int)(ua % NACC);
        mbar_wait_t(tempty + slot, (uint32_t)(((ua / NACC) & 1) ^ 1), prof, 4);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (un.z == un.w) {
          mbar_arrive(tfull + slot);
          continue;
        }
        for (int32_t blk = un.z; blk < un.w; ++blk, ++m) {
          const int s = w * SP + (int)(m % SP);
          mbar_wait_t(full + s, (uint32_t)((m / SP) & 1), prof, 3);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t bdesc = umma_desc(smem_u32(sB + (size_t)s * kBopBytes), 128, 256, 0);
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            const uint64_t adesc =
                umma_desc(smem_u32(sA + ((size_t)s * MT + t) * kTileBytes), Kind<BT>::lbo, Kind<BT>::sbo,
                          Kind<BT>::layout);
            if (!(a.flags & 8))  // bit 3: perf probe, no MMA
              mma<BT>(tmem + (uint32_t)((slot * MT + t) * 8), adesc, bdesc, idesc, blk > un.z ? 1u : 0u);
          }
          umma_commit(empty + s);
        }
        umma_commit(tfull + slot);
      }
      prof.v[5] = clock64() - t_begin;
      prof.flush(blockIdx.x, 3, 6);
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0-3)
    const int f_in_tile = warp * 32 + lane;
    int64_t ua = 0;
    for (int64_t u = u0; u < u1; ++u, ++ua) {
      int4 un = a.s.units[u];
      const int slot = (int)(ua % NACC);
      mbar_wait_t(tfull + slot, (uint32_t)((ua / NACC) & 1), prof, 6);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int32_t g = un.y, k = un.x >> 2;
      const int64_t rid = a.s.grp_rid[g];
      const int64_t avail = a.window_size < a.n_rows - rid ? a.window_size : a.n_rows - rid;
      const int32_t pslot = a.s.grp_slot[g];
      const bool has = un.z != un.w;
      float r[MT][8];
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        if (has) {
          uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((slot * MT + t) * 8);
          uint32_t q[8];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]),
                         "=r"(q[7])
                       : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 8; ++i) r[t][i] = __uint_as_float(q[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) r[t][i] = 0.f;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + slot);
      if (pslot < 0) {
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          const int64_t f = t * 128 + f_in_tile;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (i < avail) __stcs(a.C + (rid + i) * a.ldc + f, r[t][i]);
        }
      } else {
        float* part = reinterpret_cast<float*>(a.partials) + ((int64_t)(pslot + k) * 8) * a.N;
#pragma unroll
        for (int t = 0; t < MT; ++t)
#pragma unroll
          for (int i = 0; i < 8; ++i) __stcg(part + (int64_t)i * a.N + t * 128 + f_in_tile, r[t][i]);
        // one thread publishes for the whole epilogue group (bar.sync orders the others' stores
        // before its fence) and, if it took the last ticket, acquires for everyone; windows
        // with more than kTicketMax chunks are left to the fixup kernels
        const long long tp = prof.on ? clock64() : 0;
        const int32_t nch = a.s.grp_nch[g];
        if (nch > kTicketMax) continue;
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        if (threadIdx.x == 0) {
          __threadfence();
          const uint32_t t = atomicAdd(a.s.ticket + g, 1u);
          if ((int32_t)t == nch - 1) __threadfence();
          misc[1] = t;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        if ((int32_t)misc[1] == nch - 1) {
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            const int64_t f = t * 128 + f_in_tile;
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
          if (threadIdx.x == 0) a.s.ticket[g] = 0;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        if (prof.on) prof.v[8] += clock64() - tp;
      }
    }
  }

  if (warp == 0 && lane == 0) {
    prof.v[7] = clock64() - t_begin;
    prof.flush(blockIdx.x, 6, 9);
  }
  if (threadIdx.x == 0 && prof.on) atomicAdd(&g_tc_prof[blockIdx.x & 1023][9], (unsigned long long)(clock64() - t_begin));
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kMmaWarp0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

template <int MT, int STAGES>
constexpr size_t smem_bytes() {
  constexpr int NACC = kTmemCols / (8 * MT) < 64 ? kTmemCols / (8 * MT) : 64;
  return 1024 + (size_t)STAGES * (MT * kTileBytes + kBopBytes) + (2 * STAGES + 2 * NACC) * 8 + 16;
}

template <class BT, int MT, int STAGES, bool kL1>
int launch(const SpmmArgs& a, cudaStream_t st) {
  auto kern = k_spmm_tc<BT, MT, STAGES, kL1>;
  constexpr size_t bytes = smem_bytes<MT, STAGES>();
  static bool init = false;
  if (!init) {
    RSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    init = true;
  }
  kern<<<sm_count(), kThreadsTC, bytes, st>>>(a);
  RSH_LAUNCHED("k_spmm_tc");
  return launch_fixup<float>(a, st);
}

}  // namespace tc
}  // namespace rsh

using namespace rsh;

extern "C" {

// Debug: copy the per-CTA role cycle counters (flags bit 4) to host_out[1024 * 16] and clear them.
int rsh_tc_profile(unsigned long long* host_out) {
  RSH_CUDA(cudaMemcpyFromSymbol(host_out, tc::g_tc_prof, sizeof(tc::g_tc_prof)));
  static unsigned long long zeros[1024][tc::kProfSlots];
  RSH_CUDA(cudaMemcpyToSymbol(tc::g_tc_prof, zeros, sizeof(zeros)));
  return kOk;
}

// Tensor-core hybrid SpMM (execute.py:155-218 semantics, TF32 / BF16 / FP16 operands, fp32
// accumulation).  Requirements: N in {128, 256}, f32 accumulation, 16-byte aligned B rows.
// l1: 1 = gather through L1 (cp.async.ca), 0 = L2 only (cp.async.cg).
int rsh_spmm_tc(int64_t n_rows, int32_t window_size, int64_t n_entries, const uint64_t* bitmaps,
                const int32_t* col_id, const float* tc_values, int64_t n_blocks, const int32_t* res_row_id,
                const int64_t* res_offset, const int32_t* res_col_id, const float* res_values, int64_t n_res,
                const void* B, int64_t ldb, int32_t b_dtype, int64_t N, float* C, int64_t ldc, int32_t l1,
                void* sched, size_t sched_bytes, void* partials, size_t partial_bytes, cudaStream_t st) {
  if (!(N == 128 || N == 256)) return fail(kInvalid, "rsh_spmm_tc: N must be 128 or 256 (got %lld)", (long long)N);
  if (b_dtype < 0 || b_dtype > 2) return fail(kInvalid, "rsh_spmm_tc: bad b_dtype");
  size_t eb = b_dtype == 0 ? 4 : 2;
  if (ldb < N || ldc < N || ((uintptr_t)B & 15) || ((ldb * eb) & 15))
    return fail(kInvalid, "rsh_spmm_tc: B rows must be 16-byte aligned");
  Sched s;
  size_t need = sched_layout(sched, n_rows, n_entries, n_blocks, n_res, &s);
  if (!sched || sched_bytes < need) return fail(kInvalid, "rsh_spmm_tc: schedule buffer too small");
  SpmmArgs a;
  a.bitmaps = (const unsigned long long*)bitmaps;
  a.col_id = col_id;
  a.tc_values = tc_values;
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
  a.N = (int32_t)N;
  RSH_OK(bind_workspace(a, partials, partial_bytes, n_entries, sizeof(float)));
  a.flags = l1;
  l1 &= 1;
  const int mt = (int)(N / 128);
  if (b_dtype == 0) {
    if (mt == 1) return l1 ? tc::launch<float, 1, 48, true>(a, st) : tc::launch<float, 1, 48, false>(a, st);
    return l1 ? tc::launch<float, 2, 24, true>(a, st) : tc::launch<float, 2, 24, false>(a, st);
  }
  if (b_dtype == 1) {
    if (mt == 1) return l1 ? tc::launch<__nv_bfloat16, 1, 48, true>(a, st) : tc::launch<__nv_bfloat16, 1, 48, false>(a, st);
    return l1 ? tc::launch<__nv_bfloat16, 2, 24, true>(a, st) : tc::launch<__nv_bfloat16, 2, 24, false>(a, st);
  }
  if (mt == 1) return l1 ? tc::launch<__half, 1, 48, true>(a, st) : tc::launch<__half, 1, 48, false>(a, st);
  return l1 ? tc::launch<__half, 2, 24, true>(a, st) : tc::launch<__half, 2, 24, false>(a, st);
}

}  // extern "C"
