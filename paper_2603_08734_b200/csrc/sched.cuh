// Work-unit schedule shared by the CUDA-core (spmm_cc.cu) and tensor-core (spmm_tc.cu) SpMM
// kernels, plus the per-lane vector helpers and the warp-level residual / zero-row bodies.
#pragma once
#include "common.cuh"
#include <cub/cub.cuh>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace rsh {

constexpr int kChunkMin = 32;   // smallest blocks-per-unit a schedule may use (sizes buffers)
constexpr int kChunkMax = 1023; // largest: a unit's per-row totals (<= 8 x chunk) fit 16 bits
constexpr int kChunkCC = 32;    // CUDA-core path: one warp walks a unit serially
constexpr int kChunkTC = 256;   // tensor-core path: a unit stays in one TMEM accumulator
constexpr int kTicketMax = 256; // windows with more chunks are reduced by the fixup kernels
constexpr int kFixSeg = 32;     // chunks per first-level fixup segment
constexpr int kResRows = 16;    // residual rows per unit
constexpr int kZeroRows = 32;   // uncovered rows per unit

enum UnitType { kUnitWindow = 0, kUnitResidual = 1, kUnitZero = 2 };

// header: int64 [0]=groups [1]=window units [2]=all units [3]=partial slots [4]=uncovered rows
//         [5]=blocks per window unit (the fixed chunking) [6]=windows reduced by the fixup
//         kernels (more than kTicketMax chunks) [7]=their first-level fix-up segments
//         [8]=device address of the row-major window list (rsh_schedule_rowmajor), [9]=its tc nnz
//         (0 = no list), [11]=device address of its unit headers (k_unit_headers, 3 x int4 per unit)
// counters: uint32 [0]=next unit [1]=warps done
struct Sched {
  int64_t* header;
  int64_t* unit_cost;  // exclusive prefix of window-unit cost (blocks + 1), [max_units + 1]
  int64_t* unit_cost_raw;
  uint32_t* counters;
  int32_t *head, *grp_rid, *grp_b0, *grp_b1, *grp_nch, *grp_multi, *grp_slot, *unit_base, *slot_base, *big;
  int32_t* seg_base;  // exclusive prefix of fix-up segments over the big windows
  uint32_t* ticket;
  int32_t* vstart;
  uint8_t* flags;
  int32_t* pc;
  uint8_t* uncov_flag;
  int32_t* uncovered;
  int4* units;
  void* cub;
  size_t cub_bytes;
  int64_t max_units;
};

inline size_t sched_layout(void* base, int64_t n_rows, int64_t n_entries, int64_t n_blocks, int64_t n_res, Sched* s) {
  Carve cv(base);
  int64_t E = n_entries;
  s->header = cv.take<int64_t>(16);
  s->counters = cv.take<uint32_t>(4);
  s->head = cv.take<int32_t>(E + 1);
  s->grp_rid = cv.take<int32_t>(E + 1);
  s->grp_b0 = cv.take<int32_t>(E + 1);
  s->grp_b1 = cv.take<int32_t>(E + 1);
  s->grp_nch = cv.take<int32_t>(E + 1);
  s->grp_multi = cv.take<int32_t>(E + 1);
  s->big = cv.take<int32_t>(E + 1);
  s->seg_base = cv.take<int32_t>(E + 2);
  s->grp_slot = cv.take<int32_t>(E + 1);
  s->unit_base = cv.take<int32_t>(E + 1);
  s->slot_base = cv.take<int32_t>(E + 1);
  s->ticket = cv.take<uint32_t>(E + 1);
  s->vstart = cv.take<int32_t>(n_blocks + 1);
  int64_t big = n_rows > E ? n_rows : E;
  big = big > n_blocks ? big : n_blocks;
  s->flags = cv.take<uint8_t>(big + 1);
  s->pc = cv.take<int32_t>(n_blocks + 1);
  s->uncov_flag = cv.take<uint8_t>(n_rows + 1);
  s->uncovered = cv.take<int32_t>(n_rows + 1);
  s->max_units = E + n_blocks / kChunkMin + 1 + (n_res + kResRows - 1) / kResRows + (n_rows + kZeroRows - 1) / kZeroRows + 4;
  s->units = cv.take<int4>(s->max_units);
  s->unit_cost = cv.take<int64_t>(s->max_units + 1);
  s->unit_cost_raw = cv.take<int64_t>(s->max_units + 1);
  size_t a = 0, b = 0;
  cub::DeviceSelect::Flagged(nullptr, a, cub::CountingInputIterator<int32_t>(0), (uint8_t*)nullptr, (int32_t*)nullptr,
                             (int64_t*)nullptr, (int)(big + 1));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr, (int)(big + 1));
  size_t c2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, c2, (int64_t*)nullptr, (int64_t*)nullptr, (int)(s->max_units + 1));
  b = b > c2 ? b : c2;
  s->cub_bytes = a > b ? a : b;
  s->cub = cv.take<char>(s->cub_bytes);
  return cv.used + 256;
}

// ------------------------------------------------------------------------------------------
// vector load / store helpers (VEC consecutive features per lane)
// ------------------------------------------------------------------------------------------

template <class BT>
__device__ __forceinline__ float to_f(BT x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <>
__device__ __forceinline__ float to_f<__half>(__half x) { return __half2float(x); }

template <int VEC, class BT>
__device__ __forceinline__ void load_vec(const BT* __restrict__ p, float (&o)[VEC]) {
  constexpr int bytes = VEC * (int)sizeof(BT);
  if constexpr (bytes % 16 == 0) {
#pragma unroll
    for (int q = 0; q < bytes / 16; ++q) {
      uint4 u = __ldg(reinterpret_cast<const uint4*>(p) + q);
      const BT* e = reinterpret_cast<const BT*>(&u);
#pragma unroll
      for (int t = 0; t < 16 / (int)sizeof(BT); ++t) o[q * (16 / sizeof(BT)) + t] = to_f<BT>(e[t]);
    }
  } else if constexpr (bytes == 8) {
    uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    const BT* e = reinterpret_cast<const BT*>(&u);
#pragma unroll
    for (int t = 0; t < VEC; ++t) o[t] = to_f<BT>(e[t]);
  } else if constexpr (bytes == 4) {
    uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(p));
    const BT* e = reinterpret_cast<const BT*>(&u);
#pragma unroll
    for (int t = 0; t < VEC; ++t) o[t] = to_f<BT>(e[t]);
  } else {
#pragma unroll
    for (int t = 0; t < VEC; ++t) o[t] = to_f<BT>(p[t]);
  }
}

// L2 cache policies: B rows are the reused operand (evict_last), the format stream is read once
// (evict_first)
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg_hint(const void* p, uint64_t pol) {
  uint4 u;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p), "l"(pol));
  return u;
}
__device__ __forceinline__ uint32_t ldg_hint32(const void* p, uint64_t pol) {
  uint32_t u;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(u) : "l"(p), "l"(pol));
  return u;
}
__device__ __forceinline__ unsigned long long ldg_hint64(const void* p, uint64_t pol) {
  unsigned long long u;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(u) : "l"(p), "l"(pol));
  return u;
}

__device__ __forceinline__ int4 make_int4_u(uint4 u) { return make_int4((int)u.x, (int)u.y, (int)u.z, (int)u.w); }

// load_vec with an L2 policy (16-byte multiples; other widths fall back to load_vec)
template <int VEC, class BT>
__device__ __forceinline__ void load_vec_pol(const BT* __restrict__ p, float (&o)[VEC], uint64_t pol) {
  constexpr int bytes = VEC * (int)sizeof(BT);
  if constexpr (bytes % 16 == 0) {
#pragma unroll
    for (int q = 0; q < bytes / 16; ++q) {
      uint4 u = ldg_hint(reinterpret_cast<const uint4*>(p) + q, pol);
      const BT* e = reinterpret_cast<const BT*>(&u);
#pragma unroll
      for (int t = 0; t < 16 / (int)sizeof(BT); ++t) o[q * (16 / sizeof(BT)) + t] = to_f<BT>(e[t]);
    }
  } else {
    load_vec<VEC, BT>(p, o);
  }
}

template <int VEC, class AccT>
__device__ __forceinline__ void store_c(float* __restrict__ p, const AccT (&a)[VEC]) {
  if constexpr (VEC % 4 == 0) {
#pragma unroll
    for (int q = 0; q < VEC / 4; ++q)
      __stcs(reinterpret_cast<float4*>(p) + q, make_float4((float)a[4 * q], (float)a[4 * q + 1], (float)a[4 * q + 2],
                                                           (float)a[4 * q + 3]));
  } else if constexpr (VEC == 2) {
    __stcs(reinterpret_cast<float2*>(p), make_float2((float)a[0], (float)a[1]));
  } else {
#pragma unroll
    for (int t = 0; t < VEC; ++t) __stcs(p + t, (float)a[t]);
  }
}

struct SpmmArgs {
  const unsigned long long* bitmaps;
  const int32_t* col_id;
  const float* tc_values;
  const int32_t* res_row;
  const int64_t* res_off;
  const int32_t* res_col;
  const float* res_val;
  const void* B;
  int64_t ldb;
  float* C;
  int64_t ldc;
  int64_t n_rows;
  int32_t N;
  int32_t window_size;
  Sched s;
  void* partials;
  int64_t part_slots;  // 8-row partial slots the caller's workspace holds
  int32_t flags;  // tensor-core path knobs (bit 1: skip the consumer-side proxy fence)
};

// Per-launch mutable state lives in the CALLER's workspace, not in the schedule, so one schedule
// can serve concurrent launches (one workspace each): uint32 [0] next unit, [1] warps done,
// [2..3] unused, [4 .. 4 + n_entries] per-window tickets, then the chunk partials (256-B
// aligned).  The caller zero-fills a workspace once; every launch leaves the control words zero.
inline size_t spmm_ctl_bytes(int64_t n_entries) { return ((size_t)(4 + n_entries + 1) * 4 + 255) & ~size_t(255); }

inline int bind_workspace(SpmmArgs& a, void* ws, size_t ws_bytes, int64_t n_entries, size_t acc_bytes) {
  const size_t ctl = spmm_ctl_bytes(n_entries);
  if (!ws || ((uintptr_t)ws & 15) || ws_bytes < ctl)
    return fail(kInvalid, "rsh_spmm: workspace (%zu bytes) smaller than its control block (%zu); size it with "
                          "rsh_partials_bytes", ws_bytes, ctl);
  a.s.counters = reinterpret_cast<uint32_t*>(ws);
  a.s.ticket = reinterpret_cast<uint32_t*>(ws) + 4;
  a.partials = reinterpret_cast<char*>(ws) + ctl;
  a.part_slots = (int64_t)((ws_bytes - ctl) / (8 * (size_t)a.N * acc_bytes));
  return kOk;
}

// every SpMM kernel checks, once per CTA, that the workspace holds the schedule's partial slots
// (header[3]); a short workspace is a caller bug and fails the launch instead of writing past it
__device__ __forceinline__ void check_workspace(const SpmmArgs& a) {
  if (threadIdx.x == 0 && a.s.header[3] > a.part_slots) __trap();
}


// One residual row set [i0, i1) (execute.py:184-193): lane owns VEC consecutive features,
// entries are broadcast 32 at a time, B rows read with 128-bit loads, C row stored once.
template <int VEC, class BT, class AccT>
__device__ __forceinline__ void residual_rows(const SpmmArgs& a, int32_t i0, int32_t i1, int n_fc) {
  const int lane = threadIdx.x & 31;
  const BT* B = reinterpret_cast<const BT*>(a.B);
  for (int32_t i = i0; i < i1; ++i) {
    int64_t r = a.res_row[i];
    int64_t s0 = a.res_off[i], s1 = a.res_off[i + 1];
    for (int fc = 0; fc < n_fc; ++fc) {
      int f0 = fc * 32 * VEC + lane * VEC;
      bool active = f0 < a.N;
      AccT acc[VEC];
#pragma unroll
      for (int t = 0; t < VEC; ++t) acc[t] = AccT(0);
      for (int64_t base = s0; base < s1; base += 32) {
        int64_t p = base + lane;
        int32_t cr = p < s1 ? __ldg(a.res_col + p) : 0;
        float vr = p < s1 ? __ldg(a.res_val + p) : 0.f;
        int cnt = s1 - base < 32 ? int(s1 - base) : 32;
        for (int q = 0; q < cnt; ++q) {
          int32_t c = __shfl_sync(0xffffffffu, cr, q);
          AccT v = AccT(__shfl_sync(0xffffffffu, vr, q));
          if (active) {
            float bv[VEC];
            load_vec<VEC, BT>(B + (int64_t)c * a.ldb + f0, bv);
#pragma unroll
            for (int t = 0; t < VEC; ++t) acc[t] = fma(v, AccT(bv[t]), acc[t]);
          }
        }
      }
      if (active) store_c<VEC, AccT>(a.C + r * a.ldc + f0, acc);
    }
  }
}

// Uncovered rows uncovered[j0, j1) are written as zeros (execute.py:163), exactly once.
template <int VEC>
__device__ __forceinline__ void zero_rows(const SpmmArgs& a, int32_t j0, int32_t j1) {
  const int lane = threadIdx.x & 31;
  for (int32_t j = j0; j < j1; ++j) {
    int64_t r = a.s.uncovered[j];
    for (int f = lane * VEC; f < a.N; f += 32 * VEC) {
      float z[VEC];
#pragma unroll
      for (int t = 0; t < VEC; ++t) z[t] = 0.f;
      store_c<VEC, float>(a.C + r * a.ldc + f, z);
    }
  }
}

}  // namespace rsh
