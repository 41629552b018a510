// Hybrid RS-Tile SpMM: persistent work-unit scheduler + CUDA-core window/residual/zero paths
// (north-star subsystems (3) and (4); the tensor-core window path lives in spmm_tc.cu).
//
// Reference executor: execute.py:155-226 (hybrid_spmm).  Semantics kept:
//   * C is written exactly once per row: window rows [rid, rid + min(window_size, n - rid))
//     are ASSIGNED (execute.py:181-182), residual rows are ASSIGNED (execute.py:191-193), every
//     other row is zero (execute.py:163) -- zero rows are their own work units, so C is never
//     memset and then overwritten.
//   * consecutive entries sharing a row_window_id form one logical window whose block
//     sequence is independent of how it was split (execute.py:136-152).  Here a logical window
//     is cut at FIXED block offsets (the schedule's chunk) from its first block; chunk partials are
//     summed in chunk order by whichever warp finishes last (atomic ticket), so the result is
//     bit-identical for every max_blocks_per_item and every scheduling order.
//   * accumulate_precision f32 / f64 (execute.py:33-49): AccT = float / double.
#include "sched.cuh"
#include <cstdlib>

namespace rsh {

// ------------------------------------------------------------------------------------------
// schedule construction
// ------------------------------------------------------------------------------------------

__global__ void k_group_heads(const int32_t* __restrict__ rwid, int64_t E, uint8_t* flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    flag[e] = (e == 0 || rwid[e] != rwid[e - 1]);
}

__global__ void k_groups(const int32_t* __restrict__ rwid, const int64_t* __restrict__ rwoff, int64_t E, Sched s,
                         int32_t chunk) {
  int64_t G = s.header[0];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g <= E; g += (int64_t)gridDim.x * blockDim.x) {
    int32_t nch = 0, multi = 0;
    if (g < G) {
      int64_t e0 = s.head[g], e1 = g + 1 < G ? s.head[g + 1] : E;
      int64_t b0 = rwoff[e0], b1 = rwoff[e1];
      s.grp_rid[g] = rwid[e0];
      s.grp_b0[g] = (int32_t)b0;
      s.grp_b1[g] = (int32_t)b1;
      int64_t c = (b1 - b0 + chunk - 1) / chunk;
      nch = (int32_t)(c > 1 ? c : 1);
      multi = nch > 1 ? nch : 0;
      s.grp_nch[g] = nch;
      s.ticket[g] = 0;
    }
    s.grp_multi[g] = multi;
    s.unit_base[g] = nch;  // scanned in place afterwards (copied through cub)
  }
}

__global__ void k_window_units(int64_t E, Sched s, int32_t chunk) {
  int64_t G = s.header[0];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
    int32_t nch = s.grp_nch[g], b0 = s.grp_b0[g], b1 = s.grp_b1[g];
    int32_t base = s.unit_base[g];
    s.grp_slot[g] = nch > 1 ? s.slot_base[g] : -1;
    for (int32_t k = 0; k < nch; ++k) {
      int32_t lo = b0 + k * chunk, hi = lo + chunk < b1 ? lo + chunk : b1;
      s.units[base + k] = make_int4(kUnitWindow | (k << 2), (int32_t)g, lo, hi);
      s.unit_cost_raw[base + k] = (hi - lo) + 1;  // blocks gathered + one window of C rows
    }
  }
}

__global__ void k_big_flags(Sched s, int64_t E) {
  int64_t G = s.header[0];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g <= E; g += (int64_t)gridDim.x * blockDim.x)
    s.flags[g] = g < G && s.grp_nch[g] > kTicketMax;
}

// first-level fix-up segments of the big windows (few windows: one thread)
__global__ void k_seg_base(Sched s) {
  const int64_t nbig = s.header[6];
  int32_t acc = 0;
  for (int64_t i = 0; i < nbig; ++i) {
    s.seg_base[i] = acc;
    acc += (s.grp_nch[s.big[i]] + kFixSeg - 1) / kFixSeg;
  }
  s.seg_base[nbig] = acc;
  s.header[7] = acc;
}

__global__ void k_uncover(Sched s, int64_t n_rows, int window_size, const int32_t* __restrict__ res_row, int64_t n_res) {
  int64_t G = s.header[0];
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = tid; g < G; g += stride) {
    int64_t rid = s.grp_rid[g];
    int64_t avail = window_size < n_rows - rid ? window_size : n_rows - rid;
    for (int64_t i = 0; i < avail; ++i) s.uncov_flag[rid + i] = 0;
  }
  for (int64_t i = tid; i < n_res; i += stride) s.uncov_flag[res_row[i]] = 0;
}

__global__ void k_popc32(const unsigned long long* __restrict__ bm, int64_t nb, int32_t* pc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nb; i += (int64_t)gridDim.x * blockDim.x)
    pc[i] = i < nb ? __popcll(bm[i]) : 0;
}

__global__ void k_popc_total(const unsigned long long* __restrict__ bm, int64_t nb, unsigned long long* tot) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.x * blockDim.x)
    s += __popcll(bm[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(tot, s);
}

__global__ void k_finish_header(Sched s, int64_t E, int64_t n_res, int32_t chunk) {
  int64_t uw = s.unit_base[E];
  int64_t ru = (n_res + kResRows - 1) / kResRows;
  int64_t z = s.header[4];
  int64_t zu = (z + kZeroRows - 1) / kZeroRows;
  s.header[1] = uw;
  s.header[2] = uw + ru + zu;
  s.header[3] = s.slot_base[E];
  s.header[5] = chunk;
  s.counters[0] = 0;
  s.counters[1] = 0;
}

__global__ void k_tail_units(Sched s, int64_t n_res) {
  int64_t uw = s.header[1], z = s.header[4];
  int64_t ru = (n_res + kResRows - 1) / kResRows, zu = (z + kZeroRows - 1) / kZeroRows;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ru + zu; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < ru) {
      int64_t lo = i * kResRows, hi = lo + kResRows < n_res ? lo + kResRows : n_res;
      s.units[uw + i] = make_int4(kUnitResidual, (int32_t)lo, (int32_t)hi, 0);
    } else {
      int64_t j = i - ru;
      int64_t lo = j * kZeroRows, hi = lo + kZeroRows < z ? lo + kZeroRows : z;
      s.units[uw + i] = make_int4(kUnitZero, (int32_t)lo, (int32_t)hi, 0);
    }
  }
}

// ------------------------------------------------------------------------------------------
// the persistent CUDA-core kernel: one warp per work unit, units fetched dynamically
// ------------------------------------------------------------------------------------------

template <int VEC, class BT, class AccT>
__device__ __forceinline__ void window_chunk(const SpmmArgs& a, int32_t b0, int32_t b1, int f0, bool active,
                                             AccT (&acc)[8][VEC]) {
  const int lane = threadIdx.x & 31;
  const BT* B = reinterpret_cast<const BT*>(a.B);
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int t = 0; t < VEC; ++t) acc[i][t] = AccT(0);
  int32_t vp = a.s.vstart[b0];
  for (int32_t blk = b0; blk < b1; ++blk) {
    unsigned long long bm = __ldg(a.bitmaps + blk);
    int32_t colreg = lane < 8 ? __ldg(a.col_id + (int64_t)blk * 8 + lane) : 0;
    int nv = __popcll(bm);
    float v0 = lane < nv ? __ldg(a.tc_values + vp + lane) : 0.f;
    float v1 = lane + 32 < nv ? __ldg(a.tc_values + vp + 32 + lane) : 0.f;
    int kk = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t rb = uint32_t(bm >> (8 * i)) & 0xffu;
      while (rb) {
        int j = __ffs(rb) - 1;
        rb &= rb - 1;
        int32_t c = __shfl_sync(0xffffffffu, colreg, j);
        float va = __shfl_sync(0xffffffffu, v0, kk & 31);
        float vb = __shfl_sync(0xffffffffu, v1, kk & 31);
        AccT v = AccT(kk < 32 ? va : vb);
        ++kk;
        if (active) {
          float bv[VEC];
          load_vec<VEC, BT>(B + (int64_t)c * a.ldb + f0, bv);
#pragma unroll
          for (int t = 0; t < VEC; ++t) acc[i][t] = fma(v, AccT(bv[t]), acc[i][t]);
        }
      }
    }
    vp += nv;
  }
}

constexpr int kListCap = 384;  // (col, value) entries per warp list

// Stream list[beg, end) of one window row: kPF B-row gathers in flight before their FMAs.
// Stream list[beg, end) of one window row with kPF B-row gathers in flight before their FMAs.
// G > 1 (narrow rows, N = 128 / G fp32 features): the warp splits into G lane groups that take
// alternate entries with full 16-byte loads, and the G partial sums are combined by a fixed
// xor-shuffle tree at the end (deterministic).
template <int VEC, class BT, int kPF, int G>
__device__ __forceinline__ void row_from_list(const SpmmArgs& a, const int2* list, int beg, int end, int f0, bool active,
                                              float (&acc)[VEC], uint64_t pol) {
  const BT* B = reinterpret_cast<const BT*>(a.B);
  const int grp = G > 1 ? (int)(threadIdx.x & 31) / (32 / G) : 0;
#pragma unroll
  for (int t = 0; t < VEC; ++t) acc[t] = 0.f;
  int e0 = beg;
  for (; e0 + kPF * G <= end; e0 += kPF * G) {
    float bv[kPF][VEC];
    float vv[kPF];
#pragma unroll
    for (int p = 0; p < kPF; ++p) {
      const int2 cv = list[e0 + p * G + grp];
      vv[p] = __int_as_float(cv.y);
      if (active) load_vec_pol<VEC, BT>(B + (int64_t)cv.x * a.ldb + f0, bv[p], pol);
    }
    if (active) {
#pragma unroll
      for (int p = 0; p < kPF; ++p)
#pragma unroll
        for (int t = 0; t < VEC; ++t) acc[t] = fmaf(vv[p], bv[p][t], acc[t]);
    }
  }
  for (int e = e0 + grp; e < end; e += G) {
    const int2 cv = list[e];
    if (active) {
      float bv[VEC];
      load_vec_pol<VEC, BT>(B + (int64_t)cv.x * a.ldb + f0, bv, pol);
#pragma unroll
      for (int t = 0; t < VEC; ++t) acc[t] = fmaf(__int_as_float(cv.y), bv[t], acc[t]);
    }
  }
  if constexpr (G > 1) {
#pragma unroll
    for (int off = 16; off >= 32 / G; off >>= 1)
#pragma unroll
      for (int t = 0; t < VEC; ++t) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], off);
  }
}

// fp32 window unit, walked ROW by row.  The unit's (<= 32) blocks are listed once as (col,
// value) pairs in shared memory, grouped by window row -- lane l owns block l; packed warp scans
// of the per-row popcounts place every entry, and each lane only visits its set bits -- then
// each row streams its segment with kPF gathers in flight.  One accumulator row (VEC registers)
// instead of eight leaves the registers for gathers in flight; the accumulation order (blocks in
// order, columns in order within a block) is the block walk's.  Units with more than kListCap
// nonzeros are listed one row at a time.
template <int VEC, class BT, int kPF, int G>
__device__ __forceinline__ void window_rows(const SpmmArgs& a, int4 un, int64_t rid, int64_t avail, int32_t slot,
                                            int32_t k, int n_fc, int2* list, int* tab) {
  const int lane = threadIdx.x & 31;
  const int32_t b0 = un.z, b1 = un.w;
  if (b1 - b0 > 32) __trap();  // the row walk lists at most one block per lane
  const int32_t blk = b0 + lane;
  const bool mine = blk < b1;
  // L2 policy: B rows evict_last (reused across windows), the format stream evict_first
  const bool hints = !(a.flags & 4);
  const uint64_t pol_b = hints ? policy_evict_last() : 0, pol_a = hints ? policy_evict_first() : 0;
  const unsigned long long bm = mine ? (hints ? ldg_hint64(a.bitmaps + blk, pol_a) : __ldg(a.bitmaps + blk)) : 0ull;
  const int32_t vs = mine ? __ldg(a.s.vstart + blk) : 0;
  const int nrows = slot < 0 ? (int)avail : 8;
  auto meta_col = [&](int j) -> int32_t {
    const int32_t* p = a.col_id + (int64_t)blk * 8 + j;
    return hints ? (int32_t)ldg_hint32(p, pol_a) : __ldg(p);
  };
  auto meta_val = [&](int r) -> int32_t {
    const float* p = a.tc_values + vs + r;
    return hints ? (int32_t)ldg_hint32(p, pol_a) : __float_as_int(__ldg(p));
  };
  // per-row counts of this lane's block, packed 4 rows x 16 bits per word
  unsigned long long p0 = 0, p1 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    p0 |= (unsigned long long)__popc(uint32_t(bm >> (8 * i)) & 0xffu) << (16 * i);
    p1 |= (unsigned long long)__popc(uint32_t(bm >> (8 * (i + 4))) & 0xffu) << (16 * i);
  }
  unsigned long long q0 = p0, q1 = p1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t0 = __shfl_up_sync(0xffffffffu, q0, o);
    const unsigned long long t1 = __shfl_up_sync(0xffffffffu, q1, o);
    if (lane >= o) {
      q0 += t0;
      q1 += t1;
    }
  }
  const unsigned long long tot0 = __shfl_sync(0xffffffffu, q0, 31), tot1 = __shfl_sync(0xffffffffu, q1, 31);
  // inclusive prefix over rows of the row totals (fields never overflow 16 bits)
  const unsigned long long rp0 = tot0 * 0x0001000100010001ull;
  const unsigned long long rp1 = tot1 * 0x0001000100010001ull + (rp0 >> 48) * 0x0001000100010001ull;
  const int total = (int)(rp1 >> 48);
  auto row_end = [&](int i) -> int {
    return (int)(((i < 4 ? rp0 : rp1) >> (16 * (i & 3))) & 0xffffull);
  };
  if (total <= kListCap) {
    const unsigned long long e0 = q0 - p0, e1 = q1 - p1;  // exclusive lane prefixes
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row_beg = i ? row_end(i - 1) : 0;
      const int lane_off = (int)(((i < 4 ? e0 : e1) >> (16 * (i & 3))) & 0xffffull);
      tab[lane * 8 + i] = row_beg + lane_off;
    }
    __syncwarp();
    unsigned long long rem = bm;
    int vrank = 0;
    while (rem) {
      const int bit = __ffsll((long long)rem) - 1;
      rem &= rem - 1;
      const int i = bit >> 3, j = bit & 7;
      const uint32_t byte = uint32_t(bm >> (8 * i)) & 0xffu;
      const int pos = tab[lane * 8 + i] + __popc(byte & ((1u << j) - 1u));
      list[pos] = make_int2(meta_col(j), meta_val(vrank));
      ++vrank;
    }
    __syncwarp();
    for (int i = 0; i < nrows; ++i) {
      const int beg = i ? row_end(i - 1) : 0, end = row_end(i);
      for (int fc = 0; fc < n_fc; ++fc) {
        const int f0 = G > 1 ? (lane % (32 / G)) * VEC : fc * 32 * VEC + lane * VEC;
        const bool active = f0 < a.N;
        float acc[VEC];
        row_from_list<VEC, BT, kPF, G>(a, list, beg, end, f0, active, acc, pol_b);
        if (active && (G == 1 || lane < 32 / G)) {
          if (slot < 0) {
            store_c<VEC, float>(a.C + (rid + i) * a.ldc + f0, acc);
          } else {
            float* part = reinterpret_cast<float*>(a.partials) + ((int64_t)(slot + k) * 8 + i) * a.N + f0;
#pragma unroll
            for (int t = 0; t < VEC; ++t) __stcg(part + t, acc[t]);
          }
        }
      }
    }
    __syncwarp();
    return;
  }
  // dense unit: one row at a time (each row has at most 32 x 8 = 256 entries)
  for (int i = 0; i < nrows; ++i) {
    const uint32_t byte = uint32_t(bm >> (8 * i)) & 0xffu;
    const int cnt = __popc(byte);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int rtotal = __shfl_sync(0xffffffffu, incl, 31);
    int pos = incl - cnt;
    int vrank = i ? __popcll(bm & ((1ull << (8 * i)) - 1ull)) : 0;
    uint32_t rb = byte;
    while (rb) {
      const int j = __ffs(rb) - 1;
      rb &= rb - 1;
      list[pos++] = make_int2(meta_col(j), meta_val(vrank));
      ++vrank;
    }
    __syncwarp();
    for (int fc = 0; fc < n_fc; ++fc) {
      const int f0 = G > 1 ? (lane % (32 / G)) * VEC : fc * 32 * VEC + lane * VEC;
      const bool active = f0 < a.N;
      float acc[VEC];
      row_from_list<VEC, BT, kPF, G>(a, list, 0, rtotal, f0, active, acc, pol_b);
      if (active && (G == 1 || lane < 32 / G)) {
        if (slot < 0) {
          store_c<VEC, float>(a.C + (rid + i) * a.ldc + f0, acc);
        } else {
          float* part = reinterpret_cast<float*>(a.partials) + ((int64_t)(slot + k) * 8 + i) * a.N + f0;
#pragma unroll
          for (int t = 0; t < VEC; ++t) __stcg(part + t, acc[t]);
        }
      }
    }
    __syncwarp();
  }
}

// Multi-chunk window: the warp that finishes the last chunk sums the chunk partials in chunk order
// (last-finisher ticket) and writes the window rows -- deterministic and split-invariant.  Windows
// with more than kTicketMax chunks are left to the fix-up kernels.
template <int VEC, class AccT>
__device__ __forceinline__ void window_ticket_reduce(const SpmmArgs& a, int32_t g, int32_t slot, int64_t rid,
                                                     int64_t avail, int n_fc) {
  const int lane = threadIdx.x & 31;
  if (a.s.grp_nch[g] > kTicketMax) return;
  __threadfence();
  __syncwarp();
  uint32_t t = 0;
  if (lane == 0) t = atomicAdd(a.s.ticket + g, 1u);
  t = __shfl_sync(0xffffffffu, t, 0);
  const int32_t nch = a.s.grp_nch[g];
  if ((int32_t)t != nch - 1) return;
  __threadfence();
  for (int fc = 0; fc < n_fc; ++fc) {
    const int f0 = fc * 32 * VEC + lane * VEC;
    if (f0 >= a.N) continue;
    for (int i = 0; i < avail; ++i) {
      AccT sum[VEC];
#pragma unroll
      for (int q = 0; q < VEC; ++q) sum[q] = AccT(0);
      // partials summed in chunk order; loads issued 8 chunks ahead of the adds
      const AccT* part0 = reinterpret_cast<const AccT*>(a.partials) + (int64_t)i * a.N + f0;
      const int64_t cstride = (int64_t)8 * a.N;
      int kk = 0;
      for (; kk + 8 <= nch; kk += 8) {
        AccT buf[8][VEC];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int q = 0; q < VEC; ++q) buf[u][q] = __ldcg(part0 + (int64_t)(slot + kk + u) * cstride + q);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int q = 0; q < VEC; ++q) sum[q] += buf[u][q];
      }
      for (; kk < nch; ++kk)
#pragma unroll
        for (int q = 0; q < VEC; ++q) sum[q] += __ldcg(part0 + (int64_t)(slot + kk) * cstride + q);
      store_c<VEC, AccT>(a.C + (rid + i) * a.ldc + f0, sum);
    }
  }
  if (lane == 0) a.s.ticket[g] = 0;
}

template <int VEC, class BT, class AccT, int MINB = 4, int PF = 4, int G = 1>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_cc(SpmmArgs a) {
  __shared__ int2 s_list[kThreads / 32][kListCap];  // per-warp (col, value) list of a window unit
  __shared__ int s_tab[kThreads / 32][256];          // per-warp list offsets (lane, row)
  check_workspace(a);
  const int lane = threadIdx.x & 31;
  const int64_t total_units = a.s.header[2];
  const int n_fc = (a.N + 32 * VEC - 1) / (32 * VEC);
  const BT* B = reinterpret_cast<const BT*>(a.B);
  for (;;) {
    uint32_t u = 0;
    if (lane == 0) u = atomicAdd(a.s.counters, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if ((int64_t)u >= total_units) break;
    int4 un = a.s.units[u];
    int type = un.x & 3;
    if (type == kUnitWindow) {
      int32_t g = un.y, k = un.x >> 2;
      int64_t rid = a.s.grp_rid[g];
      int64_t avail = a.window_size < a.n_rows - rid ? a.window_size : a.n_rows - rid;
      int32_t slot = a.s.grp_slot[g];
      if constexpr (std::is_same<AccT, float>::value) {
        window_rows<VEC, BT, PF, G>(a, un, rid, avail, slot, k, G > 1 ? 1 : n_fc, s_list[threadIdx.x >> 5],
                                   s_tab[threadIdx.x >> 5]);
      } else
      for (int fc = 0; fc < n_fc; ++fc) {
        int f0 = fc * 32 * VEC + lane * VEC;
        bool active = f0 < a.N;
        AccT acc[8][VEC];
        window_chunk<VEC, BT, AccT>(a, un.z, un.w, f0, active, acc);
        if (slot < 0) {
          if (active) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i < avail) store_c<VEC, AccT>(a.C + (rid + i) * a.ldc + f0, acc[i]);
          }
        } else if (active) {
          AccT* part = reinterpret_cast<AccT*>(a.partials) + ((int64_t)(slot + k) * 8) * a.N;
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int t = 0; t < VEC; ++t) __stcg(part + (int64_t)i * a.N + f0 + t, acc[i][t]);
        }
      }
      if (slot >= 0) window_ticket_reduce<VEC, AccT>(a, g, slot, rid, avail, n_fc);
    } else if (type == kUnitResidual) {
      residual_rows<VEC, BT, AccT>(a, un.y, un.z, n_fc);
    } else {
      zero_rows<VEC>(a, un.y, un.z);
    }
  }
  // last warp out rewinds the counters so the next launch needs no memset
  __syncwarp();
  if (lane == 0) {
    uint32_t total_warps = (gridDim.x * blockDim.x) >> 5;
    if (atomicAdd(a.s.counters + 1, 1u) == total_warps - 1) {
      a.s.counters[0] = 0;
      a.s.counters[1] = 0;
    }
  }
}

__global__ void k_max_rel(const float* __restrict__ c, const float* __restrict__ r, int64_t rows, int64_t N,
                          int64_t ldc, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * N; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = i / N, f = i % N;
    double x = c[row * ldc + f], y = r[row * ldc + f];
    double d = fabs(x - y) / fmax(fabs(y), 1.0);
    m = fmax(m, d);
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// ------------------------------------------------------------------------------------------
// fixup of very long windows: partials of windows with more than kTicketMax chunks are summed
// by the whole GPU in a fixed two-level order (segments of kFixSeg chunks, then segments), so the
// result stays deterministic and independent of the format's split segments.
// ------------------------------------------------------------------------------------------

template <class AccT>
__global__ void k_fixup_segments(SpmmArgs a) {
  const int64_t nbig = a.s.header[6], nsegs = a.s.header[7];
  const int64_t N = a.N;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  AccT* P = reinterpret_cast<AccT*>(a.partials);
  for (int64_t t = tid; t < nsegs * 8 * N; t += stride) {
    const int64_t f = t % N, i = (t / N) % 8, sg = t / (8 * N);
    int64_t lo = 0, hi = nbig - 1;  // big window owning global segment sg
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (a.s.seg_base[mid] <= sg) lo = mid; else hi = mid - 1;
    }
    const int32_t g = a.s.big[lo];
    const int32_t nch = a.s.grp_nch[g], slot = a.s.grp_slot[g];
    const int c0 = (int)(sg - a.s.seg_base[lo]) * kFixSeg, c1 = c0 + kFixSeg < nch ? c0 + kFixSeg : nch;
    const AccT* src = P + ((int64_t)slot * 8 + i) * N + f;
    AccT sum = AccT(0);
    int c = c0;
    for (; c + 8 <= c1; c += 8) {
      AccT v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (int64_t)(c + u) * 8 * N);
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; c < c1; ++c) sum += __ldcg(src + (int64_t)c * 8 * N);
    __stcg(P + ((int64_t)(slot + c0) * 8 + i) * N + f, sum);
  }
}

template <class AccT>
__global__ void k_fixup_rows(SpmmArgs a) {
  const int64_t nbig = a.s.header[6];
  const int64_t N = a.N;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  const AccT* P = reinterpret_cast<const AccT*>(a.partials);
  for (int64_t t = tid; t < nbig * 8 * N; t += stride) {
    const int64_t f = t % N, i = (t / N) % 8, gi = t / (8 * N);
    const int32_t g = a.s.big[gi];
    const int64_t rid = a.s.grp_rid[g];
    const int64_t avail = a.window_size < a.n_rows - rid ? a.window_size : a.n_rows - rid;
    if (i >= avail) continue;
    const int32_t nch = a.s.grp_nch[g], slot = a.s.grp_slot[g];
    const int nseg = (nch + kFixSeg - 1) / kFixSeg;
    AccT sum = AccT(0);
    for (int sg = 0; sg < nseg; ++sg) sum += __ldcg(P + ((int64_t)(slot + sg * kFixSeg) * 8 + i) * N + f);
    __stcs(a.C + (rid + i) * a.ldc + f, (float)sum);
  }
}

template <class AccT>
int launch_fixup(const SpmmArgs& a, cudaStream_t st) {
  if (a.flags & 8192) return kOk;  // the caller knows the schedule has no fix-up windows
  const unsigned blocks = (unsigned)(2 * sm_count());
  k_fixup_segments<AccT><<<blocks, kThreads, 0, st>>>(a);
  RSH_LAUNCHED("k_fixup_segments");
  k_fixup_rows<AccT><<<blocks, kThreads, 0, st>>>(a);
  RSH_LAUNCHED("k_fixup_rows");
  return kOk;
}
template int launch_fixup<float>(const SpmmArgs&, cudaStream_t);


// ------------------------------------------------------------------------------------------
// the streaming CUDA-core kernel (fp32 accumulation): one warp per work unit, the unit's
// nonzeros listed once in row-major order and then gathered as ONE flat stream with kDepth B-row
// loads always in flight -- row boundaries are crossed without draining the pipeline.
//
// Why shared memory is kept tiny: the gathers are L1-allocating LDG.128s, and an SM can only
// have as many bytes in flight as its L1 can hold lines for (L1 = 228 KB minus shared memory).
// The list is 8 bytes per nonzero (kCap entries per warp) and nothing else is staged.
//
// Per unit:
//   1. window unit: lane l owns block b0 + l; two packed warp scans of the per-row popcounts give
//      every nonzero its row-major list position, and each lane copies its (col, value) pairs
//      into the list with 4-byte cp.async (no register round trip, all copies in flight at
//      once).  Residual unit: its entries are already contiguous (res_col / res_val).  Units
//      longer than kCap entries are listed and streamed in pieces; the row sum carries over.
//   2. stream: entry e's B row is requested kDepth entries before its FMA; a row's sum is stored
//      when the stream crosses the row's end (rows without nonzeros store zeros, as the reference
//      assigns every window row, execute.py:181-182).
// The per-row accumulation order -- blocks in order, columns ascending inside a block -- is the
// block walk's and the reference's (execute.py:171-182), so results are bit-identical to
// k_spmm_cc and independent of the schedule.
// ------------------------------------------------------------------------------------------

constexpr int kMaxRows = 16;   // rows per unit (8 window rows; kResRows residual rows)
static_assert(kResRows <= kMaxRows, "residual unit larger than the stream row table");

struct UnitDesc {
  long long s0;      // residual unit: first entry
  long long rid;     // window unit: first row
  const int2* ulist; // pre-built row-major window list (nullptr: list from the bitmaps)
  int v0;            // window unit: first value index (its list range starts there)
  int window, to_part, total, nrows, g, slot, avail, b0, b1;
  uint32_t next;     // the unit claimed for after this one
};

template <int kCap>
struct StreamSmem {
  int2 list[kCap];
  int rend[kMaxRows + 1];          // row-major list end of each unit row
  long long rowoff[kMaxRows];      // element offset of each unit row in C (or the partials)
  UnitDesc u;
  int4 nh[3];                      // the unit's header (k_unit_headers)
};

// Unit headers (schedule time, with the row-major list): everything the streaming kernel's unit
// setup otherwise chases through four dependent loads (unit -> group row / slot / value start ->
// bitmaps -> per-row totals), as three int4 per unit:
//   [0] = {units.x (type | chunk << 2), group, first row, partial slot (-1: rows go to C)}
//   [1] = {first list index, list entries, first block, end block}
//   [2] = the 8 per-row list ends (inclusive prefix), 16 bits each
// Residual and zero units keep their raw unit in [0] ([1], [2] zero).
__global__ void k_unit_headers(Sched s, const unsigned long long* __restrict__ bitmaps, int4* __restrict__ hdr) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_units = s.header[2];
  for (int64_t u = warp0; u < n_units; u += nwarps) {
    const int4 un = s.units[u];
    if ((un.x & 3) != kUnitWindow) {
      if (lane < 3) hdr[3 * u + lane] = lane == 0 ? un : make_int4(0, 0, 0, 0);
      continue;
    }
    unsigned long long t0 = 0, t1 = 0;
    for (int32_t blk = un.z + lane; blk < un.w; blk += 32) {
      const unsigned long long bm = bitmaps[blk];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        t0 += (unsigned long long)__popc(uint32_t(bm >> (8 * i)) & 0xffu) << (16 * i);
        t1 += (unsigned long long)__popc(uint32_t(bm >> (8 * (i + 4))) & 0xffu) << (16 * i);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      t0 += __shfl_xor_sync(0xffffffffu, t0, o);
      t1 += __shfl_xor_sync(0xffffffffu, t1, o);
    }
    const unsigned long long rp0 = t0 * 0x0001000100010001ull;
    const unsigned long long rp1 = t1 * 0x0001000100010001ull + (rp0 >> 48) * 0x0001000100010001ull;
    if (lane == 0) {
      const int32_t g = un.y, slot = s.grp_slot[g];
      hdr[3 * u] = make_int4(un.x, g, s.grp_rid[g], slot < 0 ? -1 : slot + (un.x >> 2));
      hdr[3 * u + 1] = make_int4(s.vstart[un.z], (int)(rp1 >> 48), un.z, un.w);
      hdr[3 * u + 2] = make_int4((int)(uint32_t)rp0, (int)(uint32_t)(rp0 >> 32), (int)(uint32_t)rp1,
                                 (int)(uint32_t)(rp1 >> 32));
    }
  }
}

// format-stream copy with an L2 policy (the nonzero stream is read once: evict_first)
__device__ __forceinline__ void cp_async4_sp(uint32_t saddr, const void* g, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(saddr), "l"(g), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async4_s(uint32_t saddr, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// raw (undecoded) B-row slice of one lane: VEC elements of BT as 32-bit words
template <int VEC, class BT>
struct RawVec {
  static constexpr int kWords = (VEC * (int)sizeof(BT) + 3) / 4;
  uint32_t w[kWords];
};

template <int VEC, class BT, bool kNoL1>
__device__ __forceinline__ void raw_load(const BT* p, RawVec<VEC, BT>& r, uint64_t pol) {
  constexpr int bytes = VEC * (int)sizeof(BT);
  if constexpr (bytes % 16 == 0) {
#pragma unroll
    for (int q = 0; q < bytes / 16; ++q) {
      const uint4* a = reinterpret_cast<const uint4*>(p) + q;
      if constexpr (kNoL1)
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
            : "=r"(r.w[4 * q]), "=r"(r.w[4 * q + 1]), "=r"(r.w[4 * q + 2]), "=r"(r.w[4 * q + 3])
            : "l"(a), "l"(pol));
      else
        asm("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
            : "=r"(r.w[4 * q]), "=r"(r.w[4 * q + 1]), "=r"(r.w[4 * q + 2]), "=r"(r.w[4 * q + 3])
            : "l"(a), "l"(pol));
    }
  } else if constexpr (bytes == 8) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    r.w[0] = u.x;
    r.w[1] = u.y;
  } else if constexpr (bytes == 4) {
    r.w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
  } else {  // 2-byte slice (VEC 1 of a half type)
    r.w[0] = (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p));
  }
}

template <int VEC, class BT>
__device__ __forceinline__ void raw_fma(const RawVec<VEC, BT>& r, float v, float (&acc)[VEC]) {
  const BT* e = reinterpret_cast<const BT*>(r.w);
#pragma unroll
  for (int t = 0; t < VEC; ++t) acc[t] = fmaf(v, to_f<BT>(e[t]), acc[t]);
}

// List positions [P0, P0 + kCap) of a window unit; on the first piece the unit's row table is
// written too.  With the pre-decoded row-major list (units of any length) a piece is one
// coalesced copy; without it (units of <= 32 blocks, lane l owning block b0 + l) every lane
// re-derives its block's row offsets and copies its nonzeros bit by bit.
template <int kCap>
__device__ __forceinline__ void window_fill(const SpmmArgs& a, StreamSmem<kCap>& sm, int P0, uint64_t pol_a) {
  const int lane = threadIdx.x & 31;
  if (P0 == 0 && sm.u.ulist) {
    // list mode (units of any length): the row table from the per-row totals of all blocks
    unsigned long long t0 = 0, t1 = 0;
    for (int32_t blk = sm.u.b0 + lane; blk < sm.u.b1; blk += 32) {
      const unsigned long long bm = ldg_hint64(a.bitmaps + blk, pol_a);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        t0 += (unsigned long long)__popc(uint32_t(bm >> (8 * i)) & 0xffu) << (16 * i);
        t1 += (unsigned long long)__popc(uint32_t(bm >> (8 * (i + 4))) & 0xffu) << (16 * i);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      t0 += __shfl_xor_sync(0xffffffffu, t0, o);
      t1 += __shfl_xor_sync(0xffffffffu, t1, o);
    }
    const unsigned long long rp0 = t0 * 0x0001000100010001ull;
    const unsigned long long rp1 = t1 * 0x0001000100010001ull + (rp0 >> 48) * 0x0001000100010001ull;
    if (lane < 8) {
      sm.rend[lane] = (int)(((lane < 4 ? rp0 : rp1) >> (16 * (lane & 3))) & 0xffffull);
      const int64_t rid = sm.u.rid;
      sm.rowoff[lane] = sm.u.slot < 0 ? (rid + lane) * a.ldc : ((int64_t)sm.u.slot * 8 + lane) * a.N;
    }
    if (lane == 0) sm.u.total = (int)(rp1 >> 48);
    __syncwarp();
  }
  if (sm.u.ulist) {  // the row table is set; copy this piece of the pre-decoded list
    const uint32_t list_s = (uint32_t)__cvta_generic_to_shared(sm.list);
    const int n = sm.u.total - P0 < kCap ? sm.u.total - P0 : kCap;
    const int2* src = sm.u.ulist + sm.u.v0 + P0;
    for (int p = lane; p < n; p += 32)
      asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(list_s + 8u * p),
                   "l"(src + p), "l"(pol_a) : "memory");
    cp_async_wait_all();
    __syncwarp();
    return;
  }
  if (sm.u.b1 - sm.u.b0 > 32) __trap();  // long units need the row-major list (rsh_schedule_rowmajor)
  const int32_t blk = sm.u.b0 + lane;
  const bool mine = blk < sm.u.b1;
  const unsigned long long bm = mine ? ldg_hint64(a.bitmaps + blk, pol_a) : 0ull;
  const int32_t vs = mine ? __ldg(a.s.vstart + blk) : 0;
  unsigned long long p0 = 0, p1 = 0;  // this lane's per-row counts, 4 rows x 16 bits per word
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    p0 |= (unsigned long long)__popc(uint32_t(bm >> (8 * i)) & 0xffu) << (16 * i);
    p1 |= (unsigned long long)__popc(uint32_t(bm >> (8 * (i + 4))) & 0xffu) << (16 * i);
  }
  unsigned long long q0 = p0, q1 = p1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t0 = __shfl_up_sync(0xffffffffu, q0, o);
    const unsigned long long t1 = __shfl_up_sync(0xffffffffu, q1, o);
    if (lane >= o) {
      q0 += t0;
      q1 += t1;
    }
  }
  const unsigned long long tot0 = __shfl_sync(0xffffffffu, q0, 31), tot1 = __shfl_sync(0xffffffffu, q1, 31);
  const unsigned long long rp0 = tot0 * 0x0001000100010001ull;  // inclusive prefix of the row totals
  const unsigned long long rp1 = tot1 * 0x0001000100010001ull + (rp0 >> 48) * 0x0001000100010001ull;
  if (P0 == 0) {
    if (lane < 8) {
      sm.rend[lane] = (int)(((lane < 4 ? rp0 : rp1) >> (16 * (lane & 3))) & 0xffffull);
      const int64_t rid = sm.u.rid;
      sm.rowoff[lane] = sm.u.slot < 0 ? (rid + lane) * a.ldc : ((int64_t)sm.u.slot * 8 + lane) * a.N;
    }
    if (lane == 0) sm.u.total = (int)(rp1 >> 48);
  }
  // F(i) = list start of this lane's row-i segment minus the lane's nonzeros before row i, so a
  // nonzero of rank r (its value index within the block) lands at F(row) + r.  Packed 4 x 16 bit.
  const unsigned long long ex0 = q0 - p0, ex1 = q1 - p1;  // exclusive lane prefixes per row
  const unsigned long long beg0 = (rp0 << 16), beg1 = (rp1 << 16) | (rp0 >> 48);  // row starts
  const unsigned long long below0 = (p0 * 0x0001000100010001ull) << 16;          // nnz of rows < i
  const unsigned long long below1 = ((p1 * 0x0001000100010001ull) << 16) + ((p0 * 0x0001000100010001ull) >> 48) * 0x0001000100010001ull;
  // fields stay non-negative: below(i) <= beg(i) + ex(i) always (a lane's own rows < i are part of the list before row i)
  const unsigned long long F0 = beg0 + ex0 - below0, F1 = beg1 + ex1 - below1;
  const uint32_t list_s = (uint32_t)__cvta_generic_to_shared(sm.list);
  const int32_t* cbase = a.col_id + (int64_t)blk * 8;
  const float* vbase = a.tc_values + vs;
  const int P1 = P0 + kCap;
  unsigned long long rem = bm;
  int r = 0;
  while (rem) {
    const int bit = __ffsll((long long)rem) - 1;
    rem &= rem - 1;
    const int i = bit >> 3;
    const int pos = (int)((((i < 4 ? F0 : F1) >> (16 * (i & 3))) & 0xffffull)) + r;
    if (pos >= P0 && pos < P1) {
      const uint32_t d = list_s + (uint32_t)(pos - P0) * 8u;
      if (a.flags & 1024) {
        cp_async4_s(d, cbase + (bit & 7));
        cp_async4_s(d + 4, vbase + r);
      } else {
        cp_async4_sp(d, cbase + (bit & 7), pol_a);
        cp_async4_sp(d + 4, vbase + r, pol_a);
      }
    }
    ++r;
  }
  cp_async_wait_all();
  __syncwarp();
}

// Row-major window list (schedule time, once per format): every window unit's nonzeros as
// (col_id, value) pairs in the order the stream consumes them -- rows in order, blocks in order
// inside a row, columns ascending inside a block.  A unit's pairs occupy the same index range as
// its values ([vstart[b0], vstart[b1])), so the list needs no offsets of its own.
__global__ void k_rowmajor_list(Sched s, const unsigned long long* __restrict__ bitmaps,
                                const int32_t* __restrict__ col_id, const float* __restrict__ tc_values, int2* ulist) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_units = s.header[1];  // window units come first
  for (int64_t uidx = warp0; uidx < n_units; uidx += nwarps) {
    const int4 un = s.units[uidx];
    const int32_t v0 = s.vstart[un.z];
    // pass 1: per-row totals over all blocks of the unit (4 rows x 16 bits per word; a unit has
    // at most 8 x 64 x 1024 ... fields stay below 2^16 for units of <= 1024 blocks)
    unsigned long long t0 = 0, t1 = 0;
    for (int32_t blk = un.z + lane; blk < un.w; blk += 32) {
      const unsigned long long bm = bitmaps[blk];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        t0 += (unsigned long long)__popc(uint32_t(bm >> (8 * i)) & 0xffu) << (16 * i);
        t1 += (unsigned long long)__popc(uint32_t(bm >> (8 * (i + 4))) & 0xffu) << (16 * i);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      t0 += __shfl_xor_sync(0xffffffffu, t0, o);
      t1 += __shfl_xor_sync(0xffffffffu, t1, o);
    }
    const unsigned long long rp0 = t0 * 0x0001000100010001ull;  // inclusive prefix of the row totals
    const unsigned long long rp1 = t1 * 0x0001000100010001ull + (rp0 >> 48) * 0x0001000100010001ull;
    const unsigned long long beg0 = (rp0 << 16), beg1 = (rp1 << 16) | (rp0 >> 48);  // row starts
    // pass 2: 32 blocks at a time; acc = entries of each row placed by earlier chunks
    unsigned long long acc0 = 0, acc1 = 0;
    for (int32_t c0 = un.z; c0 < un.w; c0 += 32) {
      const int32_t blk = c0 + lane;
      const bool mine = blk < un.w;
      const unsigned long long bm = mine ? bitmaps[blk] : 0ull;
      const int32_t vs = mine ? s.vstart[blk] : 0;
      unsigned long long p0 = 0, p1 = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        p0 |= (unsigned long long)__popc(uint32_t(bm >> (8 * i)) & 0xffu) << (16 * i);
        p1 |= (unsigned long long)__popc(uint32_t(bm >> (8 * (i + 4))) & 0xffu) << (16 * i);
      }
      unsigned long long q0 = p0, q1 = p1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long x0 = __shfl_up_sync(0xffffffffu, q0, o);
        const unsigned long long x1 = __shfl_up_sync(0xffffffffu, q1, o);
        if (lane >= o) {
          q0 += x0;
          q1 += x1;
        }
      }
      const unsigned long long ex0 = q0 - p0, ex1 = q1 - p1;
      const unsigned long long below0 = (p0 * 0x0001000100010001ull) << 16;
      const unsigned long long below1 =
          ((p1 * 0x0001000100010001ull) << 16) + ((p0 * 0x0001000100010001ull) >> 48) * 0x0001000100010001ull;
      // F(i) = row start + earlier chunks' entries of row i + this lane's exclusive offset - the
      // lane's nonzeros in rows < i (a nonzero of block rank r lands at F(row) + r)
      const unsigned long long F0 = beg0 + acc0 + ex0 - below0, F1 = beg1 + acc1 + ex1 - below1;
      unsigned long long rem = bm;
      int r = 0;
      while (rem) {
        const int bit = __ffsll((long long)rem) - 1;
        rem &= rem - 1;
        const int i = bit >> 3;
        const int pos = (int)((((i < 4 ? F0 : F1) >> (16 * (i & 3))) & 0xffffull)) + r;
        ulist[v0 + pos] = make_int2(col_id[(int64_t)blk * 8 + (bit & 7)], __float_as_int(tc_values[vs + r]));
        ++r;
      }
      acc0 += __shfl_sync(0xffffffffu, q0, 31);
      acc1 += __shfl_sync(0xffffffffu, q1, 31);
    }
  }
}

template <int kCap>
__device__ __forceinline__ void residual_fill(const SpmmArgs& a, StreamSmem<kCap>& sm, int P0) {
  const int lane = threadIdx.x & 31;
  const int64_t s0 = sm.u.s0 + P0;
  const int total = sm.u.total;
  const int n = total - P0 < kCap ? total - P0 : kCap;
  const uint32_t list_s = (uint32_t)__cvta_generic_to_shared(sm.list);
  for (int p = lane; p < n; p += 32) {
    cp_async4_s(list_s + 8u * p, a.res_col + s0 + p);
    cp_async4_s(list_s + 8u * p + 4, a.res_val + s0 + p);
  }
  cp_async_wait_all();
  __syncwarp();
}

// Stream the unit's row-major list (pieces of kCap positions) with kDepth B-row loads in flight.
// Bf = B + this lane's first feature; out = C (or the partials) + the same feature offset.
// Entries are consumed in groups of kDepth: a group that stays inside the current row (the
// common case) runs without any per-entry row test; only groups that reach a row end take the
// per-entry path that stores finished rows.
template <int VEC, class BT, int kDepth, bool kFull, bool kNoL1, int kCap, int kG>
__device__ __forceinline__ void stream_rows(const SpmmArgs& a, StreamSmem<kCap>& sm, const BT* __restrict__ Bf,
                                            bool active, int fc, float* __restrict__ out, uint64_t pol_b,
                                            uint64_t pol_a) {
  const char* const Bc = reinterpret_cast<const char*>(Bf);
  const uint32_t rstride = (uint32_t)(a.ldb * (int64_t)sizeof(BT));  // bytes per B row (< 4 GiB, checked on the host)
  const int total = sm.u.total;
  const bool single = total <= kCap;
  const int nrows = sm.u.nrows;
  // kG lane groups (narrow rows: a group of 32/kG lanes covers all N features) stream disjoint
  // row ranges of the unit, split where the running entry count crosses total * g / kG; every
  // row is still summed by one group in list order
  int r0 = 0, r1 = nrows;
  if constexpr (kG > 1) {
    const int g = (int)(threadIdx.x & 31) / (32 / kG);
    const int t0 = (int)((int64_t)total * g / kG), t1 = (int)((int64_t)total * (g + 1) / kG);
    r0 = 0;
    r1 = 0;
    for (int r = 0; r < nrows; ++r) {
      const int e = sm.rend[r];
      r0 += (g > 0 && e <= t0);
      r1 += (e <= t1);
    }
    if (g == kG - 1) r1 = nrows;
  }
  const int gb = r0 ? sm.rend[r0 - 1] : 0;                 // this group's entries [gb, ge)
  const int ge = r1 ? sm.rend[r1 - 1] : 0;
  float acc[VEC];
#pragma unroll
  for (int t = 0; t < VEC; ++t) acc[t] = 0.f;
  int cur = r0;
  int nxt_end = sm.rend[cur];
  auto flush = [&]() {
    if (kFull || active) store_c<VEC, float>(out + sm.rowoff[cur], acc);
#pragma unroll
    for (int t = 0; t < VEC; ++t) acc[t] = 0.f;
    ++cur;
    nxt_end = sm.rend[cur];
  };
  auto issue = [&](int idx, RawVec<VEC, BT>& r, float& v) {
    const int2 cv = sm.list[idx];
    v = __int_as_float(cv.y);
    if (kFull || active)
      raw_load<VEC, BT, kNoL1>(reinterpret_cast<const BT*>(Bc + (uint64_t)(uint32_t)cv.x * rstride), r, pol_b);
  };
  for (int P0 = 0; P0 < total; P0 += kCap) {
    if (P0 > 0 || (fc > 0 && !single)) {
      __syncwarp();  // the previous piece's list reads are done
      if (sm.u.window) window_fill<kCap>(a, sm, P0, pol_a);
      else residual_fill<kCap>(a, sm, P0);
    }
    const int len = total - P0 < kCap ? total - P0 : kCap;
    const int lb = gb - P0 > 0 ? gb - P0 : 0;              // this group's part of the piece
    const int le = ge - P0 < len ? ge - P0 : len;
    RawVec<VEC, BT> rb[kDepth];
    float vv[kDepth];
#pragma unroll
    for (int p = 0; p < kDepth; ++p)
      if (lb + p < le) issue(lb + p, rb[p], vv[p]);
    int base = lb;
    // steady state: every refill index base + kDepth + p is inside the group's part
    for (; base + 2 * kDepth <= le; base += kDepth) {
      if (P0 + base + kDepth - 1 < nxt_end) {
#pragma unroll
        for (int p = 0; p < kDepth; ++p) {
          if (kFull || active) raw_fma<VEC, BT>(rb[p], vv[p], acc);
          issue(base + kDepth + p, rb[p], vv[p]);
        }
      } else {
#pragma unroll
        for (int p = 0; p < kDepth; ++p) {
          while (P0 + base + p >= nxt_end) flush();
          if (kFull || active) raw_fma<VEC, BT>(rb[p], vv[p], acc);
          issue(base + kDepth + p, rb[p], vv[p]);
        }
      }
    }
    // drain: the last one or two groups of entries
    for (; base < le; base += kDepth) {
#pragma unroll
      for (int p = 0; p < kDepth; ++p) {
        const int e = base + p;
        if (e < le) {
          while (P0 + e >= nxt_end) flush();
          if (kFull || active) raw_fma<VEC, BT>(rb[p], vv[p], acc);
          if (e + kDepth < le) issue(e + kDepth, rb[p], vv[p]);
        }
      }
    }
  }
  while (cur < r1) flush();
}

// cp.async of 16 bytes (a unit header word) into shared memory
__device__ __forceinline__ void cp_async16_s(uint32_t saddr, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}

// A window unit's state from its header (k_unit_headers): row table, C / partial row offsets,
// descriptor fields; the caller copies the list afterwards.
template <int kCap>
__device__ __forceinline__ void apply_header(const SpmmArgs& a, StreamSmem<kCap>& sm, const int2* ulist) {
  const int lane = threadIdx.x & 31;
  const int4 h0 = sm.nh[0], h1 = sm.nh[1];
  const int64_t rid = h0.z;
  const int32_t slot = h0.w;
  if (lane < 8) {
    const int4 h2 = sm.nh[2];
    const uint32_t w = lane < 2 ? (uint32_t)h2.x : lane < 4 ? (uint32_t)h2.y : lane < 6 ? (uint32_t)h2.z : (uint32_t)h2.w;
    sm.rend[lane] = (int)((w >> (16 * (lane & 1))) & 0xffffu);
    sm.rowoff[lane] = slot < 0 ? (rid + lane) * a.ldc : ((int64_t)slot * 8 + lane) * a.N;
  }
  if (lane == 0) {
    const int64_t avail = a.window_size < a.n_rows - rid ? a.window_size : a.n_rows - rid;
    sm.u.window = 1;
    sm.u.to_part = slot >= 0;
    sm.u.g = h0.y;
    sm.u.slot = slot;
    sm.u.rid = rid;
    sm.u.avail = (int)avail;
    sm.u.nrows = slot < 0 ? (int)avail : 8;
    sm.u.v0 = h1.x;
    sm.u.total = h1.y;
    sm.u.b0 = h1.z;
    sm.u.b1 = h1.w;
    sm.u.ulist = ulist;
  }
  __syncwarp();
}

template <int kCap>
__device__ __forceinline__ void list_copy(StreamSmem<kCap>& sm, uint64_t pol_a) {
  const int lane = threadIdx.x & 31;
  const uint32_t list_s = (uint32_t)__cvta_generic_to_shared(sm.list);
  const int n = sm.u.total < kCap ? sm.u.total : kCap;
  const int2* src = sm.u.ulist + sm.u.v0;
  for (int p = lane; p < n; p += 32)
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(list_s + 8u * p),
                 "l"(src + p), "l"(pol_a) : "memory");
  cp_async_wait_all();
  __syncwarp();
}

template <int VEC, class BT, int kDepth, int MINB, bool kFull, bool kNoL1, int kCap, int kG>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_stream(SpmmArgs a) {
  __shared__ StreamSmem<kCap> smem_all[kThreads / 32];
  StreamSmem<kCap>& sm = smem_all[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  check_workspace(a);
  const int64_t total_units = a.s.header[2];
  // kG > 1: lane groups of 32/kG lanes, each covering all N = (32/kG) * VEC features
  const int n_fc = kG > 1 ? 1 : (a.N + 32 * VEC - 1) / (32 * VEC);
  const BT* B = reinterpret_cast<const BT*>(a.B);
  const uint64_t pol_b = policy_evict_last(), pol_a = policy_evict_first();
  // list mode with unit headers: a unit's setup is one 48-byte header read plus its list copy
  // instead of the chain unit -> group row / slot / value start -> bitmaps -> list (prefetching
  // the next unit's header during this one measured no better).  Flags bit 7 keeps the chain.
  const int2* ulist = (a.s.header[9] && !(a.flags & 4096)) ? reinterpret_cast<const int2*>(a.s.header[8]) : nullptr;
  const int4* hdrs = (ulist && !(a.flags & 128)) ? reinterpret_cast<const int4*>(a.s.header[11]) : nullptr;
  const uint32_t nh_s = (uint32_t)__cvta_generic_to_shared(sm.nh);

  uint32_t u = 0;
  if (lane == 0) u = atomicAdd(a.s.counters, 1u);
  u = __shfl_sync(0xffffffffu, u, 0);
  while ((int64_t)u < total_units) {
    int4 un;
    if (hdrs) {
      if (lane < 3) cp_async16_s(nh_s + 16u * lane, hdrs + 3 * (int64_t)u + lane);
      cp_async_wait_all();
      __syncwarp();
      un = sm.nh[0];
    } else {
      un = a.s.units[u];
    }
    // claim the next unit now: the atomic's round trip overlaps this unit's work
    uint32_t nx = 0;
    if (lane == 0) nx = atomicAdd(a.s.counters, 1u);
    const int type = un.x & 3;
    if (type == kUnitZero) {
      zero_rows<VEC>(a, un.y, un.z);
    } else {
      if (type == kUnitWindow) {
        if (hdrs) {
          apply_header<kCap>(a, sm, ulist);
          list_copy<kCap>(sm, pol_a);
        } else {
          if (lane == 0) {
            const int32_t g = un.y;
            const int64_t rid = a.s.grp_rid[g];
            const int32_t slot = a.s.grp_slot[g];
            sm.u.window = 1;
            sm.u.to_part = slot >= 0;
            sm.u.g = g;
            // chunk k of a multi-chunk window writes partial slot (slot + k)
            sm.u.slot = slot < 0 ? -1 : slot + (un.x >> 2);
            sm.u.rid = rid;
            const int64_t avail = a.window_size < a.n_rows - rid ? a.window_size : a.n_rows - rid;
            sm.u.avail = (int)avail;
            sm.u.nrows = slot < 0 ? (int)avail : 8;
            sm.u.b0 = un.z;
            sm.u.b1 = un.w;
            sm.u.ulist = ulist;
            sm.u.v0 = sm.u.ulist ? a.s.vstart[un.z] : 0;
          }
          __syncwarp();
          window_fill<kCap>(a, sm, 0, pol_a);
        }
      } else {
        const int32_t i0 = un.y, i1 = un.z;
        const int nr = i1 - i0;
        const int64_t s0 = __ldg(a.res_off + i0);
        if (lane < nr) {
          sm.rend[lane] = (int)(__ldg(a.res_off + i0 + lane + 1) - s0);
          sm.rowoff[lane] = (int64_t)__ldg(a.res_row + i0 + lane) * a.ldc;
        }
        if (lane == 0) {
          sm.u.window = 0;
          sm.u.to_part = 0;
          sm.u.total = (int)(__ldg(a.res_off + i1) - s0);
          sm.u.nrows = nr;
          sm.u.s0 = s0;
          sm.u.slot = -1;
        }
        __syncwarp();
        residual_fill<kCap>(a, sm, 0);
      }
      float* const out_base = sm.u.to_part ? reinterpret_cast<float*>(a.partials) : a.C;
      for (int fc = 0; fc < n_fc; ++fc) {
        const int f0 = kG > 1 ? (lane % (32 / kG)) * VEC : fc * 32 * VEC + lane * VEC;
        stream_rows<VEC, BT, kDepth, kFull, kNoL1, kCap, kG>(a, sm, B + f0, f0 < a.N, fc, out_base + f0, pol_b,
                                                            pol_a);
      }
      if (sm.u.window && sm.u.to_part)
        window_ticket_reduce<VEC, float>(a, sm.u.g, a.s.grp_slot[sm.u.g], sm.u.rid, sm.u.avail, n_fc);
    }
    __syncwarp();
    u = __shfl_sync(0xffffffffu, nx, 0);
  }
  // last warp out rewinds the counters so the next launch needs no memset
  __syncwarp();
  if (lane == 0) {
    const uint32_t total_warps = (gridDim.x * blockDim.x) >> 5;
    if (atomicAdd(a.s.counters + 1, 1u) == total_warps - 1) {
      a.s.counters[0] = 0;
      a.s.counters[1] = 0;
    }
  }
}

template <int VEC, class BT, int kDepth, int MINB, bool kFull, bool kNoL1, int kCap, int kG = 1>
int launch_stream_k(const SpmmArgs& a, cudaStream_t st) {
  auto kern = k_spmm_stream<VEC, BT, kDepth, MINB, kFull, kNoL1, kCap, kG>;
  // persistent grid: resident CTAs per SM x SMs, computed once (thread-safe static init)
  static const int blocks = [&] {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0) != cudaSuccess) per_sm = 1;
    return (per_sm > 0 ? per_sm : 1) * sm_count();
  }();
  kern<<<blocks, kThreads, 0, st>>>(a);
  RSH_LAUNCHED("k_spmm_stream");
  return launch_fixup<float>(a, st);
}

template <int VEC, class BT, int kDepth, int MINB, int kCap = 320>
int launch_stream(const SpmmArgs& a, cudaStream_t st) {
  const bool full = a.N % (32 * VEC) == 0;
  if (a.flags & 256) {  // gathers bypass L1 allocation (tuning experiment)
    if (full) return launch_stream_k<VEC, BT, kDepth, MINB, true, true, kCap>(a, st);
    return launch_stream_k<VEC, BT, kDepth, MINB, false, true, kCap>(a, st);
  }
  if (full) return launch_stream_k<VEC, BT, kDepth, MINB, true, false, kCap>(a, st);
  return launch_stream_k<VEC, BT, kDepth, MINB, false, false, kCap>(a, st);
}

// narrow rows (N = 16 B x 32 lanes / kG): kG lane groups stream disjoint row ranges of a unit
template <int VEC, class BT, int kG>
int launch_stream_groups(const SpmmArgs& a, cudaStream_t st) {
  switch ((a.flags >> 3) & 7) {  // pipeline depth / occupancy variants (tuning knob)
    case 1: return launch_stream_k<VEC, BT, 4, 4, true, false, 320, kG>(a, st);
    case 3: return launch_stream_k<VEC, BT, 8, 3, true, false, 320, kG>(a, st);
    default: return launch_stream_k<VEC, BT, 6, 4, true, false, 320, kG>(a, st);
  }
}

// pipeline depth / occupancy / list-size variants (tuning knob: flags bits 3-5)
template <int VEC, class BT>
int dispatch_stream(const SpmmArgs& a, cudaStream_t st) {
  switch ((a.flags >> 3) & 7) {
    case 1: return launch_stream<VEC, BT, 4, 4>(a, st);
    case 2: return launch_stream<VEC, BT, 6, 4>(a, st);  // the default (case 0)
    case 3: return launch_stream<VEC, BT, 8, 3>(a, st);
    case 4: return launch_stream<VEC, BT, 4, 4, 256>(a, st);
    case 5: return launch_stream<VEC, BT, 6, 4, 256>(a, st);
    case 6: return launch_stream<VEC, BT, 4, 4, 448>(a, st);
    default: return launch_stream<VEC, BT, 6, 4>(a, st);
  }
}

template <int VEC, class BT, class AccT, int MINB, int PF, int G = 1>
int launch_cc_v(const SpmmArgs& a, cudaStream_t st) {
  auto kern = k_spmm_cc<VEC, BT, AccT, MINB, PF, G>;
  // persistent grid: resident CTAs per SM x SMs, computed once (thread-safe static init)
  static const int blocks = [&] {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0) != cudaSuccess) per_sm = 1;
    return (per_sm > 0 ? per_sm : 1) * sm_count();
  }();
  kern<<<blocks, kThreads, 0, st>>>(a);
  RSH_LAUNCHED("k_spmm_cc");
  return launch_fixup<AccT>(a, st);
}

template <int VEC, class BT, class AccT>
int launch_cc(const SpmmArgs& a, cudaStream_t st) {
  if constexpr (std::is_same<AccT, float>::value && VEC == 4) {
    // occupancy / gathers-in-flight trade-off (tuning knob, flags bits 1-2)
    switch (a.flags & 3) {
      case 1: return launch_cc_v<VEC, BT, AccT, 3, 8>(a, st);
      case 2: return launch_cc_v<VEC, BT, AccT, 4, 8>(a, st);
      case 3: return launch_cc_v<VEC, BT, AccT, 4, 4>(a, st);
      default: break;
    }
  }
  return launch_cc_v<VEC, BT, AccT, 3, 4>(a, st);
}

template <class BT, class AccT>
int dispatch_vec(const SpmmArgs& a, int vec, cudaStream_t st) {
  switch (vec) {
    case 8: return launch_cc<8, BT, AccT>(a, st);
    case 4: return launch_cc<4, BT, AccT>(a, st);
    case 2: return launch_cc<2, BT, AccT>(a, st);
    default: return launch_cc<1, BT, AccT>(a, st);
  }
}

}  // namespace rsh

using namespace rsh;

extern "C" {

size_t rsh_schedule_bytes(int64_t n_rows, int64_t n_entries, int64_t n_blocks, int64_t n_res) {
  Sched s;
  return sched_layout(nullptr, n_rows, n_entries, n_blocks, n_res, &s);
}

// Work-unit schedule for one RS-Tile format (execute.py:136-168 restated as device data):
// logical windows, fixed-offset chunks of chunk_blocks blocks (kChunkCC for the CUDA-core
// kernel, kChunkTC for the tensor-core kernel), partial slots, per-block value starts,
// uncovered rows.
// header_out (device int64[8]) receives [groups, window units, units, partial slots, uncovered].
int rsh_schedule(int64_t n_rows, int32_t window_size, const int32_t* row_window_id, const int64_t* row_window_offset,
                 int64_t n_entries, const uint64_t* bitmaps, int64_t n_blocks, const int32_t* res_row_id, int64_t n_res,
                 int32_t chunk_blocks, void* sched, size_t sched_bytes, int64_t* header_out, cudaStream_t st) {
  if (n_rows < 0 || n_entries < 0 || n_blocks < 0 || n_res < 0 || window_size < 1 || window_size > 8)
    return fail(kInvalid, "rsh_schedule: bad sizes");
  // units pack per-row counts of up to chunk_blocks x 8 nonzeros into 16-bit fields
  if (chunk_blocks < kChunkMin || chunk_blocks > kChunkMax)
    return fail(kInvalid, "rsh_schedule: chunk_blocks %d outside [%d, %d]", chunk_blocks, kChunkMin, kChunkMax);
  if (n_blocks >= (1LL << 31) || n_rows >= (1LL << 31)) return fail(kInvalid, "rsh_schedule: index limit");
  Sched s;
  size_t need = sched_layout(sched, n_rows, n_entries, n_blocks, n_res, &s);
  if (!sched || sched_bytes < need) return fail(kInvalid, "rsh_schedule: buffer %zu < %zu bytes", sched_bytes, need);
  int64_t E = n_entries;
  RSH_CUDA(cudaMemsetAsync(s.header, 0, 16 * sizeof(int64_t), st));
  size_t cb;
  if (E) {
    k_group_heads<<<grid_1d(E), kThreads, 0, st>>>(row_window_id, E, s.flags);
    RSH_LAUNCHED("k_group_heads");
    cb = s.cub_bytes;
    RSH_CUDA(cub::DeviceSelect::Flagged(s.cub, cb, cub::CountingInputIterator<int32_t>(0), s.flags, s.head,
                                        s.header, (int)E, st));
  }
  k_groups<<<grid_1d(E + 1), kThreads, 0, st>>>(row_window_id, row_window_offset, E, s, chunk_blocks);
  RSH_LAUNCHED("k_groups");
  // unit_base currently holds nch; scan it (through grp_slot as scratch), multi -> slot_base
  cb = s.cub_bytes;
  RSH_CUDA(cudaMemcpyAsync(s.grp_slot, s.unit_base, (E + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(s.cub, cb, s.grp_slot, s.unit_base, (int)(E + 1), st));
  cb = s.cub_bytes;
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(s.cub, cb, s.grp_multi, s.slot_base, (int)(E + 1), st));
  RSH_CUDA(cudaMemsetAsync(s.unit_cost_raw, 0, (s.max_units + 1) * sizeof(int64_t), st));
  if (E) {
    k_window_units<<<grid_1d(E), kThreads, 0, st>>>(E, s, chunk_blocks);
    RSH_LAUNCHED("k_window_units");
  }
  cb = s.cub_bytes;
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(s.cub, cb, s.unit_cost_raw, s.unit_cost, (int)(s.max_units + 1), st));
  // windows with more than kTicketMax chunks: reduced by the fixup kernels, not by tickets
  k_big_flags<<<grid_1d(E + 1), kThreads, 0, st>>>(s, E);
  RSH_LAUNCHED("k_big_flags");
  cb = s.cub_bytes;
  RSH_CUDA(cub::DeviceSelect::Flagged(s.cub, cb, cub::CountingInputIterator<int32_t>(0), s.flags, s.big,
                                      s.header + 6, (int)(E + 1), st));
  k_seg_base<<<1, 1, 0, st>>>(s);
  RSH_LAUNCHED("k_seg_base");
  // per-block value starts (execute.py:167-168)
  k_popc32<<<grid_1d(n_blocks + 1), kThreads, 0, st>>>((const unsigned long long*)bitmaps, n_blocks, s.pc);
  cb = s.cub_bytes;
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(s.cub, cb, s.pc, s.vstart, (int)(n_blocks + 1), st));
  // vstart (int32) must not wrap: tc nonzeros < 2^31, summed exactly in 64 bits
  if (n_blocks * 64 >= (1LL << 31)) {
    int64_t* tot = s.header + 10;
    RSH_CUDA(cudaMemsetAsync(tot, 0, sizeof(int64_t), st));
    k_popc_total<<<grid_1d(n_blocks, kThreads) > 4096 ? 4096 : grid_1d(n_blocks), kThreads, 0, st>>>(
        (const unsigned long long*)bitmaps, n_blocks, (unsigned long long*)tot);
    RSH_LAUNCHED("k_popc_total");
    int64_t h = 0;
    RSH_CUDA(cudaMemcpyAsync(&h, tot, sizeof(h), cudaMemcpyDeviceToHost, st));
    RSH_CUDA(cudaStreamSynchronize(st));
    if (h >= (1LL << 31)) return fail(kInvalid, "rsh_schedule: %lld tensor-core nonzeros exceed the 32-bit index limit", (long long)h);
  }
  // uncovered rows
  if (n_rows) {
    RSH_CUDA(cudaMemsetAsync(s.uncov_flag, 1, n_rows, st));
    k_uncover<<<grid_1d(E + n_res + 1), kThreads, 0, st>>>(s, n_rows, window_size, res_row_id, n_res);
    RSH_LAUNCHED("k_uncover");
    cb = s.cub_bytes;
    RSH_CUDA(cub::DeviceSelect::Flagged(s.cub, cb, cub::CountingInputIterator<int32_t>(0), s.uncov_flag, s.uncovered,
                                        s.header + 4, (int)n_rows, st));
  }
  k_finish_header<<<1, 1, 0, st>>>(s, E, n_res, chunk_blocks);
  k_tail_units<<<grid_1d(n_res / kResRows + n_rows / kZeroRows + 2), kThreads, 0, st>>>(s, n_res);
  RSH_LAUNCHED("schedule tail");
  if (header_out) RSH_CUDA(cudaMemcpyAsync(header_out, s.header, 8 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  return kOk;
}

// Row-major window list for the streaming kernel (k_rowmajor_list): int2 ulist[tc_nnz] built from
// the format once per schedule; its address is recorded in the schedule so rsh_spmm_cc copies
// each unit's list with one coalesced read instead of decoding bitmaps.  Results are
// bit-identical with or without it.
// bytes rsh_schedule_rowmajor needs: the list (8 per tc nonzero) + scratch to reorder units
size_t rsh_rowmajor_bytes(int64_t n_rows, int64_t n_entries, int64_t n_blocks, int64_t n_res, int64_t tc_nnz) {
  Sched s;
  sched_layout(nullptr, n_rows, n_entries, n_blocks, n_res, &s);
  const int64_t mu = s.max_units;
  Carve cv(nullptr);
  cv.take<int2>(tc_nnz > 0 ? tc_nnz : 1);
  cv.take<unsigned long long>(mu);
  cv.take<unsigned long long>(mu);
  cv.take<int4>(mu);
  cv.take<int4>(3 * mu);  // unit headers (k_unit_headers)
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (int4*)nullptr, (int4*)nullptr, (int)mu);
  cv.take<char>(t);
  return cv.used + 256;
}

// longest-first order of the window units (key: chunks of the unit's window, descending; then
// the original position): the chunks of long windows start first instead of forming the
// kernel's tail, chunk order inside a window and the order of single-chunk windows are kept,
// residual and zero units keep their slots.
__global__ void k_unit_keys(Sched s, unsigned long long* keys) {
  const int64_t n_wu = s.header[1];
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < s.max_units; u += (int64_t)gridDim.x * blockDim.x) {
    if (u < n_wu) {
      const int4 un = s.units[u];
      const uint32_t nch = (uint32_t)s.grp_nch[un.y];
      keys[u] = ((unsigned long long)(0xFFFFFFFFu - nch) << 32) | (uint32_t)u;
    } else {
      keys[u] = ~0ull;
    }
  }
}

// Row-major window list for the streaming kernel (k_rowmajor_list): int2 pairs per tc nonzero
// built from the format once per schedule (plus the window units put longest-first); its
// address is recorded in the schedule so rsh_spmm_cc copies each unit's list with one coalesced
// read instead of decoding bitmaps.  Results are bit-identical with or without it for a given
// schedule.  ulist_bytes >= rsh_rowmajor_bytes(...).
int rsh_schedule_rowmajor(int64_t n_rows, int64_t n_entries, const uint64_t* bitmaps, const int32_t* col_id,
                          const float* tc_values, int64_t n_blocks, int64_t tc_nnz, int64_t n_res, void* sched,
                          size_t sched_bytes, void* ulist, size_t ulist_bytes, cudaStream_t st) {
  Sched s;
  const size_t need = sched_layout(sched, n_rows, n_entries, n_blocks, n_res, &s);
  if (!sched || sched_bytes < need) return fail(kInvalid, "rsh_schedule_rowmajor: schedule buffer too small");
  if (tc_nnz < 0 || tc_nnz >= (1LL << 31))
    return fail(kInvalid, "rsh_schedule_rowmajor: %lld nonzeros exceed the 32-bit index limit", (long long)tc_nnz);
  if (!ulist || ulist_bytes < rsh_rowmajor_bytes(n_rows, n_entries, n_blocks, n_res, tc_nnz))
    return fail(kInvalid, "rsh_schedule_rowmajor: list buffer smaller than rsh_rowmajor_bytes()");
  if ((uintptr_t)ulist & 15) return fail(kInvalid, "rsh_schedule_rowmajor: list must be 16-byte aligned");
  Carve cv(ulist);
  int2* list = cv.take<int2>(tc_nnz > 0 ? tc_nnz : 1);
  unsigned long long* keys = cv.take<unsigned long long>(s.max_units);
  unsigned long long* keys2 = cv.take<unsigned long long>(s.max_units);
  int4* units2 = cv.take<int4>(s.max_units);
  int4* uhdr = cv.take<int4>(3 * s.max_units);
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (int4*)nullptr, (int4*)nullptr, (int)s.max_units);
  void* tmp = cv.take<char>(t);
  if (tc_nnz) {
    k_rowmajor_list<<<8 * sm_count(), kThreads, 0, st>>>(s, (const unsigned long long*)bitmaps, col_id, tc_values,
                                                          list);
    RSH_LAUNCHED("k_rowmajor_list");
  }
  if (!getenv("RSH_NO_LPT")) {
    k_unit_keys<<<grid_1d(s.max_units), kThreads, 0, st>>>(s, keys);
    RSH_LAUNCHED("k_unit_keys");
    RSH_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, keys, keys2, s.units, units2, (int)s.max_units, 0, 64, st));
    RSH_CUDA(cudaMemcpyAsync(s.units, units2, s.max_units * sizeof(int4), cudaMemcpyDeviceToDevice, st));
  }
  k_unit_headers<<<8 * sm_count(), kThreads, 0, st>>>(s, (const unsigned long long*)bitmaps, uhdr);
  RSH_LAUNCHED("k_unit_headers");
  const int64_t hdr[4] = {(int64_t)(uintptr_t)list, tc_nnz, 0, (int64_t)(uintptr_t)uhdr};
  RSH_CUDA(cudaMemcpyAsync(s.header + 8, hdr, sizeof(hdr), cudaMemcpyHostToDevice, st));
  RSH_CUDA(cudaStreamSynchronize(st));  // hdr lives on this host stack frame
  return kOk;
}

// bytes of chunk-partial workspace rsh_spmm needs (partial_slots from the schedule header)
size_t rsh_partials_bytes(int64_t n_entries, int64_t partial_slots, int64_t N, int32_t accum) {
  return spmm_ctl_bytes(n_entries) +
         (size_t)(partial_slots > 0 ? partial_slots : 1) * 8 * (size_t)N * (accum ? sizeof(double) : sizeof(float));
}

// execute.py:155-218.  b_dtype: 0 f32, 1 bf16, 2 f16.  accum: 0 f32, 1 f64.  math: 0 = CUDA-core
// (fp32 FMA, exact f32 products), 1 = tensor-core window path (see spmm_tc.cu).
int rsh_spmm_cc(int64_t n_rows, int32_t window_size, int64_t n_entries, const uint64_t* bitmaps, const int32_t* col_id,
                const float* tc_values, int64_t n_blocks, const int32_t* res_row_id, const int64_t* res_offset,
                const int32_t* res_col_id, const float* res_values, int64_t n_res, const void* B, int64_t ldb,
                int32_t b_dtype, int64_t N, float* C, int64_t ldc, int32_t accum, void* sched, size_t sched_bytes,
                void* partials, size_t partial_bytes, cudaStream_t st) {
  if (N < 1 || N > (1 << 30) || ldb < N || ldc < N || !B || !C) return fail(kInvalid, "rsh_spmm: bad dense operands");
  if (b_dtype < 0 || b_dtype > 2 || accum < 0 || accum > 32767) return fail(kInvalid, "rsh_spmm: bad dtype/accum");
  Sched s;
  size_t need = sched_layout(sched, n_rows, n_entries, n_blocks, n_res, &s);
  if (!sched || sched_bytes < need) return fail(kInvalid, "rsh_spmm: schedule buffer too small");
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
  RSH_OK(bind_workspace(a, partials, partial_bytes, n_entries, (accum & 1) ? sizeof(double) : sizeof(float)));
  a.flags = accum >> 1;  // tuning knobs: bits 0-1 row-walk occupancy variant, bit 2 no L2 cache hints,
                         // bits 3-5 stream depth/occupancy variant, bit 6 row-walk kernel instead of the stream,
                         // bit 8 stream gathers bypass L1 allocation, bit 10 list copies without L2 hint, bit 11 no lane groups, bit 12 ignore the row-major list,
                         // bit 13 no window exceeds kTicketMax chunks (schedule header[6] == 0): skip the fix-up launches
  accum &= 1;
  // widest per-lane vector that tiles N and keeps loads aligned
  size_t esz = b_dtype == 0 ? 4 : 2;
  int vec = 8;
  while (vec > 1 && (N % vec || ldb % vec || ldc % vec || 32 * vec > N ||
                     ((uintptr_t)B % (vec * esz)) || ((uintptr_t)C % (vec * 4 < 16 ? vec * 4 : 16))))
    vec >>= 1;
  if (accum == 1 && vec > 4) vec = 4;
  // the stream kernel addresses B rows with a 32-bit byte stride
  if (ldb * (int64_t)esz >= (1LL << 32)) a.flags |= 64;
  // A schedule with units above 32 blocks (chunk_blocks > 32) needs the row-major list and the
  // streaming kernel for f32 accumulation; the kernels trap on a unit they cannot walk.
  if (accum == 0 && !(a.flags & 64)) {
    // streaming kernel: the f32-accumulation default (flags bit 6 selects the row-walk kernel)
    const bool al16 = !((uintptr_t)B & 15) && !((uintptr_t)C & 15) && (ldb * (int64_t)esz) % 16 == 0 && ldc % 4 == 0;
    if (al16 && !(a.flags & 2048)) {  // narrow rows: 16-byte lanes in groups (flags bit 11 disables)
      if (b_dtype == 0 && N == 64) return launch_stream_groups<4, float, 2>(a, st);
      if (b_dtype == 0 && N == 32) return launch_stream_groups<4, float, 4>(a, st);
      if (b_dtype == 1 && N == 128) return launch_stream_groups<8, __nv_bfloat16, 2>(a, st);
      if (b_dtype == 1 && N == 64) return launch_stream_groups<8, __nv_bfloat16, 4>(a, st);
      if (b_dtype == 2 && N == 128) return launch_stream_groups<8, __half, 2>(a, st);
      if (b_dtype == 2 && N == 64) return launch_stream_groups<8, __half, 4>(a, st);
    }
    if (b_dtype == 0) {
      if (vec >= 4) return dispatch_stream<4, float>(a, st);
      if (vec == 2) return dispatch_stream<2, float>(a, st);
      return launch_stream<1, float, 6, 4>(a, st);
    }
    if (b_dtype == 1) {
      if (vec == 8) return dispatch_stream<8, __nv_bfloat16>(a, st);
      if (vec == 4) return launch_stream<4, __nv_bfloat16, 6, 4>(a, st);
      if (vec == 2) return launch_stream<2, __nv_bfloat16, 6, 4>(a, st);
      return launch_stream<1, __nv_bfloat16, 6, 4>(a, st);
    }
    if (vec == 8) return dispatch_stream<8, __half>(a, st);
    if (vec == 4) return launch_stream<4, __half, 6, 4>(a, st);
    if (vec == 2) return launch_stream<2, __half, 6, 4>(a, st);
    return launch_stream<1, __half, 6, 4>(a, st);
  }
  if (accum == 0 && b_dtype == 0 && (N == 64 || N == 32) && ldb % 4 == 0 && ldc % 4 == 0 && !((uintptr_t)B & 15) &&
      !((uintptr_t)C & 15)) {
    // narrow fp32 rows: lane groups take alternate list entries with 16-byte loads
    if (N == 64) return launch_cc_v<4, float, float, 3, 4, 2>(a, st);
    return launch_cc_v<4, float, float, 3, 4, 4>(a, st);
  }
  if (accum == 0) {
    if (b_dtype == 0) return dispatch_vec<float, float>(a, vec, st);
    if (b_dtype == 1) return dispatch_vec<__nv_bfloat16, float>(a, vec, st);
    return dispatch_vec<__half, float>(a, vec, st);
  }
  if (b_dtype == 0) return dispatch_vec<float, double>(a, vec, st);
  if (b_dtype == 1) return dispatch_vec<__nv_bfloat16, double>(a, vec, st);
  return dispatch_vec<__half, double>(a, vec, st);
}

// max |c - r| / max(|r|, 1) over rows x N (core.py:398-408), as a double in out[0]
int rsh_max_relative_error(const float* c, const float* r, int64_t rows, int64_t N, int64_t ldc, double* out,
                           cudaStream_t st) {
  RSH_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
  if (rows * N == 0) return kOk;
  k_max_rel<<<grid_1d(rows * N, kThreads) > 4096 ? 4096 : grid_1d(rows * N), kThreads, 0, st>>>(
      c, r, rows, N, ldc, (unsigned long long*)out);
  RSH_LAUNCHED("k_max_rel");
  return kOk;
}

}  // extern "C"
