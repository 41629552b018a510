// Device validation and decoding of an RS-Tile format (tile.py:176-307).
//
// rsh_validate fills a small report of structural facts (first offending index per check); the
// host turns the report into the reference's messages in the reference's order (tile.py:176-267).
// rsh_decode expands the format back into (row, col, value) triples -- every value slot knows its
// block, bit and therefore its row and column -- sorts them by (row, col) with a radix sort and
// emits CSR (tile.py:270-307).
#include "common.cuh"
#include <cub/cub.cuh>

namespace rsh {

// report slots (int64), all "first offending index" slots start at INT64_MAX
enum Rep : int {
  kOff0 = 0,          // row_window_offset[0]
  kOffLast,           // row_window_offset[E]
  kOffNonMono,        // first e with off[e+1] < off[e]
  kColMin, kColMax,   // col_id range
  kRwidMin, kRwidMax, // row_window_id range
  kPopSum,            // sum of popcounts
  kPopFirstOver,      // first block b with cum[b+1] > n_values
  kBitBeyond,         // first block with a bit beyond its window's last row
  kResOff0, kResOffLast, kResNonMono,
  kResRowNonInc,      // first i with row_id[i+1] <= row_id[i]
  kResRowMin, kResRowMax,
  kResColMin, kResColMax,
  kResInWindow,       // first residual index whose row lies in a window's range
  kDupHead,           // first entry re-opening a row window that an earlier group used
  kRepSlots
};


__global__ void k_rep_init(int64_t* rep) {
  int i = threadIdx.x;
  if (i < kRepSlots) {
    int64_t v = INT64_MAX;
    if (i == kColMax || i == kRwidMax || i == kResRowMax || i == kResColMax) v = INT64_MIN;
    if (i == kPopSum || i == kOff0 || i == kOffLast || i == kResOff0 || i == kResOffLast) v = 0;
    rep[i] = v;
  }
}

// Block-level reductions so that each CTA issues one atomic per report slot.
template <class Op>
__device__ __forceinline__ int64_t block_reduce(int64_t v, Op op, int64_t* s_red) {
  for (int o = 16; o; o >>= 1) v = op(v, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) s_red[w] = v;
  __syncthreads();
  if (w == 0) {
    // lanes past the last warp repeat warp 0's value: harmless for min / max, wrong for a sum
    v = l < (int)(blockDim.x >> 5) ? s_red[l] : (Op::kIdempotent ? s_red[0] : 0);
    for (int o = 16; o; o >>= 1) v = op(v, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)v, o));
  }
  return v;  // valid in thread 0
}
struct Min { static constexpr bool kIdempotent = true; __device__ int64_t operator()(int64_t a, int64_t b) const { return a < b ? a : b; } };
struct Max { static constexpr bool kIdempotent = true; __device__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; } };
struct Sum { static constexpr bool kIdempotent = false; __device__ int64_t operator()(int64_t a, int64_t b) const { return a + b; } };

__device__ __forceinline__ void amin_s(int64_t* p, int64_t v) { atomicMin((long long*)p, (long long)v); }
__device__ __forceinline__ void amax_s(int64_t* p, int64_t v) { atomicMax((long long*)p, (long long)v); }

// entry of a block: the e with off[e] <= b < off[e+1] (offsets monotone)
__device__ __forceinline__ int64_t entry_of(const int64_t* __restrict__ off, int64_t E, int64_t b) {
  int64_t lo = 0, hi = E - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// tile.py:185-204 / 223-238: offsets, ranges, popcount sum, bits beyond the window's last row
__global__ void k_val_tc(const int32_t* __restrict__ rwid, const int64_t* __restrict__ off, int64_t E,
                         const uint64_t* __restrict__ bm, int64_t nb, const int32_t* __restrict__ col, int64_t ncol,
                         int64_t n_rows, int32_t wsize, int check_bits, int64_t* rep) {
  __shared__ int64_t s_red[32];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  int64_t nonmono = INT64_MAX, rmin = INT64_MAX, rmax = INT64_MIN, cmin = INT64_MAX, cmax = INT64_MIN;
  int64_t pop = 0, beyond = INT64_MAX;
  for (int64_t e = tid; e < E; e += stride) {
    if (off[e + 1] < off[e] && nonmono == INT64_MAX) nonmono = e;
    rmin = min(rmin, (int64_t)rwid[e]);
    rmax = max(rmax, (int64_t)rwid[e]);
  }
  for (int64_t i = tid; i < ncol; i += stride) {
    cmin = min(cmin, (int64_t)col[i]);
    cmax = max(cmax, (int64_t)col[i]);
  }
  for (int64_t b = tid; b < nb; b += stride) {
    const uint64_t m = bm[b];
    pop += __popcll(m);
    if (check_bits && E && m && beyond == INT64_MAX) {
      const int64_t rid = rwid[entry_of(off, E, b)];
      const int64_t avail = wsize < n_rows - rid ? wsize : n_rows - rid;
      if (((63 - __clzll((long long)m)) >> 3) >= avail) beyond = b;
    }
  }
  nonmono = block_reduce(nonmono, Min(), s_red);
  if (threadIdx.x == 0 && nonmono != INT64_MAX) amin_s(rep + kOffNonMono, nonmono);
  rmin = block_reduce(rmin, Min(), s_red);
  if (threadIdx.x == 0 && E) amin_s(rep + kRwidMin, rmin);
  rmax = block_reduce(rmax, Max(), s_red);
  if (threadIdx.x == 0 && E) amax_s(rep + kRwidMax, rmax);
  cmin = block_reduce(cmin, Min(), s_red);
  if (threadIdx.x == 0 && ncol) amin_s(rep + kColMin, cmin);
  cmax = block_reduce(cmax, Max(), s_red);
  if (threadIdx.x == 0 && ncol) amax_s(rep + kColMax, cmax);
  pop = block_reduce(pop, Sum(), s_red);
  if (threadIdx.x == 0 && pop) atomicAdd((unsigned long long*)(rep + kPopSum), (unsigned long long)pop);
  beyond = block_reduce(beyond, Min(), s_red);
  if (threadIdx.x == 0 && beyond != INT64_MAX) amin_s(rep + kBitBeyond, beyond);
  if (tid == 0) {
    rep[kOff0] = off[0];
    rep[kOffLast] = off[E];
  }
}

__global__ void k_popc64(const uint64_t* __restrict__ bm, int64_t nb, int64_t* pc) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= nb; b += (int64_t)gridDim.x * blockDim.x)
    pc[b] = b < nb ? __popcll(bm[b]) : 0;
}

// tile.py:211-218: first block whose running popcount exceeds the value count
__global__ void k_pop_over(const int64_t* __restrict__ cum, int64_t nb, int64_t nvals, int64_t* rep) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    if (cum[b + 1] > nvals) amin_s(rep + kPopFirstOver, b);
}

// tile.py:240-254: residual offsets and ranges
__global__ void k_val_res(const int32_t* __restrict__ row, const int64_t* __restrict__ roff, int64_t R,
                          const int32_t* __restrict__ col, int64_t ncol, int64_t* rep) {
  __shared__ int64_t s_red[32];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  int64_t nonmono = INT64_MAX, noninc = INT64_MAX, rmin = INT64_MAX, rmax = INT64_MIN, cmin = INT64_MAX,
          cmax = INT64_MIN;
  for (int64_t i = tid; i < R; i += stride) {
    if (roff[i + 1] < roff[i] && nonmono == INT64_MAX) nonmono = i;
    if (i + 1 < R && row[i + 1] <= row[i] && noninc == INT64_MAX) noninc = i;
    rmin = min(rmin, (int64_t)row[i]);
    rmax = max(rmax, (int64_t)row[i]);
  }
  for (int64_t p = tid; p < ncol; p += stride) {
    cmin = min(cmin, (int64_t)col[p]);
    cmax = max(cmax, (int64_t)col[p]);
  }
  nonmono = block_reduce(nonmono, Min(), s_red);
  if (threadIdx.x == 0 && nonmono != INT64_MAX) amin_s(rep + kResNonMono, nonmono);
  noninc = block_reduce(noninc, Min(), s_red);
  if (threadIdx.x == 0 && noninc != INT64_MAX) amin_s(rep + kResRowNonInc, noninc);
  rmin = block_reduce(rmin, Min(), s_red);
  if (threadIdx.x == 0 && R) amin_s(rep + kResRowMin, rmin);
  rmax = block_reduce(rmax, Max(), s_red);
  if (threadIdx.x == 0 && R) amax_s(rep + kResRowMax, rmax);
  cmin = block_reduce(cmin, Min(), s_red);
  if (threadIdx.x == 0 && ncol) amin_s(rep + kResColMin, cmin);
  cmax = block_reduce(cmax, Max(), s_red);
  if (threadIdx.x == 0 && ncol) amax_s(rep + kResColMax, cmax);
  if (tid == 0) {
    rep[kResOff0] = roff[0];
    rep[kResOffLast] = roff[R];
  }
}

// tile.py:258-266: rows covered by [rid, rid + window_size) of every entry
__global__ void k_cover_entries(const int32_t* __restrict__ rwid, int64_t E, int32_t wsize, int64_t n_rows, uint8_t* cov) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rid = rwid[e];
    for (int64_t i = 0; i < wsize && rid + i < n_rows; ++i) cov[rid + i] = 1;
  }
}
__global__ void k_res_in_window(const int32_t* __restrict__ row, int64_t R, const uint8_t* __restrict__ cov, int64_t* rep) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x)
    if (cov[row[i]]) amin_s(rep + kResInWindow, i);
}

// tile.py:197-206: the first entry e that opens a group (rwid[e] != rwid[e-1]) whose row id already
// headed an earlier group.  Heads are sorted stably by row id (non-heads carry a sentinel key
// above every int32); in each run of equal keys all but the first are offenders, and the smallest
// such entry index is the reference's first report.
__global__ void k_head_keys(const int32_t* __restrict__ rwid, int64_t E, int64_t* keys, int64_t* idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    keys[e] = (e == 0 || rwid[e] != rwid[e - 1]) ? (int64_t)rwid[e] : INT64_MAX;
    idx[e] = e;
  }
}
__global__ void k_dup_sorted(const int64_t* __restrict__ keys, const int64_t* __restrict__ idx, int64_t E, int64_t* rep) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x)
    if (keys[i] != INT64_MAX && keys[i] == keys[i - 1]) amin_s(rep + kDupHead, idx[i]);
}

// ---- decode -------------------------------------------------------------------------------

__global__ void k_decode_tc(const int32_t* __restrict__ rwid, const int64_t* __restrict__ off, int64_t E,
                            const uint64_t* __restrict__ bm, const int32_t* __restrict__ col,
                            const int64_t* __restrict__ vstart, int64_t nb, int64_t n_cols, int64_t* keys, int32_t* idx) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rid = rwid[entry_of(off, E, b)];
    unsigned long long m = bm[b];
    int64_t v = vstart[b];
    while (m) {
      const int bit = __ffsll((long long)m) - 1;
      m &= m - 1;
      keys[v] = (rid + (bit >> 3)) * n_cols + col[b * 8 + (bit & 7)];
      idx[v] = (int32_t)v;
      ++v;
    }
  }
}
__global__ void k_decode_res(const int32_t* __restrict__ row, const int64_t* __restrict__ roff, int64_t R,
                             const int32_t* __restrict__ col, int64_t base, int64_t n_cols, int64_t* keys, int32_t* idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = roff[i]; p < roff[i + 1]; ++p) {
      keys[base + p] = (int64_t)row[i] * n_cols + col[p];
      idx[base + p] = (int32_t)(base + p);
    }
}
__global__ void k_decode_emit(const int64_t* __restrict__ keys, const int32_t* __restrict__ idx, int64_t nnz,
                              int64_t n_cols, const float* __restrict__ tc_vals, int64_t tc_nnz,
                              const float* __restrict__ res_vals, int32_t* out_col, float* out_val, int64_t* row_cnt,
                              int64_t* dup) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = keys[p];
    out_col[p] = (int32_t)(k % n_cols);
    const int32_t s = idx[p];
    out_val[p] = s < tc_nnz ? tc_vals[s] : res_vals[s - tc_nnz];
    atomicAdd((unsigned long long*)(row_cnt + k / n_cols), 1ull);
    if (p + 1 < nnz && keys[p + 1] == k) atomicMin((unsigned long long*)dup, (unsigned long long)p);
  }
}

}  // namespace rsh

using namespace rsh;

extern "C" {

int rsh_report_slots(void) { return kRepSlots; }

size_t rsh_validate_workspace(int64_t n_rows, int64_t n_entries, int64_t n_blocks) {
  Carve cv(nullptr);
  cv.take<int64_t>(n_blocks + 1);
  cv.take<int64_t>(n_blocks + 1);
  cv.take<uint8_t>(n_rows + 1);
  for (int i = 0; i < 4; ++i) cv.take<int64_t>(n_entries + 1);
  size_t a = 0, b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_blocks + 1));
  cub::DeviceRadixSort::SortPairs(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int64_t*)nullptr,
                                  (int64_t*)nullptr, (int)(n_entries + 1));
  cv.take<char>(a > b ? a : b);
  return cv.used + 256;
}

// tile.py:176-267: structural facts of a format into rep[rsh_report_slots()] (device int64).
// The caller has checked the two length preconditions the reference returns early on
// (offsets of length E+1 and R+1).  check_bits / check_cover gate the two checks the reference
// runs only on an otherwise clean format; the host runs a second pass with them set.
int rsh_validate(int64_t n_rows, int64_t n_cols, int32_t window_size, const int32_t* row_window_id,
                 const int64_t* row_window_offset, int64_t n_entries, const uint64_t* bitmaps, const int32_t* col_id,
                 int64_t n_col_id, int64_t n_blocks, int64_t n_values, const int32_t* res_row_id,
                 const int64_t* res_offset, int64_t n_res, const int32_t* res_col_id, int64_t n_res_col,
                 int32_t check_bits, int32_t check_cover, int64_t* rep, void* ws, size_t ws_bytes, cudaStream_t st) {
  (void)n_cols;
  size_t need = rsh_validate_workspace(n_rows, n_entries, n_blocks);
  if (!rep || !ws || ws_bytes < need) return fail(kInvalid, "rsh_validate: workspace too small");
  if (n_entries > INT32_MAX || n_blocks > INT32_MAX) return fail(kInvalid, "rsh_validate: format too large");
  Carve cv(ws);
  int64_t* pc = cv.take<int64_t>(n_blocks + 1);
  int64_t* cum = cv.take<int64_t>(n_blocks + 1);
  uint8_t* cov = cv.take<uint8_t>(n_rows + 1);
  int64_t* hk = cv.take<int64_t>(n_entries + 1);
  int64_t* hi = cv.take<int64_t>(n_entries + 1);
  int64_t* hk2 = cv.take<int64_t>(n_entries + 1);
  int64_t* hi2 = cv.take<int64_t>(n_entries + 1);
  size_t a = 0, b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_blocks + 1));
  cub::DeviceRadixSort::SortPairs(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int64_t*)nullptr,
                                  (int64_t*)nullptr, (int)(n_entries + 1));
  const size_t cb = a > b ? a : b;
  void* tmp = cv.take<char>(cb);
  const unsigned cap = 4 * sm_count();
  k_rep_init<<<1, 32, 0, st>>>(rep);
  unsigned g = grid_1d(n_col_id > n_blocks ? n_col_id : n_blocks);
  k_val_tc<<<g > cap ? cap : g, kThreads, 0, st>>>(row_window_id, row_window_offset, n_entries, bitmaps, n_blocks,
                                                   col_id, n_col_id, n_rows, window_size, check_bits, rep);
  RSH_LAUNCHED("k_val_tc");
  if (n_blocks) {
    k_popc64<<<grid_1d(n_blocks + 1), kThreads, 0, st>>>(bitmaps, n_blocks, pc);
    size_t t = cb;
    RSH_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t, pc, cum, (int)(n_blocks + 1), st));
    k_pop_over<<<grid_1d(n_blocks), kThreads, 0, st>>>(cum, n_blocks, n_values, rep);
  }
  g = grid_1d(n_res > n_res_col ? n_res : n_res_col);
  k_val_res<<<g > cap ? cap : g, kThreads, 0, st>>>(res_row_id, res_offset, n_res, res_col_id, n_res_col, rep);
  RSH_LAUNCHED("k_val_res");
  if (n_entries > 1) {
    k_head_keys<<<grid_1d(n_entries), kThreads, 0, st>>>(row_window_id, n_entries, hk, hi);
    size_t t = cb;
    RSH_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, hk, hk2, hi, hi2, (int)n_entries, 0, 64, st));
    k_dup_sorted<<<grid_1d(n_entries), kThreads, 0, st>>>(hk2, hi2, n_entries, rep);
  }
  if (check_cover && n_res && n_entries) {
    RSH_CUDA(cudaMemsetAsync(cov, 0, n_rows + 1, st));
    k_cover_entries<<<grid_1d(n_entries), kThreads, 0, st>>>(row_window_id, n_entries, window_size, n_rows, cov);
    k_res_in_window<<<grid_1d(n_res), kThreads, 0, st>>>(res_row_id, n_res, cov, rep);
  }
  RSH_LAUNCHED("validate");
  return kOk;
}

size_t rsh_decode_workspace(int64_t n_rows, int64_t nnz, int64_t n_blocks) {
  Carve cv(nullptr);
  cv.take<int64_t>(n_rows + 1);
  cv.take<int64_t>(n_blocks + 1);
  cv.take<int64_t>(n_blocks + 1);
  cv.take<int64_t>(nnz + 1);
  cv.take<int64_t>(nnz + 1);
  cv.take<int32_t>(nnz + 1);
  cv.take<int32_t>(nnz + 1);
  size_t a = 0, b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_blocks + 1));
  cub::DeviceRadixSort::SortPairs(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)(nnz + 1));
  size_t c = 0;
  cub::DeviceScan::InclusiveSum(nullptr, c, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_rows + 1));
  a = a > b ? a : b;
  cv.take<char>(a > c ? a : c);
  return cv.used + 256;
}

// tile.py:270-307 on a VALID format: out_row_ptr[n_rows+1], out_col_idx[nnz], out_values[nnz]
// (nnz = tc values + residual nnz); dup_out[0] = first position of a duplicate (row, col), or
// UINT64_MAX when the decoded triples are canonical.
int rsh_decode(int64_t n_rows, int64_t n_cols, const int32_t* row_window_id, const int64_t* row_window_offset,
               int64_t n_entries, const uint64_t* bitmaps, const int32_t* col_id, const float* tc_values,
               int64_t n_blocks, int64_t tc_nnz, const int32_t* res_row_id, const int64_t* res_offset, int64_t n_res,
               const int32_t* res_col_id, const float* res_values, int64_t res_nnz, int64_t* out_row_ptr,
               int32_t* out_col_idx, float* out_values, int64_t* dup_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int64_t nnz = tc_nnz + res_nnz;
  size_t need = rsh_decode_workspace(n_rows, nnz, n_blocks);
  if (!ws || ws_bytes < need) return fail(kInvalid, "rsh_decode: workspace too small");
  if (n_cols > 0 && n_rows > (INT64_MAX / n_cols)) return fail(kInvalid, "rsh_decode: key overflow");
  Carve cv(ws);
  int64_t* rcnt = cv.take<int64_t>(n_rows + 1);
  int64_t* pc = cv.take<int64_t>(n_blocks + 1);
  int64_t* vstart = cv.take<int64_t>(n_blocks + 1);
  int64_t* keys = cv.take<int64_t>(nnz + 1);
  int64_t* keys2 = cv.take<int64_t>(nnz + 1);
  int32_t* idx = cv.take<int32_t>(nnz + 1);
  int32_t* idx2 = cv.take<int32_t>(nnz + 1);
  size_t a = 0, b = 0, c = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_blocks + 1));
  cub::DeviceRadixSort::SortPairs(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)(nnz + 1));
  cub::DeviceScan::InclusiveSum(nullptr, c, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_rows + 1));
  size_t cb = a > b ? a : b;
  cb = cb > c ? cb : c;
  void* tmp = cv.take<char>(cb);
  RSH_CUDA(cudaMemsetAsync(dup_out, 0xff, sizeof(int64_t), st));
  RSH_CUDA(cudaMemsetAsync(out_row_ptr, 0, (n_rows + 1) * sizeof(int64_t), st));
  RSH_CUDA(cudaMemsetAsync(rcnt, 0, (n_rows + 1) * sizeof(int64_t), st));
  k_popc64<<<grid_1d(n_blocks + 1), kThreads, 0, st>>>(bitmaps, n_blocks, pc);
  size_t t = cb;
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t, pc, vstart, (int)(n_blocks + 1), st));
  if (n_blocks && n_entries)
    k_decode_tc<<<grid_1d(n_blocks), kThreads, 0, st>>>(row_window_id, row_window_offset, n_entries, bitmaps, col_id,
                                                         vstart, n_blocks, n_cols, keys, idx);
  if (n_res) k_decode_res<<<grid_1d(n_res), kThreads, 0, st>>>(res_row_id, res_offset, n_res, res_col_id, tc_nnz, n_cols, keys, idx);
  RSH_LAUNCHED("decode expand");
  if (nnz) {
    t = cb;
    RSH_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, keys, keys2, idx, idx2, (int)nnz, 0, 64, st));
    k_decode_emit<<<grid_1d(nnz), kThreads, 0, st>>>(keys2, idx2, nnz, n_cols, tc_values, tc_nnz, res_values,
                                                     out_col_idx, out_values, rcnt, dup_out);
    RSH_LAUNCHED("decode emit");
  }
  if (n_rows) {
    t = cb;
    RSH_CUDA(cub::DeviceScan::InclusiveSum(tmp, t, rcnt, out_row_ptr + 1, (int)n_rows, st));
  }
  return kOk;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// core.py:380-395 oracle_spmm: C = A @ B from the CSR, every row accumulated in f64 in CSR order
// (values and B widened to f64 exactly, as the reference's astype(np.float64)), stored as f32;
// rows without nonzeros are zero.  Warp per row, lanes across features.
// ---------------------------------------------------------------------------------------------
namespace rsh {
__global__ void k_csr_spmm_f64(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               const float* __restrict__ v, int64_t n_rows, const float* __restrict__ B, int64_t ldb,
                               int64_t N, float* __restrict__ C, int64_t ldc) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n_rows; r += nw) {
    const int64_t s = rp[r], e = rp[r + 1];
    for (int64_t f = lane; f < N; f += 32) {
      double acc = 0.0;
      for (int64_t p = s; p < e; ++p) acc += (double)__ldg(v + p) * (double)__ldg(B + (int64_t)__ldg(ci + p) * ldb + f);
      C[r * ldc + f] = (float)acc;
    }
  }
}

// metrics.py:28-63 tile_density: one thread per row-window head (consecutive equal row_window_id
// are one window, tile.py segments); the OR of the window's blocks' row bytes gives its occupied
// rows.  out[0] += windows, out[1] += occupied window rows.
__global__ void k_tile_density(const int32_t* __restrict__ rwid, const int64_t* __restrict__ off, int64_t E,
                               const unsigned long long* __restrict__ bm, unsigned long long* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E) return;
  if (e > 0 && rwid[e] == rwid[e - 1]) return;
  int64_t e2 = e + 1;
  while (e2 < E && rwid[e2] == rwid[e]) ++e2;
  unsigned long long acc = 0;
  for (int64_t b = off[e]; b < off[e2]; ++b) acc |= bm[b];
  uint32_t rows = 0;
  for (int i = 0; i < 8; ++i) rows += ((acc >> (8 * i)) & 0xffull) != 0;
  atomicAdd(out, 1ull);
  atomicAdd(out + 1, (unsigned long long)rows);
}
}  // namespace rsh

extern "C" {

int rsh_csr_spmm_f64(const int64_t* row_ptr, const int32_t* col_idx, const float* values, int64_t n_rows,
                     const float* B, int64_t ldb, int64_t N, float* C, int64_t ldc, cudaStream_t st) {
  if (n_rows < 0 || N < 0 || ldb < N || ldc < N) return rsh::fail(rsh::kInvalid, "rsh_csr_spmm_f64: bad shape");
  if (n_rows == 0 || N == 0) return rsh::kOk;
  if (!row_ptr || !B || !C) return rsh::fail(rsh::kInvalid, "rsh_csr_spmm_f64: null operand");
  int64_t blocks = (n_rows + 7) / 8;
  const int64_t cap = 32LL * rsh::sm_count();
  if (blocks > cap) blocks = cap;
  rsh::k_csr_spmm_f64<<<(unsigned)blocks, 256, 0, st>>>(row_ptr, col_idx, values, n_rows, B, ldb, N, C, ldc);
  RSH_LAUNCHED("k_csr_spmm_f64");
  return rsh::kOk;
}

// out (device uint64[2]) = [windows, occupied window rows]
int rsh_tile_density(const int32_t* row_window_id, const int64_t* row_window_offset, int64_t n_entries,
                     const uint64_t* bitmaps, unsigned long long* out, cudaStream_t st) {
  if (!out) return rsh::fail(rsh::kInvalid, "rsh_tile_density: null output");
  if (n_entries > 0 && (!row_window_id || !row_window_offset || !bitmaps))
    return rsh::fail(rsh::kInvalid, "rsh_tile_density: null format array");
  RSH_CUDA(cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), st));
  if (n_entries <= 0) return rsh::kOk;
  rsh::k_tile_density<<<rsh::grid_1d(n_entries), rsh::kThreads, 0, st>>>(
      row_window_id, row_window_offset, n_entries, (const unsigned long long*)bitmaps, out);
  RSH_LAUNCHED("k_tile_density");
  return rsh::kOk;
}

}  // extern "C"
