// On-device row classifier, partition scan and RS-Tile builder (north-star subsystem (1)).
//
// Reference algorithm (rstile 0.1.0, /root/reference/pkg/src/rstile):
//   partition.py:101-116  column_increment      -> k_classify (delta only where it can matter)
//   partition.py:119-141  partition_rows        -> k_tile_maps / k_scan_tiles / k_visit + select
//   partition.py:144-180  window_columns/split  -> k_first_flags + scan + k_window_blocks, k_split
//   tile.py:102-173       build_rstile          -> k_slots (bitmaps, col_id), popcount scan,
//                                                  k_values, k_entries, residual offsets/gather
// The sequential scan of partition.py becomes an exclusive scan over per-row state automata
// (state = rows still to skip inside the current window), which is associative, so the whole
// partition is three grid passes plus two stream compactions.  Window column compaction needs
// no sort: an element is the "first occurrence" of its column if no earlier row of the window
// holds it; the compact rank of column c is then sum_j #firsts(row j, < c), read off a single
// global prefix sum of the first-occurrence flags with one binary search per window row.
// Values land at vstart[blk] + popc(bitmap & below(bit)), which is exactly the
// lexsort((bit, blk)) order of tile.py:123.  Every output is bit-exact with the reference.
#include "common.cuh"
#include <cub/cub.cuh>

namespace rsh {

constexpr int kEmpty = 0, kResid = 1, kHead = 2;
constexpr int kRowsPerThread = 16;
constexpr int kTileRows = kThreads * kRowsPerThread;  // 4096 rows per scan tile
constexpr int kElemsPerThread = 8;

// ------------------------------------------------------------------------------------------
// classification (partition.py:101-116, 129-137)
// ------------------------------------------------------------------------------------------

// kind = RESID  <=>  nz <= tau_nnz && delta < tau_inc, with delta = #head columns absent from
// rows r+1 .. min(r+W, n)-1.  delta <= nz, so nz < tau_inc already decides RESID, and the
// count can stop once it reaches tau_inc.  Interior window rows get a kind too; the scan only
// consults the kinds of rows it visits, exactly as the reference only tests visited rows.
__global__ void k_classify(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n,
                           int W, int64_t tau_nnz, int64_t tau_inc, uint8_t* __restrict__ kind) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = rp[r], e = rp[r + 1], nz = e - s;
    uint8_t k;
    if (nz == 0) k = kEmpty;
    else if (nz > tau_nnz) k = kHead;
    else if (nz < tau_inc) k = kResid;
    else {
      int64_t end = r + W < n ? r + W : n;
      int64_t missing = 0;
      for (int64_t p = s; p < e && missing < tau_inc; ++p) {
        int32_t c = ci[p];
        bool found = false;
        for (int64_t t = r + 1; t < end && !found; ++t) found = row_has(rp, ci, t, c);
        missing += !found;
      }
      k = missing < tau_inc ? kResid : kHead;
    }
    kind[r] = k;
  }
}

// ------------------------------------------------------------------------------------------
// partition scan (partition.py:127-140)
// ------------------------------------------------------------------------------------------
// A map packs next_state(s) for s = 0..7 in 3-bit fields.  Row r's map is
//   head row:  s > 0 ? s-1 : W-1      other rows:  s > 0 ? s-1 : 0
// and a row is visited by the reference scan iff the state entering it is 0.

__device__ __forceinline__ uint32_t map_identity() {
  uint32_t m = 0;
#pragma unroll
  for (int s = 0; s < 8; ++s) m |= uint32_t(s) << (3 * s);
  return m;
}
__device__ __forceinline__ uint32_t map_row(bool head, int W) {
  uint32_t m = uint32_t(head ? W - 1 : 0);
#pragma unroll
  for (int s = 1; s < 8; ++s) m |= uint32_t(s - 1) << (3 * s);
  return m;
}
__device__ __forceinline__ uint32_t map_apply(uint32_t m, uint32_t s) { return (m >> (3 * s)) & 7u; }
// first a, then b
__device__ __forceinline__ uint32_t map_then(uint32_t a, uint32_t b) {
  uint32_t out = 0;
#pragma unroll
  for (int s = 0; s < 8; ++s) out |= map_apply(b, map_apply(a, s)) << (3 * s);
  return out;
}

// exclusive scan of maps over the block (thread order); returns this thread's prefix,
// *total gets the composition of all threads' maps.
__device__ uint32_t block_scan_maps(uint32_t m, uint32_t* total) {
  __shared__ uint32_t warp_tot[kThreads / 32];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = m;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc = map_then(o, inc);
  }
  uint32_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) exc = map_identity();
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  uint32_t before = map_identity();
  for (int w = 0; w < warp; ++w) before = map_then(before, warp_tot[w]);
  if (total) {
    uint32_t t = map_identity();
    for (int w = 0; w < kThreads / 32; ++w) t = map_then(t, warp_tot[w]);
    *total = t;
  }
  __syncthreads();
  return map_then(before, exc);
}

__device__ __forceinline__ uint32_t thread_rows_map(const uint8_t* __restrict__ kind, int64_t n, int W,
                                                    int64_t r0) {
  uint32_t m = map_identity();
#pragma unroll
  for (int k = 0; k < kRowsPerThread; ++k) {
    int64_t r = r0 + k;
    if (r < n) m = map_then(m, map_row(kind[r] == kHead, W));
  }
  return m;
}

__global__ void k_tile_maps(const uint8_t* __restrict__ kind, int64_t n, int W, uint32_t* tile_map) {
  int64_t r0 = (int64_t)blockIdx.x * kTileRows + (int64_t)threadIdx.x * kRowsPerThread;
  uint32_t tot;
  block_scan_maps(thread_rows_map(kind, n, W, r0), &tot);
  if (threadIdx.x == 0) tile_map[blockIdx.x] = tot;
}

// one block: state entering each tile, starting from state 0 at row 0
__global__ void k_scan_tiles(const uint32_t* __restrict__ tile_map, int64_t n_tiles, uint8_t* state_in) {
  int64_t per = (n_tiles + kThreads - 1) / kThreads;
  int64_t t0 = threadIdx.x * per, t1 = t0 + per < n_tiles ? t0 + per : n_tiles;
  uint32_t m = map_identity();
  for (int64_t t = t0; t < t1; ++t) m = map_then(m, tile_map[t]);
  uint32_t pre = block_scan_maps(m, nullptr);
  uint32_t s = map_apply(pre, 0);
  for (int64_t t = t0; t < t1; ++t) {
    state_in[t] = (uint8_t)s;
    s = map_apply(tile_map[t], s);
  }
}

__global__ void k_visit(const uint8_t* __restrict__ kind, int64_t n, int W, const uint8_t* __restrict__ state_in,
                        uint8_t* head_flag, uint8_t* resid_flag) {
  int64_t r0 = (int64_t)blockIdx.x * kTileRows + (int64_t)threadIdx.x * kRowsPerThread;
  uint32_t pre = block_scan_maps(thread_rows_map(kind, n, W, r0), nullptr);
  uint32_t s = map_apply(pre, state_in[blockIdx.x]);
#pragma unroll
  for (int k = 0; k < kRowsPerThread; ++k) {
    int64_t r = r0 + k;
    if (r < n) {
      uint8_t kd = kind[r];
      head_flag[r] = (s == 0 && kd == kHead);
      resid_flag[r] = (s == 0 && kd == kResid);
      s = map_apply(map_row(kd == kHead, W), s);
    }
  }
}

// ------------------------------------------------------------------------------------------
// window column planning (partition.py:144-146, 167)
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ int64_t win_rows(int64_t start, int W, int64_t n) {
  return W < n - start ? W : n - start;
}
// rows of window w: explicit counts when the caller has them (arbitrary valid plans), else the
// (start, min(W, n - start)) windows partition_rows emits (partition.py:139)
__device__ __forceinline__ int64_t win_cnt(const int32_t* __restrict__ wc, int64_t w, int64_t start, int W, int64_t n) {
  return wc ? (int64_t)wc[w] : win_rows(start, W, n);
}

__global__ void k_mark_rows(const int32_t* __restrict__ win_start, const int32_t* __restrict__ win_count,
                            int64_t n_win, int W, int64_t n, int32_t* row_win) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_win; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = win_start[w], c = win_cnt(win_count, w, s, W, n);
    for (int64_t i = 0; i < c; ++i) row_win[s + i] = (int32_t)w;
  }
}

// first[p] = 1 iff p lies in a window row and no earlier row of that window holds its column;
// flags cover positions 0..nnz (the extra slot stays 0 so the exclusive scan ends in the total)
__global__ void k_first_flags(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n,
                              int64_t nnz, const int32_t* __restrict__ row_win,
                              const int32_t* __restrict__ win_start, int32_t* first) {
  int64_t p0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kElemsPerThread;
  if (p0 > nnz) return;
  if (p0 == nnz) { first[nnz] = 0; return; }
  int64_t p1 = p0 + kElemsPerThread < nnz ? p0 + kElemsPerThread : nnz;
  int64_t r = row_of(rp, n, p0);
  for (int64_t p = p0; p < p1; ++p) {
    while (rp[r + 1] <= p) ++r;
    int32_t w = row_win[r];
    int32_t f = 0;
    if (w >= 0) {
      int32_t c = ci[p];
      f = 1;
      for (int64_t j = win_start[w]; j < r && f; ++j) f = !row_has(rp, ci, j, c);
    }
    first[p] = f;
  }
  if (p1 == nnz && p0 < nnz) first[nnz] = 0;
}

__global__ void k_window_blocks(const int64_t* __restrict__ rp, int64_t n, int W,
                                const int32_t* __restrict__ win_start, const int32_t* __restrict__ win_count,
                                int64_t n_win, const int32_t* __restrict__ prefix, int64_t* nblocks,
                                int64_t* longest) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_win; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = win_start[w], c = win_cnt(win_count, w, s, W, n);
    int64_t distinct = (int64_t)prefix[rp[s + c]] - prefix[rp[s]];
    nblocks[w] = (distinct + 7) / 8;
    int64_t lg = 0;
    for (int64_t i = 0; i < c; ++i) {
      int64_t z = rp[s + i + 1] - rp[s + i];
      lg = z > lg ? z : lg;
    }
    longest[w] = lg;
  }
}

// ------------------------------------------------------------------------------------------
// split_long_work (partition.py:149-180)
// ------------------------------------------------------------------------------------------

__global__ void k_split(const int64_t* __restrict__ nblocks, const int64_t* __restrict__ longest, int64_t n_win,
                        int64_t bound, int on_row_nnz, double factor, double mean, int64_t* chunk,
                        int64_t* n_seg) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_win; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t nb = nblocks[w], ch = 0;
    if (bound > 0 && nb > bound) {
      ch = bound;
    } else if (on_row_nnz && nb > 1 && mean > 0.0) {
      double cap = factor * mean;
      int64_t lg = longest[w];
      if ((double)lg > cap) {
        int64_t pieces = (int64_t)ceil((double)lg / cap);
        int64_t c2 = (nb + pieces - 1) / pieces;
        ch = c2 > 1 ? c2 : 1;
      }
    }
    if (!(ch && ch < nb)) ch = 0;
    chunk[w] = ch;
    n_seg[w] = ch ? (nb + ch - 1) / ch : 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) n_seg[n_win] = 0;
}

__global__ void k_copy_tail0(const int64_t* __restrict__ src, int64_t n, int64_t* dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = i < n ? src[i] : 0;
}

// ------------------------------------------------------------------------------------------
// build (tile.py:115-144)
// ------------------------------------------------------------------------------------------

// compact rank of column c inside window w = #distinct window columns < c
__device__ __forceinline__ int64_t window_rank(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                               const int32_t* __restrict__ prefix, int64_t s, int64_t cnt,
                                               int32_t c) {
  int64_t rank = 0;
  for (int64_t j = s; j < s + cnt; ++j) {
    int64_t a = rp[j], b = rp[j + 1];
    int64_t k = lower_bound(ci + a, b - a, c);
    rank += (int64_t)prefix[a + k] - prefix[a];
  }
  return rank;
}

__global__ void k_slots(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n, int64_t nnz,
                        int W, const int32_t* __restrict__ row_win, const int32_t* __restrict__ win_start,
                        const int32_t* __restrict__ win_count,
                        const int32_t* __restrict__ prefix, const int64_t* __restrict__ block_base,
                        unsigned long long* bitmaps, int32_t* col_id, uint32_t* slot) {
  int64_t p0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kElemsPerThread;
  if (p0 >= nnz) return;
  int64_t p1 = p0 + kElemsPerThread < nnz ? p0 + kElemsPerThread : nnz;
  int64_t r = row_of(rp, n, p0);
  for (int64_t p = p0; p < p1; ++p) {
    while (rp[r + 1] <= p) ++r;
    int32_t w = row_win[r];
    if (w < 0) continue;
    int64_t s = win_start[w];
    int32_t c = ci[p];
    int64_t rank = window_rank(rp, ci, prefix, s, win_cnt(win_count, w, s, W, n), c);
    int64_t blk = block_base[w] + (rank >> 3);
    int bit = int(r - s) * 8 + int(rank & 7);
    atomicOr(bitmaps + blk, 1ull << bit);
    int64_t sl = blk * 8 + (rank & 7);
    if (prefix[p + 1] - prefix[p]) col_id[sl] = c;
    slot[p] = (uint32_t)sl;
  }
}

__global__ void k_popc(const unsigned long long* __restrict__ bm, int64_t nb, int32_t* pc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nb; i += (int64_t)gridDim.x * blockDim.x)
    pc[i] = i < nb ? __popcll(bm[i]) : 0;
}

__global__ void k_values(const int64_t* __restrict__ rp, const float* __restrict__ vals, int64_t n, int64_t nnz,
                         const int32_t* __restrict__ row_win, const int32_t* __restrict__ win_start,
                         const uint32_t* __restrict__ slot, const unsigned long long* __restrict__ bitmaps,
                         const int32_t* __restrict__ vstart, float* tc_values) {
  int64_t p0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kElemsPerThread;
  if (p0 >= nnz) return;
  int64_t p1 = p0 + kElemsPerThread < nnz ? p0 + kElemsPerThread : nnz;
  int64_t r = row_of(rp, n, p0);
  for (int64_t p = p0; p < p1; ++p) {
    while (rp[r + 1] <= p) ++r;
    int32_t w = row_win[r];
    if (w < 0) continue;
    int64_t sl = slot[p];
    int64_t blk = sl >> 3;
    int bit = int(r - win_start[w]) * 8 + int(sl & 7);
    unsigned long long below = bit ? (bitmaps[blk] & ((1ull << bit) - 1ull)) : 0ull;
    tc_values[vstart[blk] + __popcll(below)] = vals[p];
  }
}

__global__ void k_entries(const int32_t* __restrict__ win_start, int64_t n_win, const int64_t* __restrict__ block_base,
                          const int64_t* __restrict__ chunk, const int64_t* __restrict__ entry_base,
                          int32_t* rwid, int64_t* rwoff) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_win; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t e0 = entry_base[w], e1 = entry_base[w + 1], ch = chunk[w];
    for (int64_t e = e0; e < e1; ++e) {
      rwid[e] = win_start[w];
      rwoff[e] = block_base[w] + (e - e0) * ch;
    }
    if (w == n_win - 1) rwoff[e1] = block_base[n_win];
  }
  if (n_win == 0 && blockIdx.x == 0 && threadIdx.x == 0) rwoff[0] = 0;
}

// ------------------------------------------------------------------------------------------
// residual part (tile.py:146-165)
// ------------------------------------------------------------------------------------------

__global__ void k_res_counts(const int64_t* __restrict__ rp, const int32_t* __restrict__ rows, int64_t nr,
                             int64_t* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nr; i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = i < nr ? rp[rows[i] + 1] - rp[rows[i]] : 0;
}

__global__ void k_res_gather(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                             const float* __restrict__ vals, const int32_t* __restrict__ rows, int64_t nr,
                             const int64_t* __restrict__ off, int32_t* out_col, float* out_val) {
  int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < nr;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t s = rp[rows[i]], e = rp[rows[i] + 1], o = off[i];
    for (int64_t p = s + lane; p < e; p += 32) {
      out_col[o + p - s] = ci[p];
      out_val[o + p - s] = vals[p];
    }
  }
}

}  // namespace rsh

// ==========================================================================================
// C ABI
// ==========================================================================================
using namespace rsh;

namespace {

struct PartitionWs {
  uint8_t *kind, *head, *resid, *state_in;
  uint32_t* tile_map;
  void* cub;
  size_t cub_bytes;
};

size_t partition_layout(void* base, int64_t n, PartitionWs* o) {
  Carve cv(base);
  int64_t tiles = (n + kTileRows - 1) / kTileRows;
  o->kind = cv.take<uint8_t>(n);
  o->head = cv.take<uint8_t>(n);
  o->resid = cv.take<uint8_t>(n);
  o->state_in = cv.take<uint8_t>(tiles);
  o->tile_map = cv.take<uint32_t>(tiles);
  size_t cb = 0;
  cub::DeviceSelect::Flagged(nullptr, cb, cub::CountingInputIterator<int32_t>(0), (uint8_t*)nullptr,
                             (int32_t*)nullptr, (int64_t*)nullptr, (int)(n > 0 ? n : 1));
  o->cub_bytes = cb;
  o->cub = cv.take<char>(cb);
  return cv.used + 256;
}

}  // namespace

namespace rsh {

// ------------------------------------------------------------------------------------------
// transpose (for the GNN backward pass): A^T as a canonical CSR.  A stable radix
// sort of the nonzeros by column keeps them in row order inside every column, so each row of
// A^T lists its columns (A's rows) strictly increasing -- the canonical CSR the builder expects.
// ------------------------------------------------------------------------------------------

__global__ void k_row_ids(const int64_t* __restrict__ rp, int64_t n_rows, int32_t* rid) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = rp[r]; p < rp[r + 1]; ++p) rid[p] = (int32_t)r;
}

__global__ void k_iota32(int32_t* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (int32_t)i;
}

__global__ void k_col_counts(const int32_t* __restrict__ col, int64_t nnz, int64_t* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)(cnt + col[i]), 1ull);
}

__global__ void k_transpose_gather(const int32_t* __restrict__ perm, const int32_t* __restrict__ rid,
                                   const float* __restrict__ values, int64_t nnz, int32_t* out_col, float* out_val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = perm[i];
    out_col[i] = rid[p];
    out_val[i] = values[p];
  }
}

}  // namespace rsh

namespace rsh {
__global__ void k_window_nnz(const int64_t* __restrict__ rp, int64_t n_rows, const int32_t* __restrict__ ws,
                             const int32_t* __restrict__ wc, int64_t n_win, int32_t window_size,
                             unsigned long long* out) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long v = 0;
  if (w < n_win) {
    const int64_t s = ws[w];
    int64_t c = wc ? (int64_t)wc[w] : (n_rows - s < window_size ? n_rows - s : window_size);
    v = (unsigned long long)(rp[s + c] - rp[s]);
  }
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}
}  // namespace rsh

extern "C" {

size_t rsh_partition_workspace(int64_t n_rows) {
  PartitionWs w;
  return partition_layout(nullptr, n_rows, &w);
}

// partition.py:119-141 (+ column_increment :101-116).  win_start / resid_rows need capacity
// n_rows; counts[0] = #windows, counts[1] = #residual rows (device int64[2]).
int rsh_partition(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int32_t window_size,
                  int64_t tau_nnz, int64_t tau_inc, int32_t* win_start, int32_t* resid_rows,
                  int64_t* counts, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n_rows < 0 || window_size < 1 || window_size > 8 || tau_nnz < 0 || tau_inc < 0)
    return fail(kInvalid, "rsh_partition: bad arguments (n_rows=%lld W=%d tau=(%lld,%lld))",
                (long long)n_rows, window_size, (long long)tau_nnz, (long long)tau_inc);
  if (n_rows >= (1LL << 31)) return fail(kInvalid, "rsh_partition: n_rows exceeds the 32-bit index limit");
  if (n_rows == 0) {
    RSH_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), st));
    return kOk;
  }
  PartitionWs w;
  size_t need = partition_layout(ws, n_rows, &w);
  if (!ws || ws_bytes < need) return fail(kInvalid, "rsh_partition: workspace %zu < %zu bytes", ws_bytes, need);
  int64_t tiles = (n_rows + kTileRows - 1) / kTileRows;
  k_classify<<<grid_1d(n_rows), kThreads, 0, st>>>(row_ptr, col_idx, n_rows, window_size, tau_nnz, tau_inc, w.kind);
  k_tile_maps<<<(unsigned)tiles, kThreads, 0, st>>>(w.kind, n_rows, window_size, w.tile_map);
  k_scan_tiles<<<1, kThreads, 0, st>>>(w.tile_map, tiles, w.state_in);
  k_visit<<<(unsigned)tiles, kThreads, 0, st>>>(w.kind, n_rows, window_size, w.state_in, w.head, w.resid);
  RSH_LAUNCHED("partition kernels");
  size_t cb = w.cub_bytes;
  RSH_CUDA(cub::DeviceSelect::Flagged(w.cub, cb, cub::CountingInputIterator<int32_t>(0), w.head, win_start,
                                      counts, (int)n_rows, st));
  RSH_CUDA(cub::DeviceSelect::Flagged(w.cub, cb, cub::CountingInputIterator<int32_t>(0), w.resid, resid_rows,
                                      counts + 1, (int)n_rows, st));
  return kOk;
}

// --- window planning ------------------------------------------------------------------------

size_t rsh_plan_workspace(int64_t n_rows, int64_t nnz, int64_t n_win) {
  Carve cv(nullptr);
  cv.take<int32_t>(n_rows);         // row_win
  cv.take<int32_t>(nnz + 1);        // first flags
  cv.take<int64_t>(n_win + 1);      // n_seg / scratch
  size_t a = 0, b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int)(nnz + 1));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_win + 1));
  cv.take<char>(a > b ? a : b);
  return cv.used + 256;
}

// Window columns (partition.py:144-146): prefix[0..nnz] = exclusive scan of first-occurrence
// flags (caller buffer, reused by rsh_build_fill); row_win[n_rows] maps rows to windows (caller
// buffer, reused); nblocks[w] = ceil(distinct/8) (partition.py:167); longest[w] = max row nnz.
// Then split_long_work (partition.py:149-180): chunk[w] (0 = unsplit), entry_base[0..n_win] and
// block_base[0..n_win] are exclusive scans of segment and block counts.
int rsh_plan_windows(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t nnz,
                     int32_t window_size, const int32_t* win_start, const int32_t* win_count, int64_t n_win,
                     int64_t max_blocks_per_item,
                     int32_t split_on_row_nnz, double split_factor, int32_t* row_win, int32_t* prefix,
                     int64_t* nblocks, int64_t* longest, int64_t* chunk, int64_t* entry_base,
                     int64_t* block_base, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n_rows < 0 || nnz < 0 || n_win < 0 || window_size < 1 || window_size > 8)
    return fail(kInvalid, "rsh_plan_windows: bad arguments");
  // prefix[] and the cub scans index nonzeros with int32 (the reference's INDEX_LIMIT, core.py)
  if (nnz + 1 >= (1LL << 31) || n_rows >= (1LL << 31))
    return fail(kInvalid, "rsh_plan_windows: %lld nonzeros exceed the 32-bit index limit", (long long)nnz);
  size_t need = rsh_plan_workspace(n_rows, nnz, n_win);
  if (!ws || ws_bytes < need) return fail(kInvalid, "rsh_plan_windows: workspace %zu < %zu bytes", ws_bytes, need);
  Carve cv(ws);
  cv.take<int32_t>(n_rows);
  int32_t* first = cv.take<int32_t>(nnz + 1);
  int64_t* nseg = cv.take<int64_t>(n_win + 1);
  size_t a = 0, b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int)(nnz + 1));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_win + 1));
  size_t cb = a > b ? a : b;
  void* cubtmp = cv.take<char>(cb);

  if (n_rows) RSH_CUDA(cudaMemsetAsync(row_win, 0xff, n_rows * sizeof(int32_t), st));
  if (n_win) k_mark_rows<<<grid_1d(n_win), kThreads, 0, st>>>(win_start, win_count, n_win, window_size, n_rows, row_win);
  k_first_flags<<<grid_1d(nnz / kElemsPerThread + 1), kThreads, 0, st>>>(row_ptr, col_idx, n_rows, nnz, row_win,
                                                                          win_start, first);
  RSH_LAUNCHED("k_first_flags");
  size_t t = cb;
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, t, first, prefix, (int)(nnz + 1), st));
  if (n_win) {
    k_window_blocks<<<grid_1d(n_win), kThreads, 0, st>>>(row_ptr, n_rows, window_size, win_start, win_count,
                                                          n_win, prefix, nblocks, longest);
  }
  double mean = n_rows ? (double)nnz / (double)n_rows : 0.0;
  k_split<<<grid_1d(n_win + 1), kThreads, 0, st>>>(nblocks, longest, n_win, max_blocks_per_item, split_on_row_nnz,
                                                    split_factor, mean, chunk, nseg);
  RSH_LAUNCHED("k_split");
  t = cb;
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, t, nseg, entry_base, (int)(n_win + 1), st));
  k_copy_tail0<<<grid_1d(n_win + 1), kThreads, 0, st>>>(nblocks, n_win, nseg);
  RSH_LAUNCHED("k_copy_tail0");
  t = cb;
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, t, nseg, block_base, (int)(n_win + 1), st));
  return kOk;
}

// --- fill ---------------------------------------------------------------------------------

size_t rsh_fill_workspace(int64_t nnz, int64_t n_blocks) {
  Carve cv(nullptr);
  cv.take<uint32_t>(nnz);
  cv.take<int32_t>(n_blocks + 1);
  cv.take<int32_t>(n_blocks + 1);
  size_t a = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int)(n_blocks + 1));
  cv.take<char>(a);
  return cv.used + 256;
}

// tile.py:115-144.  Writes bitmaps[n_blocks], col_id[8*n_blocks], tc_values[window nnz] and,
// when chunk != NULL, the entry arrays row_window_id[n_entries], row_window_offset[n_entries+1]
// (with chunk == NULL the caller supplies explicit segments itself).
int rsh_build_fill(const int64_t* row_ptr, const int32_t* col_idx, const float* values, int64_t n_rows,
                   int64_t nnz, int32_t window_size, const int32_t* win_start, const int32_t* win_count,
                   int64_t n_win, const int32_t* row_win, const int32_t* prefix, const int64_t* block_base, int64_t n_blocks,
                   const int64_t* chunk, const int64_t* entry_base, int32_t* row_window_id,
                   int64_t* row_window_offset, uint64_t* bitmaps, int32_t* col_id, float* tc_values, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  if (n_blocks < 0 || 8 * n_blocks >= (1LL << 32))
    return fail(kInvalid, "rsh_build_fill: %lld blocks exceed the 32-bit slot limit", (long long)n_blocks);
  if (nnz < 0 || nnz + 1 >= (1LL << 31))
    return fail(kInvalid, "rsh_build_fill: %lld nonzeros exceed the 32-bit index limit", (long long)nnz);
  size_t need = rsh_fill_workspace(nnz, n_blocks);
  if (!ws || ws_bytes < need) return fail(kInvalid, "rsh_build_fill: workspace %zu < %zu bytes", ws_bytes, need);
  Carve cv(ws);
  uint32_t* slot = cv.take<uint32_t>(nnz);
  int32_t* pc = cv.take<int32_t>(n_blocks + 1);
  int32_t* vstart = cv.take<int32_t>(n_blocks + 1);
  size_t cb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cb, (int32_t*)nullptr, (int32_t*)nullptr, (int)(n_blocks + 1));
  void* cubtmp = cv.take<char>(cb);
  if (n_blocks) {
    RSH_CUDA(cudaMemsetAsync(bitmaps, 0, n_blocks * sizeof(uint64_t), st));
    RSH_CUDA(cudaMemsetAsync(col_id, 0, 8 * n_blocks * sizeof(int32_t), st));
  }
  if (nnz && n_win) {
    k_slots<<<grid_1d(nnz / kElemsPerThread + 1), kThreads, 0, st>>>(
        row_ptr, col_idx, n_rows, nnz, window_size, row_win, win_start, win_count, prefix, block_base,
        (unsigned long long*)bitmaps, col_id, slot);
    RSH_LAUNCHED("k_slots");
    k_popc<<<grid_1d(n_blocks + 1), kThreads, 0, st>>>((const unsigned long long*)bitmaps, n_blocks, pc);
    size_t t = cb;
    RSH_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, t, pc, vstart, (int)(n_blocks + 1), st));
    k_values<<<grid_1d(nnz / kElemsPerThread + 1), kThreads, 0, st>>>(
        row_ptr, values, n_rows, nnz, row_win, win_start, slot, (const unsigned long long*)bitmaps, vstart,
        tc_values);
    RSH_LAUNCHED("k_values");
  }
  if (chunk && n_win) {
    k_entries<<<grid_1d(n_win), kThreads, 0, st>>>(win_start, n_win, block_base, chunk, entry_base, row_window_id,
                                                   row_window_offset);
    RSH_LAUNCHED("k_entries");
  } else if (n_win == 0 && row_window_offset) {
    // no windows: the entry arrays are empty and row_window_offset = [0] (callers may pass a NULL
    // chunk here, as torch hands out address 0 for empty tensors)
    RSH_CUDA(cudaMemsetAsync(row_window_offset, 0, sizeof(int64_t), st));
  }
  return kOk;
}

// --- residual part (tile.py:146-165) --------------------------------------------------------

size_t rsh_residual_workspace(int64_t n_res) {
  Carve cv(nullptr);
  cv.take<int64_t>(n_res + 1);
  size_t a = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_res + 1));
  cv.take<char>(a);
  return cv.used + 256;
}

// offsets[0..n_res] = [0] + cumsum(row nnz); then (phase 2) col/value runs in plan order
int rsh_residual_offsets(const int64_t* row_ptr, const int32_t* resid_rows, int64_t n_res, int64_t* offsets,
                         void* ws, size_t ws_bytes, cudaStream_t st) {
  size_t need = rsh_residual_workspace(n_res);
  if (!ws || ws_bytes < need) return fail(kInvalid, "rsh_residual_offsets: workspace too small");
  Carve cv(ws);
  int64_t* cnt = cv.take<int64_t>(n_res + 1);
  size_t cb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cb, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_res + 1));
  void* cubtmp = cv.take<char>(cb);
  k_res_counts<<<grid_1d(n_res + 1), kThreads, 0, st>>>(row_ptr, resid_rows, n_res, cnt);
  RSH_LAUNCHED("k_res_counts");
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, cb, cnt, offsets, (int)(n_res + 1), st));
  return kOk;
}

int rsh_residual_gather(const int64_t* row_ptr, const int32_t* col_idx, const float* values,
                        const int32_t* resid_rows, int64_t n_res, const int64_t* offsets, int32_t* res_col_id,
                        float* res_values, cudaStream_t st) {
  if (n_res == 0) return kOk;
  k_res_gather<<<grid_1d(n_res * 32), kThreads, 0, st>>>(row_ptr, col_idx, values, resid_rows, n_res, offsets,
                                                          res_col_id, res_values);
  RSH_LAUNCHED("k_res_gather");
  return kOk;
}

}  // extern "C"

// ==========================================================================================
// row permutation (reorder.py:138-151 permute_rows): out row i = source row order[i]
// ==========================================================================================
namespace rsh {

__global__ void k_perm_counts(const int64_t* __restrict__ rp, const int64_t* __restrict__ order, int64_t n,
                              int64_t* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = i < n ? rp[order[i] + 1] - rp[order[i]] : 0;
}

__global__ void k_perm_copy(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, const float* __restrict__ va,
                            const int64_t* __restrict__ order, int64_t n, const int64_t* __restrict__ out_rp,
                            int32_t* out_ci, float* out_va) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t s = rp[order[i]], e = rp[order[i] + 1], o = out_rp[i];
    for (int64_t p = s + lane; p < e; p += 32) {
      out_ci[o + p - s] = ci[p];
      out_va[o + p - s] = va[p];
    }
  }
}

}  // namespace rsh

extern "C" {

size_t rsh_permute_workspace(int64_t n_rows) {
  rsh::Carve cv(nullptr);
  cv.take<int64_t>(n_rows + 1);
  size_t a = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_rows + 1));
  cv.take<char>(a);
  return cv.used + 256;
}

// reorder.py:138-151.  order: device int64[n_rows], a permutation of 0..n_rows-1 (the caller
// validates it, as Permutation does, reorder.py:95-107).  Writes out_row_ptr[n_rows+1],
// out_col_idx[nnz], out_values[nnz].
int rsh_permute_rows(const int64_t* row_ptr, const int32_t* col_idx, const float* values, int64_t n_rows,
                     const int64_t* order, int64_t* out_row_ptr, int32_t* out_col_idx, float* out_values, void* ws,
                     size_t ws_bytes, cudaStream_t st) {
  using namespace rsh;
  if (n_rows < 0) return fail(kInvalid, "rsh_permute_rows: bad n_rows");
  size_t need = rsh_permute_workspace(n_rows);
  if (!ws || ws_bytes < need) return fail(kInvalid, "rsh_permute_rows: workspace too small");
  Carve cv(ws);
  int64_t* cnt = cv.take<int64_t>(n_rows + 1);
  size_t cb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cb, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_rows + 1));
  void* tmp = cv.take<char>(cb);
  k_perm_counts<<<grid_1d(n_rows + 1), kThreads, 0, st>>>(row_ptr, order, n_rows, cnt);
  RSH_LAUNCHED("k_perm_counts");
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(tmp, cb, cnt, out_row_ptr, (int)(n_rows + 1), st));
  if (n_rows) {
    k_perm_copy<<<grid_1d(n_rows * 32), kThreads, 0, st>>>(row_ptr, col_idx, values, order, n_rows, out_row_ptr,
                                                            out_col_idx, out_values);
    RSH_LAUNCHED("k_perm_copy");
  }
  return kOk;
}

size_t rsh_transpose_workspace(int64_t n_rows, int64_t n_cols, int64_t nnz) {
  rsh::Carve cv(nullptr);
  cv.take<int32_t>(nnz + 1);  // row id per nonzero
  cv.take<int32_t>(nnz + 1);  // sorted keys
  cv.take<int32_t>(nnz + 1);  // identity
  cv.take<int32_t>(nnz + 1);  // permutation
  cv.take<int64_t>(n_cols + 1);
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                  (int)(nnz > 0 ? nnz : 1));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_cols + 1));
  cv.take<char>(a > b ? a : b);
  (void)n_rows;
  return cv.used + 256;
}

// A^T of a canonical CSR A (n_rows x n_cols): out_row_ptr[n_cols+1], out_col_idx[nnz],
// out_values[nnz]; canonical (strictly increasing columns per row), deterministic.
int rsh_transpose_csr(const int64_t* row_ptr, const int32_t* col_idx, const float* values, int64_t n_rows,
                      int64_t n_cols, int64_t nnz, int64_t* out_row_ptr, int32_t* out_col_idx, float* out_values,
                      void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace rsh;
  if (n_rows < 0 || n_cols < 0 || nnz < 0 || nnz >= (1LL << 31) || n_rows >= (1LL << 31))
    return fail(kInvalid, "rsh_transpose_csr: bad sizes (nnz and rows must fit int32)");
  const size_t need = rsh_transpose_workspace(n_rows, n_cols, nnz);
  if (!ws || ws_bytes < need) return fail(kInvalid, "rsh_transpose_csr: workspace too small");
  Carve cv(ws);
  int32_t* rid = cv.take<int32_t>(nnz + 1);
  int32_t* keys = cv.take<int32_t>(nnz + 1);
  int32_t* iota = cv.take<int32_t>(nnz + 1);
  int32_t* perm = cv.take<int32_t>(nnz + 1);
  int64_t* cnt = cv.take<int64_t>(n_cols + 1);
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                  (int)(nnz > 0 ? nnz : 1));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n_cols + 1));
  size_t cb = a > b ? a : b;
  void* tmp = cv.take<char>(cb);
  RSH_CUDA(cudaMemsetAsync(cnt, 0, (n_cols + 1) * sizeof(int64_t), st));
  if (nnz) {
    k_col_counts<<<grid_1d(nnz), kThreads, 0, st>>>(col_idx, nnz, cnt);
    k_row_ids<<<grid_1d(n_rows), kThreads, 0, st>>>(row_ptr, n_rows, rid);
    k_iota32<<<grid_1d(nnz), kThreads, 0, st>>>(iota, nnz);
    RSH_LAUNCHED("transpose prep");
    int bits = 1;
    while (bits < 31 && (1LL << bits) < n_cols) ++bits;
    size_t t = cb;
    RSH_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, col_idx, keys, iota, perm, (int)nnz, 0, bits, st));
    k_transpose_gather<<<grid_1d(nnz), kThreads, 0, st>>>(perm, rid, values, nnz, out_col_idx, out_values);
    RSH_LAUNCHED("k_transpose_gather");
  }
  size_t t = cb;
  RSH_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t, cnt, out_row_ptr, (int)(n_cols + 1), st));
  return kOk;
}

// Nonzeros the window part of the format holds (the size of TcPart.values, tile.py:123-131):
// sum over windows of row_ptr[start + count] - row_ptr[start]; count NULL means
// min(window_size, n_rows - start).  out: device int64[1].
int rsh_window_nnz(const int64_t* row_ptr, int64_t n_rows, const int32_t* win_start, const int32_t* win_count,
                   int64_t n_win, int32_t window_size, long long* out, cudaStream_t st) {
  if (!out) return fail(kInvalid, "rsh_window_nnz: null output");
  // win_count may be null: every window then spans min(window_size, rows left) rows
  if (n_win > 0 && (!row_ptr || !win_start || (!win_count && window_size < 1) || n_rows < 0))
    return fail(kInvalid, "rsh_window_nnz: bad arguments");
  RSH_CUDA(cudaMemsetAsync(out, 0, sizeof(long long), st));
  if (n_win <= 0) return kOk;
  k_window_nnz<<<grid_1d(n_win), kThreads, 0, st>>>(row_ptr, n_rows, win_start, win_count, n_win, window_size,
                                                     (unsigned long long*)out);
  RSH_LAUNCHED("k_window_nnz");
  return kOk;
}

}  // extern "C"
