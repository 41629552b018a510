// Locality-aware row reordering (reference reorder.py:1-481, PAPER Alg. 3) on
// device, with the two inherently sequential steps (Kruskal forest + DFS linearisation, the
// objective's left-to-right sum) as host C++ in the same library.
//
//   column weights  d_j^-alpha                         reorder.py:33-42    k_col_weights
//   row weight sums (bincount order)                   reorder.py:73-76    k_row_wsum
//   candidates + top-k weighted-Jaccard kNN           reorder.py:158-230  k_knn (warp per row)
//   Kruskal forest, DFS order                          reorder.py:268-321  rsh_mst_order (host)
//   objective: sum of (1 - sim) over adjacent pairs    reorder.py:96-101   k_pair_dis + host sum
//   windowed 2-opt                                     reorder.py:328-380  k_two_opt (warp per window)
//
// Similarities are the reference's: sim(r,u) = min(1, wi / (wsum[r] + wsum[u] - wi)) with wi the
// weight sum over the shared columns (ascending column order), 1 for two empty rows, 0 when the
// denominator is not positive.
#include "common.cuh"
#include <thread>
#include <cub/cub.cuh>
#include <algorithm>
#include <vector>
#include <numeric>

namespace rsh {

__global__ void k_col_degree_i64(const int32_t* __restrict__ col, int64_t nnz, unsigned long long* deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(deg + col[i], 1ull);
}

__global__ void k_col_weights(const unsigned long long* __restrict__ deg, int64_t n_cols, double alpha, double* w) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_cols; c += (int64_t)gridDim.x * blockDim.x)
    w[c] = deg[c] ? pow((double)deg[c], -alpha) : 0.0;
}

__global__ void k_row_wsum(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n_rows,
                           const double* __restrict__ w, double* wsum) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t p = rp[r]; p < rp[r + 1]; ++p) s += w[ci[p]];
    wsum[r] = s;
  }
}

// reorder.py:62-81 (_SimCache.sim): weighted Jaccard of the column supports of rows r and u
__device__ __forceinline__ double row_sim(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                          const double* __restrict__ w, const double* __restrict__ wsum,
                                          int64_t r, int64_t u) {
  if (r == u) return 1.0;
  int64_t a = rp[r], ae = rp[r + 1], b = rp[u], be = rp[u + 1];
  if (a == ae && b == be) return 1.0;
  double wi = 0.0;
  if ((ae - a) > 8 * (be - b) || (be - b) > 8 * (ae - a)) {
    // lopsided pair (a near-dense row): walk the short row, binary-search the long one; the
    // shared columns are still summed in ascending order
    if ((ae - a) > (be - b)) {
      int64_t t = a; a = b; b = t;
      t = ae; ae = be; be = t;
    }
    for (; a < ae; ++a) {
      const int32_t x = ci[a];
      int64_t lo = b, hi = be;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ci[mid] < x) lo = mid + 1; else hi = mid;
      }
      if (lo < be && ci[lo] == x) wi += w[x];
      b = lo;
    }
  } else
  while (a < ae && b < be) {
    const int32_t x = ci[a], y = ci[b];
    if (x == y) {
      wi += w[x];
      ++a;
      ++b;
    } else if (x < y) {
      ++a;
    } else {
      ++b;
    }
  }
  const double tot = wsum[r] + wsum[u] - wi;
  if (tot <= 0.0) return 0.0;
  const double v = wi / tot;
  return v < 1.0 ? v : 1.0;
}

constexpr int kKnnCap = 1024;   // distinct candidates tracked per row (power of two)
constexpr int kKnnWarps = 4;    // rows per 128-thread block

struct KnnSmem {
  int32_t key[kKnnCap];
  int32_t cnt[kKnnCap];
  unsigned long long sk[kKnnCap];  // sort keys: (0xFFFF - cnt) << 41 | u << 10 | slot
  double sim[kKnnCap];
};

// reorder.py:158-230.  Candidates: rows sharing a column with r (through A^T), counted per shared
// column; when more than max_candidates, the max_candidates with the largest count (ties to the
// lower row) are kept; then the top k by similarity (ties to the lower row), similarity > 0.
// Columns of degree > hub_cap are not walked for candidates (the reference walks all; with
// hub_cap >= the largest column degree and <= kKnnCap candidates per row the lists are the
// reference's).  stats[0] += rows whose candidates overflowed kKnnCap.
__global__ void __launch_bounds__(32 * kKnnWarps) k_knn(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                       int64_t n_rows, const int64_t* __restrict__ trp,
                                                       const int32_t* __restrict__ tci, const double* __restrict__ w,
                                                       const double* __restrict__ wsum, int k, int max_cand,
                                                       int64_t hub_cap, int32_t* nbr, double* nsim, int32_t* ncount,
                                                       unsigned long long* stats, int32_t* cand, int32_t* cand_cnt) {
  extern __shared__ __align__(16) unsigned char knn_smem[];
  KnnSmem& sm = reinterpret_cast<KnnSmem*>(knn_smem)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp0; r < n_rows; r += nwarps) {
    for (int i = lane; i < kKnnCap; i += 32) {
      sm.key[i] = -1;
      sm.cnt[i] = 0;
    }
    __syncwarp();
    bool overflow = false;
    for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
      const int32_t c = ci[p];
      const int64_t b0 = trp[c], b1 = trp[c + 1];
      if (b1 - b0 > hub_cap) continue;
      for (int64_t q = b0 + lane; q < b1; q += 32) {
        const int32_t u = tci[q];
        if (u == r) continue;
        uint32_t h = ((uint32_t)u * 2654435761u) & (kKnnCap - 1);
        int probe = 0;
        for (; probe < kKnnCap; ++probe) {
          const int32_t cur = sm.key[h];
          if (cur == u) break;
          if (cur == -1) {
            const int32_t prev = atomicCAS(&sm.key[h], -1, u);
            if (prev == -1 || prev == u) break;
          }
          h = (h + 1) & (kKnnCap - 1);
        }
        if (probe == kKnnCap) {
          overflow = true;
          continue;
        }
        sm.cnt[h] += 1;  // distinct u per column step: no two lanes touch one slot
      }
      // a full table ends the walk: the candidate set is truncated either way
      if (__any_sync(0xffffffffu, overflow)) {
        overflow = true;
        break;
      }
    }
    overflow = __any_sync(0xffffffffu, overflow);
    if (overflow && lane == 0) atomicAdd(stats, 1ull);
    // compact the occupied slots; when more than max_cand, sort them by (count desc, row asc)
    int n_occ = 0;
    for (int base = 0; base < kKnnCap; base += 32) {
      const int i = base + lane;
      const int32_t u = sm.key[i];
      const bool occ = u >= 0;
      const unsigned bal = __ballot_sync(0xffffffffu, occ);
      if (occ) {
        const int cn = sm.cnt[i] < 0xFFFF ? sm.cnt[i] : 0xFFFF;
        sm.sk[n_occ + __popc(bal & ((1u << lane) - 1u))] =
            ((unsigned long long)(0xFFFF - cn) << 41) | ((unsigned long long)u << 10) | (unsigned)i;
      }
      n_occ += __popc(bal);
    }
    __syncwarp();
    if (n_occ > max_cand) {
      int P = 32;
      while (P < n_occ) P <<= 1;
      for (int i = n_occ + lane; i < P; i += 32) sm.sk[i] = ~0ull;
      __syncwarp();
      for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int i = lane; i < P; i += 32) {
            const int j = i ^ stride;
            if (j > i) {
              const bool up = (i & size) == 0;
              const unsigned long long x = sm.sk[i], y = sm.sk[j];
              if ((x > y) == up) {
                sm.sk[i] = y;
                sm.sk[j] = x;
              }
            }
          }
          __syncwarp();
        }
      }
    }
    const int n_cand = n_occ < max_cand ? n_occ : max_cand;
    if (cand) {
      // build_candidates (reorder.py:168-194): the kept rows in ascending order
      int P = 32;
      while (P < n_cand) P <<= 1;
      for (int i = lane; i < P; i += 32)
        sm.sk[i] = i < n_cand ? ((sm.sk[i] >> 10) & 0x7FFFFFFFull) : ~0ull;
      __syncwarp();
      for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int i = lane; i < P; i += 32) {
            const int j = i ^ stride;
            if (j > i) {
              const bool up = (i & size) == 0;
              const unsigned long long x = sm.sk[i], y = sm.sk[j];
              if ((x > y) == up) {
                sm.sk[i] = y;
                sm.sk[j] = x;
              }
            }
          }
          __syncwarp();
        }
      }
      for (int i = lane; i < n_cand; i += 32) cand[r * (int64_t)max_cand + i] = (int32_t)sm.sk[i];
      if (lane == 0) cand_cnt[r] = n_cand;
      __syncwarp();
      continue;
    }
    // exact similarities of the kept candidates
    for (int i = lane; i < n_cand; i += 32) {
      const int64_t u = (int64_t)((sm.sk[i] >> 10) & 0x7FFFFFFFull);
      sm.sim[i] = row_sim(rp, ci, w, wsum, r, u);
    }
    __syncwarp();
    // top k by (similarity desc, row asc), similarity > 0
    int taken = 0;
    for (int t = 0; t < k; ++t) {
      double best = 0.0;
      int32_t bu = 0x7FFFFFFF;
      int bi = -1;
      for (int i = lane; i < n_cand; i += 32) {
        const double s = sm.sim[i];
        const int32_t u = (int32_t)((sm.sk[i] >> 10) & 0x7FFFFFFFull);
        if (s > 0.0 && (s > best || (s == best && u < bu))) {
          best = s;
          bu = u;
          bi = i;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int32_t ou = __shfl_xor_sync(0xffffffffu, bu, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && ou < bu)) {
          best = ob;
          bu = ou;
          bi = oi;
        }
      }
      if (bi < 0) break;
      if (lane == 0) {
        nbr[r * k + t] = bu;
        nsim[r * k + t] = best;
        sm.sim[bi] = -1.0;  // taken
      }
      __syncwarp();
      ++taken;
    }
    if (lane == 0) ncount[r] = taken;
    __syncwarp();
  }
}

// 1 - sim of every adjacent pair of an order (the objective's terms, reorder.py:96-101)
__global__ void k_pair_dis(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ w,
                           const double* __restrict__ wsum, const int64_t* __restrict__ order, int64_t m, double* dis) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i + 1 < m; i += (int64_t)gridDim.x * blockDim.x)
    dis[i] = 1.0 - row_sim(rp, ci, w, wsum, order[i], order[i + 1]);
}

// reorder.py:328-380, one warp per window [s, e).  Within the window the reference's sequential
// scan is kept exactly: for each i, the lowest j whose reversal strictly improves is applied and
// the scan continues at j + 1 on the modified order (candidate j's are scored 32 at a time).
// Windows of one launch are disjoint and a move may only touch positions s+1 .. e-2 (its
// boundary edges read positions s .. e-1), so concurrent windows never read each other's
// elements; launches alternate the window offset.  Every applied move strictly lowers the
// objective, so the result is never worse than the input.
__global__ void k_two_opt(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ w,
                          const double* __restrict__ wsum, int64_t* order, int64_t m, int window, int64_t offset,
                          unsigned long long* improved) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_win = (m - offset + window - 1) / window;
  for (int64_t wi = warp0; wi < n_win; wi += nwarps) {
    const int64_t s = offset + wi * window;
    const int64_t e = s + window < m ? s + window : m;
    bool any = false;
    for (int64_t i = s + 1; i + 1 < e; ++i) {
      int64_t j0 = i + 1;
      while (j0 + 1 < e) {
        const int64_t oi_1 = order[i - 1], oi = order[i];
        const double d_left = 1.0 - row_sim(rp, ci, w, wsum, oi_1, oi);
        const int64_t j = j0 + lane;
        bool good = false;
        if (j + 1 < e) {
          const int64_t oj = order[j], oj1 = order[j + 1];
          const double before = d_left + (1.0 - row_sim(rp, ci, w, wsum, oj, oj1));
          const double after = (1.0 - row_sim(rp, ci, w, wsum, oi_1, oj)) + (1.0 - row_sim(rp, ci, w, wsum, oi, oj1));
          good = after < before - 1e-12;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, good);
        if (bal) {
          const int64_t jj = j0 + __ffs(bal) - 1;
          // reverse order[i .. jj]
          const int64_t len = jj - i + 1;
          for (int64_t t = lane; t < len / 2; t += 32) {
            const int64_t x = order[i + t];
            order[i + t] = order[jj - t];
            order[jj - t] = x;
          }
          __syncwarp();
          any = true;
          j0 = jj + 1;
        } else {
          j0 += 32;
        }
      }
    }
    if (any && lane == 0) atomicAdd(improved, 1ull);
  }
}

}  // namespace rsh

using namespace rsh;

extern "C" {

size_t rsh_reorder_workspace(int64_t n_rows, int64_t n_cols) {
  Carve cv(nullptr);
  cv.take<unsigned long long>(n_cols + 1);
  cv.take<unsigned long long>(4);
  cv.take<double>(n_rows + 1);
  (void)n_rows;
  return cv.used + 256;
}

// reorder.py:33-42 + the row sums of _SimCache (reorder.py:73-76): w[n_cols], wsum[n_rows]
int rsh_column_weights(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                       double alpha, double* w, double* wsum, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!(alpha > 0.0)) return fail(kInvalid, "alpha must be positive");
  if (!ws || ws_bytes < rsh_reorder_workspace(n_rows, n_cols)) return fail(kInvalid, "rsh_column_weights: workspace too small");
  Carve cv(ws);
  unsigned long long* deg = cv.take<unsigned long long>(n_cols + 1);
  RSH_CUDA(cudaMemsetAsync(deg, 0, (n_cols + 1) * sizeof(unsigned long long), st));
  if (nnz) k_col_degree_i64<<<grid_1d(nnz), kThreads, 0, st>>>(col_idx, nnz, deg);
  if (n_cols) k_col_weights<<<grid_1d(n_cols), kThreads, 0, st>>>(deg, n_cols, alpha, w);
  if (n_rows) k_row_wsum<<<grid_1d(n_rows), kThreads, 0, st>>>(row_ptr, col_idx, n_rows, w, wsum);
  RSH_LAUNCHED("rsh_column_weights");
  return kOk;
}

// reorder.py:158-230 (build_candidates + build_knn).  A^T (at_*) gives the rows of each column.
// Outputs nbr[n_rows*k], nsim[n_rows*k], ncount[n_rows]; stats[0] = rows whose candidate set
// overflowed the per-row table (device uint64[1]).
int rsh_knn(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, const int64_t* at_row_ptr,
            const int32_t* at_col_idx, const double* w, const double* wsum, int32_t k, int32_t max_candidates,
            int64_t hub_cap, int32_t* nbr, double* nsim, int32_t* ncount, unsigned long long* stats, cudaStream_t st) {
  if (k < 1) return fail(kInvalid, "k must be at least 1");
  if (max_candidates < 1) return fail(kInvalid, "max_candidates must be at least 1");
  RSH_CUDA(cudaMemsetAsync(stats, 0, sizeof(unsigned long long), st));
  if (!n_rows) return kOk;
  const size_t smem = sizeof(KnnSmem) * kKnnWarps;
  RSH_CUDA(cudaFuncSetAttribute(k_knn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t blocks = (n_rows + kKnnWarps - 1) / kKnnWarps;
  const int64_t cap = 16LL * sm_count();
  if (blocks > cap) blocks = cap;
  k_knn<<<(unsigned)blocks, 32 * kKnnWarps, smem, st>>>(row_ptr, col_idx, n_rows, at_row_ptr, at_col_idx, w, wsum, k,
                                                       max_candidates, hub_cap, nbr, nsim, ncount, stats, nullptr, nullptr);
  RSH_LAUNCHED("k_knn");
  return kOk;
}

// 1 - sim over the m-1 adjacent pairs of a device order (the objective's terms)
// reorder.py:168-194 build_candidates: per row r, the rows sharing a column with r (r excluded),
// the max_candidates with the largest shared-column count when more (ties to the lower row), in
// ascending order: cand[r * max_candidates .. + cand_cnt[r]].  stats[0] += rows whose candidate set
// overflowed the per-row table (then truncated: the caller treats that as an error).
int rsh_candidates(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, const int64_t* at_row_ptr,
                   const int32_t* at_col_idx, int32_t max_candidates, int64_t hub_cap, int32_t* cand,
                   int32_t* cand_cnt, unsigned long long* stats, cudaStream_t st) {
  if (max_candidates < 1) return fail(kInvalid, "max_candidates must be at least 1");
  if (max_candidates > kKnnCap) return fail(kInvalid, "max_candidates above the device table (%d)", kKnnCap);
  if (!stats) return fail(kInvalid, "rsh_candidates: null stats");
  RSH_CUDA(cudaMemsetAsync(stats, 0, sizeof(unsigned long long), st));
  if (!n_rows) return kOk;
  if (!row_ptr || !at_row_ptr || !cand || !cand_cnt) return fail(kInvalid, "rsh_candidates: null array");
  const size_t smem = sizeof(KnnSmem) * kKnnWarps;
  RSH_CUDA(cudaFuncSetAttribute(k_knn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t blocks = (n_rows + kKnnWarps - 1) / kKnnWarps;
  const int64_t cap = 16LL * sm_count();
  if (blocks > cap) blocks = cap;
  k_knn<<<(unsigned)blocks, 32 * kKnnWarps, smem, st>>>(row_ptr, col_idx, n_rows, at_row_ptr, at_col_idx, nullptr, nullptr,
                                                       1, max_candidates, hub_cap, nullptr, nullptr, nullptr, stats,
                                                       cand, cand_cnt);
  RSH_LAUNCHED("k_knn(candidates)");
  return kOk;
}

int rsh_pair_dis(const int64_t* row_ptr, const int32_t* col_idx, const double* w, const double* wsum,
                 const int64_t* order, int64_t m, double* dis, cudaStream_t st) {
  if (m > 1) {
    k_pair_dis<<<grid_1d(m), kThreads, 0, st>>>(row_ptr, col_idx, w, wsum, order, m, dis);
    RSH_LAUNCHED("k_pair_dis");
  }
  return kOk;
}

// One 2-opt sweep over disjoint windows starting at `offset`; improved (device uint64[1]) is
// incremented once per window that applied a move.
int rsh_two_opt_sweep(const int64_t* row_ptr, const int32_t* col_idx, const double* w, const double* wsum,
                      int64_t* order, int64_t m, int32_t window, int64_t offset, unsigned long long* improved,
                      cudaStream_t st) {
  if (window < 2) return fail(kInvalid, "window must be at least 2");
  if (m < 3 || offset >= m) return kOk;
  const int64_t n_win = (m - offset + window - 1) / window;
  int64_t blocks = (n_win + 7) / 8;
  if (blocks > 64LL * sm_count()) blocks = 64LL * sm_count();
  k_two_opt<<<(unsigned)(blocks > 0 ? blocks : 1), 256, 0, st>>>(row_ptr, col_idx, w, wsum, order, m, window, offset,
                                                                improved);
  RSH_LAUNCHED("k_two_opt");
  return kOk;
}

// reorder.py:268-321 (mst_order) on HOST arrays: Kruskal forest over the undirected kNN edges
// with weight 1 - sim (ties on the lower, then the higher endpoint), each tree walked depth-first
// from its lowest vertex with children in descending similarity (ties to the lower row), trees
// by ascending root, then isolated vertices ascending.  order_out[m] (host int64).
int rsh_mst_order(int64_t m, int32_t k, const int32_t* nbr, const double* nsim, const int32_t* ncount,
                  int64_t* order_out) {
  if (m < 0 || k < 1) return fail(kInvalid, "rsh_mst_order: bad sizes");
  struct E {
    int64_t u, v;
    double s;
  };
  std::vector<E> dir;
  dir.reserve((size_t)m * k);
  for (int64_t r = 0; r < m; ++r)
    for (int t = 0; t < ncount[r]; ++t) {
      const int64_t u = nbr[r * k + t];
      dir.push_back(r < u ? E{r, u, nsim[r * k + t]} : E{u, r, nsim[r * k + t]});
    }
  // undirected edge set; a pair listed by both endpoints keeps the value met last (dict update)
  std::vector<size_t> idx(dir.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
    return dir[a].u != dir[b].u ? dir[a].u < dir[b].u : dir[a].v < dir[b].v;
  });
  std::vector<E> edges;
  for (size_t i = 0; i < idx.size(); ++i) {
    if (i + 1 < idx.size() && dir[idx[i + 1]].u == dir[idx[i]].u && dir[idx[i + 1]].v == dir[idx[i]].v) continue;
    edges.push_back(dir[idx[i]]);
  }
  std::stable_sort(edges.begin(), edges.end(), [](const E& a, const E& b) {
    const double wa = 1.0 - a.s, wb = 1.0 - b.s;
    if (wa != wb) return wa < wb;
    if (a.u != b.u) return a.u < b.u;
    return a.v < b.v;
  });
  std::vector<int64_t> parent(m), rnk(m, 0);
  std::iota(parent.begin(), parent.end(), 0);
  auto find = [&](int64_t x) {
    int64_t root = x;
    while (parent[root] != root) root = parent[root];
    while (parent[x] != root) {
      const int64_t nx = parent[x];
      parent[x] = root;
      x = nx;
    }
    return root;
  };
  std::vector<std::vector<std::pair<int64_t, double>>> adj(m);
  std::vector<char> has_adj(m, 0);
  for (const E& e : edges) {
    int64_t rx = find(e.u), ry = find(e.v);
    if (rx == ry) continue;
    if (rnk[rx] < rnk[ry]) std::swap(rx, ry);
    parent[ry] = rx;
    if (rnk[rx] == rnk[ry]) ++rnk[rx];
    adj[e.u].push_back({e.v, e.s});
    adj[e.v].push_back({e.u, e.s});
    has_adj[e.u] = has_adj[e.v] = 1;
  }
  std::vector<int64_t> comp_min(m, -1), roots;
  for (int64_t v = 0; v < m; ++v)
    if (has_adj[v]) {
      const int64_t r = find(v);
      if (comp_min[r] < 0 || v < comp_min[r]) comp_min[r] = v;
    }
  for (int64_t r = 0; r < m; ++r)
    if (comp_min[r] >= 0) roots.push_back(comp_min[r]);
  std::sort(roots.begin(), roots.end());
  std::vector<char> visited(m, 0);
  int64_t pos = 0;
  std::vector<int64_t> stack;
  std::vector<std::pair<int64_t, double>> children;
  for (int64_t start : roots) {
    stack.assign(1, start);
    while (!stack.empty()) {
      const int64_t x = stack.back();
      stack.pop_back();
      if (visited[x]) continue;
      visited[x] = 1;
      order_out[pos++] = x;
      children.clear();
      for (const auto& t : adj[x])
        if (!visited[t.first]) children.push_back(t);
      // push worst first, pop best: key (s ascending, row descending)
      std::stable_sort(children.begin(), children.end(), [](const auto& a, const auto& b) {
        if (a.second != b.second) return a.second < b.second;
        return a.first > b.first;
      });
      for (const auto& c : children) stack.push_back(c.first);
    }
  }
  for (int64_t v = 0; v < m; ++v)
    if (!visited[v]) order_out[pos++] = v;
  return kOk;
}

// reorder.py:386-446 (isolation_adjust) on HOST arrays, an exact restatement: rows whose
// similarity to both sequence neighbours is below iso_threshold are taken out and, in ascending
// row order, reinserted right after their most similar non-isolated row (candidates: rows
// sharing a column, ascending; ties to the lower row; empty rows match the first other empty
// non-isolated row); rows without a positive match go to the tail ascending.  w / wsum are the
// column weights and row weight sums (rsh_column_weights).  hub_cap < 0: walk every column (the
// reference); otherwise candidate walks skip columns with more rows.  Returns the number of
// isolated rows in *n_isolated.
int rsh_isolation_adjust(int64_t m, int64_t n_cols, const int64_t* rp, const int32_t* ci, const double* w,
                         const double* wsum, const int64_t* order_in, double iso_threshold, int64_t hub_cap,
                         int64_t* order_out, int64_t* n_isolated) {
  if (!(iso_threshold >= 0.0 && iso_threshold <= 1.0)) return fail(kInvalid, "iso_threshold must lie in [0, 1]");
  *n_isolated = 0;
  for (int64_t i = 0; i < m; ++i) order_out[i] = order_in[i];
  if (m <= 1 || iso_threshold == 0.0) return kOk;
  // weighted Jaccard (reorder.py:41-52): the shared columns' weights summed in ascending column
  // order -- by merging, or, for lopsided pairs (hub rows), by binary-searching the short row's
  // columns in the long row (same columns, same order, so the same double)
  auto sim = [&](int64_t r, int64_t u) -> double {
    if (r == u) return 1.0;
    int64_t a = rp[r], ae = rp[r + 1], b = rp[u], be = rp[u + 1];
    if (a == ae && b == be) return 1.0;
    double wi = 0.0;
    if (ae - a > 16 * (be - b) || be - b > 16 * (ae - a)) {
      if (ae - a > be - b) {
        std::swap(a, b);
        std::swap(ae, be);
      }
      int64_t lo = b;
      for (; a < ae; ++a) {
        const int32_t c = ci[a];
        int64_t hi = be;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (ci[mid] < c) lo = mid + 1; else hi = mid;
        }
        if (lo < be && ci[lo] == c) wi += w[c];
      }
    } else {
      while (a < ae && b < be) {
        if (ci[a] == ci[b]) {
          wi += w[ci[a]];
          ++a;
          ++b;
        } else if (ci[a] < ci[b]) {
          ++a;
        } else {
          ++b;
        }
      }
    }
    const double tot = wsum[r] + wsum[u] - wi;
    if (tot <= 0.0) return 0.0;
    const double v = wi / tot;
    return v < 1.0 ? v : 1.0;
  };
  std::vector<char> iso(m, 0);
  std::vector<int64_t> isolated;
  for (int64_t pos = 0; pos < m; ++pos) {
    const int64_t r = order_in[pos];
    const bool left = pos > 0 && sim(order_in[pos - 1], r) >= iso_threshold;
    const bool right = pos < m - 1 && sim(r, order_in[pos + 1]) >= iso_threshold;
    if (!left && !right) {
      iso[r] = 1;
      isolated.push_back(r);
    }
  }
  *n_isolated = (int64_t)isolated.size();
  if (isolated.empty()) return kOk;
  // base sequence as a linked list (insert-after is O(1))
  const int64_t NIL = -1;
  std::vector<int64_t> next(m, NIL);
  int64_t head = NIL, last = NIL;
  for (int64_t pos = 0; pos < m; ++pos) {
    const int64_t r = order_in[pos];
    if (iso[r]) continue;
    if (last == NIL) head = r; else next[last] = r;
    last = r;
  }
  // inverted index: rows of each column, ascending
  std::vector<int64_t> cstart(n_cols + 1, 0);
  for (int64_t p = 0; p < rp[m]; ++p) ++cstart[ci[p] + 1];
  for (int64_t c = 0; c < n_cols; ++c) cstart[c + 1] += cstart[c];
  std::vector<int64_t> fillp(cstart.begin(), cstart.end() - 1), crow(rp[m]);
  for (int64_t r = 0; r < m; ++r)
    for (int64_t p = rp[r]; p < rp[r + 1]; ++p) crow[fillp[ci[p]]++] = r;
  std::vector<int64_t> empties;
  for (int64_t r = 0; r < m; ++r)
    if (rp[r + 1] == rp[r]) empties.push_back(r);
  std::sort(isolated.begin(), isolated.end());
  // the best match of every isolated row depends only on the static similarities and flags, so
  // it is computed in parallel; the insertions then run in ascending row order (reorder.py:386-446)
  const int64_t n_iso = (int64_t)isolated.size();
  std::vector<int64_t> best_of(n_iso, NIL);
  int64_t first_empty = NIL;  // the first non-isolated empty row (empty isolated rows' match)
  for (const int64_t u : empties)
    if (!iso[u]) {
      first_empty = u;
      break;
    }
  auto work = [&](int64_t i0, int64_t i1) {
    std::vector<int64_t> cand;
    std::vector<char> seen(m, 0);
    for (int64_t i = i0; i < i1; ++i) {
      const int64_t r = isolated[i];
      int64_t best = NIL;
      if (rp[r + 1] == rp[r]) {
        best = first_empty;  // u != r holds: r is isolated, first_empty is not
      } else {
        cand.clear();
        for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
          const int32_t c = ci[p];
          if (hub_cap >= 0 && cstart[c + 1] - cstart[c] > hub_cap) continue;
          for (int64_t q = cstart[c]; q < cstart[c + 1]; ++q)
            if (!seen[crow[q]]) {
              seen[crow[q]] = 1;
              cand.push_back(crow[q]);
            }
        }
        for (const int64_t u : cand) seen[u] = 0;
        // the reference scans candidates in ascending order and keeps the first strict maximum:
        // the largest similarity > 0, ties to the lower row -- order-free, so no sort
        double best_sim = 0.0;
        for (const int64_t u : cand) {
          if (u == r || iso[u]) continue;
          const double sv = sim(r, u);
          if (sv > best_sim || (sv == best_sim && sv > 0.0 && u < best)) {
            best = u;
            best_sim = sv;
          }
        }
      }
      best_of[i] = best;
    }
  };
  const int64_t n_threads = std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), 64);
  if (n_iso < 4096 || n_threads == 1) {
    work(0, n_iso);
  } else {
    std::vector<std::thread> pool;
    const int64_t per = (n_iso + n_threads - 1) / n_threads;
    for (int64_t t = 0; t < n_threads; ++t) {
      const int64_t i0 = t * per, i1 = std::min(n_iso, i0 + per);
      if (i0 < i1) pool.emplace_back(work, i0, i1);
    }
    for (auto& th : pool) th.join();
  }
  std::vector<int64_t> tail;
  for (int64_t i = 0; i < n_iso; ++i) {
    const int64_t r = isolated[i], best = best_of[i];
    if (best == NIL) {
      tail.push_back(r);
    } else {
      next[r] = next[best];
      next[best] = r;
      if (last == best) last = r;
    }
  }
  int64_t pos = 0;
  for (int64_t x = head; x != NIL; x = next[x]) order_out[pos++] = x;
  for (const int64_t r : tail) order_out[pos++] = r;
  return pos == m ? kOk : fail(kInvalid, "rsh_isolation_adjust: internal error (lost rows)");
}

// the objective's left-to-right sum (reorder.py:96-101) over host terms
double rsh_sum_sequential(const double* x, int64_t n) {
  double t = 0.0;
  for (int64_t i = 0; i < n; ++i) t += x[i];
  return t;
}

}  // extern "C"
