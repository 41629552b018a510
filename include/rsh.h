/*
 * rsh.h -- C ABI of librsh.so, the B200 (sm_100a) RSH-SpMM hot path.
 *
 * The reference (rstile 0.1.0, /root/reference/pkg/src/rstile) has no native layer: its
 * boundary is the Python API (__init__.py:79-139).  Each entry point below replaces one
 * reference function (cited), with the reference's algorithm rewritten as device kernels.
 *
 * Conventions
 *   - every pointer argument is DEVICE memory unless stated; every call is stream-ordered on
 *     the caller's cudaStream_t and returns before the work completes;
 *   - the caller owns and allocates every buffer, including workspaces (sized by the matching
 *     *_workspace / *_bytes query); the library never allocates or frees caller memory;
 *   - return value: 0 ok, 1 invalid argument (-> ValueError), 2 format (-> FormatError),
 *     3 CUDA/launch error (-> RuntimeError); rsh_last_error() gives a thread-local message;
 *   - no global mutable state besides cached per-kernel launch sizes and a diagnostic launch
 *     counter: calls are reentrant.  A schedule (rsh_schedule) is read-only during SpMM
 *     launches; every launch's mutable state (work counter, window tickets, chunk partials)
 *     lives in the caller's SpMM workspace, so concurrent launches sharing one schedule need one
 *     workspace each (e.g. one per stream).  One process per GPU for multi-GPU use.
 *   - dtypes follow the reference format (tile.py:43-82): row_window_id int32,
 *     row_window_offset int64, bitmaps uint64, col_id int32, values float32; residual row_id
 *     int32, row_nnz_offset int64, col_id int32, values float32.  CSR: row_ptr int64,
 *     col_idx int32, values float32 (core.py:26-47).
 */
#ifndef RSH_H_
#define RSH_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- plumbing --------------------------------------------------------------------------- */
const char* rsh_last_error(void);
int rsh_abi_version(void);
/* kernels launched through this library by the process so far (diagnostic; the bench reports
 * the launches inside its timed region from it) */
unsigned long long rsh_launch_count(void);
/* host pointers: compute capability and SM count of the current device */
int rsh_device_info(int32_t* major, int32_t* minor, int32_t* sms);

/* ---- adaptive row partition: partition.py:119-141 partition_rows (+ column_increment
 *      partition.py:101-116).  win_start / resid_rows need capacity n_rows (int32);
 *      counts[0] = #windows, counts[1] = #residual rows (device int64[2]).  Window i covers
 *      rows [win_start[i], win_start[i] + min(window_size, n_rows - win_start[i])). -------- */
size_t rsh_partition_workspace(int64_t n_rows);
int rsh_partition(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int32_t window_size,
                  int64_t tau_nnz, int64_t tau_inc, int32_t* win_start, int32_t* resid_rows, int64_t* counts,
                  void* ws, size_t ws_bytes, cudaStream_t stream);

/* ---- window columns + split_long_work: partition.py:144-180.  win_count may be NULL
 *      (counts = min(window_size, n_rows - start)).  Outputs: row_win[n_rows] (window of each
 *      row or -1), prefix[nnz+1] (exclusive scan of first-occurrence flags), nblocks[n_win]
 *      = ceil(|window_columns|/8), longest[n_win] = longest row, chunk[n_win] = segment
 *      length (0: unsplit), entry_base/block_base[n_win+1] exclusive scans.
 *      max_blocks_per_item <= 0 means None. ----------------------------------------------- */
size_t rsh_plan_workspace(int64_t n_rows, int64_t nnz, int64_t n_win);
int rsh_plan_windows(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t nnz,
                     int32_t window_size, const int32_t* win_start, const int32_t* win_count, int64_t n_win,
                     int64_t max_blocks_per_item, int32_t split_on_row_nnz, double split_factor, int32_t* row_win,
                     int32_t* prefix, int64_t* nblocks, int64_t* longest, int64_t* chunk, int64_t* entry_base,
                     int64_t* block_base, void* ws, size_t ws_bytes, cudaStream_t stream);

/* ---- RS-Tile build: tile.py:102-144 build_rstile (TC part).  With chunk == NULL the
 *      entry arrays are not written (the caller supplies explicit segments). -------------- */
/* TcPart.values size (tile.py:123-131): sum over windows of their rows' nonzeros; win_count NULL
 * means min(window_size, n_rows - start).  out: device int64[1]. */
int rsh_window_nnz(const int64_t* row_ptr, int64_t n_rows, const int32_t* win_start, const int32_t* win_count,
                   int64_t n_win, int32_t window_size, long long* out, cudaStream_t stream);
size_t rsh_fill_workspace(int64_t nnz, int64_t n_blocks);
int rsh_build_fill(const int64_t* row_ptr, const int32_t* col_idx, const float* values, int64_t n_rows,
                   int64_t nnz, int32_t window_size, const int32_t* win_start, const int32_t* win_count,
                   int64_t n_win, const int32_t* row_win, const int32_t* prefix, const int64_t* block_base,
                   int64_t n_blocks, const int64_t* chunk, const int64_t* entry_base, int32_t* row_window_id,
                   int64_t* row_window_offset, uint64_t* bitmaps, int32_t* col_id, float* tc_values, void* ws,
                   size_t ws_bytes, cudaStream_t stream);

/* ---- residual part: tile.py:146-165 ------------------------------------------------------ */
size_t rsh_residual_workspace(int64_t n_res);
int rsh_residual_offsets(const int64_t* row_ptr, const int32_t* resid_rows, int64_t n_res, int64_t* offsets,
                         void* ws, size_t ws_bytes, cudaStream_t stream);
int rsh_residual_gather(const int64_t* row_ptr, const int32_t* col_idx, const float* values,
                        const int32_t* resid_rows, int64_t n_res, const int64_t* offsets, int32_t* res_col_id,
                        float* res_values, cudaStream_t stream);

/* ---- row permutation: reorder.py:138-151 permute_rows (out row i = source row order[i]);
 *      order is a device int64 permutation of 0..n_rows-1 (validated by the caller). -------- */
size_t rsh_permute_workspace(int64_t n_rows);
int rsh_permute_rows(const int64_t* row_ptr, const int32_t* col_idx, const float* values, int64_t n_rows,
                     const int64_t* order, int64_t* out_row_ptr, int32_t* out_col_idx, float* out_values, void* ws,
                     size_t ws_bytes, cudaStream_t stream);

/* ---- transpose: A^T as a canonical CSR (the GNN backward operand; no
 *      reference counterpart -- the reference has no autograd).  Deterministic (stable radix
 *      sort by column).  nnz and n_rows must fit int32. ------------------------------------ */
size_t rsh_transpose_workspace(int64_t n_rows, int64_t n_cols, int64_t nnz);
int rsh_transpose_csr(const int64_t* row_ptr, const int32_t* col_idx, const float* values, int64_t n_rows,
                      int64_t n_cols, int64_t nnz, int64_t* out_row_ptr, int32_t* out_col_idx, float* out_values,
                      void* ws, size_t ws_bytes, cudaStream_t stream);

/* ---- locality-aware row reordering (reorder.py:1-481).  Device: column
 *      weights d^-alpha and row sums (reorder.py:33-42,73-76), candidates + top-k weighted-Jaccard
 *      kNN through A^T (reorder.py:158-230), objective terms, windowed 2-opt sweeps
 *      (reorder.py:328-380).  Host (plain host pointers): Kruskal forest + DFS order
 *      (reorder.py:268-321) and the objective's left-to-right sum. ------------------------- */
size_t rsh_reorder_workspace(int64_t n_rows, int64_t n_cols);
int rsh_column_weights(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                       double alpha, double* w, double* wsum, void* ws, size_t ws_bytes, cudaStream_t stream);
int rsh_knn(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, const int64_t* at_row_ptr,
            const int32_t* at_col_idx, const double* w, const double* wsum, int32_t k, int32_t max_candidates,
            int64_t hub_cap, int32_t* nbr, double* nsim, int32_t* ncount, unsigned long long* stats,
            cudaStream_t stream);
/* reorder.py:168-194 build_candidates: rows sharing a column with each row (itself excluded), the
 * max_candidates (<= 1024) with the most shared columns when more (ties to the lower row), ascending:
 * cand[r * max_candidates .. + cand_cnt[r]]; stats[0] = rows whose candidate set overflowed the
 * per-row device table (their lists are truncated). */
int rsh_candidates(const int64_t* row_ptr, const int32_t* col_idx, int64_t n_rows, const int64_t* at_row_ptr,
                   const int32_t* at_col_idx, int32_t max_candidates, int64_t hub_cap, int32_t* cand,
                   int32_t* cand_cnt, unsigned long long* stats, cudaStream_t stream);
int rsh_pair_dis(const int64_t* row_ptr, const int32_t* col_idx, const double* w, const double* wsum,
                 const int64_t* order, int64_t m, double* dis, cudaStream_t stream);
int rsh_two_opt_sweep(const int64_t* row_ptr, const int32_t* col_idx, const double* w, const double* wsum,
                      int64_t* order, int64_t m, int32_t window, int64_t offset, unsigned long long* improved,
                      cudaStream_t stream);
int rsh_mst_order(int64_t m, int32_t k, const int32_t* nbr, const double* nsim, const int32_t* ncount,
                  int64_t* order_out);
int rsh_isolation_adjust(int64_t m, int64_t n_cols, const int64_t* row_ptr, const int32_t* col_idx, const double* w,
                         const double* wsum, const int64_t* order_in, double iso_threshold, int64_t hub_cap,
                         int64_t* order_out, int64_t* n_isolated);
double rsh_sum_sequential(const double* x, int64_t n);

/* ---- persistent-kernel schedule: execute.py:136-168 (_window_groups, value starts) as device
 *      data.  Logical windows are cut into units of chunk_blocks blocks (>= 32; rsh_spmm_cc is
 *      tuned for 32, rsh_spmm_tc for 256) at fixed offsets, so results never depend on the
 *      format's split segments.  header_out (device int64[8], may be NULL) = [groups, window
 *      units, units, partial slots, uncovered rows, chunk_blocks, 0, 0]. ------------------- */
size_t rsh_schedule_bytes(int64_t n_rows, int64_t n_entries, int64_t n_blocks, int64_t n_res);
int rsh_schedule(int64_t n_rows, int32_t window_size, const int32_t* row_window_id,
                 const int64_t* row_window_offset, int64_t n_entries, const uint64_t* bitmaps, int64_t n_blocks,
                 const int32_t* res_row_id, int64_t n_res, int32_t chunk_blocks, void* sched, size_t sched_bytes,
                 int64_t* header_out, cudaStream_t stream);
/* SpMM workspace: a control block (work counter, per-window tickets) + chunk partials for
 * partial_slots (schedule header[3]) 8-row slots.  16-byte aligned, ZERO-FILLED by the caller
 * before its first use (every launch leaves the control block zero again); one workspace per
 * concurrently running launch.  A launch whose workspace holds fewer partial slots than its
 * schedule needs traps (the kernel checks header[3] against the size passed). */
size_t rsh_partials_bytes(int64_t n_entries, int64_t partial_slots, int64_t n_features, int32_t accum);

/* ---- row-major window list (optional, once per schedule; no reference counterpart): the
 *      window units' nonzeros as int2 (col_id, value) pairs in stream order (the buffer,
 *      16-byte aligned, also holds the scratch that puts the window units longest-first and a
 *      48-byte header per unit -- row, partial slot, list range, per-row list ends; size it with
 *      rsh_rowmajor_bytes).  rsh_spmm_cc then sets a unit up from its header and copies its list
 *      coalesced instead of decoding bitmaps; results are bit-identical with or without it.  The
 *      buffer must outlive the schedule's use (its addresses are recorded in the schedule).  The
 *      list is a SNAPSHOT of col_id and tc_values: rsh_spmm_cc then reads the pairs from it, not
 *      from its own col_id / tc_values arguments, so a caller that changes the values (same
 *      sparsity) must rebuild the list (paper_2603_08734_b200.device keys its cached plan on the
 *      arrays' identity and version for this). */
size_t rsh_rowmajor_bytes(int64_t n_rows, int64_t n_entries, int64_t n_blocks, int64_t n_res, int64_t tc_nnz);
int rsh_schedule_rowmajor(int64_t n_rows, int64_t n_entries, const uint64_t* bitmaps, const int32_t* col_id,
                          const float* tc_values, int64_t n_blocks, int64_t tc_nnz, int64_t n_res, void* sched,
                          size_t sched_bytes, void* ulist, size_t ulist_bytes, cudaStream_t stream);

/* ---- hybrid SpMM: execute.py:155-218 hybrid_spmm.  C[n_rows x N] (row stride ldc) is
 *      fully written: window rows assigned, residual rows assigned, all other rows zero.
 *      B[n_cols x N] row stride ldb; b_dtype 0 f32, 1 bf16, 2 f16; accum bit 0: 0 f32, 1 f64;
 *      accum bits 1..14 are kernel-variant knobs (spmm_cc.cu), bit 14 = "the schedule has no
 *      window beyond 256 chunks (header[6] == 0): skip the two fix-up launches".
 *      sched/partials: the schedule and the caller's workspace (rsh_partials_bytes).
 *      rsh_spmm_cc: one persistent CUDA-core launch (exact FP32 products). -------------- */
int rsh_spmm_cc(int64_t n_rows, int32_t window_size, int64_t n_entries, const uint64_t* bitmaps,
                const int32_t* col_id, const float* tc_values, int64_t n_blocks, const int32_t* res_row_id,
                const int64_t* res_offset, const int32_t* res_col_id, const float* res_values, int64_t n_res,
                const void* B, int64_t ldb, int32_t b_dtype, int64_t N, float* C, int64_t ldc, int32_t accum,
                void* sched, size_t sched_bytes, void* partials, size_t partial_bytes, cudaStream_t stream);

/* rsh_tc_fragments: schedule-time image of every 8x8 block in the MMA's shared-memory operand
 * layout (K-major core matrices), decoded once per (format, operand type) from the bitmaps and the
 * bit-ordered values (tile.py:123-131): b_dtype 0 -> tf32 (cvt.rna, 256 B per block), 1 -> bf16,
 * 2 -> fp16 (round to nearest, 128 B per block).  out_bytes >= rsh_tc_fragment_bytes(). */
size_t rsh_tc_fragment_bytes(int64_t n_blocks, int32_t b_dtype);
int rsh_tc_fragments(int64_t n_rows, int64_t n_entries, const uint64_t* bitmaps, const float* tc_values,
                     int64_t n_blocks, int64_t n_res, int32_t b_dtype, const void* sched, size_t sched_bytes,
                     void* out, size_t out_bytes, cudaStream_t stream);

/* rsh_spmm_tc: the same contract with the window blocks on the tensor cores (tcgen05.mma,
 * fp32 accumulation in TMEM): b_dtype 0 -> TF32 operands, 1 -> BF16, 2 -> FP16.  N in
 * {32, 64, 128, 256} (fp32 B) or {64, 128, 256} (half B); B rows 16-byte aligned.  b_rows = rows
 * of B (the TMA tensor map's extent: B rows are staged into shared memory by tile::gather4, and
 * padding slots read as zeros); fragments = rsh_tc_fragments(..., b_dtype) of this format.
 * Residual / uncovered rows run on CUDA cores in the same launch.  For N >= 128 half of each
 * pipeline's super-stages are staged by 16-byte cp.async (the LSU) beside the TMA.  flags:
 * bit 13 = "no window needs the fix-up kernels" (as rsh_spmm_cc's accum bit 14); bits 0 / 2 / 5 /
 * 6 are perf probes (skip the gathers / MMAs / epilogue stores / fragment copies; results
 * invalid). */
int rsh_spmm_tc(int64_t n_rows, int32_t window_size, int64_t n_entries, const uint64_t* bitmaps,
                const int32_t* col_id, const void* fragments, size_t fragment_bytes, int64_t n_blocks,
                const int32_t* res_row_id, const int64_t* res_offset, const int32_t* res_col_id,
                const float* res_values, int64_t n_res, const void* B, int64_t b_rows, int64_t ldb,
                int32_t b_dtype, int64_t N, float* C, int64_t ldc, int32_t flags, void* sched,
                size_t sched_bytes, void* partials, size_t partial_bytes, cudaStream_t stream);

/* ---- format checks and decode: tile.py:176-267 validate_rstile, tile.py:270-307 decode_rstile.
 *      rsh_validate writes rsh_report_slots() int64 facts (first offending index per check,
 *      ranges, popcount sum) that the host turns into the reference's messages; rsh_decode
 *      rebuilds CSR (row_ptr[n_rows+1], col_idx/values[tc_nnz + res_nnz]) from a valid format,
 *      dup_out[0] = first duplicate position or -1 (non-canonical result). ------------------ */
int rsh_report_slots(void);
size_t rsh_validate_workspace(int64_t n_rows, int64_t n_entries, int64_t n_blocks);
int rsh_validate(int64_t n_rows, int64_t n_cols, int32_t window_size, const int32_t* row_window_id,
                 const int64_t* row_window_offset, int64_t n_entries, const uint64_t* bitmaps, const int32_t* col_id,
                 int64_t n_col_id, int64_t n_blocks, int64_t n_values, const int32_t* res_row_id,
                 const int64_t* res_offset, int64_t n_res, const int32_t* res_col_id, int64_t n_res_col,
                 int32_t check_bits, int32_t check_cover, int64_t* rep, void* ws, size_t ws_bytes,
                 cudaStream_t stream);
size_t rsh_decode_workspace(int64_t n_rows, int64_t nnz, int64_t n_blocks);
int rsh_decode(int64_t n_rows, int64_t n_cols, const int32_t* row_window_id, const int64_t* row_window_offset,
               int64_t n_entries, const uint64_t* bitmaps, const int32_t* col_id, const float* tc_values,
               int64_t n_blocks, int64_t tc_nnz, const int32_t* res_row_id, const int64_t* res_offset, int64_t n_res,
               const int32_t* res_col_id, const float* res_values, int64_t res_nnz, int64_t* out_row_ptr,
               int32_t* out_col_idx, float* out_values, int64_t* dup_out, void* ws, size_t ws_bytes,
               cudaStream_t stream);

/* ---- verification: core.py:398-408 max_relative_error, result in out[0] (device double) - */
int rsh_max_relative_error(const float* c, const float* ref, int64_t rows, int64_t n_features, int64_t ldc,
                           double* out, cudaStream_t stream);
/* core.py:380-395 oracle_spmm from the CSR: f64 accumulation per row in CSR order, f32 store */
int rsh_csr_spmm_f64(const int64_t* row_ptr, const int32_t* col_idx, const float* values, int64_t n_rows,
                     const float* B, int64_t ldb, int64_t N, float* C, int64_t ldc, cudaStream_t stream);

/* ---- structure metrics: metrics.py:28-63 tile_density.  out (device uint64[2]) = [row windows
 *      (consecutive equal row_window_id), occupied rows of those windows]. ------------------- */
int rsh_tile_density(const int32_t* row_window_id, const int64_t* row_window_offset, int64_t n_entries,
                     const uint64_t* bitmaps, unsigned long long* out, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* RSH_H_ */
