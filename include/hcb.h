/*
 * hcb.h -- C-ABI of libhcb.so, the B200 (sm_100a) IPGC hot path.
 *
 * The reference (hybridcolor, /root/reference/pkg) crosses into native code at
 * exactly one place: the kernel-module plugin API that `_backend.get_kernels()`
 * hands to the round functions (pkg/src/hybridcolor/_backend.py:13-44,
 * _kernels.pyx:25-187).  The hc_k_* entry points below are that API, one per
 * reference function, over DEVICE int64 buffers with the same argument meaning.
 * hc_solve replaces the whole `color_graph` round loop
 * (driver.py:122-176 + coloring.py:113-176 + worklist.py:77-91) with a single
 * device-resident solve.  Graph construction / generation / verification
 * entry points replace graph.py:184-201 and driver.py:179-204.
 *
 * Conventions (all entry points):
 *   - plain pointers + sizes, no torch types;  `d_` pointers are device
 *     pointers (borrowed for the duration of the call), `h_` are host.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *   - the library never allocates device memory: scratch comes from a
 *     caller-owned workspace sized by the matching *_workspace_bytes query.
 *   - return HC_OK (0) or a negative HC_ERR_* code; hc_last_error() gives the
 *     message of the last failure on the calling host thread.
 *   - one device per call (the caller selects it); reentrant per stream.
 */
#ifndef HCB_H_
#define HCB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HC_OK 0
#define HC_ERR_INVALID (-1)      /* bad argument (ValueError in the reference)        */
#define HC_ERR_CUDA (-2)         /* CUDA runtime / launch failure                       */
#define HC_ERR_WL_OVERFLOW (-3)  /* worklist overflow: worklist.py:50-58, 79-83         */
#define HC_ERR_WORKSPACE (-4)    /* workspace too small                                 */
#define HC_ERR_UNCOLORED (-5)    /* colors_used on a 0 entry: driver.py:183-184         */
#define HC_ERR_DUPLICATE (-6)    /* duplicate push in one iteration: worklist.py:85-88  */
#define HC_ERR_RECORDS (-7)      /* per-round record buffer too small (rounds returned) */
#define HC_ERR_TIMEOUT (-8)      /* multi-GPU: a peer missed a cross-GPU barrier       */
#define HC_ERR_STALLED (-9)      /* solve exceeded n rounds (broken invariant; a bug)   */

#define HC_MODE_DATA 0   /* driver.py:149-150 */
#define HC_MODE_TOPO 1   /* driver.py:147-148 */
#define HC_MODE_HYBRID 2 /* driver.py:151-152 */

/* One RoundRecord (driver.py:47-54); `topo` is mode_used == "topo". */
typedef struct hc_round_rec {
    int64_t round;
    int64_t topo;
    int64_t wl_in;
    int64_t wl_out;
    int64_t conflicts;
    int64_t ns; /* device %globaltimer nanoseconds spent in the round */
} hc_round_rec;

const char *hc_last_error(void);
int hc_version(void);
/* number of SMs and the solver's resident CTAs per SM on the current device */
int hc_device_info(int *h_num_sms, int *h_ctas_per_sm);

/* ------------------------------------------------------------------ */
/* Kernel-module plugin API (the reference's native operator surface). */
/* All arrays int64 and C-contiguous on the device, exactly as in       */
/* _kernels.pyx; `active` is uint8.  Scalar results are accumulated in  */
/* the caller's device scalar d_acc (int64[1], zeroed by the call) and  */
/* copied to the host pointer after the stream is synchronised.         */
/* ------------------------------------------------------------------ */

/* _kernels.pyx:29-58 assign_from_list */
int hc_k_assign_from_list(const int64_t *d_row_offsets, const int64_t *d_col_indices,
                          const int64_t *d_colors_read, int64_t *d_colors_write, int64_t *d_stamp,
                          const int64_t *d_nodes, int64_t num_list, int64_t round_no,
                          int64_t max_degree, void *stream);
/* _kernels.pyx:61-91 assign_sweep; *h_processed = nodes with colors_read==0 */
int hc_k_assign_sweep(const int64_t *d_row_offsets, const int64_t *d_col_indices,
                      const int64_t *d_colors_read, int64_t *d_colors_write, int64_t *d_stamp,
                      int64_t num_nodes, int64_t round_no, int64_t max_degree,
                      int64_t *d_acc, int64_t *h_processed, void *stream);
/* _kernels.pyx:94-120 resolve_from_list; *h_conflicts = sum of k_u */
int hc_k_resolve_from_list(const int64_t *d_row_offsets, const int64_t *d_col_indices,
                           const int64_t *d_colors_read, int64_t *d_colors_write,
                           const int64_t *d_stamp, const int64_t *d_nodes, int64_t num_list,
                           int64_t round_no, int64_t *d_next_ids, int64_t capacity,
                           int64_t *d_cursor, int64_t *d_acc, int64_t *h_conflicts,
                           void *stream);
/* _kernels.pyx:123-149 resolve_sweep */
int hc_k_resolve_sweep(const int64_t *d_row_offsets, const int64_t *d_col_indices,
                       const int64_t *d_colors_read, int64_t *d_colors_write,
                       const int64_t *d_stamp, int64_t num_nodes, int64_t round_no,
                       int64_t *d_next_ids, int64_t capacity, int64_t *d_cursor,
                       int64_t *d_acc, int64_t *h_conflicts, void *stream);
/* _kernels.pyx:152-168 bench_from_list */
int hc_k_bench_from_list(const int64_t *d_nodes, int64_t num_list, uint8_t *d_active,
                         int64_t cutoff, int64_t *d_next_ids, int64_t capacity,
                         int64_t *d_cursor, void *stream);
/* _kernels.pyx:171-187 bench_sweep */
int hc_k_bench_sweep(uint8_t *d_active, int64_t num_nodes, int64_t cutoff, int64_t *d_next_ids,
                     int64_t capacity, int64_t *d_cursor, void *stream);

/* Commits between phases, coloring.py:105-110:
 *   _commit_list:    colors_read[nodes] = colors_write[nodes]
 *   _commit_stamped: colors_read[u] = colors_write[u] where stamp[u] == round_no */
int hc_k_commit_list(int64_t *d_colors_read, const int64_t *d_colors_write, const int64_t *d_nodes,
                     int64_t num_list, void *stream);
int hc_k_commit_stamped(int64_t *d_colors_read, const int64_t *d_colors_write,
                        const int64_t *d_stamp, int64_t num_nodes, int64_t round_no, void *stream);

/* Worklist.swap_and_sort (worklist.py:77-91): d_sorted[0..m) = ascending
 * d_next[0..m) with m = *d_cursor; duplicate ids -> HC_ERR_DUPLICATE, m >
 * capacity -> HC_ERR_WL_OVERFLOW.  *h_count = m.  Workspace: capacity+1 int64. */
size_t hc_wl_sort_workspace_bytes(int64_t capacity);
int hc_wl_swap_and_sort(const int64_t *d_next, const int64_t *d_cursor, int64_t capacity,
                        int64_t *d_sorted, int64_t *h_count, void *d_ws, size_t ws_bytes,
                        void *stream);

/* ------------------------------------------------------------------ */
/* Device-resident solve (replaces the color_graph round loop).         */
/* ------------------------------------------------------------------ */

/* CSR: d_row_offsets int64[n+1], d_col_indices int32[m], symmetric, with each
 * row's lower-id neighbours first (build_csr's sorted rows qualify; any other
 * CSR goes through hc_csr_check_lower_first / hc_csr_partition_lower_first,
 * which the Python layer does for every caller-supplied graph).  thr_count = ceil(H*n)
 * computed by the host exactly as driver.py:138.  Output d_colors int64[n]
 * (0 never appears on success).  d_rec receives up to max_rec round records;
 * *h_rounds = total rounds.  If rounds > max_rec the solve still completes,
 * the first max_rec records are kept and HC_ERR_RECORDS is returned. */
size_t hc_solve_workspace_bytes(int64_t num_nodes, int64_t num_edges);
/* Storage-format overrides for tests and experiments (per calling host thread):
 * force int64 row offsets, forbid 16-bit state words, forbid 16-bit delta
 * columns.  Defaults (0, 0, 0) let hc_solve pick per graph. */
int hc_solve_set_formats(int force_wide_offsets, int no_x16, int no_c16);
/* Graphs whose every degree is <= 16 (grids, meshes, road networks) run a
 * bin-0-only instantiation (less shared memory, more resident CTAs);
 * allow = 0 forces the general kernel (tests / experiments). */
int hc_solve_set_small(int allow);
/* Bin-0-only graphs whose every degree is <= 4 and every |v-u| < 2^15
 * (grids) store each row as one 8-byte word of int16 deltas (ELL4) next to
 * the CSR and run the ELL4 instantiation; allow = 0 forces the offset +
 * column path (per calling host thread; tests / experiments). */
int hc_solve_set_ell(int allow);
/* Graphs whose every degree is <= 128 (ER-2^25, grids) keep 8-bit state words
 * (colors <= 127; a larger tentative color redoes the solve with 16-bit
 * words); allow = 0 forces 16-bit words (per calling host thread). */
int hc_solve_set_x8(int allow);
/* Live lower lists (resolve keeps each node's still-uncolored lower
 * neighbours, compacted in place): mode -1 = per graph (hubs present and
 * >= 2^25 half-edges), 0 = off, 1 = on (per calling host thread). */
int hc_solve_set_live(int mode);
/* L2 residency of the state words (per calling host thread).  When the
 * state-word array is 16 MB .. L2/3 and the graph is bin-0-only (every
 * degree <= 16: grids and meshes of ~8-40 M nodes) hc_solve launches the solve kernel with the array as a persisting
 * access-policy window and sets the device's persisting set-aside
 * (cudaLimitPersistingL2CacheSize, a device-wide limit) to exactly its
 * size; after the solve a stream-ordered pass demotes those lines to normal
 * (the context's other persisting lines are left alone).  allow = 0: never
 * touch the limit or set a window. */
int hc_solve_set_l2_window(int allow);
int hc_solve(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
             int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors,
             hc_round_rec *d_rec, int64_t max_rec, int64_t *h_rounds, void *d_ws,
             size_t ws_bytes, void *stream);

/* hc_solve plus per-round edge-visit statistics (for the roofline's
 * algorithmic byte count): d_stats int64[2*max_rec], round t (1-based) gets
 * d_stats[2(t-1)] = sum of degrees over nodes assigned in round t and
 * d_stats[2(t-1)+1] = lower-id neighbours scanned by resolve in round t. */
int hc_solve_stats(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                   int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors,
                   hc_round_rec *d_rec, int64_t max_rec, int64_t *h_rounds, int64_t *d_stats,
                   void *d_ws, size_t ws_bytes, void *stream);

/* Graph-capturable solve: a per-graph plan plus sync-free launches.
 *
 * hc_solve_plan runs the per-graph preprocessing of hc_solve once (degree
 * binning, narrowed offsets, delta / ELL4 columns) into d_ws, reads the
 * verdicts back (ONE host synchronisation) and fixes the kernel choice in
 * *h_plan.  16-bit state words are planned only where they are exact
 * (max degree <= 16384), so a launch never needs the 32-bit redo.
 *
 * hc_solve_launch then solves on the planned graph with stream-ordered work
 * only (state reset, the cooperative solve kernel, the L2 demotion, a
 * device-to-device copy of (rounds, record overflow / stall flag, format
 * overflow) into d_info int64[3]): no host synchronisation, so it can be
 * captured into a CUDA graph and replayed.  d_ws must be the planned
 * workspace and the graph must be unchanged; results equal hc_solve's.
 * d_info[1] != 0 means HC_ERR_RECORDS (1) or HC_ERR_STALLED (2). */
typedef struct hc_solve_plan {
    int64_t num_nodes, num_edges;
    int32_t narrow, x16, c16, small, ell, live;
    int64_t totals_offset;  /* bucket totals inside d_ws (copied into each launch's control block) */
    int64_t reserved[3];
} hc_solve_plan;
int hc_solve_plan_graph(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                        int64_t num_edges, void *d_ws, size_t ws_bytes, hc_solve_plan *h_plan, void *stream);
int hc_solve_launch(const hc_solve_plan *h_plan, const int64_t *d_row_offsets, const int32_t *d_col_indices,
                    int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec, int64_t max_rec,
                    int64_t *d_info, void *d_ws, size_t ws_bytes, void *stream);

/* Bench-only "Plain" data-driven baseline (the paper's IrGL Plain,
 * PAPER.md:268-283, 301-332): the same solve, but losers are pushed with
 * warp-aggregated atomics into one dense, unordered list per degree bin
 * (_kernels.pyx:114-118 without the sort of worklist.py:84), so data-driven
 * rounds walk a fragmented list.  Same arguments and results as hc_solve. */
int hc_solve_plain(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                   int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec,
                   int64_t max_rec, int64_t *h_rounds, void *d_ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ */
/* Device-resident multi-GPU solve over NVLink peer memory (SURVEY.md   */
/* §8(e); replaces driver.py:122-176 on a 1D vertex partition).  One    */
/* process (or one stream) per rank; rank r owns nodes [lo, hi) and     */
/* runs ONE persistent kernel for the whole solve.  Every rank has a    */
/* "shared region" (hc_mg_shared_bytes, zero-initialised once by the    */
/* caller) holding its replica of the state words plus a mailbox; all   */
/* ranks' regions are mapped into every rank (hc_mg_ipc_* between       */
/* processes, plain pointers within one).  Owned boundary words are     */
/* stored straight into every peer's replica (NVLink stores), and the   */
/* per-round grid barriers are cross-GPU barriers that also all-reduce  */
/* (|W'|, conflicts) for the identical hybrid decision on every rank    */
/* (driver.py:145-152).  Colors, rounds and per-round records are       */
/* bit-identical to hc_solve for every partition.                       */
/*   h_bounds[world+1]: the partition (rank r owns [h_bounds[r],        */
/*     h_bounds[r+1]); every rank passes the same array).  A boundary   */
/*     word goes only to the ranks holding a neighbour of it.           */
/*   The CSR is the rank's SHARD ("each GPU holds its  */
/*     CSR rows"): d_row_offsets int64[hi-lo+1] (row r = node lo+r,     */
/*     offsets into d_col_indices), d_col_indices int32[num_edges]      */
/*     (global ids; num_edges = the shard's half-edges), rows as        */
/*     build_csr makes them (hc_build_csr_rows).  num_nodes is global;  */
/*     global_max_degree (the all-reduced max over ranks) fixes the     */
/*     state-word width and kernel family, which every rank must share. */
/*   hc_mg_solve: preprocessing (synchronous) + launch (asynchronous);  */
/*     d_colors int64[hi-lo] receives the owned colors; every rank's    */
/*     d_rec gets the same global records; ctas = 0: all resident CTAs; */
/*     timeout_ms bounds each cross-GPU wait (<= 0: 60 s).  ctas > 0:   */
/*     the caller sizes the grid (several ranks sharing one GPU, e.g.   */
/*     tests) and guarantees co-residency; it is a regular launch.      */
/*   hc_mg_wait: synchronises the stream, *h_rounds = rounds; returns   */
/*     HC_ERR_TIMEOUT if a peer missed a barrier (the shared regions    */
/*     must then be re-zeroed on every rank before the next solve).     */
/* ------------------------------------------------------------------ */
#define HC_IPC_HANDLE_BYTES 64
size_t hc_mg_shared_bytes(int64_t num_nodes);
size_t hc_mg_workspace_bytes(int64_t num_nodes, int64_t shard_edges, int64_t lo, int64_t hi);
/* The one allocation the library makes: a shared region in its own
 * cudaMalloc allocation (zeroed), so it is IPC-exportable whatever the
 * caller's allocator does (e.g. virtual-memory segments).  Freed by
 * hc_mg_free_shared after every peer closed its mapping. */
int hc_mg_alloc_shared(size_t bytes, void **h_dptr);
int hc_mg_free_shared(void *d_ptr);
/* export a device pointer for another process: cudaIpc handle of the
 * allocation that contains it + the pointer's offset in it */
int hc_mg_ipc_export(const void *d_ptr, void *h_handle, int64_t *h_offset);
int hc_mg_ipc_import(const void *h_handle, int64_t offset, void **h_dptr);
int hc_mg_ipc_close(void *d_ptr, int64_t offset);
int hc_mg_solve(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                int64_t num_edges, const int64_t *h_bounds, int rank, int world, void *const *h_shared,
                int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec, int64_t max_rec,
                int ctas, int64_t timeout_ms, int64_t global_max_degree, void *d_ws, size_t ws_bytes,
                void *stream);
/* hc_mg_solve == hc_mg_prepare + hc_mg_launch.  Ranks sharing one GPU
 * prepare all ranks first, then launch all (preprocessing kernels must not
 * queue behind another rank's persistent kernel). */
int hc_mg_prepare(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                  int64_t num_edges, const int64_t *h_bounds, int rank, int world, void *const *h_shared,
                  int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec, int64_t max_rec,
                  int ctas, int64_t timeout_ms, int64_t global_max_degree, void *d_ws, size_t ws_bytes,
                  void *stream);
int hc_mg_launch(void *d_ws, void *stream);
int hc_mg_wait(void *d_ws, int64_t *h_rounds, void *stream);
/* How a rank's boundary words reach its peers (per calling host thread; tests /
 * experiments): 0 = per round, the cheaper of (1) mirroring every boundary
 * store and (2) copying the boundary zones at the end of each phase. */
int hc_mg_set_exchange(int mode);

/* ------------------------------------------------------------------ */
/* 1D-partitioned multi-GPU solve: per-phase kernels  */
/* over the owned range [lo, hi) with a replicated state word X[n]      */
/* (0 / T / C|0x80000000).  Collectives between phases are the caller's */
/* (torch.distributed / NCCL).  Work items: d_list[0..count) or, when   */
/* d_list is NULL, the topology sweep lo..lo+count-1 with the activity   */
/* test.  Boundary flags are relative to lo (flags[u-lo]); only boundary */
/* nodes emit exchange pairs.  Counters are device int64, accumulated.   */
/* ------------------------------------------------------------------ */
int hc_dist_boundary(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t lo, int64_t hi,
                     uint8_t *d_flags, void *stream);
int hc_dist_assign(const int64_t *d_row_offsets, const int32_t *d_col_indices, uint32_t *d_X,
                   const int32_t *d_list, int64_t count, int64_t lo, const uint8_t *d_boundary,
                   int32_t *d_out_ids, uint32_t *d_out_vals, int64_t *d_out_cnt, void *stream);
int hc_dist_resolve(const int64_t *d_row_offsets, const int32_t *d_col_indices, uint32_t *d_X,
                    const int32_t *d_list, int64_t count, int64_t lo, const uint8_t *d_boundary,
                    int32_t *d_next, int64_t *d_next_cnt, int32_t *d_out_ids, uint32_t *d_out_vals,
                    int64_t *d_out_cnt, int64_t *d_conflicts, void *stream);
int hc_dist_apply(uint32_t *d_X, const int32_t *d_ids, const uint32_t *d_vals, int64_t count, void *stream);
int hc_dist_colors(const uint32_t *d_X, int64_t lo, int64_t hi, int64_t *d_colors, void *stream);

/* ------------------------------------------------------------------ */
/* §3 micro-benchmark pair (bench.py:67-161, _kernels.pyx:152-187):     */
/* one persistent kernel runs the whole pipe of `variant` (0 push_wl,   */
/* 1 push_nowl) over n nodes deactivating `batch` lowest-id active     */
/* nodes per iteration; per iteration it records the push phase's      */
/* device nanoseconds, the worklist size before, and the cutoff id.    */
/* ------------------------------------------------------------------ */
size_t hc_push_bench_workspace_bytes(int64_t num_nodes);
int hc_push_bench(int64_t num_nodes, int64_t batch, int variant, int64_t *d_rec_ns, int64_t *d_rec_size,
                  int64_t *d_rec_cutoff, int64_t max_iters, int64_t *h_iters, void *d_ws, size_t ws_bytes,
                  void *stream);

/* ------------------------------------------------------------------ */
/* Graph construction / generators / verification.                      */
/* ------------------------------------------------------------------ */

/* build_csr (graph.py:184-201) on device: d_edges int64[2*m] (src,dst pairs,
 * all in [0,n)).  Outputs d_row_offsets int64[n+1] and d_col_indices int32
 * with capacity 2*m; *h_num_edges = directed half-edges after symmetrise /
 * drop loops / dedupe.  Workspace sized by hc_build_csr_workspace_bytes. */
size_t hc_build_csr_workspace_bytes(int64_t num_nodes, int64_t num_pairs);
int hc_build_csr(const int64_t *d_edges, int64_t num_pairs, int64_t num_nodes,
                 int64_t *d_row_offsets, int32_t *d_col_indices, int64_t *h_num_edges,
                 void *d_ws, size_t ws_bytes, void *stream);

/* Rows [lo, hi) of build_csr (a multi-GPU shard): d_row_offsets
 * int64[hi-lo+1] (row r = node lo+r), d_col_indices int32[dir_capacity] with
 * global ids; dir_capacity >= the rows' directed entries before dedupe (their
 * hc_edge_degrees sum), else HC_ERR_WORKSPACE.  Rows equal the same rows of
 * hc_build_csr (graph.py:184-201).  hc_build_csr == rows [0, n). */
size_t hc_build_csr_rows_workspace_bytes(int64_t num_nodes, int64_t lo, int64_t hi, int64_t dir_capacity);
int hc_build_csr_rows(const int64_t *d_edges, int64_t num_pairs, int64_t num_nodes, int64_t lo, int64_t hi,
                      int64_t dir_capacity, int64_t *d_row_offsets, int32_t *d_col_indices,
                      int64_t *h_num_edges, void *d_ws, size_t ws_bytes, void *stream);
/* d_deg int64[n]: per node the half-edges of the pair list with loops
 * dropped and duplicates kept (graph.py:191-192 before np.unique) -- the
 * prefix the multi-GPU partition is cut on before any shard exists. */
int hc_edge_degrees(const int64_t *d_edges, int64_t num_pairs, int64_t num_nodes, int64_t *d_deg, void *stream);

/* Synthetic edge streams (bit-identical to
 * oracle/ipgc_oracle.c orc_gen_*).  d_edges int64[2*m]. */
int hc_gen_grid(int64_t rows, int64_t cols, int64_t *d_edges, void *stream);
int hc_gen_er(int64_t num_nodes, int64_t num_pairs, uint64_t seed, int64_t *d_edges, void *stream);
int hc_gen_rmat(int scale, int64_t num_pairs, uint64_t seed, int64_t *d_edges, void *stream);

/* verify_coloring (driver.py:188-204): *h_bad = #edges u<v with equal colors
 * or colors[u]==0.  colors_used (driver.py:179-185): max color, 0 for n==0,
 * HC_ERR_UNCOLORED if any entry < 1. */
int hc_verify(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
              const int64_t *d_colors, int64_t *d_acc, int64_t *h_bad, void *stream);
/* verify_coloring over a shard's rows [lo, hi) (row offsets as in
 * hc_build_csr_rows; d_colors indexed by global id) -- the multi-GPU
 * RunReport sums it over ranks. */
int hc_verify_rows(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t lo, int64_t hi,
                   const int64_t *d_colors, int64_t *d_acc, int64_t *h_bad, void *stream);
/* d_acc: int64[2] device scratch */
int hc_colors_used(const int64_t *d_colors, int64_t num_nodes, int64_t *d_acc, int64_t *h_used,
                   void *stream);
/* MatrixMarket coordinate entries (graph.py:105-181) parsed on the device.
 * d_bytes = the file content AFTER the size line (the host parses banner and
 * size line); universal_newlines: '\r' also ends a line (files read in text
 * mode).  Entry k (k-th non-blank, non-comment line) -> d_edges[2k..2k+1] =
 * (row-1, col-1), int64[2*nnz].  On return *h_num_entries = entry lines; if
 * some line is bad, *h_err_line / *h_err_code / h_err_span[2] (byte span)
 * name the FIRST bad line (the reference raises there), else *h_err_line=-1.
 * *h_first_nonascii = offset of the first byte >= 0x80 or -1. */
#define HC_MTX_FEW_FIELDS 1  /* "entry needs at least two coordinates" */
#define HC_MTX_NON_INTEGER 2 /* "non-integer coordinate"               */
#define HC_MTX_BOUNDS 3      /* "coordinate (r, c) outside declared bounds" */
#define HC_MTX_TOO_MANY 4    /* "more than the declared nnz entries"   */
size_t hc_mtx_workspace_bytes(int64_t num_bytes);
int hc_mtx_parse(const uint8_t *d_bytes, int64_t num_bytes, int universal_newlines, int64_t rows, int64_t cols,
                 int64_t nnz, int64_t *d_edges, int64_t *h_num_entries, int64_t *h_err_line, int *h_err_code,
                 int64_t *h_err_span, int64_t *h_first_nonascii, void *d_ws, size_t ws_bytes, void *stream);

/* degree_stats (graph.py:204-217): min, max and the element at sorted index
 * n/2 (np.partition) of the degree array, on the device (radix select). */
size_t hc_degree_stats_workspace_bytes(void);
int hc_degree_stats(const int64_t *d_row_offsets, int64_t num_nodes, int64_t *h_min, int64_t *h_median,
                    int64_t *h_max, void *d_ws, size_t ws_bytes, void *stream);

/* int64 -> int32 column conversion for uploads of reference CsrGraph arrays */
int hc_narrow_i64_i32(const int64_t *d_in, int32_t *d_out, int64_t count, void *stream);
/* Lower-id-first rows.  hc_solve / hc_mg_solve stop a row's conflict scan at
 * its first neighbour >= u, so they need each row's lower-id neighbours to be
 * a prefix of the row (true for build_csr output, graph.py:193-197, which is
 * sorted).  The reference scans whole rows (_kernels.pyx:106-113), so it
 * accepts any order; callers with an arbitrary CSR run the check and, when it
 * reports rows, the stable partition (v < u first) into a second column array.
 * Colors and every record are row-order independent, so the result is the
 * reference's.  d_acc: int64[1] device scratch. */
int hc_csr_check_lower_first(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                             int64_t *d_acc, int64_t *h_bad_rows, void *stream);
int hc_csr_partition_lower_first(const int64_t *d_row_offsets, const int32_t *d_col_in, int32_t *d_col_out,
                                 int64_t num_nodes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HCB_H_ */
