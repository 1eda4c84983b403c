/*
 * tfg.h -- C-ABI of libtfg, the B200 (sm_100a) tile-fusion library for
 * D = A (B C):  A square CSR, C dense, B dense (GeMM-SpMM) or CSR
 * (SpMM-SpMM).
 *
 * This is the drop-in boundary under the reference's C++ operator API.  The
 * reference (arXiv 2407.00243 artifact, /root/reference/proj) is a
 * header-only C++ template library with no FFI; the C++ headers in
 * include/tilefuse/ keep its names and signatures and forward to these
 * entry points.  Each function cites the reference interface it replaces.
 *
 * Conventions
 *   - plain pointers and sizes, no torch / C++ types;
 *   - every function returns a tfg_status; tfg_last_error() holds the
 *     message of the last failure on the calling thread;
 *   - TFG_EINVAL maps to std::invalid_argument and TFG_ERUNTIME to
 *     std::runtime_error in the C++ mirror, as the reference throws them;
 *   - "d_" pointers are device (HBM) pointers, "h_" pointers host pointers;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *     All device work is asynchronous on that stream unless stated.
 * There is no CPU fallback: every compute entry point launches sm_100a
 * kernels and fails with TFG_ECUDA when no B200 is present.
 */
#ifndef TFG_H
#define TFG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TFG_OK = 0,
  TFG_EINVAL = 1,   /* std::invalid_argument in the reference */
  TFG_ERUNTIME = 2, /* std::runtime_error in the reference    */
  TFG_ECUDA = 3     /* CUDA error / no device                  */
} tfg_status;

typedef enum { TFG_F32 = 0, TFG_F64 = 1 } tfg_dtype;

/* == tilefuse::SchedulerConfig (include/tilefuse/scheduler.hpp:15-24),
 * same field order, meaning and defaults (tfg_config_default). */
typedef struct {
  int32_t ct_size;              /* coarse tile width heuristic (2048)   */
  int32_t num_workers;          /* p (1)                                 */
  uint64_t cache_size_words;    /* per-worker budget in scalars (163840) */
  int32_t b_cols;               /* columns of B when dense (32)          */
  int32_t c_cols;               /* columns of C (32)                     */
  double index_to_scalar_ratio; /* index word / scalar word (0.5)        */
  int32_t b_is_dense;           /* GeMM-SpMM when 1 (1)                  */
  int32_t whole_b_cost;         /* charge all of B (0)                   */
} tfg_config;

typedef struct tfg_schedule tfg_schedule; /* device-resident FusedSchedule */
typedef struct tfg_plan tfg_plan;         /* executor plan bound to a problem */

const char *tfg_last_error(void);
void tfg_config_default(tfg_config *cfg);
/* library build / device facts: writes the sm arch the code was built for
 * (100 for sm_100a) and the number of SMs of the current device (0 if none) */
tfg_status tfg_device_info(int32_t *built_arch, int32_t *sm_count);

/* ---------------------------------------------------------------------
 * Inspector (replaces scheduler.hpp:67-111 / scheduler.cpp:124-252)
 * ------------------------------------------------------------------- */

/* choose_tile_size -- scheduler.hpp:67, scheduler.cpp:124-129.
 * Host arithmetic on three scalars.  EINVAL if any input < 1. */
tfg_status tfg_choose_tile_size(int32_t n, int32_t num_workers,
                                int32_t ct_size, int32_t *out);

/* build_schedule -- scheduler.hpp:101-102, scheduler.cpp:212-245.
 * GPU inspector over a device-resident CSR pattern (row_ptr n_rows+1,
 * col_idx nnz; columns strictly increasing per row).  Produces a schedule
 * bit-identical to the reference's (tile order, i ranges, j lists and
 * double costs) for the same config.  EINVAL for non-square / empty input
 * or config values < 1 (scheduler.cpp:115-128).  Synchronises `stream`
 * before returning (the schedule's shape is needed on the host). */
tfg_status tfg_build_schedule(int32_t n_rows, int32_t n_cols, int64_t nnz,
                              const int32_t *d_row_ptr,
                              const int32_t *d_col_idx,
                              const tfg_config *cfg, void *stream,
                              tfg_schedule **out);

/* Same, from host arrays (copies the pattern to the device first): the
 * entry the C++ mirror's build_schedule(const SparsityView&, ...) uses. */
tfg_status tfg_build_schedule_host(int32_t n_rows, int32_t n_cols,
                                   const int32_t *h_row_ptr,
                                   const int32_t *h_col_idx,
                                   const tfg_config *cfg, void *stream,
                                   tfg_schedule **out);

/* Sizes of a schedule: n, tile size t, tiles per wavefront, j rows per
 * wavefront, and the inspector's device time in seconds. */
tfg_status tfg_schedule_info(const tfg_schedule *s, int32_t *n,
                             int32_t *tile_size, int64_t n_tiles[2],
                             int64_t n_jrows[2], double *inspect_seconds);

/* Flat export of wavefront `wave` into host buffers sized from
 * tfg_schedule_info: i_lo/i_hi/cost[n_tiles], j_off[n_tiles+1] (int64),
 * j_rows[n_jrows].  Any pointer may be NULL to skip that array. */
tfg_status tfg_schedule_export(const tfg_schedule *s, int wave,
                               int32_t *h_i_lo, int32_t *h_i_hi,
                               double *h_cost, int64_t *h_j_off,
                               int32_t *h_j_rows);

/* Import a schedule built elsewhere (e.g. by the reference, or reloaded
 * from schedule JSON, schedule_io.cpp:28-54) from host flat arrays. */
tfg_status tfg_schedule_import(int32_t n, int32_t tile_size,
                               const int64_t n_tiles[2],
                               const int32_t *const h_i_lo[2],
                               const int32_t *const h_i_hi[2],
                               const double *const h_cost[2],
                               const int64_t *const h_j_off[2],
                               const int32_t *const h_j_rows[2],
                               tfg_schedule **out);

void tfg_schedule_destroy(tfg_schedule *s);

/* fused_ratio -- scheduler.hpp:105, scheduler.cpp:247-252 (Eq. 2). */
double tfg_fused_ratio(const tfg_schedule *s);

/* validate_schedule -- scheduler.hpp:109-111, scheduler.cpp:254-390.
 * Host-side checker over host CSR pattern + a schedule (the verify path,
 * not the hot path).  *pass = 1 when no violation; the first message goes
 * to msg (may be NULL); tfg_validate_messages returns all of them. */
tfg_status tfg_validate_schedule(int32_t n_rows, int32_t n_cols,
                                 const int32_t *h_row_ptr,
                                 const int32_t *h_col_idx,
                                 const tfg_schedule *s, const tfg_config *cfg,
                                 int32_t *pass, int64_t *n_violations,
                                 int64_t *over_budget_width1, char *msg,
                                 size_t msg_cap);

/* Every violation message of the calling thread's last
 * tfg_validate_schedule, newline separated (ValidationReport::violations,
 * scheduler.hpp:60-65).  *needed = bytes including the terminator. */
tfg_status tfg_validate_messages(char *buf, size_t cap, size_t *needed);

/* tile_cost -- scheduler.hpp:86-87, scheduler.cpp:196-200 (Eq. 3 over the
 * tile's j rows; distinct columns anywhere in the matrix).  Host pattern;
 * runs the inspector's cost kernel on the device. */
tfg_status tfg_tile_cost(int32_t n, const int32_t *h_row_ptr, const int32_t *h_col_idx,
                         int32_t i_lo, int32_t i_hi, const int32_t *h_j_rows, int64_t n_j,
                         const tfg_config *cfg, double *cost);

/* split_tile -- scheduler.hpp:89-97, scheduler.cpp:66-93 / :202-210: the
 * inspector's split kernel on one tile whose j rows read only columns in
 * [i_lo, i_hi) (the tiles step 1 produces; EINVAL otherwise).  Pieces in DFS
 * pre-order (cost-bounded or width 1), j rows per piece by h_j_off; demoted
 * rows ascending.  Buffers: pieces <= i_hi - i_lo, j / demoted <= n_j. */
tfg_status tfg_split_tile(int32_t n, const int32_t *h_row_ptr, const int32_t *h_col_idx,
                          int32_t i_lo, int32_t i_hi, const int32_t *h_j_rows, int64_t n_j,
                          const tfg_config *cfg, int64_t *n_pieces, int32_t *h_lo,
                          int32_t *h_hi, double *h_cost, int64_t *h_j_off, int32_t *h_j_out,
                          int64_t *n_demoted, int32_t *h_demoted);

/* balance -- scheduler.hpp:80-82, scheduler.cpp:163-194: greedy contiguous
 * chunking of a weight list (the inspector's k_balance).  h_chunk_start
 * [num_chunks + 1]: chunk c is items [start[c], start[c + 1]); trailing
 * chunks may be empty.  EINVAL when num_chunks < 1. */
tfg_status tfg_balance(int64_t n_items, const int64_t *h_weights, int64_t num_chunks,
                       int64_t *h_chunk_start);

/* ---------------------------------------------------------------------
 * Executor (replaces kernels.hpp:182-236: fused_gemm_spmm,
 * fused_spmm_spmm, unfused_gemm_spmm, unfused_spmm_spmm)
 * ------------------------------------------------------------------- */

/* FusedProblem<T> (kernels.hpp:16-43) as device pointers. */
typedef struct {
  int32_t dtype;      /* tfg_dtype                                    */
  int32_t n;          /* A is n x n                                   */
  int32_t b_is_dense; /* 1: B dense n x b_cols; 0: B CSR n x b_cols   */
  int32_t b_rows;     /* must equal n   (kernels.hpp:38-39)           */
  int32_t b_cols;
  int32_t c_rows;     /* must equal b_cols (kernels.hpp:40-41)         */
  int32_t c_cols;
  int64_t a_nnz;
  int64_t b_nnz;      /* CSR B only                                   */
  const int32_t *d_a_row_ptr;
  const int32_t *d_a_col_idx;
  const void *d_a_val;
  const int32_t *d_b_row_ptr; /* CSR B */
  const int32_t *d_b_col_idx;
  const void *d_b_val;
  const void *d_b_dense;      /* dense B, row-major n x b_cols */
  const void *d_c;            /* row-major c_rows x c_cols     */
} tfg_problem;

/* Bind a problem to a schedule (NULL = the unfused executor,
 * kernels.hpp:128-155 / 212-236) and precompute the device execution plan:
 * D1 spill set, tile work lists, long-row splits, scratch.  Checks exactly
 * what the reference executors check: problem.check() (kernels.hpp:35-42),
 * sched.n == n (kernels.hpp:93-94); the GeMM/SpMM distinction is the
 * problem's b_is_dense.  The schedule may be destroyed after this call. */
tfg_status tfg_plan_create(const tfg_problem *p, const tfg_schedule *s,
                           void *stream, tfg_plan **out);

/* Plan options (tfg_plan_create_ex).  Default: every SpMM term of a
 * grid-stencil row is one fused multiply-add (results within the north-star
 * tolerance of the reference, 1e-12 / 1e-5 max-norm).  REFERENCE_BITS: the
 * reference's separately rounded multiply and add in the same ascending
 * order (kernels.hpp:75-79), so SpMM results are bit-identical to it. */
#define TFG_PLAN_REFERENCE_BITS 1u

/* tfg_plan_create with options; row_lo = 0, row_hi = -1 is the whole
 * problem, a row block is a multi-GPU partition (tfg_plan_create_partition).
 * Device operands must be 16-byte aligned (cudaMalloc guarantees 256). */
tfg_status tfg_plan_create_ex(const tfg_problem *p, const tfg_schedule *s, uint32_t flags,
                              int32_t row_lo, int32_t row_hi, void *stream, tfg_plan **out);

/* Multi-GPU row-block partition: the plan of the rank owning
 * rows [row_lo, row_hi).  It runs the wavefront-0 tiles whose i_lo lies in
 * the block (the caller cuts at tile boundaries, so fused rows need no
 * remote D1) and the wavefront-1 rows j in the block; every D1 row some
 * wavefront-1 row reads is written to the plan's D1 buffer (global row
 * indexing) so it can be sent to peers.  D rows this rank computes are
 * written into d_d at their global positions. */
tfg_status tfg_plan_create_partition(const tfg_problem *p, const tfg_schedule *s,
                                     int32_t row_lo, int32_t row_hi,
                                     void *stream, tfg_plan **out);

/* The plan's D1 scratch (n x c_cols, dtype of the problem): the halo
 * exchange writes received rows into it between the two stages. */
tfg_status tfg_plan_d1(const tfg_plan *plan, void **d_d1);

/* Run one half of tfg_plan_execute: stage 0 = wavefront 0 (first op and
 * fused tiles), stage 1 = wavefront 1 (SpMM over D1).  The kernel boundary
 * between them is the wavefront barrier (kernels.hpp:118-119). */
tfg_status tfg_plan_execute_stage(tfg_plan *plan, int32_t stage, void *d_d,
                                  void *stream);

/* D = A (B C) into the caller's device buffer d_d (n x c_cols row-major,
 * fully overwritten).  Asynchronous on `stream`; no host synchronisation,
 * no allocation, no host<->device traffic. */
tfg_status tfg_plan_execute(tfg_plan *plan, void *d_d, void *stream);

/* RunStats (kernels.hpp:46-50) the plan's execution performs:
 * first_op_rows, second_op_rows (both n for a valid schedule). */
tfg_status tfg_plan_stats(const tfg_plan *plan, int64_t *first_op_rows,
                          int64_t *second_op_rows, int64_t *nnz_processed);

/* Plan facts for roofline accounting: number of D1 rows spilled to HBM
 * (|S|, rows read by wavefront 1), fused j rows, kernel launches per
 * execute, and bytes of device scratch held. */
tfg_status tfg_plan_info(const tfg_plan *plan, int64_t *spill_rows,
                         int64_t *fused_rows, int32_t *launches,
                         int64_t *scratch_bytes);

/* Which kernel runs each stage, as a NUL-terminated string of the form
 * "first_op=<k> fused=<k> wave1=<k>" (k: stencil3d, stencil2d, band, strip,
 * tcgen05, gemm, ...); for reports and tests.  Truncated to len - 1 chars. */
tfg_status tfg_plan_kernels(const tfg_plan *plan, char *buf, int32_t len);

/* Execute once with CUDA events around each stage on `stream`, wait, and
 * report device milliseconds and algorithmic HBM bytes (each input byte read
 * once, each output byte written once) per stage:
 *   [0] first op of wavefront-0 tiles that fuse no row (or all rows, unfused)
 *   [1] fused wavefront-0 tiles      [2] wavefront-1 / second-op SpMM.
 * Used for the roofline numbers; not for the hot loop. */
tfg_status tfg_plan_profile(tfg_plan *plan, void *d_d, void *stream,
                            double stage_ms[3], int64_t stage_bytes[3]);

void tfg_plan_destroy(tfg_plan *plan);

/* One-shot host entry used by the C++ mirror for the reference's
 * by-value API: copies host A, B, C to the device, builds the plan, runs
 * it and copies D back into h_d (n x c_cols).  Host pointers in `p`
 * (the d_ fields are read as host addresses).  s may be NULL (unfused). */
tfg_status tfg_run_host(const tfg_problem *host_problem,
                        const tfg_schedule *s, void *h_d);

/* Row-range helpers (kernels.hpp:159-180) on host operands, computed by the
 * GPU kernels.  gemm: rows [row_lo, row_hi) of D1 = B*C written into h_d1
 * (b_rows x c_cols; other rows untouched); EINVAL if b_cols != c_rows or the
 * range is out of bounds.  spmm: rows h_rows[] of D = A*X written into h_d
 * (a_rows x x_cols; other rows untouched); EINVAL if a_cols != x_rows. */
tfg_status tfg_gemm_rows_host(int32_t dtype, const void *h_b, int32_t b_rows,
                              int32_t b_cols, const void *h_c, int32_t c_rows,
                              int32_t c_cols, int32_t row_lo, int32_t row_hi,
                              void *h_d1);
tfg_status tfg_spmm_rows_host(int32_t dtype, int32_t a_rows, int32_t a_cols,
                              const int32_t *h_row_ptr, const int32_t *h_col_idx,
                              const void *h_values, const void *h_x,
                              int32_t x_rows, int32_t x_cols,
                              const int32_t *h_rows, int64_t n_rows, void *h_d);

/* ---------------------------------------------------------------------
 * Multi-GPU row-block partition.  The reference has no
 * distributed mode; its wavefront barrier (kernels.hpp:102-120) is where the
 * one exchange step sits: wavefront 0 is communication-free when the cuts
 * fall on tile boundaries (the dependence closure, scheduler.cpp:336-351),
 * and before wavefront 1 each rank needs the D1 rows its wavefront-1 rows
 * read from other blocks.  One process per GPU; the caller owns the NCCL
 * communicator (any NCCL already loaded in the process is used, else
 * libnccl.so.2).
 * ------------------------------------------------------------------- */
typedef struct tfg_halo tfg_halo;
#define TFG_HALO_AUTO 0      /* cost model picks EXCHANGE or RECOMPUTE          */
#define TFG_HALO_EXCHANGE 1  /* NCCL send/recv of the D1 halo rows              */
#define TFG_HALO_RECOMPUTE 2 /* GeMM-SpMM: halo D1 rows recomputed from local B */

/* NCCL communicator helpers (same NCCL library the exchange calls). */
tfg_status tfg_nccl_unique_id(void *id_out, size_t cap /* >= 128 */);
tfg_status tfg_nccl_comm_init(int32_t nranks, const void *id, int32_t rank, void **comm);
tfg_status tfg_nccl_comm_destroy(void *comm);

/* Row-block cuts for `world` ranks at wavefront-0 tile starts, balanced by
 * estimated bytes per row (first op + wavefront-1 gathers), written to
 * h_bounds[world + 1].  h_row_ptr: A's host row_ptr. */
tfg_status tfg_partition_bounds(const tfg_schedule *s, const int32_t *h_row_ptr,
                                int32_t b_cols, int32_t c_cols, int32_t dtype,
                                int32_t b_is_dense, int32_t world, int32_t *h_bounds);

/* The halo of rank `rank`'s partition plan (tfg_plan_create_partition /
 * _ex with its row block): per-peer recv / send D1 row lists computed on the
 * device from the replicated pattern and schedule; with EXCHANGE the
 * wavefront-1 rows that read only local D1 are split off so they run while
 * NCCL moves the halo.  mode: TFG_HALO_*; AUTO compares the NVLink time of
 * the halo rows with recomputing them from B (GeMM-SpMM only). */
tfg_status tfg_halo_create(tfg_plan *plan, const tfg_schedule *s, const int32_t *h_bounds,
                           int32_t world, int32_t rank, int32_t mode, void *stream,
                           tfg_halo **out);
tfg_status tfg_halo_info(const tfg_halo *h, int32_t *mode, int64_t *recv_rows,
                         int64_t *send_rows, double *t_exchange_us, double *t_recompute_us);
void tfg_halo_destroy(tfg_halo *h);

/* One step of the partitioned product on this rank into d_d (global row
 * indexing; this rank's rows written): wavefront 0; then the halo (grouped
 * ncclSend/ncclRecv on an internal stream, overlapped with the local-only
 * wavefront-1 rows) or its recomputation; then the remaining wavefront-1
 * rows.  nccl_comm: ncclComm_t (may be NULL for RECOMPUTE or world 1). */
tfg_status tfg_plan_execute_dist(tfg_plan *plan, tfg_halo *halo, void *nccl_comm, void *d_d,
                                 void *stream);

/* Test / debug: the step of ALL `world` ranks on one GPU, sequentially, the
 * NCCL transfer replaced by device copies between the ranks' halo buffers
 * (plans[r], halos[r], d[r] of rank r). */
tfg_status tfg_plan_execute_dist_emulated(tfg_plan **plans, tfg_halo **halos, int32_t world,
                                          void **d, void *stream);

/* Halo pack / unpack of D1 rows around a caller-driven exchange.  rows:
 * device int32 list. */
tfg_status tfg_gather_rows(int32_t dtype, const void *d_src, int32_t cols,
                           const int32_t *d_rows, int64_t n_rows,
                           void *d_dst, void *stream);
tfg_status tfg_scatter_rows(int32_t dtype, const void *d_src, int32_t cols,
                            const int32_t *d_rows, int64_t n_rows,
                            void *d_dst, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TFG_H */
