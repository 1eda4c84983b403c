/*
 * tf_oracle.h -- CPU restatement of the reference tile-fusion path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the libtfg CUDA
 * library, the paper_2407_00243_b200 package, the C++ mirror headers) may
 * link, load or call this.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py use it, and only as the
 * checker or the timed CPU baseline.
 *
 * Parity status: PINNED.  The restatement is checked (tests/test_oracle_pins.py)
 * against (1) the known-answer values hard-coded in the reference's own unit
 * tests (test_scheduler.cpp, test_kernels.cpp, tests/python/test_smoke.py) and
 * (2) golden vectors produced by the reference itself, compiled from
 * /root/reference/proj/src by oracle/Makefile into oracle/_ref/ and dumped by
 * tests/golden/make_golden.py.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 */
#ifndef TF_ORACLE_H
#define TF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirror of tilefuse::SchedulerConfig (include/tilefuse/scheduler.hpp:15-24). */
typedef struct {
  int32_t ct_size;
  int32_t num_workers;
  uint64_t cache_size_words;
  int32_t b_cols;
  int32_t c_cols;
  double index_to_scalar_ratio;
  int32_t b_is_dense;
  int32_t whole_b_cost;
} tfo_config;

/* Flat two-wavefront schedule (FusedSchedule, scheduler.hpp:39-49).
 * Wave w has n_tiles[w] tiles; tile v owns j_rows[w][j_off[w][v] .. j_off[w][v+1]). */
typedef struct {
  int32_t n;
  int32_t tile_size;
  int64_t n_tiles[2];
  int32_t *i_lo[2];
  int32_t *i_hi[2];
  double *cost[2];
  int64_t *j_off[2];
  int32_t *j_rows[2];
} tfo_schedule;

/* status: 0 ok, 1 invalid_argument, 2 runtime error; message via tfo_last_error */
const char *tfo_last_error(void);

int tfo_choose_tile_size(int32_t n, int32_t p, int32_t ct, int32_t *out);

/* step1_coarse_fuse (scheduler.cpp:131-161).  tile_j_off has ceil(n/t)+1
 * entries, tile_j_rows and unfused have n entries capacity.  */
int tfo_step1(int32_t n_rows, int32_t n_cols, const int32_t *row_ptr,
              const int32_t *col_idx, int32_t t, int64_t *tile_j_off,
              int32_t *tile_j_rows, int32_t *unfused, int64_t *n_unfused);

/* balance (scheduler.cpp:163-194); chunk_off has num_chunks+1 entries */
int tfo_balance(const int32_t *rows, int64_t m, const int32_t *row_weight,
                int64_t num_chunks, int64_t *chunk_off);

/* tile_cost (scheduler.cpp:29-64, 196-200) */
int tfo_tile_cost(int32_t n_rows, const int32_t *row_ptr,
                  const int32_t *col_idx, int32_t i_lo, int32_t i_hi,
                  const int32_t *j_rows, int64_t nj, const tfo_config *cfg,
                  double *out);

/* split_tile (scheduler.cpp:202-210).  Output is a 1-wave tfo_schedule in
 * wave 0 (pieces) plus demoted rows (sorted) in a malloc'd array. */
int tfo_split_tile(int32_t n_rows, const int32_t *row_ptr,
                   const int32_t *col_idx, int32_t i_lo, int32_t i_hi,
                   const int32_t *j_rows, int64_t nj, const tfo_config *cfg,
                   tfo_schedule *pieces, int32_t **demoted, int64_t *n_demoted);

/* build_schedule (scheduler.cpp:212-245) */
int tfo_build_schedule(int32_t n_rows, int32_t n_cols, const int32_t *row_ptr,
                       const int32_t *col_idx, const tfo_config *cfg,
                       tfo_schedule *out);
void tfo_schedule_free(tfo_schedule *s);
void tfo_free(void *p);

/* fused_ratio (scheduler.cpp:247-252) */
double tfo_fused_ratio(const tfo_schedule *s);

/* validate_schedule (scheduler.cpp:254-390).  Returns pass (1/0); writes the
 * number of violations, the width-1 over-budget count and the first message. */
int tfo_validate_schedule(int32_t n_rows, int32_t n_cols,
                          const int32_t *row_ptr, const int32_t *col_idx,
                          const tfo_schedule *s, const tfo_config *cfg,
                          int64_t *n_violations, int64_t *over_budget_width1,
                          char *first_msg, size_t msg_cap);
/* all violation messages joined by '\n' (malloc'd) */
int tfo_validate_schedule_all(int32_t n_rows, int32_t n_cols,
                              const int32_t *row_ptr, const int32_t *col_idx,
                              const tfo_schedule *s, const tfo_config *cfg,
                              char **messages);

/* Executors (kernels.hpp:88-155, 182-236).  sched == NULL runs the unfused
 * two-phase order.  b_row_ptr == NULL means B is dense (n x b_cols row
 * major); otherwise B is CSR with b_cols columns.  C is b_cols x c_cols.
 * d is n x c_cols (overwritten).  stats (3 x int64, may be NULL) accumulate
 * first_op_rows, second_op_rows, nnz_processed as RunStats does. */
int tfo_run_f64(int32_t n, const int32_t *a_row_ptr, const int32_t *a_col_idx,
                const double *a_val, const int32_t *b_row_ptr,
                const int32_t *b_col_idx, const double *b_val,
                const double *b_dense, int32_t b_cols, const double *c,
                int32_t c_cols, const tfo_schedule *sched, double *d,
                int64_t *stats);
int tfo_run_f32(int32_t n, const int32_t *a_row_ptr, const int32_t *a_col_idx,
                const float *a_val, const int32_t *b_row_ptr,
                const int32_t *b_col_idx, const float *b_val,
                const float *b_dense, int32_t b_cols, const float *c,
                int32_t c_cols, const tfo_schedule *sched, float *d,
                int64_t *stats);
/* Same as tfo_run_* but with the reference's OpenMP structure across
 * `workers` threads (kernels.hpp:105-106 dynamic,1 per wavefront;
 * kernels.hpp:138-149 static for unfused).  Used for the CPU baseline. */
int tfo_run_f64_mt(int32_t n, const int32_t *a_row_ptr,
                   const int32_t *a_col_idx, const double *a_val,
                   const int32_t *b_row_ptr, const int32_t *b_col_idx,
                   const double *b_val, const double *b_dense, int32_t b_cols,
                   const double *c, int32_t c_cols, const tfo_schedule *sched,
                   double *d, int workers);
int tfo_run_f32_mt(int32_t n, const int32_t *a_row_ptr,
                   const int32_t *a_col_idx, const float *a_val,
                   const int32_t *b_row_ptr, const int32_t *b_col_idx,
                   const float *b_val, const float *b_dense, int32_t b_cols,
                   const float *c, int32_t c_cols, const tfo_schedule *sched,
                   float *d, int workers);

/* ---- deterministic generators used by the reference tests ------------ */
/* std::mt19937_64 raw outputs */
void tfo_mt64_stream(uint64_t seed, uint64_t *out, int64_t count);
/* gen_random_sparse<double> (generate.hpp:15-63): malloc'd CSR */
int tfo_gen_random_sparse(int32_t n, double density, uint64_t seed,
                          int32_t **row_ptr, int32_t **col_idx,
                          double **values);
/* gen_banded (generate.hpp:66-94) */
int tfo_gen_banded(int32_t n, int32_t half_bw, int32_t **row_ptr,
                   int32_t **col_idx, double **values);
/* tests/support.hpp:68-75 random_dense: U(-1,1) via libstdc++
 * uniform_real_distribution over mt19937_64; writes rows*cols doubles */
void tfo_random_dense(int32_t rows, int32_t cols, uint64_t seed, double *out);
/* tests/support.hpp:50-66 gen_rect_random */
int tfo_gen_rect_random(int32_t rows, int32_t cols, double density,
                        uint64_t seed, int32_t **row_ptr, int32_t **col_idx,
                        double **values);

#ifdef __cplusplus
}
#endif
#endif
