// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// the reference headers and sources where they lie under
// /root/reference/proj (nothing is copied into this repo) into
// oracle/_ref/libtfref.so, with the reference's own flags (-O3 -DNDEBUG
// -fopenmp, no -march: CMakeLists.txt:3-13).  Used to
//   * pin the C restatement (oracle/tf_oracle.c) against the real code,
//   * dump golden vectors (tests/golden/make_golden.py),
//   * time the reference CPU path (bench.py --impl reference and the
//     cpu_baseline leg).
// The product path never loads this library.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "tilefuse/csr.hpp"
#include "tilefuse/dense.hpp"
#include "tilefuse/generate.hpp"
#include "tilefuse/kernels.hpp"
#include "tilefuse/scheduler.hpp"
#include "../tests/support.hpp"  // resolved under /root/reference/proj/include/..

#include "tf_oracle.h"

using namespace tilefuse;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

SchedulerConfig to_cfg(const tfo_config* c) {
  SchedulerConfig cfg;
  cfg.ct_size = c->ct_size;
  cfg.num_workers = c->num_workers;
  cfg.cache_size_words = c->cache_size_words;
  cfg.b_cols = c->b_cols;
  cfg.c_cols = c->c_cols;
  cfg.index_to_scalar_ratio = c->index_to_scalar_ratio;
  cfg.b_is_dense = c->b_is_dense != 0;
  cfg.whole_b_cost = c->whole_b_cost != 0;
  return cfg;
}

SparsityView view(int32_t n_rows, int32_t n_cols, const int32_t* rp,
                  const int32_t* ci) {
  const std::size_t nnz = rp[n_rows];
  return SparsityView(n_rows, n_cols,
                      std::span<const index_t>(rp, (std::size_t)n_rows + 1),
                      std::span<const index_t>(ci, nnz));
}

void flatten(const std::vector<FusedTile>& tiles, tfo_schedule* out, int w) {
  const std::size_t nt = tiles.size();
  std::size_t total = 0;
  for (const auto& t : tiles) total += t.j_rows.size();
  out->n_tiles[w] = (int64_t)nt;
  out->i_lo[w] = (int32_t*)malloc((nt + 1) * sizeof(int32_t));
  out->i_hi[w] = (int32_t*)malloc((nt + 1) * sizeof(int32_t));
  out->cost[w] = (double*)malloc((nt + 1) * sizeof(double));
  out->j_off[w] = (int64_t*)malloc((nt + 1) * sizeof(int64_t));
  out->j_rows[w] = (int32_t*)malloc((total + 1) * sizeof(int32_t));
  int64_t off = 0;
  for (std::size_t v = 0; v < nt; ++v) {
    out->i_lo[w][v] = tiles[v].i_lo;
    out->i_hi[w][v] = tiles[v].i_hi;
    out->cost[w][v] = tiles[v].cost;
    out->j_off[w][v] = off;
    if (!tiles[v].j_rows.empty())
      std::memcpy(out->j_rows[w] + off, tiles[v].j_rows.data(),
                  tiles[v].j_rows.size() * sizeof(int32_t));
    off += (int64_t)tiles[v].j_rows.size();
  }
  out->j_off[w][nt] = off;
}

FusedSchedule unflatten(const tfo_schedule* s) {
  FusedSchedule fs;
  fs.n = s->n;
  fs.tile_size = s->tile_size;
  fs.wavefronts.resize(2);
  for (int w = 0; w < 2; ++w)
    for (int64_t v = 0; v < s->n_tiles[w]; ++v) {
      FusedTile t;
      t.i_lo = s->i_lo[w][v];
      t.i_hi = s->i_hi[w][v];
      t.cost = s->cost[w][v];
      t.j_rows.assign(s->j_rows[w] + s->j_off[w][v],
                      s->j_rows[w] + s->j_off[w][v + 1]);
      fs.wavefronts[w].push_back(std::move(t));
    }
  return fs;
}

void export_csr(const CsrMatrix<double>& m, int32_t** rp, int32_t** ci,
                double** v) {
  *rp = (int32_t*)malloc((m.row_ptr.size() + 1) * sizeof(int32_t));
  *ci = (int32_t*)malloc((m.col_idx.size() + 1) * sizeof(int32_t));
  *v = (double*)malloc((m.values.size() + 1) * sizeof(double));
  std::memcpy(*rp, m.row_ptr.data(), m.row_ptr.size() * sizeof(int32_t));
  if (!m.col_idx.empty())
    std::memcpy(*ci, m.col_idx.data(), m.col_idx.size() * sizeof(int32_t));
  if (!m.values.empty())
    std::memcpy(*v, m.values.data(), m.values.size() * sizeof(double));
}

template <class T>
CsrMatrix<T> make_csr(int32_t rows, int32_t cols, const int32_t* rp,
                      const int32_t* ci, const T* v) {
  CsrMatrix<T> m;
  m.n_rows = rows;
  m.n_cols = cols;
  m.row_ptr.assign(rp, rp + rows + 1);
  m.col_idx.assign(ci, ci + rp[rows]);
  m.values.assign(v, v + rp[rows]);
  return m;
}

template <class T>
DenseMatrix<T> make_dense(int32_t rows, int32_t cols, const T* p) {
  DenseMatrix<T> m(rows, cols);
  std::memcpy(m.data.data(), p, (std::size_t)rows * cols * sizeof(T));
  return m;
}

struct ProblemHandle {
  int is_f64;
  FusedProblem<double> p64;
  FusedProblem<float> p32;
};

}  // namespace

extern "C" {

const char* tfr_last_error(void) { return g_err.c_str(); }

int tfr_choose_tile_size(int32_t n, int32_t p, int32_t ct, int32_t* out) {
  return guard([&] { *out = choose_tile_size(n, p, ct); });
}

int tfr_step1(int32_t n_rows, int32_t n_cols, const int32_t* rp,
              const int32_t* ci, int32_t t, int64_t* tile_j_off,
              int32_t* tile_j_rows, int32_t* unfused, int64_t* n_unfused) {
  return guard([&] {
    auto s = step1_coarse_fuse(view(n_rows, n_cols, rp, ci), t);
    int64_t off = 0;
    for (std::size_t v = 0; v < s.tiles.size(); ++v) {
      tile_j_off[v] = off;
      for (auto j : s.tiles[v].j_rows) tile_j_rows[off++] = j;
    }
    tile_j_off[s.tiles.size()] = off;
    for (std::size_t q = 0; q < s.unfused_rows.size(); ++q)
      unfused[q] = s.unfused_rows[q];
    *n_unfused = (int64_t)s.unfused_rows.size();
  });
}

int tfr_balance(const int32_t* rows, int64_t m, const int32_t* w,
                int32_t n_weights, int64_t num_chunks, int64_t* chunk_off) {
  return guard([&] {
    std::vector<index_t> r(rows, rows + m), wt(w, w + n_weights);
    auto chunks = balance(r, wt, (std::size_t)num_chunks);
    int64_t off = 0;
    for (std::size_t c = 0; c < chunks.size(); ++c) {
      chunk_off[c] = off;
      off += (int64_t)chunks[c].size();
    }
    chunk_off[chunks.size()] = off;
  });
}

int tfr_tile_cost(int32_t n_rows, const int32_t* rp, const int32_t* ci,
                  int32_t i_lo, int32_t i_hi, const int32_t* j_rows,
                  int64_t nj, const tfo_config* cfg, double* out) {
  return guard([&] {
    FusedTile t{i_lo, i_hi, std::vector<index_t>(j_rows, j_rows + nj), 0.0};
    *out = tile_cost(view(n_rows, n_rows, rp, ci), t, to_cfg(cfg));
  });
}

int tfr_split_tile(int32_t n_rows, const int32_t* rp, const int32_t* ci,
                   int32_t i_lo, int32_t i_hi, const int32_t* j_rows,
                   int64_t nj, const tfo_config* cfg, tfo_schedule* pieces,
                   int32_t** demoted, int64_t* n_demoted) {
  return guard([&] {
    FusedTile t{i_lo, i_hi, std::vector<index_t>(j_rows, j_rows + nj), 0.0};
    auto r = split_tile(view(n_rows, n_rows, rp, ci), t, to_cfg(cfg));
    std::memset(pieces, 0, sizeof *pieces);
    pieces->n = n_rows;
    flatten(r.pieces, pieces, 0);
    flatten({}, pieces, 1);
    *demoted = (int32_t*)malloc((r.demoted_rows.size() + 1) * 4);
    for (std::size_t q = 0; q < r.demoted_rows.size(); ++q)
      (*demoted)[q] = r.demoted_rows[q];
    *n_demoted = (int64_t)r.demoted_rows.size();
  });
}

int tfr_build_schedule(int32_t n_rows, int32_t n_cols, const int32_t* rp,
                       const int32_t* ci, const tfo_config* cfg,
                       tfo_schedule* out, double* seconds) {
  return guard([&] {
    std::memset(out, 0, sizeof *out);
    const auto t0 = std::chrono::steady_clock::now();
    auto s = build_schedule(view(n_rows, n_cols, rp, ci), to_cfg(cfg));
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    out->n = s.n;
    out->tile_size = s.tile_size;
    for (int w = 0; w < 2; ++w) flatten(s.wavefronts[w], out, w);
  });
}

double tfr_fused_ratio(const tfo_schedule* s) {
  return fused_ratio(unflatten(s));
}

int tfr_validate_schedule(int32_t n_rows, int32_t n_cols, const int32_t* rp,
                          const int32_t* ci, const tfo_schedule* s,
                          const tfo_config* cfg, int64_t* n_violations,
                          int64_t* over_budget_width1, char* first_msg,
                          size_t cap) {
  auto rep = validate_schedule(view(n_rows, n_cols, rp, ci), unflatten(s),
                               to_cfg(cfg));
  *n_violations = (int64_t)rep.violations.size();
  *over_budget_width1 = (int64_t)rep.over_budget_width1;
  if (first_msg && cap) {
    first_msg[0] = 0;
    if (!rep.violations.empty())
      std::strncpy(first_msg, rep.violations.front().c_str(), cap - 1),
          first_msg[cap - 1] = 0;
  }
  return rep.pass ? 1 : 0;
}

int tfr_gen_random_sparse(int32_t n, double density, uint64_t seed,
                          int32_t** rp, int32_t** ci, double** v) {
  return guard([&] {
    export_csr(gen_random_sparse<double>(n, density, seed), rp, ci, v);
  });
}

int tfr_gen_banded(int32_t n, int32_t hb, int32_t** rp, int32_t** ci,
                   double** v) {
  return guard([&] { export_csr(gen_banded<double>(n, hb), rp, ci, v); });
}

void tfr_random_dense(int32_t rows, int32_t cols, uint64_t seed, double* out) {
  auto m = tf_test::random_dense<double>(rows, cols, seed);
  std::memcpy(out, m.data.data(), m.data.size() * sizeof(double));
}

int tfr_gen_rect_random(int32_t rows, int32_t cols, double density,
                        uint64_t seed, int32_t** rp, int32_t** ci,
                        double** v) {
  return guard([&] {
    export_csr(tf_test::gen_rect_random(rows, cols, density, seed), rp, ci,
               v);
  });
}

// ---- problem handles for executor parity and CPU-baseline timing ----
// is_f64: 1 double, 0 float.  b_rp == nullptr -> dense B.
void* tfr_problem_create(int is_f64, int32_t n, const int32_t* a_rp,
                         const int32_t* a_ci, const void* a_v,
                         const int32_t* b_rp, const int32_t* b_ci,
                         const void* b_v, const void* b_dense, int32_t b_cols,
                         const void* c, int32_t c_rows, int32_t c_cols) {
  auto* h = new ProblemHandle;
  h->is_f64 = is_f64;
  if (is_f64) {
    h->p64.a = make_csr<double>(n, n, a_rp, a_ci, (const double*)a_v);
    if (b_rp)
      h->p64.b = make_csr<double>(n, b_cols, b_rp, b_ci, (const double*)b_v);
    else
      h->p64.b = make_dense<double>(n, b_cols, (const double*)b_dense);
    h->p64.c = make_dense<double>(c_rows, c_cols, (const double*)c);
  } else {
    h->p32.a = make_csr<float>(n, n, a_rp, a_ci, (const float*)a_v);
    if (b_rp)
      h->p32.b = make_csr<float>(n, b_cols, b_rp, b_ci, (const float*)b_v);
    else
      h->p32.b = make_dense<float>(n, b_cols, (const float*)b_dense);
    h->p32.c = make_dense<float>(c_rows, c_cols, (const float*)c);
  }
  return h;
}

void tfr_problem_destroy(void* h) { delete (ProblemHandle*)h; }

void* tfr_schedule_import(const tfo_schedule* s) {
  return new FusedSchedule(unflatten(s));
}
void tfr_schedule_destroy(void* s) { delete (FusedSchedule*)s; }

// mode: 0 fused, 1 unfused.  d_out may be null (timing only).
// seconds = steady_clock time of the executor call alone, which includes
// the executor's own zeroed D1/D allocation (kernels.hpp:97-98).
int tfr_problem_run(void* hp, const void* sched, int mode, int workers,
                    void* d_out, int64_t* stats, double* seconds) {
  auto* h = (ProblemHandle*)hp;
  return guard([&] {
    RunStats st;
    auto go = [&](auto& p, auto* out_t) {
      using T = std::remove_pointer_t<decltype(out_t)>;
      const bool dense = p.b_is_dense();
      const auto t0 = std::chrono::steady_clock::now();
      DenseMatrix<T> d;
      if (mode == 0) {
        const auto& s = *(const FusedSchedule*)sched;
        d = dense ? fused_gemm_spmm(p, s, workers, &st)
                  : fused_spmm_spmm(p, s, workers, &st);
      } else {
        d = dense ? unfused_gemm_spmm(p, workers, &st)
                  : unfused_spmm_spmm(p, workers, &st);
      }
      const auto t1 = std::chrono::steady_clock::now();
      if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
      if (out_t) std::memcpy(out_t, d.data.data(), d.data.size() * sizeof(T));
    };
    if (h->is_f64)
      go(h->p64, (double*)d_out);
    else
      go(h->p32, (float*)d_out);
    if (stats) {
      stats[0] = st.first_op_rows;
      stats[1] = st.second_op_rows;
      stats[2] = st.nnz_processed;
    }
  });
}

}  // extern "C"
