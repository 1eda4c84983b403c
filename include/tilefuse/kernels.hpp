// tilefuse/kernels.hpp -- drop-in executor API over libtfg (tfg.h).
//
// Same names and signatures as the reference (include/tilefuse/kernels.hpp:
// FusedProblem :16-43, RunStats :46-50, fused_gemm_spmm / fused_spmm_spmm
// :182-208, unfused_* :212-236) and the same std::invalid_argument
// contracts.  The work runs on the B200: operands are copied to HBM, the
// schedule is executed by the sm_100a kernels, D comes back by value.
// `workers` is validated (>= 1) as the reference does and otherwise unused.
// For "inspect once, execute many" without per-call copies use the
// device-resident tfg_plan_* entry points directly.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <type_traits>
#include <variant>

#include "tfg.h"
#include "tilefuse/csr.hpp"
#include "tilefuse/dense.hpp"
#include "tilefuse/scheduler.hpp"

namespace tilefuse {

template <class T>
struct FusedProblem {
  CsrMatrix<T> a;
  std::variant<DenseMatrix<T>, CsrMatrix<T>> b;
  DenseMatrix<T> c;

  bool b_is_dense() const { return std::holds_alternative<DenseMatrix<T>>(b); }
  index_t n() const { return a.n_rows; }
  index_t b_rows() const {
    return b_is_dense() ? std::get<DenseMatrix<T>>(b).n_rows : std::get<CsrMatrix<T>>(b).n_rows;
  }
  index_t b_cols() const {
    return b_is_dense() ? std::get<DenseMatrix<T>>(b).n_cols : std::get<CsrMatrix<T>>(b).n_cols;
  }
  index_t c_cols() const { return c.n_cols; }
  void check() const {
    if (!a.square()) throw std::invalid_argument("problem: A must be square");
    if (b_rows() != a.n_cols) throw std::invalid_argument("problem: B must have n rows");
    if (c.n_rows != b_cols()) throw std::invalid_argument("problem: C rows must match B cols");
  }
};

struct RunStats {
  std::int64_t first_op_rows = 0;
  std::int64_t second_op_rows = 0;
  std::int64_t nnz_processed = 0;
};

namespace detail {

inline void require_workers(int workers) {
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
}

template <class T>
tfg_problem host_problem(const FusedProblem<T>& p) {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "float or double");
  tfg_problem h{};
  h.dtype = std::is_same_v<T, double> ? TFG_F64 : TFG_F32;
  h.n = p.a.n_rows;
  h.b_rows = p.b_rows();
  h.b_cols = p.b_cols();
  h.c_rows = p.c.n_rows;
  h.c_cols = p.c.n_cols;
  h.a_nnz = p.a.nnz();
  h.d_a_row_ptr = p.a.row_ptr.data();
  h.d_a_col_idx = p.a.col_idx.data();
  h.d_a_val = p.a.values.data();
  if (p.b_is_dense()) {
    h.b_is_dense = 1;
    h.d_b_dense = std::get<DenseMatrix<T>>(p.b).data.data();
  } else {
    const auto& b = std::get<CsrMatrix<T>>(p.b);
    h.b_is_dense = 0;
    h.b_nnz = b.nnz();
    h.d_b_row_ptr = b.row_ptr.data();
    h.d_b_col_idx = b.col_idx.data();
    h.d_b_val = b.values.data();
  }
  h.d_c = p.c.data.data();
  return h;
}

template <class T>
DenseMatrix<T> run_on_device(const FusedProblem<T>& p, const FusedSchedule* sched,
                             RunStats* stats) {
  DenseMatrix<T> d(p.a.n_rows, p.c_cols());
  const tfg_problem h = host_problem(p);
  if (sched) {
    if (sched->n != p.a.n_rows)
      throw std::invalid_argument("schedule and problem disagree on n");
    auto ds = upload(*sched);
    tfg_check(tfg_run_host(&h, ds.h, d.data.data()));
  } else {
    tfg_check(tfg_run_host(&h, nullptr, d.data.data()));
  }
  if (stats) {
    if (sched) {
      for (const auto& w : sched->wavefronts)
        for (const auto& t : w) {
          stats->first_op_rows += t.i_hi - t.i_lo;
          stats->second_op_rows += static_cast<std::int64_t>(t.j_rows.size());
        }
    } else {
      stats->first_op_rows += p.a.n_rows;
      stats->second_op_rows += p.a.n_rows;
    }
  }
  return d;
}

}  // namespace detail

// Rows [row_lo, row_hi) of D1 = B*C (kernels.hpp:159-169), on the GPU.
template <class T>
void gemm(const DenseMatrix<T>& b, const DenseMatrix<T>& c, index_t row_lo, index_t row_hi,
          DenseMatrix<T>& d1) {
  if (b.n_cols != c.n_rows) throw std::invalid_argument("gemm: inner dimensions disagree");
  if (d1.n_rows != b.n_rows || d1.n_cols != c.n_cols)
    throw std::invalid_argument("gemm: output shape mismatch");
  detail::tfg_check(tfg_gemm_rows_host(std::is_same_v<T, double> ? TFG_F64 : TFG_F32,
                                       b.data.data(), b.n_rows, b.n_cols, c.data.data(), c.n_rows,
                                       c.n_cols, row_lo, row_hi, d1.data.data()));
}

// Rows j_list of D = A*X (kernels.hpp:171-180), on the GPU.
template <class T>
void spmm(const CsrMatrix<T>& a, const DenseMatrix<T>& x, std::span<const index_t> j_list,
          DenseMatrix<T>& d) {
  if (a.n_cols != x.n_rows) throw std::invalid_argument("spmm: inner dimensions disagree");
  if (d.n_rows != a.n_rows || d.n_cols != x.n_cols)
    throw std::invalid_argument("spmm: output shape mismatch");
  const index_t dummy = 0;
  detail::tfg_check(tfg_spmm_rows_host(
      std::is_same_v<T, double> ? TFG_F64 : TFG_F32, a.n_rows, a.n_cols, a.row_ptr.data(),
      a.col_idx.empty() ? &dummy : a.col_idx.data(), a.values.data(), x.data.data(), x.n_rows,
      x.n_cols, j_list.empty() ? &dummy : j_list.data(), (int64_t)j_list.size(), d.data.data()));
}

template <class T>
DenseMatrix<T> fused_gemm_spmm(const FusedProblem<T>& problem, const FusedSchedule& sched,
                               int workers, RunStats* stats = nullptr) {
  problem.check();
  if (!problem.b_is_dense()) throw std::invalid_argument("fused_gemm_spmm: B must be dense");
  detail::require_workers(workers);
  return detail::run_on_device(problem, &sched, stats);
}

template <class T>
DenseMatrix<T> fused_spmm_spmm(const FusedProblem<T>& problem, const FusedSchedule& sched,
                               int workers, RunStats* stats = nullptr) {
  problem.check();
  if (problem.b_is_dense()) throw std::invalid_argument("fused_spmm_spmm: B must be sparse");
  detail::require_workers(workers);
  return detail::run_on_device(problem, &sched, stats);
}

template <class T>
DenseMatrix<T> unfused_gemm_spmm(const FusedProblem<T>& problem, int workers,
                                 RunStats* stats = nullptr) {
  problem.check();
  if (!problem.b_is_dense()) throw std::invalid_argument("unfused_gemm_spmm: B must be dense");
  detail::require_workers(workers);
  return detail::run_on_device<T>(problem, nullptr, stats);
}

template <class T>
DenseMatrix<T> unfused_spmm_spmm(const FusedProblem<T>& problem, int workers,
                                 RunStats* stats = nullptr) {
  problem.check();
  if (problem.b_is_dense()) throw std::invalid_argument("unfused_spmm_spmm: B must be sparse");
  detail::require_workers(workers);
  return detail::run_on_device<T>(problem, nullptr, stats);
}

}  // namespace tilefuse
