// C++ conformance program for the drop-in headers (include/tilefuse/*.hpp)
// against libtfg.  Written against the reference's public API only, replaying
// known answers from its unit tests (test_scheduler.cpp, test_kernels.cpp).
// Exit 0 when every check passes; prints one line per failed check.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "tilefuse/csr.hpp"
#include "tilefuse/dense.hpp"
#include "tilefuse/kernels.hpp"
#include "tilefuse/scheduler.hpp"
#include "tilefuse/verify.hpp"

using namespace tilefuse;

static int g_fail = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
      ++g_fail;                                                         \
    }                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, E)                                        \
  do {                                                                  \
    bool thrown = false;                                                \
    try {                                                               \
      (void)(expr);                                                     \
    } catch (const E&) {                                                \
      thrown = true;                                                    \
    } catch (...) {                                                     \
    }                                                                   \
    if (!thrown) {                                                      \
      std::printf("FAIL %s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #E); \
      ++g_fail;                                                         \
    }                                                                   \
  } while (0)

static CsrMatrix<double> banded(index_t n, index_t hb) {
  std::vector<Triplet<double>> t;
  for (index_t r = 0; r < n; ++r)
    for (index_t c = std::max<index_t>(0, r - hb); c <= std::min<index_t>(n - 1, r + hb); ++c)
      t.push_back({r, c, 1.0});
  return csr_from_triplets<double>(n, n, t);
}

static CsrMatrix<double> random_sparse(index_t n, double density, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::vector<Triplet<double>> t;
  for (index_t r = 0; r < n; ++r) {
    bool any = false;
    for (index_t c = 0; c < n; ++c)
      if (u(rng) < density) {
        t.push_back({r, c, 0.1 + 0.9 * u(rng)});
        any = true;
      }
    if (!any) t.push_back({r, r, 1.0});
  }
  return csr_from_triplets<double>(n, n, t);
}

template <class T>
static DenseMatrix<T> rand_dense(index_t r, index_t c, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  DenseMatrix<T> m(r, c);
  for (auto& x : m.data) x = static_cast<T>(u(rng));
  return m;
}

int main() {
  // choose_tile_size (test_scheduler.cpp:31-43)
  CHECK(choose_tile_size(10000, 3, 2048) == 2048);
  CHECK(choose_tile_size(4096, 8, 2048) == 512);
  CHECK(choose_tile_size(8, 3, 4) == 3);
  CHECK_THROWS_AS(choose_tile_size(0, 1, 1), std::invalid_argument);

  // step 1 on banded(16,1) at t = 4 (test_scheduler.cpp:69-79)
  const auto b16 = banded(16, 1);
  const auto s1 = step1_coarse_fuse(b16, 4);
  CHECK(s1.tiles.size() == 4);
  CHECK((s1.tiles[0].j_rows == std::vector<index_t>{0, 1, 2}));
  CHECK((s1.tiles[1].j_rows == std::vector<index_t>{5, 6}));
  CHECK((s1.tiles[3].j_rows == std::vector<index_t>{13, 14, 15}));
  CHECK((s1.unfused_rows == std::vector<index_t>{3, 4, 7, 8, 11, 12}));

  // build_schedule (test_scheduler.cpp:356-367, test_smoke.py:93-103)
  SchedulerConfig cfg;
  cfg.ct_size = 4;
  cfg.num_workers = 2;
  const auto s = build_schedule(b16, cfg);
  CHECK(s.wavefronts.size() == 2);
  CHECK(fused_ratio(s) == 0.3125);
  CHECK(validate_schedule(b16, s, cfg).pass);
  CHECK(s.wavefronts[0][0].i_lo == 0 && s.wavefronts[0][0].i_hi == 4);
  auto bad = s;
  bad.wavefronts[0][0].i_hi -= 1;
  CHECK(!validate_schedule(b16, bad, cfg).pass);
  CsrMatrix<double> rect = CsrMatrix<double>::checked(2, 3, {0, 1, 2}, {0, 1}, {1.0, 1.0});
  CHECK_THROWS_AS(build_schedule(rect, cfg), std::invalid_argument);
  CHECK_THROWS_AS(CsrMatrix<double>::checked(1, 2, {0, 1}, {5}, {1.0}), std::invalid_argument);

  // gemm / spmm known answers through the executors (test_kernels.cpp:26-64)
  {
    FusedProblem<double> p;
    p.a = csr_from_triplets<double>(2, 2, {{0, 0, 1.0}, {1, 1, 1.0}});
    DenseMatrix<double> b(2, 2), c(2, 2);
    b.data = {1, 2, 3, 4};
    c.data = {5, 6, 7, 8};
    p.b = b;
    p.c = c;
    CHECK((unfused_gemm_spmm(p, 1).data == std::vector<double>{19, 22, 43, 50}));
    FusedProblem<double> q;
    q.a = csr_from_triplets<double>(2, 2, {{0, 1, 2.0}, {1, 0, 3.0}});
    q.b = csr_from_triplets<double>(2, 2, {{0, 0, 1.0}, {1, 1, 1.0}});
    DenseMatrix<double> x(2, 2);
    x.data = {1, 2, 3, 4};
    q.c = x;
    CHECK((unfused_spmm_spmm(q, 1).data == std::vector<double>{6, 8, 3, 6}));
  }

  // gemm / spmm row-range helpers (test_kernels.cpp:26-64)
  {
    DenseMatrix<double> b(2, 2), c(2, 2), d1(2, 2);
    b.data = {1, 2, 3, 4};
    c.data = {5, 6, 7, 8};
    gemm(b, c, 0, 2, d1);
    CHECK((d1.data == std::vector<double>{19, 22, 43, 50}));
    DenseMatrix<double> part(2, 2);
    gemm(b, c, 1, 2, part);
    CHECK((part.data == std::vector<double>{0, 0, 43, 50}));
    DenseMatrix<double> wrong(3, 2);
    CHECK_THROWS_AS(gemm(b, c, 0, 2, wrong), std::invalid_argument);
    const auto a = csr_from_triplets<double>(2, 2, {{0, 1, 2.0}, {1, 0, 3.0}});
    DenseMatrix<double> x(2, 2), d(2, 2);
    x.data = {1, 2, 3, 4};
    const std::vector<index_t> all{0, 1}, one{1};
    spmm(a, x, all, d);
    CHECK((d.data == std::vector<double>{6, 8, 3, 6}));
    DenseMatrix<double> pd(2, 2);
    spmm(a, x, one, pd);
    CHECK((pd.data == std::vector<double>{0, 0, 3, 6}));
    DenseMatrix<double> xbad(3, 2);
    CHECK_THROWS_AS(spmm(a, xbad, all, d), std::invalid_argument);
  }

  // fused vs dense oracle, fused == unfused bitwise, stats, errors
  // (test_kernels.cpp:66-229)
  {
    const auto a = random_sparse(64, 0.08, 21);
    SchedulerConfig c2;
    c2.ct_size = 8;
    c2.num_workers = 2;
    c2.cache_size_words = 4096;
    c2.b_cols = 20;
    c2.c_cols = 9;
    FusedProblem<double> p{a, rand_dense<double>(64, 20, 77), rand_dense<double>(20, 9, 78)};
    const auto sched = build_schedule(a, c2);
    CHECK(validate_schedule(a, sched, c2).pass);
    RunStats st;
    const auto d = fused_gemm_spmm(p, sched, 2, &st);
    CHECK(compare(d, dense_oracle(p), kTolDouble).pass);
    CHECK(st.first_op_rows == 64 && st.second_op_rows == 64);
    CHECK(d.data == unfused_gemm_spmm(p, 3).data);
    CHECK_THROWS_AS(fused_gemm_spmm(p, sched, 0), std::invalid_argument);
    CHECK_THROWS_AS(fused_spmm_spmm(p, sched, 1), std::invalid_argument);
    const auto other = build_schedule(banded(8, 1), c2);
    CHECK_THROWS_AS(fused_gemm_spmm(p, other, 1), std::invalid_argument);
    auto badc = p;
    badc.c = rand_dense<double>(5, 9, 3);
    CHECK_THROWS_AS(fused_gemm_spmm(badc, sched, 1), std::invalid_argument);

    FusedProblem<double> sp{a, random_sparse(64, 0.2, 5), rand_dense<double>(64, 7, 79)};
    SchedulerConfig c3 = c2;
    c3.b_is_dense = false;
    c3.c_cols = 7;
    const auto ss = build_schedule(a, c3);
    const auto ds = fused_spmm_spmm(sp, ss, 2);
    CHECK(compare(ds, dense_oracle(sp), kTolDouble).pass);
    CHECK(ds.data == unfused_spmm_spmm(sp, 1).data);

    FusedProblem<float> pf{CsrMatrix<float>{a.n_rows, a.n_cols, a.row_ptr, a.col_idx,
                                            std::vector<float>(a.values.begin(), a.values.end())},
                           rand_dense<float>(64, 8, 4), rand_dense<float>(8, 8, 5)};
    SchedulerConfig c4 = c2;
    c4.b_cols = 8;
    c4.c_cols = 8;
    c4.index_to_scalar_ratio = 1.0;
    CHECK(compare(fused_gemm_spmm(pf, build_schedule(a, c4), 2), dense_oracle(pf), kTolSingle).pass);
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "PASSED", g_fail);
  return g_fail ? 1 : 0;
}
