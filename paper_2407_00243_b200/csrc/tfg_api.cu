// tfg_api.cu -- extern "C" entry points of libtfg (declared in include/tfg.h).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "tfg_common.cuh"

struct tfg_plan;

namespace tfg {

void build_schedule_device(int32_t n_rows, int32_t n_cols, int64_t nnz,
                           const int32_t* rp, const int32_t* ci,
                           const tfg_config& cfg, cudaStream_t st,
                           tfg_schedule& out);
void plan_create(const tfg_problem& pr, const tfg_schedule* s, cudaStream_t st,
                 tfg_plan& pl);
void plan_execute(tfg_plan& pl, void* d, cudaStream_t st, cudaEvent_t* ev);
size_t plan_scratch_bytes(const tfg_plan& pl);
void gather_rows(int dtype, const void* src, int cols, const int* rows, int64_t n,
                 void* dst, cudaStream_t st);
double tile_cost_device(int n, const int* rp, const int* ci, int i_lo, int i_hi,
                        const int* jrows, int nj, const tfg_config& cfg, cudaStream_t st);
void split_tile_device(int n, const int* rp, const int* ci, int i_lo, int i_hi, const int* jrows,
                       int nj, const tfg_config& cfg, cudaStream_t st, std::vector<int>& lo,
                       std::vector<int>& hi, std::vector<double>& cost,
                       std::vector<int64_t>& joff, std::vector<int>& jout,
                       std::vector<int>& demoted);
void balance_device(int64_t U, const int64_t* h_w, int64_t num_chunks, int64_t* h_starts,
                    cudaStream_t st);
void scatter_rows(int dtype, const void* src, int cols, const int* rows, int64_t n,
                  void* dst, cudaStream_t st);

namespace {
thread_local std::string g_last_error;
thread_local std::string g_violations;  // all messages of the last tfg_validate_schedule
}
void set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {

// Host restatement of the Eq.-3 footprint for the verify path
// (validate_schedule's cost bound, scheduler.cpp:353-370).
double host_tile_cost(int n, const int32_t* rp, const int32_t* ci, int lo, int hi,
                      const int32_t* j, int64_t nj, const tfg_config& cfg,
                      std::vector<int64_t>& mark, int64_t& epoch) {
  const double t = (double)(hi - lo), jc = (double)nj;
  double nnzj = 0.0, uc = 0.0;
  const int64_t ep = ++epoch;
  for (int64_t q = 0; q < nj; ++q)
    for (int k = rp[j[q]]; k < rp[j[q] + 1]; ++k) {
      ++nnzj;
      if (mark[ci[k]] != ep) {
        mark[ci[k]] = ep;
        ++uc;
      }
    }
  const double cc = cfg.c_cols, bc = cfg.b_cols;
  if (cfg.b_is_dense) {
    const double first = cfg.whole_b_cost ? (double)n : t;
    const double idx = std::ceil((nnzj + jc + 1.0) * cfg.index_to_scalar_ratio);
    return (uc + t + jc) * cc + first * bc + idx;
  }
  double nb = 0.0;
  for (int i = lo; i < hi; ++i) nb += rp[i + 1] - rp[i];
  const double idx = std::ceil((nnzj + jc + 1.0 + nb + t + 1.0) * cfg.index_to_scalar_ratio);
  return (nb + nnzj + uc + t + jc) * cc + idx;
}

struct HostSched {
  int32_t n, t;
  std::vector<int32_t> ilo[2], ihi[2], jrows[2];
  std::vector<double> cost[2];
  std::vector<int64_t> joff[2];
};

HostSched download(const tfg_schedule& s) {
  HostSched h;
  h.n = s.n;
  h.t = s.tile_size;
  for (int w = 0; w < 2; ++w) {
    const int64_t nt = s.n_tiles[w];
    h.ilo[w].resize(nt);
    h.ihi[w].resize(nt);
    h.cost[w].resize(nt);
    h.joff[w].resize(nt + 1);
    h.jrows[w].resize(s.n_jrows[w]);
    if (nt) {
      TFG_CUDA(cudaMemcpy(h.ilo[w].data(), s.i_lo[w].p, nt * 4, cudaMemcpyDeviceToHost));
      TFG_CUDA(cudaMemcpy(h.ihi[w].data(), s.i_hi[w].p, nt * 4, cudaMemcpyDeviceToHost));
      TFG_CUDA(cudaMemcpy(h.cost[w].data(), s.cost[w].p, nt * 8, cudaMemcpyDeviceToHost));
    }
    TFG_CUDA(cudaMemcpy(h.joff[w].data(), s.j_off[w].p, (nt + 1) * 8, cudaMemcpyDeviceToHost));
    if (s.n_jrows[w])
      TFG_CUDA(cudaMemcpy(h.jrows[w].data(), s.j_rows[w].p, s.n_jrows[w] * 4,
                          cudaMemcpyDeviceToHost));
  }
  return h;
}

}  // namespace
}  // namespace tfg

using namespace tfg;

extern "C" {

const char* tfg_last_error(void) { return g_last_error.c_str(); }

void tfg_config_default(tfg_config* c) {
  c->ct_size = 2048;
  c->num_workers = 1;
  c->cache_size_words = 160 * 1024;
  c->b_cols = 32;
  c->c_cols = 32;
  c->index_to_scalar_ratio = 0.5;
  c->b_is_dense = 1;
  c->whole_b_cost = 0;
}

tfg_status tfg_device_info(int32_t* built_arch, int32_t* sms) {
  return guard([&] {
    if (built_arch) *built_arch = 100;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
    cudaGetLastError();
    if (sms) *sms = count > 0 ? sm_count() : 0;
  });
}

tfg_status tfg_choose_tile_size(int32_t n, int32_t p, int32_t ct, int32_t* out) {
  return guard([&] {
    if (n < 1 || p < 1 || ct < 1)
      throw invalid_argument("choose_tile_size: all inputs must be >= 1");
    *out = ((n + ct - 1) / ct) >= p ? ct : (n + p - 1) / p;
  });
}

tfg_status tfg_build_schedule(int32_t n_rows, int32_t n_cols, int64_t nnz,
                              const int32_t* d_row_ptr, const int32_t* d_col_idx,
                              const tfg_config* cfg, void* stream, tfg_schedule** out) {
  return guard([&] {
    *out = nullptr;
    auto* s = new tfg_schedule;
    try {
      build_schedule_device(n_rows, n_cols, nnz, d_row_ptr, d_col_idx, *cfg,
                            as_stream(stream), *s);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

tfg_status tfg_build_schedule_host(int32_t n_rows, int32_t n_cols, const int32_t* h_row_ptr,
                                   const int32_t* h_col_idx, const tfg_config* cfg,
                                   void* stream, tfg_schedule** out) {
  return guard([&] {
    *out = nullptr;
    if (n_rows != n_cols) throw invalid_argument("build_schedule: matrix must be square");
    if (n_rows < 1) throw invalid_argument("build_schedule: matrix must be nonempty");
    cudaStream_t st = as_stream(stream);
    const int64_t nnz = h_row_ptr[n_rows];
    dbuf<int32_t> rp(n_rows + 1), ci(std::max<int64_t>(nnz, 1));
    h2d(rp.p, h_row_ptr, n_rows + 1, st);
    h2d(ci.p, h_col_idx, nnz, st);
    auto* s = new tfg_schedule;
    try {
      build_schedule_device(n_rows, n_cols, nnz, rp.p, ci.p, *cfg, st, *s);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

tfg_status tfg_schedule_info(const tfg_schedule* s, int32_t* n, int32_t* t,
                             int64_t n_tiles[2], int64_t n_jrows[2], double* secs) {
  return guard([&] {
    if (!s) throw invalid_argument("null schedule");
    if (n) *n = s->n;
    if (t) *t = s->tile_size;
    for (int w = 0; w < 2; ++w) {
      if (n_tiles) n_tiles[w] = s->n_tiles[w];
      if (n_jrows) n_jrows[w] = s->n_jrows[w];
    }
    if (secs) *secs = s->inspect_seconds;
  });
}

tfg_status tfg_schedule_export(const tfg_schedule* s, int w, int32_t* i_lo, int32_t* i_hi,
                               double* cost, int64_t* j_off, int32_t* j_rows) {
  return guard([&] {
    if (!s || w < 0 || w > 1) throw invalid_argument("schedule_export: bad arguments");
    const int64_t nt = s->n_tiles[w];
    if (nt) {
      if (i_lo) TFG_CUDA(cudaMemcpy(i_lo, s->i_lo[w].p, nt * 4, cudaMemcpyDeviceToHost));
      if (i_hi) TFG_CUDA(cudaMemcpy(i_hi, s->i_hi[w].p, nt * 4, cudaMemcpyDeviceToHost));
      if (cost) TFG_CUDA(cudaMemcpy(cost, s->cost[w].p, nt * 8, cudaMemcpyDeviceToHost));
    }
    if (j_off) TFG_CUDA(cudaMemcpy(j_off, s->j_off[w].p, (nt + 1) * 8, cudaMemcpyDeviceToHost));
    if (j_rows && s->n_jrows[w])
      TFG_CUDA(cudaMemcpy(j_rows, s->j_rows[w].p, s->n_jrows[w] * 4, cudaMemcpyDeviceToHost));
  });
}

tfg_status tfg_schedule_import(int32_t n, int32_t tile_size, const int64_t n_tiles[2],
                               const int32_t* const h_i_lo[2], const int32_t* const h_i_hi[2],
                               const double* const h_cost[2], const int64_t* const h_j_off[2],
                               const int32_t* const h_j_rows[2], tfg_schedule** out) {
  return guard([&] {
    *out = nullptr;
    auto* s = new tfg_schedule;
    try {
      s->n = n;
      s->tile_size = tile_size;
      for (int w = 0; w < 2; ++w) {
        const int64_t nt = n_tiles[w];
        const int64_t nj = h_j_off[w][nt];
        if (h_j_off[w][0] != 0 || nj < 0) throw invalid_argument("schedule_import: bad j_off");
        s->n_tiles[w] = nt;
        s->n_jrows[w] = nj;
        s->i_lo[w].alloc(nt + 1);
        s->i_hi[w].alloc(nt + 1);
        s->cost[w].alloc(nt + 1);
        s->j_off[w].alloc(nt + 1);
        s->j_rows[w].alloc(nj + 1);
        if (nt) {
          TFG_CUDA(cudaMemcpy(s->i_lo[w].p, h_i_lo[w], nt * 4, cudaMemcpyHostToDevice));
          TFG_CUDA(cudaMemcpy(s->i_hi[w].p, h_i_hi[w], nt * 4, cudaMemcpyHostToDevice));
          TFG_CUDA(cudaMemcpy(s->cost[w].p, h_cost[w], nt * 8, cudaMemcpyHostToDevice));
        }
        TFG_CUDA(cudaMemcpy(s->j_off[w].p, h_j_off[w], (nt + 1) * 8, cudaMemcpyHostToDevice));
        if (nj) TFG_CUDA(cudaMemcpy(s->j_rows[w].p, h_j_rows[w], nj * 4, cudaMemcpyHostToDevice));
        for (int64_t q = 0; q < nj; ++q)
          if (h_j_rows[w][q] < 0 || h_j_rows[w][q] >= n)
            throw invalid_argument("schedule_import: j row out of range");
        for (int64_t v = 0; v < nt; ++v)
          if (h_i_lo[w][v] < 0 || h_i_hi[w][v] > n || h_i_lo[w][v] > h_i_hi[w][v] ||
              h_j_off[w][v + 1] < h_j_off[w][v])
            throw invalid_argument("schedule_import: tile out of range");
      }
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void tfg_schedule_destroy(tfg_schedule* s) { delete s; }

double tfg_fused_ratio(const tfg_schedule* s) {
  if (!s || s->n < 1) return 0.0;
  return (double)s->n_jrows[0] / (2.0 * (double)s->n);
}

tfg_status tfg_validate_schedule(int32_t n_rows, int32_t n_cols, const int32_t* rp,
                                 const int32_t* ci, const tfg_schedule* s,
                                 const tfg_config* cfg, int32_t* pass, int64_t* nviol,
                                 int64_t* ob1, char* msg, size_t cap) {
  return guard([&] {
    std::vector<std::string> v;
    int64_t over = 0;
    auto fail = [&](std::string m) { v.push_back(std::move(m)); };
    const HostSched h = download(*s);
    const int n = n_rows;
    bool square = n_rows == n_cols;
    if (!square) fail("matrix is not square");
    if (h.n != n) fail("schedule n does not match matrix");
    if (square && h.n == n) {
      std::vector<std::pair<int, int>> ranges;
      for (size_t q = 0; q < h.ilo[0].size(); ++q) {
        const int lo = h.ilo[0][q], hi = h.ihi[0][q];
        if (lo >= hi) {
          fail("wavefront-0 tile with empty i_range [" + std::to_string(lo) + "," +
               std::to_string(hi) + ")");
          continue;
        }
        if (lo < 0 || hi > n) {
          fail("i_range out of bounds");
          continue;
        }
        ranges.emplace_back(lo, hi);
      }
      std::sort(ranges.begin(), ranges.end());
      int expect = 0;
      bool contiguous = true;
      for (auto& [lo, hi] : ranges) {
        if (lo != expect) {
          fail("i coverage gap or overlap at " + std::to_string(lo) + " (expected " +
               std::to_string(expect) + ")");
          contiguous = false;
          break;
        }
        expect = hi;
      }
      if (contiguous && !ranges.empty() && expect != n)
        fail("i coverage stops at " + std::to_string(expect));
      if (ranges.empty() && n > 0) fail("wavefront 0 covers nothing");
      for (size_t q = 0; q < h.ilo[1].size(); ++q)
        if (h.ilo[1][q] != h.ihi[1][q]) {
          fail("wavefront-1 tile carries a nonempty i_range");
          break;
        }
      std::vector<char> seen(n, 0);
      int64_t seen_count = 0;
      for (int w = 0; w < 2; ++w)
        for (size_t t = 0; t + 1 < h.joff[w].size(); ++t) {
          int prev = -1;
          for (int64_t q = h.joff[w][t]; q < h.joff[w][t + 1]; ++q) {
            const int j = h.jrows[w][q];
            if (j < 0 || j >= n) {
              fail("j out of range: " + std::to_string(j));
              continue;
            }
            if (j <= prev) fail("j_list not strictly ascending");
            prev = j;
            if (seen[j])
              fail("j appears twice: " + std::to_string(j));
            else {
              seen[j] = 1;
              ++seen_count;
            }
          }
        }
      if (seen_count != n)
        fail("j coverage incomplete: " + std::to_string(seen_count) + " of " +
             std::to_string(n));
      for (size_t t = 0; t < h.ilo[0].size(); ++t) {
        bool ok = true;
        for (int64_t q = h.joff[0][t]; q < h.joff[0][t + 1] && ok; ++q) {
          const int j = h.jrows[0][q];
          if (j < 0 || j >= n) continue;
          for (int k = rp[j]; k < rp[j + 1]; ++k)
            if (ci[k] < h.ilo[0][t] || ci[k] >= h.ihi[0][t]) {
              fail("row " + std::to_string(j) + " fused into [" + std::to_string(h.ilo[0][t]) +
                   "," + std::to_string(h.ihi[0][t]) + ") but depends on " +
                   std::to_string(ci[k]));
              ok = false;
              break;
            }
        }
      }
      std::vector<int64_t> mark(n + 1, 0);
      int64_t epoch = 0;
      const double budget = (double)cfg->cache_size_words;
      for (int w = 0; w < 2; ++w)
        for (size_t t = 0; t + 1 < h.joff[w].size(); ++t) {
          const int64_t b = h.joff[w][t], e = h.joff[w][t + 1];
          bool bad = false;
          for (int64_t q = b; q < e; ++q) bad |= h.jrows[w][q] < 0 || h.jrows[w][q] >= n;
          if (bad) continue;
          const double cost = host_tile_cost(n, rp, ci, h.ilo[w][t], h.ihi[w][t],
                                             h.jrows[w].data() + b, e - b, *cfg, mark, epoch);
          if (cost <= budget) continue;
          const bool irreducible = w == 0 ? (h.ihi[w][t] - h.ilo[w][t]) <= 1 : (e - b) <= 1;
          if (irreducible)
            ++over;
          else
            fail("splittable tile exceeds cache budget (cost " + std::to_string(cost) + ")");
        }
      const int64_t p = cfg->num_workers;
      if (h.t < 1) {
        fail("tile_size must be >= 1");
      } else {
        const int64_t avail0 = ((int64_t)n + h.t - 1) / h.t;
        if ((int64_t)h.ilo[0].size() < std::min(p, avail0))
          fail("wavefront 0 has too few tiles for " + std::to_string(p) + " workers");
      }
      const int64_t w1_rows = (int64_t)h.jrows[1].size();
      if ((int64_t)h.ilo[1].size() < std::min(p, w1_rows))
        fail("wavefront 1 has too few tiles for " + std::to_string(p) + " workers");
    }
    *pass = v.empty() ? 1 : 0;
    if (nviol) *nviol = (int64_t)v.size();
    if (ob1) *ob1 = over;
    // every violation, newline separated (scheduler.cpp:258-261 keeps them all)
    std::string all;
    for (size_t q = 0; q < v.size(); ++q) all += (q ? "\n" : "") + v[q];
    g_violations = all;
    if (msg && cap) {
      msg[0] = 0;
      if (!v.empty()) {
        std::strncpy(msg, v.front().c_str(), cap - 1);
        msg[cap - 1] = 0;
      }
    }
  });
}

tfg_status tfg_validate_messages(char* buf, size_t cap, size_t* needed) {
  return guard([&] {
    if (needed) *needed = g_violations.size() + 1;
    if (buf && cap) {
      const size_t k = std::min(cap - 1, g_violations.size());
      std::memcpy(buf, g_violations.data(), k);
      buf[k] = 0;
    }
  });
}

// ---- single inspector steps (scheduler.hpp:80-97) ------------------------
namespace {
struct HostPattern {  // a host CSR pattern on the device for one call
  dbuf<int32_t> rp, ci, jr;
  HostPattern(int32_t n, const int32_t* h_rp, const int32_t* h_ci, const int32_t* h_j, int64_t nj,
              cudaStream_t st)
      : rp(n + 1), ci(std::max<int64_t>(h_rp[n], 1)), jr(std::max<int64_t>(nj, 1)) {
    h2d(rp.p, h_rp, n + 1, st);
    h2d(ci.p, h_ci, h_rp[n], st);
    h2d(jr.p, h_j, nj, st);
  }
};
void check_tile_args(int32_t n, const int32_t* h_rp, const int32_t* h_j, int64_t nj,
                     const tfg_config* cfg, const char* who) {
  if (!h_rp || !cfg || (nj > 0 && !h_j)) throw invalid_argument(std::string(who) + ": null argument");
  if (n < 1) throw invalid_argument(std::string(who) + ": matrix must be nonempty");
  for (int64_t q = 0; q < nj; ++q)
    if (h_j[q] < 0 || h_j[q] >= n) throw invalid_argument(std::string(who) + ": j row out of range");
}
}  // namespace

tfg_status tfg_tile_cost(int32_t n, const int32_t* h_row_ptr, const int32_t* h_col_idx,
                         int32_t i_lo, int32_t i_hi, const int32_t* h_j_rows, int64_t n_j,
                         const tfg_config* cfg, double* cost) {
  return guard([&] {
    check_tile_args(n, h_row_ptr, h_j_rows, n_j, cfg, "tile_cost");
    cudaStream_t st = nullptr;
    HostPattern hp(n, h_row_ptr, h_col_idx, h_j_rows, n_j, st);
    *cost = tile_cost_device(n, hp.rp.p, hp.ci.p, i_lo, i_hi, hp.jr.p, (int)n_j, *cfg, st);
  });
}

tfg_status tfg_split_tile(int32_t n, const int32_t* h_row_ptr, const int32_t* h_col_idx,
                          int32_t i_lo, int32_t i_hi, const int32_t* h_j_rows, int64_t n_j,
                          const tfg_config* cfg, int64_t* n_pieces, int32_t* h_lo, int32_t* h_hi,
                          double* h_cost, int64_t* h_j_off, int32_t* h_j_out, int64_t* n_demoted,
                          int32_t* h_demoted) {
  return guard([&] {
    check_tile_args(n, h_row_ptr, h_j_rows, n_j, cfg, "split_tile");
    for (int64_t q = 0; q < n_j; ++q) {  // j rows of a step-1 tile: columns inside it
      const int j = h_j_rows[q];
      for (int k = h_row_ptr[j]; k < h_row_ptr[j + 1]; ++k)
        if (h_col_idx[k] < i_lo || h_col_idx[k] >= i_hi)
          throw invalid_argument("split_tile: a j row reads outside the tile's i range");
    }
    cudaStream_t st = nullptr;
    HostPattern hp(n, h_row_ptr, h_col_idx, h_j_rows, n_j, st);
    std::vector<int> lo, hi, jout, dem;
    std::vector<double> cost;
    std::vector<int64_t> joff;
    split_tile_device(n, hp.rp.p, hp.ci.p, i_lo, i_hi, hp.jr.p, (int)n_j, *cfg, st, lo, hi, cost,
                      joff, jout, dem);
    *n_pieces = (int64_t)lo.size();
    *n_demoted = (int64_t)dem.size();
    if (h_lo) std::copy(lo.begin(), lo.end(), h_lo);
    if (h_hi) std::copy(hi.begin(), hi.end(), h_hi);
    if (h_cost) std::copy(cost.begin(), cost.end(), h_cost);
    if (h_j_off) std::copy(joff.begin(), joff.end(), h_j_off);
    if (h_j_out) std::copy(jout.begin(), jout.end(), h_j_out);
    if (h_demoted) std::copy(dem.begin(), dem.end(), h_demoted);
  });
}

tfg_status tfg_balance(int64_t n_items, const int64_t* h_weights, int64_t num_chunks,
                       int64_t* h_chunk_start) {
  return guard([&] {
    if (num_chunks < 1) throw invalid_argument("balance: num_chunks must be >= 1");
    if (n_items < 0 || (n_items > 0 && !h_weights) || !h_chunk_start)
      throw invalid_argument("balance: null argument");
    balance_device(n_items, h_weights, num_chunks, h_chunk_start, nullptr);
  });
}

}  // extern "C"
