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
void scatter_rows(int dtype, const void* src, int cols, const int* rows, int64_t n,
                  void* dst, cudaStream_t st);

namespace {
thread_local std::string g_last_error;
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
    if (msg && cap) {
      msg[0] = 0;
      if (!v.empty()) {
        std::strncpy(msg, v.front().c_str(), cap - 1);
        msg[cap - 1] = 0;
      }
    }
  });
}

// ---- host generators (generate.hpp:15-94), std::mt19937_64 as the reference
static void export_csr(const std::vector<int32_t>& rp, const std::vector<int32_t>& ci,
                       const std::vector<double>& v, int32_t** orp, int32_t** oci,
                       double** ov) {
  *orp = (int32_t*)std::malloc((rp.size() + 1) * sizeof(int32_t));
  *oci = (int32_t*)std::malloc((ci.size() + 1) * sizeof(int32_t));
  *ov = (double*)std::malloc((v.size() + 1) * sizeof(double));
  std::memcpy(*orp, rp.data(), rp.size() * sizeof(int32_t));
  if (!ci.empty()) std::memcpy(*oci, ci.data(), ci.size() * sizeof(int32_t));
  if (!v.empty()) std::memcpy(*ov, v.data(), v.size() * sizeof(double));
}

tfg_status tfg_gen_random_sparse(int32_t n, double density, uint64_t seed, int32_t** orp,
                                 int32_t** oci, double** ov) {
  return guard([&] {
    if (n < 1) throw invalid_argument("gen_random_sparse: n must be >= 1");
    if (!(density > 0.0) || density > 1.0)
      throw invalid_argument("gen_random_sparse: density must be in (0,1]");
    std::mt19937_64 rng(seed);
    auto unit_open = [&] { return ((double)(rng() >> 11) + 0.5) * 0x1.0p-53; };
    auto value = [&] { return 0.1 + 0.9 * (double)(rng() >> 11) * 0x1.0p-53; };
    std::vector<int32_t> rp{0}, ci;
    std::vector<double> v;
    const bool full = density >= 1.0;
    const double log_skip = full ? 0.0 : std::log1p(-density);
    for (int32_t r = 0; r < n; ++r) {
      const size_t start = ci.size();
      if (full) {
        for (int32_t c = 0; c < n; ++c) {
          ci.push_back(c);
          v.push_back(value());
        }
      } else {
        int64_t c = -1;
        for (;;) {
          c += 1 + (int64_t)std::floor(std::log(unit_open()) / log_skip);
          if (c >= n) break;
          ci.push_back((int32_t)c);
          v.push_back(value());
        }
      }
      if (ci.size() == start) {
        ci.push_back(r);
        v.push_back(value());
      }
      rp.push_back((int32_t)ci.size());
    }
    export_csr(rp, ci, v, orp, oci, ov);
  });
}

tfg_status tfg_gen_banded(int32_t n, int32_t hb, int32_t** orp, int32_t** oci, double** ov) {
  return guard([&] {
    if (n < 1) throw invalid_argument("gen_banded: n must be >= 1");
    if (hb < 0 || hb >= n) throw invalid_argument("gen_banded: need 0 <= half_bandwidth < n");
    std::vector<int32_t> rp{0}, ci;
    std::vector<double> v;
    for (int32_t r = 0; r < n; ++r) {
      for (int32_t c = std::max(0, r - hb); c <= std::min(n - 1, r + hb); ++c) {
        ci.push_back(c);
        v.push_back(1.0);
      }
      rp.push_back((int32_t)ci.size());
    }
    export_csr(rp, ci, v, orp, oci, ov);
  });
}

void tfg_free(void* p) { std::free(p); }

}  // extern "C"
