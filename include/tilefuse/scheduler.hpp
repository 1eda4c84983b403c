// tilefuse/scheduler.hpp -- drop-in inspector API over libtfg (tfg.h).
//
// Keeps the reference's names, types and signatures
// (include/tilefuse/scheduler.hpp:15-111): choose_tile_size,
// step1_coarse_fuse, balance, tile_cost, split_tile, build_schedule,
// fused_ratio and validate_schedule all run the GPU inspector's kernels.  build_schedule runs the sm_100a
// GPU inspector and returns the same FusedSchedule, bit for bit, as the
// reference's CPU inspector for the same SchedulerConfig.  Link with
// -ltfg (paper_2407_00243_b200/libtfg.so).
#pragma once

#include <cstddef>
#include <cstdint>
#include <algorithm>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "tfg.h"
#include "tilefuse/csr.hpp"

namespace tilefuse {

struct SchedulerConfig {
  index_t ct_size = 2048;
  int num_workers = 1;
  std::size_t cache_size_words = 160 * 1024;
  index_t b_cols = 32;
  index_t c_cols = 32;
  double index_to_scalar_ratio = 0.5;
  bool b_is_dense = true;
  bool whole_b_cost = false;
};

struct FusedTile {
  index_t i_lo = 0;
  index_t i_hi = 0;
  std::vector<index_t> j_rows;
  double cost = 0.0;
  index_t width() const { return i_hi - i_lo; }
};

struct FusedSchedule {
  index_t n = 0;
  index_t tile_size = 0;
  std::vector<std::vector<FusedTile>> wavefronts;
  std::size_t num_tiles() const {
    std::size_t k = 0;
    for (const auto& w : wavefronts) k += w.size();
    return k;
  }
};

struct IntermediateSchedule {
  index_t n = 0;
  index_t tile_size = 0;
  std::vector<FusedTile> tiles;
  std::vector<index_t> unfused_rows;
};

struct ValidationReport {
  bool pass = true;
  std::vector<std::string> violations;
  std::size_t over_budget_width1 = 0;
};

namespace detail {

inline void tfg_check(tfg_status st) {
  if (st == TFG_OK) return;
  if (st == TFG_EINVAL) throw std::invalid_argument(tfg_last_error());
  throw std::runtime_error(tfg_last_error());
}

inline tfg_config to_c(const SchedulerConfig& c) {
  tfg_config o;
  o.ct_size = c.ct_size;
  o.num_workers = c.num_workers;
  o.cache_size_words = static_cast<uint64_t>(c.cache_size_words);
  o.b_cols = c.b_cols;
  o.c_cols = c.c_cols;
  o.index_to_scalar_ratio = c.index_to_scalar_ratio;
  o.b_is_dense = c.b_is_dense ? 1 : 0;
  o.whole_b_cost = c.whole_b_cost ? 1 : 0;
  return o;
}

// RAII owner of a device schedule handle.
struct DeviceSchedule {
  tfg_schedule* h = nullptr;
  DeviceSchedule() = default;
  explicit DeviceSchedule(tfg_schedule* s) : h(s) {}
  DeviceSchedule(const DeviceSchedule&) = delete;
  DeviceSchedule& operator=(const DeviceSchedule&) = delete;
  DeviceSchedule(DeviceSchedule&& o) noexcept : h(o.h) { o.h = nullptr; }
  ~DeviceSchedule() { if (h) tfg_schedule_destroy(h); }
};

inline FusedSchedule download(const tfg_schedule* s) {
  int32_t n = 0, t = 0;
  int64_t nt[2], nj[2];
  tfg_check(tfg_schedule_info(s, &n, &t, nt, nj, nullptr));
  FusedSchedule out;
  out.n = n;
  out.tile_size = t;
  out.wavefronts.resize(2);
  for (int w = 0; w < 2; ++w) {
    std::vector<int32_t> lo(nt[w] + 1), hi(nt[w] + 1), jr(nj[w] + 1);
    std::vector<double> cost(nt[w] + 1);
    std::vector<int64_t> off(nt[w] + 1);
    tfg_check(tfg_schedule_export(s, w, lo.data(), hi.data(), cost.data(), off.data(), jr.data()));
    out.wavefronts[w].resize(static_cast<std::size_t>(nt[w]));
    for (int64_t v = 0; v < nt[w]; ++v) {
      FusedTile& tile = out.wavefronts[w][static_cast<std::size_t>(v)];
      tile.i_lo = lo[v];
      tile.i_hi = hi[v];
      tile.cost = cost[v];
      tile.j_rows.assign(jr.begin() + off[v], jr.begin() + off[v + 1]);
    }
  }
  return out;
}

inline DeviceSchedule upload(const FusedSchedule& s) {
  if (s.wavefronts.size() != 2)
    throw std::invalid_argument("schedule: expected exactly 2 wavefronts");
  std::vector<int32_t> lo[2], hi[2], jr[2];
  std::vector<double> cost[2];
  std::vector<int64_t> off[2];
  int64_t nt[2];
  for (int w = 0; w < 2; ++w) {
    off[w].push_back(0);
    for (const auto& tile : s.wavefronts[w]) {
      lo[w].push_back(tile.i_lo);
      hi[w].push_back(tile.i_hi);
      cost[w].push_back(tile.cost);
      jr[w].insert(jr[w].end(), tile.j_rows.begin(), tile.j_rows.end());
      off[w].push_back(static_cast<int64_t>(jr[w].size()));
    }
    nt[w] = static_cast<int64_t>(s.wavefronts[w].size());
    lo[w].push_back(0);
    hi[w].push_back(0);
    cost[w].push_back(0.0);
    jr[w].push_back(0);
  }
  const int32_t* plo[2] = {lo[0].data(), lo[1].data()};
  const int32_t* phi[2] = {hi[0].data(), hi[1].data()};
  const double* pc[2] = {cost[0].data(), cost[1].data()};
  const int64_t* po[2] = {off[0].data(), off[1].data()};
  const int32_t* pj[2] = {jr[0].data(), jr[1].data()};
  tfg_schedule* h = nullptr;
  tfg_check(tfg_schedule_import(s.n, s.tile_size, nt, plo, phi, pc, po, pj, &h));
  return DeviceSchedule(h);
}

inline DeviceSchedule build_device(const SparsityView& a, const SchedulerConfig& cfg) {
  const tfg_config c = to_c(cfg);
  tfg_schedule* h = nullptr;
  const int32_t dummy = 0;
  tfg_check(tfg_build_schedule_host(a.n_rows, a.n_cols, a.row_ptr.data(),
                                    a.col_idx.empty() ? &dummy : a.col_idx.data(), &c, nullptr,
                                    &h));
  return DeviceSchedule(h);
}

}  // namespace detail

// scheduler.cpp:124-129
inline index_t choose_tile_size(index_t n, int num_workers, index_t ct_size) {
  int32_t out = 0;
  detail::tfg_check(tfg_choose_tile_size(n, num_workers, ct_size, &out));
  return out;
}

// scheduler.cpp:212-245 -- runs the GPU inspector.
inline FusedSchedule build_schedule(const SparsityView& a, const SchedulerConfig& cfg) {
  auto d = detail::build_device(a, cfg);
  return detail::download(d.h);
}

// scheduler.cpp:131-161 -- the GPU inspector with p = 1, ct = t and an
// unbounded budget performs step 1 only: wavefront 0 is the coarse tiles,
// wavefront 1 the (ascending) leftovers.
inline IntermediateSchedule step1_coarse_fuse(const SparsityView& a, index_t tile_size) {
  if (!a.square()) throw std::invalid_argument("step1_coarse_fuse: matrix must be square");
  if (a.n_rows < 1) throw std::invalid_argument("step1_coarse_fuse: matrix must be nonempty");
  if (tile_size < 1) throw std::invalid_argument("step1_coarse_fuse: tile_size must be >= 1");
  SchedulerConfig cfg;
  cfg.ct_size = tile_size;
  cfg.num_workers = 1;
  cfg.cache_size_words = std::numeric_limits<std::size_t>::max();
  FusedSchedule s = build_schedule(a, cfg);
  IntermediateSchedule out;
  out.n = s.n;
  out.tile_size = s.tile_size;
  out.tiles = std::move(s.wavefronts[0]);
  for (auto& t : out.tiles) t.cost = 0.0;
  for (const auto& t : s.wavefronts[1])
    out.unfused_rows.insert(out.unfused_rows.end(), t.j_rows.begin(), t.j_rows.end());
  return out;
}

// scheduler.cpp:163-194 -- the inspector's k_balance on the list's weights
// (weight of an item = row_weight[row]).
inline std::vector<std::vector<index_t>> balance(const std::vector<index_t>& rows,
                                                 const std::vector<index_t>& row_weight,
                                                 std::size_t num_chunks) {
  std::vector<int64_t> w(rows.size());
  for (std::size_t q = 0; q < rows.size(); ++q) {
    const auto r = static_cast<std::size_t>(rows[q]);
    if (r >= row_weight.size()) throw std::invalid_argument("balance: row without a weight");
    w[q] = row_weight[r];
  }
  std::vector<int64_t> start(num_chunks + 1, 0);
  detail::tfg_check(tfg_balance(static_cast<int64_t>(rows.size()), w.empty() ? nullptr : w.data(),
                                static_cast<int64_t>(num_chunks), start.data()));
  std::vector<std::vector<index_t>> out(num_chunks);
  for (std::size_t c = 0; c < num_chunks; ++c)
    out[c].assign(rows.begin() + start[c], rows.begin() + start[c + 1]);
  return out;
}

// scheduler.cpp:196-200 (Eq. 3) -- the inspector's cost kernel on one tile.
inline double tile_cost(const SparsityView& a, const FusedTile& tile, const SchedulerConfig& cfg) {
  const tfg_config c = detail::to_c(cfg);
  double cost = 0.0;
  const int32_t dummy = 0;
  detail::tfg_check(tfg_tile_cost(a.n_rows, a.row_ptr.data(),
                                  a.col_idx.empty() ? &dummy : a.col_idx.data(), tile.i_lo,
                                  tile.i_hi, tile.j_rows.empty() ? &dummy : tile.j_rows.data(),
                                  static_cast<int64_t>(tile.j_rows.size()), &c, &cost));
  return cost;
}

struct SplitResult {
  std::vector<FusedTile> pieces;      // cost-bounded or width 1, DFS pre-order
  std::vector<index_t> demoted_rows;  // rows evicted while splitting (ascending)
};

// scheduler.cpp:66-93 / :202-210 -- the inspector's split kernel on one tile
// (a tile step 1 produces: its j rows read only columns inside it).
inline SplitResult split_tile(const SparsityView& a, FusedTile tile, const SchedulerConfig& cfg) {
  const tfg_config c = detail::to_c(cfg);
  const auto w = static_cast<std::size_t>(std::max<index_t>(tile.i_hi - tile.i_lo, 1));
  const std::size_t nj = tile.j_rows.size();
  std::vector<int32_t> lo(w), hi(w), jout(nj + 1), dem(nj + 1);
  std::vector<double> cost(w);
  std::vector<int64_t> joff(w + 1);
  int64_t np = 0, nd = 0;
  const int32_t dummy = 0;
  detail::tfg_check(tfg_split_tile(a.n_rows, a.row_ptr.data(),
                                   a.col_idx.empty() ? &dummy : a.col_idx.data(), tile.i_lo,
                                   tile.i_hi, nj ? tile.j_rows.data() : &dummy,
                                   static_cast<int64_t>(nj), &c, &np, lo.data(), hi.data(),
                                   cost.data(), joff.data(), jout.data(), &nd, dem.data()));
  SplitResult r;
  for (int64_t q = 0; q < np; ++q) {
    FusedTile p;
    p.i_lo = lo[q];
    p.i_hi = hi[q];
    p.cost = cost[q];
    p.j_rows.assign(jout.begin() + joff[q], jout.begin() + joff[q + 1]);
    r.pieces.push_back(std::move(p));
  }
  r.demoted_rows.assign(dem.begin(), dem.begin() + nd);
  return r;
}

// scheduler.cpp:247-252 (Eq. 2)
inline double fused_ratio(const FusedSchedule& sched) {
  if (sched.n < 1 || sched.wavefronts.empty()) return 0.0;
  std::size_t fused = 0;
  for (const auto& t : sched.wavefronts[0]) fused += t.j_rows.size();
  return static_cast<double>(fused) / (2.0 * static_cast<double>(sched.n));
}

// scheduler.cpp:254-390 (verify path; every violation, in the reference's
// check order).
inline ValidationReport validate_schedule(const SparsityView& a, const FusedSchedule& sched,
                                          const SchedulerConfig& cfg) {
  ValidationReport rep;
  if (sched.wavefronts.size() != 2) {
    rep.pass = false;
    rep.violations.push_back("expected exactly 2 wavefronts, got " +
                             std::to_string(sched.wavefronts.size()));
    return rep;
  }
  auto d = detail::upload(sched);
  const tfg_config c = detail::to_c(cfg);
  int32_t pass = 0;
  int64_t nv = 0, ob = 0;
  char msg[512];
  const int32_t dummy = 0;
  detail::tfg_check(tfg_validate_schedule(a.n_rows, a.n_cols, a.row_ptr.data(),
                                          a.col_idx.empty() ? &dummy : a.col_idx.data(), d.h, &c,
                                          &pass, &nv, &ob, msg, sizeof msg));
  rep.pass = pass != 0;
  rep.over_budget_width1 = static_cast<std::size_t>(ob);
  if (!rep.pass) {
    std::size_t need = 0;
    detail::tfg_check(tfg_validate_messages(nullptr, 0, &need));
    std::string all(need, '\0');
    detail::tfg_check(tfg_validate_messages(&all[0], need, &need));
    all.resize(need ? need - 1 : 0);
    std::size_t b = 0;
    while (b <= all.size()) {
      const std::size_t e = std::min(all.find('\n', b), all.size());
      if (e > b) rep.violations.push_back(all.substr(b, e - b));
      b = e + 1;
    }
  }
  return rep;
}

}  // namespace tilefuse
