// tfg_inspector.cu -- GPU tile-fusion inspector ("Algorithm 1").
//
// Rebuilds the reference's build_schedule (scheduler.cpp:212-245) as device
// passes over the CSR row pointers, producing a bit-identical schedule:
//
//   1. classify  (step1_coarse_fuse, scheduler.cpp:131-161): one thread per
//      row decides fused tile v = front/t (iff back < tile end), the own-index
//      tile for empty rows, or the unfused bucket.  A stable radix sort on the
//      bucket key groups rows per tile in ascending j (the reference appends
//      rows to each tile in j order).
//   2. split     (split_rec, scheduler.cpp:66-93): one CTA per coarse tile
//      runs the recursive bisection as an explicit DFS stack.  Eq.-3 cost per
//      node: nnz_J by block reduction, distinct columns uc by a shared-memory
//      bitmap over the node's i-range (every column of a fused row lies inside
//      its tile), nnz_B = row_ptr[hi] - row_ptr[lo] in O(1).  Children are
//      built by a stable block-scan partition; straddling rows are demoted.
//      Pieces are emitted in DFS order (left before right).
//   3. compact wavefront 0 by scans (tile order, then DFS order).
//   4. unfused rows = step-1 leftovers + demoted rows, radix-sorted.
//   5. balance   (scheduler.cpp:163-194): the greedy chunking has a
//      sequential dependency across chunks, so one warp walks the chunks and
//      finds each chunk end by a 32-ary search over the prefix sum of row
//      weights (the reserve rule caps it).
//   6. bisect_by_count (scheduler.cpp:95-113): one CTA per chunk, DFS by
//      row count; distinct columns via a per-CTA epoch-marked array in HBM
//      (the reference's CostScratch, scheduler.cpp:19-27, one per CTA).
//   7. compact wavefront 1 (pieces are contiguous runs of the sorted list).
//
// Costs are computed in double with the reference's exact operation order
// (scheduler.cpp:47-63); every intermediate is an integer below 2^53 except
// the single product by index_to_scalar_ratio, so the bits match.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include <chrono>
#include <vector>

#include "tfg_common.cuh"

namespace tfg {
namespace {

struct CostParams {
  double c_cols, b_cols, ratio, budget, n_rows;
  int b_is_dense, whole_b;
};

// tile_cost_ws formula, scheduler.cpp:47-63, same left-to-right order.
__device__ __forceinline__ double eq3_cost(const CostParams& cp, long long uc,
                                           long long nnzj, long long jc,
                                           long long t, long long nnzb) {
  const double dt = (double)t, djc = (double)jc, dn = (double)nnzj,
               du = (double)uc;
  if (cp.b_is_dense) {
    const double first = cp.whole_b ? cp.n_rows : dt;
    const double idx =
        ceil(__dmul_rn(__dadd_rn(__dadd_rn(dn, djc), 1.0), cp.ratio));
    double r = __dadd_rn(__dadd_rn(du, dt), djc);
    r = __dmul_rn(r, cp.c_cols);
    r = __dadd_rn(r, __dmul_rn(first, cp.b_cols));
    return __dadd_rn(r, idx);
  }
  const double db = (double)nnzb;
  double s = __dadd_rn(__dadd_rn(dn, djc), 1.0);
  s = __dadd_rn(__dadd_rn(__dadd_rn(s, db), dt), 1.0);
  const double idx = ceil(__dmul_rn(s, cp.ratio));
  double r = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(db, dn), du), dt), djc);
  r = __dmul_rn(r, cp.c_cols);
  return __dadd_rn(r, idx);
}

// ---- 1. classify ------------------------------------------------------
__global__ void k_classify(int n, int t, int nt, const int* __restrict__ rp,
                           const int* __restrict__ ci, uint32_t* key,
                           int* rows) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += gridDim.x * blockDim.x) {
    const int b = rp[j], e = rp[j + 1];
    int k;
    if (b == e) {
      k = j / t;
    } else {
      const int v = ci[b] / t;
      const long long hi = min((long long)(v + 1) * t, (long long)n);
      k = ((long long)ci[e - 1] < hi) ? v : nt;
    }
    key[j] = (uint32_t)k;
    rows[j] = j;
  }
}

// seg_off[k] = first sorted position with key >= k, k in [0, nt+1].
__global__ void k_seg_bounds(int n, int nt, const uint32_t* __restrict__ skey,
                             int* seg_off) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += gridDim.x * blockDim.x) {
    const int kp = p == 0 ? -1 : (int)skey[p - 1];
    const int kc = (int)skey[p];
    for (int k = kp + 1; k <= kc; ++k) seg_off[k] = p;
    if (p == n - 1)
      for (int k = kc + 1; k <= nt + 1; ++k) seg_off[k] = n;
  }
}

// ---- 2. split (one CTA per coarse tile) --------------------------------
struct Node {
  int lo, hi, start, len;
};

constexpr int kSplitThreads = 256;

template <class T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  T s = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
  return s;
}

__global__ void __launch_bounds__(kSplitThreads)
    k_split(int n, int t, int base, const int* __restrict__ rp,
            const int* __restrict__ ci, const int* __restrict__ seg_off,
            int* buf, int* tmp, int* demoted, int* n_demoted,
            uint32_t* gbitmap, int bm_words, int smem_bitmap, CostParams cp,
            int* pc_lo, int* pc_hi, int* pc_start, int* pc_len,
            double* pc_cost, int* piece_cnt) {
  extern __shared__ uint32_t sbm[];
  __shared__ Node stack[72];
  __shared__ int sp, s_emit, s_npieces;
  __shared__ long long red[kSplitThreads / 32];
  using Scan = cub::BlockScan<int, kSplitThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;

  const int tid = threadIdx.x;
  const int v = blockIdx.x;
  const int tlo = base + (int)((long long)v * t);
  const int thi = (int)min((long long)tlo + t, (long long)n);
  uint32_t* bm = smem_bitmap ? sbm : gbitmap + (size_t)v * bm_words;

  if (tid == 0) {
    sp = 0;
    s_npieces = 0;
    stack[sp++] = Node{tlo, thi, seg_off[v], seg_off[v + 1] - seg_off[v]};
  }
  __syncthreads();
  while (true) {
    if (sp == 0) break;
    const Node nd = stack[sp - 1];
    __syncthreads();
    if (tid == 0) --sp;
    const int w0 = (nd.lo - tlo) >> 5, w1 = (nd.hi - 1 - tlo) >> 5;
    for (int w = w0 + tid; w <= w1; w += blockDim.x) bm[w] = 0u;
    __syncthreads();
    long long my_nnz = 0;
    for (int q = tid; q < nd.len; q += blockDim.x) {
      const int j = buf[nd.start + q];
      const int b = rp[j], e = rp[j + 1];
      my_nnz += e - b;
      for (int k = b; k < e; ++k) {
        const int c = ci[k];
        if (c < nd.lo || c >= nd.hi) continue;  // impossible for valid CSR
        const int r = c - tlo;
        atomicOr(&bm[r >> 5], 1u << (r & 31));
      }
    }
    __syncthreads();
    long long my_uc = 0;
    for (int w = w0 + tid; w <= w1; w += blockDim.x) my_uc += __popc(bm[w]);
    const long long nnzj = block_sum(my_nnz, red);
    const long long uc = block_sum(my_uc, red);
    if (tid == 0) {
      const long long nnzb = (long long)rp[nd.hi] - rp[nd.lo];
      const double cost = eq3_cost(cp, uc, nnzj, nd.len, nd.hi - nd.lo, nnzb);
      const int emit = (cost <= cp.budget) || (nd.hi - nd.lo <= 1);
      s_emit = emit;
      if (emit) {
        const int slot = tlo + s_npieces++;
        pc_lo[slot] = nd.lo;
        pc_hi[slot] = nd.hi;
        pc_start[slot] = nd.start;
        pc_len[slot] = nd.len;
        pc_cost[slot] = cost;
      }
    }
    __syncthreads();
    if (s_emit) {
      __syncthreads();
      continue;
    }
    // Stable three-way partition: left (all cols < mid, or empty & j < mid),
    // right (all cols >= mid, or empty & j >= mid), demoted (straddling).
    const int mid = nd.lo + (nd.hi - nd.lo) / 2;
    long long my_l = 0;
    for (int q = tid; q < nd.len; q += blockDim.x) {
      const int j = buf[nd.start + q];
      const int b = rp[j], e = rp[j + 1];
      my_l += (b == e) ? (j < mid) : (ci[e - 1] < mid);
    }
    const int n_left = (int)block_sum(my_l, red);
    int base_l = 0, base_r = 0;
    for (int q0 = 0; q0 < nd.len; q0 += blockDim.x) {
      const int q = q0 + tid;
      int cls = 3, j = -1;  // 0 left, 1 right, 2 demoted, 3 none
      if (q < nd.len) {
        j = buf[nd.start + q];
        const int b = rp[j], e = rp[j + 1];
        if (b == e)
          cls = j < mid ? 0 : 1;
        else if (ci[e - 1] < mid)
          cls = 0;
        else if (ci[b] >= mid)
          cls = 1;
        else
          cls = 2;
      }
      int rl, rr, tl, tr;
      Scan(scan_tmp).ExclusiveSum(cls == 0 ? 1 : 0, rl, tl);
      __syncthreads();
      Scan(scan_tmp).ExclusiveSum(cls == 1 ? 1 : 0, rr, tr);
      __syncthreads();
      if (cls == 0) tmp[nd.start + base_l + rl] = j;
      if (cls == 1) tmp[nd.start + n_left + base_r + rr] = j;
      if (cls == 2) demoted[atomicAdd(n_demoted, 1)] = j;
      base_l += tl;
      base_r += tr;
    }
    __syncthreads();
    const int kept = base_l + base_r;
    for (int q = tid; q < kept; q += blockDim.x)
      buf[nd.start + q] = tmp[nd.start + q];
    if (tid == 0) {
      stack[sp++] = Node{mid, nd.hi, nd.start + n_left, base_r};
      stack[sp++] = Node{nd.lo, mid, nd.start, n_left};
    }
    __syncthreads();
  }
  if (tid == 0) piece_cnt[v] = s_npieces;
}

// tile_cost (scheduler.cpp:29-64, :196-200) of one arbitrary tile: distinct
// columns of its j rows (anywhere in the matrix) by a global bitmap, then
// the Eq. 3 formula in the reference's operation order.
__global__ void __launch_bounds__(kSplitThreads)
    k_tile_cost(int i_lo, int i_hi, const int* __restrict__ rp, const int* __restrict__ ci,
                const int* __restrict__ jrows, int nj, uint32_t* bm, int bm_words, CostParams cp,
                double* cost) {
  __shared__ long long red[kSplitThreads / 32];
  long long my_nnz = 0;
  for (int q = threadIdx.x; q < nj; q += blockDim.x) {
    const int j = jrows[q];
    for (int k = rp[j]; k < rp[j + 1]; ++k) atomicOr(&bm[ci[k] >> 5], 1u << (ci[k] & 31));
    my_nnz += rp[j + 1] - rp[j];
  }
  __syncthreads();
  long long my_uc = 0;
  for (int w = threadIdx.x; w < bm_words; w += blockDim.x) my_uc += __popc(bm[w]);
  const long long nnzj = block_sum(my_nnz, red);
  const long long uc = block_sum(my_uc, red);
  if (threadIdx.x == 0)
    *cost = eq3_cost(cp, uc, nnzj, nj, i_hi - i_lo, (long long)rp[i_hi] - rp[i_lo]);
}

// ---- 3. wavefront-0 compaction ----------------------------------------
__global__ void k_w0_emit(int nt, int t, const int* __restrict__ piece_cnt,
                          const int* __restrict__ piece_base,
                          const int* pc_lo, const int* pc_hi,
                          const int* pc_start, const int* pc_len,
                          const double* pc_cost, int* i_lo, int* i_hi,
                          double* cost, int64_t* jcnt, int* jstart) {
  for (int v = blockIdx.x; v < nt; v += gridDim.x) {
    const int tlo = (int)((long long)v * t);
    const int base = piece_base[v];
    for (int k = threadIdx.x; k < piece_cnt[v]; k += blockDim.x) {
      const int g = base + k;
      i_lo[g] = pc_lo[tlo + k];
      i_hi[g] = pc_hi[tlo + k];
      cost[g] = pc_cost[tlo + k];
      jcnt[g] = pc_len[tlo + k];
      jstart[g] = pc_start[tlo + k];
    }
  }
}

__global__ void k_copy_pieces(int64_t np, const int64_t* __restrict__ j_off,
                              const int* __restrict__ jstart,
                              const int* __restrict__ buf, int* j_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = warp; g < np; g += nwarps) {
    const int64_t o = j_off[g];
    const int len = (int)(j_off[g + 1] - o);
    const int s = jstart[g];
    for (int q = lane; q < len; q += 32) j_rows[o + q] = buf[s + q];
  }
}

// ---- 4. unfused list ------------------------------------------------------
__global__ void k_gather_unfused(int n1, const int* __restrict__ step1_unf,
                                 int nd, const int* __restrict__ demoted,
                                 uint32_t* out) {
  const int total = n1 + nd;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += gridDim.x * blockDim.x)
    out[q] = (uint32_t)(q < n1 ? step1_unf[q] : demoted[q - n1]);
}

__global__ void k_row_weights(int64_t U, const uint32_t* __restrict__ unf,
                              const int* __restrict__ rp, int64_t* w) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < U;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)unf[q];
    w[q] = rp[j + 1] - rp[j];
  }
}

// ---- 5. balance (one warp) ----------------------------------------------
// Largest e in [lo, hi] with P[e] <= target, given P[lo] <= target.
__device__ int64_t warp_last_leq(const int64_t* __restrict__ P, int64_t lo,
                                 int64_t hi, long long target) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    int64_t idx = lo + (int64_t)(lane + 1) * step;
    if (idx > hi) idx = hi;
    const bool pred = P[idx] <= target;
    const unsigned bal = __ballot_sync(0xffffffffu, pred);
    const int k = __popc(bal);  // monotone: true...true false...false
    const int64_t idx_k1 = __shfl_sync(0xffffffffu, idx, k > 0 ? k - 1 : 0);
    const int64_t idx_k = __shfl_sync(0xffffffffu, idx, k < 32 ? k : 31);
    if (k == 32) return hi;
    const int64_t nlo = k > 0 ? idx_k1 : lo;
    hi = idx_k - 1;
    lo = nlo;
  }
  const int64_t idx = lo + lane + 1;
  const bool pred = idx <= hi && P[idx] <= target;
  const int k = __popc(__ballot_sync(0xffffffffu, pred));
  return lo + k;
}

__global__ void k_balance(int64_t U, int64_t num_chunks,
                          const int64_t* __restrict__ P, int64_t* chunk_s,
                          int64_t* n_chunks_out) {
  if (threadIdx.x >= 32) return;
  int64_t s = 0;
  long long rem = P[U];
  int64_t c = 0;
  for (; c < num_chunks && s < U; ++c) {
    const int64_t rc = num_chunks - c;
    const long long ideal = (rem + rc - 1) / rc;
    const long long target = P[s] + ideal;
    int64_t e = warp_last_leq(P, s, U, target);
    const int64_t lim = U - rc + 1;
    if (e > lim) e = lim;
    if (e < s + 1) e = s + 1;
    if (threadIdx.x == 0) chunk_s[c] = s;
    rem -= P[e] - P[s];
    s = e;
  }
  if (threadIdx.x == 0) {
    chunk_s[c] = s;
    *n_chunks_out = c;
  }
}

// ---- 6. bisect_by_count (one CTA per chunk, persistent) -------------------
constexpr int kBisectThreads = 512;

__global__ void __launch_bounds__(kBisectThreads)
    k_bisect(int64_t nck, const int64_t* __restrict__ chunk_s,
             const uint32_t* __restrict__ unf, const int64_t* __restrict__ P,
             const int* __restrict__ rp, const int* __restrict__ ci,
             int* marks_all, int n, CostParams cp, uint8_t* pc1_flag,
             double* pc1_cost) {
  __shared__ int64_t st_s[72], st_l[72];
  __shared__ int sp, s_emit;
  __shared__ long long red[kBisectThreads / 32];
  int* marks = marks_all + (size_t)blockIdx.x * n;
  int epoch = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t c = blockIdx.x; c < nck; c += gridDim.x) {
    if (threadIdx.x == 0) {
      sp = 0;
      st_s[sp] = chunk_s[c];
      st_l[sp] = chunk_s[c + 1] - chunk_s[c];
      ++sp;
    }
    __syncthreads();
    while (true) {
      if (sp == 0) break;
      const int64_t s = st_s[sp - 1], len = st_l[sp - 1];
      __syncthreads();
      if (threadIdx.x == 0) --sp;
      ++epoch;
      long long my_uc = 0;
      for (int64_t q = wid; q < len; q += nw) {
        const int j = (int)unf[s + q];
        const int b = rp[j], e = rp[j + 1];
        for (int k = b + lane; k < e; k += 32) {
          const int old = atomicExch(&marks[ci[k]], epoch);
          my_uc += old != epoch;
        }
      }
      const long long uc = block_sum(my_uc, red);
      if (threadIdx.x == 0) {
        const long long nnzj = P[s + len] - P[s];
        const double cost = eq3_cost(cp, uc, nnzj, len, 0, 0);
        const int emit = (cost <= cp.budget) || (len <= 1);
        s_emit = emit;
        if (emit) {
          pc1_flag[s] = 1;
          pc1_cost[s] = cost;
        } else {
          const int64_t half = len / 2;
          st_s[sp] = s + half;
          st_l[sp] = len - half;
          ++sp;
          st_s[sp] = s;
          st_l[sp] = half;
          ++sp;
        }
      }
      __syncthreads();
    }
    __syncthreads();
  }
}

// ---- 7. wavefront-1 compaction --------------------------------------------
__global__ void k_w1_emit(int64_t U, const uint8_t* __restrict__ flag,
                          const int64_t* __restrict__ pos,
                          const double* __restrict__ pc1_cost, int* i_lo,
                          int* i_hi, double* cost, int64_t* j_off) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < U;
       q += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[q]) continue;
    const int64_t g = pos[q];
    i_lo[g] = 0;
    i_hi[g] = 0;
    cost[g] = pc1_cost[q];
    j_off[g] = q;
  }
}

__global__ void k_u8_to_i64(int64_t U, const uint8_t* f, int64_t* o) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < U;
       q += (int64_t)gridDim.x * blockDim.x)
    o[q] = f[q];
}

// CUB helpers with a reusable scratch buffer.
struct CubScratch {
  dbuf<unsigned char> buf;
  void* get(size_t bytes) {
    if (bytes > buf.n) buf.alloc(bytes + (bytes >> 2) + 256);
    return buf.p;
  }
};

template <class T>
T fetch(const T* d, cudaStream_t s) {
  T h{};
  TFG_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  TFG_CUDA(cudaStreamSynchronize(s));
  return h;
}

inline int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (g > cap) g = cap;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

// The GPU inspector entry (C-ABI wrapper lives in tfg_api.cu).
void build_schedule_device(int32_t n_rows, int32_t n_cols, int64_t nnz,
                           const int32_t* rp, const int32_t* ci,
                           const tfg_config& cfg, cudaStream_t st,
                           tfg_schedule& out) {
  (void)nnz;
  if (n_rows != n_cols)
    throw invalid_argument("build_schedule: matrix must be square");
  if (n_rows < 1) throw invalid_argument("build_schedule: matrix must be nonempty");
  if (cfg.num_workers < 1 || cfg.ct_size < 1)
    throw invalid_argument("choose_tile_size: all inputs must be >= 1");
  const auto t0 = std::chrono::steady_clock::now();
  const int n = n_rows;
  const int p = cfg.num_workers, ct = cfg.ct_size;
  const int t = ((n + ct - 1) / ct) >= p ? ct : (n + p - 1) / p;
  const int nt = (int)(((int64_t)n + t - 1) / t);

  CostParams cp;
  cp.c_cols = (double)cfg.c_cols;
  cp.b_cols = (double)cfg.b_cols;
  cp.ratio = cfg.index_to_scalar_ratio;
  cp.budget = (double)cfg.cache_size_words;
  cp.n_rows = (double)n;
  cp.b_is_dense = cfg.b_is_dense != 0;
  cp.whole_b = cfg.whole_b_cost != 0;

  CubScratch cub_tmp;
  size_t tb = 0;

  // 1. classify + stable group by tile
  dbuf<uint32_t> key(n), skey(n);
  dbuf<int> rows(n), buf(n), tmp(n), seg_off(nt + 2);
  k_classify<<<grid_for(n, 256), 256, 0, st>>>(n, t, nt, rp, ci, key.p, rows.p);
  TFG_LAUNCH_CHECK();
  const int kbits = ceil_log2_bits((uint64_t)nt);
  TFG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, skey.p, rows.p,
                                           buf.p, n, 0, kbits, st));
  TFG_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp.get(tb), tb, key.p, skey.p,
                                           rows.p, buf.p, n, 0, kbits, st));
  k_seg_bounds<<<grid_for(n, 256), 256, 0, st>>>(n, nt, skey.p, seg_off.p);
  TFG_LAUNCH_CHECK();

  // 2. split each coarse tile
  const int bm_words = (t + 31) / 32 + 2;
  const size_t bm_bytes = (size_t)bm_words * 4;
  const bool smem_bm = bm_bytes <= 160 * 1024;
  dbuf<uint32_t> gbm;
  if (!smem_bm) gbm.alloc((size_t)bm_words * nt);
  if (smem_bm && bm_bytes > 48 * 1024)
    TFG_CUDA(cudaFuncSetAttribute(k_split, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)bm_bytes));
  dbuf<int> demoted(n), n_demoted(1), pc_lo(n), pc_hi(n), pc_start(n),
      pc_len(n), piece_cnt(nt), piece_base(nt);
  dbuf<double> pc_cost(n);
  TFG_CUDA(cudaMemsetAsync(n_demoted.p, 0, sizeof(int), st));
  k_split<<<nt, kSplitThreads, smem_bm ? bm_bytes : 0, st>>>(
      n, t, 0, rp, ci, seg_off.p, buf.p, tmp.p, demoted.p, n_demoted.p, gbm.p,
      bm_words, smem_bm ? 1 : 0, cp, pc_lo.p, pc_hi.p, pc_start.p, pc_len.p,
      pc_cost.p, piece_cnt.p);
  TFG_LAUNCH_CHECK();

  // 3. compact wavefront 0
  TFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, piece_cnt.p, piece_base.p, nt, st));
  TFG_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp.get(tb), tb, piece_cnt.p,
                                         piece_base.p, nt, st));
  const int last_base = fetch(piece_base.p + nt - 1, st);
  const int last_cnt = fetch(piece_cnt.p + nt - 1, st);
  const int64_t P0 = (int64_t)last_base + last_cnt;
  out.n = n;
  out.tile_size = t;
  out.n_tiles[0] = P0;
  out.i_lo[0].alloc(P0 + 1);
  out.i_hi[0].alloc(P0 + 1);
  out.cost[0].alloc(P0 + 1);
  out.j_off[0].alloc(P0 + 1);
  dbuf<int64_t> jcnt(P0 + 1);
  dbuf<int> jstart(P0 + 1);
  k_w0_emit<<<grid_for((int64_t)nt * 32, 32) , 128, 0, st>>>(
      nt, t, piece_cnt.p, piece_base.p, pc_lo.p, pc_hi.p, pc_start.p, pc_len.p,
      pc_cost.p, out.i_lo[0].p, out.i_hi[0].p, out.cost[0].p, jcnt.p, jstart.p);
  TFG_LAUNCH_CHECK();
  TFG_CUDA(cudaMemsetAsync(jcnt.p + P0, 0, sizeof(int64_t), st));
  TFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, jcnt.p, out.j_off[0].p, P0 + 1, st));
  TFG_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp.get(tb), tb, jcnt.p,
                                         out.j_off[0].p, P0 + 1, st));
  const int64_t F = fetch(out.j_off[0].p + P0, st);
  out.n_jrows[0] = F;
  out.j_rows[0].alloc(F + 1);
  if (P0 > 0) {
    k_copy_pieces<<<grid_for(P0 * 32, 256), 256, 0, st>>>(
        P0, out.j_off[0].p, jstart.p, buf.p, out.j_rows[0].p);
    TFG_LAUNCH_CHECK();
  }

  // 4. unfused rows = step-1 leftovers (sorted bucket nt) + demoted, sorted
  const int seg_nt = fetch(seg_off.p + nt, st);
  const int n1 = n - seg_nt;
  const int nd = fetch(n_demoted.p, st);
  const int64_t U = (int64_t)n1 + nd;
  out.n_jrows[1] = U;
  if (U == 0) {
    out.n_tiles[1] = 0;
    out.i_lo[1].alloc(1);
    out.i_hi[1].alloc(1);
    out.cost[1].alloc(1);
    out.j_off[1].alloc(1);
    TFG_CUDA(cudaMemsetAsync(out.j_off[1].p, 0, sizeof(int64_t), st));
    out.j_rows[1].alloc(1);
  } else {
    dbuf<uint32_t> unf_in(U), unf(U);
    k_gather_unfused<<<grid_for(U, 256), 256, 0, st>>>(
        n1, buf.p + seg_nt, nd, demoted.p, unf_in.p);
    // note: buf[seg_nt..n) was never touched by k_split (it owns only tile
    // segments), so it still holds the ascending step-1 leftovers.
    TFG_LAUNCH_CHECK();
    const int rbits = ceil_log2_bits((uint64_t)(n - 1));
    TFG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, unf_in.p, unf.p, (int)U, 0, rbits, st));
    TFG_CUDA(cub::DeviceRadixSort::SortKeys(cub_tmp.get(tb), tb, unf_in.p,
                                            unf.p, (int)U, 0, rbits, st));
    dbuf<int64_t> w(U), P(U + 1);
    k_row_weights<<<grid_for(U, 256), 256, 0, st>>>(U, unf.p, rp, w.p);
    TFG_LAUNCH_CHECK();
    TFG_CUDA(cudaMemsetAsync(P.p, 0, sizeof(int64_t), st));
    TFG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, w.p, P.p + 1, U, st));
    TFG_CUDA(cub::DeviceScan::InclusiveSum(cub_tmp.get(tb), tb, w.p, P.p + 1, U, st));

    // 5. balance
    const int64_t by_ct = (U + ct - 1) / ct;
    const int64_t chunks = std::max<int64_t>((int64_t)p, by_ct);
    dbuf<int64_t> chunk_s(chunks + 1), nck_d(1);
    k_balance<<<1, 32, 0, st>>>(U, chunks, P.p, chunk_s.p, nck_d.p);
    TFG_LAUNCH_CHECK();
    const int64_t nck = fetch(nck_d.p, st);

    // 6. bisect_by_count
    dbuf<uint8_t> flag(U);
    dbuf<double> pc1_cost(U);
    TFG_CUDA(cudaMemsetAsync(flag.p, 0, U, st));
    int64_t G = std::min<int64_t>(nck, (int64_t)sm_count() * 2);
    const int64_t mark_cap = (int64_t)1 << 29;  // ints of mark scratch (2 GiB)
    G = std::max<int64_t>(1, std::min<int64_t>(G, mark_cap / n));
    dbuf<int> marks((size_t)G * n);
    TFG_CUDA(cudaMemsetAsync(marks.p, 0, marks.bytes(), st));
    k_bisect<<<(int)G, kBisectThreads, 0, st>>>(nck, chunk_s.p, unf.p, P.p, rp,
                                                ci, marks.p, n, cp, flag.p,
                                                pc1_cost.p);
    TFG_LAUNCH_CHECK();

    // 7. compact wavefront 1
    dbuf<int64_t> f64(U), pos(U);
    k_u8_to_i64<<<grid_for(U, 256), 256, 0, st>>>(U, flag.p, f64.p);
    TFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, f64.p, pos.p, U, st));
    TFG_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp.get(tb), tb, f64.p, pos.p, U, st));
    const int64_t P1 = fetch(pos.p + U - 1, st) + fetch(f64.p + U - 1, st);
    out.n_tiles[1] = P1;
    out.i_lo[1].alloc(P1 + 1);
    out.i_hi[1].alloc(P1 + 1);
    out.cost[1].alloc(P1 + 1);
    out.j_off[1].alloc(P1 + 1);
    k_w1_emit<<<grid_for(U, 256), 256, 0, st>>>(U, flag.p, pos.p, pc1_cost.p,
                                                out.i_lo[1].p, out.i_hi[1].p,
                                                out.cost[1].p, out.j_off[1].p);
    TFG_LAUNCH_CHECK();
    TFG_CUDA(cudaMemcpyAsync(out.j_off[1].p + P1, &U, sizeof(int64_t),
                             cudaMemcpyHostToDevice, st));
    out.j_rows[1].alloc(U);
    TFG_CUDA(cudaMemcpyAsync(out.j_rows[1].p, unf.p, U * sizeof(int32_t),
                             cudaMemcpyDeviceToDevice, st));
  }
  TFG_CUDA(cudaStreamSynchronize(st));
  out.inspect_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}


// ---- single-step entry points (scheduler.hpp:80-97): the same kernels the
// pipeline runs, on one tile / one list -------------------------------------
static CostParams cost_params(const tfg_config& cfg, int n) {
  CostParams cp;
  cp.c_cols = (double)cfg.c_cols;
  cp.b_cols = (double)cfg.b_cols;
  cp.ratio = cfg.index_to_scalar_ratio;
  cp.budget = (double)cfg.cache_size_words;
  cp.n_rows = (double)n;
  cp.b_is_dense = cfg.b_is_dense != 0;
  cp.whole_b = cfg.whole_b_cost != 0;
  return cp;
}

double tile_cost_device(int n, const int* rp, const int* ci, int i_lo, int i_hi,
                        const int* jrows, int nj, const tfg_config& cfg, cudaStream_t st) {
  if (i_lo < 0 || i_hi > n || i_lo > i_hi) throw invalid_argument("tile_cost: i_range out of bounds");
  const int bm_words = (n + 31) / 32;
  dbuf<uint32_t> bm(bm_words);
  TFG_CUDA(cudaMemsetAsync(bm.p, 0, (size_t)bm_words * 4, st));
  dbuf<double> cost(1);
  k_tile_cost<<<1, kSplitThreads, 0, st>>>(i_lo, i_hi, rp, ci, jrows, nj, bm.p, bm_words,
                                          cost_params(cfg, n), cost.p);
  TFG_LAUNCH_CHECK();
  double h = 0;
  TFG_CUDA(cudaMemcpyAsync(&h, cost.p, sizeof h, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaStreamSynchronize(st));
  return h;
}

// split_tile through k_split on one coarse tile (base = i_lo, width t =
// i_hi - i_lo): pieces in DFS pre-order, demoted rows ascending.  j rows must
// lie inside the tile (the tiles step 1 produces).
void split_tile_device(int n, const int* rp, const int* ci, int i_lo, int i_hi, const int* jrows,
                       int nj, const tfg_config& cfg, cudaStream_t st, std::vector<int>& lo,
                       std::vector<int>& hi, std::vector<double>& cost,
                       std::vector<int64_t>& joff, std::vector<int>& jout,
                       std::vector<int>& demoted) {
  if (i_lo < 0 || i_hi > n || i_lo >= i_hi) throw invalid_argument("split_tile: i_range out of bounds");
  const int t = i_hi - i_lo;
  dbuf<int> seg(3), buf(std::max(nj, 1)), tmp(std::max(nj, 1)), dem(std::max(nj, 1)), ndem(1);
  const int so[3] = {0, nj, nj};
  TFG_CUDA(cudaMemcpyAsync(seg.p, so, sizeof so, cudaMemcpyHostToDevice, st));
  if (nj) TFG_CUDA(cudaMemcpyAsync(buf.p, jrows, (size_t)nj * 4, cudaMemcpyDeviceToDevice, st));
  TFG_CUDA(cudaMemsetAsync(ndem.p, 0, 4, st));
  const int bm_words = (t + 31) / 32 + 2;
  dbuf<uint32_t> gbm(bm_words);
  dbuf<int> pc_lo(n), pc_hi(n), pc_start(n), pc_len(n), pcnt(1);
  dbuf<double> pc_cost(n);
  k_split<<<1, kSplitThreads, 0, st>>>(n, t, i_lo, rp, ci, seg.p, buf.p, tmp.p, dem.p, ndem.p,
                                       gbm.p, bm_words, 0, cost_params(cfg, n), pc_lo.p, pc_hi.p,
                                       pc_start.p, pc_len.p, pc_cost.p, pcnt.p);
  TFG_LAUNCH_CHECK();
  int np = 0, nd = 0;
  TFG_CUDA(cudaMemcpyAsync(&np, pcnt.p, 4, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaMemcpyAsync(&nd, ndem.p, 4, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaStreamSynchronize(st));
  std::vector<int> start(np), len(np), rows(std::max(nj, 1));
  lo.resize(np);
  hi.resize(np);
  cost.resize(np);
  demoted.resize(nd);
  TFG_CUDA(cudaMemcpyAsync(lo.data(), pc_lo.p + i_lo, (size_t)np * 4, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaMemcpyAsync(hi.data(), pc_hi.p + i_lo, (size_t)np * 4, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaMemcpyAsync(cost.data(), pc_cost.p + i_lo, (size_t)np * 8, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaMemcpyAsync(start.data(), pc_start.p + i_lo, (size_t)np * 4, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaMemcpyAsync(len.data(), pc_len.p + i_lo, (size_t)np * 4, cudaMemcpyDeviceToHost, st));
  if (nj) TFG_CUDA(cudaMemcpyAsync(rows.data(), buf.p, (size_t)nj * 4, cudaMemcpyDeviceToHost, st));
  if (nd) TFG_CUDA(cudaMemcpyAsync(demoted.data(), dem.p, (size_t)nd * 4, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaStreamSynchronize(st));
  std::sort(demoted.begin(), demoted.end());
  joff.assign(1, 0);
  jout.clear();
  for (int q = 0; q < np; ++q) {
    jout.insert(jout.end(), rows.begin() + start[q], rows.begin() + start[q] + len[q]);
    joff.push_back((int64_t)jout.size());
  }
}

// balance through k_balance: chunk starts over a weight list
void balance_device(int64_t U, const int64_t* h_w, int64_t num_chunks, int64_t* h_starts,
                    cudaStream_t st) {
  if (num_chunks < 1) throw invalid_argument("balance: num_chunks must be >= 1");
  std::vector<int64_t> P(U + 1, 0);
  for (int64_t q = 0; q < U; ++q) P[q + 1] = P[q] + h_w[q];
  dbuf<int64_t> Pd(U + 1), cs(num_chunks + 1), nc(1);
  TFG_CUDA(cudaMemcpyAsync(Pd.p, P.data(), (size_t)(U + 1) * 8, cudaMemcpyHostToDevice, st));
  k_balance<<<1, 32, 0, st>>>(U, num_chunks, Pd.p, cs.p, nc.p);
  TFG_LAUNCH_CHECK();
  int64_t c = 0;
  TFG_CUDA(cudaMemcpyAsync(&c, nc.p, 8, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaStreamSynchronize(st));
  TFG_CUDA(cudaMemcpyAsync(h_starts, cs.p, (size_t)(c + 1) * 8, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaStreamSynchronize(st));
  for (int64_t k = c + 1; k <= num_chunks; ++k) h_starts[k] = U;  // trailing empty chunks
}

}  // namespace tfg
