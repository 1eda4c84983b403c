// tfg_executor.cu -- sm_100a executors for D = A (B C) under a two-wavefront
// tile-fusion schedule (kernels.hpp:88-155 fused_run / unfused_run).
//
// Execution of a plan (one stream, kernel boundaries = wavefront barriers):
//
//   (a) first op for wavefront-0 tiles that fuse no second-op row: a dense
//       register-tiled GEMM (B dense) or a CSR SpMM with X = C (B sparse),
//       writing D1 rows to HBM -- every such row is read by wavefront 1.
//   (b) the fused wavefront-0 kernel: one CTA per (tile, column slice).  The
//       tile's D1 slice is computed into shared memory; only rows that some
//       wavefront-1 row reads (the spill set S) are also written to HBM; the
//       tile's fused D rows are then computed from shared memory.  D1 rows
//       outside S never touch HBM (the paper's fused tile).  Tiles too wide
//       for shared memory stage through HBM/L2 inside the same CTA.
//   (c) wavefront 1: CSR SpMM over the wavefront-1 rows reading D1 from HBM;
//       rows longer than kLongRow are split into fixed segments whose
//       partial rows are combined in a fixed order (no atomics: the result is
//       bitwise reproducible run to run).
//
// Numerics.  The SpMM kernels reproduce the reference's per-element order
// exactly: out[q] = ((0 + a0*x0) + a1*x1) + ... in ascending nonzero order
// with separately rounded products and sums (kernels.hpp:71-80), so every
// SpMM row shorter than kLongRow is bit-identical to the reference.  The
// dense first op accumulates B[i,j]*C[j,k] in ascending j with fused
// multiply-add (within the north-star tolerance); fused and unfused paths
// use the same per-element order, so they agree bitwise with each other.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <memory>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tfg_common.cuh"
#include "tfg_device.cuh"
#include "tfg_tc.cuh"
#include "tfg_stencil.cuh"
#include "tfg_nccl.cuh"

namespace tfg {
namespace {

constexpr int kLongRow = 4096;  // rows with more nonzeros are segmented
constexpr int kSegLen = 2048;   // nonzeros per segment

using namespace dev;

// ---- SpMM over a row list (short rows) ------------------------------------
// A group of LPR lanes walks a strip of STRIP rows (STRIP <= LPR) in order.
// The strip's row bounds are loaded once (lane q holds row q), the index
// chunk of the next row is prefetched while the current row's X rows are
// gathered, and X gathers are issued UNR at a time (predicated), so each
// row costs about one dependent memory round trip.  Per-element order stays
// ascending with separately rounded mul/add (kernels.hpp:75-79).
template <class T, int VEC, int LPR, int NCH, int UNR, int MINB = 1, int STRIP = LPR,
          bool FMA = false>
__global__ void __launch_bounds__(256, MINB)
    k_spmm_strip(int64_t nrows, const int* __restrict__ rows, int row0,
                 const int* __restrict__ rp, const int* __restrict__ ci,
                 const T* __restrict__ av, const T* __restrict__ X, int ldx,
                 T* __restrict__ out, int ldo) {
  static_assert(STRIP >= 1 && STRIP <= LPR, "strip");
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR;
  const int64_t base = g * STRIP;
  if (base >= nrows) return;
  const int gl = threadIdx.x & (LPR - 1);
  const unsigned gmask = group_mask(LPR);
  const int cnt = (int)(nrows - base < STRIP ? nrows - base : STRIP);
  int my_r = 0, my_b = 0, my_e = 0;
  if (gl < cnt) {
    my_r = rows ? __ldg(rows + base + gl) : row0 + (int)(base + gl);
    my_b = __ldg(rp + my_r);
    my_e = __ldg(rp + my_r + 1);
  }
  int q = 0;
  int e = __shfl_sync(gmask, my_e, 0, LPR);
  int k0 = __shfl_sync(gmask, my_b, 0, LPR);
  int c = 0;
  T a = T(0);
  if (k0 + gl < e) {
    c = __ldg(ci + k0 + gl);
    a = __ldg(av + k0 + gl);
  }
  T acc[NCH][VEC];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[ch][v] = T(0);
  while (q < cnt) {
    const int n_here = min(LPR, e - k0);
    // next cursor: same row, next chunk -- or the next row's first chunk
    const bool row_done = k0 + LPR >= e;
    int nq = q, nk0 = k0 + LPR, ne = e;
    if (row_done) {
      nq = q + 1;
      const int src = nq < cnt ? nq : 0;
      nk0 = __shfl_sync(gmask, my_b, src, LPR);
      ne = __shfl_sync(gmask, my_e, src, LPR);
    }
    int c2 = 0;
    T a2 = T(0);
    if (nq < cnt && nk0 + gl < ne) {
      c2 = __ldg(ci + nk0 + gl);
      a2 = __ldg(av + nk0 + gl);
    }
    for (int u0 = 0; u0 < n_here; u0 += UNR) {
      int cu[UNR];
      T au[UNR];
      T x[UNR][NCH][VEC];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        cu[u] = __shfl_sync(gmask, c, (u0 + u) & (LPR - 1), LPR);
        au[u] = __shfl_sync(gmask, a, (u0 + u) & (LPR - 1), LPR);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (u0 + u < n_here) {
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
            ldv<T, VEC>(x[u][ch], X + (size_t)cu[u] * ldx + (ch * LPR + gl) * VEC);
        }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (u0 + u < n_here) {
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int v = 0; v < VEC; ++v)
              acc[ch][v] = madd<T, FMA>(acc[ch][v], au[u], x[u][ch][v]);
        }
    }
    if (row_done) {
      const int r = __shfl_sync(gmask, my_r, q, LPR);
      T* o = out + (size_t)r * ldo;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        stv<T, VEC>(o + (ch * LPR + gl) * VEC, acc[ch]);
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[ch][v] = T(0);
      }
    }
    q = nq;
    k0 = nk0;
    e = ne;
    c = c2;
    a = a2;
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- band-staged SpMM (TMA bulk copies into shared memory) -------------------
// For matrices whose consecutive rows reuse a few contiguous ranges of X rows
// (stencils, banded matrices), the plan cuts the row list into blocks of R
// rows and records, per block, the union of X rows it reads as <= kBandRuns
// contiguous runs plus a compact local index record (uint16 row offsets and
// uint16 stage slots).  A persistent CTA double-buffers blocks: one thread
// issues cp.async.bulk copies of the runs (row-major X rows are contiguous)
// and of the index record, completing on an mbarrier; all threads cp.async
// the block's values from the live CSR.  Rows are then summed from shared
// memory in the reference order (bit-identical), so each X row crosses
// L2->SM once per block instead of once per nonzero.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// the CTA's cp.async copies issued so far arrive on the barrier when complete
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "n"(BYTES));
}

constexpr int kBandRuns = 32;
// diagonal lines of a stencil matrix: diagonals [first[l], first[l] + cnt[l])
// of the ascending global offset set have consecutive column offsets
struct DiaLines {
  int nlines = 0, ndiag = 0;
  int first[16] = {}, cnt[16] = {};
};
constexpr int kBandMG = 4;  // rows per register-reuse mini-group
constexpr size_t kBandSmemMax = 200 * 1024;

// For a regular mini-group (every row has the global diagonal set) each
// diagonal line's X rows are loaded once into a sliding register window and
// applied to all 4 rows: row q, diagonal d of a line reads window slot q + d.
// Per row the terms are still added in ascending column order (lines and
// diagonals ascend), separately rounded -- the reference's order.  Other
// mini-groups take the per-row path.
template <class T, int VEC, int NCH>
__device__ __forceinline__ void band_dia_group(const T* __restrict__ xs, const T* __restrict__ vs,
                                               const uint16_t* lrp, const uint16_t* lsl, int cc,
                                               int q0, const DiaLines& dl, int lane,
                                               T* __restrict__ out_row0, int ldo) {
  constexpr int M = 4, WMAX = M + 4;
  T acc[M][NCH][VEC];
#pragma unroll
  for (int q = 0; q < M; ++q)
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[q][ch][v] = T(0);
  int e[M];
#pragma unroll
  for (int q = 0; q < M; ++q) e[q] = lrp[q0 + q];
  for (int l = 0; l < dl.nlines; ++l) {
    const int d0 = dl.first[l], dc = dl.cnt[l];
    const int base = lsl[e[0] + d0];  // slot of X row (row q0 + offset of d0)
    T w[WMAX][NCH][VEC];
#pragma unroll
    for (int k = 0; k < WMAX; ++k)
      if (k < M + dc - 1)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
          ldv<T, VEC>(w[k][ch], xs + (size_t)(base + k) * cc + (ch * 32 + lane) * VEC);
#pragma unroll
    for (int q = 0; q < M; ++q)
#pragma unroll
      for (int d = 0; d < 5; ++d)
        if (d < dc) {
          const T a = vs[e[q] + d0 + d];
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int v = 0; v < VEC; ++v)
              acc[q][ch][v] = fops<T>::add(acc[q][ch][v], fops<T>::mul(a, w[q + d][ch][v]));
        }
  }
#pragma unroll
  for (int q = 0; q < M; ++q)
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
      stv<T, VEC>(out_row0 + (size_t)q * ldo + (ch * 32 + lane) * VEC, acc[q][ch]);
}

// One row of a staged band block, a whole warp (LPR = 32) per row, reference
// order.
template <class T, int VEC, int NCH>
__device__ __forceinline__ void band_row_warp(const T* __restrict__ xs, const T* __restrict__ vs,
                                              const uint16_t* lrp, const uint16_t* lsl, int cc,
                                              int r, int lane, T* __restrict__ o) {
  const int eb = lrp[r], ee = lrp[r + 1];
  T acc[NCH][VEC];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[ch][v] = T(0);
  for (int e0 = eb; e0 < ee; e0 += 32) {
    const int sl = e0 + lane < ee ? lsl[e0 + lane] : 0;
    const int cnt = min(32, ee - e0);
    for (int u = 0; u < cnt; ++u) {
      const int su = __shfl_sync(0xffffffffu, sl, u);
      const T au = vs[e0 + u];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        T x[VEC];
        ldv<T, VEC>(x, xs + (size_t)su * cc + (ch * 32 + lane) * VEC);
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[ch][v] = fops<T>::add(acc[ch][v], fops<T>::mul(au, x[v]));
      }
    }
  }
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) stv<T, VEC>(o + (ch * 32 + lane) * VEC, acc[ch]);
}

// All rows of a staged block with the stencil consumer: regular mini-groups
// (bit g of the record's mask) through band_dia_group, the rest row by row.
template <class T, int VEC, int NCH, int NWARPS>
__device__ __forceinline__ void band_block_dia(const T* __restrict__ xs, const T* __restrict__ vs,
                                               const uint16_t* lrp, const uint16_t* lsl, int cc,
                                               int nr, const DiaLines& dl, int warp, int lane,
                                               T* __restrict__ out_r0, int ldo) {
  const int nnzb = lrp[nr];
  const uint32_t reg = (uint32_t)lsl[nnzb] | ((uint32_t)lsl[nnzb + 1] << 16);
  const int nmg = (nr + 3) / 4;
  for (int g = warp; g < nmg; g += NWARPS) {
    if ((reg >> g) & 1u) {
      band_dia_group<T, VEC, NCH>(xs, vs, lrp, lsl, cc, 4 * g, dl, lane,
                                  out_r0 + (size_t)(4 * g) * ldo, ldo);
      continue;
    }
    for (int r = 4 * g; r < min(4 * g + 4, nr); ++r)
      band_row_warp<T, VEC, NCH>(xs, vs, lrp, lsl, cc, r, lane, out_r0 + (size_t)r * ldo);
  }
}

template <class T, int VEC, int LPR, int NCH, int STAGES, bool DIA = false>
__global__ void __launch_bounds__(288, (DIA && NCH == 1) ? 2 : 1)
    k_spmm_band3(int nblk, int R, int row0, int nrows, const int* __restrict__ rp,
                 const T* __restrict__ av, const int* __restrict__ run_begin,
                 const int* __restrict__ run_start, const int* __restrict__ run_len,
                 const int64_t* __restrict__ idx_off, const uint16_t* __restrict__ lidx,
                 int stage_cap, int idx_cap, int val_cap, const T* __restrict__ X, int ldx,
                 T* __restrict__ out, int ldo, const DiaLines* __restrict__ dlp = nullptr) {
  static_assert(!DIA || LPR == 32, "DIA consumer: a warp per row");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int cc = ldx;
  const size_t xbytes = (size_t)stage_cap * cc * sizeof(T);
  const size_t ibytes = ((size_t)idx_cap * 2 + 15) / 16 * 16;
  const size_t vbytes = ((size_t)val_cap * sizeof(T) + 15) / 16 * 16;
  const size_t bufbytes = xbytes + ibytes + vbytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NCONS = 8;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  const int nmine = blockIdx.x < nblk ? (nblk - 1 - blockIdx.x) / G + 1 : 0;
  if (warp == NCONS) {
    // ---------------- producer ----------------
    int m_k0 = 0, m_k1 = 0, m_rb = 0, m_re = 0;
    int64_t m_i0 = 0, m_i1 = 0;
    auto load_meta = [&](int base) {
      const int itl = base + lane;
      if (itl < nmine) {
        const int b = blockIdx.x + itl * G;
        const int r_lo = row0 + b * R;
        const int r_hi = min(r_lo + R, row0 + nrows);
        m_k0 = __ldg(rp + r_lo);
        m_k1 = __ldg(rp + r_hi);
        m_rb = __ldg(run_begin + b);
        m_re = __ldg(run_begin + b + 1);
        m_i0 = __ldg(idx_off + b);
        m_i1 = __ldg(idx_off + b + 1);
      }
    };
    load_meta(0);
    // runs of the current block: lane q holds run q
    auto load_runs = [&](int it, int& rs, int& rl) {
      const int rb = __shfl_sync(0xffffffffu, m_rb, it & 31);
      const int re = __shfl_sync(0xffffffffu, m_re, it & 31);
      rs = 0;
      rl = 0;
      if (rb + lane < re) {
        rs = __ldg(run_start + rb + lane);
        rl = __ldg(run_len + rb + lane);
      }
    };
    int rs = 0, rl = 0;
    if (nmine > 0) load_runs(0, rs, rl);
    for (int it = 0; it < nmine; ++it) {
      const int s = it % STAGES;
      const int k0 = __shfl_sync(0xffffffffu, m_k0, it & 31);
      const int k1 = __shfl_sync(0xffffffffu, m_k1, it & 31);
      const int64_t i0 = __shfl_sync(0xffffffffu, m_i0, it & 31);
      const int64_t i1 = __shfl_sync(0xffffffffu, m_i1, it & 31);
      // offsets of this block's runs in the stage (exclusive warp scan)
      int off = rl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, off, o);
        if (lane >= o) off += y;
      }
      const int total_rows = __shfl_sync(0xffffffffu, off, 31);
      off -= rl;
      const int my_rs = rs, my_rl = rl;
      // prefetch the next block's metadata / runs while this one is issued
      if (it + 1 < nmine) {
        if (((it + 1) & 31) == 0) load_meta(it + 1);
        load_runs(it + 1, rs, rl);
      }
      mbar_wait(&empty[s], (unsigned)(((it / STAGES) & 1) ^ 1));
      unsigned char* base = smem_raw + (size_t)s * bufbytes;
      T* xs = reinterpret_cast<T*>(base);
      uint16_t* is = reinterpret_cast<uint16_t*>(base + xbytes);
      T* vs = reinterpret_cast<T*>(base + xbytes + ibytes);
      for (int k = k0 + lane; k < k1; k += 32) cp_async_small<sizeof(T)>(vs + (k - k0), av + k);
      cp_async_mbar_arrive(&full[s]);
      __syncwarp();
      if (lane == 0)
        mbar_arrive_expect_tx(&full[s], (unsigned)((size_t)total_rows * cc * sizeof(T) +
                                                   (size_t)(i1 - i0) * 2));
      __syncwarp();
      if (my_rl > 0) {
        const char* src = reinterpret_cast<const char*>(X + (size_t)my_rs * cc);
        char* dst = reinterpret_cast<char*>(xs + (size_t)off * cc);
        size_t left = (size_t)my_rl * cc * sizeof(T);
        while (left) {
          const unsigned chunk = (unsigned)min(left, (size_t)32768);
          bulk_g2s(dst, src, chunk, &full[s]);
          dst += chunk;
          src += chunk;
          left -= chunk;
        }
      }
      if (lane == 0 && i1 > i0) bulk_g2s(is, lidx + i0, (unsigned)((i1 - i0) * 2), &full[s]);
    }
    cp_async_wait<0>();
    return;
  }
  // ---------------- consumers ----------------
  const int gl = threadIdx.x & (LPR - 1);
  const unsigned gmask = group_mask(LPR);
  const int group = threadIdx.x / LPR, ngroups = (NCONS * 32) / LPR;
  __shared__ DiaLines dl_s;
  if constexpr (DIA) {
    if (threadIdx.x == 0) dl_s = *dlp;
    asm volatile("bar.sync 1, 256;\n" ::: "memory");  // consumer warps only
  }
  const DiaLines& dl = dl_s;
  for (int it = 0; it < nmine; ++it) {
    const int b = blockIdx.x + it * G;
    const int s = it % STAGES;
    mbar_wait(&full[s], (unsigned)((it / STAGES) & 1));
    const unsigned char* base = smem_raw + (size_t)s * bufbytes;
    const T* xs = reinterpret_cast<const T*>(base);
    const uint16_t* is = reinterpret_cast<const uint16_t*>(base + xbytes);
    const T* vs = reinterpret_cast<const T*>(base + xbytes + ibytes);
    const int r_lo = row0 + b * R;
    const int nr = min(R, row0 + nrows - r_lo);
    const uint16_t* lrp = is;
    const uint16_t* lsl = is + nr + 1;
    if constexpr (DIA) {
      band_block_dia<T, VEC, NCH, NCONS>(xs, vs, lrp, lsl, cc, nr, dl, warp, gl,
                                         out + (size_t)r_lo * ldo, ldo);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      continue;
    }
    for (int r = group; r < nr; r += ngroups) {

      const int eb = lrp[r], ee = lrp[r + 1];
      T acc[NCH][VEC];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[ch][v] = T(0);
      for (int e0 = eb; e0 < ee; e0 += LPR) {
        const int sl = e0 + gl < ee ? lsl[e0 + gl] : 0;
        const int cnt = min(LPR, ee - e0);
#pragma unroll 4
        for (int u = 0; u < cnt; ++u) {
          const int su = __shfl_sync(gmask, sl, u, LPR);
          const T au = vs[e0 + u];  // broadcast load: 1 wavefront vs 2 for a 64-bit shuffle
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            T x[VEC];
            ldv<T, VEC>(x, xs + (size_t)su * cc + (ch * LPR + gl) * VEC);
#pragma unroll
            for (int v = 0; v < VEC; ++v)
              acc[ch][v] = fops<T>::add(acc[ch][v], fops<T>::mul(au, x[v]));
          }
        }
      }
      T* o = out + (size_t)(r_lo + r) * ldo;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) stv<T, VEC>(o + (ch * LPR + gl) * VEC, acc[ch]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// Generic SpMM (any column count): one warp per row, scalar columns.
template <class T>
__global__ void __launch_bounds__(256)
    k_spmm_rows_generic(int64_t nrows, const int* __restrict__ rows, int row0,
                        const int* __restrict__ rp, const int* __restrict__ ci,
                        const T* __restrict__ av, const T* __restrict__ X,
                        int ldx, int cc, T* __restrict__ out, int ldo) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= nrows) return;
  const int lane = threadIdx.x & 31;
  const int r = rows ? __ldg(rows + g) : row0 + (int)g;
  const int kb = __ldg(rp + r), ke = __ldg(rp + r + 1);
  for (int cb = 0; cb < cc; cb += 32) {
    const int col = cb + lane;
    T acc = T(0);
    for (int k = kb; k < ke; ++k) {
      const int c = __ldg(ci + k);
      const T a = __ldg(av + k);
      if (col < cc) acc = fops<T>::add(acc, fops<T>::mul(a, X[(size_t)c * ldx + col]));
    }
    if (col < cc) out[(size_t)r * ldo + col] = acc;
  }
}

// Long rows: segment partials then an ordered combine.
template <class T>
__global__ void __launch_bounds__(256)
    k_spmm_segments(int64_t nseg, const int* __restrict__ seg_k0,
                    const int* __restrict__ seg_k1, const int* __restrict__ ci,
                    const T* __restrict__ av, const T* __restrict__ X, int ldx,
                    int cc, T* __restrict__ partial) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= nseg) return;
  const int lane = threadIdx.x & 31;
  const int kb = seg_k0[g], ke = seg_k1[g];
  for (int cb = 0; cb < cc; cb += 32) {
    const int col = cb + lane;
    T acc = T(0);
    int k = kb;
    for (; k + 4 <= ke; k += 4) {
      int c[4];
      T a[4], x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        c[q] = __ldg(ci + k + q);
        a[q] = __ldg(av + k + q);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = col < cc ? X[(size_t)c[q] * ldx + col] : T(0);
#pragma unroll
      for (int q = 0; q < 4; ++q) acc = fops<T>::add(acc, fops<T>::mul(a[q], x[q]));
    }
    for (; k < ke; ++k) {
      const int c = __ldg(ci + k);
      const T a = __ldg(av + k);
      if (col < cc) acc = fops<T>::add(acc, fops<T>::mul(a, X[(size_t)c * ldx + col]));
    }
    if (col < cc) partial[(size_t)g * cc + col] = acc;
  }
}

template <class T>
__global__ void __launch_bounds__(256)
    k_segment_combine(int64_t nlong, const int* __restrict__ long_rows,
                      const int64_t* __restrict__ long_seg_off,
                      const T* __restrict__ partial, int cc,
                      T* __restrict__ out, int ldo) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= nlong) return;
  const int lane = threadIdx.x & 31;
  const int r = long_rows[g];
  const int64_t s0 = long_seg_off[g], s1 = long_seg_off[g + 1];
  for (int col = lane; col < cc; col += 32) {
    T acc = partial[(size_t)s0 * cc + col];
    for (int64_t s = s0 + 1; s < s1; ++s)
      acc = fops<T>::add(acc, partial[(size_t)s * cc + col]);
    out[(size_t)r * ldo + col] = acc;
  }
}

// Vectorised long-row segments: LPR lanes per segment (16-byte gathers),
// partial rows to scratch, then an ordered combine per long row.
template <class T, int VEC, int LPR, int NCH, int UNR = 4, int MINB = 1, bool FMA = false>
__global__ void __launch_bounds__(256, MINB)
    k_spmm_segments_vec(int64_t nseg, const int* __restrict__ seg_k0,
                        const int* __restrict__ seg_k1, const int* __restrict__ ci,
                        const T* __restrict__ av, const T* __restrict__ X, int ldx,
                        T* __restrict__ partial) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR;
  if (g >= nseg) return;
  const int gl = threadIdx.x & (LPR - 1);
  const unsigned gmask = group_mask(LPR);
  auto xl = [&](int c, int ch, T(&x)[VEC]) {
    ldv<T, VEC>(x, X + (size_t)c * ldx + (ch * LPR + gl) * VEC);
  };
  T acc[NCH][VEC];
  spmm_row<T, VEC, LPR, NCH, decltype(xl), UNR, FMA>(seg_k0[g], seg_k1[g], ci, av, gl, gmask, xl, acc);
  T* o = partial + (size_t)g * ldx;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) stv<T, VEC>(o + (ch * LPR + gl) * VEC, acc[ch]);
}

template <class T, int VEC, int LPR, int NCH>
__global__ void __launch_bounds__(256)
    k_segment_combine_vec(int64_t nlong, const int* __restrict__ long_rows,
                          const int64_t* __restrict__ long_seg_off,
                          const T* __restrict__ partial, int cc, T* __restrict__ out,
                          int ldo) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR;
  if (g >= nlong) return;
  const int gl = threadIdx.x & (LPR - 1);
  const int r = long_rows[g];
  const int64_t s0 = long_seg_off[g], s1 = long_seg_off[g + 1];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    const int col = (ch * LPR + gl) * VEC;
    T acc[VEC];
    ldv<T, VEC>(acc, partial + (size_t)s0 * cc + col);
    // the longest row has hundreds of segments: 8 independent loads in
    // flight, then the adds in segment order (the same fixed order)
    int64_t sg = s0 + 1;
    for (; sg + 8 <= s1; sg += 8) {
      T x[8][VEC];
#pragma unroll
      for (int u = 0; u < 8; ++u) ldv<T, VEC>(x[u], partial + (size_t)(sg + u) * cc + col);
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = fops<T>::add(acc[v], x[u][v]);
    }
    for (; sg < s1; ++sg) {
      T x[VEC];
      ldv<T, VEC>(x, partial + (size_t)sg * cc + col);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = fops<T>::add(acc[v], x[v]);
    }
    stv<T, VEC>(out + (size_t)r * ldo + col, acc);
  }
}

// ---- dense first op: D1[rows, :] = B[rows, :] C, register tiled ----------
// Per element: acc = fma(B[i,j], C[j,k], acc) for j ascending from 0, the
// same sequence the fused kernel uses, so fused and unfused agree bitwise.
template <class T, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    k_gemm_blocks(int64_t nblk, const int* __restrict__ blk_r0,
                  const int* __restrict__ blk_cnt, const T* __restrict__ B,
                  int bc, const T* __restrict__ C, int cc,
                  T* __restrict__ D1, int ldd) {
  constexpr int NT = (BM / TM) * (BN / TN);
  __shared__ __align__(16) T As[BK][BM];
  __shared__ __align__(16) T Cs[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int n0 = blockIdx.y * BN;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int r0 = blk_r0[blk], cnt = blk_cnt[blk];
    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
    for (int k0 = 0; k0 < bc; k0 += BK) {
      const int kn = min(BK, bc - k0);
      for (int e = tid; e < BM * BK; e += NT) {
        const int m = e / BK, kk = e % BK;
        As[kk][m] = (m < cnt && kk < kn) ? B[(size_t)(r0 + m) * bc + k0 + kk] : T(0);
      }
      for (int e = tid; e < BK * BN; e += NT) {
        const int kk = e / BN, nn = e % BN;
        Cs[kk][nn] = (kk < kn && n0 + nn < cc) ? C[(size_t)(k0 + kk) * cc + n0 + nn] : T(0);
      }
      __syncthreads();
      for (int kk = 0; kk < kn; ++kk) {
        T a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = Cs[kk][tx * TN + j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fops<T>::fma(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int m = ty * TM + i;
      if (m >= cnt) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int col = n0 + tx * TN + j;
        if (col < cc) D1[(size_t)(r0 + m) * ldd + col] = acc[i][j];
      }
    }
  }
}

// ---- dense first op v2: cp.async 3-stage pipeline -------------------------
// CTA tile BM rows x BN columns of D1 = B C, K streamed in BK chunks (both
// the B row block and the C chunk) through a 3-stage cp.async ring; each
// thread owns a TM x TN register tile.  Per element the k loop ascends with
// fused multiply-add from 0 -- the same sequence k_gemm_blocks and the fused
// kernel use, so every path produces identical bits.
template <class T, int BM, int BN, int BK, int TM, int TN, int STAGES>
struct GemmCfg {
  static constexpr int V = 16 / (int)sizeof(T);  // elements per 16 B
  static constexpr int PAD = V;                  // keeps 16 B alignment, shifts banks
  static constexpr int THREADS = (BM / TM) * (BN / TN);
  static constexpr int B_LD = BK + PAD;
  static constexpr int C_LD = BN + PAD;
  static constexpr size_t SMEM =
      (size_t)STAGES * ((size_t)BM * B_LD + (size_t)BK * C_LD) * sizeof(T);
  static_assert(THREADS == 256 || THREADS == 128, "128 or 256 threads per CTA");
  static_assert(BK % V == 0 && TN % V == 0, "vector widths");
};

// Column (inside the BN slice) of a thread's accumulator vector starting at j
// (a multiple of V): the thread's TN / V vectors are BN / TN vectors apart, so
// the 16-byte loads of the C chunk and the D1 stores of the BN / TN threads of
// a row are contiguous (tx * TN + j put them 2 vectors apart: 2-way
// shared-memory bank conflicts on every C load of the fp64 tile).
template <int BN, int TN, int V>
__device__ __forceinline__ int gemm_col(int tx, int j) {
  return (j / V) * (BN / TN) * V + tx * V;
}

// acc[TM][TN] += B[r0 .. r0+cnt) x C[:, n0 .. n0+BN) ; rows >= cnt read zeros.
template <class T, int BM, int BN, int BK, int TM, int TN, int STAGES>
__device__ __forceinline__ void gemm_block(const T* __restrict__ B, int bc,
                                           const T* __restrict__ C, int cc, int n0,
                                           int r0, int cnt, T* smem, T (&acc)[TM][TN]) {
  using G = GemmCfg<T, BM, BN, BK, TM, TN, STAGES>;
  constexpr int V = G::V;
  T* sb = smem;                                        // [STAGES][BM][B_LD]
  T* sc = smem + (size_t)STAGES * BM * G::B_LD;        // [STAGES][BK][C_LD]
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int nk = (bc + BK - 1) / BK;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  auto load_stage = [&](int stg, int kc) {
    const int k0 = kc * BK;
    T* bdst = sb + (size_t)stg * BM * G::B_LD;
    for (int e = tid; e < BM * (BK / V); e += G::THREADS) {
      const int m = e / (BK / V), kv = (e % (BK / V)) * V;
      const bool ok = m < cnt && k0 + kv < bc;
      const T* src = ok ? B + (size_t)(r0 + m) * bc + k0 + kv : B;
      cp_async16(bdst + m * G::B_LD + kv, src, ok ? 16 : 0);
    }
    T* cdst = sc + (size_t)stg * BK * G::C_LD;
    for (int e = tid; e < BK * (BN / V); e += G::THREADS) {
      const int kk = e / (BN / V), nv = (e % (BN / V)) * V;
      const bool ok = k0 + kk < bc;
      const T* src = ok ? C + (size_t)(k0 + kk) * cc + n0 + nv : C;
      cp_async16(cdst + kk * G::C_LD + nv, src, ok ? 16 : 0);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kc + STAGES - 1;
      if (nxt < nk) load_stage(nxt % STAGES, nxt);
      cp_async_commit();
    }
    const int stg = kc % STAGES;
    const T* bs = sb + (size_t)stg * BM * G::B_LD;
    const T* cs = sc + (size_t)stg * BK * G::C_LD;
    const int kn = min(BK, bc - kc * BK);
    for (int k0 = 0; k0 < kn; k0 += V) {
      T a[TM][V];
#pragma unroll
      for (int i = 0; i < TM; ++i) ldv<T, V>(a[i], bs + (ty * TM + i) * G::B_LD + k0);
      const int kv = min(V, kn - k0);
#pragma unroll
      for (int kk = 0; kk < V; ++kk) {
        if (kk < kv) {
          T b[TN];
#pragma unroll
          for (int j = 0; j < TN; j += V) {
            T tmp[V];
            ldv<T, V>(tmp, cs + (k0 + kk) * G::C_LD + gemm_col<BN, TN, V>(tx, j));
#pragma unroll
            for (int q = 0; q < V; ++q) b[j + q] = tmp[q];
          }
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = fops<T>::fma(a[i][kk], b[j], acc[i][j]);
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Pipeline pieces shared by the streamed GEMM kernels: one K-chunk load of
// (B row block, C chunk) into ring stage `stg`, and one chunk of FMAs.
template <class T, int BM, int BN, int BK, int TM, int TN, int STAGES>
__device__ __forceinline__ void gemm_load_chunk(const T* __restrict__ B, int bc,
                                                const T* __restrict__ C, int cc, int n0,
                                                int r0, int cnt, int kc, int stg, T* smem) {
  using G = GemmCfg<T, BM, BN, BK, TM, TN, STAGES>;
  constexpr int V = G::V;
  T* bdst = smem + (size_t)stg * BM * G::B_LD;
  T* cdst = smem + (size_t)STAGES * BM * G::B_LD + (size_t)stg * BK * G::C_LD;
  const int k0 = kc * BK;
  for (int e = threadIdx.x; e < BM * (BK / V); e += G::THREADS) {
    const int m = e / (BK / V), kv = (e % (BK / V)) * V;
    const bool ok = m < cnt && k0 + kv < bc;
    cp_async16(bdst + m * G::B_LD + kv, ok ? B + (size_t)(r0 + m) * bc + k0 + kv : B, ok ? 16 : 0);
  }
  for (int e = threadIdx.x; e < BK * (BN / V); e += G::THREADS) {
    const int kk = e / (BN / V), nv = (e % (BN / V)) * V;
    const bool ok = k0 + kk < bc;
    cp_async16(cdst + kk * G::C_LD + nv, ok ? C + (size_t)(k0 + kk) * cc + n0 + nv : C, ok ? 16 : 0);
  }
}

template <class T, int BM, int BN, int BK, int TM, int TN, int STAGES>
__device__ __forceinline__ void gemm_compute_chunk(int bc, int kc, int stg, const T* smem,
                                                   T (&acc)[TM][TN]) {
  using G = GemmCfg<T, BM, BN, BK, TM, TN, STAGES>;
  constexpr int V = G::V;
  const int tx = threadIdx.x % (BN / TN), ty = threadIdx.x / (BN / TN);
  const T* bs = smem + (size_t)stg * BM * G::B_LD;
  const T* cs = smem + (size_t)STAGES * BM * G::B_LD + (size_t)stg * BK * G::C_LD;
  const int kn = min(BK, bc - kc * BK);
  if (kn == BK) {  // full chunk: compile-time trip counts, fully unrolled
#pragma unroll
    for (int k0 = 0; k0 < BK; k0 += V) {
      T a[TM][V];
#pragma unroll
      for (int i = 0; i < TM; ++i) ldv<T, V>(a[i], bs + (ty * TM + i) * G::B_LD + k0);
#pragma unroll
      for (int kk = 0; kk < V; ++kk) {
        T b[TN];
#pragma unroll
        for (int j = 0; j < TN; j += V) {
          T tmp[V];
          ldv<T, V>(tmp, cs + (k0 + kk) * G::C_LD + gemm_col<BN, TN, V>(tx, j));
#pragma unroll
          for (int q = 0; q < V; ++q) b[j + q] = tmp[q];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fops<T>::fma(a[i][kk], b[j], acc[i][j]);
      }
    }
    return;
  }
  for (int k0 = 0; k0 < kn; k0 += V) {
    T a[TM][V];
#pragma unroll
    for (int i = 0; i < TM; ++i) ldv<T, V>(a[i], bs + (ty * TM + i) * G::B_LD + k0);
    const int kv = min(V, kn - k0);
#pragma unroll
    for (int kk = 0; kk < V; ++kk) {
      if (kk < kv) {
        T b[TN];
#pragma unroll
        for (int j = 0; j < TN; j += V) {
          T tmp[V];
          ldv<T, V>(tmp, cs + (k0 + kk) * G::C_LD + gemm_col<BN, TN, V>(tx, j));
#pragma unroll
          for (int q = 0; q < V; ++q) b[j + q] = tmp[q];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fops<T>::fma(a[i][kk], b[j], acc[i][j]);
      }
    }
  }
}

// Streamed GEMM: the CTA's row blocks blk = blockIdx.x + j*gridDim.x are
// flattened with their K chunks into one cp.async ring, so loads of the next
// block overlap the current block's FMAs and epilogue.
template <class T, int BM, int BN, int BK, int TM, int TN, int STAGES>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    k_gemm_stream(int64_t nblk, const int* __restrict__ blk_r0, const int* __restrict__ blk_cnt,
                  const T* __restrict__ B, int bc, const T* __restrict__ C, int cc,
                  T* __restrict__ D1, int ldd) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  constexpr int V = 16 / (int)sizeof(T);
  const int n0 = blockIdx.y * BN;
  const int tx = threadIdx.x % (BN / TN), ty = threadIdx.x / (BN / TN);
  const int nk = (bc + BK - 1) / BK;
  const int64_t nmine = blockIdx.x < nblk ? (nblk - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = nmine * nk;
  auto load = [&](int64_t t) {
    const int64_t blk = blockIdx.x + (t / nk) * gridDim.x;
    gemm_load_chunk<T, BM, BN, BK, TM, TN, STAGES>(B, bc, C, cc, n0, blk_r0[blk], blk_cnt[blk],
                                                   (int)(t % nk), (int)(t % STAGES), smem);
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < total) load(s);
    cp_async_commit();
  }
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
  for (int64_t t = 0; t < total; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (t + STAGES - 1 < total) load(t + STAGES - 1);
    cp_async_commit();
    const int kc = (int)(t % nk);
    gemm_compute_chunk<T, BM, BN, BK, TM, TN, STAGES>(bc, kc, (int)(t % STAGES), smem, acc);
    if (kc == nk - 1) {
      const int64_t blk = blockIdx.x + (t / nk) * gridDim.x;
      const int r0 = blk_r0[blk], cnt = blk_cnt[blk];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int m = ty * TM + i;
        if (m < cnt) {
          T* o = D1 + (size_t)(r0 + m) * ldd + n0;
#pragma unroll
          for (int j = 0; j < TN; j += V) {
            T tmp[V];
#pragma unroll
            for (int q = 0; q < V; ++q) tmp[q] = acc[i][j + q];
            stv<T, V>(o + gemm_col<BN, TN, V>(tx, j), tmp);
          }
        }
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
      }
    }
  }
  cp_async_wait<0>();
}

template <class T, int BM, int BN, int BK, int TM, int TN, int STAGES>
__global__ void __launch_bounds__(256)
    k_gemm_v2(int64_t nblk, const int* __restrict__ blk_r0, const int* __restrict__ blk_cnt,
              const T* __restrict__ B, int bc, const T* __restrict__ C, int cc,
              T* __restrict__ D1, int ldd) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const int n0 = blockIdx.y * BN;
  const int tx = threadIdx.x % (BN / TN), ty = threadIdx.x / (BN / TN);
  constexpr int V = 16 / (int)sizeof(T);
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int r0 = blk_r0[blk], cnt = blk_cnt[blk];
    T acc[TM][TN];
    gemm_block<T, BM, BN, BK, TM, TN, STAGES>(B, bc, C, cc, n0, r0, cnt, smem, acc);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int m = ty * TM + i;
      if (m < cnt) {
        T* o = D1 + (size_t)(r0 + m) * ldd + n0;
#pragma unroll
        for (int j = 0; j < TN; j += V) {
          T tmp[V];
#pragma unroll
          for (int q = 0; q < V; ++q) tmp[q] = acc[i][j + q];
          stv<T, V>(o + gemm_col<BN, TN, V>(tx, j), tmp);
        }
      }
    }
  }
}

// ---- fused wavefront-0 kernel ----------------------------------------------
// blockIdx.x = fused tile, blockIdx.y = column slice [c0, c0+cs).
// smem: [stage: w_cap x cs][C slice: bc x cs (dense B only)]
template <class T>
__global__ void __launch_bounds__(256)
    k_fused_tiles(int64_t ntiles, const int* __restrict__ t_ilo,
                  const int* __restrict__ t_ihi,
                  const int64_t* __restrict__ t_joff,
                  const int* __restrict__ jrows, int w_cap, int cs, int cc,
                  int b_dense, const T* __restrict__ Bd, int bc,
                  const int* __restrict__ brp, const int* __restrict__ bci,
                  const T* __restrict__ bv, const T* __restrict__ C,
                  const int* __restrict__ arp, const int* __restrict__ aci,
                  const T* __restrict__ av, const uint8_t* __restrict__ spill,
                  T* D1, T* __restrict__ D) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* stage = reinterpret_cast<T*>(smem_raw);
  T* Cs = stage + (size_t)w_cap * cs;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int c0 = blockIdx.y * cs;
  const int csn = min(cs, cc - c0);  // columns in this slice
  constexpr int MAXQ = 4;            // cs <= 128
  if (b_dense) {
    for (int e = threadIdx.x; e < bc * cs; e += blockDim.x) {
      const int j = e / cs, col = e % cs;
      Cs[e] = col < csn ? C[(size_t)j * cc + c0 + col] : T(0);
    }
    __syncthreads();
  }
  for (int64_t v = blockIdx.x; v < ntiles; v += gridDim.x) {
    const int ilo = t_ilo[v], ihi = t_ihi[v];
    const bool in_smem = (ihi - ilo) <= w_cap;
    // phase 1: D1 slice of rows [ilo, ihi)
    for (int i = ilo + warp; i < ihi; i += nwarps) {
      T acc[MAXQ];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) acc[q] = T(0);
      if (b_dense) {
        const T* brow = Bd + (size_t)i * bc;
        for (int j0 = 0; j0 < bc; j0 += 32) {
          const T bvv = j0 + lane < bc ? brow[j0 + lane] : T(0);
          const int cnt = min(32, bc - j0);
          for (int u = 0; u < cnt; ++u) {
            const T b = __shfl_sync(0xffffffffu, bvv, u);
            const T* crow = Cs + (size_t)(j0 + u) * cs;
#pragma unroll
            for (int q = 0; q < MAXQ; ++q) {
              const int col = lane + 32 * q;
              if (col < csn) acc[q] = fops<T>::fma(b, crow[col], acc[q]);
            }
          }
        }
      } else {
        const int kb = brp[i], ke = brp[i + 1];
        for (int k = kb; k < ke; ++k) {
          const int c = __ldg(bci + k);
          const T a = __ldg(bv + k);
          const T* xrow = C + (size_t)c * cc + c0;
#pragma unroll
          for (int q = 0; q < MAXQ; ++q) {
            const int col = lane + 32 * q;
            if (col < csn) acc[q] = fops<T>::add(acc[q], fops<T>::mul(a, xrow[col]));
          }
        }
      }
      const bool sp = spill[i] != 0;
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int col = lane + 32 * q;
        if (col < csn) {
          if (in_smem) stage[(size_t)(i - ilo) * cs + col] = acc[q];
          if (sp || !in_smem) D1[(size_t)i * cc + c0 + col] = acc[q];
        }
      }
    }
    __syncthreads();
    // phase 2: fused D rows from the staged slice
    const int64_t jb = t_joff[v], je = t_joff[v + 1];
    for (int64_t q0 = jb + warp; q0 < je; q0 += nwarps) {
      const int j = jrows[q0];
      const int kb = __ldg(arp + j), ke = __ldg(arp + j + 1);
      T acc[MAXQ];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) acc[q] = T(0);
      for (int k = kb; k < ke; ++k) {
        const int c = __ldg(aci + k);
        const T a = __ldg(av + k);
        const T* xrow = in_smem ? stage + (size_t)(c - ilo) * cs
                                : D1 + (size_t)c * cc + c0;
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int col = lane + 32 * q;
          if (col < csn) acc[q] = fops<T>::add(acc[q], fops<T>::mul(a, xrow[col]));
        }
      }
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int col = lane + 32 * q;
        if (col < csn) D[(size_t)j * cc + c0 + col] = acc[q];
      }
    }
    __syncthreads();
  }
}

// ---- fused wavefront-0 kernel v2 (dense B) ----------------------------------
// Persistent CTAs over fused tiles; blockIdx.y = column slice of width BN.
// Phase 1 runs the pipelined GEMM over the tile's i-range in BM-row blocks;
// the epilogue writes D1 rows that wavefront 1 reads (spill) to HBM and the
// rows the tile's own fused rows read (slot >= 0) to a shared-memory stage.
// Phase 2 computes the tile's fused D rows from the stage (LPR lanes per row,
// reference order).  Tiles whose staged set exceeds the stage capacity were
// marked "wide" at plan time: all their rows spill and phase 2 reads HBM/L2.
template <class T, int BM, int BN, int BK, int TM, int TN, int LPR>
__global__ void __launch_bounds__(256)
    k_fused_gemm_tiles(int64_t ntiles, const int* __restrict__ t_ilo,
                       const int* __restrict__ t_ihi, const int64_t* __restrict__ t_joff,
                       const int* __restrict__ jrows, const uint8_t* __restrict__ t_wide,
                       const int* __restrict__ slot, const T* __restrict__ B, int bc,
                       const T* __restrict__ C, int cc, const int* __restrict__ arp,
                       const int* __restrict__ aci, const T* __restrict__ av,
                       const uint8_t* __restrict__ spill, T* D1, T* __restrict__ D) {
  constexpr int STAGES = 3;
  using G = GemmCfg<T, BM, BN, BK, TM, TN, STAGES>;
  constexpr int V = G::V;
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int NCH = BN / (LPR * VEC);
  static_assert(NCH >= 1 && NCH * LPR * VEC == BN, "slice width");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* gsm = reinterpret_cast<T*>(smem_raw);
  T* stage = gsm + G::SMEM / sizeof(T);
  const int n0 = blockIdx.y * BN;
  const int tx = threadIdx.x % (BN / TN), ty = threadIdx.x / (BN / TN);
  const int gl = threadIdx.x & (LPR - 1);
  const unsigned gmask = group_mask(LPR);
  const int group = threadIdx.x / LPR, ngroups = blockDim.x / LPR;
  const int nk = (bc + BK - 1) / BK;

  // cursor over this CTA's (tile, row block, k chunk) sequence
  struct Cur {
    int64_t v;
    int r0, ihi, kc;
  };
  auto start = [&](Cur& c) {
    c.v = blockIdx.x;
    c.kc = 0;
    if (c.v < ntiles) {
      c.r0 = t_ilo[c.v];
      c.ihi = t_ihi[c.v];
    }
  };
  auto next = [&](Cur& c) {
    if (++c.kc < nk) return;
    c.kc = 0;
    c.r0 += BM;
    if (c.r0 >= c.ihi) {
      c.v += gridDim.x;
      if (c.v < ntiles) {
        c.r0 = t_ilo[c.v];
        c.ihi = t_ihi[c.v];
      }
    }
  };
  Cur lc, cu;
  start(lc);
  start(cu);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (lc.v < ntiles) {
      gemm_load_chunk<T, BM, BN, BK, TM, TN, STAGES>(B, bc, C, cc, n0, lc.r0,
                                                     min(BM, lc.ihi - lc.r0), lc.kc, s, gsm);
      next(lc);
    }
    cp_async_commit();
  }
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
  for (int64_t t = 0; cu.v < ntiles; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (lc.v < ntiles) {
      gemm_load_chunk<T, BM, BN, BK, TM, TN, STAGES>(B, bc, C, cc, n0, lc.r0,
                                                     min(BM, lc.ihi - lc.r0), lc.kc,
                                                     (int)((t + STAGES - 1) % STAGES), gsm);
      next(lc);
    }
    cp_async_commit();
    gemm_compute_chunk<T, BM, BN, BK, TM, TN, STAGES>(bc, cu.kc, (int)(t % STAGES), gsm, acc);
    if (cu.kc == nk - 1) {
      const int64_t v = cu.v;
      const int r0 = cu.r0, cnt = min(BM, cu.ihi - cu.r0);
      const bool wide = t_wide[v] != 0;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int m = ty * TM + i;
        if (m < cnt) {
          const int row = r0 + m;
          const int sl = wide ? -1 : __ldg(slot + row);
          const bool sp = wide || spill[row];
#pragma unroll
          for (int j = 0; j < TN; j += V) {
            T tmp[V];
#pragma unroll
            for (int q = 0; q < V; ++q) tmp[q] = acc[i][j + q];
            const int col = gemm_col<BN, TN, V>(tx, j);
            if (sp) stv<T, V>(D1 + (size_t)row * cc + n0 + col, tmp);
            if (sl >= 0) stv<T, V>(stage + (size_t)sl * BN + col, tmp);
          }
        }
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
      }
      if (r0 + BM >= cu.ihi) {  // last block of the tile: fused rows from the stage
        __syncthreads();
        const int64_t jb = t_joff[v], je = t_joff[v + 1];
        for (int64_t q = jb + group; q < je; q += ngroups) {
          const int j = jrows[q];
          const int kb = __ldg(arp + j), ke = __ldg(arp + j + 1);
          T acc2[NCH][VEC];
          if (wide) {
            auto xl = [&](int c, int ch, T(&x)[VEC]) {
              ldv<T, VEC>(x, D1 + (size_t)c * cc + n0 + (ch * LPR + gl) * VEC);
            };
            spmm_row<T, VEC, LPR, NCH>(kb, ke, aci, av, gl, gmask, xl, acc2);
          } else {
            auto xl = [&](int c, int ch, T(&x)[VEC]) {
              ldv<T, VEC>(x, stage + (size_t)__ldg(slot + c) * BN + (ch * LPR + gl) * VEC);
            };
            spmm_row<T, VEC, LPR, NCH>(kb, ke, aci, av, gl, gmask, xl, acc2);
          }
          T* o = D + (size_t)j * cc + n0;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) stv<T, VEC>(o + (ch * LPR + gl) * VEC, acc2[ch]);
        }
        __syncthreads();
      }
    }
    next(cu);
  }
  cp_async_wait<0>();
}

// Fused-row index stream of the tensor-core tiles: per nonzero, the stage
// slot of its column (staged tile) or the column itself (wide tile).
__global__ void k_fused_xidx(int64_t nrows, const int* __restrict__ jrows,
                             const int64_t* __restrict__ off, const uint8_t* __restrict__ rwide,
                             const int* __restrict__ arp, const int* __restrict__ aci,
                             const int* __restrict__ slot, int* __restrict__ xidx) {
  const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (q >= nrows) return;
  const int lane = threadIdx.x & 31;
  const int j = jrows[q];
  const int kb = arp[j], ke = arp[j + 1];
  const bool w = rwide[q] != 0;
  int* o = xidx + off[q] - kb;
  for (int k = kb + lane; k < ke; k += 32) {
    const int c = aci[k];
    o[k] = w ? c : slot[c];
  }
}

// slot[i] = position of D1 row i in its tile's stage (-1: not read by the
// tile's fused rows).  One warp per fused tile, rows ascending.
__global__ void k_assign_slots(int64_t ntiles, const int* __restrict__ t_ilo,
                               const int* __restrict__ t_ihi, const uint8_t* __restrict__ mark,
                               int* slot, int* t_count) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= ntiles) return;
  const int lane = threadIdx.x & 31;
  const int ilo = t_ilo[w], ihi = t_ihi[w];
  int base = 0;
  for (int i0 = ilo; i0 < ihi; i0 += 32) {
    const int i = i0 + lane;
    const bool m = i < ihi && mark[i];
    const unsigned bal = __ballot_sync(0xffffffffu, m);
    if (i < ihi) slot[i] = m ? base + __popc(bal & ((1u << lane) - 1u)) : -1;
    base += __popc(bal);
  }
  if (lane == 0) t_count[w] = base;
}

// spill[c] = 1 for every column c of every wavefront-1 row
__global__ void k_mark_spill(int64_t nrows, const int* __restrict__ rows,
                             const int* __restrict__ rp,
                             const int* __restrict__ ci, uint8_t* spill) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= nrows) return;
  const int lane = threadIdx.x & 31;
  const int r = rows[g];
  for (int k = rp[r] + lane; k < rp[r + 1]; k += 32) spill[ci[k]] = 1;
}

// mark[c] = 1 for every column of the listed rows (distinct-row accounting)
__global__ void k_mark_cols(int64_t nrows, const int* __restrict__ rows,
                            const int* __restrict__ rp, const int* __restrict__ ci,
                            uint8_t* mark) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= nrows) return;
  const int lane = threadIdx.x & 31;
  const int r = rows[g];
  for (int k = rp[r] + lane; k < rp[r + 1]; k += 32) mark[ci[k]] = 1;
}

__global__ void k_count_u8(int64_t n, const uint8_t* f, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += f[i];
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}

template <class T>
__global__ void k_gather_rows(const T* __restrict__ src, int cols,
                              const int* __restrict__ rows, int64_t n,
                              T* __restrict__ dst) {
  const int64_t total = n * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols;
    const int c = (int)(e % cols);
    dst[e] = src[(size_t)rows[r] * cols + c];
  }
}
// Multi-GPU halo: bit q of mask[c] is set when a wavefront-1 row owned by
// rank q (row block [bounds[q], bounds[q+1])) reads column c.
__global__ void k_mark_readers(int64_t nrows, const int* __restrict__ rows,
                               const int* __restrict__ rp, const int* __restrict__ ci,
                               const int* __restrict__ bounds, int world,
                               unsigned* __restrict__ mask) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  const int j = rows[w];
  int q = 0;
  while (q + 1 < world && j >= bounds[q + 1]) ++q;
  for (int k = rp[j] + lane; k < rp[j + 1]; k += 32) atomicOr(mask + ci[k], 1u << q);
}

// flag[i] = 1 when row rows[i] reads a column outside [lo, hi)
__global__ void k_reads_remote(int64_t nrows, const int* __restrict__ rows,
                               const int* __restrict__ rp, const int* __restrict__ ci, int lo,
                               int hi, uint8_t* __restrict__ flag) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  const int j = rows[w];
  bool remote = false;
  for (int k = rp[j] + lane; k < rp[j + 1] && !remote; k += 32) remote = ci[k] < lo || ci[k] >= hi;
  remote = __any_sync(0xffffffffu, remote);
  if (lane == 0) flag[w] = remote;
}

// D[rows[i], :] = 0 (empty rows of a row list), 16-byte stores
__global__ void k_zero_rows(int64_t nrows, const int* __restrict__ rows, int row_bytes,
                            unsigned char* __restrict__ out) {
  const int per = row_bytes / 16;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nrows * per) return;
  const int64_t i = t / per;
  const int q = (int)(t - i * per);
  reinterpret_cast<uint4*>(out + (size_t)rows[i] * row_bytes)[q] = make_uint4(0, 0, 0, 0);
}

template <class T>
__global__ void k_scatter_rows(const T* __restrict__ src, int cols,
                               const int* __restrict__ rows, int64_t n,
                               T* __restrict__ dst) {
  const int64_t total = n * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols;
    const int c = (int)(e % cols);
    dst[(size_t)rows[r] * cols + c] = src[e];
  }
}

inline int blocks_for(int64_t threads, int per_block = 256) {
  int64_t b = (threads + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, b);
}

}  // namespace

// ===========================================================================
// Row-SpMM work list: short rows (one group per row) + segmented long rows.
// ===========================================================================
struct SpmmWork {
  int64_t n_short = 0, n_long = 0, n_seg = 0;
  size_t elem_ = 8;
  // side stream for the long rows (runs beside the short-row kernel)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  SpmmWork() = default;
  SpmmWork(const SpmmWork&) = delete;
  SpmmWork& operator=(const SpmmWork&) = delete;
  ~SpmmWork() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
  }
  // reference-bits mode: grid-stencil rows with separately rounded mul and
  // add (bit-identical to spmm_row); default one FMA per term (tfg.h)
  bool exact = false;
  bool skewed = false;  // row lengths vary a lot: one row per lane group
  // band-staged layout (k_spmm_band3)
  bool banded = false;
  int band_R = 0, band_blocks = 0, stage_cap = 0, idx_cap = 0, val_cap = 0;
  size_t band_smem = 0;
  dbuf<int> run_begin, run_start, run_len;
  dbuf<int64_t> idx_off;
  dbuf<uint16_t> lidx;
  std::vector<int> blk_xlo, blk_xhi;  // per band block: X rows read [lo, hi] (hi < lo: none)
  // stencil (diagonal) structure: every row of a "regular" 4-row mini-group
  // has exactly the global diagonal set; diagonals form lines of <= 5
  // consecutive offsets (k_spmm_band3 DIA consumer)
  bool dia = false;
  DiaLines dia_lines{};
  dbuf<DiaLines> dia_dev;

  // Blocks of R consecutive rows whose X rows form <= kBandRuns contiguous
  // runs; adopted only when it at least halves the X rows gathered.
  void build_band(int row0, int64_t nrows, const std::vector<int>& rp,
                  const std::vector<int>& ci, int cc, size_t elem, cudaStream_t st) {
    detect_dia(row0, nrows, rp, ci, cc, elem);
    // smallest stage budget that admits a band layout (more CTAs per SM); the
    // stencil consumer wants >= 8 mini-groups (R >= 32) per block
    for (int kb : {40, 64, 100}) {
      if (dia && kb == 40 && (size_t)cc * elem == 512) continue;
      build_band_budget(row0, nrows, rp, ci, cc, elem, st, (size_t)kb * 1024);
      if (banded) return;
    }
  }

  std::vector<int> dia_offs;  // the global diagonal offsets (col - row), ascending

  void detect_dia(int row0, int64_t nrows, const std::vector<int>& rp, const std::vector<int>& ci,
                  int cc, size_t elem) {
    dia = false;
    dia_offs.clear();
    if ((size_t)cc * elem != 512 && (size_t)cc * elem != 1024) return;
    std::vector<int> offs;
    for (int64_t r = row0; r < row0 + nrows; ++r)
      for (int k = rp[r]; k < rp[r + 1]; ++k) {
        const int o = ci[k] - (int)r;
        if (std::find(offs.begin(), offs.end(), o) == offs.end()) {
          offs.push_back(o);
          if (offs.size() > 32) return;
        }
      }
    std::sort(offs.begin(), offs.end());
    DiaLines L{};
    L.ndiag = (int)offs.size();
    for (int d = 0; d < (int)offs.size();) {
      int e = d + 1;
      while (e < (int)offs.size() && offs[e] == offs[e - 1] + 1 && e - d < 5) ++e;
      if (L.nlines == 16) return;
      L.first[L.nlines] = d;
      L.cnt[L.nlines] = e - d;
      ++L.nlines;
      d = e;
    }
    dia_offs = offs;
    dia_lines = L;
    dia = true;
  }

  // mini-group g (rows 4g..4g+3 of the block) is regular: all four rows exist
  // and each has exactly the global diagonal set
  bool dia_regular(int r_lo, int nr, int g, const std::vector<int>& rp,
                   const std::vector<int>& ci) const {
    if (4 * g + 3 >= nr) return false;
    for (int q = 0; q < 4; ++q) {
      const int r = r_lo + 4 * g + q;
      if (rp[r + 1] - rp[r] != (int)dia_offs.size()) return false;
      for (int d = 0; d < (int)dia_offs.size(); ++d)
        if (ci[rp[r] + d] - r != dia_offs[d]) return false;
    }
    return true;
  }

  void build_band_budget(int row0, int64_t nrows, const std::vector<int>& rp,
                         const std::vector<int>& ci, int cc, size_t elem, cudaStream_t st,
                         size_t budget) {
    const size_t row_bytes = (size_t)cc * elem;
    int64_t nnz_total = (int64_t)rp[row0 + nrows] - rp[row0];
    if (nnz_total <= 0) return;
    for (int R : {256, 128, 64, 32, 16, 8, 4}) {
      const int nb = (int)((nrows + R - 1) / R);
      std::vector<int> rb{0}, rs, rl, li, bxlo, bxhi;
      std::vector<int64_t> io{0};
      int64_t staged_total = 0;
      int scap = 0, icap = 0, vcap = 0;
      bool ok = true;
      std::vector<int> cols;
      for (int b = 0; b < nb && ok; ++b) {
        const int r_lo = row0 + b * R;
        const int r_hi = (int)std::min<int64_t>(r_lo + R, row0 + nrows);
        const int k0 = rp[r_lo], k1 = rp[r_hi];
        cols.assign(ci.begin() + k0, ci.begin() + k1);
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        // runs, merging gaps of up to 2 rows
        std::vector<std::pair<int, int>> runs;
        for (int c : cols) {
          if (!runs.empty() && c <= runs.back().first + runs.back().second + 2)
            runs.back().second = c - runs.back().first + 1;
          else
            runs.emplace_back(c, 1);
        }
        int staged = 0;
        for (auto& r : runs) staged += r.second;
        const int nr = r_hi - r_lo;
        // slots of every entry (runs are in ascending column order, so slot
        // order == column order)
        std::vector<int> run_off;
        {
          int off = 0;
          for (auto& r : runs) {
            run_off.push_back(off);
            off += r.second;
          }
        }
        std::vector<int> slots(k1 - k0);
        for (int k = k0; k < k1; ++k) {
          const int c = ci[k];
          size_t q = std::upper_bound(runs.begin(), runs.end(), std::make_pair(c, INT32_MAX)) -
                     runs.begin() - 1;
          slots[k - k0] = run_off[q] + (c - runs[q].first);
        }
        const bool rec_dia = dia && R <= 128 && R >= 32;
        const int irec = ((nr + 1 + (k1 - k0) + (rec_dia ? 2 : 0)) + 7) / 8 * 8;
        const size_t need = (size_t)staged * row_bytes + (size_t)irec * 2 +
                            ((size_t)(k1 - k0) * elem + 15) / 16 * 16;
        if ((int)runs.size() > kBandRuns || staged > 65535 || need > budget) {
          ok = false;
          break;
        }
        scap = std::max(scap, staged);
        icap = std::max(icap, irec);
        vcap = std::max(vcap, k1 - k0);
        staged_total += staged;
        for (auto& r : runs) {
          rs.push_back(r.first);
          rl.push_back(r.second);
        }
        bxlo.push_back(runs.empty() ? 1 : runs.front().first);
        bxhi.push_back(runs.empty() ? 0 : runs.back().first + runs.back().second - 1);
        rb.push_back((int)rs.size());
        // index record: row offsets, slots, [mini-group offsets, union entries]
        const size_t rec0 = li.size();
        for (int r = r_lo; r <= r_hi; ++r) li.push_back(rp[r] - k0);
        for (int v : slots) li.push_back(v);
        if (rec_dia) {
          uint32_t mask = 0;
          for (int g = 0; g < (nr + 3) / 4; ++g)
            if (dia_regular(r_lo, nr, g, rp, ci)) mask |= 1u << g;
          li.push_back((int)(mask & 0xffffu));
          li.push_back((int)(mask >> 16));
        }
        while ((li.size() - rec0) % 8) li.push_back(0);
        io.push_back((int64_t)li.size());
      }
      if (!ok) continue;
      {
        const size_t buf = (size_t)scap * row_bytes + ((size_t)icap * 2 + 15) / 16 * 16 +
                           ((size_t)vcap * elem + 15) / 16 * 16;
        if (2 * buf > kBandSmemMax) continue;  // two stages must fit one CTA
      }
      if ((double)staged_total > 0.5 * (double)nnz_total) return;  // not worth it
      banded = true;
      band_R = R;
      band_blocks = nb;
      // the stencil consumer needs >= 8 mini-groups per block (one per warp)
      if (!(dia && R <= 128 && R >= 32)) dia = false;
      if (dia) {
        dia_dev.alloc(1);
        h2d(dia_dev.p, &dia_lines, 1, st);
      }
      blk_xlo.swap(bxlo);
      blk_xhi.swap(bxhi);
      stage_cap = scap;
      idx_cap = icap;
      val_cap = vcap;
      std::vector<uint16_t> l16(li.begin(), li.end());
      run_begin.alloc(rb.size());
      h2d(run_begin.p, rb.data(), rb.size(), st);
      run_start.alloc(rs.size() + 1);
      h2d(run_start.p, rs.data(), rs.size(), st);
      run_len.alloc(rl.size() + 1);
      h2d(run_len.p, rl.data(), rl.size(), st);
      idx_off.alloc(io.size());
      h2d(idx_off.p, io.data(), io.size(), st);
      lidx.alloc(l16.size() + 8);
      h2d(lidx.p, l16.data(), l16.size(), st);
      const size_t buf = (size_t)scap * row_bytes + ((size_t)icap * 2 + 15) / 16 * 16 +
                         ((size_t)vcap * elem + 15) / 16 * 16;
      band_smem = 2 * buf;
      TFG_CUDA(cudaStreamSynchronize(st));
      return;
    }
  }
  // grid stencil: the plane-streaming kernel replaces everything above
  // (tfg_stencil.cu); set by the plan when every row is in the list
  std::unique_ptr<StencilPlan> stencil;
  bool identity = false;  // short rows are exactly [row0, row0 + n_short)
  int row0 = 0;
  dbuf<int> short_rows, long_rows, seg_k0, seg_k1;
  // empty rows of a non-stencil list: D rows zero-filled by one streaming
  // kernel instead of costing a lane group's row iteration each
  int64_t n_empty = 0;
  dbuf<int> empty_rows;
  dbuf<int64_t> long_seg_off;
  dbuf<unsigned char> partial;

  void build(const std::vector<int>& rows, const std::vector<int>& rp, int cc,
             size_t elem, cudaStream_t st, const std::vector<int>* ci = nullptr,
             bool stencil_rows = false) {  // stencil_rows: the stencil kernel takes them
    std::vector<int> sh, lg, k0, k1;
    std::vector<int64_t> off{0};
    sh.reserve(rows.size());
    // Power-law rows: one lane group would walk a row of thousands of
    // nonzeros alone while the rest of the GPU idles, so skewed lists split
    // every row longer than ~8x the mean into segments of that length.
    int long_thr = kLongRow, seg_len = kSegLen;
    if (!rows.empty()) {
      int64_t tot = 0;
      int mx = 0;
      for (int r : rows) {
        tot += rp[r + 1] - rp[r];
        mx = std::max(mx, rp[r + 1] - rp[r]);
      }
      const double mean = (double)tot / (double)rows.size();
      // 16 x the mean (8: cfg5 wavefront 1 6.09 ms, 16: 5.93, cfg3 equal)
      const int thr = std::max(256, (int)(16.0 * mean));
      if (mx > thr && thr < kLongRow) {
        long_thr = thr;
        seg_len = thr;
      }
    }
    std::vector<int> em;
    em.reserve(rows.size());
    for (int r : rows) {
      const int b = rp[r], e = rp[r + 1];
      if (e == b && !stencil_rows && ((size_t)cc * elem) % 16 == 0) {
        em.push_back(r);
      } else if (e - b <= long_thr) {
        sh.push_back(r);
      } else {
        lg.push_back(r);
        for (int k = b; k < e; k += seg_len) {
          k0.push_back(k);
          k1.push_back(std::min(e, k + seg_len));
        }
        off.push_back((int64_t)k0.size());
      }
    }
    n_empty = (int64_t)em.size();
    if (n_empty) {
      empty_rows.alloc(em.size());
      h2d(empty_rows.p, em.data(), em.size(), st);
    }
    if (!sh.empty()) {  // skew: longest short row vs the mean
      int64_t tot = 0;
      int mx = 0;
      for (int r : sh) {
        tot += rp[r + 1] - rp[r];
        mx = std::max(mx, rp[r + 1] - rp[r]);
      }
      const double mean = (double)tot / (double)sh.size();
      // one row per lane group when rows are skewed, or when strips of 32
      // rows would leave the GPU with too few warps (small row lists)
      skewed = mx > 8.0 * std::max(mean, 1.0) ||
               (int64_t)sh.size() < (int64_t)sm_count() * 32 * 32;
      // skewed lists: longest rows first (the lane groups of a warp then walk
      // rows of similar length, and the long rows start early)
      static const bool sort_on = [] {
        const char* e = getenv("TFG_W1_SORT");
        return !e || atoi(e) > 0;
      }();
      if (skewed && sort_on && !stencil_rows) {
        // stable counting sort by descending length (lengths <= long_thr); a
        // comparison sort of millions of rows costs ~0.2 s of plan creation
        std::vector<int64_t> start((size_t)mx + 2, 0);
        for (int r : sh) ++start[(size_t)(mx - (rp[r + 1] - rp[r])) + 1];
        for (size_t l = 1; l < start.size(); ++l) start[l] += start[l - 1];
        std::vector<int> sorted(sh.size());
        for (int r : sh) sorted[(size_t)start[(size_t)(mx - (rp[r + 1] - rp[r]))]++] = r;
        sh.swap(sorted);
      }
    }
    n_short = (int64_t)sh.size();
    n_long = (int64_t)lg.size();
    n_seg = (int64_t)k0.size();
    identity = false;
    if (n_short > 0 && n_long == 0) {
      bool id = true;
      for (int64_t q = 1; q < n_short && id; ++q) id = sh[q] == sh[q - 1] + 1;
      if (id) {
        identity = true;
        row0 = sh[0];
      }
    }
    if (!identity) {
      short_rows.alloc(sh.size());
      h2d(short_rows.p, sh.data(), sh.size(), st);
    }
    long_rows.alloc(lg.size());
    h2d(long_rows.p, lg.data(), lg.size(), st);
    seg_k0.alloc(k0.size());
    seg_k1.alloc(k1.size());
    h2d(seg_k0.p, k0.data(), k0.size(), st);
    h2d(seg_k1.p, k1.data(), k1.size(), st);
    long_seg_off.alloc(off.size());
    h2d(long_seg_off.p, off.data(), off.size(), st);
    partial.alloc((size_t)n_seg * cc * elem);
    TFG_CUDA(cudaStreamSynchronize(st));
    const int vec = 16 / (int)elem;
    elem_ = elem;
    if (ci && identity && !stencil_rows && (cc % vec == 0) &&
        (cc / vec == 8 || cc / vec == 16 || cc / vec == 32 || cc / vec == 64))
      build_band(row0, n_short, rp, *ci, cc, elem, st);
    if (getenv("TFG_DEBUG"))
      fprintf(stderr,
              "[tfg] spmm work: short=%lld long=%lld identity=%d skewed=%d banded=%d R=%d "
              "blocks=%d stage_cap=%d smem=%zu ci=%d\n",
              (long long)n_short, (long long)n_long, (int)identity, (int)skewed, (int)banded,
              band_R, band_blocks, stage_cap, band_smem, ci ? 1 : 0);
    if (n_long > 0 && n_short > 0 && !side) {
      TFG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      TFG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      TFG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
  }
  size_t bytes() const {
    return short_rows.bytes() + long_rows.bytes() + seg_k0.bytes() + seg_k1.bytes() +
           long_seg_off.bytes() + partial.bytes() +
           run_begin.bytes() + run_start.bytes() + run_len.bytes() + idx_off.bytes() +
           lidx.bytes() + empty_rows.bytes();
  }
  int launches() const {
    return (n_short > 0) + 2 * (n_long > 0) + (n_empty > 0);
  }
};

template <class T>
static void spmm_dispatch_short(const SpmmWork& w, const int* rp, const int* ci,
                                const T* av, const T* X, int cc, T* out,
                                cudaStream_t st) {
  if (w.n_short == 0) return;
  constexpr int VEC = 16 / sizeof(T);
  if (w.banded) {
    // band-staged blocks (k_spmm_band3): 2-stage ring, 8 consumer warps; the
    // stencil (diagonal-line) consumer where every mini-group qualifies
    const int L = cc / VEC;
    const size_t smem = w.band_smem;
#define TFG_BAND(LPR, NCH)                                                                   \
  {                                                                                          \
    auto kern = k_spmm_band3<T, VEC, LPR, NCH, 2>;                                           \
    if constexpr (LPR == 32)                                                                 \
      if (w.dia) kern = k_spmm_band3<T, VEC, LPR, NCH, 2, true>;                             \
    TFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                                  (int)smem));                                               \
    int occ = 1;                                                                             \
    TFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 288, smem));          \
    const int grid = (int)std::min<int64_t>(w.band_blocks, (int64_t)sm_count() * std::max(occ, 1)); \
    kern<<<grid, 288, smem, st>>>(w.band_blocks, w.band_R, w.row0, (int)w.n_short, rp, av,   \
                                  w.run_begin.p, w.run_start.p, w.run_len.p, w.idx_off.p,    \
                                  w.lidx.p, w.stage_cap, w.idx_cap, w.val_cap, X, cc, out, cc, \
                                  w.dia ? w.dia_dev.p : nullptr);                            \
    TFG_LAUNCH_CHECK();                                                                      \
    return;                                                                                  \
  }
    if (L == 8) TFG_BAND(8, 1)
    if (L == 16) TFG_BAND(16, 1)
    if (L == 32) TFG_BAND(32, 1)
    if (L == 64) TFG_BAND(32, 2)
#undef TFG_BAND
  }
  const int* rows = w.identity ? nullptr : w.short_rows.p;
  const int row0 = w.identity ? w.row0 : 0;
  const int64_t n = w.n_short;
  // skewed lists: one row per lane group, 2 gathers in flight at full
  // occupancy (cfg3 1.02 -> 0.76 ms); uniform lists: strips of LPR rows
#define TFG_SPMM_CASE(LPR, NCH)                                                        \
  if (w.skewed)                                                                        \
    k_spmm_strip<T, VEC, LPR, NCH, 2, 8, 1><<<blocks_for(n * LPR), 256, 0, st>>>(       \
        n, rows, row0, rp, ci, av, X, cc, out, cc);                                    \
  else                                                                                 \
    k_spmm_strip<T, VEC, LPR, NCH, 4, 4><<<blocks_for((n + LPR - 1) / LPR * LPR), 256, 0, st>>>( \
        n, rows, row0, rp, ci, av, X, cc, out, cc);                                    \
  TFG_LAUNCH_CHECK();                                                                  \
  return;
  if (cc % VEC == 0) {
    switch (cc / VEC) {
      case 4: TFG_SPMM_CASE(4, 1)
      case 8: TFG_SPMM_CASE(8, 1)
      case 16: TFG_SPMM_CASE(16, 1)
      case 32: TFG_SPMM_CASE(32, 1)
      case 64: TFG_SPMM_CASE(32, 2)
      default: break;
    }
  }
#undef TFG_SPMM_CASE
  k_spmm_rows_generic<T><<<blocks_for(n * 32), 256, 0, st>>>(n, rows, row0, rp, ci, av,
                                                               X, cc, cc, out, cc);
  TFG_LAUNCH_CHECK();
}

template <class T>
static void spmm_long(const SpmmWork& w, const int* ci, const T* av, const T* X, int cc, T* out,
                      cudaStream_t st) {
  T* partial = reinterpret_cast<T*>(w.partial.p);
  constexpr int VEC = 16 / sizeof(T);
  const int L = cc % VEC == 0 ? cc / VEC : 0;
#define TFG_SEG(LPR, NCH)                                                                     \
  {                                                                                           \
    /* 8 gathers in flight per lane group: cfg5 wavefront 1 10.3 -> 9.1 ms (vs 4) */          \
    k_spmm_segments_vec<T, VEC, LPR, NCH, 8><<<blocks_for(w.n_seg * LPR), 256, 0, st>>>(      \
        w.n_seg, w.seg_k0.p, w.seg_k1.p, ci, av, X, cc, partial);                             \
    TFG_LAUNCH_CHECK();                                                                       \
    k_segment_combine_vec<T, VEC, LPR, NCH><<<blocks_for(w.n_long * LPR), 256, 0, st>>>(      \
        w.n_long, w.long_rows.p, w.long_seg_off.p, partial, cc, out, cc);                     \
    TFG_LAUNCH_CHECK();                                                                       \
    return;                                                                                   \
  }
  if (L == 8) TFG_SEG(8, 1)
  if (L == 16) TFG_SEG(16, 1)
  if (L == 32) TFG_SEG(32, 1)
  if (L == 64) TFG_SEG(32, 2)
#undef TFG_SEG
  k_spmm_segments<T><<<blocks_for(w.n_seg * 32), 256, 0, st>>>(
      w.n_seg, w.seg_k0.p, w.seg_k1.p, ci, av, X, cc, cc, partial);
  TFG_LAUNCH_CHECK();
  k_segment_combine<T><<<blocks_for(w.n_long * 32), 256, 0, st>>>(
      w.n_long, w.long_rows.p, w.long_seg_off.p, partial, cc, out, cc);
  TFG_LAUNCH_CHECK();
}

// D rows of the empty rows of the list (no other kernel touches them)
template <class T>
static void spmm_zero_empty(const SpmmWork& w, int cc, T* out, cudaStream_t st) {
  const int rb = cc * (int)sizeof(T);
  const int64_t thr = w.n_empty * (rb / 16);
  k_zero_rows<<<(unsigned)((thr + 255) / 256), 256, 0, st>>>(
      w.n_empty, w.empty_rows.p, rb, reinterpret_cast<unsigned char*>(out));
  TFG_LAUNCH_CHECK();
}

// The empty rows of a forked list can be zeroed early, on the side stream,
// beside whatever the main stream runs before this list (spmm_run then joins
// the side stream as it does for the long rows).
static bool spmm_can_zero_early(const SpmmWork& w) {
  static const bool on = [] {  // TFG_ZERO_EARLY=0: keep the zero fill in front of wavefront 1
    const char* e = getenv("TFG_ZERO_EARLY");
    return !e || atoi(e) > 0;
  }();
  return on && !w.stencil && w.side && w.n_long && w.n_short && w.n_empty;
}
template <class T>
static void spmm_zero_early(const SpmmWork& w, int cc, T* out, cudaStream_t st) {
  TFG_CUDA(cudaEventRecord(w.ev_fork, st));
  TFG_CUDA(cudaStreamWaitEvent(w.side, w.ev_fork, 0));
  spmm_zero_empty<T>(w, cc, out, w.side);
}

template <class T>
static void spmm_run(const SpmmWork& w, const int* rp, const int* ci,
                     const T* av, const T* X, int cc, T* out, cudaStream_t st,
                     bool empty_done = false) {
  if (w.stencil) {
    stencil_run(*w.stencil, rp, ci, av, out, st, w.exact);
    return;
  }
  // short and long (segmented) rows are independent: the long rows run on a
  // side stream beside the short-row kernel (latency-bound gathers both)
  const bool fork = w.side && w.n_long && w.n_short;
  if (fork) {
    TFG_CUDA(cudaEventRecord(w.ev_fork, st));
    TFG_CUDA(cudaStreamWaitEvent(w.side, w.ev_fork, 0));
  }
  if (w.n_long) spmm_long<T>(w, ci, av, X, cc, out, fork ? w.side : st);
  if (w.n_empty && !empty_done) spmm_zero_empty<T>(w, cc, out, st);
  spmm_dispatch_short<T>(w, rp, ci, av, X, cc, out, st);
  if (fork) {
    TFG_CUDA(cudaEventRecord(w.ev_join, w.side));
    TFG_CUDA(cudaStreamWaitEvent(st, w.ev_join, 0));
  }
}

}  // namespace tfg

// ===========================================================================
// The plan behind tfg_plan.
// ===========================================================================
namespace tfg {
struct PlanProfileCtx {
  std::vector<int> fo_rows, second_rows, arp, brp;
};
}  // namespace tfg

struct tfg_plan {
  tfg_problem p{};
  size_t elem = 8;
  bool has_sched = false;
  bool zero_d = false;  // schedule does not cover every j row
  // (a) first op for j-less wavefront-0 tiles / all rows when unfused
  int64_t n_fo_blocks = 0;
  int gemm_kind = 0;             // 0 generic k_gemm_blocks, else k_gemm_v2 config id
  int gemm_bm = 64;
  tfg::dbuf<int> fo_r0, fo_cnt;  // dense B: GEMM row blocks
  tfg::dbuf<int> fo_ihi;         // r0 + cnt (tensor-core first op)
  tfg::TcPlan tc;                // fp32 dense B: tcgen05 3xTF32 first op (tfg_tc.cu)
  tfg::dbuf<int64_t> fx_off;     // tc fused rows: offsets into fx_idx (ft_jrows order)
  tfg::dbuf<int> fx_idx;         // per fused nonzero: stage slot (staged tile) or D1 row (wide)
  tfg::dbuf<int> fx_aoff;        // per fused row: arp[j] - fx_off[q] (value offset)
  tfg::SpmmWork fo_sparse;       // sparse B: SpMM rows with X = C
  // (b) fused tiles
  int64_t n_ftiles = 0;
  tfg::dbuf<int> ft_ilo, ft_ihi, ft_jrows;
  tfg::dbuf<int64_t> ft_joff;
  int w_cap = 0, cs = 0, n_slices = 0;
  size_t fused_smem = 0;
  int64_t ft_nrows = 0;      // fused (non-empty) j rows in the fused tiles
  bool fused_v2 = false;     // dense-B pipelined GEMM tiles with slot staging
  tfg::dbuf<int> slot;       // D1 row -> stage slot within its tile (-1 none)
  tfg::dbuf<uint8_t> ft_wide;
  tfg::dbuf<int> ft_order;   // tc fused tiles: balanced tile order of the persistent grid
  int stage_cap = 0;
  int64_t n_wide = 0;
  // (c) wavefront 1 / unfused second op
  tfg::SpmmWork second;
  tfg::dbuf<uint8_t> spill;
  tfg::dbuf<unsigned char> d1;
  // accounting
  int64_t spill_rows = 0, fused_rows = 0;
  int64_t first_rows = 0, second_rows = 0, nnz_processed = 0;
  int launches = 0;
  int row_lo = 0, row_hi = 0;  // row block of a partition plan (multi-GPU)
  std::vector<int> w1_rows;    // partition plans: the wavefront-1 row list (tfg_halo_create)
  // algorithmic (compulsory) HBM bytes per stage: (a) first op, (b) fused
  // tiles, (c) wavefront-1 SpMM -- each input byte read once, each output
  // byte written once (the roofline numerator)
  int64_t stage_bytes[3] = {0, 0, 0};
  int64_t d1_read_rows = 0;  // distinct D1 rows wavefront 1 reads
  bool stage_bytes_done = false;
  std::unique_ptr<tfg::PlanProfileCtx> prof;  // host lists kept for compute_stage_bytes
};

// Multi-GPU halo of one rank's partition plan (tfg_halo_create).
struct tfg_halo {
  int world = 1, rank = 0;
  int mode = TFG_HALO_EXCHANGE;
  int64_t n_recv = 0, n_send = 0;
  std::vector<int64_t> recv_off, send_off;  // per peer, rows (world + 1)
  tfg::dbuf<int> recv_rows, send_rows;      // global D1 rows, grouped by peer
  tfg::dbuf<unsigned char> recv_buf, send_buf;
  // recompute mode: first-op row blocks covering the halo rows
  int64_t n_rblk = 0;
  tfg::dbuf<int> r_r0, r_cnt, r_ihi;
  // wavefront 1 split: rows reading only local D1 run during the exchange
  bool split = false;
  tfg::SpmmWork interior, boundary;
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_recv = nullptr;
  double t_exchange_us = 0, t_recompute_us = 0;  // the cost model's estimates
  ~tfg_halo() {
    if (ev_packed) cudaEventDestroy(ev_packed);
    if (ev_recv) cudaEventDestroy(ev_recv);
    if (comm) cudaStreamDestroy(comm);
  }
};

namespace tfg {

static constexpr int kGemmBM = 64, kGemmBN = 64, kGemmBK = 16, kGemmTM = 4, kGemmTN = 4;
static constexpr size_t kFusedSmemCap = 200 * 1024;
// the row-group layout is analysed on the host at plan time up to this nnz
static constexpr int64_t kGroupMaxNnz = 96ll << 20;
static constexpr size_t kFusedSmemMax = 227 * 1024;  // sm_100 opt-in max per CTA

// FMA first-op GEMM tilings (measured best): FP32 BN =
// 128 -> 128x128 blocks of 8x8 thread tiles, BN = 64 -> 128x64 of 8x4;
// FP64 BN = 64 -> 64x64 blocks of 8x4 tiles, 128 threads (cfg1 first op
// 0.062 ms with 4x4 tiles -> 0.047 ms: more, smaller blocks).

// shared memory of the pipelined GEMM configuration a plan uses
static size_t fused_gemm_smem(const tfg_plan& pl) {
  if (pl.elem == 4) {
    return pl.gemm_kind == 2 ? GemmCfg<float, 128, 128, 32, 8, 8, 3>::SMEM
                             : GemmCfg<float, 128, 64, 32, 8, 4, 3>::SMEM;
  }
  return pl.gemm_kind == 2 ? GemmCfg<double, 64, 128, 16, 4, 8, 3>::SMEM
                           : GemmCfg<double, 64, 64, 16, 4, 4, 3>::SMEM;
}

// The band layout pays only for identity row lists of similar-length rows
// (the skew test of SpmmWork::build): skip copying column indices otherwise.
static bool band_candidate(const std::vector<int>& rows, const std::vector<int>& rp) {
  if (rows.empty()) return false;
  for (size_t q = 1; q < rows.size(); ++q)
    if (rows[q] != rows[q - 1] + 1) return false;
  int64_t tot = 0;
  int mx = 0;
  for (int r : rows) {
    tot += rp[r + 1] - rp[r];
    mx = std::max(mx, rp[r + 1] - rp[r]);
  }
  return mx <= 8.0 * std::max((double)tot / (double)rows.size(), 1.0);
}

static StencilGeom probe_stencil(int64_t n, const std::vector<int>& rp, const int* rp_d,
                                 const int* ci_d, cudaStream_t st) {
  StencilGeom g;
  if (stencil_env_enabled() && n <= INT32_MAX) stencil_detect((int)n, rp, rp_d, ci_d, g, st);
  return g;
}

// The row list is a whole-plane slab of the grid (what the stencil kernel runs).
static bool stencil_rows(const std::vector<int>& rows, const StencilGeom& g, int cc,
                         size_t elem) {
  if (g.nx == 0 || rows.empty() || (size_t)cc * elem % 512 != 0) return false;
  const int64_t nxy = (int64_t)g.nx * g.ny;
  for (size_t q = 1; q < rows.size(); ++q)
    if (rows[q] != rows[q - 1] + 1) return false;
  return rows[0] % nxy == 0 && (int64_t)rows.size() % nxy == 0;
}

static void attach_stencil(SpmmWork& w, const StencilGeom& g, const void* X, int cc,
                           size_t elem) {
  w.stencil.reset();
  if (g.nx == 0 || !w.identity || w.n_short == 0 || w.n_long != 0) return;
  // the rows must be whole grid planes (a partition's slab of z)
  const int64_t nxy = (int64_t)g.nx * g.ny;
  if (w.row0 % nxy != 0 || w.n_short % nxy != 0) return;
  auto sp = std::make_unique<StencilPlan>();
  if (!stencil_prepare(*sp, g, X, cc, (int)elem, (int)(w.row0 / nxy),
                       (int)((w.row0 + w.n_short) / nxy)))
    return;
  if (getenv("TFG_DEBUG"))
    fprintf(stderr,
            "[tfg] stencil spmm: grid %d x %d x %d K=%d tile %d x %d zc %d ns %d slices %d "
            "items %lld grid %d smem %zu\n",
            g.nx, g.ny, g.nz, g.K, sp->tx, sp->ty, sp->zc, sp->ns, sp->slices,
            (long long)sp->items, sp->grid, sp->smem);
  w.stencil = std::move(sp);
}

// Algorithmic (compulsory) HBM bytes of each stage, the roofline numerator
// (DESIGN.md section 4): each input byte read once, each output written once.
static void compute_stage_bytes(tfg_plan& pl, cudaStream_t st) {
  if (pl.stage_bytes_done || !pl.prof) return;
  const tfg_problem& pr = pl.p;
  const int n = pr.n, cc = pr.c_cols, bc = pr.b_cols;
  const std::vector<int>& fo_rows = pl.prof->fo_rows;
  const std::vector<int>& second_rows = pl.prof->second_rows;
  const std::vector<int>& arp = pl.prof->arp;
  const std::vector<int>& brp = pl.prof->brp;

    const int64_t el = (int64_t)pl.elem;
    auto csr_rows_bytes = [&](const std::vector<int>& rows, const std::vector<int>& rp) {
      int64_t b = 0;
      for (int r : rows) b += 4 + (int64_t)(rp[r + 1] - rp[r]) * (4 + el);
      return b;
    };
    // distinct X rows referenced by `rows` of the CSR (rp_d, ci_d)
    auto distinct_cols = [&](const std::vector<int>& rows, const int* rp_d, const int* ci_d,
                             int ncols) -> int64_t {
      if (rows.empty()) return 0;
      dbuf<int> rows_d(rows.size());
      h2d(rows_d.p, rows.data(), rows.size(), st);
      dbuf<uint8_t> mark(ncols);
      TFG_CUDA(cudaMemsetAsync(mark.p, 0, ncols, st));
      k_mark_cols<<<blocks_for((int64_t)rows.size() * 32), 256, 0, st>>>(
          (int64_t)rows.size(), rows_d.p, rp_d, ci_d, mark.p);
      TFG_LAUNCH_CHECK();
      dbuf<unsigned long long> cnt(1);
      TFG_CUDA(cudaMemsetAsync(cnt.p, 0, 8, st));
      k_count_u8<<<256, 256, 0, st>>>(ncols, mark.p, cnt.p);
      TFG_LAUNCH_CHECK();
      unsigned long long h = 0;
      d2h(&h, cnt.p, 1, st);
      TFG_CUDA(cudaStreamSynchronize(st));
      return (int64_t)h;
    };
    const int64_t ra = (int64_t)fo_rows.size();
    if (ra) {
      if (pr.b_is_dense)
        pl.stage_bytes[0] = ra * bc * el + (int64_t)bc * cc * el + ra * cc * el;
      else
        pl.stage_bytes[0] = csr_rows_bytes(fo_rows, brp) +
                            distinct_cols(fo_rows, pr.d_b_row_ptr, pr.d_b_col_idx, bc) * cc * el +
                            ra * cc * el;
    }
    if (pl.n_ftiles) {
      std::vector<int> ti, tj;  // first-op rows and fused j rows of fused tiles
      std::vector<int> ilo(pl.n_ftiles), ihi(pl.n_ftiles);
      d2h(ilo.data(), pl.ft_ilo.p, pl.n_ftiles, st);
      d2h(ihi.data(), pl.ft_ihi.p, pl.n_ftiles, st);
      tj.resize(pl.ft_nrows);
      d2h(tj.data(), pl.ft_jrows.p, pl.ft_nrows, st);
      std::vector<uint8_t> sp(n);
      d2h(sp.data(), pl.spill.p, n, st);
      TFG_CUDA(cudaStreamSynchronize(st));
      int64_t spilled = 0;
      for (int64_t v = 0; v < pl.n_ftiles; ++v)
        for (int i = ilo[v]; i < ihi[v]; ++i) {
          ti.push_back(i);
          spilled += sp[i];
        }
      const int64_t w = (int64_t)ti.size();
      int64_t b = 0;
      if (pr.b_is_dense)
        b = w * bc * el + (int64_t)bc * cc * el;
      else
        b = csr_rows_bytes(ti, brp) + distinct_cols(ti, pr.d_b_row_ptr, pr.d_b_col_idx, bc) * cc * el;
      b += csr_rows_bytes(tj, arp) + (int64_t)tj.size() * cc * el + spilled * cc * el;
      pl.stage_bytes[1] = b;
    }
    if (!second_rows.empty())
      pl.d1_read_rows = distinct_cols(second_rows, pr.d_a_row_ptr, pr.d_a_col_idx, n);
      pl.stage_bytes[2] = csr_rows_bytes(second_rows, arp) + pl.d1_read_rows * cc * el +
                          (int64_t)second_rows.size() * cc * el;
    pl.stage_bytes_done = true;
  pl.prof.reset();
}

void plan_create(const tfg_problem& pr, const tfg_schedule* s, cudaStream_t st,
                 tfg_plan& pl, int row_lo = 0, int row_hi = -1, uint32_t flags = 0) {
  AllocScope scope(st);  // temporaries stream-ordered: no device-wide sync on free
  // problem.check() -- kernels.hpp:35-42; require_workers is the caller's.
  if (pr.dtype != TFG_F32 && pr.dtype != TFG_F64)
    throw invalid_argument("problem: unknown dtype");
  if (pr.n < 1) throw invalid_argument("problem: A must be square");
  if (pr.b_rows != pr.n) throw invalid_argument("problem: B must have n rows");
  if (pr.c_rows != pr.b_cols)
    throw invalid_argument("problem: C rows must match B cols");
  if (pr.c_cols < 1 || pr.b_cols < 1)
    throw invalid_argument("problem: B and C need at least one column");
  if (s && s->n != pr.n)
    throw invalid_argument("schedule and problem disagree on n");
  // the SpMM kernels read X rows with 16-byte vector loads (tfg.h: operands
  // 16-byte aligned, as cudaMalloc returns them)
  if (!pr.b_is_dense && (uintptr_t)pr.d_c % 16 != 0)
    throw invalid_argument("problem: C must be 16-byte aligned");
  if ((uintptr_t)pr.d_a_val % 16 != 0 || (!pr.b_is_dense && (uintptr_t)pr.d_b_val % 16 != 0))
    throw invalid_argument("problem: CSR values must be 16-byte aligned");

  pl.p = pr;
  pl.elem = pr.dtype == TFG_F64 ? 8 : 4;
  pl.has_sched = s != nullptr;
  pl.fo_sparse.exact = pl.second.exact = (flags & TFG_PLAN_REFERENCE_BITS) != 0;
  // TFG_DEBUG: wall time of each plan-creation phase
  const bool dbg_t = getenv("TFG_DEBUG") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!dbg_t) return;
    TFG_CUDA(cudaStreamSynchronize(st));
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[tfg] plan phase %-24s %8.2f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  const int n = pr.n, cc = pr.c_cols, bc = pr.b_cols;
  if (row_hi < 0) row_hi = n;
  if (row_lo < 0 || row_hi > n || row_lo > row_hi)
    throw invalid_argument("plan: partition rows out of range");
  const bool partial = row_lo != 0 || row_hi != n;
  pl.row_lo = row_lo;
  pl.row_hi = row_hi;

  std::vector<int> arp(n + 1), brp;
  d2h(arp.data(), pr.d_a_row_ptr, n + 1, st);
  if (!pr.b_is_dense) {
    brp.resize(n + 1);
    d2h(brp.data(), pr.d_b_row_ptr, n + 1, st);
  }
  TFG_CUDA(cudaStreamSynchronize(st));
  pl.nnz_processed = arp[n];
  pl.d1.alloc((size_t)n * cc * pl.elem);
  pl.spill.alloc(n);
  phase("row_ptr + d1 alloc");

  std::vector<int> fo_rows;  // first-op rows handled by stage (a)
  std::vector<int> second_rows;
  std::vector<int> zero_rows;  // empty fused rows, written by the SpMM stage
  StencilGeom gB;              // B's grid-stencil geometry (sparse B), probed once
  if (pr.b_is_dense) {
    // fast path: cp.async pipelined GEMM when the shapes and pointers allow
    const int V = 16 / (int)pl.elem;
    const bool aligned = ((uintptr_t)pr.d_b_dense % 16 == 0) && ((uintptr_t)pr.d_c % 16 == 0) &&
                         (bc % V == 0);
    pl.gemm_kind = 0;
    pl.gemm_bm = kGemmBM;
    if (aligned && cc % 128 == 0)
      pl.gemm_kind = 2;  // BN = 128
    else if (aligned && cc % 64 == 0)
      pl.gemm_kind = 1;  // BN = 64
    if (pl.gemm_kind)
      pl.gemm_bm = pl.elem == 4 ? 128 : 64;
    if (pl.gemm_kind && pl.elem == 4 &&
        tc_prepare(pl.tc, static_cast<const float*>(pr.d_b_dense), n, bc, cc))
      pl.gemm_bm = 128;
  }
  phase("gemm/tc prepare");
  if (!s) {
    for (int i = row_lo; i < row_hi; ++i) fo_rows.push_back(i);
    second_rows = fo_rows;
    pl.first_rows = row_hi - row_lo;
    pl.second_rows = row_hi - row_lo;
    pl.spill_rows = n;
  } else {
    const int64_t nt0 = s->n_tiles[0];
    std::vector<int> ilo(nt0), ihi(nt0);
    std::vector<int64_t> joff(nt0 + 1);
    d2h(ilo.data(), s->i_lo[0].p, nt0, st);
    d2h(ihi.data(), s->i_hi[0].p, nt0, st);
    d2h(joff.data(), s->j_off[0].p, nt0 + 1, st);
    const int64_t nj1 = s->n_jrows[1];
    second_rows.resize(nj1);
    d2h(second_rows.data(), s->j_rows[1].p, nj1, st);
    TFG_CUDA(cudaStreamSynchronize(st));
    if (partial) {  // this rank owns the wavefront-1 rows of its row block
      std::vector<int> mine;
      for (int j : second_rows)
        if (j >= row_lo && j < row_hi) mine.push_back(j);
      second_rows.swap(mine);
    }
    std::vector<int> jr0(s->n_jrows[0]);
    d2h(jr0.data(), s->j_rows[0].p, jr0.size(), st);
    TFG_CUDA(cudaStreamSynchronize(st));
    std::vector<int> f_ilo, f_ihi, f_rows;
    std::vector<int64_t> f_joff{0};
    f_rows.reserve(jr0.size());
    zero_rows.reserve(jr0.size());
    f_ilo.reserve(nt0);
    f_ihi.reserve(nt0);
    f_joff.reserve(nt0 + 1);
    int w_max = 0;
    int64_t fused_here = 0;
    for (int64_t v = 0; v < nt0; ++v) {
      if (ilo[v] < row_lo || ilo[v] >= row_hi) continue;  // tiles partitioned by i_lo
      fused_here += joff[v + 1] - joff[v];
      pl.first_rows += ihi[v] - ilo[v];
      // empty fused rows need no D1 (D row = 0): the SpMM stage writes them
      const size_t before = f_rows.size();
      for (int64_t q = joff[v]; q < joff[v + 1]; ++q) {
        const int j = jr0[q];
        if (arp[j + 1] > arp[j])
          f_rows.push_back(j);
        else
          zero_rows.push_back(j);
      }
      if (f_rows.size() == before) {
        for (int i = ilo[v]; i < ihi[v]; ++i) fo_rows.push_back(i);
      } else {
        f_ilo.push_back(ilo[v]);
        f_ihi.push_back(ihi[v]);
        f_joff.push_back((int64_t)f_rows.size());
        w_max = std::max(w_max, ihi[v] - ilo[v]);
      }
    }
    phase("schedule d2h + tile lists");
    pl.fused_rows = fused_here;
    pl.second_rows = fused_here + (int64_t)second_rows.size();
    pl.zero_d = !partial && pl.second_rows != n;
    pl.n_ftiles = (int64_t)f_ilo.size();
    if (pl.n_ftiles) {
      pl.ft_ilo.alloc(pl.n_ftiles);
      pl.ft_ihi.alloc(pl.n_ftiles);
      pl.ft_joff.alloc(pl.n_ftiles + 1);
      h2d(pl.ft_ilo.p, f_ilo.data(), f_ilo.size(), st);
      h2d(pl.ft_ihi.p, f_ihi.data(), f_ihi.size(), st);
      h2d(pl.ft_joff.p, f_joff.data(), f_joff.size(), st);
      pl.ft_jrows.alloc(f_rows.size());
      h2d(pl.ft_jrows.p, f_rows.data(), f_rows.size(), st);
      pl.ft_nrows = (int64_t)f_rows.size();
        phase("  ft lists uploaded");
      if (pr.b_is_dense && pl.gemm_kind) {
        // v2: stage only the D1 rows the tile's fused rows read
        const int BN = pl.gemm_kind == 2 ? 128 : 64;
        pl.fused_v2 = true;
        pl.cs = BN;
        pl.n_slices = cc / BN;
        dbuf<uint8_t> mark(n);
        TFG_CUDA(cudaMemsetAsync(mark.p, 0, n, st));
        k_mark_cols<<<blocks_for((int64_t)f_rows.size() * 32), 256, 0, st>>>(
            (int64_t)f_rows.size(), pl.ft_jrows.p, pr.d_a_row_ptr, pr.d_a_col_idx, mark.p);
        TFG_LAUNCH_CHECK();
        pl.slot.alloc(n);
        TFG_CUDA(cudaMemsetAsync(pl.slot.p, 0xff, (size_t)n * 4, st));
        dbuf<int> tcount(pl.n_ftiles);
        k_assign_slots<<<blocks_for(pl.n_ftiles * 32), 256, 0, st>>>(
            pl.n_ftiles, pl.ft_ilo.p, pl.ft_ihi.p, mark.p, pl.slot.p, tcount.p);
        TFG_LAUNCH_CHECK();
        std::vector<int> tc(pl.n_ftiles);
        d2h(tc.data(), tcount.p, tc.size(), st);
        TFG_CUDA(cudaStreamSynchronize(st));
        phase("  marks + slots");
        const size_t gsm = fused_gemm_smem(pl);
        // stage capacity: two CTAs per SM when the GEMM ring leaves room
        const size_t per_cta = 2 * gsm + 16 * 1024 <= kFusedSmemMax ? kFusedSmemMax / 2 - 1024
                                                                   : kFusedSmemMax;
        size_t cap_bytes = per_cta > gsm ? per_cta - gsm : 0;
        int max_need = 0;
        for (int c : tc) max_need = std::max(max_need, c);
        size_t row_bytes = (size_t)BN * pl.elem;
        if (pl.tc.on) {  // tensor-core tiles: one CTA per SM, stage after ring + C
          // column slice: wider slices read B fewer times, narrower ones leave
          // more shared memory for staged D1 rows; fused rows of tiles that do
          // not fit gather D1 from L2 (weighted 2x: random 4-16 B-per-lane
          // gathers against streamed TMA blocks)
          std::vector<int64_t> tnnz(pl.n_ftiles, 0);
          int64_t ft_rows = 0;
          for (int64_t v = 0; v < pl.n_ftiles; ++v) {
            ft_rows += f_ihi[v] - f_ilo[v];
            for (int64_t q = f_joff[v]; q < f_joff[v + 1]; ++q)
              tnnz[v] += arp[f_rows[q] + 1] - arp[f_rows[q]];
          }
          int best_bn = pl.tc.bn;
          double best = 1e300;
          for (int bnc = pl.tc.bn; bnc >= 32 && cc % bnc == 0; bnc /= 2) {
            const int capc = (int)std::min<size_t>(tc_stage_bytes_bn(pl.tc, bnc) / ((size_t)bnc * 4),
                                                   (size_t)max_need);
            int64_t wide_nnz = 0;
            for (int64_t v = 0; v < pl.n_ftiles; ++v)
              if (tc[v] > capc) wide_nnz += tnnz[v];
            const double cost = (double)(cc / bnc) * ft_rows * bc * 4 + 2.0 * wide_nnz * cc * 4;
            if (getenv("TFG_DEBUG"))
              fprintf(stderr, "[tfg] tc candidate bn %d cap %d wide-nnz %lld cost %.3g\n", bnc, capc,
                      (long long)wide_nnz, cost);
            if (cost < best) {
              best = cost;
              best_bn = bnc;
            }
          }
          if (best_bn != pl.tc.bn) tc_set_bn(pl.tc, best_bn);
          if (getenv("TFG_DEBUG")) {
            const int capc = (int)std::min<size_t>(
                tc_stage_bytes(pl.tc) / ((size_t)pl.tc.bn * 4), (size_t)max_need);
            int64_t wn = 0, an = 0;
            for (int64_t v = 0; v < pl.n_ftiles; ++v) {
              an += tnnz[v];
              if (tc[v] > capc) wn += tnnz[v];
            }
            fprintf(stderr, "[tfg] tc bn %d slices %d cap %d wide-nnz %.3f of %lld\n", pl.tc.bn,
                    pl.tc.slices, capc, an ? (double)wn / an : 0.0, (long long)an);
          }
          cap_bytes = tc_stage_bytes(pl.tc);
          row_bytes = (size_t)pl.tc.bn * 4;
          pl.cs = pl.tc.bn;
          pl.n_slices = pl.tc.slices;
        }
        const int cap = (int)std::min<size_t>(cap_bytes / row_bytes, (size_t)max_need);
        std::vector<uint8_t> wide(pl.n_ftiles);
        for (int64_t v = 0; v < pl.n_ftiles; ++v) {
          wide[v] = tc[v] > cap;
          pl.n_wide += wide[v];
        }
        pl.ft_wide.alloc(pl.n_ftiles);
        h2d(pl.ft_wide.p, wide.data(), wide.size(), st);
        phase("  slice choice");
        pl.stage_cap = cap;
        pl.fused_smem = gsm + (size_t)cap * BN * pl.elem;
        if (pl.tc.on) {
          tc_finalize(pl.tc, cap);
          pl.fused_smem = pl.tc.smem;
          {
            // balanced tile order for the persistent grid: tiles by estimated
            // cost (B bytes streamed + fused-row gathers, L2 gathers of tiles
            // too wide for the stage weighted 2x), longest first onto the
            // least-loaded CTA (cfg3: per-SM active cycles max / avg 1.15)
            const int64_t G = tc_grid(pl.tc, pl.n_ftiles);
            std::vector<double> cost(pl.n_ftiles);
            std::vector<int64_t> idx(pl.n_ftiles);
            for (int64_t v = 0; v < pl.n_ftiles; ++v) {
              const int64_t rows128 = ((int64_t)(f_ihi[v] - f_ilo[v]) + 127) / 128 * 128;
              int64_t fnnz = 0;  // nonzeros of the tile's fused rows
              for (int64_t q = f_joff[v]; q < f_joff[v + 1]; ++q)
                fnnz += arp[f_rows[q] + 1] - arp[f_rows[q]];
              cost[v] = (double)rows128 * bc * 4 + (wide[v] ? 2.0 : 1.0) * (double)fnnz * pl.tc.bn * 4;
              idx[v] = v;
            }
            std::stable_sort(idx.begin(), idx.end(),
                             [&](int64_t x, int64_t y) { return cost[x] > cost[y]; });
            std::vector<std::vector<int>> per((size_t)G);
            std::vector<std::pair<double, int64_t>> heap;  // (load, cta), min first
            for (int64_t b = 0; b < G; ++b) heap.emplace_back(0.0, b);
            auto cmp = [](const std::pair<double, int64_t>& x, const std::pair<double, int64_t>& y) {
              return x.first > y.first || (x.first == y.first && x.second > y.second);
            };
            std::make_heap(heap.begin(), heap.end(), cmp);
            size_t kmax = 0;
            for (int64_t v : idx) {
              std::pop_heap(heap.begin(), heap.end(), cmp);
              auto& top = heap.back();
              per[(size_t)top.second].push_back((int)v);
              kmax = std::max(kmax, per[(size_t)top.second].size());
              top.first += cost[v];
              std::push_heap(heap.begin(), heap.end(), cmp);
            }
            std::vector<int> order(kmax * (size_t)G, -1);
            for (int64_t b = 0; b < G; ++b)
              for (size_t k = 0; k < per[(size_t)b].size(); ++k) order[k * (size_t)G + (size_t)b] = per[(size_t)b][k];
            pl.ft_order.alloc(order.size());
            h2d(pl.ft_order.p, order.data(), order.size(), st);
            TFG_CUDA(cudaStreamSynchronize(st));  // order is a local
          }
          // fused rows address the stage (or D1) directly: no slot lookup per
          // nonzero in the kernel
          std::vector<int64_t> off(f_rows.size() + 1, 0);
          std::vector<uint8_t> rwide(f_rows.size());
          std::vector<int> aoff(f_rows.size());
          for (int64_t v = 0; v < pl.n_ftiles; ++v)
            for (int64_t q = f_joff[v]; q < f_joff[v + 1]; ++q) {
              rwide[q] = wide[v];
              off[q + 1] = off[q] + (arp[f_rows[q] + 1] - arp[f_rows[q]]);
              aoff[q] = (int)(arp[f_rows[q]] - off[q]);
            }
          pl.fx_aoff.alloc(aoff.size());
          h2d(pl.fx_aoff.p, aoff.data(), aoff.size(), st);
          pl.fx_off.alloc(off.size());
          h2d(pl.fx_off.p, off.data(), off.size(), st);
          pl.fx_idx.alloc(std::max<int64_t>(off.back(), 1));
          dbuf<uint8_t> drw(rwide.size());
          h2d(drw.p, rwide.data(), rwide.size(), st);
          k_fused_xidx<<<blocks_for((int64_t)f_rows.size() * 32), 256, 0, st>>>(
              (int64_t)f_rows.size(), pl.ft_jrows.p, pl.fx_off.p, drw.p, pr.d_a_row_ptr,
              pr.d_a_col_idx, pl.slot.p, pl.fx_idx.p);
          TFG_LAUNCH_CHECK();
          TFG_CUDA(cudaStreamSynchronize(st));
        }
        if (getenv("TFG_DEBUG")) {
          int64_t rows = 0, pad128 = 0, slots = 0, small = 0;
          int wmax = 0;
          for (int64_t v = 0; v < pl.n_ftiles; ++v) {
            const int w = f_ihi[v] - f_ilo[v];
            rows += w;
            pad128 += (w + 127) / 128 * 128;
            slots += tc[v];
            small += w < 128;
            wmax = std::max(wmax, w);
          }
          fprintf(stderr,
                  "[tfg] fused tiles %lld rows %lld (pad128 %lld) wmax %d small %lld slots %lld "
                  "fused_rows %lld cap %d wide %lld first_rows(unfused) %zu\n",
                  (long long)pl.n_ftiles, (long long)rows, (long long)pad128, wmax,
                  (long long)small, (long long)slots, (long long)f_rows.size(), cap,
                  (long long)pl.n_wide, fo_rows.size());
        }
      } else {
        // generic fused kernel: column slice = whole cc when the widest tile fits
        int cs = std::min(cc, 128);
        auto need = [&](int w, int c) {
          return (size_t)w * c * pl.elem + (pr.b_is_dense ? (size_t)bc * c * pl.elem : 0);
        };
        while (cs > 32 && need(w_max, cs) > kFusedSmemCap) cs = (cs + 1) / 2;
        const size_t c_bytes = pr.b_is_dense ? (size_t)bc * cs * pl.elem : 0;
        if (c_bytes + (size_t)cs * pl.elem > kFusedSmemCap)
          throw runtime_error("fused executor: C slice does not fit in shared memory");
        int w_cap = (int)std::min<size_t>((size_t)w_max,
                                          (kFusedSmemCap - c_bytes) / ((size_t)cs * pl.elem));
        pl.cs = cs;
        pl.w_cap = std::max(w_cap, 0);
        pl.n_slices = (cc + cs - 1) / cs;
        pl.fused_smem = (size_t)pl.w_cap * cs * pl.elem + c_bytes;
      }
    }
    phase("fused tiles");
    // spill set S = columns of wavefront-1 rows
    TFG_CUDA(cudaMemsetAsync(pl.spill.p, 0, n, st));
    if (nj1) {
      k_mark_spill<<<blocks_for(nj1 * 32), 256, 0, st>>>(nj1, s->j_rows[1].p, pr.d_a_row_ptr,
                                                          pr.d_a_col_idx, pl.spill.p);
      TFG_LAUNCH_CHECK();
    }
    dbuf<unsigned long long> cnt(1);
    TFG_CUDA(cudaMemsetAsync(cnt.p, 0, 8, st));
    k_count_u8<<<256, 256, 0, st>>>(n, pl.spill.p, cnt.p);
    TFG_LAUNCH_CHECK();
    unsigned long long h = 0;
    d2h(&h, cnt.p, 1, st);
    TFG_CUDA(cudaStreamSynchronize(st));
    pl.spill_rows = (int64_t)h;
  }
  if (!s) TFG_CUDA(cudaMemsetAsync(pl.spill.p, 1, n, st));
  phase("spill set");

  // (a) first-op work
  if (pr.b_is_dense) {
    const int BMb = pl.gemm_bm;
    std::vector<int> r0, cnt;
    size_t q = 0;
    while (q < fo_rows.size()) {
      size_t e = q + 1;
      while (e < fo_rows.size() && fo_rows[e] == fo_rows[e - 1] + 1 &&
             (int)(e - q) < BMb)
        ++e;
      r0.push_back(fo_rows[q]);
      cnt.push_back((int)(e - q));
      q = e;
    }
    pl.n_fo_blocks = (int64_t)r0.size();
    pl.fo_r0.alloc(r0.size());
    pl.fo_cnt.alloc(cnt.size());
    h2d(pl.fo_r0.p, r0.data(), r0.size(), st);
    h2d(pl.fo_cnt.p, cnt.data(), cnt.size(), st);
    if (pl.tc.on) {
      std::vector<int> ihi(r0.size());
      for (size_t k = 0; k < r0.size(); ++k) ihi[k] = r0[k] + cnt[k];
      pl.fo_ihi.alloc(ihi.size());
      h2d(pl.fo_ihi.p, ihi.data(), ihi.size(), st);
    }
  } else {
    if (pr.b_cols == n && pr.b_nnz > 0) gB = probe_stencil(n, brp, pr.d_b_row_ptr, pr.d_b_col_idx, st);
    // host column indices only for the band layout (not a grid stencil)
    std::vector<int> bci;
    if (gB.nx == 0 && pr.b_nnz > 0 && pr.b_nnz <= kGroupMaxNnz) {
      bci.resize(pr.b_nnz);
      d2h(bci.data(), pr.d_b_col_idx, bci.size(), st);
      TFG_CUDA(cudaStreamSynchronize(st));
    }
    pl.fo_sparse.build(fo_rows, brp, cc, pl.elem, st, bci.empty() ? nullptr : &bci,
                       stencil_rows(fo_rows, gB, cc, pl.elem));
    attach_stencil(pl.fo_sparse, gB, pr.d_c, cc, pl.elem);
  }
  phase("first-op work");
  // (c) second-op work (wavefront-1 rows, then the empty fused rows)
  if (!zero_rows.empty()) {  // ascending union, O(n) (a sort of millions of rows costs 0.5 s)
    std::vector<uint8_t> in(n, 0);
    for (int r : second_rows) in[r] = 1;
    for (int r : zero_rows) in[r] = 1;
    const size_t total = second_rows.size() + zero_rows.size();
    second_rows.clear();
    second_rows.reserve(total);
    for (int r = 0; r < n; ++r)
      if (in[r]) second_rows.push_back(r);
  }
  {
    // A aliased with B (SpMM-SpMM with B = A): same pattern, same geometry
    const bool same = !pr.b_is_dense && pr.d_a_row_ptr == pr.d_b_row_ptr &&
                      pr.d_a_col_idx == pr.d_b_col_idx && pr.b_cols == n;
    const StencilGeom gA =
        same ? gB : (arp[n] > 0 ? probe_stencil(n, arp, pr.d_a_row_ptr, pr.d_a_col_idx, st)
                                : StencilGeom{});
    phase("wave-1 row union + stencil probe");
    // host column indices only for the band layout: not a stencil, and a
    // list that is not skewed (R-MAT rows never band-stage)
    std::vector<int> aci;
    if (gA.nx == 0 && arp[n] > 0 && arp[n] <= kGroupMaxNnz && band_candidate(second_rows, arp)) {
      aci.resize(arp[n]);
      d2h(aci.data(), pr.d_a_col_idx, aci.size(), st);
      TFG_CUDA(cudaStreamSynchronize(st));
    }
    pl.second.build(second_rows, arp, cc, pl.elem, st, aci.empty() ? nullptr : &aci,
                    stencil_rows(second_rows, gA, cc, pl.elem));
    if (partial) pl.w1_rows = second_rows;
    attach_stencil(pl.second, gA, pl.d1.p, cc, pl.elem);
  }
  phase("wave-1 work");

  // algorithmic bytes per stage: computed on first use (tfg_plan_profile);
  // the drop-in by-value call never needs them
  pl.prof.reset(new PlanProfileCtx{std::move(fo_rows), std::move(second_rows), std::move(arp),
                                   std::move(brp)});
  pl.launches = 0;
  if (pl.tc.on && (pl.n_fo_blocks > 0 || pl.n_ftiles > 0)) pl.launches += 1;  // C split
  if (pr.b_is_dense)
    pl.launches += pl.n_fo_blocks > 0;
  else
    pl.launches += pl.fo_sparse.launches();
  pl.launches += pl.n_ftiles > 0;
  pl.launches += pl.second.launches();
  TFG_CUDA(cudaStreamSynchronize(st));
}

template <class T, int BM, int BN, int BK, int TM, int TN>
static void launch_gemm_v2_cfg(int64_t nblk, const int* r0, const int* cnt, const T* B, int bc,
                               const T* C, int cc, T* D1, cudaStream_t st) {
  using G = GemmCfg<T, BM, BN, BK, TM, TN, 3>;
  auto kern = k_gemm_stream<T, BM, BN, BK, TM, TN, 3>;
  static bool attr = false;
  if (!attr) {
    TFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
    attr = true;
  }
  int per_sm = 1;
  TFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::THREADS, G::SMEM));
  const int64_t gx = std::min<int64_t>(nblk, (int64_t)sm_count() * std::max(per_sm, 1));
  kern<<<dim3((unsigned)gx, cc / BN), G::THREADS, G::SMEM, st>>>(nblk, r0, cnt, B, bc, C, cc, D1,
                                                                 cc);
  TFG_LAUNCH_CHECK();
}

template <class T, int BM, int BN, int BK, int TM, int TN, int LPR>
static void launch_fused_v2_cfg(tfg_plan& pl, T* D1, T* D, cudaStream_t st) {
  const tfg_problem& pr = pl.p;
  auto kern = k_fused_gemm_tiles<T, BM, BN, BK, TM, TN, LPR>;
  TFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pl.fused_smem));
  int per_sm = 1;
  TFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, pl.fused_smem));
  const int64_t gx = std::min<int64_t>(pl.n_ftiles, (int64_t)sm_count() * std::max(per_sm, 1));
  kern<<<dim3((unsigned)gx, pl.n_slices), 256, pl.fused_smem, st>>>(
      pl.n_ftiles, pl.ft_ilo.p, pl.ft_ihi.p, pl.ft_joff.p, pl.ft_jrows.p, pl.ft_wide.p, pl.slot.p,
      static_cast<const T*>(pr.d_b_dense), pr.b_cols, static_cast<const T*>(pr.d_c),
      pr.c_cols, pr.d_a_row_ptr, pr.d_a_col_idx, static_cast<const T*>(pr.d_a_val), pl.spill.p, D1,
      D);
  TFG_LAUNCH_CHECK();
}

template <class T>
static void launch_fused_v2(tfg_plan& pl, T* D1, T* D, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    if (pl.gemm_kind == 2)
      launch_fused_v2_cfg<T, 128, 128, 32, 8, 8, 32>(pl, D1, D, st);
    else
      launch_fused_v2_cfg<T, 128, 64, 32, 8, 4, 16>(pl, D1, D, st);
  } else {
    if (pl.gemm_kind == 2)
      launch_fused_v2_cfg<T, 64, 128, 16, 4, 8, 32>(pl, D1, D, st);
    else
      launch_fused_v2_cfg<T, 64, 64, 16, 4, 4, 32>(pl, D1, D, st);
  }
}

template <class T>
static void launch_gemm_v2(tfg_plan& pl, int64_t nblk, const int* r0, const int* cnt, const T* B,
                           int bc, const T* C, int cc, T* D1, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    if (pl.gemm_kind == 2)
      launch_gemm_v2_cfg<T, 128, 128, 32, 8, 8>(nblk, r0, cnt, B, bc, C, cc, D1, st);
    else
      launch_gemm_v2_cfg<T, 128, 64, 32, 8, 4>(nblk, r0, cnt, B, bc, C, cc, D1, st);
  } else {
    if (pl.gemm_kind == 2)
      launch_gemm_v2_cfg<T, 64, 128, 16, 4, 8>(nblk, r0, cnt, B, bc, C, cc, D1, st);
    else
      launch_gemm_v2_cfg<T, 64, 64, 16, 8, 4>(nblk, r0, cnt, B, bc, C, cc, D1, st);
  }
}

// Dense first op D1[rows] = B[rows] C over row blocks (r0, cnt; ihi = r0 +
// cnt for the tensor-core kernel): the plan's first-op kernel on any block
// list (the plan's own, or a multi-GPU halo recomputed locally).
template <class T>
static void first_op_blocks(tfg_plan& pl, int64_t nblk, const int* r0, const int* cnt,
                            const int* ihi, T* D1, cudaStream_t st) {
  const tfg_problem& pr = pl.p;
  const int cc = pr.c_cols, bc = pr.b_cols;
  const T* C = static_cast<const T*>(pr.d_c);
  if (!nblk) return;
  if (pl.tc.on) {
    if constexpr (sizeof(T) == 4)
      tc_run(pl.tc, pr.n, bc, cc, nblk, r0, ihi, nullptr, nullptr, nullptr, nullptr, nullptr,
             nullptr, nullptr, nullptr, nullptr, reinterpret_cast<float*>(D1), nullptr, st);
  } else if (pl.gemm_kind) {
    launch_gemm_v2<T>(pl, nblk, r0, cnt, static_cast<const T*>(pr.d_b_dense), bc, C, cc, D1, st);
  } else {
    const int gy = (cc + kGemmBN - 1) / kGemmBN;
    const int64_t gx = std::min<int64_t>(nblk, (int64_t)sm_count() * 16);
    k_gemm_blocks<T, kGemmBM, kGemmBN, kGemmBK, kGemmTM, kGemmTN>
        <<<dim3((unsigned)gx, gy), (kGemmBM / kGemmTM) * (kGemmBN / kGemmTN), 0, st>>>(
            nblk, r0, cnt, static_cast<const T*>(pr.d_b_dense), bc, C, cc, D1, cc);
    TFG_LAUNCH_CHECK();
  }
}

template <class T>
static void plan_execute_t(tfg_plan& pl, T* D, cudaStream_t st, cudaEvent_t* ev = nullptr,
                           int part = -1) {
  const tfg_problem& pr = pl.p;
  const int cc = pr.c_cols, bc = pr.b_cols;
  T* D1 = reinterpret_cast<T*>(pl.d1.p);
  const T* C = static_cast<const T*>(pr.d_c);
  bool empty_done = false;
  if (part == 1) goto wave1;
  if (pl.zero_d) TFG_CUDA(cudaMemsetAsync(D, 0, (size_t)pr.n * cc * sizeof(T), st));
  if (ev) TFG_CUDA(cudaEventRecord(ev[0], st));
  // D rows of empty wavefront-1 rows: written beside the first op (its kernels
  // leave HBM write bandwidth idle), not in front of the wavefront-1 gathers
  if (part == -1 && spmm_can_zero_early(pl.second)) {
    spmm_zero_early<T>(pl.second, cc, D, st);
    empty_done = true;
  }
  // (a)
  if constexpr (sizeof(T) == 4) {
    if (pl.tc.on && (pl.n_fo_blocks || pl.n_ftiles))
      tc_prep_c(pl.tc, reinterpret_cast<const float*>(C), bc, cc, st);
  }
  if (pr.b_is_dense) {
    first_op_blocks<T>(pl, pl.n_fo_blocks, pl.fo_r0.p, pl.fo_cnt.p, pl.fo_ihi.p, D1, st);
  } else {
    spmm_run<T>(pl.fo_sparse, pr.d_b_row_ptr, pr.d_b_col_idx,
                static_cast<const T*>(pr.d_b_val), C, cc, D1, st);
  }
  if (ev) TFG_CUDA(cudaEventRecord(ev[1], st));
  // (b)
  if (pl.n_ftiles && pl.fused_v2 && pl.tc.on) {
    if constexpr (sizeof(T) == 4)
      tc_run(pl.tc, pr.n, bc, cc, pl.n_ftiles, pl.ft_ilo.p, pl.ft_ihi.p, pl.ft_joff.p,
             pl.ft_jrows.p, pl.ft_wide.p, pl.slot.p, pl.spill.p, pl.fx_aoff.p, pl.fx_off.p,
             pl.fx_idx.p, static_cast<const float*>(pr.d_a_val), reinterpret_cast<float*>(D1),
             reinterpret_cast<float*>(D), st, pl.ft_order.p, (int64_t)pl.ft_order.n);
  } else if (pl.n_ftiles && pl.fused_v2) {
    launch_fused_v2<T>(pl, D1, D, st);
  } else if (pl.n_ftiles) {
    if (pl.fused_smem > 48 * 1024)
      TFG_CUDA(cudaFuncSetAttribute(k_fused_tiles<T>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)pl.fused_smem));
    const int64_t gx = std::min<int64_t>(pl.n_ftiles, 65535);
    k_fused_tiles<T><<<dim3((unsigned)gx, pl.n_slices), 256, pl.fused_smem, st>>>(
        pl.n_ftiles, pl.ft_ilo.p, pl.ft_ihi.p, pl.ft_joff.p, pl.ft_jrows.p, pl.w_cap,
        pl.cs, cc, pr.b_is_dense, static_cast<const T*>(pr.d_b_dense), bc, pr.d_b_row_ptr,
        pr.d_b_col_idx, static_cast<const T*>(pr.d_b_val), C, pr.d_a_row_ptr,
        pr.d_a_col_idx, static_cast<const T*>(pr.d_a_val), pl.spill.p, D1, D);
    TFG_LAUNCH_CHECK();
  }
  if (ev) TFG_CUDA(cudaEventRecord(ev[2], st));
  if (part == 0) return;
wave1:
  // (c)
  spmm_run<T>(pl.second, pr.d_a_row_ptr, pr.d_a_col_idx,
              static_cast<const T*>(pr.d_a_val), D1, cc, D, st, empty_done);
  if (ev) TFG_CUDA(cudaEventRecord(ev[3], st));
}

void plan_execute(tfg_plan& pl, void* d, cudaStream_t st, cudaEvent_t* ev = nullptr) {
  if (pl.p.dtype == TFG_F64)
    plan_execute_t<double>(pl, static_cast<double*>(d), st, ev);
  else
    plan_execute_t<float>(pl, static_cast<float*>(d), st, ev);
}

// part 0: wavefront 0 (first op + fused tiles); part 1: wavefront-1 SpMM.
// The multi-GPU driver runs the D1 halo exchange between the two.
void plan_execute_part(tfg_plan& pl, void* d, cudaStream_t st, int part) {
  if (pl.p.dtype == TFG_F64)
    plan_execute_t<double>(pl, static_cast<double*>(d), st, nullptr, part);
  else
    plan_execute_t<float>(pl, static_cast<float*>(d), st, nullptr, part);
}

void gather_rows(int dtype, const void* src, int cols, const int* rows, int64_t n,
                 void* dst, cudaStream_t st) {
  if (n == 0) return;
  const int g = (int)std::min<int64_t>((n * cols + 255) / 256, (int64_t)sm_count() * 16);
  if (dtype == TFG_F64)
    k_gather_rows<double><<<g, 256, 0, st>>>(static_cast<const double*>(src), cols, rows, n,
                                             static_cast<double*>(dst));
  else
    k_gather_rows<float><<<g, 256, 0, st>>>(static_cast<const float*>(src), cols, rows, n,
                                            static_cast<float*>(dst));
  TFG_LAUNCH_CHECK();
}

void scatter_rows(int dtype, const void* src, int cols, const int* rows, int64_t n,
                  void* dst, cudaStream_t st) {
  if (n == 0) return;
  const int g = (int)std::min<int64_t>((n * cols + 255) / 256, (int64_t)sm_count() * 16);
  if (dtype == TFG_F64)
    k_scatter_rows<double><<<g, 256, 0, st>>>(static_cast<const double*>(src), cols, rows, n,
                                              static_cast<double*>(dst));
  else
    k_scatter_rows<float><<<g, 256, 0, st>>>(static_cast<const float*>(src), cols, rows, n,
                                             static_cast<float*>(dst));
  TFG_LAUNCH_CHECK();
}

size_t plan_scratch_bytes(const tfg_plan& pl) {
  return pl.d1.bytes() + pl.spill.bytes() + pl.fo_r0.bytes() + pl.fo_cnt.bytes() +
         pl.fo_sparse.bytes() + pl.ft_ilo.bytes() + pl.ft_ihi.bytes() + pl.ft_joff.bytes() +
         pl.ft_jrows.bytes() + pl.second.bytes();
}


// ---------------------------------------------------------------------------
// Multi-GPU row-block partition: cuts, halo, one step.
// ---------------------------------------------------------------------------

// Row-block cuts at wavefront-0 tile starts, balanced by estimated bytes per
// row: the first op (B row + D1 row) plus the second op (A row + one gathered
// D1 row per nonzero + D row) -- the wavefront-1 gathers dominate skewed
// matrices, so equal row counts would not balance them.
void partition_bounds(const tfg_schedule& s, const int* rp, int bc, int cc, size_t elem,
                      bool b_dense, int world, int* bounds) {
  const int n = s.n;
  std::vector<int> ilo(s.n_tiles[0]);
  d2h(ilo.data(), s.i_lo[0].p, ilo.size(), nullptr);
  TFG_CUDA(cudaStreamSynchronize(nullptr));
  std::sort(ilo.begin(), ilo.end());
  if (ilo.empty() || ilo[0] != 0) ilo.insert(ilo.begin(), 0);
  std::vector<double> P(n + 1, 0.0);
  const double e = (double)elem;
  for (int i = 0; i < n; ++i) {
    const double nnz = rp[i + 1] - rp[i];
    const double first = b_dense ? (double)bc * e + cc * e : nnz * (4 + e) + cc * e;
    const double second = nnz * (4 + e + cc * e) + cc * e;
    P[i + 1] = P[i] + first + second;
  }
  bounds[0] = 0;
  for (int k = 1; k < world; ++k) {
    const double target = P[n] * k / world;
    const int row = (int)(std::lower_bound(P.begin(), P.end(), target) - P.begin());
    auto it = std::lower_bound(ilo.begin(), ilo.end(), row);
    int c = it == ilo.end() ? ilo.back() : *it;
    if (it != ilo.begin()) {
      const int prev = *(it - 1);
      if (it == ilo.end() || std::fabs(P[prev] - target) < std::fabs(P[c] - target)) c = prev;
    }
    bounds[k] = std::max(c, bounds[k - 1]);
  }
  bounds[world] = n;
}

void halo_create(tfg_plan& pl, const tfg_schedule& s, const int* bounds, int world, int rank,
                 int mode, tfg_halo& h, cudaStream_t st) {
  const tfg_problem& pr = pl.p;
  const int n = pr.n, cc = pr.c_cols;
  if (world < 1 || world > 32 || rank < 0 || rank >= world)
    throw invalid_argument("halo: world must be in [1, 32] and rank in [0, world)");
  if (bounds[0] != 0 || bounds[world] != n) throw invalid_argument("halo: bounds must span [0, n]");
  for (int q = 0; q < world; ++q)
    if (bounds[q] > bounds[q + 1]) throw invalid_argument("halo: bounds must be ascending");
  if (bounds[rank] != pl.row_lo || bounds[rank + 1] != pl.row_hi)
    throw invalid_argument("halo: the plan is not this rank's partition plan");
  if (mode == TFG_HALO_RECOMPUTE && !pr.b_is_dense)
    throw invalid_argument("halo: recompute needs a dense B (GeMM-SpMM)");
  h.world = world;
  h.rank = rank;
  const int lo = pl.row_lo, hi = pl.row_hi;
  // readers of every D1 row, from every rank's wavefront-1 rows
  dbuf<int> bd(world + 1);
  h2d(bd.p, bounds, world + 1, st);
  dbuf<unsigned> mask(n);
  TFG_CUDA(cudaMemsetAsync(mask.p, 0, (size_t)n * 4, st));
  const int64_t nj1 = s.n_jrows[1];
  if (nj1) {
    k_mark_readers<<<blocks_for(nj1 * 32), 256, 0, st>>>(nj1, s.j_rows[1].p, pr.d_a_row_ptr,
                                                          pr.d_a_col_idx, bd.p, world, mask.p);
    TFG_LAUNCH_CHECK();
  }
  std::vector<unsigned> m(n);
  d2h(m.data(), mask.p, n, st);
  TFG_CUDA(cudaStreamSynchronize(st));
  std::vector<int> recv, send;
  h.recv_off.assign(1, 0);
  h.send_off.assign(1, 0);
  for (int q = 0; q < world; ++q) {
    if (q != rank)
      for (int i = bounds[q]; i < bounds[q + 1]; ++i)
        if (m[i] >> rank & 1u) recv.push_back(i);
    h.recv_off.push_back((int64_t)recv.size());
    if (q != rank)
      for (int i = lo; i < hi; ++i)
        if (m[i] >> q & 1u) send.push_back(i);
    h.send_off.push_back((int64_t)send.size());
  }
  h.n_recv = (int64_t)recv.size();
  h.n_send = (int64_t)send.size();
  const size_t rb = (size_t)cc * pl.elem;
  // cost model: NVLink transfer of the halo rows vs recomputing them from
  // the locally resident B rows (B row read + D1 row write at HBM speed)
  const double nvlink = 700e9, hbm = 6500e9;
  h.t_exchange_us = (double)h.n_recv * rb / nvlink * 1e6;
  h.t_recompute_us = pr.b_is_dense ? (double)h.n_recv * ((double)pr.b_cols * pl.elem + rb) / hbm * 1e6 : 1e300;
  h.mode = mode == TFG_HALO_AUTO ? (pr.b_is_dense && h.t_recompute_us < h.t_exchange_us
                                        ? TFG_HALO_RECOMPUTE : TFG_HALO_EXCHANGE)
                                 : mode;
  h.recv_rows.alloc(std::max<int64_t>(h.n_recv, 1));
  h2d(h.recv_rows.p, recv.data(), recv.size(), st);
  h.send_rows.alloc(std::max<int64_t>(h.n_send, 1));
  h2d(h.send_rows.p, send.data(), send.size(), st);
  if (h.mode == TFG_HALO_RECOMPUTE) {
    std::vector<int> r0, cnt, ihi;
    for (size_t q = 0; q < recv.size();) {
      size_t e = q + 1;
      while (e < recv.size() && recv[e] == recv[e - 1] + 1 && (int)(e - q) < pl.gemm_bm) ++e;
      r0.push_back(recv[q]);
      cnt.push_back((int)(e - q));
      ihi.push_back(recv[q] + (int)(e - q));
      q = e;
    }
    h.n_rblk = (int64_t)r0.size();
    h.r_r0.alloc(std::max<size_t>(r0.size(), 1));
    h.r_cnt.alloc(std::max<size_t>(r0.size(), 1));
    h.r_ihi.alloc(std::max<size_t>(r0.size(), 1));
    h2d(h.r_r0.p, r0.data(), r0.size(), st);
    h2d(h.r_cnt.p, cnt.data(), cnt.size(), st);
    h2d(h.r_ihi.p, ihi.data(), ihi.size(), st);
  } else {
    h.recv_buf.alloc(std::max<size_t>((size_t)h.n_recv * rb, 16));
    h.send_buf.alloc(std::max<size_t>((size_t)h.n_send * rb, 16));
    TFG_CUDA(cudaStreamCreateWithFlags(&h.comm, cudaStreamNonBlocking));
    TFG_CUDA(cudaEventCreateWithFlags(&h.ev_packed, cudaEventDisableTiming));
    TFG_CUDA(cudaEventCreateWithFlags(&h.ev_recv, cudaEventDisableTiming));
    // wavefront-1 rows that read only local D1 overlap the exchange (row-list
    // kernels; a grid-stencil slab keeps its one plane-streaming pass)
    if (!pl.second.stencil && !pl.w1_rows.empty() && h.n_recv > 0) {
      const int64_t nr = (int64_t)pl.w1_rows.size();
      dbuf<int> rows(nr);
      h2d(rows.p, pl.w1_rows.data(), nr, st);
      dbuf<uint8_t> flag(nr);
      k_reads_remote<<<blocks_for(nr * 32), 256, 0, st>>>(nr, rows.p, pr.d_a_row_ptr,
                                                           pr.d_a_col_idx, lo, hi, flag.p);
      TFG_LAUNCH_CHECK();
      std::vector<uint8_t> f(nr);
      d2h(f.data(), flag.p, nr, st);
      std::vector<int> arp(n + 1);
      d2h(arp.data(), pr.d_a_row_ptr, n + 1, st);
      TFG_CUDA(cudaStreamSynchronize(st));
      std::vector<int> in_rows, bd_rows;
      for (int64_t q = 0; q < nr; ++q) (f[q] ? bd_rows : in_rows).push_back(pl.w1_rows[q]);
      h.interior.exact = h.boundary.exact = pl.second.exact;
      h.interior.build(in_rows, arp, cc, pl.elem, st);
      h.boundary.build(bd_rows, arp, cc, pl.elem, st);
      h.split = true;
    }
  }
  TFG_CUDA(cudaStreamSynchronize(st));
}

// The step in phases (execute_dist runs them in order with NCCL between
// 0 and 2; the single-GPU emulation moves the buffers itself).
// phase 0: wavefront 0, then pack the rows peers need (or recompute the halo)
template <class T>
static void dist_phase0(tfg_plan& pl, tfg_halo& h, T* D, cudaStream_t st) {
  const int cc = pl.p.c_cols;
  T* D1 = reinterpret_cast<T*>(pl.d1.p);
  plan_execute_t<T>(pl, D, st, nullptr, 0);  // no communication
  if (h.mode == TFG_HALO_RECOMPUTE) {  // the halo's D1 rows from the resident B rows
    first_op_blocks<T>(pl, h.n_rblk, h.r_r0.p, h.r_cnt.p, h.r_ihi.p, D1, st);
    return;
  }
  if (h.n_send) {
    k_gather_rows<T><<<blocks_for(h.n_send * cc), 256, 0, st>>>(
        D1, cc, h.send_rows.p, h.n_send, reinterpret_cast<T*>(h.send_buf.p));
    TFG_LAUNCH_CHECK();
  }
}
// phase 2: the wavefront-1 rows that read only local D1 (while the halo moves)
template <class T>
static void dist_phase2(tfg_plan& pl, tfg_halo& h, T* D, cudaStream_t st) {
  const tfg_problem& pr = pl.p;
  if (h.mode == TFG_HALO_EXCHANGE && h.split)
    spmm_run<T>(h.interior, pr.d_a_row_ptr, pr.d_a_col_idx, static_cast<const T*>(pr.d_a_val),
                reinterpret_cast<const T*>(pl.d1.p), pr.c_cols, D, st);
}
// phase 3: unpack the received rows, then the rest of wavefront 1
template <class T>
static void dist_phase3(tfg_plan& pl, tfg_halo& h, T* D, cudaStream_t st) {
  const tfg_problem& pr = pl.p;
  const int cc = pr.c_cols;
  T* D1 = reinterpret_cast<T*>(pl.d1.p);
  if (h.mode == TFG_HALO_EXCHANGE && h.n_recv) {
    k_scatter_rows<T><<<blocks_for(h.n_recv * cc), 256, 0, st>>>(
        reinterpret_cast<const T*>(h.recv_buf.p), cc, h.recv_rows.p, h.n_recv, D1);
    TFG_LAUNCH_CHECK();
  }
  if (h.mode == TFG_HALO_EXCHANGE && h.split)
    spmm_run<T>(h.boundary, pr.d_a_row_ptr, pr.d_a_col_idx, static_cast<const T*>(pr.d_a_val),
                D1, cc, D, st);
  else
    plan_execute_t<T>(pl, D, st, nullptr, 1);
}

template <class T>
static void execute_dist_t(tfg_plan& pl, tfg_halo& h, void* comm, T* D, cudaStream_t st) {
  const int cc = pl.p.c_cols;
  dist_phase0<T>(pl, h, D, st);
  const bool xfer = h.mode == TFG_HALO_EXCHANGE && h.world > 1 && (h.n_recv || h.n_send);
  if (xfer) {
    if (!comm) throw invalid_argument("plan_execute_dist: exchange needs an NCCL communicator");
    const ncclDataType_t dt = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
    TFG_CUDA(cudaEventRecord(h.ev_packed, st));
    TFG_CUDA(cudaStreamWaitEvent(h.comm, h.ev_packed, 0));
    const NcclApi& nc = nccl();
    auto* c = static_cast<ncclComm_t>(comm);
    nccl_check(nc.GroupStart(), "ncclGroupStart");
    for (int q = 0; q < h.world; ++q) {
      const int64_t ns = h.send_off[q + 1] - h.send_off[q], nr = h.recv_off[q + 1] - h.recv_off[q];
      if (ns)
        nccl_check(nc.Send(reinterpret_cast<T*>(h.send_buf.p) + h.send_off[q] * cc, (size_t)ns * cc,
                           dt, q, c, h.comm), "ncclSend");
      if (nr)
        nccl_check(nc.Recv(reinterpret_cast<T*>(h.recv_buf.p) + h.recv_off[q] * cc, (size_t)nr * cc,
                           dt, q, c, h.comm), "ncclRecv");
    }
    nccl_check(nc.GroupEnd(), "ncclGroupEnd");
    TFG_CUDA(cudaEventRecord(h.ev_recv, h.comm));
  }
  dist_phase2<T>(pl, h, D, st);  // overlaps the NCCL transfer
  if (xfer) TFG_CUDA(cudaStreamWaitEvent(st, h.ev_recv, 0));
  dist_phase3<T>(pl, h, D, st);
}

// All ranks of a partitioned step on ONE GPU, one after another, the NCCL
// transfer replaced by device copies between the ranks' halo buffers (every
// rank's memory is local): checks cuts, halo lists and the split without a
// second GPU.  No kernel waits on another.
template <class T>
static void execute_dist_emulated_t(tfg_plan** pls, tfg_halo** hs, int world, void** ds,
                                    cudaStream_t st) {
  for (int r = 0; r < world; ++r) dist_phase0<T>(*pls[r], *hs[r], static_cast<T*>(ds[r]), st);
  for (int r = 0; r < world; ++r) {
    tfg_halo& h = *hs[r];
    if (h.mode != TFG_HALO_EXCHANGE) continue;
    const size_t rb = (size_t)pls[r]->p.c_cols * sizeof(T);
    for (int q = 0; q < world; ++q) {  // rows r receives from q = rows q sends to r
      const tfg_halo& g = *hs[q];
      const int64_t nr = h.recv_off[q + 1] - h.recv_off[q];
      if (nr != g.send_off[r + 1] - g.send_off[r])
        throw runtime_error("halo emulation: send / recv lists of a rank pair disagree");
      if (nr)
        TFG_CUDA(cudaMemcpyAsync(h.recv_buf.p + h.recv_off[q] * rb, g.send_buf.p + g.send_off[r] * rb,
                                 (size_t)nr * rb, cudaMemcpyDeviceToDevice, st));
    }
  }
  for (int r = 0; r < world; ++r) {
    dist_phase2<T>(*pls[r], *hs[r], static_cast<T*>(ds[r]), st);
    dist_phase3<T>(*pls[r], *hs[r], static_cast<T*>(ds[r]), st);
  }
}

void execute_dist(tfg_plan& pl, tfg_halo& h, void* comm, void* d, cudaStream_t st) {
  if (pl.p.dtype == TFG_F64)
    execute_dist_t<double>(pl, h, comm, static_cast<double*>(d), st);
  else
    execute_dist_t<float>(pl, h, comm, static_cast<float*>(d), st);
}

void execute_dist_emulated(tfg_plan** pls, tfg_halo** hs, int world, void** ds, cudaStream_t st) {
  if (pls[0]->p.dtype == TFG_F64)
    execute_dist_emulated_t<double>(pls, hs, world, ds, st);
  else
    execute_dist_emulated_t<float>(pls, hs, world, ds, st);
}

}  // namespace tfg

// ===========================================================================
// C-ABI: plans (include/tfg.h)
// ===========================================================================
using namespace tfg;

extern "C" {

tfg_status tfg_plan_create(const tfg_problem* p, const tfg_schedule* s, void* stream,
                           tfg_plan** out) {
  return guard([&] {
    *out = nullptr;
    if (!p) throw invalid_argument("plan_create: null problem");
    auto* pl = new tfg_plan;
    try {
      plan_create(*p, s, as_stream(stream), *pl);
    } catch (...) {
      delete pl;
      throw;
    }
    *out = pl;
  });
}

tfg_status tfg_plan_create_ex(const tfg_problem* p, const tfg_schedule* s, uint32_t flags,
                              int32_t row_lo, int32_t row_hi, void* stream, tfg_plan** out) {
  return guard([&] {
    *out = nullptr;
    if (!p) throw invalid_argument("plan_create: null problem");
    if (flags & ~(uint32_t)TFG_PLAN_REFERENCE_BITS) throw invalid_argument("plan_create: unknown flags");
    auto* pl = new tfg_plan;
    try {
      plan_create(*p, s, as_stream(stream), *pl, row_lo, row_hi < 0 ? -1 : row_hi, flags);
    } catch (...) {
      delete pl;
      throw;
    }
    *out = pl;
  });
}

tfg_status tfg_plan_create_partition(const tfg_problem* p, const tfg_schedule* s,
                                     int32_t row_lo, int32_t row_hi, void* stream,
                                     tfg_plan** out) {
  return guard([&] {
    *out = nullptr;
    if (!p) throw invalid_argument("plan_create: null problem");
    auto* pl = new tfg_plan;
    try {
      plan_create(*p, s, as_stream(stream), *pl, row_lo, row_hi);
    } catch (...) {
      delete pl;
      throw;
    }
    *out = pl;
  });
}

tfg_status tfg_partition_bounds(const tfg_schedule* s, const int32_t* h_row_ptr, int32_t b_cols,
                                int32_t c_cols, int32_t dtype, int32_t b_is_dense, int32_t world,
                                int32_t* h_bounds) {
  return guard([&] {
    if (!s || !h_row_ptr || !h_bounds || world < 1)
      throw invalid_argument("partition_bounds: bad arguments");
    partition_bounds(*s, h_row_ptr, b_cols, c_cols, dtype == TFG_F64 ? 8 : 4, b_is_dense != 0,
                     world, h_bounds);
  });
}

tfg_status tfg_halo_create(tfg_plan* pl, const tfg_schedule* s, const int32_t* h_bounds,
                           int32_t world, int32_t rank, int32_t mode, void* stream,
                           tfg_halo** out) {
  return guard([&] {
    *out = nullptr;
    if (!pl || !s || !h_bounds) throw invalid_argument("halo_create: null argument");
    if (mode < TFG_HALO_AUTO || mode > TFG_HALO_RECOMPUTE) throw invalid_argument("halo_create: bad mode");
    auto* h = new tfg_halo;
    try {
      halo_create(*pl, *s, h_bounds, world, rank, mode, *h, as_stream(stream));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

tfg_status tfg_halo_info(const tfg_halo* h, int32_t* mode, int64_t* recv_rows, int64_t* send_rows,
                         double* t_exchange_us, double* t_recompute_us) {
  return guard([&] {
    if (!h) throw invalid_argument("halo_info: null halo");
    if (mode) *mode = h->mode;
    if (recv_rows) *recv_rows = h->n_recv;
    if (send_rows) *send_rows = h->n_send;
    if (t_exchange_us) *t_exchange_us = h->t_exchange_us;
    if (t_recompute_us) *t_recompute_us = h->t_recompute_us;
  });
}

void tfg_halo_destroy(tfg_halo* h) { delete h; }

tfg_status tfg_plan_execute_dist_emulated(tfg_plan** plans, tfg_halo** halos, int32_t world,
                                          void** d, void* stream) {
  return guard([&] {
    if (!plans || !halos || !d || world < 1) throw invalid_argument("execute_dist_emulated: bad arguments");
    for (int r = 0; r < world; ++r) {
      if (!plans[r] || !halos[r] || !d[r]) throw invalid_argument("execute_dist_emulated: null entry");
      if (halos[r]->world != world || halos[r]->rank != r)
        throw invalid_argument("execute_dist_emulated: halos must be ranks 0..world-1 of one partition");
    }
    execute_dist_emulated(plans, halos, world, d, as_stream(stream));
  });
}

tfg_status tfg_plan_execute_dist(tfg_plan* pl, tfg_halo* h, void* nccl_comm, void* d, void* stream) {
  return guard([&] {
    if (!pl || !h || !d) throw invalid_argument("plan_execute_dist: null argument");
    if ((uintptr_t)d % 16 != 0) throw invalid_argument("plan_execute: D must be 16-byte aligned");
    execute_dist(*pl, *h, nccl_comm, d, as_stream(stream));
  });
}

tfg_status tfg_plan_d1(const tfg_plan* pl, void** d1) {
  return guard([&] {
    if (!pl) throw invalid_argument("plan_d1: null plan");
    *d1 = pl->d1.p;
  });
}

tfg_status tfg_plan_execute_stage(tfg_plan* pl, int32_t stage, void* d, void* stream) {
  return guard([&] {
    if (!pl || !d) throw invalid_argument("plan_execute_stage: null plan or output");
    if (stage < 0 || stage > 1) throw invalid_argument("plan_execute_stage: stage 0 or 1");
    if ((uintptr_t)d % 16 != 0) throw invalid_argument("plan_execute: D must be 16-byte aligned");
    plan_execute_part(*pl, d, as_stream(stream), stage);
  });
}

tfg_status tfg_plan_execute(tfg_plan* pl, void* d, void* stream) {
  return guard([&] {
    if (!pl || !d) throw invalid_argument("plan_execute: null plan or output");
    if ((uintptr_t)d % 16 != 0) throw invalid_argument("plan_execute: D must be 16-byte aligned");
    plan_execute(*pl, d, as_stream(stream));
  });
}

tfg_status tfg_plan_stats(const tfg_plan* pl, int64_t* fr, int64_t* sr, int64_t* nnz) {
  return guard([&] {
    if (!pl) throw invalid_argument("plan_stats: null plan");
    if (fr) *fr = pl->first_rows;
    if (sr) *sr = pl->second_rows;
    if (nnz) *nnz = pl->nnz_processed;
  });
}

tfg_status tfg_plan_info(const tfg_plan* pl, int64_t* spill_rows, int64_t* fused_rows,
                         int32_t* launches, int64_t* scratch_bytes) {
  return guard([&] {
    if (!pl) throw invalid_argument("plan_info: null plan");
    if (spill_rows) *spill_rows = pl->spill_rows;
    if (fused_rows) *fused_rows = pl->fused_rows;
    if (launches) *launches = pl->launches + (pl->zero_d ? 1 : 0);
    if (scratch_bytes) *scratch_bytes = (int64_t)plan_scratch_bytes(*pl);
  });
}

tfg_status tfg_plan_kernels(const tfg_plan* pl, char* buf, int32_t len) {
  return guard([&] {
    if (!pl || !buf || len < 1) throw invalid_argument("plan_kernels: null plan or buffer");
    auto spmm_kind = [](const SpmmWork& w) -> std::string {
      if (w.n_short == 0 && w.n_long == 0 && !w.n_empty) return "none";
      std::string k;
      if (w.stencil)
        k = w.stencil->g.d3 ? "stencil3d" : "stencil2d";
      else if (w.banded)
        k = w.dia ? "band-dia" : "band";
      else
        k = w.skewed ? "strip-skewed" : "strip";
      if (w.n_long) k += "+segments";
      return k;
    };
    std::string fo;
    if (pl->p.b_is_dense)
      fo = pl->n_fo_blocks == 0 ? "none" : (pl->tc.on ? "tcgen05" : (pl->gemm_kind ? "gemm-v2" : "gemm"));
    else
      fo = spmm_kind(pl->fo_sparse);
    std::string fu = pl->n_ftiles == 0 ? "none"
                     : (pl->fused_v2 ? (pl->tc.on ? "tcgen05-tiles" : "gemm-tiles") : "tiles");
    std::string w1 = spmm_kind(pl->second);
    const std::string s = "first_op=" + fo + " fused=" + fu + " wave1=" + w1;
    const size_t n = std::min(s.size(), (size_t)len - 1);
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  });
}

void tfg_plan_destroy(tfg_plan* pl) { delete pl; }

tfg_status tfg_plan_profile(tfg_plan* pl, void* d, void* stream, double stage_ms[3],
                            int64_t stage_bytes[3]) {
  return guard([&] {
    if (!pl || !d) throw invalid_argument("plan_profile: null plan or output");
    cudaStream_t st = as_stream(stream);
    compute_stage_bytes(*pl, st);
    cudaEvent_t ev[4];
    for (auto& e : ev) TFG_CUDA(cudaEventCreate(&e));
    plan_execute(*pl, d, st, ev);
    TFG_CUDA(cudaEventSynchronize(ev[3]));
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      TFG_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
      if (stage_ms) stage_ms[k] = ms;
      if (stage_bytes) stage_bytes[k] = pl->stage_bytes[k];
    }
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

tfg_status tfg_run_host(const tfg_problem* hp, const tfg_schedule* s, void* h_d) {
  return guard([&] {
    if (!hp) throw invalid_argument("run_host: null problem");
    const tfg_problem& h = *hp;
    if (h.n < 1) throw invalid_argument("problem: A must be square");
    const size_t el = h.dtype == TFG_F64 ? 8 : 4;
    // The plan needs only the patterns (A's, and a sparse B's) on the device:
    // row pointers and column indices go first, alone on the link; then the
    // values, B and C stream in on a second stream, issued from a second host
    // thread (so a pageable, hence synchronous, copy overlaps too), while the
    // plan is built; execution waits for both.
    cudaStream_t sa = nullptr, sb = nullptr;
    TFG_CUDA(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
    TFG_CUDA(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    struct Streams {
      cudaStream_t a, b;
      ~Streams() {
        cudaStreamSynchronize(a);
        cudaStreamDestroy(a);
        cudaStreamDestroy(b);
      }
    } streams{sa, sb};
    AllocScope scope(sa);  // the inputs and D: stream-ordered, pooled across calls
    const int64_t annz = h.d_a_row_ptr[h.n];
    dbuf<int32_t> arp(h.n + 1), aci(std::max<int64_t>(annz, 1));
    dbuf<unsigned char> av(std::max<int64_t>(annz, 1) * el);
    dbuf<int32_t> brp, bci;
    dbuf<unsigned char> bv, bd, c;
    tfg_problem d = h;
    d.a_nnz = annz;
    d.d_a_row_ptr = arp.p;
    d.d_a_col_idx = aci.p;
    d.d_a_val = av.p;
    c.alloc((size_t)std::max(h.c_rows, 1) * std::max(h.c_cols, 1) * el);
    d.d_c = c.p;
    if (h.b_is_dense) {
      bd.alloc((size_t)std::max(h.b_rows, 1) * std::max(h.b_cols, 1) * el);
      d.d_b_dense = bd.p;
    }
    const bool b_is_a = !h.b_is_dense && h.d_b_row_ptr == h.d_a_row_ptr &&
                        h.d_b_col_idx == h.d_a_col_idx && h.d_b_val == h.d_a_val &&
                        h.b_rows == h.n;  // B is A: upload once
    int64_t bnnz = 0;
    if (!h.b_is_dense) {
      if (b_is_a) {
        d.b_nnz = annz;
        d.d_b_row_ptr = arp.p;
        d.d_b_col_idx = aci.p;
        d.d_b_val = av.p;
      } else {
        bnnz = h.d_b_row_ptr[h.b_rows];
        brp.alloc(h.b_rows + 1);
        bci.alloc(std::max<int64_t>(bnnz, 1));
        bv.alloc(std::max<int64_t>(bnnz, 1) * el);
        d.b_nnz = bnnz;
        d.d_b_row_ptr = brp.p;
        d.d_b_col_idx = bci.p;
        d.d_b_val = bv.p;
      }
    }
    int dev = 0;
    TFG_CUDA(cudaGetDevice(&dev));
    // patterns first (sa), then everything else (sb) once they are through
    h2d(arp.p, h.d_a_row_ptr, h.n + 1, sa);
    h2d(aci.p, h.d_a_col_idx, annz, sa);
    if (!h.b_is_dense && !b_is_a) {
      h2d(brp.p, h.d_b_row_ptr, h.b_rows + 1, sa);
      h2d(bci.p, h.d_b_col_idx, bnnz, sa);
    }
    cudaEvent_t patterns = nullptr;  // allocations made and patterns uploaded, in sa's order
    TFG_CUDA(cudaEventCreateWithFlags(&patterns, cudaEventDisableTiming));
    struct Ev {
      cudaEvent_t e;
      ~Ev() { cudaEventDestroy(e); }
    } ev{patterns};
    TFG_CUDA(cudaEventRecord(patterns, sa));
    cudaError_t berr = cudaSuccess;
    // in pieces, at most two queued at a time: the copy engine serves copies
    // in submission order, so the plan's own small uploads (work lists, on
    // sa) wait for two pieces instead of for the whole of B
    cudaEvent_t piece_ev[2] = {nullptr, nullptr};
    for (auto& e : piece_ev) TFG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct PieceEv {
      cudaEvent_t* e;
      ~PieceEv() {
        cudaEventDestroy(e[0]);
        cudaEventDestroy(e[1]);
      }
    } piece_guard{piece_ev};
    size_t piece_no = 0;
    auto upload = [&](void* dst, const void* src, size_t bytes) {
      constexpr size_t kPiece = (size_t)16 << 20;
      for (size_t o = 0; o < bytes && berr == cudaSuccess; o += kPiece, ++piece_no) {
        if (piece_no >= 2) berr = cudaEventSynchronize(piece_ev[piece_no & 1]);
        if (berr == cudaSuccess)
          berr = cudaMemcpyAsync(static_cast<unsigned char*>(dst) + o,
                                 static_cast<const unsigned char*>(src) + o,
                                 std::min(kPiece, bytes - o), cudaMemcpyHostToDevice, sb);
        if (berr == cudaSuccess) berr = cudaEventRecord(piece_ev[piece_no & 1], sb);
      }
    };
    std::thread upload_b([&] {
      berr = cudaSetDevice(dev);
      if (berr == cudaSuccess) berr = cudaStreamWaitEvent(sb, patterns, 0);
      if (berr == cudaSuccess && h.b_is_dense)
        upload(bd.p, h.d_b_dense, (size_t)h.b_rows * h.b_cols * el);
      if (berr == cudaSuccess) upload(c.p, h.d_c, (size_t)h.c_rows * h.c_cols * el);
      if (berr == cudaSuccess && annz > 0) upload(av.p, h.d_a_val, (size_t)annz * el);
      if (berr == cudaSuccess && !h.b_is_dense && !b_is_a && bnnz > 0)
        upload(bv.p, h.d_b_val, (size_t)bnnz * el);
      if (berr == cudaSuccess) berr = cudaStreamSynchronize(sb);
    });
    struct Join {
      std::thread& t;
      ~Join() {
        if (t.joinable()) t.join();
      }
    } join{upload_b};
    const bool dbg_t = getenv("TFG_DEBUG") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what, bool sync) {
      if (!dbg_t) return;
      if (sync) cudaStreamSynchronize(sa);
      fprintf(stderr, "[tfg] run_host %-22s at %8.2f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count());
    };
    mark("patterns queued", false);
    UploadScope staged(sa);  // the plan's work lists bypass the busy H2D copy engine
    tfg_plan pl;
    plan_create(d, s, sa, pl);  // overlaps the upload of values, B and C
    mark("plan created", false);
    dbuf<unsigned char> dd((size_t)h.n * h.c_cols * el);
    upload_b.join();
    TFG_CUDA(berr);
    mark("operands uploaded", false);
    plan_execute(pl, dd.p, sa);
    mark("executed", true);
    d2h(static_cast<unsigned char*>(h_d), dd.p, (size_t)h.n * h.c_cols * el, sa);
    TFG_CUDA(cudaStreamSynchronize(sa));
    mark("D downloaded", false);
  });
}

tfg_status tfg_gather_rows(int32_t dtype, const void* src, int32_t cols, const int32_t* rows,
                           int64_t n, void* dst, void* stream) {
  return guard([&] { gather_rows(dtype, src, cols, rows, n, dst, as_stream(stream)); });
}

tfg_status tfg_scatter_rows(int32_t dtype, const void* src, int32_t cols, const int32_t* rows,
                            int64_t n, void* dst, void* stream) {
  return guard([&] { scatter_rows(dtype, src, cols, rows, n, dst, as_stream(stream)); });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Row-range helpers (kernels.hpp:159-180): host operands, GPU kernels.
// ---------------------------------------------------------------------------
extern "C" {

tfg_status tfg_gemm_rows_host(int32_t dtype, const void* h_b, int32_t b_rows, int32_t b_cols,
                              const void* h_c, int32_t c_rows, int32_t c_cols, int32_t row_lo,
                              int32_t row_hi, void* h_d1) {
  return guard([&] {
    if (b_cols != c_rows) throw invalid_argument("gemm: inner dimensions disagree");
    if (row_lo < 0 || row_hi > b_rows || row_lo > row_hi)
      throw invalid_argument("gemm: row range out of bounds");
    if (row_hi == row_lo) return;
    const size_t el = dtype == TFG_F64 ? 8 : 4;
    cudaStream_t st = nullptr;
    const int nr = row_hi - row_lo;
    dbuf<unsigned char> b((size_t)nr * b_cols * el), c((size_t)c_rows * c_cols * el),
        d((size_t)nr * c_cols * el);
    h2d(b.p, static_cast<const unsigned char*>(h_b) + (size_t)row_lo * b_cols * el,
        (size_t)nr * b_cols * el, st);
    h2d(c.p, static_cast<const unsigned char*>(h_c), (size_t)c_rows * c_cols * el, st);
    std::vector<int> r0, cnt;
    for (int r = 0; r < nr; r += kGemmBM) {
      r0.push_back(r);
      cnt.push_back(std::min(kGemmBM, nr - r));
    }
    dbuf<int> dr0(r0.size()), dcnt(cnt.size());
    h2d(dr0.p, r0.data(), r0.size(), st);
    h2d(dcnt.p, cnt.data(), cnt.size(), st);
    const int gy = (c_cols + kGemmBN - 1) / kGemmBN;
    const int gx = (int)std::min<size_t>(r0.size(), (size_t)sm_count() * 16);
    if (dtype == TFG_F64)
      k_gemm_blocks<double, kGemmBM, kGemmBN, kGemmBK, kGemmTM, kGemmTN>
          <<<dim3(gx, gy), 256, 0, st>>>((int64_t)r0.size(), dr0.p, dcnt.p,
                                         reinterpret_cast<const double*>(b.p), b_cols,
                                         reinterpret_cast<const double*>(c.p), c_cols,
                                         reinterpret_cast<double*>(d.p), c_cols);
    else
      k_gemm_blocks<float, kGemmBM, kGemmBN, kGemmBK, kGemmTM, kGemmTN>
          <<<dim3(gx, gy), 256, 0, st>>>((int64_t)r0.size(), dr0.p, dcnt.p,
                                         reinterpret_cast<const float*>(b.p), b_cols,
                                         reinterpret_cast<const float*>(c.p), c_cols,
                                         reinterpret_cast<float*>(d.p), c_cols);
    TFG_LAUNCH_CHECK();
    d2h(static_cast<unsigned char*>(h_d1) + (size_t)row_lo * c_cols * el, d.p,
        (size_t)nr * c_cols * el, st);
    TFG_CUDA(cudaStreamSynchronize(st));
  });
}

tfg_status tfg_spmm_rows_host(int32_t dtype, int32_t a_rows, int32_t a_cols,
                              const int32_t* h_rp, const int32_t* h_ci, const void* h_av,
                              const void* h_x, int32_t x_rows, int32_t x_cols,
                              const int32_t* h_rows, int64_t n_list, void* h_d) {
  return guard([&] {
    if (a_cols != x_rows) throw invalid_argument("spmm: inner dimensions disagree");
    for (int64_t q = 0; q < n_list; ++q)
      if (h_rows[q] < 0 || h_rows[q] >= a_rows) throw invalid_argument("spmm: row out of range");
    if (n_list == 0) return;
    const size_t el = dtype == TFG_F64 ? 8 : 4;
    cudaStream_t st = nullptr;
    const int64_t nnz = h_rp[a_rows];
    dbuf<int32_t> rp(a_rows + 1), ci(std::max<int64_t>(nnz, 1));
    dbuf<unsigned char> av(std::max<int64_t>(nnz, 1) * el), x((size_t)x_rows * x_cols * el),
        d((size_t)a_rows * x_cols * el);
    h2d(rp.p, h_rp, a_rows + 1, st);
    h2d(ci.p, h_ci, nnz, st);
    h2d(av.p, static_cast<const unsigned char*>(h_av), nnz * el, st);
    h2d(x.p, static_cast<const unsigned char*>(h_x), (size_t)x_rows * x_cols * el, st);
    // rows not in the list keep the caller's values
    h2d(d.p, static_cast<const unsigned char*>(h_d), (size_t)a_rows * x_cols * el, st);
    std::vector<int> rows(h_rows, h_rows + n_list);
    std::vector<int> rph(h_rp, h_rp + a_rows + 1);
    SpmmWork w;
    w.build(rows, rph, x_cols, el, st);
    if (dtype == TFG_F64)
      spmm_run<double>(w, rp.p, ci.p, reinterpret_cast<const double*>(av.p),
                       reinterpret_cast<const double*>(x.p), x_cols,
                       reinterpret_cast<double*>(d.p), st);
    else
      spmm_run<float>(w, rp.p, ci.p, reinterpret_cast<const float*>(av.p),
                      reinterpret_cast<const float*>(x.p), x_cols, reinterpret_cast<float*>(d.p),
                      st);
    d2h(static_cast<unsigned char*>(h_d), d.p, (size_t)a_rows * x_cols * el, st);
    TFG_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
