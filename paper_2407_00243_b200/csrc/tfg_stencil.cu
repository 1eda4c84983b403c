// tfg_stencil.cu -- plane-streaming SpMM for grid stencils (see tfg_stencil.cuh).
#include "tfg_stencil.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tfg_device.cuh"

namespace tfg {
namespace {

using dev::fops;
using dev::ldv;
using dev::stv;

constexpr int kMaxNS = 8;      // plane ring depth cap
constexpr size_t kSliceBytes = 512;  // column slice of X / out per CTA
constexpr size_t kSmemBudget = 224 * 1024;
// value slots per warp: 3-D output planes keep their values for three steps
// (z-sliding accumulators) and load them four planes ahead; 2-D: two ahead
template <bool D3>
constexpr int kValueSlots = D3 ? 5 : 3;

// One sparse operand (a stencil CSR) of a kernel.
struct OpArgs {
  unsigned used;  // 27-bit mask of the stencil's neighbours (bit ((dz+1)*3+(dy+1))*3+(dx+1))
  int K;     // nonzeros of a full row
  int full;  // the stencil is the whole 3x3 (x3) box: compile-time value offsets
  int8_t rank[27];
  const int* rp;
  const int* ci;
  const void* av;
};

struct StencilArgs {
  int n, nx, ny, nz, nxy;
  int zb, ze;  // planes [zb, ze) are computed (a row-block partition)
  int zc, ns, slices, ntx, nty, cc;
  long long items;
  int plane_elems;
  OpArgs op;
  void* out;
  int nzc;  // z chunks per tile
};

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void s_bar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s_u32(b)), "r"(count));
}
__device__ __forceinline__ void s_bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void s_bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void s_bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n ST_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      " @!p bra ST_WAIT_%=;\n}\n" ::"r"(s_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                       int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(s_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(s_u32(bar))
      : "memory");
}

// Tile geometry.  2-D (9-point family): a tile is NW * M consecutive points
// of one grid line, the sliding axis is y.  3-D (27-point family): a tile is
// M x NW points of the (x, y) plane, one tile line per warp, sliding along z.
template <bool D3, int NW, int M>
struct Tile {
  static constexpr int TX = D3 ? M : M * NW;
  static constexpr int TY = D3 ? NW : 1;
  static constexpr int ROW = TX + 2;           // plane row length incl. halo
  static constexpr int TYH = D3 ? NW + 2 : 1;  // plane rows incl. halo
};

// Work item -> (column slice, x tile, y tile, z chunk); slices vary fastest so
// co-resident CTAs share their tiles' halo rows in L2.
__device__ __forceinline__ void decode_item(const StencilArgs& a, long long it, int& cs, int& itx,
                                            int& ity, int& izc) {
  cs = (int)(it % a.slices);
  long long t = it / a.slices;
  itx = (int)(t % a.ntx);
  t /= a.ntx;
  ity = (int)(t % a.nty);
  izc = (int)(t / a.nty);
}

template <int BYTES>
__device__ __forceinline__ void cp_async_ca(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s_u32(dst)), "l"(src),
               "n"(BYTES)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Values of a warp's M consecutive rows are contiguous in the CSR: lanes load
// them (one step ahead, coalesced) into registers and stage them in the
// warp's shared-memory buffer, so the per-nonzero value reads are broadcast
// shared loads instead of dependent global loads.
template <class T, int VR>
__device__ __forceinline__ void load_vals(const T* __restrict__ av, int v0, int v1, int lane,
                                          T (&vr)[VR]) {
#pragma unroll
  for (int i = 0; i < VR; ++i) {
    const int k = v0 + lane + 32 * i;
    vr[i] = k < v1 ? __ldg(av + k) : T(0);
  }
}

// acc += v * x: one fused multiply-add per element (default: within the
// north-star tolerance, half the FP issue slots), or the reference's
// separately rounded mul and add (EXACT: bit-identical to spmm_row)
template <class T, int VEC, bool EXACT>
__device__ __forceinline__ void axpy(T (&acc)[VEC], T v, const T (&x)[VEC]) {
#pragma unroll
  for (int e = 0; e < VEC; ++e)
    acc[e] = EXACT ? fops<T>::add(acc[e], fops<T>::mul(v, x[e])) : fops<T>::fma(v, x[e], acc[e]);
}

// One output plane z of a warp's M points.  P0/P1/P2: the shared-memory
// planes z-1, z, z+1 of the tile (zero-filled outside the grid); rpl: lane
// m <= M holds row_ptr of point m; valid: points inside the grid; sv: the
// rows' values from row_ptr[point 0].
// 27-bit neighbour masks, bit ((dz+1)*3 + (dy+1))*3 + (dx+1)
constexpr unsigned nb_bits(int axis, int d) {  // all neighbours with offset d along axis (0 x, 1 y, 2 z)
  unsigned m = 0;
  for (int q = 0; q < 27; ++q) {
    const int dx = q % 3 - 1, dy = (q / 3) % 3 - 1, dz = q / 9 - 1;
    if ((axis == 0 ? dx : (axis == 1 ? dy : dz)) == d) m |= 1u << q;
  }
  return m;
}

// One output plane of a warp's M points into acc.  P0/P1/P2: the
// shared-memory planes z-1, z, z+1 of the tile (zero-filled outside the
// grid); rpl: lane m <= M holds row_ptr of point m; valid: points inside the
// grid; sv: the rows' values from row_ptr[point 0]; (px, py, pz): grid
// position of point 0.
// Padded value layout of a full-box group (PAD): point m's three values of
// line l at sv[m * 4 * NL + 4 * l + j] -- one 16-byte aligned group per line
// -- so a point's line values come in one (fp32) or two (fp64) shared loads.
template <bool D3>
__device__ __forceinline__ int pad_index(int t) {  // t = m * K + 3 l + j
  constexpr int K = D3 ? 27 : 9;
  const int m = t / K, r = t - m * K;
  const int l = r / 3;
  return m * (4 * (D3 ? 9 : 3)) + 4 * l + (r - 3 * l);
}

// The per-point paths of one output plane's M points (grid faces and rows
// missing in-grid neighbours), restricted to the neighbours with dz + 1 in
// [dz_lo, dz_hi): all three planes at once (0, 3), or one input plane at a
// time in ascending dz (the z-sliding loop; P0 = P1 = P2 = that plane).  acc
// is accumulated into, not cleared.
template <class T, bool D3, int M, int ROW, bool EXACT>
__device__ __forceinline__ void stencil_slow(const StencilArgs& a, const OpArgs& op,
                                             const T* __restrict__ P0, const T* __restrict__ P1,
                                             const T* __restrict__ P2, const T* __restrict__ sv,
                                             int rpl, unsigned valid, int wy, int col0, int rbase,
                                             int px, int py, int pz, int lane, int dz_lo, int dz_hi,
                                             T (&acc)[M][16 / sizeof(T)]) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int CW = (int)(kSliceBytes / sizeof(T));
  constexpr int NL = D3 ? 9 : 3;
  const int v0 = __shfl_sync(0xffffffffu, rpl, 0);
  // Grid-face points: a row whose nonzero count equals the number of its
  // in-grid stencil neighbours holds exactly those (every nonzero was checked
  // to be an in-grid neighbour at plan time), so its value for neighbour bit
  // q sits at popc(mask & (2^q - 1)) -- the same compile-time loop as the
  // fast path, predicated per point.  Other rows (missing in-grid
  // neighbours) walk their own CSR entries.
  int vb[M + 1];
#pragma unroll
  for (int m = 0; m <= M; ++m) vb[m] = __shfl_sync(0xffffffffu, rpl, m);
  unsigned pm[M];
  unsigned geo = 0;
  {
    unsigned face = op.used;
    if (D3) {
      if (py == 0) face &= ~nb_bits(1, -1);
      if (py == a.ny - 1) face &= ~nb_bits(1, 1);
    }
    if (pz == 0) face &= ~nb_bits(D3 ? 2 : 2, -1);
    if (pz == a.nz - 1) face &= ~nb_bits(2, 1);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      unsigned pmm = face;
      if (px + m == 0) pmm &= ~nb_bits(0, -1);
      if (px + m == a.nx - 1) pmm &= ~nb_bits(0, 1);
      pm[m] = pmm;
      if (((valid >> m) & 1u) && vb[m + 1] - vb[m] == __popc(pmm)) geo |= 1u << m;
    }
  }
  if (geo) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int dz = D3 ? l / 3 - 1 : l - 1;
      const int dy = D3 ? l % 3 - 1 : 0;
      const int li = (dz + 1) * 3 + (dy + 1);
      if (!(op.used & (7u << (3 * li)))) continue;
      if (dz + 1 < dz_lo || dz + 1 >= dz_hi) continue;
      const T* P = dz < 0 ? P0 : (dz == 0 ? P1 : P2);
      const T* base = P + ((D3 ? (wy + 1 + dy) * ROW : 0) + col0) * CW + lane * VEC;
      // the line's values of all M points first (independent shared loads,
      // absent neighbours read a dummy slot), then the predicated updates:
      // a face group costs about what an interior group does, so the CTA's
      // other warps are not held at the plane ring by it
      T vl[M][3];
      unsigned pr = 0;  // bit 3 m + j: point m has neighbour dx = j - 1 on this line
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const unsigned bits = ((geo >> m) & 1u) ? (pm[m] >> (3 * li)) & 7u : 0u;
        pr |= bits << (3 * m);
        // value index of the line's first present neighbour, then +1 per bit
        int idx = vb[m] - v0 + __popc(pm[m] & ((1u << (3 * li)) - 1u));
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const bool has = (bits >> j) & 1u;
          vl[m][j] = sv[has ? idx : 0];
          idx += has;
        }
      }
#pragma unroll
      for (int k = 0; k < M + 2; ++k) {
        T xr[VEC];
        ldv<T, VEC>(xr, base + k * CW);
        // this row is neighbour dx = -1 of point k, 0 of k - 1, +1 of k - 2
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int m = k - j;
          if (m < 0 || m >= M) continue;
          if ((pr >> (3 * m + j)) & 1u) axpy<T, VEC, EXACT>(acc[m], vl[m][j], xr);
        }
      }
    }
  }
  const unsigned irr = valid & ~geo;
  if (irr) {  // rows missing in-grid neighbours: their own CSR order
    // the rows' column indices, lane-parallel and all issued up front
    // (one memory round trip for the group, not one per nonzero)
    int cl[M];
#pragma unroll
    for (int m = 0; m < M; ++m)
      cl[m] = ((irr >> m) & 1u) && vb[m] + lane < vb[m + 1] ? __ldg(op.ci + vb[m] + lane) : 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      if (!((irr >> m) & 1u)) continue;
      const int r = rbase + m;
      for (int k = vb[m]; k < vb[m + 1]; ++k) {  // <= 27 nonzeros: one lane each
        int o = __shfl_sync(0xffffffffu, cl[m], k - vb[m]) - r;
        int dz = 0, dy = 0;
        if (D3) {
          dz = o > a.nxy / 2 ? 1 : (o < -(a.nxy / 2) ? -1 : 0);
          o -= dz * a.nxy;
          dy = o > a.nx / 2 ? 1 : (o < -(a.nx / 2) ? -1 : 0);
          o -= dy * a.nx;
        } else {
          dz = o > a.nx / 2 ? 1 : (o < -(a.nx / 2) ? -1 : 0);
          o -= dz * a.nx;
        }
        if (dz + 1 < dz_lo || dz + 1 >= dz_hi) continue;  // warp-uniform
        const T* P = dz < 0 ? P0 : (dz == 0 ? P1 : P2);
        const int yy = D3 ? wy + 1 + dy : 0;
        T xr[VEC];
        ldv<T, VEC>(xr, P + (yy * ROW + col0 + m + 1 + o) * CW + lane * VEC);
        axpy<T, VEC, EXACT>(acc[m], sv[k - v0], xr);
      }
    }
  }
}

template <class T, bool D3, int M, int ROW, bool PAD, bool EXACT>
__device__ __forceinline__ void stencil_compute(const StencilArgs& a, const OpArgs& op,
                                                const T* __restrict__ P0, const T* __restrict__ P1,
                                                const T* __restrict__ P2, const T* __restrict__ sv,
                                                int rpl, unsigned valid, int wy, int col0,
                                                int rbase, int px, int py, int pz, int lane,
                                                T (&acc)[M][16 / sizeof(T)]) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int CW = (int)(kSliceBytes / sizeof(T));
  constexpr int NL = D3 ? 9 : 3;
  const int v0 = __shfl_sync(0xffffffffu, rpl, 0);
  const int vM = __shfl_sync(0xffffffffu, rpl, M);
  // every row has <= K nonzeros, so M * K of them means all M rows are full;
  // the window rows of points outside the tile are still in the plane
  // buffer (or the next shared-memory region), so the fast path computes all
  // M points and stores only the valid ones
  const bool fast = op.full && valid != 0 && vM - v0 == M * 3 * NL;
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[m][v] = T(0);
  if (fast && PAD) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int dz = D3 ? l / 3 - 1 : l - 1;
      const int dy = D3 ? l % 3 - 1 : 0;
      const T* P = dz < 0 ? P0 : (dz == 0 ? P1 : P2);
      const T* base = P + ((D3 ? (wy + 1 + dy) * ROW : 0) + col0) * CW + lane * VEC;
      T vl[M][4];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const T* q = sv + m * 4 * NL + 4 * l;
        if constexpr (sizeof(T) == 8) {
          T v01[2];
          ldv<T, 2>(v01, q);
          vl[m][0] = v01[0];
          vl[m][1] = v01[1];
          vl[m][2] = q[2];
        } else {
          ldv<T, 4>(vl[m], q);
        }
      }
#pragma unroll
      for (int k = 0; k < M + 2; ++k) {
        T xr[VEC];
        ldv<T, VEC>(xr, base + k * CW);
        if (k < M) axpy<T, VEC, EXACT>(acc[k], vl[k][0], xr);
        if (k >= 1 && k - 1 < M) axpy<T, VEC, EXACT>(acc[k - 1], vl[k - 1][1], xr);
        if (k >= 2) axpy<T, VEC, EXACT>(acc[k - 2], vl[k - 2][2], xr);
      }
    }
    return;
  }
  if (fast) {
    // whole box, every point interior: point m's value for line l, dx is
    // sv[m * K + 3 * l + dx + 1] -- all offsets compile-time
    constexpr int K = 3 * NL;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int dz = D3 ? l / 3 - 1 : l - 1;
      const int dy = D3 ? l % 3 - 1 : 0;
      const T* P = dz < 0 ? P0 : (dz == 0 ? P1 : P2);
      const T* base = P + ((D3 ? (wy + 1 + dy) * ROW : 0) + col0) * CW + lane * VEC;
#pragma unroll
      for (int k = 0; k < M + 2; ++k) {
        T xr[VEC];
        ldv<T, VEC>(xr, base + k * CW);
        if (k < M) axpy<T, VEC, EXACT>(acc[k], sv[k * K + 3 * l], xr);
        if (k >= 1 && k - 1 < M) axpy<T, VEC, EXACT>(acc[k - 1], sv[(k - 1) * K + 3 * l + 1], xr);
        if (k >= 2) axpy<T, VEC, EXACT>(acc[k - 2], sv[(k - 2) * K + 3 * l + 2], xr);
      }
    }
    return;
  }
  stencil_slow<T, D3, M, ROW, EXACT>(a, op, P0, P1, P2, sv, rpl, valid, wy, col0, rbase, px, py, pz,
                                     lane, 0, 3, acc);
}

template <class T, bool D3, int M, int ROW, bool PAD, bool EXACT>
__device__ __forceinline__ void stencil_points(const StencilArgs& a, const OpArgs& op,
                                               const T* __restrict__ P0, const T* __restrict__ P1,
                                               const T* __restrict__ P2, const T* __restrict__ sv,
                                               int rpl, unsigned valid, int wy, int col0,
                                               int rbase, int px, int py, int pz,
                                               T* __restrict__ outp, int ostride, int lane) {
  constexpr int VEC = 16 / sizeof(T);
  T acc[M][VEC];
  stencil_compute<T, D3, M, ROW, PAD, EXACT>(a, op, P0, P1, P2, sv, rpl, valid, wy, col0, rbase,
                                             px, py, pz, lane, acc);
#pragma unroll
  for (int m = 0; m < M; ++m)
    if ((valid >> m) & 1u) stv<T, VEC>(outp + (size_t)m * ostride, acc[m]);
}

// z-sliding accumulation (3-D full-box interior groups).  Instead of reading
// the three X planes z-1, z, z+1 again for every output plane (each X row 9
// times), one pass over the NEWEST plane p adds its rows to three output
// planes at once: as dz = +1 of output p-1 (accA, that plane's values of
// lines 6..8), dz = 0 of output p (accB, lines 3..5) and dz = -1 of output
// p+1 (accC, lines 0..2) -- each X row is read from shared memory 3 times
// instead of 9.  An output plane still receives its terms in ascending
// (dz, dy, dx) order (dz = -1 from plane z-1 first, then plane z, then z+1,
// each in dy, dx order), so the bits equal stencil_compute's.  MASK selects
// the live targets (bit 0 accA, 1 accB, 2 accC): planes that are not full-box
// groups, or lie outside the item, are skipped.
template <class T, int M, int ROW, bool EXACT, int MASK>
__device__ __forceinline__ void slide_plane(const T* __restrict__ P, int wy, int col0, int lane,
                                            const T* __restrict__ svA, const T* __restrict__ svB,
                                            const T* __restrict__ svC,
                                            T (&accA)[M][16 / sizeof(T)],
                                            T (&accB)[M][16 / sizeof(T)],
                                            T (&accC)[M][16 / sizeof(T)]) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int CW = (int)(kSliceBytes / sizeof(T));
  constexpr int NL = 9;
  auto load_line = [&](const T* sv, int l, T(&vl)[M][4]) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const T* q = sv + m * 4 * NL + 4 * l;
      if constexpr (sizeof(T) == 8) {
        T v01[2];
        ldv<T, 2>(v01, q);
        vl[m][0] = v01[0];
        vl[m][1] = v01[1];
        vl[m][2] = q[2];
      } else {
        ldv<T, 4>(vl[m], q);
      }
    }
  };
#pragma unroll
  for (int dyi = 0; dyi < 3; ++dyi) {
    const T* base = P + ((wy + dyi) * ROW + col0) * CW + lane * VEC;
    T vA[M][4], vB[M][4], vC[M][4];
    if constexpr ((MASK & 1) != 0) load_line(svA, 6 + dyi, vA);
    if constexpr ((MASK & 2) != 0) load_line(svB, 3 + dyi, vB);
    if constexpr ((MASK & 4) != 0) load_line(svC, dyi, vC);
#pragma unroll
    for (int k = 0; k < M + 2; ++k) {
      T xr[VEC];
      ldv<T, VEC>(xr, base + k * CW);
      if constexpr ((MASK & 4) != 0) {  // dz = -1 terms come first in their output's order
        if (k < M) axpy<T, VEC, EXACT>(accC[k], vC[k][0], xr);
        if (k >= 1 && k - 1 < M) axpy<T, VEC, EXACT>(accC[k - 1], vC[k - 1][1], xr);
        if (k >= 2) axpy<T, VEC, EXACT>(accC[k - 2], vC[k - 2][2], xr);
      }
      if constexpr ((MASK & 2) != 0) {
        if (k < M) axpy<T, VEC, EXACT>(accB[k], vB[k][0], xr);
        if (k >= 1 && k - 1 < M) axpy<T, VEC, EXACT>(accB[k - 1], vB[k - 1][1], xr);
        if (k >= 2) axpy<T, VEC, EXACT>(accB[k - 2], vB[k - 2][2], xr);
      }
      if constexpr ((MASK & 1) != 0) {
        if (k < M) axpy<T, VEC, EXACT>(accA[k], vA[k][0], xr);
        if (k >= 1 && k - 1 < M) axpy<T, VEC, EXACT>(accA[k - 1], vA[k - 1][1], xr);
        if (k >= 2) axpy<T, VEC, EXACT>(accA[k - 2], vA[k - 2][2], xr);
      }
    }
  }
}

template <class T, int M, int ROW, bool EXACT>
__device__ __forceinline__ void slide_plane_masked(unsigned mask, const T* __restrict__ P, int wy,
                                                   int col0, int lane, const T* __restrict__ svA,
                                                   const T* __restrict__ svB,
                                                   const T* __restrict__ svC,
                                                   T (&accA)[M][16 / sizeof(T)],
                                                   T (&accB)[M][16 / sizeof(T)],
                                                   T (&accC)[M][16 / sizeof(T)]) {
  switch (mask) {  // warp-uniform
#define TFG_SLIDE(MK)                                                                          \
  case MK:                                                                                     \
    slide_plane<T, M, ROW, EXACT, MK>(P, wy, col0, lane, svA, svB, svC, accA, accB, accC);     \
    break;
    TFG_SLIDE(1) TFG_SLIDE(2) TFG_SLIDE(3) TFG_SLIDE(4) TFG_SLIDE(5) TFG_SLIDE(6) TFG_SLIDE(7)
#undef TFG_SLIDE
    default: break;
  }
}

template <class T, bool D3, int NW, int M, int MINB, bool EXACT>
__global__ void __launch_bounds__((NW + 1) * 32, MINB)
    k_spmm_stencil(const __grid_constant__ CUtensorMap xmap, const StencilArgs a) {
  using TL = Tile<D3, NW, M>;
  constexpr int CW = (int)(kSliceBytes / sizeof(T));
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxNS], empty[kMaxNS];
  T* planes = reinterpret_cast<T*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ns = a.ns;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      s_bar_init(&full[s], 1);
      s_bar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const uint32_t plane_bytes = (uint32_t)a.plane_elems * sizeof(T);
  if (warp == NW) {
    // ---------------- producer: one 4-D TMA copy per tile plane ----------------
    if (lane == 0) {
      uint32_t g = 0;
      for (long long it = blockIdx.x; it < a.items; it += gridDim.x) {
        int cs, itx, ity, izc;
        decode_item(a, it, cs, itx, ity, izc);
        const int z0 = a.zb + izc * a.zc, z1 = min(z0 + a.zc, a.ze);
        const int c1 = itx * TL::TX - 1;
        const int c2 = D3 ? ity * TL::TY - 1 : 0;
        const CUtensorMap* map = &xmap;
        for (int p = z0 - 1; p <= z1; ++p, ++g) {
          const int s = (int)(g % ns);
          const uint32_t k = g / ns;
          if (k > 0) s_bar_wait(&empty[s], (k - 1) & 1u);
          s_bar_expect(&full[s], plane_bytes);
          tma_4d(planes + (size_t)s * a.plane_elems, map, cs * CW, c1, c2, p, &full[s]);
        }
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  // Per warp, the values and row pointers of its points stream into shared
  // memory by cp.async, values two output planes ahead and row pointers four
  // ahead (one commit group per plane), so no consumer instruction waits on
  // a global load.
  constexpr int VR = (M * (D3 ? 27 : 9) + 31) / 32;  // value elements per lane and plane
  constexpr int VS0 = VR * 32;
  constexpr int VS = VS0 > M * 4 * (D3 ? 9 : 3) ? VS0 : M * 4 * (D3 ? 9 : 3);  // value slot
  // 3-D: z-sliding accumulators (slide_plane); an output plane's values are
  // then in use over three steps, so its ring is deeper and loaded further ahead
  constexpr bool SLIDE = D3;
  constexpr int VSL = kValueSlots<D3>;  // value slots per warp
  T* svb = reinterpret_cast<T*>(smem_raw + (size_t)ns * plane_bytes) + (size_t)warp * VSL * VS;
  int* srp = reinterpret_cast<int*>(reinterpret_cast<T*>(smem_raw + (size_t)ns * plane_bytes) +
                                    (size_t)NW * VSL * VS) + warp * 8 * 16;
  const int wy = D3 ? warp : 0, wx = D3 ? 0 : warp;
  int pidx[VR];  // padded slot position of this lane's value elements (loop invariant)
#pragma unroll
  for (int i = 0; i < VR; ++i) pidx[i] = pad_index<D3>(lane + 32 * i);
  int s0 = 0;        // ring slot of the current item's plane z-1
  uint32_t p0 = 0;   // its full-barrier phase parity
  const OpArgs& opa = a.op;
  const T* __restrict__ av = static_cast<const T*>(opa.av);
  T* const outb = static_cast<T*>(a.out);
  for (long long it = blockIdx.x; it < a.items; it += gridDim.x) {
    int cs, itx, ity, izc;
    decode_item(a, it, cs, itx, ity, izc);
    const int z0 = a.zb + izc * a.zc, z1 = min(z0 + a.zc, a.ze);
    const int nzl = z1 - z0;
    const int x = itx * TL::TX + wx * M;
    const int y = D3 ? ity * TL::TY + wy : 0;
    const bool yvalid = y < a.ny;
    const bool live = yvalid && x < a.nx && lane <= M;
    unsigned valid = 0;
#pragma unroll
    for (int m = 0; m < M; ++m)
      if (yvalid && x + m < a.nx) valid |= 1u << m;
    const int r0 = (z0 * a.ny + y) * a.nx + x;  // point 0 at output plane z0
    auto issue_rp = [&](int jj) {
      if (live && jj < nzl) cp_async_ca<4>(srp + (jj & 7) * 16 + lane, opa.rp + min(r0 + jj * a.nxy + lane, a.n));
    };
    const bool wlive = yvalid && x < a.nx;  // warp-uniform: the warp has points
    // Staging of an output plane's values, and with it the plane's path
    // (3-D; recorded in the row-pointer slot's spare word for fast_at):
    //  2  interior full-box group: value t of the group at padded slot pidx
    //  1  every point of the group is a grid-face point holding exactly its
    //     in-grid neighbours: the same padded slots by neighbour POSITION, a
    //     zero stored where a neighbour lies outside the grid -- the X plane
    //     is zero-filled there too, so the full-box code adds an exact +0 and
    //     face, edge and corner groups cost what interior groups do
    //  0  anything else (rows missing in-grid neighbours): values as stored,
    //     per-point paths
    auto issue_vals = [&](int jj) {  // row pointers of plane jj must be visible
      if (!wlive || jj >= nzl) return;
      const int* rpl = srp + (jj & 7) * 16;
      const int v0 = rpl[0], v1 = rpl[M];
      T* dst = svb + (jj % VSL) * VS;
      // the compute side takes the padded full-box path exactly when this holds
      const bool pad = opa.full && valid != 0 && v1 - v0 == M * (D3 ? 27 : 9);
      if constexpr (SLIDE) {
        int mode = pad ? 2 : 0;
        unsigned face = 0;
        if (!pad && opa.full && valid != 0) {
          const int pz = z0 + jj;
          face = (1u << 27) - 1u;
          if (y == 0) face &= ~nb_bits(1, -1);
          if (y == a.ny - 1) face &= ~nb_bits(1, 1);
          if (pz == 0) face &= ~nb_bits(2, -1);
          if (pz == a.nz - 1) face &= ~nb_bits(2, 1);
          // lanes 0..M-1 check their point: outside the grid, or exactly its in-grid neighbours
          bool ok = true;
          if (lane < M && ((valid >> lane) & 1u)) {
            unsigned pmm = face;
            if (x + lane == 0) pmm &= ~nb_bits(0, -1);
            if (x + lane == a.nx - 1) pmm &= ~nb_bits(0, 1);
            ok = rpl[lane + 1] - rpl[lane] == __popc(pmm);
          }
          mode = __all_sync(0xffffffffu, ok) ? 1 : 0;
        }
        if (lane == 0) srp[(jj & 7) * 16 + 15] = mode;
        if (mode == 1) {
#pragma unroll
          for (int i = 0; i < VR; ++i) {
            const int t = lane + 32 * i;  // neighbour position t = m * 27 + q
            if (t >= M * 27) continue;
            const int m = t / 27, q = t - m * 27;
            unsigned pmm = ((valid >> m) & 1u) ? face : 0u;
            if (x + m == 0) pmm &= ~nb_bits(0, -1);
            if (x + m == a.nx - 1) pmm &= ~nb_bits(0, 1);
            if ((pmm >> q) & 1u)
              cp_async_ca<sizeof(T)>(dst + pidx[i], av + rpl[m] + __popc(pmm & ((1u << q) - 1u)));
            else
              dst[pidx[i]] = T(0);
          }
          return;
        }
      }
#pragma unroll
      for (int i = 0; i < VR; ++i) {
        const int t = lane + 32 * i;
        if (v0 + t < v1) cp_async_ca<sizeof(T)>(dst + (pad ? pidx[i] : t), av + v0 + t);
      }
    };
    // the group at output plane jj of this item takes the full-box code (warp-uniform)
    auto fast_at = [&](int jj) {
      if (jj < 0 || jj >= nzl || !opa.full || valid == 0) return false;
      if constexpr (SLIDE)
        return srp[(jj & 7) * 16 + 15] != 0;
      else
        return srp[(jj & 7) * 16 + M] - srp[(jj & 7) * 16] == M * (D3 ? 27 : 9);
    };
    constexpr int VEC = 16 / sizeof(T);
    if constexpr (SLIDE) {
      // ---- z-sliding loop: one pass per INPUT plane p = z0-1 .. z1 ----
      // Plane p (iteration pi = p - z0 + 1) adds dz = +1 to output pi-2
      // (acc3[0]), dz = 0 to output pi-1 (acc3[1]) and dz = -1 to output pi
      // (acc3[2]); output pi-2 is then complete and stored.  Full-box and
      // grid-face groups go through slide_plane (all live targets in one
      // pass over the plane's rows), rows missing in-grid neighbours through
      // stencil_slow restricted to this plane.  Each plane is read once and
      // released: the ring holds the plane in use plus the prefetch depth.
      T acc3[3][M][VEC];
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc3[q][m][v] = T(0);
      // values of output jj: issued at iteration jj - 2, used at jj .. jj + 2;
      // row pointers of jj: issued at jj - 4 (the values' addresses)
      issue_rp(0);
      issue_rp(1);
      issue_rp(2);
      issue_rp(3);
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
      issue_vals(0);
      issue_vals(1);
      cp_async_commit();
      bool f0 = false, f1 = false;  // outputs pi-2, pi-1 take the full-box code
      for (int pi = 0; pi < nzl + 2; ++pi) {
        if (pi == 0)
          cp_async_wait<0>();
        else
          cp_async_wait<1>();  // values up to output pi, row pointers up to pi + 2
        __syncwarp();
        issue_vals(pi + 2);
        issue_rp(pi + 4);
        cp_async_commit();
        s_bar_wait(&full[s0], p0);
        const T* P = planes + (size_t)s0 * a.plane_elems;
        const bool f2 = fast_at(pi);
        const T* sv0 = svb + ((pi + VSL - 2) % VSL) * VS;
        const T* sv1 = svb + ((pi + VSL - 1) % VSL) * VS;
        const T* sv2 = svb + (pi % VSL) * VS;
        slide_plane_masked<T, M, TL::ROW, EXACT>((f0 ? 1u : 0u) | (f1 ? 2u : 0u) | (f2 ? 4u : 0u), P,
                                                 wy, wx * M, lane, sv0, sv1, sv2, acc3[0], acc3[1],
                                                 acc3[2]);
        // groups with rows missing in-grid neighbours: per-point paths, this plane only
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int jo = pi - 2 + q;  // output plane of target q, neighbour dz = 1 - q
          const bool fq = q == 0 ? f0 : (q == 1 ? f1 : f2);
          if (fq || jo < 0 || jo >= nzl || valid == 0) continue;
          const int rpl = live ? srp[(jo & 7) * 16 + lane] : 0;
          stencil_slow<T, D3, M, TL::ROW, EXACT>(a, opa, P, P, P, svb + (jo % VSL) * VS, rpl, valid, wy,
                                                 wx * M, r0 + jo * a.nxy, x, y, z0 + jo, lane, 2 - q,
                                                 3 - q, acc3[q]);
        }
        if (pi >= 2) {
          T* const outp = outb + (size_t)(r0 + (pi - 2) * a.nxy) * a.cc + (size_t)cs * CW + lane * VEC;
#pragma unroll
          for (int m = 0; m < M; ++m)
            if ((valid >> m) & 1u) stv<T, VEC>(outp + (size_t)m * a.cc, acc3[0][m]);
        }
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            acc3[0][m][v] = acc3[1][m][v];
            acc3[1][m][v] = acc3[2][m][v];
            acc3[2][m][v] = T(0);
          }
        f0 = f1;
        f1 = f2;
        __syncwarp();
        if (lane == 0) s_bar_arrive(&empty[s0]);
        if (++s0 == ns) s0 = 0, p0 ^= 1u;
      }
    } else {
      issue_rp(0);
      issue_rp(1);
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
      issue_vals(0);
      issue_rp(2);
      cp_async_commit();
      issue_vals(1);
      issue_rp(3);
      cp_async_commit();
      for (int j = 0; j < nzl; ++j) {
        cp_async_wait<1>();  // values of plane j, row pointers of plane j + 2
        __syncwarp();
        issue_vals(j + 2);
        issue_rp(j + 4);
        cp_async_commit();
        const int rp_j = live ? srp[(j & 7) * 16 + lane] : 0;
        // ring positions of planes z-1 (s0), z (s1), z+1 (s2)
        int s1 = s0 + 1, s2;
        uint32_t p1 = p0, p2;
        if (s1 == ns) s1 = 0, p1 ^= 1u;
        s2 = s1 + 1;
        p2 = p1;
        if (s2 == ns) s2 = 0, p2 ^= 1u;
        if (j == 0) {
          s_bar_wait(&full[s0], p0);
          s_bar_wait(&full[s1], p1);
        }
        s_bar_wait(&full[s2], p2);
        const int rb = r0 + j * a.nxy;
        stencil_points<T, D3, M, TL::ROW, true, EXACT>(
            a, opa, planes + (size_t)s0 * a.plane_elems, planes + (size_t)s1 * a.plane_elems,
            planes + (size_t)s2 * a.plane_elems, svb + (j % VSL) * VS, rp_j, valid, wy, wx * M, rb,
            x, y, z0 + j, outb + (size_t)rb * a.cc + (size_t)cs * CW + lane * VEC, a.cc, lane);
        __syncwarp();
        if (lane == 0) {
          s_bar_arrive(&empty[s0]);
          if (j == nzl - 1) {
            s_bar_arrive(&empty[s1]);
            s_bar_arrive(&empty[s2]);
          }
        }
        if (j == nzl - 1) {  // the next item starts at the plane after s2
          s0 = s2 + 1;
          p0 = p2;
          if (s0 == ns) s0 = 0, p0 ^= 1u;
        } else {
          s0 = s1;
          p0 = p1;
        }
      }
    }
    cp_async_wait<0>();
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int env_int(const char* name, int def) {
  const char* e = getenv(name);
  return e ? atoi(e) : def;
}

// Every nonzero of the CSR decomposes as an in-grid neighbour of its row and
// every row's columns strictly increase (the kernel finds a neighbour's value
// by its rank in the row).  One warp per row; *fail set on the first
// violation; *used gathers the 27-bit neighbour mask.
__global__ void k_check_geom(int n, const int* __restrict__ rp, const int* __restrict__ ci, int nx,
                             int ny, int* __restrict__ fail, unsigned* __restrict__ used) {
  const long long nxy = (long long)nx * ny;
  const int nz = (int)(n / nxy);
  const int lane = threadIdx.x & 31;
  unsigned mask = 0;
  bool bad = false;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n && !bad;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int x = (int)(r % nx), y = (int)((r / nx) % ny), z = (int)(r / nxy);
    const int b = rp[r], e = rp[r + 1];
    for (int k = b + lane; k < e; k += 32) {
      const int c = ci[k];
      if (k > b && c <= ci[k - 1]) bad = true;
      long long o = (long long)c - r;
      int dz, dy = 0;
      if (ny > 1) {
        dz = o > nxy / 2 ? 1 : (o < -(nxy / 2) ? -1 : 0);
        o -= dz * nxy;
        dy = o > nx / 2 ? 1 : (o < -(nx / 2) ? -1 : 0);
        o -= (long long)dy * nx;
      } else {
        dz = o > nx / 2 ? 1 : (o < -(nx / 2) ? -1 : 0);
        o -= (long long)dz * nx;
      }
      const int dx = (int)o;
      if (dx < -1 || dx > 1 || x + dx < 0 || x + dx >= nx || y + dy < 0 || y + dy >= ny ||
          z + dz < 0 || z + dz >= nz)
        bad = true;
      else
        mask |= 1u << (((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1));
    }
    bad = __any_sync(0xffffffffu, bad);
  }
  mask = __reduce_or_sync(0xffffffffu, mask);
  if (lane == 0) {
    if (bad) atomicExch(fail, 1);
    if (mask) atomicOr(used, mask);
  }
}

bool check_geom(int n, const int* rp_d, const int* ci_d, int nx, int ny, StencilGeom& g,
                cudaStream_t st) {
  const int64_t nxy = (int64_t)nx * ny;
  if (nx < 3 || (ny > 1 && ny < 3) || n % nxy != 0) return false;
  dbuf<int> flag(2);
  TFG_CUDA(cudaMemsetAsync(flag.p, 0, 8, st));
  const int64_t threads = (int64_t)n * 32;
  const int blocks = (int)std::min<int64_t>((threads + 255) / 256, (int64_t)sm_count() * 64);
  k_check_geom<<<blocks, 256, 0, st>>>(n, rp_d, ci_d, nx, ny, flag.p,
                                       reinterpret_cast<unsigned*>(flag.p + 1));
  TFG_LAUNCH_CHECK();
  int h[2] = {0, 0};
  TFG_CUDA(cudaMemcpyAsync(h, flag.p, 8, cudaMemcpyDeviceToHost, st));
  TFG_CUDA(cudaStreamSynchronize(st));
  if (h[0] || h[1] == 0) return false;
  g.nx = nx;
  g.ny = ny;
  g.nz = (int)(n / nxy);
  g.d3 = ny > 1;
  g.K = 0;
  for (int q = 0; q < 27; ++q) g.rank[q] = ((unsigned)h[1] >> q & 1u) ? (int8_t)g.K++ : (int8_t)-1;
  return g.K > 0;
}

}  // namespace

int stencil_env_enabled() { return env_int("TFG_STENCIL", 1); }

bool stencil_detect(int n, const std::vector<int>& rp, const int* rp_d, const int* ci_d,
                    StencilGeom& g, cudaStream_t st) {
  g = StencilGeom{};
  if (n < 9 || (int)rp.size() < n + 1 || rp[n] == 0) return false;
  // candidate geometries from the offsets (col - row) of a sample of rows
  // (a grid stencil's interior rows carry its whole offset set); every
  // candidate is then checked over ALL nonzeros on the device
  std::vector<int64_t> offs;
  std::vector<int> cols;
  for (int q = 0; q < 64; ++q) {
    const int r = (int)(((int64_t)2 * q + 1) * n / 128);
    const int b = rp[r], e = rp[r + 1];
    if (e <= b || e - b > 64) continue;
    cols.resize(e - b);
    TFG_CUDA(cudaMemcpyAsync(cols.data(), ci_d + b, (size_t)(e - b) * 4, cudaMemcpyDeviceToHost, st));
    TFG_CUDA(cudaStreamSynchronize(st));
    for (int c : cols) {
      const int64_t o = (int64_t)c - r;
      if (std::find(offs.begin(), offs.end(), o) == offs.end()) {
        offs.push_back(o);
        if (offs.size() > 27) return false;
      }
    }
  }
  std::sort(offs.begin(), offs.end());
  std::vector<int64_t> pos;
  for (int64_t o : offs)
    if (o >= 2) pos.push_back(o);
  if (pos.empty()) return false;
  // x stride: the smallest offset >= 2 is nx + dx for some dx in {-1, 0, 1}
  for (int64_t nxc : {pos[0] + 1, pos[0], pos[0] - 1}) {
    if (nxc < 3 || nxc > n) continue;
    if (check_geom(n, rp_d, ci_d, (int)nxc, 1, g, st)) return true;
    // 3-D: the smallest offset beyond the x line is nx*ny + dy*nx + dx
    for (int64_t o2 : pos) {
      if (o2 <= nxc + 1) continue;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int64_t nxy = o2 - dy * nxc - dx;
          if (nxy % nxc != 0) continue;
          const int64_t nyc = nxy / nxc;
          if (nyc < 3 || n % nxy != 0) continue;
          if (check_geom(n, rp_d, ci_d, (int)nxc, (int)nyc, g, st)) return true;
        }
      break;
    }
  }
  g = StencilGeom{};
  return false;
}

bool stencil_prepare(StencilPlan& sp, const StencilGeom& g, const void* X, int cc, int elem,
                     int zb, int ze) {
  sp.on = false;
  if (ze < 0) ze = g.nz;
  if (zb < 0 || ze > g.nz || zb >= ze) return false;
  sp.zb = zb;
  sp.ze = ze;
  const int nzr = ze - zb;
  if (!stencil_env_enabled() || g.nx == 0) return false;
  if ((size_t)cc * elem % kSliceBytes != 0 || (uintptr_t)X % 16 != 0) return false;
  auto enc = encode_tiled();
  if (!enc) return false;
  sp.g = g;
  sp.elem = elem;
  sp.cc = cc;
  sp.M = 4;  // 8 points per warp measured slower (register pressure, fewer warps)
  sp.cw = (int)(kSliceBytes / elem);
  sp.slices = (int)((size_t)cc * elem / kSliceBytes);
  // warps per CTA: 2-D tiles of 4 warps (32 points, small planes, several
  // CTAs per SM with a deep ring); 3-D tiles of 8 x 8 points (one CTA per SM)
  const int nw_env = env_int("TFG_STENCIL_NW", 0);
  sp.nw = nw_env == 4 || nw_env == 8 ? nw_env : 4;
  if (g.d3) {
    sp.ty = sp.nw;
    sp.tx = sp.M;
    sp.tyh = sp.ty + 2;
  } else {
    sp.ty = 1;
    sp.tx = sp.M * sp.nw;
    sp.tyh = 1;
  }
  sp.ntx = (g.nx + sp.tx - 1) / sp.tx;
  sp.nty = (g.ny + sp.ty - 1) / sp.ty;
  sp.plane_bytes = (size_t)sp.cw * (sp.tx + 2) * sp.tyh * elem;
  // per warp: 3 value slots + 8 row-pointer slots (consumer cp.async ring)
  const size_t vslot = std::max<size_t>((sp.M * (g.d3 ? 27 : 9) + 31) / 32 * 32,
                                        (size_t)sp.M * 4 * (g.d3 ? 9 : 3));
  const size_t vbytes = (size_t)sp.nw * ((g.d3 ? kValueSlots<true> : kValueSlots<false>) * vslot * elem +
                                         8 * 16 * 4);
  // CTAs per SM, then the deepest ring that fits (>= 3 planes in use)
  const int per_env = env_int("TFG_STENCIL_CTAS", 0);
  // 3-D, 4 warps: 2 CTAs per SM with a 4-plane ring measured best (cfg4 per
  // pass: 1.264 ms; 3 CTAs with the 2-plane ring they leave room for: 1.281)
  int per_sm = per_env > 0 ? std::min(per_env, sp.nw == 8 ? 2 : 4)
                           : (sp.nw == 8 ? (g.d3 ? 1 : 2) : (g.d3 ? 2 : 3));
  // 2-D: planes z-1, z, z+1 in use; 3-D (z-sliding): one plane in use + prefetch
  const int min_ns = g.d3 ? 2 : 3;
  int ns = 0;
  for (; per_sm >= 1; --per_sm) {
    const size_t budget = kSmemBudget / per_sm - (per_sm > 1 ? 1024 : 0);
    ns = (int)std::min<size_t>(kMaxNS, (budget - std::min(budget, vbytes)) / sp.plane_bytes);
    if (ns >= min_ns) break;
  }
  if (per_sm < 1 || ns < min_ns) return false;
  const int ns_env = env_int("TFG_STENCIL_NS", 0);
  if (ns_env >= min_ns) ns = std::min(ns, ns_env);
  sp.ns = ns;
  sp.smem = ns * sp.plane_bytes + vbytes;
  sp.per_sm = per_sm;
  sp.grid = sm_count() * per_sm;
  // z chunk: balance items over the persistent grid (each item re-reads two
  // halo planes)
  const int64_t tiles = (int64_t)sp.ntx * sp.nty * sp.slices;
  const int zc_env = env_int("TFG_STENCIL_ZC", 0);
  int best = nzr;
  double best_cost = 1e300;
  // 2-D: short chunks measured best on cfg2 (16 planes: 0.239 ms vs 0.26 at
  // 24-28).  3-D: an item pays its two extra planes and a prologue, and face
  // groups cost what interior groups do, so long chunks win (cfg4 per pass:
  // 16 planes 1.355 ms, 32 1.313, 64 1.304, 128 1.297)
  for (int zc = std::min(8, nzr); zc <= (g.d3 ? std::max(1, nzr) : std::min(16, std::max(1, nzr)));
       ++zc) {
    const int64_t nzc = (nzr + zc - 1) / zc;
    const int64_t items = tiles * nzc;
    const double waves = (double)((items + sp.grid - 1) / sp.grid);
    const double cost = waves * (zc + 2);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = zc;
    }
  }
  sp.zc = zc_env > 0 ? zc_env : best;
  sp.nzc = (nzr + sp.zc - 1) / sp.zc;
  sp.items = tiles * sp.nzc;
  sp.grid = (int)std::min<int64_t>(sp.grid, sp.items);
  cuuint64_t dims[4] = {(cuuint64_t)cc, (cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz};
  cuuint64_t strides[3] = {(cuuint64_t)cc * elem, (cuuint64_t)cc * elem * g.nx,
                           (cuuint64_t)cc * elem * g.nx * g.ny};
  cuuint32_t box[4] = {(cuuint32_t)sp.cw, (cuuint32_t)(sp.tx + 2), (cuuint32_t)sp.tyh, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (enc(&sp.xmap, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
          4, const_cast<void*>(X), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  sp.on = true;
  return true;
}

template <class T, bool D3, int NW, int MINB, bool EXACT>
static void stencil_launch(const StencilPlan& sp, const StencilArgs& a, cudaStream_t st) {
  auto kern = k_spmm_stencil<T, D3, NW, 4, MINB, EXACT>;
  TFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.smem));
  kern<<<sp.grid, (NW + 1) * 32, sp.smem, st>>>(sp.xmap, a);
  TFG_LAUNCH_CHECK();
}

// register budget cut for the resident CTAs per SM the plan chose
template <class T, bool D3, bool EXACT>
static void stencil_launch_d(const StencilPlan& sp, const StencilArgs& a, cudaStream_t st) {
  const int r = sp.per_sm;
  if (sp.nw == 8) {
    if (r >= 2)
      stencil_launch<T, D3, 8, 2, EXACT>(sp, a, st);
    else
      stencil_launch<T, D3, 8, 1, EXACT>(sp, a, st);
  } else {
    if (r >= 4)
      stencil_launch<T, D3, 4, 4, EXACT>(sp, a, st);
    else if (r == 3)
      stencil_launch<T, D3, 4, 3, EXACT>(sp, a, st);
    else
      stencil_launch<T, D3, 4, 2, EXACT>(sp, a, st);
  }
}

template <class T>
static void stencil_launch_t(const StencilPlan& sp, const StencilArgs& a, cudaStream_t st,
                             bool exact) {
  if (sp.g.d3) {
    if (exact)
      stencil_launch_d<T, true, true>(sp, a, st);
    else
      stencil_launch_d<T, true, false>(sp, a, st);
  } else {
    if (exact)
      stencil_launch_d<T, false, true>(sp, a, st);
    else
      stencil_launch_d<T, false, false>(sp, a, st);
  }
}

void stencil_run(const StencilPlan& sp, const int* rp, const int* ci, const void* av, void* out,
                 cudaStream_t st, bool exact) {
  StencilArgs a{};
  const StencilGeom& g = sp.g;
  a.n = g.nx * g.ny * g.nz;
  a.nx = g.nx;
  a.ny = g.ny;
  a.nz = g.nz;
  a.nxy = g.nx * g.ny;
  a.zb = sp.zb;
  a.ze = sp.ze;

  a.zc = sp.zc;
  a.ns = sp.ns;
  a.slices = sp.slices;
  a.ntx = sp.ntx;
  a.nty = sp.nty;
  a.cc = sp.cc;
  a.items = sp.items;
  a.nzc = sp.nzc;
  a.plane_elems = (int)(sp.plane_bytes / sp.elem);
  a.op.K = g.K;
  a.op.full = g.K == (g.d3 ? 27 : 9);
  memcpy(a.op.rank, g.rank, sizeof(g.rank));
  a.op.used = 0;
  for (int q = 0; q < 27; ++q)
    if (g.rank[q] >= 0) a.op.used |= 1u << q;
  a.op.rp = rp;
  a.op.ci = ci;
  a.op.av = av;
  a.out = out;
  if (sp.elem == 8)
    stencil_launch_t<double>(sp, a, st, exact);
  else
    stencil_launch_t<float>(sp, a, st, exact);
}

}  // namespace tfg
