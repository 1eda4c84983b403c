// tfg_stencil.cuh -- SpMM for CSR matrices that are stencils on a regular grid.
//
// The SpMM-SpMM configurations of BASELINE.json (9-point on 1024^2, 27-point
// on 128^3) are matrices whose every nonzero (r, c) joins a grid point r to a
// neighbour: c - r = dz*nx*ny + dy*nx + dx with dx, dy, dz in {-1, 0, 1} and
// the neighbour inside the grid.  For those the plan replaces the row-list
// SpMM (kernels.hpp:71-80, spmm_row) by a plane-streaming kernel: a CTA owns a
// tile of the grid's (x, y) plane and walks the z axis; each X plane of the
// tile (with a one-point halo) is fetched by ONE 4-D TMA copy into a ring of
// shared-memory planes, so every X row crosses L2 -> SM about once instead
// of once per nonzero.  A warp computes M consecutive points of a tile line,
// streaming the M + 2 X rows of each (dz, dy) line through registers and
// adding each row's product to the up-to-three points that use it.  Every
// output row still sums its nonzeros from 0 in ascending column order with
// separate multiply and add roundings, so the result is bit-identical to the
// reference's spmm_row.  Rows with fewer nonzeros than the full stencil (grid
// faces) take a per-row path inside the same kernel, reading their column
// indices; full rows never read col_idx.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "tfg_common.cuh"

namespace tfg {

struct StencilGeom {
  int nx = 0, ny = 1, nz = 0;  // row r = (z * ny + y) * nx + x
  bool d3 = false;             // ny > 1: 27-point family; else 9-point family
  int K = 0;                   // nonzeros of a full (interior) row
  // rank[((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1)]: position of that neighbour
  // in a full row's CSR order, -1 when the stencil does not use it
  int8_t rank[27] = {};
};

struct StencilPlan {
  bool on = false;
  StencilGeom g;
  int elem = 8;
  int cc = 0;
  int M = 8;            // points per warp
  int nw = 8;           // compute warps per CTA
  int tx = 0, ty = 1;   // tile of the (x, y) plane, points
  int tyh = 1;          // tile rows incl. halo along y (ty + 2, or 1 in 2-D)
  int zc = 0;           // z planes (outputs) per work item
  int zb = 0, ze = 0;   // planes computed (row-block partitions: a slab)
  int ns = 3;           // shared-memory plane ring depth
  int cw = 0;           // column slice per CTA (elements, 512 bytes)
  int slices = 0;       // cc / cw
  int ntx = 0, nty = 0, nzc = 0;
  int64_t items = 0;
  size_t plane_bytes = 0, smem = 0;
  size_t plane2_bytes = 0;  // fused kernel: D1 plane
  StencilGeom g2;           // fused kernel: A's stencil (g is B's)
  int per_sm = 1;       // resident CTAs per SM the launch is built for
  int grid = 0;
  alignas(64) CUtensorMap xmap;  // X as (cc, nx, ny, nz), box (cw, tx + 2, tyh, 1)
};

// Detect the stencil structure of an n x n CSR: candidate geometries from a
// sample of rows (host row_ptr, a few device column indices), each checked
// over every nonzero on the device (in-grid neighbour, strictly increasing
// columns).  false: not a grid stencil.
bool stencil_detect(int n, const std::vector<int>& rp, const int* rp_d, const int* ci_d,
                    StencilGeom& g, cudaStream_t st);
// Tile the grid for X (n x cc row-major, element size elem bytes) and encode
// the X tensor map.  false: shape not supported (the plan keeps its SpMM).
// Planes [zb, ze) only (a row-block partition; -1: the whole grid).
bool stencil_prepare(StencilPlan& sp, const StencilGeom& g, const void* X, int cc, int elem,
                     int zb = 0, int ze = -1);
// out[r, :] = sum_k av[k] * X[ci[k], :] over every row r of the matrix, in
// ascending k; exact: separately rounded mul and add (the reference's bits),
// else one fused multiply-add per term.
void stencil_run(const StencilPlan& sp, const int* rp, const int* ci, const void* av, void* out,
                 cudaStream_t st, bool exact);
int stencil_env_enabled();  // TFG_STENCIL (default 1)

}  // namespace tfg
