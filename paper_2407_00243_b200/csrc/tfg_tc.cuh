// tfg_tc.cuh -- FP32 first op D1 = B C on the 5th-generation tensor cores
// (tcgen05, TMEM accumulators, TMA-fed shared memory), 3xTF32 split so the
// result stays within the fp32 tolerance of the north star (1e-5 max-norm).
//
// Used for dense-B fp32 problems with bCol % 32 == 0 by both the first-op
// stage (row blocks that fuse nothing) and the fused wavefront-0 tiles (the
// same kernel then also computes the tile's fused D rows from the staged D1
// rows, kernels.hpp:104-116).  Every first-op path of a plan uses the same
// kernel, so fused and unfused execution stay bit-identical.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "tfg_common.cuh"

namespace tfg {

struct TcPlan {
  bool on = false;
  int bn = 0;         // column slice (MMA N)
  int slices = 0;     // cc / bn (gridDim.y)
  int kchunks = 0;    // bc / 32
  int raw = 4;        // raw B slots in the shared-memory ring
  int stage_cap = 0;  // staged D1 rows per fused tile
  size_t smem = 0;    // dynamic shared memory per CTA
  alignas(64) CUtensorMap bmap;  // B: n x bc fp32, box 32 x 128, 128B swizzle
  dbuf<float> cimg;   // C split into tf32 hi/lo, K-major, swizzled (smem image)
};

// Shape eligibility + tensor map + C image buffer.  false: use the FFMA path.
bool tc_prepare(TcPlan& tc, const float* B, int n, int bc, int cc);
// Shared memory left for the fused stage (bytes) once the ring and C fit.
size_t tc_stage_bytes(const TcPlan& tc);
size_t tc_stage_bytes_bn(const TcPlan& tc, int bn);
// Narrow the column slice (more slices, more room for the fused stage).
void tc_set_bn(TcPlan& tc, int bn);
void tc_finalize(TcPlan& tc, int stage_cap);
// Split + swizzle C into the image (one tiny kernel per execution).
void tc_prep_c(const TcPlan& tc, const float* C, int bc, int cc, cudaStream_t st);
// Tiles [ilo, ihi) of B's rows.  joff == nullptr: first-op mode (every row of
// every tile is written to D1, no fused rows).  Otherwise rows are written to
// D1 when spill[row] or the tile is wide, to the stage when slot[row] >= 0,
// and the tile's fused rows jrows[joff[v] .. joff[v+1]) are computed into D.
// fx_off / fx_idx: the fused rows' nonzeros as stage slots (staged tile) or
// D1 rows (wide tile), in jrows order; fused row q's values are
// av[fx_aoff[q] + k] for k in [fx_off[q], fx_off[q+1]) (live CSR values).
void tc_run(const TcPlan& tc, int n, int bc, int cc, int64_t ntiles, const int* ilo,
            const int* ihi, const int64_t* joff, const int* jrows, const uint8_t* wide,
            const int* slot, const uint8_t* spill, const int* fx_aoff, const int64_t* fx_off,
            const int* fx_idx, const float* av, float* D1, float* D, cudaStream_t st,
            const int* order = nullptr, int64_t norder = 0);
// CTAs along x of a launch over ntiles tiles (the persistent grid); order, when
// given, lists the tiles as order[k * tc_grid + b] = CTA b's k-th tile (-1: none)
int64_t tc_grid(const TcPlan& tc, int64_t ntiles);
int tc_env_enabled();  // TFG_TC (default 1)

}  // namespace tfg
