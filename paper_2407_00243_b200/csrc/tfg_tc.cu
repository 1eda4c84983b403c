// tfg_tc.cu -- FP32 first op on tcgen05 tensor cores (3xTF32), optionally
// fused with the wavefront-0 tile's SpMM rows.  See tfg_tc.cuh.
//
// Per CTA (one per SM, 576-704 threads, persistent over tiles):
//   warp 0      TMA producer: 128-row x 32-column fp32 blocks of B land in a
//               ring of raw shared-memory slots (128-byte swizzle); the CTA's
//               C slice (pre-split tf32 hi/lo image, K-major) is bulk-copied
//               once and stays resident.
//   warps 1-C   converters (C = 4 or 8), a block row per 4 warps: read values,
//               split x = hi + lo (tf32 each, error < 2^-20 x), free the raw
//               slot and tcgen05.st both planes into a TMEM operand stage.
//   warp C+1    one lane issues tcgen05.mma kind::tf32 with A from TMEM and
//               B (C) from shared memory, M=128, N=BN, K=8:
//               D += B_lo C_hi + B_hi C_lo + B_hi C_hi into one of two TMEM
//               accumulators; tcgen05.commit frees operand stages and hands
//               finished accumulators to the epilogue.
//   last E      epilogue (E = 16 or 8): tcgen05.ld rows out of TMEM, write D1 rows that
//               wavefront 1 reads (spill) or that no stage holds (wide tile),
//               stage rows the tile's fused rows read, then compute those
//               fused rows (spmm_row, reference order) into D.
// Shared memory carries only the raw B blocks and C: the split operand lives
// in TMEM, so the MMAs do not compete with the converters for SMEM bandwidth.
// The algorithm is the reference's (kernels.hpp:88-126: first-op rows of a
// tile, then its fused rows); only the arithmetic of the dense product is the
// tensor cores' (error ~1e-6 relative, inside the 1e-5 fp32 tolerance).
#include "tfg_tc.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "tfg_device.cuh"

namespace tfg {
namespace {

using namespace dev;

constexpr int kStages = 4;
constexpr int kBM = 128;                      // rows per MMA block (M)
constexpr int kKC = 32;                       // K per ring chunk (one 128-byte swizzle row)
constexpr int kChunkBytes = kBM * kKC * 4;    // 16 KB
// warp roles: 0 TMA producer, 1..CONV converters, CONV+1 MMA issuer, then
// EPI epilogue / fused-row warps.  First-op launches (no fused rows) use
// 8 + 8; fused tiles 4 + 16 (the fused rows need the warps, the 4-op split
// does not).
template <int CONV, int EPI>
struct Roles {
  static constexpr int kConv = CONV;
  static constexpr int kEpi = EPI;
  static constexpr int kMmaWarp = 1 + CONV;
  static constexpr int kEpi0 = kMmaWarp + 1;
  static constexpr int kThreads = 32 * (kEpi0 + EPI);
  static_assert(CONV == 4 || CONV == 8, "converter warps");
  static_assert(EPI % 4 == 0 && EPI >= 4, "epilogue warps");
};
constexpr size_t kCMax = 128 * 1024;          // resident C slice image (hi + lo)
constexpr size_t kSmemMax = 227 * 1024;
constexpr size_t kBarBytes = 384;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n TC_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      " @!p bra TC_WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// K-major operand, 128-byte swizzle: 8-row atoms of 128 B, atoms 1 KB apart
// (SBO), version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Both tcgen05.mma and tcgen05.commit are issued from warp-uniform code by the
// lane elect.sync picks (the same lane every time for the full mask): inside
// an `if (lane == 0)` region the compiler wraps every uniform-datapath
// instruction in an ELECT / BRA.U.ANY loop, ~10 instructions per MMA that made
// the issuing thread the slowest stage of the pipeline.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          su32(bar))
      : "memory");
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// C (bc x cc, row-major) -> per column slice y and K chunk kc: [hi | lo] planes
// of BN rows (output columns) x 32 K values, 128-byte swizzled (16-byte unit
// u of row r stored at u ^ (r % 8)), i.e. the K-major operand image.
__global__ void k_tc_prep_c(const float* __restrict__ C, int bc, int cc, int bn,
                            float* __restrict__ img) {
  const int64_t total = (int64_t)bc * cc;
  const int kchunks = bc / kKC;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / cc), col = (int)(e % cc);
    const float x = C[e];
    const float h = tf32_rna(x), l = tf32_rna(x - h);
    const int y = col / bn, nl = col % bn, kc = k / kKC, kk = k % kKC;
    const size_t base = (size_t)(y * kchunks + kc) * 2 * bn * kKC;
    const size_t w = (size_t)(nl / 8) * 256 + (nl % 8) * 32 + (((kk / 4) ^ (nl % 8)) * 4) + kk % 4;
    img[base + w] = h;
    img[base + (size_t)bn * kKC + w] = l;
  }
}

// 16 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// 16 consecutive fp32 columns into this thread's TMEM lane.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};\n" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
// x = hi + lo with hi = x truncated to tf32 (exact) and lo = x - hi (exact in
// fp32, |lo| < 2^-10 |x|); the tensor core reads lo at tf32 precision, so the
// split represents x to 2^-20 relative.  Non-finite x: hi = x, lo = 0.
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = hi == x ? 0.f : x - hi;
}
// 4 x 4 transpose of float4 across each quad of lanes: on entry lane 4k + j
// holds v[c] = columns 4c .. 4c+3 of row 4k + j; on exit v[i] = columns
// 4j .. 4j+3 of row 4k + i.  A warp store of v[i] then writes 8 rows x 64
// contiguous bytes (8 lines) instead of 32 rows x 16 bytes (32 lines).
__device__ __forceinline__ float4 shfl_xor4(const float4& a, int m) {
  return make_float4(__shfl_xor_sync(0xffffffffu, a.x, m), __shfl_xor_sync(0xffffffffu, a.y, m),
                     __shfl_xor_sync(0xffffffffu, a.z, m), __shfl_xor_sync(0xffffffffu, a.w, m));
}
__device__ __forceinline__ void quad_transpose(float4 (&v)[4], int lane) {
  const bool b1 = (lane & 2) != 0, b0 = (lane & 1) != 0;
  {  // exchange 2 x 2 blocks with lane ^ 2
    const float4 s0 = b1 ? v[0] : v[2], s1 = b1 ? v[1] : v[3];
    const float4 r0 = shfl_xor4(s0, 2), r1 = shfl_xor4(s1, 2);
    if (b1) {
      v[0] = r0;
      v[1] = r1;
    } else {
      v[2] = r0;
      v[3] = r1;
    }
  }
  {  // exchange inside the 2 x 2 blocks with lane ^ 1
    const float4 s0 = b0 ? v[0] : v[1], s1 = b0 ? v[2] : v[3];
    const float4 r0 = shfl_xor4(s0, 1), r1 = shfl_xor4(s1, 1);
    if (b0) {
      v[0] = r0;
      v[2] = r1;
    } else {
      v[1] = r0;
      v[3] = r1;
    }
  }
}
// D[tmem] (+)= A[tmem] . B[smem desc]^T
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}

// TMEM columns: [0, NACC*BN) accumulators, then kOpStages x 64 operand
// columns (32 tf32 hi + 32 tf32 lo per row of the 128-row block).  Narrow
// slices get more accumulators: the MMAs then run up to NACC blocks ahead
// of the epilogue, which also computes the fused rows of finished tiles.
#ifndef TFG_TC_OPS
#define TFG_TC_OPS 4
#endif
#ifndef TFG_TC_NACC_MAX
#define TFG_TC_NACC_MAX 8
#endif
constexpr int kOpStages = TFG_TC_OPS;
constexpr uint32_t kTmemCols = 512;
template <int BN>
__host__ __device__ constexpr int nacc() {
  return ((int)kTmemCols - kOpStages * 64) / BN > TFG_TC_NACC_MAX
             ? TFG_TC_NACC_MAX
             : ((int)kTmemCols - kOpStages * 64) / BN;
}

template <int BN, int LPR, int CONV, int EPI>
__global__ void __launch_bounds__(Roles<CONV, EPI>::kThreads, 1)
    k_tc_tiles(const __grid_constant__ CUtensorMap bmap, int kchunks, int raw_stages, int dbg_arg,
               const float* __restrict__ cimg, int64_t ntiles, const int* __restrict__ t_ilo,
               const int* __restrict__ t_ihi, const int64_t* __restrict__ t_joff,
               const int* __restrict__ jrows, const uint8_t* __restrict__ t_wide,
               const int* __restrict__ slot, const uint8_t* __restrict__ spill, int stage_cap,
               int cc, const int* __restrict__ fx_aoff, const int64_t* __restrict__ fx_off,
               const int* __restrict__ fx_idx, const float* __restrict__ av, float* D1,
               float* __restrict__ D, const int* __restrict__ order) {
  // timing experiments (wrong D): only in builds with -DTFG_TC_TIMING=1, where
  // TFG_TC_DBGX selects pipeline stages to skip; 0 and folded away otherwise
#ifdef TFG_TC_TIMING
  const int dbg = dbg_arg;
#else
  constexpr int dbg = 0;
  (void)dbg_arg;
#endif
  using R = Roles<CONV, EPI>;
  constexpr int kConv = R::kConv, kEpi = R::kEpi, kMmaWarp = R::kMmaWarp, kEpi0 = R::kEpi0;
  constexpr int VEC = 4;
  // fused rows: 8 lanes per row (4 rows in flight per warp), NCH x 16 B each
  constexpr int LPR2 = 8;
  constexpr int NCH = BN / (LPR2 * VEC);
  static_assert(NCH >= 1 && NCH * LPR2 * VEC == BN, "slice width");
  static_assert(LPR >= 1, "unused");
  constexpr int NACC = nacc<BN>();
  static_assert(NACC >= 2 && NACC * BN + kOpStages * 64 <= (int)kTmemCols, "TMEM budget");
  constexpr int kEpiGroups = kEpi / 4;  // epilogue warps per TMEM lane quarter
  static_assert(BN % 16 == 0, "epilogue column chunks");
  constexpr uint32_t kIdesc = (1u << 4)                       // D format f32
                              | (2u << 7) | (2u << 10)        // A, B format tf32
                              | ((uint32_t)(BN >> 3) << 17)   // N
                              | ((uint32_t)(kBM >> 4) << 24); // M
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  const size_t cbytes = (size_t)kchunks * 2 * BN * kKC * 4;
  float* sc = reinterpret_cast<float*>(base);
  unsigned char* ring = base + cbytes;  // raw_stages x 16 KB of fp32 B blocks (swizzled)
  float* stage = reinterpret_cast<float*>(ring + (size_t)raw_stages * kChunkBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage + (size_t)stage_cap * BN);
  uint64_t* raw_full = bars;                   // [raw_stages] TMA landed
  uint64_t* raw_empty = bars + raw_stages;     // [raw_stages] converters read it
  uint64_t* op_full = raw_empty + raw_stages;  // [kOpStages] hi/lo in TMEM
  uint64_t* op_empty = op_full + kOpStages;    // [kOpStages] MMAs done with it
  uint64_t* acc_full = op_empty + kOpStages;   // [NACC]
  uint64_t* acc_empty = acc_full + NACC;       // [NACC]
  uint64_t* c_full = acc_empty + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(c_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.y * BN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < raw_stages; ++s) {
      bar_init(&raw_full[s], 1);
      bar_init(&raw_empty[s], kConv * 32);
    }
    for (int s = 0; s < kOpStages; ++s) {
      bar_init(&op_full[s], kConv * 32);
      bar_init(&op_empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      bar_init(&acc_full[a], 1);
      bar_init(&acc_empty[a], kEpi * 32);
    }
    bar_init(c_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t op_col0 = NACC * BN;

  if (warp == 0) {
    if (lane == 0) {
      const float* csrc = cimg + (size_t)blockIdx.y * kchunks * 2 * BN * kKC;
      bar_expect(c_full, (uint32_t)cbytes);
      for (size_t off = 0; off < cbytes; off += 16384)
        bulk_1d(reinterpret_cast<unsigned char*>(sc) + off,
                reinterpret_cast<const unsigned char*>(csrc) + off,
                (uint32_t)(cbytes - off < 16384 ? cbytes - off : 16384), c_full);
      int s = 0;
      uint32_t ph = 1;  // parity of the slot's previous use (first round: nothing to wait for)
      bool wrapped = false;
      for (int64_t vi = blockIdx.x; vi < ntiles; vi += gridDim.x) {
        const int64_t v = order ? order[vi] : vi;  // plan-time balanced tile order (-1: none)
        if (v < 0) continue;
        const int ilo = t_ilo[v], ihi = t_ihi[v];
        for (int r0 = ilo; r0 < ihi; r0 += kBM)
          for (int kc = 0; kc < kchunks; ++kc) {
            if (wrapped) bar_wait(&raw_empty[s], ph);
            bar_expect(&raw_full[s], kChunkBytes);
            tma_2d(ring + (size_t)s * kChunkBytes, &bmap, kc * kKC, r0, &raw_full[s]);
            if (++s == raw_stages) {
              s = 0;
              ph ^= 1u;
              wrapped = true;
            }
          }
      }
    }
  } else if (warp <= kConv) {
    // converters: one row of the 128-row block per thread (kConv = 4: both
    // 16-value halves in turn; kConv = 8: one half), TMEM lane quarter =
    // warp % 4 (the lanes a warp may access)
    const int q = warp & 3, hpart = (warp - 1) >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_bits = (uint32_t)(q * 32) << 16;
    // The converters need no tile structure: the CTA's chunks are one flat
    // sequence (chunk t lives in raw slot t % raw_stages, operand stage
    // t % kOpStages).  A thread's work is split into units of 16 values (one
    // 64-byte half row): both halves of every chunk (kConv = 4) or its own
    // half (kConv = 8).  The shared-memory loads of unit u + 1 are issued
    // before unit u is split and stored to TMEM, so the load latency (several
    // hundred cycles beside the TMA writes and the MMA operand reads) is off
    // the per-chunk critical path.
    uint32_t nchunks = 0;
    for (int64_t vi = blockIdx.x; vi < ntiles; vi += gridDim.x) {
      const int64_t v = order ? order[vi] : vi;
      if (v < 0) continue;
      nchunks += (uint32_t)((t_ihi[v] - t_ilo[v] + kBM - 1) / kBM) * (uint32_t)kchunks;
    }
    constexpr int kUnits = kConv == 4 ? 2 : 1;  // units per chunk and thread
    const uint32_t nunits = nchunks * kUnits;
    int ls = 0, cs = 0;       // raw slot of the chunk being loaded / converted
    uint32_t lph = 0;         // raw_full parity of the chunk being loaded
    const unsigned char* rowp = ring + (size_t)r * 128;
    auto load = [&](uint32_t u, float4 (&x)[4]) {
      const int hh = kUnits == 2 ? (int)(u & 1) : hpart;
      if (kUnits == 1 || (u & 1) == 0) bar_wait(&raw_full[ls], lph);
      const float4* src = reinterpret_cast<const float4*>(rowp + (size_t)ls * kChunkBytes);
#pragma unroll
      for (int k = 0; k < 4; ++k) x[k] = src[(hh * 4 + k) ^ (r & 7)];
      if (kUnits == 1 || (u & 1) == 1) {
        if (++ls == raw_stages) {
          ls = 0;
          lph ^= 1u;
        }
      }
    };
    auto convert = [&](uint32_t u, const float4 (&x)[4]) {
      const uint32_t t = u / kUnits;
      const int hh = kUnits == 2 ? (int)(u & 1) : hpart;
      const bool first = kUnits == 1 || (u & 1) == 0, last = kUnits == 1 || (u & 1) == 1;
      const int so = (int)(t % kOpStages);
      float h[16], l[16];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        split_tf32(x[k].x, h[4 * k], l[4 * k]);
        split_tf32(x[k].y, h[4 * k + 1], l[4 * k + 1]);
        split_tf32(x[k].z, h[4 * k + 2], l[4 * k + 2]);
        split_tf32(x[k].w, h[4 * k + 3], l[4 * k + 3]);
      }
      if (last) {
        // the slot is refilled by the TMA (async proxy): order this thread's
        // (completed) generic reads before that write, then release the slot
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        bar_arrive(&raw_empty[cs]);
        if (++cs == raw_stages) cs = 0;
      }
      if (first && t >= (uint32_t)kOpStages)
        bar_wait(&op_empty[so], ((t / kOpStages) - 1) & 1);
      tc_fence_after();
      const uint32_t col = tmem + lane_bits + op_col0 + (uint32_t)so * 64 + hh * 16;
      if (!(dbg & 16)) {
        tmem_st16(col, h);
        tmem_st16(col + 32, l);
      }
      if (last) {
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        bar_arrive(&op_full[so]);
      }
    };
    float4 xa[4], xb[4];
    if (nunits) load(0, xa);
    for (uint32_t u = 0; u < nunits; u += 2) {
      if (u + 1 < nunits) load(u + 1, xb);
      convert(u, xa);
      if (u + 2 < nunits) load(u + 2, xa);
      if (u + 1 < nunits) convert(u + 1, xb);
    }
  } else if (warp == kMmaWarp) {
    {  // the whole warp walks the loop; one elected lane issues (see mma_tf32_ts)
      bar_wait(c_full, 0);
      const uint32_t sc_addr = su32(sc);
      uint32_t t = 0, b = 0;
      for (int64_t vi = blockIdx.x; vi < ntiles; vi += gridDim.x) {
        const int64_t v = order ? order[vi] : vi;  // plan-time balanced tile order (-1: none)
        if (v < 0) continue;
        const int ilo = t_ilo[v], ihi = t_ihi[v];
        for (int r0 = ilo; r0 < ihi; r0 += kBM, ++b) {
          const int a = b % NACC;
          if (b >= (uint32_t)NACC) bar_wait(&acc_empty[a], ((b / NACC) - 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(a * BN);
          for (int kc = 0; kc < kchunks; ++kc, ++t) {
            const int so = t % kOpStages;
            bar_wait(&op_full[so], (t / kOpStages) & 1);
            tc_fence_after();
            const uint32_t ah = tmem + op_col0 + (uint32_t)so * 64, al = ah + 32;
            const uint32_t ch = sc_addr + (uint32_t)(kc * 2 * BN * kKC * 4),
                           cl = ch + (uint32_t)(BN * kKC * 4);
            // the C image is 1024-byte aligned and each plane a multiple of 1 KB:
            // one descriptor per plane, the K step advances its address field
            const uint64_t dh = sw128_desc(ch), dl = sw128_desc(cl);
            if (elect_one()) {
#pragma unroll
              for (int ks = 0; ks < kKC / 8; ++ks) {
                const uint64_t o = (uint64_t)(ks * 32 >> 4);  // 8 tf32 = 32 bytes of the swizzled row
                if (!(dbg & 1)) mma_tf32_ts(d, al + ks * 8, dh + o, kIdesc, (kc | ks) != 0);
                if (!(dbg & 2)) mma_tf32_ts(d, ah + ks * 8, dl + o, kIdesc, 1);
                if (!(dbg & 32)) mma_tf32_ts(d, ah + ks * 8, dh + o, kIdesc, (dbg & 1) ? (kc | ks) != 0 : 1);
              }
              mma_commit(&op_empty[so]);
              if (kc == kchunks - 1) mma_commit(&acc_full[a]);
            }
            __syncwarp();
          }
        }
      }
    }
  } else {
    // epilogue warps: TMEM lane quarter = warp % 4, column chunks of 16
    // interleaved over the kEpiGroups warps of a quarter
    const int et = threadIdx.x - kEpi0 * 32;
    const int q = warp & 3, g = (warp - kEpi0) >> 2;
    const int m = q * 32 + lane;
    const bool first_op = t_joff == nullptr;
    auto named_sync = [] { asm volatile("bar.sync 1, %0;\n" ::"n"(kEpi * 32) : "memory"); };
    const int gl = et & (LPR2 - 1);
    const unsigned gmask = group_mask(LPR2);
    const int group = et / LPR2, ngroups = kEpi * 32 / LPR2;
    uint32_t b = 0;
    for (int64_t vi = blockIdx.x; vi < ntiles; vi += gridDim.x) {
        const int64_t v = order ? order[vi] : vi;  // plan-time balanced tile order (-1: none)
        if (v < 0) continue;
      const int ilo = t_ilo[v], ihi = t_ihi[v];
      const bool wide = first_op || t_wide[v] != 0;
      for (int r0 = ilo; r0 < ihi; r0 += kBM, ++b) {
        const int a = b % NACC;
        bar_wait(&acc_full[a], (b / NACC) & 1);
        tc_fence_after();
        const int row = r0 + m;
        const bool valid = row < ihi;
        const bool sp = valid && (wide || spill[row]) && !(dbg & 4);
        const int sl = (valid && !wide && !(dbg & 8)) ? slot[row] : -1;
        // D1 rows go out transposed inside lane quads: lane 4k + j writes
        // columns 4j .. 4j+3 of rows 4k .. 4k+3 in turn (64 contiguous bytes
        // per row and instruction; the per-lane pattern cost 4x the LSU
        // store wavefronts, which the converters' shared-memory loads share)
        const unsigned spmask = __ballot_sync(0xffffffffu, sp);
        const int quad0 = lane & ~3, qj = lane & 3;
#pragma unroll
        for (int c0 = g * 16; c0 < BN; c0 += 16 * kEpiGroups) {
          float x[16];
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * BN + c0), x);
          if (sl >= 0) {
            float4* o = reinterpret_cast<float4*>(stage + (size_t)sl * BN + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              o[j] = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
          }
          if (spmask) {
            float4 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              v[j] = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
            quad_transpose(v, lane);
            float* o = D1 + (size_t)(r0 + q * 32 + quad0) * cc + n0 + c0 + 4 * qj;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if ((spmask >> (quad0 + i)) & 1u)
                *reinterpret_cast<float4*>(o + (size_t)i * cc) = v[i];
          }
        }
        tc_fence_before();
        bar_arrive(&acc_empty[a]);
      }
      if (first_op) continue;
      const int64_t jb = t_joff[v], je = t_joff[v + 1];
      if (je == jb || (dbg & 8)) continue;
      named_sync();  // staged / spilled rows visible
      for (int64_t qq = jb + group; qq < je; qq += ngroups) {
        const int j = jrows[qq];
        const int xb = (int)fx_off[qq], xe = (int)fx_off[qq + 1];
        const float* avj = av + __ldg(fx_aoff + qq);  // value of fused nonzero k: avj[k]
        float acc2[NCH][VEC];
        if (wide) {
          auto xl = [&](int c, int chn, float(&xx)[VEC]) {
            ldv<float, VEC>(xx, D1 + (size_t)c * cc + n0 + (chn * LPR2 + gl) * VEC);
          };
          spmm_row<float, VEC, LPR2, NCH>(xb, xe, fx_idx, avj, gl, gmask, xl, acc2);
        } else {
          auto xl = [&](int c, int chn, float(&xx)[VEC]) {
            ldv<float, VEC>(xx, stage + (size_t)c * BN + (chn * LPR2 + gl) * VEC);
          };
          spmm_row<float, VEC, LPR2, NCH>(xb, xe, fx_idx, avj, gl, gmask, xl, acc2);
        }
        float* o = D + (size_t)j * cc + n0;
#pragma unroll
        for (int chn = 0; chn < NCH; ++chn) stv<float, VEC>(o + (chn * LPR2 + gl) * VEC, acc2[chn]);
      }
      named_sync();  // stage free for the next tile
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(kTmemCols));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

int tc_timing_mask() {
#ifdef TFG_TC_TIMING
  const char* e = getenv("TFG_TC_DBGX");
  return e ? atoi(e) : 0;
#else
  return 0;
#endif
}

int env_raw_stages() {  // TFG_TC_RING: raw ring depth (tests stress 2)
  const char* e = getenv("TFG_TC_RING");
  const int v = e ? atoi(e) : kStages;
  return v < 2 ? 2 : (v > 8 ? 8 : v);
}

size_t fixed_bytes_bn(const TcPlan& tc, int bn) {
  return 1024 + (size_t)tc.kchunks * 2 * bn * kKC * 4 + (size_t)tc.raw * kChunkBytes + kBarBytes;
}
size_t fixed_bytes(const TcPlan& tc) { return fixed_bytes_bn(tc, tc.bn); }

}  // namespace

int tc_env_enabled() {
  const char* e = getenv("TFG_TC");
  return e ? atoi(e) : 1;
}

bool tc_prepare(TcPlan& tc, const float* B, int n, int bc, int cc) {
  tc.on = false;
  if (!tc_env_enabled()) return false;
  if (bc < kKC || bc % kKC != 0 || (uintptr_t)B % 16 != 0) return false;
  int bn = 0;
  for (int c : {128, 64, 32})  // widest slice whose split C fits (TMEM: 2*BN + 256 <= 512)
    if (cc % c == 0 && (size_t)bc * c * 8 <= kCMax) {
      bn = c;
      break;
    }
  if (!bn) return false;
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)bc, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)bc * 4};
  cuuint32_t box[2] = {(cuuint32_t)kKC, (cuuint32_t)kBM};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tc.bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(B), dims, strides, box,
          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  tc.bn = bn;
  tc.raw = env_raw_stages();
  if (fixed_bytes(tc) > kSmemMax) return false;
  tc.slices = cc / bn;
  tc.kchunks = bc / kKC;
  tc.cimg.alloc((size_t)bc * cc * 2);
  tc.stage_cap = 0;
  tc.smem = fixed_bytes(tc);
  tc.on = true;
  return true;
}

size_t tc_stage_bytes(const TcPlan& tc) { return tc_stage_bytes_bn(tc, tc.bn); }

size_t tc_stage_bytes_bn(const TcPlan& tc, int bn) {
  const size_t f = fixed_bytes_bn(tc, bn);
  return f < kSmemMax ? kSmemMax - f : 0;
}

void tc_set_bn(TcPlan& tc, int bn) {
  if (bn < 32 || bn % 32 != 0 || (tc.slices * tc.bn) % bn != 0)
    throw invalid_argument("tc: bad column slice");
  tc.slices = tc.slices * tc.bn / bn;
  tc.bn = bn;
  tc.smem = fixed_bytes(tc) + (size_t)tc.stage_cap * bn * 4;
}

void tc_finalize(TcPlan& tc, int stage_cap) {
  tc.stage_cap = stage_cap;
  tc.smem = fixed_bytes(tc) + (size_t)stage_cap * tc.bn * 4;
}

void tc_prep_c(const TcPlan& tc, const float* C, int bc, int cc, cudaStream_t st) {
  const int64_t total = (int64_t)bc * cc;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 8);
  k_tc_prep_c<<<blocks, 256, 0, st>>>(C, bc, cc, tc.bn, tc.cimg.p);
  TFG_LAUNCH_CHECK();
}

int64_t tc_grid(const TcPlan& tc, int64_t ntiles) {
  return std::min<int64_t>(ntiles, std::max<int64_t>(1, sm_count() / std::max(tc.slices, 1)));
}

void tc_run(const TcPlan& tc, int n, int bc, int cc, int64_t ntiles, const int* ilo,
            const int* ihi, const int64_t* joff, const int* jrows, const uint8_t* wide,
            const int* slot, const uint8_t* spill, const int* fx_aoff, const int64_t* fx_off,
            const int* fx_idx, const float* av, float* D1, float* D, cudaStream_t st,
            const int* order, int64_t norder) {
  (void)n;
  (void)bc;
  if (!ntiles) return;
  const bool fused = joff != nullptr;
  // first-op launches stage nothing: their shared memory goes to a deeper raw
  // ring (6 slots at bCol 256: first op 0.65 -> 0.60 ms on cfg5); TFG_TC_RING pins both
  int raw = tc.raw, stage_cap = tc.stage_cap;
  size_t smem = tc.smem;
  if (!fused) {
    stage_cap = 0;
    if (!getenv("TFG_TC_RING")) {
      const size_t base = fixed_bytes(tc) - (size_t)tc.raw * kChunkBytes;
      raw = (int)std::min<size_t>(8, (kSmemMax - base) / kChunkBytes);
      raw = std::max(raw, tc.raw);
    }
    smem = fixed_bytes(tc) + (size_t)(raw - tc.raw) * kChunkBytes;
  }
  auto launch = [&](auto kern, int threads) {
    TFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // all column slices of a tile run concurrently so B blocks are read from
    // HBM once and hit L2 for the other slices
    const int64_t gx = tc_grid(tc, ntiles);
    kern<<<dim3((unsigned)gx, (unsigned)tc.slices), threads, smem, st>>>(
        tc.bmap, tc.kchunks, raw, tc_timing_mask(), tc.cimg.p, order ? norder : ntiles, ilo, ihi, joff, jrows, wide,
        slot, spill, stage_cap, cc, fx_aoff, fx_off, fx_idx, av, D1, D, order);
  };
  using F = Roles<4, 16>;
  using U = Roles<8, 8>;
  if (tc.bn == 128)
    fused ? launch(k_tc_tiles<128, 32, 4, 16>, F::kThreads) : launch(k_tc_tiles<128, 32, 8, 8>, U::kThreads);
  else if (tc.bn == 64)
    fused ? launch(k_tc_tiles<64, 16, 4, 16>, F::kThreads) : launch(k_tc_tiles<64, 16, 8, 8>, U::kThreads);
  else
    fused ? launch(k_tc_tiles<32, 8, 4, 16>, F::kThreads) : launch(k_tc_tiles<32, 8, 8, 8>, U::kThreads);
  TFG_LAUNCH_CHECK();
}

}  // namespace tfg
