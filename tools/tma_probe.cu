// TMA streaming probe: how fast can 148 persistent CTAs pull an n x 256 fp32
// matrix through a 16 KB-slot shared-memory ring, by the shape of the copy?
//   mode 0  2-D box 32 cols x 128 rows, 128-byte swizzle (k_tc_tiles' B loads)
//   mode 1  3-D view (32, 8, n), box 32 x 2 x 64: 256 contiguous bytes per row
//   mode 2  3-D view (32, 8, n), box 32 x 8 x 16: 16 KB contiguous
//   mode 3  cp.async.bulk 1-D, 16 KB contiguous (no tensor map)
// The consumer only releases the slot.  Prints GB/s per mode and ring depth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      " @!p bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}

constexpr int kSlot = 16 * 1024;

__global__ void __launch_bounds__(64, 1)
    k_stream(const __grid_constant__ CUtensorMap map, const float* src, int mode, int ring,
             long nblocks /* 128-row blocks */) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* base = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[8], empty[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < ring; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // producer
    uint32_t t = 0;
    for (long b = blockIdx.x; b < nblocks; b += gridDim.x)
      for (int c = 0; c < 8; ++c, ++t) {  // 8 slots of 16 KB per 128-row block
        const int s = t % ring;
        if (t >= (uint32_t)ring) bar_wait(&empty[s], ((t / ring) - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&full[s])),
                     "r"(kSlot)
                     : "memory");
        unsigned char* dst = base + (size_t)s * kSlot;
        const int r0 = (int)(b * 128);
        if (mode == 0)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(su32(dst)),
              "l"(reinterpret_cast<uint64_t>(&map)), "r"(c * 32), "r"(r0), "r"(su32(&full[s]))
              : "memory");
        else if (mode == 1)  // slot c: rows r0 + 64 (c / 4) .. + 64, chunk pair c % 4
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(su32(dst)),
              "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"((c % 4) * 2),
              "r"(r0 + 64 * (c / 4)), "r"(su32(&full[s]))
              : "memory");
        else if (mode == 2)  // slot c: rows r0 + 16 c .. + 16, all 8 chunks
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(su32(dst)),
              "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(0), "r"(r0 + 16 * c),
              "r"(su32(&full[s]))
              : "memory");
        else
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
                  "r"(su32(dst)),
              "l"(src + ((size_t)r0 + 16 * c) * 256), "r"(kSlot), "r"(su32(&full[s]))
              : "memory");
      }
  } else if (threadIdx.x == 32) {  // consumer
    uint32_t t = 0;
    for (long b = blockIdx.x; b < nblocks; b += gridDim.x)
      for (int c = 0; c < 8; ++c, ++t) {
        const int s = t % ring;
        bar_wait(&full[s], (t / ring) & 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&empty[s])) : "memory");
      }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long n = 1L << 21;  // 2 GiB of fp32 x 256
  float* B;
  cudaMalloc(&B, (size_t)n * 1024);
  cudaMemset(B, 0, (size_t)n * 1024);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap maps[3];
  {
    cuuint64_t dims[2] = {256, (cuuint64_t)n};
    cuuint64_t str[1] = {1024};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    enc(&maps[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  for (int m = 1; m <= 2; ++m) {
    cuuint64_t dims[3] = {32, 8, (cuuint64_t)n};
    cuuint64_t str[2] = {128, 1024};
    cuuint32_t box[3] = {32, m == 1 ? 2u : 8u, m == 1 ? 64u : 16u}, es[3] = {1, 1, 1};
    CUresult r = enc(&maps[m], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, B, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode mode %d failed: %d\n", m, (int)r);
  }
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kSlot + 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float* flush;
  cudaMalloc(&flush, 256 << 20);
  for (int mode = 0; mode < 4; ++mode)
    for (int ring : {4, 6, 8}) {
      float best = 1e9f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaMemsetAsync(flush, rep, 256 << 20);
        cudaEventRecord(e0);
        k_stream<<<sms, 64, ring * kSlot + 1024>>>(maps[mode < 3 ? mode : 0], B, mode, ring, n / 128);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      printf("{\"mode\": %d, \"ring\": %d, \"ms\": %.4f, \"GBs\": %.1f, \"status\": \"%s\"}\n", mode,
             ring, best, (double)n * 1024 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
