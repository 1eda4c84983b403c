// TMA tile::gather4 probe: 4 rows of a row-major fp32 matrix (n x 64) by
// index into shared memory with one cp.async.bulk.tensor instruction, checked
// against the source rows, and a throughput estimate for random row gathers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_probe tools/gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_gather4(const __grid_constant__ CUtensorMap map, const int* rows, int nrows,
                          int reps, float* out, int check) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* ring = reinterpret_cast<float*>(sm) + (size_t)w * 8 * 256;  // 8 slots of 4 x 64 floats
  __shared__ __align__(8) uint64_t wbar[32][8];
  if (lane < 8) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&wbar[w][lane])));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  float acc = 0.f;
  const int gw = blockIdx.x * (blockDim.x >> 5) + w, nw = gridDim.x * (blockDim.x >> 5);
  uint32_t phase = 0;
  for (int r = 0; r < reps; ++r) {
    for (int g = gw * 32; g + 32 <= nrows; g += nw * 32) {  // 8 gathers of 4 rows in flight
      if (lane == 0) {
        for (int s = 0; s < 8; ++s) {
          const int* q = rows + g + 4 * s;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&wbar[w][s])),
                       "r"(4 * 256) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(su32(ring + s * 256)),
              "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]),
              "r"(su32(&wbar[w][s]))
              : "memory");
        }
      }
      for (int s = 0; s < 8; ++s) {
        asm volatile(
            "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra W_%=;\n}\n" ::"r"(su32(&wbar[w][s])), "r"(phase) : "memory");
        const float* x = ring + s * 256;
        if (check && r == 0)
          for (int q = 0; q < 4; ++q) {
            out[(size_t)(g + 4 * s + q) * 64 + lane] = x[q * 64 + lane];
            out[(size_t)(g + 4 * s + q) * 64 + 32 + lane] = x[q * 64 + 32 + lane];
          }
        acc += x[lane] + x[64 + lane] + x[128 + lane] + x[192 + lane];
      }
      phase ^= 1u;
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const int n = 1 << 23, cc = 64, nrows = 1 << 22;
  std::vector<float> h((size_t)n * cc);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 1000003) * 0.5f;
  std::vector<int> rows(nrows);
  uint64_t x = 88172645463325252ull;
  for (int i = 0; i < nrows; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    rows[i] = (int)(x % n);
  }
  float *d, *o;
  int* r;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, (size_t)nrows * cc * 4);
  cudaMalloc(&r, nrows * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(r, rows.data(), nrows * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)cc, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)cc * 4};
  cuuint32_t box[2] = {(cuuint32_t)cc, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult e = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)e);
  const int threads = 256, smem = 8 * 8 * 1024 + 1024;
  cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_gather4<<<148, threads, smem>>>(map, r, nrows, 1, o, 1);
  cudaError_t err = cudaDeviceSynchronize();
  printf("check run: %s\n", cudaGetErrorString(err));
  if (err != cudaSuccess) return 1;
  std::vector<float> got((size_t)nrows * cc);
  cudaMemcpy(got.data(), o, got.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  const int covered = nrows / (148 * 8 * 32) * (148 * 8 * 32);
  for (int i = 0; i < covered; ++i)
    for (int c = 0; c < cc; ++c)
      if (got[(size_t)i * cc + c] != h[(size_t)rows[i] * cc + c]) ++bad;
  printf("mismatches: %ld of %ld\n", bad, (long)covered * cc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int blocks : {148, 296}) {
    cudaEventRecord(a);
    k_gather4<<<blocks, threads, smem>>>(map, r, nrows, 4, o, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 4.0 * covered * cc * 4;
    printf("gather4 random rows, %d CTAs x 8 warps x 8 in flight: %.3f ms, %.1f GB/s\n", blocks, ms,
           bytes / (ms * 1e-3) / 1e9);
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
