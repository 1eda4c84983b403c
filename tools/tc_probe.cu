// Tensor-pipe peak probe for the roofline denominators (bench.py "tensor"
// entry): back-to-back tcgen05.mma (cta_group::1, M = 128, N = 256) with both
// operands in shared memory (128-byte swizzled K-major descriptors) into a
// TMEM accumulator, one CTA per SM, one issuing thread per CTA.  Measures
// kind::tf32 (K = 8 per instruction) and kind::f16 with bf16 inputs (K = 16)
// so the tf32 figure can be read against the driver's cuBLAS bf16 peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe tools/tc_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <int KIND, int N = 256, bool TS = false>  // 0: tf32, 1: bf16; TS: A operand in TMEM
__global__ void __launch_bounds__(128, 1) k_probe(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* base = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  unsigned char* a = base;               // 128 rows x 128 B
  unsigned char* b = base + 16 * 1024;   // 256 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = 0x3f800000u ^ (i * 2654435761u & 0x007fffffu);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t d = tmem_base;
  constexpr uint32_t fmt = KIND == 0 ? 2u : 1u;  // tf32 : bf16
  constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint64_t da = sw128_desc(su32(a)), db = sw128_desc(su32(b));
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // 4 K steps of 32 bytes inside the 128-byte atom
        const uint64_t off = (uint64_t)(k * 32) >> 4;
        if (KIND == 0 && TS)
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
              "r"(d + 256 + k * 8), "l"(db + off), "r"(idesc), "r"(it | k));
        else if (KIND == 0)
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(da + off), "l"(db + off), "r"(idesc), "r"(it | k));
        else
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(da + off), "l"(db + off), "r"(idesc), "r"(it | k));
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            su32(&bar))
        : "memory");
    asm volatile(
        "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, 1000000;\n"
        " @!p bra W_%=;\n}\n" ::"r"(su32(&bar))
        : "memory");
    t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(d), "r"(512));
}

template <int KIND, int N = 256, bool TS = false>
double run(int sms, int iters) {
  const size_t smem = 48 * 1024 + 1024;
  cudaFuncSetAttribute(k_probe<KIND, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  k_probe<KIND, N, TS><<<sms, 128, smem>>>(16, cyc);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_probe<KIND, N, TS><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double k_per = KIND == 0 ? 8 : 16;
  const double flops = 2.0 * 128 * N * k_per * 4 * (double)iters * sms;
  cudaFree(cyc);
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  double tf = 0, bf = 0;
  for (int r = 0; r < 3; ++r) {  // best of 3
    const double a = run<0>(sms, iters), b = run<1>(sms, iters);
    tf = a > tf ? a : tf;
    bf = b > bf ? b : bf;
  }
  double n64ss = 0, n64ts = 0, n128ts = 0;
  for (int r = 0; r < 3; ++r) {
    n64ss = fmax(n64ss, run<0, 64, false>(sms, iters));
    n64ts = fmax(n64ts, run<0, 64, true>(sms, iters));
    n128ts = fmax(n128ts, run<0, 128, true>(sms, iters));
  }
  printf("{\"tf32_M128_N64_SS_tflops\": %.1f, \"tf32_M128_N64_TS_tflops\": %.1f, "
         "\"tf32_M128_N128_TS_tflops\": %.1f}\n", n64ss, n64ts, n128ts);
  printf("{\"sm_count\": %d, \"tcgen05_tf32_tflops\": %.1f, \"tcgen05_bf16_tflops\": %.1f, "
         "\"shape\": \"cta_group::1 M128 N256, SS operands, 1 CTA/SM, best of 3\", \"status\": \"%s\"}\n",
         sms, tf, bf, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
