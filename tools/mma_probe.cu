// Throughput probe: FFMA vs legacy warp-level mma.sync (TF32 m16n8k8, FP64
// m8n8k4) on the B200, all operands in registers.  Decides whether a 3xTF32
// first-op GEMM can beat the FFMA one.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float s) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f);
  float t = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_tf32(float* out, float s) {
  unsigned a[4], b[2];
  float c[8][4];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(s + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(s - i);
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[j][i] = 0.f;
  for (int it = 0; it < ITERS / 8; ++it)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  float t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) t += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_dmma(double* out, double s) {
  double a = s, b = s + 1, c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
  for (int it = 0; it < ITERS / 8; ++it)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  double t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_dfma(double* out, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001 + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, 0.5);
  double t = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <class F>
static float time_it(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  float* of;
  double* od;
  cudaMalloc(&of, (size_t)blocks * threads * 8);
  cudaMalloc(&od, (size_t)blocks * threads * 8);
  const double warps = (double)blocks * threads / 32;
  float ms = time_it([&] { k_ffma<<<blocks, threads>>>(of, 0.999f); });
  std::printf("FFMA   %.1f TFLOP/s\n", (double)blocks * threads * ITERS * 16 * 2 / ms / 1e9);
  ms = time_it([&] { k_tf32<<<blocks, threads>>>(of, 0.999f); });
  std::printf("TF32 mma.sync %.1f TFLOP/s\n", warps * ITERS * 16 * 8 * 8 * 2 / ms / 1e9);
  ms = time_it([&] { k_dfma<<<blocks, threads>>>(od, 0.999); });
  std::printf("DFMA   %.1f TFLOP/s\n", (double)blocks * threads * ITERS * 16 * 2 / ms / 1e9);
  ms = time_it([&] { k_dmma<<<blocks, threads>>>(od, 0.999); });
  std::printf("DMMA mma.sync %.1f TFLOP/s\n", warps * ITERS * 8 * 8 * 4 * 2 / ms / 1e9);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
