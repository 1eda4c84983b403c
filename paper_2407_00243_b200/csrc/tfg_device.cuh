// tfg_device.cuh -- device helpers shared by the executor kernels: exact
// fp mul/add/fma wrappers, vector loads/stores, and the CSR-row SpMM routine
// whose per-element order (ascending nonzeros, separately rounded mul and
// add) makes SpMM results bit-identical to the reference (kernels.hpp:75-79).
#pragma once
#include <cuda_runtime.h>

#include <cstring>

namespace tfg {
namespace dev {

template <class T>
struct fops;
template <>
struct fops<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
};
template <>
struct fops<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
};

template <class T, int VEC>
struct VT;
template <> struct VT<double, 1> { using type = double; };
template <> struct VT<double, 2> { using type = double2; };
template <> struct VT<float, 1> { using type = float; };
template <> struct VT<float, 2> { using type = float2; };
template <> struct VT<float, 4> { using type = float4; };

template <class T, int VEC>
__device__ __forceinline__ void ldv(T (&r)[VEC], const T* p) {
  using V = typename VT<T, VEC>::type;
  const V x = *reinterpret_cast<const V*>(p);
  memcpy(r, &x, sizeof(V));
}
template <class T, int VEC>
__device__ __forceinline__ void stv(T* p, const T (&r)[VEC]) {
  using V = typename VT<T, VEC>::type;
  V x;
  memcpy(&x, r, sizeof(V));
  *reinterpret_cast<V*>(p) = x;
}
// streaming store for D (written once, never re-read by this launch)
template <class T, int VEC>
__device__ __forceinline__ void stv_cs(T* p, const T (&r)[VEC]) {
  using V = typename VT<T, VEC>::type;
  V x;
  memcpy(&x, r, sizeof(V));
  __stcs(reinterpret_cast<V*>(p), x);
}

__device__ __forceinline__ unsigned group_mask(int lpr) {
  if (lpr == 32) return 0xffffffffu;
  const int lane = threadIdx.x & 31;
  return ((1u << lpr) - 1u) << (lane & ~(lpr - 1));
}

// One CSR row times X, LPR lanes per row, each lane NCH x VEC columns.
// Per-element order = ascending nonzeros, separate mul and add
// (kernels.hpp:75-79).  XL(c, ch, out[VEC]) loads X row c, chunk ch.
// acc += a * x per term: separately rounded mul and add (the reference's
// order and rounding), or one fused multiply-add when FMA (GeMM-SpMM plans
// whose first op is already tolerance-bound; never for SpMM-SpMM parity)
template <class T, bool FMA>
__device__ __forceinline__ T madd(T acc, T a, T x) {
  if constexpr (FMA)
    return fops<T>::fma(a, x, acc);
  else
    return fops<T>::add(acc, fops<T>::mul(a, x));
}

template <class T, int VEC, int LPR, int NCH, class XL, int UNR = 4, bool FMA = false>
__device__ __forceinline__ void spmm_accum(int kb, int ke,
                                           const int* __restrict__ ci,
                                           const T* __restrict__ av, int gl,
                                           unsigned gmask, XL xl,
                                           T (&acc)[NCH][VEC]) {
  for (int k0 = kb; k0 < ke; k0 += LPR) {
    const int kk = k0 + gl;
    int c = 0;
    T a = T(0);
    if (kk < ke) {
      c = __ldg(ci + kk);
      a = __ldg(av + kk);
    }
    const int cnt = min(LPR, ke - k0);
    int u = 0;
    for (; u + UNR <= cnt; u += UNR) {
      int cu[UNR];
      T au[UNR];
      T x[UNR][NCH][VEC];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        cu[q] = __shfl_sync(gmask, c, u + q, LPR);
        au[q] = __shfl_sync(gmask, a, u + q, LPR);
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) xl(cu[q], ch, x[q][ch]);
#pragma unroll
      for (int q = 0; q < UNR; ++q)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
          for (int e = 0; e < VEC; ++e)
            acc[ch][e] = madd<T, FMA>(acc[ch][e], au[q], x[q][ch][e]);
    }
    for (; u < cnt; ++u) {
      const int cu = __shfl_sync(gmask, c, u, LPR);
      const T au = __shfl_sync(gmask, a, u, LPR);
      T x[NCH][VEC];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) xl(cu, ch, x[ch]);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          acc[ch][e] = madd<T, FMA>(acc[ch][e], au, x[ch][e]);
    }
  }
}

// acc = row kb..ke times X, from 0 (spmm_row, kernels.hpp:71-80)
template <class T, int VEC, int LPR, int NCH, class XL, int UNR = 4, bool FMA = false>
__device__ __forceinline__ void spmm_row(int kb, int ke,
                                         const int* __restrict__ ci,
                                         const T* __restrict__ av, int gl,
                                         unsigned gmask, XL xl,
                                         T (&acc)[NCH][VEC]) {
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[ch][e] = T(0);
  spmm_accum<T, VEC, LPR, NCH, XL, UNR, FMA>(kb, ke, ci, av, gl, gmask, xl, acc);
}

}  // namespace dev
}  // namespace tfg
