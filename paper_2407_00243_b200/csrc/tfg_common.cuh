// tfg_common.cuh -- shared plumbing for libtfg (errors, device buffers,
// CUB scratch, launch helpers).  sm_100a only.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

#include "tfg.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libtfg is written for sm_100a only (compile with -gencode arch=compute_100a,code=sm_100a)"
#endif

namespace tfg {

// Error classes mirror the reference's exception types.
struct invalid_argument : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct runtime_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what,
                                    const char* file, int line) {
  throw cuda_error(std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                   cudaGetErrorString(e) + ") at " + file + ":" +
                   std::to_string(line) + ": " + what);
}

#define TFG_CUDA(expr)                                            \
  do {                                                            \
    cudaError_t e__ = (expr);                                     \
    if (e__ != cudaSuccess) ::tfg::throw_cuda(e__, #expr, __FILE__, __LINE__); \
  } while (0)
#define TFG_LAUNCH_CHECK() TFG_CUDA(cudaGetLastError())

template <class F>
tfg_status guard(F&& f) {
  try {
    f();
    return TFG_OK;
  } catch (const invalid_argument& e) {
    set_last_error(e.what());
    return TFG_EINVAL;
  } catch (const cuda_error& e) {
    set_last_error(e.what());
    return TFG_ECUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TFG_ERUNTIME;
  }
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Stream-ordered allocation scope.  cudaFree synchronises the whole device,
// so temporaries freed while building a plan would wait for unrelated work
// (the by-value call uploads B on another stream meanwhile).  Inside a scope,
// dbuf allocates and frees with cudaMallocAsync / cudaFreeAsync on the
// scope's stream from the device's default pool (kept cached: release
// threshold raised once), so buffers are ordered with the work that uses them.
struct AllocScope {
  static cudaStream_t& stream() {
    static thread_local cudaStream_t s = nullptr;
    return s;
  }
  static bool& active() {
    static thread_local bool on = false;
    return on;
  }
  cudaStream_t prev_s;
  bool prev_on;
  explicit AllocScope(cudaStream_t st) : prev_s(stream()), prev_on(active()) {
    static thread_local bool pool_set = false;
    if (!pool_set) {
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      pool_set = true;
    }
    stream() = st;
    active() = true;
  }
  ~AllocScope() {
    stream() = prev_s;
    active() = prev_on;
  }
  AllocScope(const AllocScope&) = delete;
  AllocScope& operator=(const AllocScope&) = delete;
};

// Owning device allocation (cudaMalloc, or stream-ordered inside an
// AllocScope; plans and schedules are built once and executed many times, so
// allocation is never on the execute path).
template <class T>
struct dbuf {
  T* p = nullptr;
  size_t n = 0;
  dbuf() = default;
  explicit dbuf(size_t count) { alloc(count); }
  dbuf(const dbuf&) = delete;
  dbuf& operator=(const dbuf&) = delete;
  dbuf(dbuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  dbuf& operator=(dbuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~dbuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (!count) return;
    if (AllocScope::active())
      TFG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), AllocScope::stream()));
    else
      TFG_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p) {
      if (AllocScope::active())
        cudaFreeAsync(p, AllocScope::stream());
      else
        cudaFree(p);
    }
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
  T* get() const { return p; }
};

inline int ceil_log2_bits(uint64_t x) {  // bits needed to represent x
  int b = 0;
  while (x) { ++b; x >>= 1; }
  return b < 1 ? 1 : b;
}

inline int sm_count() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0;
    TFG_CUDA(cudaGetDevice(&dev));
    TFG_CUDA(cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev));
  }
  return cached;
}

// Small host->device uploads without the copy engine.  Inside the drop-in
// by-value call (tfg_run_host) the H2D copy engine is busy with gigabytes of
// operands for ~0.2 s; a plan's own work-list uploads queued behind them
// would stall plan creation for that long (measured: 130 ms).  With an
// UploadScope active, h2d() stages the bytes in a pinned arena and a copy
// kernel reads them over the bus (zero-copy), sharing only bandwidth.
struct UploadArena {
  unsigned char* base = nullptr;
  size_t cap = 0, off = 0;
  std::mutex mu;
  static UploadArena& get() {
    static UploadArena a;
    return a;
  }
};
struct UploadScope {
  static UploadArena*& active() {
    static thread_local UploadArena* a = nullptr;
    return a;
  }
  cudaStream_t st;
  bool owns = false;
  explicit UploadScope(cudaStream_t s, size_t bytes = (size_t)256 << 20) : st(s) {
    UploadArena& a = UploadArena::get();
    if (active() || !a.mu.try_lock()) return;  // nested or in use elsewhere: plain copies
    if (!a.base && cudaHostAlloc(reinterpret_cast<void**>(&a.base), bytes, cudaHostAllocDefault) ==
                       cudaSuccess)
      a.cap = bytes;
    if (!a.base) {
      cudaGetLastError();
      a.mu.unlock();
      return;
    }
    a.off = 0;
    owns = true;
    active() = &a;
  }
  ~UploadScope() {
    if (!owns) return;
    cudaStreamSynchronize(st);  // the copy kernels have read the arena
    active() = nullptr;
    UploadArena::get().mu.unlock();
  }
  UploadScope(const UploadScope&) = delete;
  UploadScope& operator=(const UploadScope&) = delete;
};
#ifdef __CUDACC__
static __global__ void k_upload_copy(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                     size_t n16, size_t bytes) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
    dst[i] = src[i];
  if (blockIdx.x == 0 && threadIdx.x < (bytes & 15)) {
    const size_t o = (n16 << 4) + threadIdx.x;
    reinterpret_cast<unsigned char*>(dst)[o] = reinterpret_cast<const unsigned char*>(src)[o];
  }
}
#endif

template <class T>
inline void h2d(T* d, const T* h, size_t count, cudaStream_t s) {
  if (!count) return;
#ifdef __CUDACC__
  if (UploadArena* a = UploadScope::active()) {
    const size_t bytes = count * sizeof(T), need = (bytes + 255) & ~(size_t)255;
    if (a->off + need <= a->cap && (reinterpret_cast<uintptr_t>(d) & 15) == 0) {
      unsigned char* stage = a->base + a->off;
      a->off += need;
      std::memcpy(stage, h, bytes);
      const size_t n16 = bytes >> 4;
      const unsigned blocks = (unsigned)std::min<size_t>(std::max<size_t>((n16 + 255) / 256, 1), 64);
      k_upload_copy<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(stage),
                                           reinterpret_cast<uint4*>(d), n16, bytes);
      TFG_LAUNCH_CHECK();
      return;
    }
  }
#endif
  TFG_CUDA(cudaMemcpyAsync(d, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <class T>
inline void d2h(T* h, const T* d, size_t count, cudaStream_t s) {
  if (count) TFG_CUDA(cudaMemcpyAsync(h, d, count * sizeof(T), cudaMemcpyDeviceToHost, s));
}

}  // namespace tfg

// The device-resident schedule behind the opaque tfg_schedule handle.
struct tfg_schedule {
  int32_t n = 0;
  int32_t tile_size = 0;
  int64_t n_tiles[2] = {0, 0};
  int64_t n_jrows[2] = {0, 0};
  double inspect_seconds = 0.0;
  tfg::dbuf<int32_t> i_lo[2], i_hi[2];
  tfg::dbuf<double> cost[2];
  tfg::dbuf<int64_t> j_off[2];
  tfg::dbuf<int32_t> j_rows[2];
};
