// npcg_internal.cuh -- shared host/device infrastructure of libnpcg.so.
//
// Context (device, stream, launch counter, event profiler), error plumbing
// (exceptions inside, status codes at the C ABI), device allocation with
// accounting, and the kernel-launch helper every launch goes through.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "npcg.h"

namespace npcg {

// Internal error: thrown by host code, converted to a status at the ABI.
struct Error {
  npcg_status code;
  std::string msg;
};

[[noreturn]] inline void fail(npcg_status s, const std::string& m) { throw Error{s, m}; }

#define NPCG_CUDA(x)                                                                      \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      ::npcg::fail(e_ == cudaErrorMemoryAllocation ? NPCG_ERR_OOM : NPCG_ERR_CUDA,        \
                   std::string(#x) + ": " + cudaGetErrorString(e_));                      \
    }                                                                                     \
  } while (0)

// Process-wide device-allocation accounting (bytes owned by the library).
void mem_account(int64_t delta);
int64_t mem_current();
int64_t mem_peak();
void mem_reset_peak();

}  // namespace npcg

struct npcg_prof_rec {
  const char* name;
  cudaEvent_t start, stop;
};

struct npcg_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int max_smem_optin = 0;
  std::string last_error;
  int64_t launches = 0;
  bool profiling = false;
  std::vector<npcg_prof_rec> prof;
  std::vector<cudaEvent_t> event_pool;
};

namespace npcg {

cudaEvent_t take_event(npcg_context* ctx);

// Runs an entry point's body: C++ exceptions become status codes (they never
// cross the ABI); the message is kept for npcg_last_error.
template <typename F>
npcg_status guard(npcg_context* ctx, F&& f) {
  try {
    if (ctx) {
      NPCG_CUDA(cudaSetDevice(ctx->device));
      ctx->last_error.clear();
    }
    f();
    return NPCG_OK;
  } catch (const Error& e) {
    if (ctx) ctx->last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->last_error = "host allocation failed";
    return NPCG_ERR_OOM;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    return NPCG_ERR_CUDA;
  }
}

// Every kernel launch of the library goes through here: counted, optionally
// bracketed by events for the in-library profiler, error-checked.
template <typename... KArgs, typename... Args>
inline void launch(npcg_context* ctx, const char* name, void (*kernel)(KArgs...), dim3 grid,
                   dim3 block, size_t smem, Args&&... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  cudaEvent_t a = nullptr, b = nullptr;
  if (ctx->profiling) {
    a = take_event(ctx);
    NPCG_CUDA(cudaEventRecord(a, ctx->stream));
  }
  kernel<<<grid, block, smem, ctx->stream>>>(std::forward<Args>(args)...);
  NPCG_CUDA(cudaGetLastError());
  ctx->launches++;
  if (ctx->profiling) {
    b = take_event(ctx);
    NPCG_CUDA(cudaEventRecord(b, ctx->stream));
    ctx->prof.push_back({name, a, b});
  }
}

// Cluster launch (thread-block clusters, cudaLaunchKernelEx).
template <typename... KArgs, typename... Args>
inline void launch_cluster(npcg_context* ctx, const char* name, void (*kernel)(KArgs...),
                           dim3 grid, dim3 block, size_t smem, unsigned cluster_x,
                           Args&&... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  cudaEvent_t a = nullptr, b = nullptr;
  if (ctx->profiling) {
    a = take_event(ctx);
    NPCG_CUDA(cudaEventRecord(a, ctx->stream));
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  NPCG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  ctx->launches++;
  if (ctx->profiling) {
    b = take_event(ctx);
    NPCG_CUDA(cudaEventRecord(b, ctx->stream));
    ctx->prof.push_back({name, a, b});
  }
}

// RAII device buffer (stream-ordered allocation on the context stream).
template <typename T>
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(npcg_context* ctx, int64_t n) { alloc(ctx, n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { swap(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      swap(o);
    }
    return *this;
  }
  void alloc(npcg_context* ctx, int64_t n) {
    if (p_ && stream_ != ctx->stream) {
      // the old buffer may still be read by work on the stream it was last
      // used on: free it on the current stream, ordered after that stream
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(e, stream_);
        cudaStreamWaitEvent(ctx->stream, e, 0);
        cudaEventDestroy(e);
      }
      stream_ = ctx->stream;
    }
    release();
    n_ = n;
    stream_ = ctx->stream;
    if (n <= 0) return;
    const size_t bytes = static_cast<size_t>(n) * sizeof(T);
    NPCG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), bytes, stream_));
    bytes_ = static_cast<int64_t>(bytes);
    mem_account(bytes_);
  }
  void release() {
    if (p_) {
      cudaFreeAsync(p_, stream_);
      mem_account(-bytes_);
    }
    p_ = nullptr;
    n_ = 0;
    bytes_ = 0;
  }
  T* get() const { return p_; }
  int64_t size() const { return n_; }
  void swap(DevBuf& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(bytes_, o.bytes_);
    std::swap(stream_, o.stream_);
  }

 private:
  T* p_ = nullptr;
  int64_t n_ = 0;
  int64_t bytes_ = 0;
  cudaStream_t stream_ = nullptr;
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- primitives (sort.cu) --------------------------------------------------
// Exclusive prefix sum; returns the total (synchronises) when `total` != null.
void exclusive_scan_i64(npcg_context* ctx, const int64_t* in, int64_t* out, int64_t n,
                        int64_t* total);
void exclusive_scan_u32(npcg_context* ctx, const uint32_t* in, uint32_t* out, int64_t n,
                        uint32_t* total);
// Stable LSD radix sort of (key, value) pairs over key bits [0, key_bits).
// keys/vals are sorted in place (double buffers allocated internally).
void radix_sort_u32(npcg_context* ctx, uint32_t* keys, uint32_t* vals, int64_t n, int key_bits);
void radix_sort_u64(npcg_context* ctx, uint64_t* keys, uint32_t* vals, int64_t n, int key_bits);
// out[p] = p
void iota_u32(npcg_context* ctx, uint32_t* out, int64_t n);
int bits_for(uint64_t max_value);  // bits needed to represent max_value

}  // namespace npcg
