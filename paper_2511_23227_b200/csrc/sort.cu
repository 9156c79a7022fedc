// sort.cu -- device primitives: exclusive scan and stable LSD radix sort.
//
// Used by the neighbor build (row offsets), the triplet orderings the
// reference API exposes (sort_triplets, triplets.cpp:135-170, a stable
// counting sort) and the compute plans (transposed CSR, per-cell lists,
// spatial order).  Hand-written; no CUB.
#include <atomic>

#include "npcg_internal.cuh"

namespace npcg {

// ---------------------------------------------------------------------------
// accounting + events
// ---------------------------------------------------------------------------
static std::atomic<int64_t> g_cur{0}, g_peak{0};
void mem_account(int64_t d) {
  const int64_t now = g_cur.fetch_add(d) + d;
  int64_t p = g_peak.load();
  while (now > p && !g_peak.compare_exchange_weak(p, now)) {
  }
}
int64_t mem_current() { return g_cur.load(); }
int64_t mem_peak() { return g_peak.load(); }
void mem_reset_peak() { g_peak.store(g_cur.load()); }

cudaEvent_t take_event(npcg_context* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  NPCG_CUDA(cudaEventCreate(&e));
  return e;
}

int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

// ---------------------------------------------------------------------------
// exclusive scan: 1024 threads x 4 items per block, recursive over block sums
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of per-thread values; returns the block total.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T& total) {
  __shared__ T warp_tot[32];
  __shared__ T block_total;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T incl = warp_incl_scan(v);
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    T x = lane < nw ? warp_tot[lane] : T(0);
    T xi = warp_incl_scan(x);
    if (lane < nw) warp_tot[lane] = xi - x;
    if (lane == nw - 1) block_total = xi;
  }
  __syncthreads();
  total = block_total;
  T r = incl - v + warp_tot[w];
  __syncthreads();
  return r;
}

template <typename T>
__global__ void scan_block_sums(const T* __restrict__ in, int64_t n, T* __restrict__ sums) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  T s = 0;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const int64_t e = base + static_cast<int64_t>(threadIdx.x) * kScanItems + it;
    if (e < n) s += in[e];
  }
  T total;
  block_excl_scan(s, total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

template <typename T>
__global__ void scan_block_apply(const T* __restrict__ in, int64_t n, T* __restrict__ out,
                                 const T* __restrict__ offsets) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const int64_t e = base + static_cast<int64_t>(threadIdx.x) * kScanItems + it;
    v[it] = e < n ? in[e] : T(0);
    s += v[it];
  }
  T total;
  T run = block_excl_scan(s, total) + (offsets ? offsets[blockIdx.x] : T(0));
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const int64_t e = base + static_cast<int64_t>(threadIdx.x) * kScanItems + it;
    if (e < n) out[e] = run;
    run += v[it];
  }
}

template <typename T>
static void exclusive_scan(npcg_context* ctx, const T* in, T* out, int64_t n, T* total) {
  if (n <= 0) {
    if (total) *total = 0;
    return;
  }
  const int64_t nb = ceil_div(n, kScanTile);
  if (nb == 1) {
    launch(ctx, "scan_apply", scan_block_apply<T>, dim3(1), dim3(kScanThreads), 0, in, n, out,
           static_cast<const T*>(nullptr));
  } else {
    DevBuf<T> sums(ctx, nb), sums_scan(ctx, nb);
    launch(ctx, "scan_sums", scan_block_sums<T>, dim3(static_cast<unsigned>(nb)),
           dim3(kScanThreads), 0, in, n, sums.get());
    exclusive_scan<T>(ctx, sums.get(), sums_scan.get(), nb, nullptr);
    launch(ctx, "scan_apply", scan_block_apply<T>, dim3(static_cast<unsigned>(nb)),
           dim3(kScanThreads), 0, in, n, out, static_cast<const T*>(sums_scan.get()));
  }
  if (total) {
    T last_in, last_out;
    NPCG_CUDA(cudaMemcpyAsync(&last_in, in + n - 1, sizeof(T), cudaMemcpyDeviceToHost,
                              ctx->stream));
    NPCG_CUDA(cudaMemcpyAsync(&last_out, out + n - 1, sizeof(T), cudaMemcpyDeviceToHost,
                              ctx->stream));
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
    *total = last_in + last_out;
  }
}

void exclusive_scan_i64(npcg_context* ctx, const int64_t* in, int64_t* out, int64_t n,
                        int64_t* total) {
  exclusive_scan<int64_t>(ctx, in, out, n, total);
}
void exclusive_scan_u32(npcg_context* ctx, const uint32_t* in, uint32_t* out, int64_t n,
                        uint32_t* total) {
  exclusive_scan<uint32_t>(ctx, in, out, n, total);
}

__global__ void iota_kernel(uint32_t* out, int64_t n) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) out[e] = static_cast<uint32_t>(e);
}
void iota_u32(npcg_context* ctx, uint32_t* out, int64_t n) {
  launch(ctx, "iota", iota_kernel, dim3(static_cast<unsigned>(ceil_div(n, 256))), dim3(256), 0,
         out, n);
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort, 8-bit digits.
//   pass = histogram (per block) -> scan (digit-major) -> stable scatter.
// The scatter ranks keys inside a block in original order: 16 rounds of 256
// keys; inside a round, warps rank with __match_any_sync and combine their
// per-digit counts through shared memory in warp order.
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 256;
constexpr int kRsRounds = 16;
constexpr int kRsTile = kRsThreads * kRsRounds;

template <typename K>
__global__ void rs_histogram(const K* __restrict__ keys, int64_t n, int shift, uint32_t mask,
                             uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  for (int d = threadIdx.x; d < 256; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile;
  const int64_t end = min(n, base + kRsTile);
  for (int64_t e = base + threadIdx.x; e < end; e += blockDim.x)
    atomicAdd(&h[static_cast<uint32_t>(keys[e] >> shift) & mask], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d <= static_cast<int>(mask); d += blockDim.x)
    hist[static_cast<int64_t>(d) * gridDim.x + blockIdx.x] = h[d];
}

template <typename K>
__global__ void rs_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                           K* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n,
                           int shift, uint32_t mask, const uint32_t* __restrict__ offs) {
  __shared__ uint32_t run[256];
  __shared__ uint32_t wcnt[kRsThreads / 32][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    run[d] = d <= static_cast<int>(mask) ? offs[static_cast<int64_t>(d) * gridDim.x + blockIdx.x]
                                         : 0u;
    for (int ww = 0; ww < kRsThreads / 32; ++ww) wcnt[ww][d] = 0;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile;
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t e = base + static_cast<int64_t>(r) * kRsThreads + threadIdx.x;
    const bool valid = e < n;
    K key = valid ? kin[e] : K(0);
    const uint32_t d = valid ? (static_cast<uint32_t>(key >> shift) & mask) : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) wcnt[w][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pos = run[d] + rank;
      for (int ww = 0; ww < w; ++ww) pos += wcnt[ww][d];
      kout[pos] = key;
      vout[pos] = vin[e];
    }
    __syncthreads();
    for (int dd = threadIdx.x; dd < 256; dd += blockDim.x) {
      uint32_t s = 0;
      for (int ww = 0; ww < kRsThreads / 32; ++ww) {
        s += wcnt[ww][dd];
        wcnt[ww][dd] = 0;
      }
      run[dd] += s;
    }
    __syncthreads();
  }
}

template <typename K>
static void radix_sort(npcg_context* ctx, K* keys, uint32_t* vals, int64_t n, int key_bits) {
  if (n <= 1 || key_bits <= 0) return;
  if (n > 0xFFFFFFFFll) fail(NPCG_ERR_SHAPE, "radix_sort: more than 2^32 items");
  const int64_t nb = ceil_div(n, kRsTile);
  DevBuf<K> k2(ctx, n);
  DevBuf<uint32_t> v2(ctx, n);
  DevBuf<uint32_t> hist(ctx, 256 * nb), offs(ctx, 256 * nb);
  K* ka = keys;
  K* kb = k2.get();
  uint32_t* va = vals;
  uint32_t* vb = v2.get();
  int passes = 0;
  for (int shift = 0; shift < key_bits; shift += 8, ++passes) {
    const int bits = key_bits - shift < 8 ? key_bits - shift : 8;
    const uint32_t mask = (1u << bits) - 1u;
    const int64_t bins = static_cast<int64_t>(mask) + 1;
    launch(ctx, "radix_hist", rs_histogram<K>, dim3(static_cast<unsigned>(nb)), dim3(kRsThreads),
           0, ka, n, shift, mask, hist.get());
    exclusive_scan_u32(ctx, hist.get(), offs.get(), bins * nb, nullptr);
    launch(ctx, "radix_scatter", rs_scatter<K>, dim3(static_cast<unsigned>(nb)),
           dim3(kRsThreads), 0, ka, va, kb, vb, n, shift, mask,
           static_cast<const uint32_t*>(offs.get()));
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (passes & 1) {
    NPCG_CUDA(cudaMemcpyAsync(keys, ka, n * sizeof(K), cudaMemcpyDeviceToDevice, ctx->stream));
    NPCG_CUDA(cudaMemcpyAsync(vals, va, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                              ctx->stream));
  }
}

void radix_sort_u32(npcg_context* ctx, uint32_t* keys, uint32_t* vals, int64_t n, int key_bits) {
  radix_sort<uint32_t>(ctx, keys, vals, n, key_bits);
}
void radix_sort_u64(npcg_context* ctx, uint64_t* keys, uint32_t* vals, int64_t n, int key_bits) {
  radix_sort<uint64_t>(ctx, keys, vals, n, key_bits);
}

}  // namespace npcg
