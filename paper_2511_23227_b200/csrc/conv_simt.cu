// conv_simt.cu -- exact-arithmetic MVMR / VVOR engines on CUDA cores.
//
// These run in the API dtype (fp32 or fp64, FMA accumulation) for every
// shape the reference accepts (any G, C_in, C_out, t).  They are the
// NPCG_MATH_EXACT path and the narrow-channel path of the north star.
//
//   mvmr            engine.cpp:444-455 -> output-stationary: one warp per
//                   (output row, group), lanes own output channels, the
//                   row's neighbor entries are walked in CSR order and
//                   reduced in registers; one plain store per output value
//                   (no atomics, deterministic).
//   mvmr_transposed engine.cpp:457-473 -> the same kernel over the
//                   transposed CSR (rows = input points) with W^T.
//   vvor            vvor.cpp:102-271 -> per kernel cell, chunks of the cell's
//                   entries accumulate dW_k tiles in registers (rows staged
//                   in shared memory); chunk partials are summed in a fixed
//                   order by a second kernel (deterministic, no atomics).
#include <type_traits>

#include "neighbors.cuh"
#include "conv.cuh"

namespace npcg {

// ---------------------------------------------------------------------------
// mvmr rows
// ---------------------------------------------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(256) k_mvmr_rows(CsrView csr, const T* __restrict__ w,
                                                   const T* __restrict__ fin, int G, int cin,
                                                   int cout, int m_base,
                                                   T* __restrict__ out) {
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= csr.n_rows * G) return;
  const int64_t row = warp / G;
  const int g = static_cast<int>(warp - row * G);
  T acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = T(0);
  const int64_t e0 = csr.row_ptr[row], e1 = csr.row_ptr[row + 1];
  for (int64_t e = e0; e < e1; ++e) {
    const int64_t j = csr.col[e];
    const int64_t k = csr.k[e];
    const T* f = fin + (j * G + g) * cin;
    const T* wm = w + ((k * G + g) * cin) * cout + m_base;
    for (int c0 = 0; c0 < cin; c0 += 32) {
      const T fv = (c0 + lane < cin) ? f[c0 + lane] : T(0);
      const int cn = cin - c0 < 32 ? cin - c0 : 32;
      if (cn == 32) {  // full chunk: unrolled, so the W loads of several channels are in flight
#pragma unroll 8
        for (int cc = 0; cc < 32; ++cc) {
          const T fc = __shfl_sync(0xffffffffu, fv, cc);
          const T* wr = wm + static_cast<int64_t>(c0 + cc) * cout;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int m = lane + 32 * r;
            if (m_base + m < cout) acc[r] = fma(__ldg(wr + m), fc, acc[r]);
          }
        }
      } else {
        for (int cc = 0; cc < cn; ++cc) {
          const T fc = __shfl_sync(0xffffffffu, fv, cc);
          const T* wr = wm + static_cast<int64_t>(c0 + cc) * cout;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int m = lane + 32 * r;
            if (m_base + m < cout) acc[r] = fma(wr[m], fc, acc[r]);
          }
        }
      }
    }
  }
  T* o = out + (row * G + g) * cout + m_base;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int m = lane + 32 * r;
    if (m_base + m < cout) o[m] = acc[r];
  }
}

// Same arithmetic (same FMA order: entries in CSR order, input channels
// ascending) with W staged once per CTA in shared memory, for the narrow
// layers whose whole W fits (config 1: 27 x 32 x 32 fp32 = 110 KB): one
// persistent CTA per SM, warps grid-striding over rows, the next entry's
// (j, k) and feature slice loaded while the current one is reduced.
template <typename T, int R>
__global__ void __launch_bounds__(1024, 1) k_mvmr_rows_ws(CsrView csr, const T* __restrict__ w,
                                                          int64_t w_elems, const T* __restrict__ fin,
                                                          int G, int cin, int cout,
                                                          T* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t ws_raw[];
  T* ws = reinterpret_cast<T*>(ws_raw);
  for (int64_t x = threadIdx.x; x < w_elems; x += blockDim.x) ws[x] = w[x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t total = csr.n_rows * G;
  for (int64_t warp = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       warp < total; warp += nw) {
    const int64_t row = warp / G;
    const int g = static_cast<int>(warp - row * G);
    T acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = T(0);
    const int64_t e0 = csr.row_ptr[row], e1 = csr.row_ptr[row + 1];
    // the next entry's cell and first feature slice are in flight while the
    // current entry is reduced
    int64_t kn = 0;
    T fn = T(0);
    if (e0 < e1) {
      kn = csr.k[e0];
      if (lane < cin) fn = fin[(static_cast<int64_t>(csr.col[e0]) * G + g) * cin + lane];
    }
    for (int64_t e = e0; e < e1; ++e) {
      const int64_t k = kn;
      const T f0 = fn;
      const int64_t j = csr.col[e];
      if (e + 1 < e1) {
        kn = csr.k[e + 1];
        if (lane < cin) fn = fin[(static_cast<int64_t>(csr.col[e + 1]) * G + g) * cin + lane];
      }
      const T* f = fin + (j * G + g) * cin;
      const T* wm = ws + ((k * G + g) * cin) * cout;
      for (int c0 = 0; c0 < cin; c0 += 32) {
        const T fv = c0 == 0 ? f0 : (c0 + lane < cin) ? f[c0 + lane] : T(0);
        const int cn = cin - c0 < 32 ? cin - c0 : 32;
#pragma unroll 8
        for (int cc = 0; cc < cn; ++cc) {
          const T fc = __shfl_sync(0xffffffffu, fv, cc);
          const T* wr = wm + (c0 + cc) * cout;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int m = lane + 32 * r;
            if (m < cout) acc[r] = fma(wr[m], fc, acc[r]);
          }
        }
      }
    }
    T* o = out + (row * G + g) * cout;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int m = lane + 32 * r;
      if (m < cout) o[m] = acc[r];
    }
  }
}

// fp32, C_in % 4 == 0: W staged transposed ([k][m][c], rows padded to an odd
// number of 16-byte groups so a warp's 16-byte reads are conflict-free), the
// input row read four channels at a time with a broadcast load -- per four
// FMAs one LDG.128 (all lanes one address) and one LDS.128 instead of four
// shuffles and four loads.  Same products, same order: channel-ascending FMAs
// per entry, entries in CSR order.
template <int R>
__global__ void __launch_bounds__(1024, 1) k_mvmr_rows_ws4(CsrView csr, const float* __restrict__ w,
                                                           int64_t kg_n, const float* __restrict__ fin,
                                                           int G, int cin, int cout, int wstride,
                                                           float* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t ws_raw[];
  float* ws = reinterpret_cast<float*>(ws_raw);
  // (the image is < 200 KB: 32-bit index arithmetic)
  const int per = cin * cout, w_total = static_cast<int>(kg_n) * per;
#pragma unroll 4
  for (int x = threadIdx.x; x < w_total; x += blockDim.x) {
    const int kg = x / per, r = x - kg * per, c = r / cout, m = r - c * cout;
    ws[(kg * cout + m) * wstride + c] = w[x];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t total = csr.n_rows * G;
  int mrow[R];
#pragma unroll
  for (int r = 0; r < R; ++r) mrow[r] = min(lane + 32 * r, cout - 1) * wstride;  // lanes past C_out: discarded
  for (int64_t warp = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       warp < total; warp += nw) {
    const int64_t row = warp / G;
    const int g = static_cast<int>(warp - row * G);
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    const int64_t e0 = csr.row_ptr[row], e1 = csr.row_ptr[row + 1];
    // the row's entries, 32 at a time: one coalesced load of (j, k) per lane,
    // broadcast by shuffles (no dependent global load per entry)
    for (int64_t eb = e0; eb < e1; eb += 32) {
    const int cnt = static_cast<int>(e1 - eb < 32 ? e1 - eb : 32);
    uint32_t jl = 0, kl = 0;
    if (lane < cnt) {
      jl = csr.col[eb + lane];
      kl = csr.k[eb + lane];
    }
    for (int x = 0; x < cnt; ++x) {
      const int64_t j = __shfl_sync(0xffffffffu, jl, x), k = __shfl_sync(0xffffffffu, kl, x);
      const float4* f4 = reinterpret_cast<const float4*>(fin + (j * G + g) * cin);
      const float* wk = ws + (k * G + g) * cout * wstride;
#pragma unroll 8
      for (int c = 0; c < cin; c += 4) {
        const float4 fv = __ldg(f4 + (c >> 2));
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float4 wv = *reinterpret_cast<const float4*>(wk + mrow[r] + c);
          acc[r] = fmaf(wv.x, fv.x, acc[r]);
          acc[r] = fmaf(wv.y, fv.y, acc[r]);
          acc[r] = fmaf(wv.z, fv.z, acc[r]);
          acc[r] = fmaf(wv.w, fv.w, acc[r]);
        }
      }
    }
    }
    float* o = out + (row * G + g) * cout;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int m = lane + 32 * r;
      if (m < cout) o[m] = acc[r];
    }
  }
}

constexpr int64_t WS_MAX_BYTES = 200 * 1024;

// fp32 rows of the transposed W image: C_in floats padded to an odd number of
// 16-byte groups
static int ws4_stride(int cin) { return (cin / 4) % 2 ? cin : cin + 4; }

template <int R>
static void launch_mvmr_ws4(npcg_context* ctx, const CsrView& csr, const float* w, int64_t kg_n,
                            const float* fin, int G, int cin, int cout, float* out) {
  const int stride = ws4_stride(cin);
  const int bytes = static_cast<int>(kg_n * cout * stride * sizeof(float));
  auto kern = k_mvmr_rows_ws4<R>;
  NPCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  launch(ctx, "mvmr_simt", kern, dim3(static_cast<unsigned>(ctx->num_sms)), dim3(1024), bytes, csr, w,
         kg_n, fin, G, cin, cout, stride, out);
}

template <typename T, int R>
static void launch_mvmr_ws(npcg_context* ctx, const CsrView& csr, const T* w, int64_t w_elems,
                           const T* fin, int G, int cin, int cout, T* out) {
  const int bytes = static_cast<int>(w_elems * sizeof(T));
  auto kern = k_mvmr_rows_ws<T, R>;
  NPCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  launch(ctx, "mvmr_simt", kern, dim3(static_cast<unsigned>(ctx->num_sms)), dim3(1024), bytes, csr, w,
         w_elems, fin, G, cin, cout, out);
}

// Rows given as a list of positions into `perm` (row = perm[list[x]]): the
// exact engine for the rows of tensor-core super-tiles beyond tile capacity.
template <typename T, int R>
__global__ void __launch_bounds__(256) k_mvmr_rows_subset(CsrView csr, const uint32_t* __restrict__ perm,
                                                          const uint32_t* __restrict__ list,
                                                          int64_t n_list, const T* __restrict__ w,
                                                          const T* __restrict__ fin, int cin,
                                                          int cout, T* __restrict__ out) {
  const int64_t x = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (x >= n_list) return;
  const int64_t row = perm[list[x]];
  T acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = T(0);
  for (int64_t e = csr.row_ptr[row]; e < csr.row_ptr[row + 1]; ++e) {
    const T* f = fin + static_cast<int64_t>(csr.col[e]) * cin;
    const T* wm = w + static_cast<int64_t>(csr.k[e]) * cin * cout;
    for (int c0 = 0; c0 < cin; c0 += 32) {
      const T fv = (c0 + lane < cin) ? f[c0 + lane] : T(0);
      const int cn = cin - c0 < 32 ? cin - c0 : 32;
      for (int cc = 0; cc < cn; ++cc) {
        const T fc = __shfl_sync(0xffffffffu, fv, cc);
        const T* wr = wm + static_cast<int64_t>(c0 + cc) * cout;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int m = lane + 32 * r;
          if (m < cout) acc[r] = fma(wr[m], fc, acc[r]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int m = lane + 32 * r;
    if (m < cout) out[row * cout + m] = acc[r];
  }
}

void mvmr_rows_subset_f32(npcg_context* ctx, const CsrView& csr, const uint32_t* perm,
                          const uint32_t* list, int64_t n_list, const float* w, const float* fin,
                          int cin, int cout, float* out) {
  if (n_list == 0) return;
  const unsigned blocks = static_cast<unsigned>(ceil_div(n_list * 32, 256));
  if (cout > 256) fail(NPCG_ERR_UNSUPPORTED, "row-subset engine: C_out <= 256");
  if (cout <= 64)
    launch(ctx, "mvmr_simt_subset", k_mvmr_rows_subset<float, 2>, dim3(blocks), dim3(256), 0, csr,
           perm, list, n_list, w, fin, cin, cout, out);
  else if (cout <= 128)
    launch(ctx, "mvmr_simt_subset", k_mvmr_rows_subset<float, 4>, dim3(blocks), dim3(256), 0, csr,
           perm, list, n_list, w, fin, cin, cout, out);
  else
    launch(ctx, "mvmr_simt_subset", k_mvmr_rows_subset<float, 8>, dim3(blocks), dim3(256), 0, csr,
           perm, list, n_list, w, fin, cin, cout, out);
}

template <typename T>
void mvmr_rows(npcg_context* ctx, const CsrView& csr, const T* w, const T* fin, int G, int cin,
               int cout, T* out, int64_t n_kernels) {
  if (csr.n_rows == 0) return;
  const int64_t w_elems = n_kernels * G * cin * cout;
  if (std::is_same<T, float>::value && n_kernels > 0 && cout <= 64 && cin % 4 == 0 &&
      n_kernels * G * cout * ws4_stride(cin) * 4 <= WS_MAX_BYTES &&
      reinterpret_cast<uintptr_t>(fin) % 16 == 0 && csr.n_rows * G >= 8 * static_cast<int64_t>(ctx->num_sms)) {
    const float* wf = reinterpret_cast<const float*>(w);
    const float* ff = reinterpret_cast<const float*>(fin);
    float* of = reinterpret_cast<float*>(out);
    if (cout <= 32)
      launch_mvmr_ws4<1>(ctx, csr, wf, n_kernels * G, ff, G, cin, cout, of);
    else
      launch_mvmr_ws4<2>(ctx, csr, wf, n_kernels * G, ff, G, cin, cout, of);
    return;
  }
  if (n_kernels > 0 && cout <= 64 && w_elems * static_cast<int64_t>(sizeof(T)) <= WS_MAX_BYTES &&
      csr.n_rows * G >= 8 * static_cast<int64_t>(ctx->num_sms)) {
    if (cout <= 32)
      launch_mvmr_ws<T, 1>(ctx, csr, w, w_elems, fin, G, cin, cout, out);
    else
      launch_mvmr_ws<T, 2>(ctx, csr, w, w_elems, fin, G, cin, cout, out);
    return;
  }
  const unsigned blocks = static_cast<unsigned>(ceil_div(csr.n_rows * G * 32, 256));
  for (int m_base = 0; m_base < cout; m_base += 256) {
    const int rem = cout - m_base;
    if (rem <= 32)
      launch(ctx, "mvmr_simt", k_mvmr_rows<T, 1>, dim3(blocks), dim3(256), 0, csr, w, fin, G, cin,
             cout, m_base, out);
    else if (rem <= 64)
      launch(ctx, "mvmr_simt", k_mvmr_rows<T, 2>, dim3(blocks), dim3(256), 0, csr, w, fin, G, cin,
             cout, m_base, out);
    else if (rem <= 128)
      launch(ctx, "mvmr_simt", k_mvmr_rows<T, 4>, dim3(blocks), dim3(256), 0, csr, w, fin, G, cin,
             cout, m_base, out);
    else
      launch(ctx, "mvmr_simt", k_mvmr_rows<T, 8>, dim3(blocks), dim3(256), 0, csr, w, fin, G, cin,
             cout, m_base, out);
  }
}

// W (K, G, Cin, Cout) -> W^T (K, G, Cout, Cin)  (tensors.hpp:113-123 transposed())
template <typename T>
__global__ void k_transpose_w(const T* __restrict__ w, int64_t KG, int cin, int cout,
                              T* __restrict__ wt) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per = static_cast<int64_t>(cin) * cout;
  if (p >= KG * per) return;
  const int64_t kg = p / per, r = p - kg * per;
  const int c = static_cast<int>(r / cout), m = static_cast<int>(r - static_cast<int64_t>(c) * cout);
  wt[kg * per + static_cast<int64_t>(m) * cin + c] = w[p];
}

template <typename T>
void transpose_w(npcg_context* ctx, const T* w, int64_t KG, int cin, int cout, T* wt) {
  const int64_t n = KG * cin * cout;
  launch(ctx, "transpose_w", k_transpose_w<T>, dim3(static_cast<unsigned>(ceil_div(n, 256))),
         dim3(256), 0, w, KG, cin, cout, wt);
}

// ---------------------------------------------------------------------------
// vvor: per-cell chunk partials + fixed-order reduction
// ---------------------------------------------------------------------------
constexpr int kVvorThreads = 256;
constexpr int kVvorOutsPerThread = 16;
constexpr int kVvorOutsPerBlock = kVvorThreads * kVvorOutsPerThread;

template <typename T>
__global__ void __launch_bounds__(kVvorThreads)
    k_vvor_chunks(const uint32_t* __restrict__ ci, const uint32_t* __restrict__ cj,
                  const int64_t* __restrict__ chunk_begin, const int64_t* __restrict__ chunk_end,
                  const T* __restrict__ gout, const T* __restrict__ fin, int G, int cin,
                  int cout, int rows_per_batch, T* __restrict__ partial) {
  extern __shared__ unsigned char smem_raw[];
  T* gs = reinterpret_cast<T*>(smem_raw);          // [rows][cout]
  T* fs = gs + static_cast<int64_t>(rows_per_batch) * cout;  // [rows][cin]
  const int64_t chunk = blockIdx.x;
  const int g = blockIdx.y;
  const int64_t o_base = static_cast<int64_t>(blockIdx.z) * kVvorOutsPerBlock;
  const int64_t per = static_cast<int64_t>(cout) * cin;
  const int64_t b0 = chunk_begin[chunk], b1 = chunk_end[chunk];
  T acc[kVvorOutsPerThread];
  int om[kVvorOutsPerThread], oc[kVvorOutsPerThread];
#pragma unroll
  for (int s = 0; s < kVvorOutsPerThread; ++s) {
    acc[s] = T(0);
    const int64_t o = o_base + threadIdx.x + static_cast<int64_t>(s) * kVvorThreads;
    om[s] = o < per ? static_cast<int>(o / cin) : -1;
    oc[s] = o < per ? static_cast<int>(o % cin) : 0;
  }
  for (int64_t e0 = b0; e0 < b1; e0 += rows_per_batch) {
    const int nr = static_cast<int>(b1 - e0 < rows_per_batch ? b1 - e0 : rows_per_batch);
    __syncthreads();
    for (int x = threadIdx.x; x < nr * cout; x += blockDim.x) {
      const int r = x / cout, m = x - r * cout;
      gs[x] = gout[(static_cast<int64_t>(ci[e0 + r]) * G + g) * cout + m];
    }
    for (int x = threadIdx.x; x < nr * cin; x += blockDim.x) {
      const int r = x / cin, c = x - r * cin;
      fs[x] = fin[(static_cast<int64_t>(cj[e0 + r]) * G + g) * cin + c];
    }
    __syncthreads();
    for (int r = 0; r < nr; ++r) {
#pragma unroll
      for (int s = 0; s < kVvorOutsPerThread; ++s)
        if (om[s] >= 0) acc[s] = fma(gs[r * cout + om[s]], fs[r * cin + oc[s]], acc[s]);
    }
  }
  T* p = partial + (chunk * G + g) * per;
#pragma unroll
  for (int s = 0; s < kVvorOutsPerThread; ++s) {
    const int64_t o = o_base + threadIdx.x + static_cast<int64_t>(s) * kVvorThreads;
    if (o < per) p[o] = acc[s];
  }
}

// grad[k][g][o] = sum over chunks c of cell k (ascending) of partial[c][g][o]
template <typename T>
__global__ void k_vvor_reduce(const T* __restrict__ partial, const int64_t* __restrict__ kc_ptr,
                              int64_t K, int G, int64_t per, T* __restrict__ grad) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= K * G * per) return;
  const int64_t k = p / (G * per), rem = p - k * G * per;
  T s = T(0);
  for (int64_t c = kc_ptr[k]; c < kc_ptr[k + 1]; ++c) s += partial[c * G * per + rem];
  grad[p] = s;
}

template <typename T>
void vvor_cells(npcg_context* ctx, const CellPlan& cells, const T* gout, const T* fin, int G,
                int cin, int cout, T* grad) {
  const int64_t K = cells.n_kernels;
  const int64_t per = static_cast<int64_t>(cout) * cin;
  const int64_t chunk_len = 4096;
  std::vector<int64_t> cb, ce, kc(K + 1, 0);
  for (int64_t k = 0; k < K; ++k) {
    kc[k] = static_cast<int64_t>(cb.size());
    for (int64_t s = cells.k_ptr_host[k]; s < cells.k_ptr_host[k + 1]; s += chunk_len) {
      cb.push_back(s);
      ce.push_back(std::min(cells.k_ptr_host[k + 1], s + chunk_len));
    }
  }
  kc[K] = static_cast<int64_t>(cb.size());
  const int64_t nch = static_cast<int64_t>(cb.size());
  const int64_t total = K * G * per;
  if (nch == 0) {
    NPCG_CUDA(cudaMemsetAsync(grad, 0, total * sizeof(T), ctx->stream));
    return;
  }
  DevBuf<int64_t> d_cb(ctx, nch), d_ce(ctx, nch), d_kc(ctx, K + 1);
  NPCG_CUDA(cudaMemcpyAsync(d_cb.get(), cb.data(), nch * 8, cudaMemcpyHostToDevice, ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(d_ce.get(), ce.data(), nch * 8, cudaMemcpyHostToDevice, ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(d_kc.get(), kc.data(), (K + 1) * 8, cudaMemcpyHostToDevice,
                            ctx->stream));
  DevBuf<T> partial(ctx, nch * G * per);
  int rows = static_cast<int>(48 * 1024 / ((cin + cout) * sizeof(T)));
  rows = rows < 1 ? 1 : (rows > 32 ? 32 : rows);
  const size_t smem = static_cast<size_t>(rows) * (cin + cout) * sizeof(T);
  const unsigned oz = static_cast<unsigned>(ceil_div(per, kVvorOutsPerBlock));
  launch(ctx, "vvor_simt", k_vvor_chunks<T>,
         dim3(static_cast<unsigned>(nch), static_cast<unsigned>(G), oz), dim3(kVvorThreads), smem,
         cells.i.get(), cells.j.get(), static_cast<const int64_t*>(d_cb.get()),
         static_cast<const int64_t*>(d_ce.get()), gout, fin, G, cin, cout, rows, partial.get());
  launch(ctx, "vvor_reduce", k_vvor_reduce<T>, dim3(static_cast<unsigned>(ceil_div(total, 256))),
         dim3(256), 0, static_cast<const T*>(partial.get()),
         static_cast<const int64_t*>(d_kc.get()), K, G, per, grad);
}

// explicit instantiations
template void mvmr_rows<float>(npcg_context*, const CsrView&, const float*, const float*, int,
                               int, int, float*, int64_t);
template void mvmr_rows<double>(npcg_context*, const CsrView&, const double*, const double*, int,
                                int, int, double*, int64_t);
template void transpose_w<float>(npcg_context*, const float*, int64_t, int, int, float*);
template void transpose_w<double>(npcg_context*, const double*, int64_t, int, int, double*);
template void vvor_cells<float>(npcg_context*, const CellPlan&, const float*, const float*, int,
                                int, int, float*);
template void vvor_cells<double>(npcg_context*, const CellPlan&, const double*, const double*,
                                 int, int, int, double*);

}  // namespace npcg
