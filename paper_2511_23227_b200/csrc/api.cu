// api.cu -- the extern "C" boundary of libnpcg.so (include/npcg.h).
//
// Every entry point: validate exactly like the reference function it replaces
// (file:line cited per function), then dispatch to the device engines.
// Exceptions (npcg::Error) are converted to status codes here and never cross
// the ABI.
#include <cstdio>
#include <memory>

#include "conv.cuh"
#include "neighbors.cuh"

using namespace npcg;

namespace npcg {
void kernel_index_batch(npcg_context* ctx, const double* c, const double* nbr, int64_t n,
                        double radius, int64_t t, int64_t* k);
void voxel_downsample_impl(npcg_context* ctx, const npcg_cloud* cloud, double voxel,
                           int64_t* kept, int64_t* parent, int64_t* out_offsets, int64_t* n_kept);
void upsample_impl(npcg_context* ctx, const int64_t* parent, int64_t n_fine, const void* coarse,
                   int64_t n_coarse, int64_t row_bytes, void* fine);
}  // namespace npcg

namespace {

__global__ void k_widen(const uint32_t* a, int64_t n, int64_t* o) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n) o[p] = a[p];
}

void need(const void* p, const char* what) {
  if (!p) fail(NPCG_ERR_INVALID, std::string(what) + " is null");
}

// engine.cpp:29-33 validate_config
void validate_config(const npcg_exec_config* c) {
  if (c->L < 1) fail(NPCG_ERR_SHAPE, "ExecConfig: L must be >= 1");
  if (c->b_out < 1 || c->b_in < 1) fail(NPCG_ERR_SHAPE, "ExecConfig: tile sizes must be >= 1");
  if (c->workers < 0) fail(NPCG_ERR_SHAPE, "ExecConfig: workers must be >= 0");
  if (c->math < NPCG_MATH_AUTO || c->math > NPCG_MATH_F32TC)
    fail(NPCG_ERR_INVALID, "ExecConfig: unknown math mode");
}

// tensors.hpp:126-131 WeightTensor::validate_shape
void validate_weight_shape(int64_t t, int64_t G, int64_t cin, int64_t cout) {
  if (t < 1 || t % 2 == 0) fail(NPCG_ERR_SHAPE, "WeightTensor: kernel resolution t must be odd and >= 1");
  if (G < 1 || cin < 1 || cout < 1)
    fail(NPCG_ERR_SHAPE, "WeightTensor: need groups >= 1, c_in_g >= 1, c_out_g >= 1");
}

size_t dsize(npcg_dtype d) { return d == NPCG_F64 ? 8 : 4; }

int64_t cube_root_exact(int64_t K) {
  for (int64_t t = 1; t * t * t <= K; ++t)
    if (t * t * t == K) return t;
  return -1;
}

// Which engine runs: the exact CUDA-core engines, the bf16 tensor-core path
// (opt-in), or the split (fp32-contract) tensor-core path.  AUTO keeps the
// reference's fp32 contract: the split path where it applies (F32, G = 1,
// C_in / C_out multiples of 16 up to 256: narrow layers included -- at C = 32
// it is 1.4x (forward) to 6x (backward) faster than the exact engines), else
// the exact engines.
TcMode use_tc(const npcg_exec_config* cfg, npcg_dtype dtype, int64_t G, int64_t cin,
              int64_t cout, int64_t K) {
  switch (cfg->math) {
    case NPCG_MATH_EXACT:
      return TcMode::none;
    case NPCG_MATH_BF16:
      if (dtype != NPCG_F32) fail(NPCG_ERR_UNSUPPORTED, "bf16 math requires F32 tensors");
      if (!tc_supported(G, cin, cout, K, TcMode::bf16, true))
        fail(NPCG_ERR_UNSUPPORTED,
             "bf16 tensor-core path needs G=1, C_in, C_out multiples of 16 up to 256, K<=128");
      return TcMode::bf16;
    case NPCG_MATH_F32TC:
      if (dtype != NPCG_F32) fail(NPCG_ERR_UNSUPPORTED, "f32tc math requires F32 tensors");
      if (!tc_supported(G, cin, cout, K, TcMode::split, true))
        fail(NPCG_ERR_UNSUPPORTED,
             "split tensor-core path needs G=1, C_in, C_out multiples of 16 up to 256, K<=128");
      return TcMode::split;
    default:
      return dtype == NPCG_F32 && tc_supported(G, cin, cout, K, TcMode::split, true)
                 ? TcMode::split
                 : TcMode::none;
  }
}

// A transient neighbor handle over a raw TripletList: CSR over rows (stable
// input order), identity spatial order.
std::unique_ptr<npcg_neighbors> handle_from_triplets(npcg_context* ctx, const npcg_triplets* T,
                                                     int64_t n_out, int64_t n_in, int64_t t) {
  auto nb = std::make_unique<npcg_neighbors>();
  nb->n_out = n_out;
  nb->n_in = n_in;
  nb->out_off = {0, n_out};
  nb->in_off = {0, n_in};
  nb->t = t;
  nb->n_kernels = t * t * t;
  nb->n_pairs = T->size;
  CsrPlan csr;
  csr_from_triplets(ctx, T, false, n_out, &csr);
  nb->row_ptr = std::move(csr.row_ptr);
  nb->col_j = std::move(csr.col);
  nb->col_k = std::move(csr.k);
  nb->perm_out.alloc(ctx, n_out);
  nb->perm_in.alloc(ctx, n_in);
  if (n_out) iota_u32(ctx, nb->perm_out.get(), n_out);
  if (n_in) iota_u32(ctx, nb->perm_in.get(), n_in);
  return nb;
}

// dst[m] = src[idx[m]] / dst[idx[m]] = src[m], rows of `width` bytes (width % 4 == 0)
template <bool SCATTER>
__global__ void k_move_rows(const uint32_t* __restrict__ src, const int64_t* __restrict__ idx,
                            int64_t n, int64_t words, uint32_t* __restrict__ dst) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= n * words) return;
  const int64_t m = x / words, w = x % words;
  if (SCATTER) dst[idx[m] * words + w] = src[m * words + w];
  else dst[m * words + w] = src[idx[m] * words + w];
}
void gather_rows(npcg_context* ctx, const void* src, const int64_t* idx, int64_t n, int64_t width,
                 void* dst) {
  if (n == 0) return;
  const int64_t words = width / 4;
  launch(ctx, "gather_rows", k_move_rows<false>, dim3(static_cast<unsigned>(ceil_div(n * words, 256))),
         dim3(256), 0, static_cast<const uint32_t*>(src), idx, n, words, static_cast<uint32_t*>(dst));
}
void scatter_rows(npcg_context* ctx, const void* src, const int64_t* idx, int64_t n, int64_t width,
                  void* dst) {
  if (n == 0) return;
  const int64_t words = width / 4;
  launch(ctx, "scatter_rows", k_move_rows<true>, dim3(static_cast<unsigned>(ceil_div(n * words, 256))),
         dim3(256), 0, static_cast<const uint32_t*>(src), idx, n, words, static_cast<uint32_t*>(dst));
}

void forward_impl(npcg_context* ctx, npcg_neighbors* nb, npcg_dtype dtype, const void* w,
                  int64_t G, int64_t cin, int64_t cout, const void* fin,
                  const npcg_exec_config* cfg, void* fout) {
  const int64_t bytes = nb->n_out * G * cout * static_cast<int64_t>(dsize(dtype));
  if (nb->n_out == 0) return;
  if (nb->n_pairs == 0) {
    NPCG_CUDA(cudaMemsetAsync(fout, 0, bytes, ctx->stream));
    return;
  }
  if (const TcMode m = use_tc(cfg, dtype, G, cin, cout, nb->n_kernels); m != TcMode::none) {
    tc_forward(ctx, nb, m, static_cast<const float*>(w), static_cast<const float*>(fin),
               static_cast<float*>(fout), static_cast<int>(cin), static_cast<int>(cout));
    return;
  }
  const CsrView v{nb->row_ptr.get(), nb->col_j.get(), nb->col_k.get(), nb->n_out, nb->n_pairs};
  if (dtype == NPCG_F32)
    mvmr_rows<float>(ctx, v, static_cast<const float*>(w), static_cast<const float*>(fin),
                     static_cast<int>(G), static_cast<int>(cin), static_cast<int>(cout),
                     static_cast<float*>(fout), nb->n_kernels);
  else
    mvmr_rows<double>(ctx, v, static_cast<const double*>(w), static_cast<const double*>(fin),
                      static_cast<int>(G), static_cast<int>(cin), static_cast<int>(cout),
                      static_cast<double*>(fout), nb->n_kernels);
}

template <typename T>
void dgrad_exact(npcg_context* ctx, npcg_neighbors* nb, const T* w, int64_t G, int64_t cin,
                 int64_t cout, const T* gout, T* grad_in) {
  build_tcsr(ctx, nb);
  DevBuf<T> wt(ctx, nb->n_kernels * G * cin * cout);
  transpose_w<T>(ctx, w, nb->n_kernels * G, static_cast<int>(cin), static_cast<int>(cout), wt.get());
  mvmr_rows<T>(ctx, nb->tcsr->view(), wt.get(), gout, static_cast<int>(G), static_cast<int>(cout),
               static_cast<int>(cin), grad_in, nb->n_kernels);
}

void backward_impl(npcg_context* ctx, npcg_neighbors* nb, npcg_dtype dtype, const void* w,
                   int64_t G, int64_t cin, int64_t cout, const void* fin, const void* gout,
                   const npcg_exec_config* cfg, void* grad_in, void* grad_w) {
  const size_t ds = dsize(dtype);
  if (nb->n_pairs == 0) {
    if (grad_in && nb->n_in)
      NPCG_CUDA(cudaMemsetAsync(grad_in, 0, nb->n_in * G * cin * ds, ctx->stream));
    if (grad_w)
      NPCG_CUDA(cudaMemsetAsync(grad_w, 0, nb->n_kernels * G * cin * cout * ds, ctx->stream));
    return;
  }
  if (const TcMode m = use_tc(cfg, dtype, G, cin, cout, nb->n_kernels); m != TcMode::none) {
    tc_backward(ctx, nb, m, static_cast<const float*>(w), static_cast<const float*>(fin),
                static_cast<const float*>(gout), static_cast<float*>(grad_in),
                static_cast<float*>(grad_w), static_cast<int>(cin), static_cast<int>(cout),
                (cfg->flags & NPCG_FLAG_FIN_UNCHANGED) != 0);
    return;
  }
  if (grad_in) {
    if (dtype == NPCG_F32)
      dgrad_exact<float>(ctx, nb, static_cast<const float*>(w), G, cin, cout,
                         static_cast<const float*>(gout), static_cast<float*>(grad_in));
    else
      dgrad_exact<double>(ctx, nb, static_cast<const double*>(w), G, cin, cout,
                          static_cast<const double*>(gout), static_cast<double*>(grad_in));
  }
  if (grad_w) {
    build_cells(ctx, nb);
    if (dtype == NPCG_F32)
      vvor_cells<float>(ctx, *nb->cells, static_cast<const float*>(gout),
                        static_cast<const float*>(fin), static_cast<int>(G), static_cast<int>(cin),
                        static_cast<int>(cout), static_cast<float*>(grad_w));
    else
      vvor_cells<double>(ctx, *nb->cells, static_cast<const double*>(gout),
                         static_cast<const double*>(fin), static_cast<int>(G),
                         static_cast<int>(cin), static_cast<int>(cout),
                         static_cast<double*>(grad_w));
  }
}

// The handle's last user (see npcg_neighbors::last_stream).
void touch(npcg_context* ctx, npcg_neighbors* nb) {
  nb->last_stream = ctx->stream;
  nb->device = ctx->device;
  nb->used = true;
}

void check_triplets_struct(const npcg_triplets* T) {
  need(T, "triplets");
  if (T->size < 0) fail(NPCG_ERR_SHAPE, "triplets: negative size");
  if (T->size > 0) {
    need(T->i, "triplets.i");
    need(T->j, "triplets.j");
    need(T->k, "triplets.k");
  }
}

}  // namespace

extern "C" {

int npcg_api_version(void) { return NPCG_API_VERSION; }

const char* npcg_status_string(npcg_status s) {
  switch (s) {
    case NPCG_OK: return "ok";
    case NPCG_ERR_OFFSET: return "OffsetError";
    case NPCG_ERR_NONFINITE: return "NonFiniteError";
    case NPCG_ERR_SHAPE: return "ShapeError";
    case NPCG_ERR_RADIUS: return "RadiusError";
    case NPCG_ERR_VOXEL: return "VoxelError";
    case NPCG_ERR_INDEX: return "IndexError";
    case NPCG_ERR_DOMAIN: return "DomainError";
    case NPCG_ERR_STATE: return "StateError";
    case NPCG_ERR_IO: return "IOError";
    case NPCG_ERR_CUDA: return "CudaError";
    case NPCG_ERR_OOM: return "OutOfMemory";
    case NPCG_ERR_INVALID: return "InvalidArgument";
    case NPCG_ERR_UNSUPPORTED: return "Unsupported";
  }
  return "unknown";
}

npcg_status npcg_context_create(int device, void* stream, npcg_context** out) {
  if (!out) return NPCG_ERR_INVALID;
  *out = nullptr;
  auto ctx = std::make_unique<npcg_context>();
  ctx->device = device;
  const npcg_status s = guard(nullptr, [&] {
    int n = 0;
    NPCG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) fail(NPCG_ERR_INVALID, "no such CUDA device");
    NPCG_CUDA(cudaSetDevice(device));
    cudaDeviceProp p{};
    NPCG_CUDA(cudaGetDeviceProperties(&p, device));
    if (p.major != 10 || p.minor != 0)
      fail(NPCG_ERR_UNSUPPORTED, std::string("libnpcg is built for sm_100a (B200); device is ") +
                                     p.name);
    ctx->num_sms = p.multiProcessorCount;
    ctx->max_smem_optin = static_cast<int>(p.sharedMemPerBlockOptin);
    ctx->stream = static_cast<cudaStream_t>(stream);
    // stream-ordered allocations come from the device's default pool; keep
    // freed blocks cached there (a caching allocator, like torch's) instead
    // of returning them to the driver at every synchronisation
    cudaMemPool_t pool;
    NPCG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = ~0ull;
    NPCG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  });
  if (s != NPCG_OK) return s;
  *out = ctx.release();
  return NPCG_OK;
}

npcg_status npcg_context_destroy(npcg_context* ctx) {
  if (!ctx) return NPCG_ERR_INVALID;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& r : ctx->prof) {
    cudaEventDestroy(r.start);
    cudaEventDestroy(r.stop);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  delete ctx;
  return NPCG_OK;
}

npcg_status npcg_context_set_stream(npcg_context* ctx, void* stream) {
  if (!ctx) return NPCG_ERR_INVALID;
  ctx->stream = static_cast<cudaStream_t>(stream);
  return NPCG_OK;
}

npcg_status npcg_context_synchronize(npcg_context* ctx) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] { NPCG_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

const char* npcg_last_error(const npcg_context* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

npcg_status npcg_launch_count(const npcg_context* ctx, int64_t* count) {
  if (!ctx || !count) return NPCG_ERR_INVALID;
  *count = ctx->launches;
  return NPCG_OK;
}

npcg_status npcg_profile_enable(npcg_context* ctx, int enable) {
  if (!ctx) return NPCG_ERR_INVALID;
  ctx->profiling = enable != 0;
  return NPCG_OK;
}

npcg_status npcg_profile_reset(npcg_context* ctx) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& r : ctx->prof) {
      ctx->event_pool.push_back(r.start);
      ctx->event_pool.push_back(r.stop);
    }
    ctx->prof.clear();
  });
}

npcg_status npcg_profile_query(npcg_context* ctx, const char* name_substr, int64_t* launches,
                               double* total_ms) {
  if (!ctx || !launches || !total_ms) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
    int64_t n = 0;
    double ms = 0.0;
    for (auto& r : ctx->prof) {
      if (name_substr && !std::strstr(r.name, name_substr)) continue;
      float t = 0.f;
      NPCG_CUDA(cudaEventElapsedTime(&t, r.start, r.stop));
      ms += t;
      ++n;
    }
    *launches = n;
    *total_ms = ms;
  });
}

npcg_status npcg_profile_dump(npcg_context* ctx, char* buf, size_t buf_len) {
  if (!ctx || !buf || buf_len == 0) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<std::pair<std::string, std::pair<int64_t, double>>> agg;
    for (auto& r : ctx->prof) {
      float t = 0.f;
      NPCG_CUDA(cudaEventElapsedTime(&t, r.start, r.stop));
      bool found = false;
      for (auto& a : agg)
        if (a.first == r.name) {
          a.second.first++;
          a.second.second += t;
          found = true;
        }
      if (!found) agg.push_back({r.name, {1, t}});
    }
    std::string s;
    for (auto& a : agg) {
      char line[256];
      std::snprintf(line, sizeof line, "%s\t%lld\t%.6f\n", a.first.c_str(),
                    static_cast<long long>(a.second.first), a.second.second);
      s += line;
    }
    std::strncpy(buf, s.c_str(), buf_len - 1);
    buf[buf_len - 1] = 0;
  });
}

npcg_status npcg_memory_stats(const npcg_context* ctx, int64_t* current_bytes,
                              int64_t* peak_bytes) {
  if (!ctx) return NPCG_ERR_INVALID;
  if (current_bytes) *current_bytes = mem_current();
  if (peak_bytes) *peak_bytes = mem_peak();
  return NPCG_OK;
}

npcg_status npcg_memory_reset_peak(npcg_context* ctx) {
  if (!ctx) return NPCG_ERR_INVALID;
  mem_reset_peak();
  return NPCG_OK;
}

// ---- geometry -------------------------------------------------------------

// spatial.cpp:56-60 + triplets.cpp:53-56
static npcg_status build_common(npcg_context* ctx, const npcg_cloud* oc, const npcg_cloud* ic,
                                double radius, int64_t t, npcg_neighbors** out) {
  if (!ctx || !out) return NPCG_ERR_INVALID;
  *out = nullptr;
  return guard(ctx, [&] {
    if (t != 0 && (t < 1 || t % 2 == 0))
      fail(NPCG_ERR_SHAPE, "conv geometry: kernel resolution t must be odd and >= 1");
    validate_cloud(ctx, oc, "queries");
    validate_cloud(ctx, ic, "targets");
    if (!(radius > 0.0)) fail(NPCG_ERR_RADIUS, "radius_search: radius must be > 0");
    if (oc->n_batches != ic->n_batches)
      fail(NPCG_ERR_SHAPE, "radius_search: query and target batch counts differ");
    auto nb = std::make_unique<npcg_neighbors>();
    build_neighbors(ctx, oc, ic, radius, t, nb.get());
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = nb.release();
  });
}

npcg_status npcg_radius_search(npcg_context* ctx, const npcg_cloud* queries,
                               const npcg_cloud* targets, double radius, npcg_neighbors** out) {
  return build_common(ctx, queries, targets, radius, 0, out);
}

npcg_status npcg_build_triplets_native(npcg_context* ctx, const npcg_cloud* out_cloud,
                                       const npcg_cloud* in_cloud, double radius, int64_t t,
                                       npcg_neighbors** out) {
  if (t == 0) {  // t = 0 is the internal "no kernel cells" marker; reject like validate_t
    if (ctx) ctx->last_error = "conv geometry: kernel resolution t must be odd and >= 1";
    return NPCG_ERR_SHAPE;
  }
  return build_common(ctx, out_cloud, in_cloud, radius, t, out);
}

npcg_status npcg_build_triplets_degraded(npcg_context* ctx, const npcg_cloud* in_cloud,
                                         double voxel_size, int64_t t, npcg_neighbors** out) {
  if (!ctx || !out) return NPCG_ERR_INVALID;
  *out = nullptr;
  return guard(ctx, [&] {
    // triplets.cpp:79-81: validate_t, then the voxel size
    if (t < 1 || t % 2 == 0)
      fail(NPCG_ERR_SHAPE, "conv geometry: kernel resolution t must be odd and >= 1");
    if (!(voxel_size > 0.0)) fail(NPCG_ERR_VOXEL, "build_triplets_degraded: voxel_size must be > 0");
    validate_cloud(ctx, in_cloud, "in_cloud");
    auto nb = std::make_unique<npcg_neighbors>();
    build_degraded(ctx, in_cloud, voxel_size, t, nb.get());
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = nb.release();
  });
}

npcg_status npcg_neighbors_sites(const npcg_neighbors* nb, int64_t* n_sites, int64_t* n_fine,
                                 int64_t* n_batches) {
  if (!nb) return NPCG_ERR_INVALID;
  if (!nb->degraded) return NPCG_ERR_STATE;
  if (n_sites) *n_sites = nb->n_out;
  if (n_fine) *n_fine = nb->n_fine;
  if (n_batches) *n_batches = static_cast<int64_t>(nb->site_offsets.size()) - 1;
  return NPCG_OK;
}

npcg_status npcg_neighbors_export_sites(npcg_context* ctx, const npcg_neighbors* nb,
                                        double* snapped_xyz, int64_t* kept, int64_t* parent,
                                        int64_t* site_offsets) {
  if (!ctx || !nb) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    if (!nb->degraded) fail(NPCG_ERR_STATE, "PointConvOp: no degraded cache");
    const int64_t ns = nb->n_out;
    if (snapped_xyz && ns)
      NPCG_CUDA(cudaMemcpyAsync(snapped_xyz, nb->site_xyz.get(), 3 * ns * sizeof(double),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    if (kept && ns)
      NPCG_CUDA(cudaMemcpyAsync(kept, nb->kept.get(), ns * sizeof(int64_t),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    if (parent && nb->n_fine)
      NPCG_CUDA(cudaMemcpyAsync(parent, nb->parent.get(), nb->n_fine * sizeof(int64_t),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    if (site_offsets)
      std::copy(nb->site_offsets.begin(), nb->site_offsets.end(), site_offsets);
  });
}

npcg_status npcg_neighbors_destroy(npcg_neighbors* nb) {
  if (!nb) return NPCG_ERR_INVALID;
  if (nb->used) {
    cudaSetDevice(nb->device);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(nb->last_stream, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone)
      cudaStreamSynchronize(nb->last_stream);
  }
  delete nb;
  return NPCG_OK;
}

npcg_status npcg_neighbors_size(const npcg_neighbors* nb, int64_t* n_pairs) {
  if (!nb || !n_pairs) return NPCG_ERR_INVALID;
  *n_pairs = nb->n_pairs;
  return NPCG_OK;
}

npcg_status npcg_neighbors_info(const npcg_neighbors* nb, int64_t* n_out, int64_t* n_in,
                                int64_t* n_kernels, double* radius) {
  if (!nb) return NPCG_ERR_INVALID;
  if (n_out) *n_out = nb->n_out;
  if (n_in) *n_in = nb->n_in;
  if (n_kernels) *n_kernels = nb->n_kernels;
  if (radius) *radius = nb->radius;
  return NPCG_OK;
}

npcg_status npcg_neighbors_export_pairs(npcg_context* ctx, const npcg_neighbors* nb,
                                        int64_t* out_index, int64_t* in_index) {
  if (!ctx || !nb) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    if (nb->n_pairs == 0) return;
    need(out_index, "out_index");
    need(in_index, "in_index");
    expand_rows_i64(ctx, nb->row_ptr.get(), nb->n_out, out_index);
    launch(ctx, "widen", k_widen, dim3(static_cast<unsigned>(ceil_div(nb->n_pairs, 256))), dim3(256),
           0, static_cast<const uint32_t*>(nb->col_j.get()), nb->n_pairs, in_index);
  });
}

npcg_status npcg_neighbors_export_triplets(npcg_context* ctx, const npcg_neighbors* nb,
                                           int32_t axis, uint32_t* i, uint32_t* j, uint32_t* k) {
  if (!ctx || !nb) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    if (nb->t == 0) fail(NPCG_ERR_STATE, "export_triplets: handle has no kernel cells (radius_search)");
    if (axis < NPCG_SORT_NONE || axis > NPCG_SORT_BY_K) fail(NPCG_ERR_INVALID, "bad sort axis");
    const int64_t n = nb->n_pairs;
    if (n == 0) return;
    need(i, "i");
    need(j, "j");
    need(k, "k");
    if (axis == NPCG_SORT_NONE || axis == NPCG_SORT_BY_I) {
      expand_rows_u32(ctx, nb->row_ptr.get(), nb->n_out, i);
      NPCG_CUDA(cudaMemcpyAsync(j, nb->col_j.get(), n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      NPCG_CUDA(cudaMemcpyAsync(k, nb->col_k.get(), n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      return;
    }
    DevBuf<uint32_t> ei(ctx, n);
    expand_rows_u32(ctx, nb->row_ptr.get(), nb->n_out, ei.get());
    const int64_t range = axis == NPCG_SORT_BY_J ? nb->n_in : nb->n_kernels;
    sort_triplets_by(ctx, ei.get(), nb->col_j.get(), nb->col_k.get(), n, axis, range, i, j, k);
  });
}

npcg_status npcg_kernel_index(npcg_context* ctx, const double* centers, const double* neighbors,
                              int64_t n, double radius, int64_t t, int64_t* k) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    // triplets.cpp:44-45
    if (t < 1 || t % 2 == 0) fail(NPCG_ERR_SHAPE, "conv geometry: kernel resolution t must be odd and >= 1");
    if (!(radius > 0.0)) fail(NPCG_ERR_RADIUS, "local_voxel_kernel_index: radius must be > 0");
    if (n <= 0) return;
    need(centers, "centers");
    need(neighbors, "neighbors");
    need(k, "k");
    kernel_index_batch(ctx, centers, neighbors, n, radius, t, k);
  });
}

npcg_status npcg_sort_triplets(npcg_context* ctx, const npcg_triplets* in, int32_t axis,
                               uint32_t* oi, uint32_t* oj, uint32_t* ok) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    check_triplets_struct(in);
    if (axis < NPCG_SORT_NONE || axis > NPCG_SORT_BY_K) fail(NPCG_ERR_INVALID, "bad sort axis");
    const int64_t n = in->size;
    if (n == 0) return;
    need(oi, "oi");
    need(oj, "oj");
    need(ok, "ok");
    if (axis == NPCG_SORT_NONE || n <= 1) {  // triplets.cpp:136-139
      NPCG_CUDA(cudaMemcpyAsync(oi, in->i, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      NPCG_CUDA(cudaMemcpyAsync(oj, in->j, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      NPCG_CUDA(cudaMemcpyAsync(ok, in->k, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      return;
    }
    const int64_t range =
        axis == NPCG_SORT_BY_I ? in->n_out : (axis == NPCG_SORT_BY_J ? in->n_in : in->n_kernels);
    sort_triplets_by(ctx, in->i, in->j, in->k, n, axis, range, oi, oj, ok);
  });
}

int32_t npcg_choose_sort_axis(int64_t n_out, int64_t n_in, int64_t n_kernels) {
  const int64_t lo = n_in < n_out ? n_in : n_out;  // triplets.cpp:172-179
  if (n_kernels <= lo) return NPCG_SORT_BY_K;
  return n_out <= n_in ? NPCG_SORT_BY_I : NPCG_SORT_BY_J;
}

// ---- engines over raw triplets ----------------------------------------------

// engine.cpp:444-455 + run_engine 284-292
npcg_status npcg_mvmr(npcg_context* ctx, npcg_dtype dtype, const void* w, int64_t t,
                      int64_t groups, int64_t c_in, int64_t c_out, const void* fin,
                      int64_t n_fin, const npcg_triplets* T, int64_t n_out,
                      const npcg_exec_config* cfg, void* out) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    need(cfg, "cfg");
    check_triplets_struct(T);
    validate_weight_shape(t, groups, c_in, c_out);
    if (dtype != NPCG_F32 && dtype != NPCG_F64) fail(NPCG_ERR_INVALID, "bad dtype");
    const int64_t K = t * t * t;
    if (T->n_kernels != K) fail(NPCG_ERR_SHAPE, "mvmr: triplet n_kernels does not match weight kernel count");
    if (T->n_in > n_fin) fail(NPCG_ERR_SHAPE, "mvmr: triplet n_in exceeds feature rows");
    if (T->n_out > n_out) fail(NPCG_ERR_SHAPE, "mvmr: triplet n_out exceeds requested output size");
    validate_config(cfg);
    if (n_out < 0) fail(NPCG_ERR_SHAPE, "mvmr: negative output size");
    if (n_fin < 0) fail(NPCG_ERR_SHAPE, "mvmr: negative feature rows");
    if (any_out_of_range(ctx, T->i, T->size, n_out)) fail(NPCG_ERR_INDEX, "triplet output index out of range");
    if (any_out_of_range(ctx, T->j, T->size, n_fin)) fail(NPCG_ERR_INDEX, "triplet input index out of range");
    if (any_out_of_range(ctx, T->k, T->size, K)) fail(NPCG_ERR_INDEX, "triplet kernel index out of range");
    if (n_out == 0) return;
    need(out, "out");
    if (T->size > 0) {
      need(w, "w");
      need(fin, "fin");
    }
    auto nb = handle_from_triplets(ctx, T, n_out, n_fin, t);
    forward_impl(ctx, nb.get(), dtype, w, groups, c_in, c_out, fin, cfg, out);
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));  // transient handle freed after the work
  });
}

// engine.cpp:457-473
npcg_status npcg_mvmr_transposed(npcg_context* ctx, npcg_dtype dtype, const void* w, int64_t t,
                                 int64_t groups, int64_t c_in, int64_t c_out, const void* gout,
                                 int64_t n_gout, const npcg_triplets* T, int64_t n_in,
                                 const npcg_exec_config* cfg, void* out) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    need(cfg, "cfg");
    check_triplets_struct(T);
    validate_weight_shape(t, groups, c_in, c_out);
    if (dtype != NPCG_F32 && dtype != NPCG_F64) fail(NPCG_ERR_INVALID, "bad dtype");
    const int64_t K = t * t * t;
    if (T->n_kernels != K)
      fail(NPCG_ERR_SHAPE, "mvmr_transposed: triplet n_kernels does not match weight kernel count");
    if (T->n_out > n_gout) fail(NPCG_ERR_SHAPE, "mvmr_transposed: triplet n_out exceeds gradient rows");
    if (T->n_in > n_in) fail(NPCG_ERR_SHAPE, "mvmr_transposed: triplet n_in exceeds requested output size");
    validate_config(cfg);
    if (n_in < 0) fail(NPCG_ERR_SHAPE, "mvmr: negative output size");
    if (n_gout < 0) fail(NPCG_ERR_SHAPE, "mvmr: negative feature rows");
    // run_engine(wt, gout, j, i, k, n_in): out_idx = j, in_idx = i
    if (any_out_of_range(ctx, T->j, T->size, n_in)) fail(NPCG_ERR_INDEX, "triplet output index out of range");
    if (any_out_of_range(ctx, T->i, T->size, n_gout)) fail(NPCG_ERR_INDEX, "triplet input index out of range");
    if (any_out_of_range(ctx, T->k, T->size, K)) fail(NPCG_ERR_INDEX, "triplet kernel index out of range");
    if (n_in == 0) return;
    need(out, "out");
    if (T->size == 0) {
      NPCG_CUDA(cudaMemsetAsync(out, 0, n_in * groups * c_in * dsize(dtype), ctx->stream));
      return;
    }
    need(w, "w");
    need(gout, "gout");
    auto nb = handle_from_triplets(ctx, T, n_gout, n_in, t);
    backward_impl(ctx, nb.get(), dtype, w, groups, c_in, c_out, nullptr, gout, cfg, out, nullptr);
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// vvor.cpp:102-123
npcg_status npcg_vvor(npcg_context* ctx, npcg_dtype dtype, const void* gout, int64_t n_gout,
                      const void* fin, int64_t n_fin, int64_t groups, int64_t c_in,
                      int64_t c_out, const npcg_triplets* T, int64_t n_kernels,
                      const npcg_exec_config* cfg, void* grad) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    need(cfg, "cfg");
    check_triplets_struct(T);
    if (dtype != NPCG_F32 && dtype != NPCG_F64) fail(NPCG_ERR_INVALID, "bad dtype");
    if (cfg->L < 1) fail(NPCG_ERR_SHAPE, "vvor: L must be >= 1");
    if (cfg->b_out < 1 || cfg->b_in < 1) fail(NPCG_ERR_SHAPE, "vvor: tile sizes must be >= 1");
    if (cfg->math < NPCG_MATH_AUTO || cfg->math > NPCG_MATH_F32TC)
      fail(NPCG_ERR_INVALID, "ExecConfig: unknown math mode");
    if (groups < 1 || c_in < 1 || c_out < 1)
      fail(NPCG_ERR_SHAPE, "FeatureTensor: need n >= 0, groups >= 1, channels >= 1");
    if (n_kernels < 1) fail(NPCG_ERR_SHAPE, "vvor: n_kernels must be >= 1");
    if (T->n_kernels > n_kernels) fail(NPCG_ERR_SHAPE, "vvor: triplet n_kernels exceeds requested kernel count");
    if (T->n_out > n_gout) fail(NPCG_ERR_SHAPE, "vvor: triplet n_out exceeds gradient rows");
    if (T->n_in > n_fin) fail(NPCG_ERR_SHAPE, "vvor: triplet n_in exceeds feature rows");
    if (any_out_of_range(ctx, T->i, T->size, n_gout)) fail(NPCG_ERR_INDEX, "vvor: output index out of range");
    if (any_out_of_range(ctx, T->j, T->size, n_fin)) fail(NPCG_ERR_INDEX, "vvor: input index out of range");
    if (any_out_of_range(ctx, T->k, T->size, n_kernels)) fail(NPCG_ERR_INDEX, "vvor: kernel index out of range");
    need(grad, "grad");
    const size_t ds = dsize(dtype);
    if (T->size == 0) {
      NPCG_CUDA(cudaMemsetAsync(grad, 0, n_kernels * groups * c_in * c_out * ds, ctx->stream));
      return;
    }
    need(gout, "gout");
    need(fin, "fin");
    // vvor accepts any n_kernels (not only t^3): use the t-less exact engine
    // unless K is a cube handled by the tensor-core path.
    const int64_t t = cube_root_exact(n_kernels);
    if (t > 0 && t % 2 == 1 && use_tc(cfg, dtype, groups, c_in, c_out, n_kernels) != TcMode::none) {
      auto nb = handle_from_triplets(ctx, T, n_gout, n_fin, t);
      backward_impl(ctx, nb.get(), dtype, nullptr, groups, c_in, c_out, fin, gout, cfg, nullptr,
                    grad);
    } else {
      if (cfg->math == NPCG_MATH_BF16 || cfg->math == NPCG_MATH_F32TC)
        fail(NPCG_ERR_UNSUPPORTED, "tensor-core vvor needs K = t^3 (t odd), G=1, C multiples of 16");
      CellPlan cells;
      cells_from_triplets(ctx, T, n_kernels, &cells);
      if (dtype == NPCG_F32)
        vvor_cells<float>(ctx, cells, static_cast<const float*>(gout),
                          static_cast<const float*>(fin), static_cast<int>(groups),
                          static_cast<int>(c_in), static_cast<int>(c_out),
                          static_cast<float*>(grad));
      else
        vvor_cells<double>(ctx, cells, static_cast<const double*>(gout),
                           static_cast<const double*>(fin), static_cast<int>(groups),
                           static_cast<int>(c_in), static_cast<int>(c_out),
                           static_cast<double*>(grad));
    }
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ---- operator path ----------------------------------------------------------

static void check_op(npcg_neighbors* nb, npcg_dtype dtype, int64_t G, int64_t cin, int64_t cout,
                     const npcg_exec_config* cfg) {
  need(nb, "neighbors");
  need(cfg, "cfg");
  if (nb->t == 0) fail(NPCG_ERR_STATE, "conv: handle has no kernel cells (radius_search handle)");
  if (dtype != NPCG_F32 && dtype != NPCG_F64) fail(NPCG_ERR_INVALID, "bad dtype");
  validate_weight_shape(nb->t, G, cin, cout);
  validate_config(cfg);
}

npcg_status npcg_conv_forward(npcg_context* ctx, npcg_neighbors* nb, npcg_dtype dtype,
                              const void* w, int64_t groups, int64_t c_in, int64_t c_out,
                              const void* fin, const npcg_exec_config* cfg, void* fout) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    check_op(nb, dtype, groups, c_in, c_out, cfg);
    touch(ctx, nb);
    if (nb->n_out == 0) return;
    need(fout, "fout");
    need(w, "w");
    if (nb->n_in > 0) need(fin, "fin");
    if (nb->degraded) {
      // conv_op.hpp:133-158: the engines see one row per site, gathered from
      // each site's representative point; the gathered rows are the
      // operator's saved input for the backward
      const int64_t width = groups * c_in * static_cast<int64_t>(dsize(dtype));
      if (nb->site_fin.size() < nb->n_in * width) nb->site_fin.alloc(ctx, nb->n_in * width);
      gather_rows(ctx, fin, nb->kept.get(), nb->n_in, width, nb->site_fin.get());
      nb->site_fin_dtype = dtype;
      nb->site_fin_width = width;
      forward_impl(ctx, nb, dtype, w, groups, c_in, c_out, nb->site_fin.get(), cfg, fout);
      return;
    }
    forward_impl(ctx, nb, dtype, w, groups, c_in, c_out, fin, cfg, fout);
  });
}

npcg_status npcg_conv_backward(npcg_context* ctx, npcg_neighbors* nb, npcg_dtype dtype,
                               const void* w, int64_t groups, int64_t c_in, int64_t c_out,
                               const void* fin, const void* gout, const npcg_exec_config* cfg,
                               void* grad_in, void* grad_w) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    check_op(nb, dtype, groups, c_in, c_out, cfg);
    touch(ctx, nb);
    need(w, "w");
    if (nb->n_out > 0) need(gout, "gout");
    if (nb->degraded) {
      // conv_op.hpp:177-202: gradients w.r.t. the rows saved by the forward;
      // site input gradients scatter back to the representative points,
      // merged-away points keep zero rows
      const int64_t width = groups * c_in * static_cast<int64_t>(dsize(dtype));
      if (fin) {
        // the operator's saved input: its site rows are gathered again (the
        // handle may have served another layer's forward since)
        if (nb->site_fin.size() < nb->n_in * width) nb->site_fin.alloc(ctx, nb->n_in * width);
        gather_rows(ctx, fin, nb->kept.get(), nb->n_in, width, nb->site_fin.get());
        nb->site_fin_dtype = dtype;
        nb->site_fin_width = width;
      } else if (nb->site_fin_dtype != dtype) {
        fail(NPCG_ERR_STATE, "PointConvOp::backward: no cached forward inputs");
      } else if (nb->site_fin_width != width) {
        fail(NPCG_ERR_SHAPE, "PointConvOp::backward: layer widths differ from the cached forward's");
      }
      DevBuf<uint8_t> gi_sites(ctx, grad_in ? std::max<int64_t>(nb->n_in * width, 1) : 0);
      backward_impl(ctx, nb, dtype, w, groups, c_in, c_out, nb->site_fin.get(), gout, cfg,
                    grad_in ? gi_sites.get() : nullptr, grad_w);
      if (grad_in && nb->n_fine) {
        NPCG_CUDA(cudaMemsetAsync(grad_in, 0, nb->n_fine * width, ctx->stream));
        scatter_rows(ctx, gi_sites.get(), nb->kept.get(), nb->n_in, width, grad_in);
      }
      return;
    }
    if (grad_w && nb->n_in > 0) need(fin, "fin");
    backward_impl(ctx, nb, dtype, w, groups, c_in, c_out, fin, gout, cfg, grad_in, grad_w);
  });
}

npcg_status npcg_neighbors_prepare(npcg_context* ctx, npcg_neighbors* nb, int32_t math) {
  if (!ctx || !nb) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    if (nb->t == 0) fail(NPCG_ERR_STATE, "prepare: handle has no kernel cells");
    touch(ctx, nb);
    if (math == NPCG_MATH_EXACT || math == NPCG_MATH_AUTO) {
      build_tcsr(ctx, nb);
      build_cells(ctx, nb);
    }
    if (math != NPCG_MATH_EXACT && tc_supported(1, 64, 64, nb->n_kernels, TcMode::bf16, false))
      tc_prepare(ctx, nb, math == NPCG_MATH_BF16 ? TcMode::bf16 : TcMode::split);
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

npcg_status npcg_neighbors_plan_stats(npcg_context* ctx, npcg_neighbors* nb, int64_t* stats) {
  if (!ctx || !nb || !stats) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    if (nb->t == 0) fail(NPCG_ERR_STATE, "plan_stats: handle has no kernel cells");
    touch(ctx, nb);
    if (!tc_supported(1, 64, 64, nb->n_kernels, TcMode::bf16, false))
      fail(NPCG_ERR_UNSUPPORTED, "no tensor-core plan for this K");
    tc_plan_stats(ctx, nb, stats);
  });
}

npcg_status npcg_debug_trace_forward(npcg_context* ctx, npcg_neighbors* nb, const float* w,
                                     const float* fin, float* fout, int64_t* trace) {
  if (!ctx || !nb || !trace) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    if (nb->t == 0 || !tc_supported(1, 64, 64, nb->n_kernels, TcMode::bf16, false))
      fail(NPCG_ERR_UNSUPPORTED, "trace: tensor-core plan needs K<=128");
    tc_trace_forward(ctx, nb, w, fin, fout, trace);
  });
}

npcg_status npcg_voxel_downsample(npcg_context* ctx, const npcg_cloud* cloud, double voxel,
                                  int64_t* kept, int64_t* parent, int64_t* out_offsets,
                                  int64_t* n_kept) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    validate_cloud(ctx, cloud, "cloud");
    if (!(voxel > 0.0)) fail(NPCG_ERR_VOXEL, "voxel_downsample: voxel_size must be > 0");
    need(out_offsets, "out_offsets");
    need(n_kept, "n_kept");
    voxel_downsample_impl(ctx, cloud, voxel, kept, parent, out_offsets, n_kept);
  });
}

// spatial.cpp:154-169 (validation at :156-160 is the caller's map / tensor
// shapes; here the widths and the parent range)
npcg_status npcg_upsample(npcg_context* ctx, npcg_dtype dtype, const int64_t* parent,
                          int64_t n_fine, const void* coarse, int64_t n_coarse, int64_t width,
                          void* fine) {
  if (!ctx) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    if (dtype != NPCG_F32 && dtype != NPCG_F64) fail(NPCG_ERR_INVALID, "bad dtype");
    if (width < 1) fail(NPCG_ERR_SHAPE, "upsample: feature width must be >= 1");
    if (n_fine < 0 || n_coarse < 0) fail(NPCG_ERR_SHAPE, "upsample: negative row count");
    if (n_fine == 0) return;
    need(parent, "parent");
    need(coarse, "coarse");
    need(fine, "fine");
    upsample_impl(ctx, parent, n_fine, coarse, n_coarse, width * static_cast<int64_t>(dsize(dtype)),
                  fine);
  });
}

}  // extern "C"

// SURVEY.md §8(b) export names for the three engines
extern "C" {
npcg_status npcg_mvmr_fwd(npcg_context* ctx, npcg_dtype dtype, const void* w, int64_t t,
                          int64_t groups, int64_t c_in, int64_t c_out, const void* fin,
                          int64_t n_fin, const npcg_triplets* triplets, int64_t n_out,
                          const npcg_exec_config* cfg, void* out) {
  return npcg_mvmr(ctx, dtype, w, t, groups, c_in, c_out, fin, n_fin, triplets, n_out, cfg, out);
}
npcg_status npcg_mvmr_dgrad(npcg_context* ctx, npcg_dtype dtype, const void* w, int64_t t,
                            int64_t groups, int64_t c_in, int64_t c_out, const void* gout,
                            int64_t n_gout, const npcg_triplets* triplets, int64_t n_in,
                            const npcg_exec_config* cfg, void* out) {
  return npcg_mvmr_transposed(ctx, dtype, w, t, groups, c_in, c_out, gout, n_gout, triplets, n_in,
                              cfg, out);
}
npcg_status npcg_vvor_wgrad(npcg_context* ctx, npcg_dtype dtype, const void* gout, int64_t n_gout,
                            const void* fin, int64_t n_fin, int64_t groups, int64_t c_in,
                            int64_t c_out, const npcg_triplets* triplets, int64_t n_kernels,
                            const npcg_exec_config* cfg, void* grad) {
  return npcg_vvor(ctx, dtype, gout, n_gout, fin, n_fin, groups, c_in, c_out, triplets, n_kernels,
                   cfg, grad);
}
}  // extern "C"
