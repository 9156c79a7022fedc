// voxel.cu -- GPU voxel_downsample, bit-exact with spatial.cpp:94-152
// (the strided path).
//
// Reference: bucket points by (batch, floor(c/v)) sorted by (key, index);
// per run: centroid = left-to-right sum over members in ascending index,
// times inv = 1.0/count; representative = nearest member to the centroid
// (d2 with the same FMA nesting as radius_search), strict '<' keeps the lowest
// index on ties; output ordered by (batch, key).
//
// Here: four stable LSD radix passes (z, y, x, batch -- each field offset to
// non-negative and sorted over exactly its bit range) reproduce the
// lexicographic (key, index) order for any coordinate range; run heads are
// flagged and scanned into output slots; one thread per run replays the
// reference's sequential fp64 arithmetic with explicit _rn intrinsics.
#include <algorithm>

#include "neighbors.cuh"

namespace npcg {

__global__ void k_vox_field(const double* __restrict__ xyz, const uint32_t* __restrict__ perm,
                            int64_t n, int axis, double voxel, long long base,
                            uint64_t* __restrict__ key) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t s = perm[p];
  const long long c = static_cast<long long>(floor(__ddiv_rn(xyz[3 * s + axis], voxel)));
  key[p] = static_cast<uint64_t>(c - base);
}

__global__ void k_vox_minmax(const double* __restrict__ xyz, int64_t n, double voxel,
                             long long* __restrict__ mn, long long* __restrict__ mx) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
#pragma unroll
  for (int a = 0; a < 3; ++a) {  // warp-reduced: one atomic per warp and axis
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    if (p < n) lo = hi = static_cast<long long>(floor(__ddiv_rn(xyz[3 * p + a], voxel)));
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const long long u = __shfl_xor_sync(0xffffffffu, lo, o), w = __shfl_xor_sync(0xffffffffu, hi, o);
      lo = u < lo ? u : lo;
      hi = w > hi ? w : hi;
    }
    if ((threadIdx.x & 31) == 0 && lo != LLONG_MAX) {
      atomicMin(&mn[a], lo);
      atomicMax(&mx[a], hi);
    }
  }
}

__global__ void k_vox_batchkey(const uint32_t* __restrict__ bid, const uint32_t* __restrict__ perm,
                               int64_t n, uint64_t* __restrict__ key) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n) key[p] = bid[perm[p]];
}

__device__ __forceinline__ bool same_voxel(const double* xyz, const uint32_t* bid, uint32_t a,
                                           uint32_t b, double v) {
  if (bid[a] != bid[b]) return false;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax)
    if (floor(__ddiv_rn(xyz[3 * a + ax], v)) != floor(__ddiv_rn(xyz[3 * b + ax], v))) return false;
  return true;
}

__global__ void k_vox_heads(const double* __restrict__ xyz, const uint32_t* __restrict__ bid,
                            const uint32_t* __restrict__ perm, int64_t n, double v,
                            uint32_t* __restrict__ head) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  head[p] = (p == 0 || !same_voxel(xyz, bid, perm[p - 1], perm[p], v)) ? 1u : 0u;
}

__global__ void k_vox_runs(const uint32_t* __restrict__ head, const uint32_t* __restrict__ slot,
                           int64_t n, int64_t* __restrict__ run_start) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n && head[p]) run_start[slot[p]] = p;
}

__global__ void k_vox_reduce(const double* __restrict__ xyz, const uint32_t* __restrict__ bid,
                             const uint32_t* __restrict__ perm,
                             const int64_t* __restrict__ run_start, int64_t n_runs, int64_t n,
                             int64_t* __restrict__ kept, int64_t* __restrict__ parent,
                             uint32_t* __restrict__ run_batch) {
  const int64_t m = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (m >= n_runs) return;
  const int64_t s0 = run_start[m], s1 = m + 1 < n_runs ? run_start[m + 1] : n;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0;
  for (int64_t s = s0; s < s1; ++s) {  // spatial.cpp:111-118, ascending index
    const double* p = xyz + 3 * static_cast<int64_t>(perm[s]);
    c0 = __dadd_rn(c0, p[0]);
    c1 = __dadd_rn(c1, p[1]);
    c2 = __dadd_rn(c2, p[2]);
  }
  const double inv = __ddiv_rn(1.0, static_cast<double>(s1 - s0));
  c0 = __dmul_rn(c0, inv);
  c1 = __dmul_rn(c1, inv);
  c2 = __dmul_rn(c2, inv);
  int64_t best = perm[s0];
  double best_d2 = 0.0;
  for (int64_t s = s0; s < s1; ++s) {  // spatial.cpp:123-133
    const uint32_t q = perm[s];
    const double* p = xyz + 3 * static_cast<int64_t>(q);
    const double dx = __dsub_rn(p[0], c0), dy = __dsub_rn(p[1], c1), dz = __dsub_rn(p[2], c2);
    const double d2 = __fma_rn(dz, dz, __fma_rn(dx, dx, __dmul_rn(dy, dy)));
    if (s == s0 || d2 < best_d2) {
      best_d2 = d2;
      best = q;
    }
    parent[q] = m;
  }
  kept[m] = best;
  run_batch[m] = bid[perm[s0]];
}

void batch_ids_of(npcg_context* ctx, const npcg_cloud* c, DevBuf<uint32_t>& bid);

void voxel_downsample_impl(npcg_context* ctx, const npcg_cloud* cloud, double voxel,
                           int64_t* kept, int64_t* parent, int64_t* out_offsets, int64_t* n_kept) {
  const int64_t n = cloud->n_points, nbat = cloud->n_batches;
  if (n == 0) {
    for (int64_t b = 0; b <= nbat; ++b) out_offsets[b] = 0;
    *n_kept = 0;
    return;
  }
  if (!kept || !parent) fail(NPCG_ERR_INVALID, "voxel_downsample: null outputs");
  DevBuf<uint32_t> bid;
  batch_ids_of(ctx, cloud, bid);
  const unsigned nb = static_cast<unsigned>(ceil_div(n, 256));
  DevBuf<long long> mn(ctx, 3), mx(ctx, 3);
  const long long lo[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX}, hi[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
  NPCG_CUDA(cudaMemcpyAsync(mn.get(), lo, sizeof lo, cudaMemcpyHostToDevice, ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(mx.get(), hi, sizeof hi, cudaMemcpyHostToDevice, ctx->stream));
  launch(ctx, "voxel_minmax", k_vox_minmax, dim3(nb), dim3(256), 0, cloud->xyz, n, voxel, mn.get(),
         mx.get());
  long long hmn[3], hmx[3];
  NPCG_CUDA(cudaMemcpyAsync(hmn, mn.get(), sizeof hmn, cudaMemcpyDeviceToHost, ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(hmx, mx.get(), sizeof hmx, cudaMemcpyDeviceToHost, ctx->stream));
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));

  // stable LSD over fields z, y, x, batch starting from index order
  DevBuf<uint32_t> perm(ctx, n);
  DevBuf<uint64_t> key(ctx, n);
  iota_u32(ctx, perm.get(), n);
  for (int axis = 2; axis >= 0; --axis) {
    const uint64_t range = static_cast<uint64_t>(hmx[axis] - hmn[axis]);
    launch(ctx, "voxel_field", k_vox_field, dim3(nb), dim3(256), 0, cloud->xyz,
           static_cast<const uint32_t*>(perm.get()), n, axis, voxel, hmn[axis], key.get());
    radix_sort_u64(ctx, key.get(), perm.get(), n, std::max(1, bits_for(range)));
  }
  if (nbat > 1) {
    launch(ctx, "voxel_batchkey", k_vox_batchkey, dim3(nb), dim3(256), 0,
           static_cast<const uint32_t*>(bid.get()), static_cast<const uint32_t*>(perm.get()), n,
           key.get());
    radix_sort_u64(ctx, key.get(), perm.get(), n, std::max(1, bits_for(nbat - 1)));
  }
  DevBuf<uint32_t> head(ctx, n), slot(ctx, n);
  launch(ctx, "voxel_heads", k_vox_heads, dim3(nb), dim3(256), 0, cloud->xyz,
         static_cast<const uint32_t*>(bid.get()), static_cast<const uint32_t*>(perm.get()), n,
         voxel, head.get());
  uint32_t runs = 0;
  exclusive_scan_u32(ctx, head.get(), slot.get(), n, &runs);
  DevBuf<int64_t> run_start(ctx, runs);
  DevBuf<uint32_t> run_batch(ctx, runs);
  launch(ctx, "voxel_runs", k_vox_runs, dim3(nb), dim3(256), 0,
         static_cast<const uint32_t*>(head.get()), static_cast<const uint32_t*>(slot.get()), n,
         run_start.get());
  launch(ctx, "voxel_reduce", k_vox_reduce, dim3(static_cast<unsigned>(ceil_div(runs, 256))),
         dim3(256), 0, cloud->xyz, static_cast<const uint32_t*>(bid.get()),
         static_cast<const uint32_t*>(perm.get()), static_cast<const int64_t*>(run_start.get()),
         static_cast<int64_t>(runs), n, kept, parent, run_batch.get());
  std::vector<uint32_t> rb(runs);
  if (runs)
    NPCG_CUDA(cudaMemcpyAsync(rb.data(), run_batch.get(), runs * 4, cudaMemcpyDeviceToHost,
                              ctx->stream));
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  // spatial.cpp:135-152 batch offsets of the kept cloud
  out_offsets[0] = 0;
  int64_t b = 0;
  for (uint32_t m = 0; m < runs; ++m)
    while (b < static_cast<int64_t>(rb[m])) out_offsets[++b] = m;
  while (b < nbat) out_offsets[++b] = runs;
  *n_kept = runs;
}

// ---- upsample (spatial.cpp:154-169): fine row m = coarse row parent[m] ----
__global__ void k_parent_oob(const int64_t* __restrict__ parent, int64_t n, int64_t bound,
                             int* __restrict__ flag) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = parent[p];
    if (v < 0 || v >= bound) *flag = 1;
  }
}

// one thread per V-sized piece of a fine row (V = 16 B when rows allow it)
template <typename V>
__global__ void k_upsample_rows(const int64_t* __restrict__ parent, int64_t n_fine, int64_t pieces,
                                const V* __restrict__ coarse, V* __restrict__ fine) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= n_fine * pieces) return;
  const int64_t m = x / pieces, q = x % pieces;
  fine[x] = __ldg(coarse + parent[m] * pieces + q);
}

void upsample_impl(npcg_context* ctx, const int64_t* parent, int64_t n_fine, const void* coarse,
                   int64_t n_coarse, int64_t row_bytes, void* fine) {
  if (n_fine == 0) return;
  {
    DevBuf<int> flag(ctx, 1);
    NPCG_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), ctx->stream));
    launch(ctx, "upsample_check", k_parent_oob,
           dim3(static_cast<unsigned>(std::min<int64_t>(ceil_div(n_fine, 256), 8 * ctx->num_sms))),
           dim3(256), 0, parent, n_fine, n_coarse, flag.get());
    int h = 0;
    NPCG_CUDA(cudaMemcpyAsync(&h, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h) fail(NPCG_ERR_INDEX, "upsample: parent index outside the coarse rows");
  }
  const bool v16 = row_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(coarse) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(fine) % 16 == 0;
  if (v16) {
    const int64_t pieces = row_bytes / 16;
    launch(ctx, "upsample", k_upsample_rows<uint4>,
           dim3(static_cast<unsigned>(ceil_div(n_fine * pieces, 256))), dim3(256), 0, parent, n_fine,
           pieces, static_cast<const uint4*>(coarse), static_cast<uint4*>(fine));
  } else {
    const int64_t pieces = row_bytes / 4;
    launch(ctx, "upsample", k_upsample_rows<uint32_t>,
           dim3(static_cast<unsigned>(ceil_div(n_fine * pieces, 256))), dim3(256), 0, parent, n_fine,
           pieces, static_cast<const uint32_t*>(coarse), static_cast<uint32_t*>(fine));
  }
}

}  // namespace npcg
