// degraded.cu -- the degraded (voxel) triplet build on the GPU,
// triplets.cpp:78-133 build_triplets_degraded, and the site gather / scatter
// the degraded PointConvOp wraps around the engines (conv_op.hpp:133-158,
// 193-202).
//
// Sites come from voxel_downsample (voxel.cu, bit-exact): one per occupied
// voxel, representative = the point nearest the centroid, in (batch, key)
// order -- so the site keys are already sorted and every neighbor lookup is
// a binary search over them (the reference uses a std::map).  Per site the
// t^3 integer offsets are visited in the reference's loop order (dx outer,
// dz inner), which is also ascending k; the handle's CSR rows keep that
// order, so exporting the triplets reproduces the reference's build order.
//
// Arithmetic (bit-exact with the reference object):
//   key_axis = (int64) floor(p_axis / v)             triplets.cpp:96-98
//   snapped  = ((double) key + 0.5) * v              triplets.cpp:101-103
#include <climits>
#include <vector>

#include "neighbors.cuh"

namespace npcg {

void voxel_downsample_impl(npcg_context* ctx, const npcg_cloud* cloud, double voxel,
                           int64_t* kept, int64_t* parent, int64_t* out_offsets, int64_t* n_kept);

namespace {

__global__ void k_site_keys(const double* __restrict__ xyz, const int64_t* __restrict__ kept,
                            int64_t ns, double v, long long* __restrict__ key,
                            double* __restrict__ snapped) {
  const int64_t m = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (m >= ns) return;
  const double* p = xyz + 3 * kept[m];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const long long c = static_cast<long long>(floor(__ddiv_rn(p[a], v)));
    key[3 * m + a] = c;
    snapped[3 * m + a] = __dmul_rn(__dadd_rn(static_cast<double>(c), 0.5), v);
  }
}

// Site whose key is (x, y, z) within [lo, hi) (one batch), or -1.
__device__ __forceinline__ int64_t find_site(const long long* __restrict__ key, int64_t lo,
                                             int64_t hi, long long x, long long y, long long z) {
  const int64_t end = hi;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const long long* q = key + 3 * mid;
    const bool less = q[0] != x ? q[0] < x : (q[1] != y ? q[1] < y : q[2] < z);
    if (less) lo = mid + 1;
    else hi = mid;
  }
  if (lo < end) {
    const long long* q = key + 3 * lo;
    if (q[0] == x && q[1] == y && q[2] == z) return lo;
  }
  return -1;
}

// Count (FILL = false) or write (FILL = true) each site's triplets.
template <bool FILL>
__global__ void k_degraded(const long long* __restrict__ key, const uint32_t* __restrict__ sbid,
                           const int64_t* __restrict__ soff, int64_t ns, int t,
                           const int64_t* __restrict__ row_ptr, int64_t* __restrict__ count,
                           uint32_t* __restrict__ col_j, uint32_t* __restrict__ col_k) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const int h = (t - 1) / 2;
  const uint32_t b = sbid[s];
  const int64_t lo = soff[b], hi = soff[b + 1];
  const long long x = key[3 * s], y = key[3 * s + 1], z = key[3 * s + 2];
  int64_t n = 0, base = FILL ? row_ptr[s] : 0;
  for (int dx = -h; dx <= h; ++dx)
    for (int dy = -h; dy <= h; ++dy)
      for (int dz = -h; dz <= h; ++dz) {
        const int64_t j = find_site(key, lo, hi, x + dx, y + dy, z + dz);
        if (j < 0) continue;
        if (FILL) {
          col_j[base + n] = static_cast<uint32_t>(j);
          col_k[base + n] = static_cast<uint32_t>(((dx + h) * t + (dy + h)) * t + (dz + h));
        }
        ++n;
      }
  if (!FILL) count[s] = n;
}

}  // namespace

void build_degraded(npcg_context* ctx, const npcg_cloud* in_cloud, double voxel, int64_t t,
                    npcg_neighbors* nb) {
  const int64_t n = in_cloud->n_points, nbat = in_cloud->n_batches;
  nb->degraded = true;
  nb->n_fine = n;
  nb->t = t;
  nb->n_kernels = t * t * t;
  nb->radius = voxel;
  nb->same_cloud = true;
  nb->site_offsets.assign(static_cast<size_t>(nbat + 1), 0);
  nb->kept.alloc(ctx, std::max<int64_t>(n, 1));
  nb->parent.alloc(ctx, std::max<int64_t>(n, 1));
  int64_t ns = 0;
  voxel_downsample_impl(ctx, in_cloud, voxel, nb->kept.get(), nb->parent.get(),
                        nb->site_offsets.data(), &ns);
  nb->n_out = nb->n_in = ns;
  nb->out_off = nb->in_off = nb->site_offsets;
  nb->site_xyz.alloc(ctx, std::max<int64_t>(3 * ns, 1));
  nb->row_ptr.alloc(ctx, ns + 1);
  if (ns == 0) {
    NPCG_CUDA(cudaMemsetAsync(nb->row_ptr.get(), 0, sizeof(int64_t), ctx->stream));
    nb->n_pairs = 0;
    nb->perm_out.alloc(ctx, 0);
    nb->perm_in.alloc(ctx, 0);
    return;
  }
  const unsigned blocks = static_cast<unsigned>(ceil_div(ns, 256));
  DevBuf<long long> key(ctx, 3 * ns);
  launch(ctx, "site_keys", k_site_keys, dim3(blocks), dim3(256), 0, in_cloud->xyz,
         static_cast<const int64_t*>(nb->kept.get()), ns, voxel, key.get(), nb->site_xyz.get());
  const npcg_cloud sites{nb->site_xyz.get(), nb->site_offsets.data(), ns, nbat};
  DevBuf<uint32_t> sbid;
  batch_ids_of(ctx, &sites, sbid);
  DevBuf<int64_t> soff(ctx, nbat + 1);
  NPCG_CUDA(cudaMemcpyAsync(soff.get(), nb->site_offsets.data(), (nbat + 1) * sizeof(int64_t),
                            cudaMemcpyHostToDevice, ctx->stream));
  DevBuf<int64_t> count(ctx, ns + 1);
  NPCG_CUDA(cudaMemsetAsync(count.get() + ns, 0, sizeof(int64_t), ctx->stream));
  launch(ctx, "degraded_count", k_degraded<false>, dim3(blocks), dim3(256), 0,
         static_cast<const long long*>(key.get()), static_cast<const uint32_t*>(sbid.get()),
         static_cast<const int64_t*>(soff.get()), ns, static_cast<int>(t),
         static_cast<const int64_t*>(nullptr), count.get(), static_cast<uint32_t*>(nullptr),
         static_cast<uint32_t*>(nullptr));
  int64_t total = 0;
  exclusive_scan_i64(ctx, count.get(), nb->row_ptr.get(), ns + 1, &total);
  nb->n_pairs = total;
  nb->col_j.alloc(ctx, std::max<int64_t>(total, 1));
  nb->col_k.alloc(ctx, std::max<int64_t>(total, 1));
  launch(ctx, "degraded_fill", k_degraded<true>, dim3(blocks), dim3(256), 0,
         static_cast<const long long*>(key.get()), static_cast<const uint32_t*>(sbid.get()),
         static_cast<const int64_t*>(soff.get()), ns, static_cast<int>(t),
         static_cast<const int64_t*>(nb->row_ptr.get()), static_cast<int64_t*>(nullptr),
         nb->col_j.get(), nb->col_k.get());
  // spatial (Morton) order of the sites for the tile plans; one cloud
  spatial_order(ctx, nb->site_xyz.get(), sbid.get(), ns, nbat, voxel, nb->perm_out);
  nb->perm_in.alloc(ctx, ns);
  NPCG_CUDA(cudaMemcpyAsync(nb->perm_in.get(), nb->perm_out.get(), ns * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, ctx->stream));
}

}  // namespace npcg
