// neighbors.cu -- GPU spatial-hash radius search + fused kernel-cell
// assignment, bit-exact with the reference.
//
// Reference: spatial.cpp:20-92 (radius_search), triplets.cpp:42-76
// (local_voxel_kernel_index, build_triplets_native), triplets.cpp:135-170
// (sort_triplets).  The reference buckets targets on a grid of edge
// `radius`, sorts (key, index) and binary-searches 27 cells per query.  Here:
//   1. per-point cell key (batch, floor(x/r), floor(y/r), floor(z/r)) in fp64
//      with IEEE division (__ddiv_rn), exactly cell_of (spatial.cpp:20-22);
//   2. an open-addressing hash table over occupied cells (owner = first
//      inserted point; keys compared by value), cell counts, a scan and a
//      scatter give per-cell point ranges -- the GPU analogue of bucket_points;
//   3. a count pass and a fill pass over the 27 neighbor cells of each query,
//      processed in spatial (Morton) order so a warp walks adjacent cells;
//      the distance test is the compiled reference recipe
//      d2 = fma(dz, dz, fma(dx, dx, dy*dy)), accepted iff r*r >= d2;
//   4. the fill pass also evaluates local_voxel_kernel_index with the exact
//      operation order sub -> add -> div -> floor -> clamp (no FMA);
//   5. each query's hits are ranked by j (the reference sorts `found`), giving
//      the (i, j) emission order of build_triplets_native.
#include <algorithm>

#include "neighbors.cuh"

#include <cstdlib>
#include <cstring>

namespace npcg {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// validation
// ---------------------------------------------------------------------------
__global__ void k_check_finite(const double* __restrict__ xyz, int64_t n3, int* flag) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n3;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (!isfinite(xyz[e])) *flag = 1;
}

void validate_cloud(npcg_context* ctx, const npcg_cloud* c, const char* what) {
  if (!c) fail(NPCG_ERR_INVALID, std::string(what) + ": null cloud");
  if (c->n_points < 0) fail(NPCG_ERR_SHAPE, std::string(what) + ": negative point count");
  if (c->n_points > 0 && !c->xyz) fail(NPCG_ERR_INVALID, std::string(what) + ": null xyz");
  // point_cloud.cpp:20-31
  if (!c->batch_offsets || c->n_batches < 1)
    fail(NPCG_ERR_OFFSET, "batch_offsets needs at least [0, N]");
  const int64_t* o = c->batch_offsets;
  if (o[0] != 0) fail(NPCG_ERR_OFFSET, "batch_offsets must start at 0");
  if (o[c->n_batches] != c->n_points)
    fail(NPCG_ERR_OFFSET,
         "batch_offsets must end at the point count (" + std::to_string(c->n_points) + ")");
  for (int64_t b = 1; b <= c->n_batches; ++b)
    if (o[b] < o[b - 1]) fail(NPCG_ERR_OFFSET, "batch_offsets must be monotone non-decreasing");
  if (c->n_points > 0xFFFFFFFEll)
    fail(NPCG_ERR_SHAPE, std::string(what) + ": more than 2^32-1 points (u32 triplet indices)");
  if (c->n_points == 0) return;
  DevBuf<int> flag(ctx, 1);
  NPCG_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), ctx->stream));
  const int64_t n3 = 3 * c->n_points;
  launch(ctx, "check_finite", k_check_finite,
         dim3(static_cast<unsigned>(std::min<int64_t>(ceil_div(n3, 256), 4 * ctx->num_sms))),
         dim3(256), 0, c->xyz, n3, flag.get());
  int h = 0;
  NPCG_CUDA(cudaMemcpyAsync(&h, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h) fail(NPCG_ERR_NONFINITE, "point coordinate is NaN or infinite");
}

// ---------------------------------------------------------------------------
// per-point batch ids and cell keys
// ---------------------------------------------------------------------------
__global__ void k_batch_ids(const int64_t* __restrict__ off, int64_t nb, int64_t n,
                            uint32_t* __restrict__ bid) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  // last b with off[b] <= p  (upper_bound - 1; handles empty batches)
  int64_t lo = 0, hi = nb + 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid] <= p) lo = mid + 1;
    else hi = mid;
  }
  bid[p] = static_cast<uint32_t>(lo - 1);
}

__device__ __forceinline__ int64_t cell_of(double c, double edge) {
  return static_cast<int64_t>(floor(__ddiv_rn(c, edge)));  // spatial.cpp:20-22
}

__global__ void k_cell_keys(const double* __restrict__ xyz, const uint32_t* __restrict__ bid,
                            int64_t n, double edge, longlong4* __restrict__ keys) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  keys[p] = make_longlong4(static_cast<long long>(bid[p]), cell_of(xyz[3 * p], edge),
                           cell_of(xyz[3 * p + 1], edge), cell_of(xyz[3 * p + 2], edge));
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}
__device__ __forceinline__ uint64_t hash_key(const longlong4& k) {
  uint64_t h = mix64(static_cast<uint64_t>(k.x) + 0x9E3779B97F4A7C15ULL);
  h = mix64(h ^ static_cast<uint64_t>(k.y));
  h = mix64(h ^ (static_cast<uint64_t>(k.z) * 0xD6E8FEB86659FD93ULL));
  h = mix64(h ^ (static_cast<uint64_t>(k.w) * 0xA0761D6478BD642FULL));
  return h;
}
__device__ __forceinline__ bool key_eq(const longlong4& a, const longlong4& b) {
  return a.x == b.x && a.y == b.y && a.z == b.z && a.w == b.w;
}

__global__ void k_hash_insert(const longlong4* __restrict__ keys, int64_t n,
                              uint32_t* __restrict__ slots, uint64_t mask,
                              uint32_t* __restrict__ cell_of_pt, uint32_t* __restrict__ cell_cnt) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const longlong4 k = keys[p];
  uint64_t h = hash_key(k) & mask;
  while (true) {
    const uint32_t cur = atomicCAS(&slots[h], kEmpty, static_cast<uint32_t>(p));
    if (cur == kEmpty || key_eq(keys[cur], k)) break;
    h = (h + 1) & mask;
  }
  cell_of_pt[p] = static_cast<uint32_t>(h);
  atomicAdd(&cell_cnt[h], 1u);
}

__global__ void k_cell_scatter(const uint32_t* __restrict__ cell_of_pt, int64_t n,
                               const uint32_t* __restrict__ cell_start,
                               uint32_t* __restrict__ cell_fill, uint32_t* __restrict__ cell_pts) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t h = cell_of_pt[p];
  cell_pts[cell_start[h] + atomicAdd(&cell_fill[h], 1u)] = static_cast<uint32_t>(p);
}

// target coordinates in cell order (a cell's candidates are contiguous: the
// probe loop reads them without the index indirection)
__global__ void k_gather_xyz(const uint32_t* __restrict__ cell_pts, const double* __restrict__ xyz, int64_t n,
                             double* __restrict__ sxyz) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int64_t p = cell_pts[q];
#pragma unroll
  for (int a = 0; a < 3; ++a) sxyz[3 * q + a] = xyz[3 * p + a];
}

__device__ __forceinline__ int64_t find_cell(const longlong4& probe,
                                             const uint32_t* __restrict__ slots, uint64_t mask,
                                             const longlong4* __restrict__ keys) {
  uint64_t h = hash_key(probe) & mask;
  while (true) {
    const uint32_t o = slots[h];
    if (o == kEmpty) return -1;
    if (key_eq(keys[o], probe)) return static_cast<int64_t>(h);
    h = (h + 1) & mask;
  }
}

// triplets.cpp:30-51 -- exact fp64 recipe, no contraction.
// The IEEE quotient is only needed when x / cell lies within rounding distance
// of an integer (floor could differ); elsewhere floor of x * (1 / cell) is the
// same integer (relative error < 2^-50 on |u| <= t + 1, margin 2^-30).
__device__ __forceinline__ double cell_floor(double x, double cell, double inv_cell) {
  const double q = __dmul_rn(x, inv_cell);
  const double f = floor(q);
  if (q - f > 0x1p-30 && f + 1.0 - q > 0x1p-30) return f;
  return floor(__ddiv_rn(x, cell));
}
__device__ __forceinline__ int64_t kernel_cell(const double* __restrict__ center,
                                               const double* __restrict__ nbr, double radius,
                                               int64_t t, double cell, double inv_cell) {
  int64_t idx[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double u = cell_floor(__dadd_rn(__dsub_rn(nbr[a], center[a]), radius), cell, inv_cell);
    int64_t c = static_cast<int64_t>(u);
    c = c < 0 ? 0 : (c > t - 1 ? t - 1 : c);
    idx[a] = c;
  }
  return (idx[0] * t + idx[1]) * t + idx[2];
}

struct Grid {
  const uint32_t* slots;
  uint64_t mask;
  const longlong4* keys;
  const uint32_t* cell_start;
  const uint32_t* cell_cnt;
  const uint32_t* cell_pts;
  const double* sxyz;  // target coordinates in cell_pts order
};

// Count (FILL=false) or fill (FILL=true) the neighbors of each query.
template <bool FILL>
__global__ void __launch_bounds__(256) k_query(const double* __restrict__ qxyz,
                                               const uint32_t* __restrict__ qbid,
                                               const uint32_t* __restrict__ qorder, int64_t nq,
                                               const double* __restrict__ txyz, Grid g,
                                               double radius, int64_t t,
                                               int64_t* __restrict__ counts,
                                               const int64_t* __restrict__ row_ptr,
                                               uint32_t* __restrict__ out_j,
                                               uint32_t* __restrict__ out_k,
                                               uint32_t* __restrict__ scr_j,
                                               uint32_t* __restrict__ scr_k, int cap,
                                               int* __restrict__ scr_over) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nq) return;
  const int64_t i = qorder ? qorder[s] : s;
  const double q[3] = {qxyz[3 * i], qxyz[3 * i + 1], qxyz[3 * i + 2]};
  const double r2 = __dmul_rn(radius, radius);  // spatial.cpp:62
  const long long b = qbid[i];
  const int64_t cx = cell_of(q[0], radius), cy = cell_of(q[1], radius),
                cz = cell_of(q[2], radius);
  const double kcell = t > 0 ? __ddiv_rn(__dmul_rn(2.0, radius), static_cast<double>(t)) : 1.0;
  const double kinv = __drcp_rn(kcell);
  int64_t pos = 0;
  if (FILL) pos = row_ptr[i];
  int64_t cnt = 0;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        const longlong4 probe = make_longlong4(b, cx + dx, cy + dy, cz + dz);
        const int64_t h = find_cell(probe, g.slots, g.mask, g.keys);
        if (h < 0) continue;
        const uint32_t s0 = g.cell_start[h], n0 = g.cell_cnt[h];
        for (uint32_t e = 0; e < n0; ++e) {
          const double* tp = g.sxyz + 3 * static_cast<int64_t>(s0 + e);
          const double ddx = __dsub_rn(q[0], tp[0]);
          const double ddy = __dsub_rn(q[1], tp[1]);
          const double ddz = __dsub_rn(q[2], tp[2]);
          const double d2 = __fma_rn(ddz, ddz, __fma_rn(ddx, ddx, __dmul_rn(ddy, ddy)));
          if (r2 >= d2) {
            const uint32_t p = g.cell_pts[s0 + e];
            if (FILL) {
              out_j[pos + cnt] = p;
              if (t > 0) out_k[pos + cnt] = static_cast<uint32_t>(kernel_cell(q, tp, radius, t, kcell, kinv));
            } else if (scr_j && cnt < cap) {  // one-pass build: the hits of row i at i * cap
              scr_j[i * cap + cnt] = p;
              if (t > 0) scr_k[i * cap + cnt] = static_cast<uint32_t>(kernel_cell(q, tp, radius, t, kcell, kinv));
            }
            ++cnt;
          }
        }
      }
  if (!FILL) {
    counts[i] = cnt;
    if (scr_over && cnt > cap) *scr_over = 1;
  }
}

// Rank-sort each row by j (j values are unique within a row).
// (in_stride > 0: row r's input entries start at r * in_stride -- the one-pass
// build's per-row scratch -- instead of at its CSR position)
__global__ void k_sort_rows(const int64_t* __restrict__ row_ptr, int64_t n_rows,
                            const uint32_t* __restrict__ in_j, const uint32_t* __restrict__ in_k,
                            uint32_t* __restrict__ out_j, uint32_t* __restrict__ out_k,
                            int64_t in_stride) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const int64_t s = row_ptr[row], len = row_ptr[row + 1] - s;
  if (in_stride) {  // shift the inputs so that in_j[s + x] is the row's x-th scratch entry
    in_j += row * in_stride - s;
    if (in_k) in_k += row * in_stride - s;
  }
  if (len <= 32) {
    const uint32_t mine = lane < len ? in_j[s + lane] : 0xFFFFFFFFu;
    uint32_t rank = 0;
    for (int l = 0; l < len; ++l) rank += __shfl_sync(0xffffffffu, mine, l) < mine;
    if (lane < len) {
      out_j[s + rank] = mine;
      if (in_k) out_k[s + rank] = in_k[s + lane];
    }
  } else {
    for (int64_t a = lane; a < len; a += 32) {
      const uint32_t mine = in_j[s + a];
      int64_t rank = 0;
      for (int64_t c = 0; c < len; ++c) rank += in_j[s + c] < mine;
      out_j[s + rank] = mine;
      if (in_k) out_k[s + rank] = in_k[s + a];
    }
  }
}

// ---------------------------------------------------------------------------
// spatial order: (batch, Morton code of the r/2 cell) -> perm
// ---------------------------------------------------------------------------
// per-axis minimum cell; warp-reduced, one atomic per warp and axis
__global__ void k_minmax_cells(const double* __restrict__ xyz, int64_t n, double inv_edge,
                               long long* __restrict__ mn) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    long long v = p < n ? static_cast<long long>(floor(xyz[3 * p + a] * inv_edge)) : LLONG_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const long long u = __shfl_xor_sync(0xffffffffu, v, o);
      v = u < v ? u : v;
    }
    if ((threadIdx.x & 31) == 0 && v != LLONG_MAX) atomicMin(&mn[a], v);
  }
}

__device__ __forceinline__ uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1fffffULL;
  v = (v | (v << 32)) & 0x1f00000000ffffULL;
  v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
  v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
  v = (v | (v << 2)) & 0x1249249249249249ULL;
  return v;
}

__global__ void k_morton_keys(const double* __restrict__ xyz, const uint32_t* __restrict__ bid,
                              int64_t n, double inv_edge, const long long* __restrict__ mn,
                              int axis_bits, uint64_t* __restrict__ keys) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const long long lim = (1ll << axis_bits) - 1;
  uint64_t c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    long long v = static_cast<long long>(floor(xyz[3 * p + a] * inv_edge)) - mn[a];
    v = v < 0 ? 0 : (v > lim ? lim : v);
    c[a] = static_cast<uint64_t>(v);
  }
  const uint64_t m = spread3(c[0]) << 2 | spread3(c[1]) << 1 | spread3(c[2]);
  keys[p] = (static_cast<uint64_t>(bid[p]) << (3 * axis_bits)) | m;
}

void spatial_order(npcg_context* ctx, const double* xyz, const uint32_t* bid, int64_t n,
                          int64_t n_batches, double edge, DevBuf<uint32_t>& perm) {
  perm.alloc(ctx, n);
  if (n == 0) return;
  DevBuf<long long> mn(ctx, 3);
  const long long big[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
  NPCG_CUDA(cudaMemcpyAsync(mn.get(), big, sizeof(big), cudaMemcpyHostToDevice, ctx->stream));
  const double inv_edge = 1.0 / edge;
  const unsigned nb = static_cast<unsigned>(ceil_div(n, 256));
  launch(ctx, "morton_min", k_minmax_cells, dim3(nb), dim3(256), 0, xyz, n, inv_edge, mn.get());
  const int bbits = bits_for(static_cast<uint64_t>(n_batches > 1 ? n_batches - 1 : 0));
  const int axis_bits = std::min(21, (64 - bbits) / 3);
  DevBuf<uint64_t> keys(ctx, n);
  launch(ctx, "morton_keys", k_morton_keys, dim3(nb), dim3(256), 0, xyz, bid, n, inv_edge,
         static_cast<const long long*>(mn.get()), axis_bits, keys.get());
  iota_u32(ctx, perm.get(), n);
  radix_sort_u64(ctx, keys.get(), perm.get(), n, 3 * axis_bits + bbits);
}

// ---------------------------------------------------------------------------
// build
// ---------------------------------------------------------------------------
void batch_ids_of(npcg_context* ctx, const npcg_cloud* c, DevBuf<uint32_t>& bid) {
  bid.alloc(ctx, c->n_points);
  if (c->n_points == 0) return;
  DevBuf<int64_t> off(ctx, c->n_batches + 1);
  NPCG_CUDA(cudaMemcpyAsync(off.get(), c->batch_offsets, (c->n_batches + 1) * sizeof(int64_t),
                            cudaMemcpyHostToDevice, ctx->stream));
  launch(ctx, "batch_ids", k_batch_ids, dim3(static_cast<unsigned>(ceil_div(c->n_points, 256))),
         dim3(256), 0, static_cast<const int64_t*>(off.get()), c->n_batches, c->n_points,
         bid.get());
}

void build_neighbors(npcg_context* ctx, const npcg_cloud* qc, const npcg_cloud* tc,
                     double radius, int64_t t, npcg_neighbors* nb) {
  const int64_t nq = qc->n_points, nt = tc->n_points;
  nb->n_out = nq;
  nb->n_in = nt;
  nb->out_off.assign(qc->batch_offsets, qc->batch_offsets + qc->n_batches + 1);
  nb->in_off.assign(tc->batch_offsets, tc->batch_offsets + tc->n_batches + 1);
  nb->t = t;
  nb->n_kernels = t > 0 ? t * t * t : 1;
  nb->radius = radius;
  // same points and the same batches: the radius relation is symmetric (the
  // transposed structure and the input spatial order come from the forward's)
  nb->same_cloud = (qc->xyz == tc->xyz && nq == nt && qc->n_batches == tc->n_batches &&
                    std::equal(qc->batch_offsets, qc->batch_offsets + qc->n_batches + 1, tc->batch_offsets));
  nb->row_ptr.alloc(ctx, nq + 1);
  NPCG_CUDA(cudaMemsetAsync(nb->row_ptr.get(), 0, (nq + 1) * sizeof(int64_t), ctx->stream));

  DevBuf<uint32_t> qbid, tbid;
  batch_ids_of(ctx, qc, qbid);
  batch_ids_of(ctx, tc, tbid);
  // spatial orders (Morton over r/2 cells): query processing order + tile plans
  spatial_order(ctx, qc->xyz, qbid.get(), nq, qc->n_batches, 0.5 * radius, nb->perm_out);
  if (nb->same_cloud) {
    nb->perm_in.alloc(ctx, nt);
    if (nt)
      NPCG_CUDA(cudaMemcpyAsync(nb->perm_in.get(), nb->perm_out.get(), nt * sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    spatial_order(ctx, tc->xyz, tbid.get(), nt, tc->n_batches, 0.5 * radius, nb->perm_in);
  }
  if (nq == 0 || nt == 0) {
    nb->n_pairs = 0;
    return;
  }

  // 1-2: target grid (cell edge = radius)
  DevBuf<longlong4> keys(ctx, nt);
  const unsigned tb = static_cast<unsigned>(ceil_div(nt, 256));
  launch(ctx, "cell_keys", k_cell_keys, dim3(tb), dim3(256), 0, tc->xyz,
         static_cast<const uint32_t*>(tbid.get()), nt, radius, keys.get());
  uint64_t hsize = 1024;
  while (hsize < static_cast<uint64_t>(2 * nt)) hsize <<= 1;
  DevBuf<uint32_t> slots(ctx, hsize), cell_cnt(ctx, hsize), cell_start(ctx, hsize),
      cell_fill(ctx, hsize), cell_of_pt(ctx, nt), cell_pts(ctx, nt);
  NPCG_CUDA(cudaMemsetAsync(slots.get(), 0xFF, hsize * 4, ctx->stream));
  NPCG_CUDA(cudaMemsetAsync(cell_cnt.get(), 0, hsize * 4, ctx->stream));
  NPCG_CUDA(cudaMemsetAsync(cell_fill.get(), 0, hsize * 4, ctx->stream));
  launch(ctx, "hash_insert", k_hash_insert, dim3(tb), dim3(256), 0,
         static_cast<const longlong4*>(keys.get()), nt, slots.get(), hsize - 1, cell_of_pt.get(),
         cell_cnt.get());
  exclusive_scan_u32(ctx, cell_cnt.get(), cell_start.get(), static_cast<int64_t>(hsize), nullptr);
  launch(ctx, "cell_scatter", k_cell_scatter, dim3(tb), dim3(256), 0,
         static_cast<const uint32_t*>(cell_of_pt.get()), nt,
         static_cast<const uint32_t*>(cell_start.get()), cell_fill.get(), cell_pts.get());
  DevBuf<double> sxyz(ctx, nt * 3);
  launch(ctx, "gather_xyz", k_gather_xyz, dim3(tb), dim3(256), 0, static_cast<const uint32_t*>(cell_pts.get()),
         tc->xyz, nt, sxyz.get());
  Grid g{slots.get(), hsize - 1, keys.get(), cell_start.get(), cell_cnt.get(), cell_pts.get(), sxyz.get()};

  // 3: count (and, when the scratch fits, keep the hits: one-pass build)
  DevBuf<int64_t> counts(ctx, nq);
  const unsigned qb = static_cast<unsigned>(ceil_div(nq, 256));
  constexpr int kCap = 64;  // hits kept per query (more: the two-pass fill below)
  const bool one_pass = static_cast<uint64_t>(nq) * kCap * 8 <= (uint64_t(4) << 30);
  DevBuf<uint32_t> scr_j, scr_k;
  DevBuf<int> scr_over;
  int h_over = 1;
  if (one_pass) {
    scr_j.alloc(ctx, nq * kCap);
    if (t > 0) scr_k.alloc(ctx, nq * kCap);
    scr_over.alloc(ctx, 1);
    NPCG_CUDA(cudaMemsetAsync(scr_over.get(), 0, sizeof(int), ctx->stream));
  }
  launch(ctx, "radius_count", k_query<false>, dim3(qb), dim3(256), 0, qc->xyz,
         static_cast<const uint32_t*>(qbid.get()), static_cast<const uint32_t*>(nb->perm_out.get()),
         nq, tc->xyz, g, radius, t, counts.get(), static_cast<const int64_t*>(nullptr),
         static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), scr_j.get(),
         t > 0 ? scr_k.get() : static_cast<uint32_t*>(nullptr), kCap,
         one_pass ? scr_over.get() : static_cast<int*>(nullptr));
  if (one_pass)
    NPCG_CUDA(cudaMemcpyAsync(&h_over, scr_over.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  int64_t total = 0;
  exclusive_scan_i64(ctx, counts.get(), nb->row_ptr.get(), nq, &total);
  NPCG_CUDA(cudaMemcpyAsync(nb->row_ptr.get() + nq, &total, sizeof(int64_t),
                            cudaMemcpyHostToDevice, ctx->stream));
  nb->n_pairs = total;
  if (total > 0xFFFFFFFFll * 64) fail(NPCG_ERR_SHAPE, "radius_search: pair count too large");

  nb->col_j.alloc(ctx, total);
  if (t > 0) nb->col_k.alloc(ctx, total);
  if (one_pass && h_over == 0) {  // every row's hits are in the scratch: rank them by j
    launch(ctx, "sort_rows", k_sort_rows, dim3(static_cast<unsigned>(ceil_div(nq * 32, 256))), dim3(256), 0,
           static_cast<const int64_t*>(nb->row_ptr.get()), nq, static_cast<const uint32_t*>(scr_j.get()),
           t > 0 ? static_cast<const uint32_t*>(scr_k.get()) : static_cast<const uint32_t*>(nullptr),
           nb->col_j.get(), t > 0 ? nb->col_k.get() : static_cast<uint32_t*>(nullptr),
           static_cast<int64_t>(kCap));
    return;
  }
  // 4: fill (j, k) in probe order, 5: rank rows by j
  DevBuf<uint32_t> tmp_j(ctx, total), tmp_k(ctx, t > 0 ? total : 0);
  launch(ctx, "radius_fill", k_query<true>, dim3(qb), dim3(256), 0, qc->xyz,
         static_cast<const uint32_t*>(qbid.get()), static_cast<const uint32_t*>(nb->perm_out.get()),
         nq, tc->xyz, g, radius, t, static_cast<int64_t*>(nullptr),
         static_cast<const int64_t*>(nb->row_ptr.get()), tmp_j.get(), tmp_k.get(),
         static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), 0, static_cast<int*>(nullptr));
  launch(ctx, "sort_rows", k_sort_rows, dim3(static_cast<unsigned>(ceil_div(nq * 32, 256))),
         dim3(256), 0, static_cast<const int64_t*>(nb->row_ptr.get()), nq,
         static_cast<const uint32_t*>(tmp_j.get()),
         t > 0 ? static_cast<const uint32_t*>(tmp_k.get()) : static_cast<const uint32_t*>(nullptr),
         nb->col_j.get(), t > 0 ? nb->col_k.get() : static_cast<uint32_t*>(nullptr), static_cast<int64_t>(0));
}

// ---------------------------------------------------------------------------
// batched kernel index (triplets.hpp:48-49)
// ---------------------------------------------------------------------------
__global__ void k_kernel_index(const double* __restrict__ c, const double* __restrict__ nbr,
                               int64_t n, double radius, int64_t t, int64_t* __restrict__ k) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double cell = __ddiv_rn(__dmul_rn(2.0, radius), static_cast<double>(t));
  k[p] = kernel_cell(c + 3 * p, nbr + 3 * p, radius, t, cell, __drcp_rn(cell));
}
void kernel_index_batch(npcg_context* ctx, const double* c, const double* nbr, int64_t n,
                        double radius, int64_t t, int64_t* k) {
  launch(ctx, "kernel_index", k_kernel_index, dim3(static_cast<unsigned>(ceil_div(n, 256))),
         dim3(256), 0, c, nbr, n, radius, t, k);
}

// ---------------------------------------------------------------------------
// row expansion, sorting, plans
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_expand_rows(const int64_t* __restrict__ row_ptr, int64_t n_rows,
                              T* __restrict__ out) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const int64_t s = row_ptr[row], e = row_ptr[row + 1];
  for (int64_t p = s + lane; p < e; p += 32) out[p] = static_cast<T>(row);
}
void expand_rows_u32(npcg_context* ctx, const int64_t* row_ptr, int64_t n_rows, uint32_t* out) {
  launch(ctx, "expand_rows", k_expand_rows<uint32_t>,
         dim3(static_cast<unsigned>(ceil_div(n_rows * 32, 256))), dim3(256), 0, row_ptr, n_rows,
         out);
}
void expand_rows_i64(npcg_context* ctx, const int64_t* row_ptr, int64_t n_rows, int64_t* out) {
  launch(ctx, "expand_rows", k_expand_rows<int64_t>,
         dim3(static_cast<unsigned>(ceil_div(n_rows * 32, 256))), dim3(256), 0, row_ptr, n_rows,
         out);
}

__global__ void k_gather3(const uint32_t* __restrict__ perm, int64_t n,
                          const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                          const uint32_t* __restrict__ c, uint32_t* __restrict__ oa,
                          uint32_t* __restrict__ ob, uint32_t* __restrict__ oc) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t s = perm[p];
  if (oa) oa[p] = a[s];
  if (ob) ob[p] = b[s];
  if (oc) oc[p] = c[s];
}

void sort_triplets_by(npcg_context* ctx, const uint32_t* i, const uint32_t* j, const uint32_t* k,
                      int64_t n, int axis, int64_t key_range, uint32_t* oi, uint32_t* oj,
                      uint32_t* ok) {
  if (n <= 0) return;
  const uint32_t* key = axis == NPCG_SORT_BY_I ? i : (axis == NPCG_SORT_BY_J ? j : k);
  DevBuf<uint32_t> keys(ctx, n), perm(ctx, n);
  NPCG_CUDA(cudaMemcpyAsync(keys.get(), key, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  iota_u32(ctx, perm.get(), n);
  const int bits = key_range > 0 ? bits_for(static_cast<uint64_t>(key_range - 1)) : 32;
  radix_sort_u32(ctx, keys.get(), perm.get(), n, bits < 32 ? bits : 32);
  launch(ctx, "gather_triplets", k_gather3, dim3(static_cast<unsigned>(ceil_div(n, 256))),
         dim3(256), 0, static_cast<const uint32_t*>(perm.get()), n, i, j, k, oi, oj, ok);
}

// Sorted keys -> CSR row pointers: position p (0 < p < n) starts rows
// key[p-1]+1 .. key[p]; p = 0 starts rows 0 .. key[0], p = n closes the rest.
__global__ void k_row_bounds(const uint32_t* __restrict__ key, int64_t n, int64_t n_rows,
                             int64_t* __restrict__ row_ptr) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p > n) return;
  const int64_t lo = p == 0 ? 0 : static_cast<int64_t>(key[p - 1]) + 1;
  const int64_t hi = p == n ? n_rows : min(static_cast<int64_t>(key[p]), n_rows);
  for (int64_t r = lo; r <= hi; ++r) row_ptr[r] = p;
}

__global__ void k_oob(const uint32_t* __restrict__ v, int64_t n, int64_t bound, int* flag) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (static_cast<int64_t>(v[p]) >= bound) *flag = 1;
}
bool any_out_of_range(npcg_context* ctx, const uint32_t* v, int64_t n, int64_t bound) {
  if (n <= 0) return false;
  DevBuf<int> flag(ctx, 1);
  NPCG_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), ctx->stream));
  launch(ctx, "index_check", k_oob,
         dim3(static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 8 * ctx->num_sms))),
         dim3(256), 0, v, n, bound, flag.get());
  int h = 0;
  NPCG_CUDA(cudaMemcpyAsync(&h, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  return h != 0;
}

// CSR of rows over `rowkey` (i or j) with entries in stable input order.
static void csr_build(npcg_context* ctx, const uint32_t* rowkey, const uint32_t* col,
                      const uint32_t* k, int64_t n, int64_t n_rows, CsrPlan* out) {
  out->n_rows = n_rows;
  out->nnz = n;
  out->row_ptr.alloc(ctx, n_rows + 1);
  out->col.alloc(ctx, n);
  out->k.alloc(ctx, n);
  if (n == 0) {
    NPCG_CUDA(cudaMemsetAsync(out->row_ptr.get(), 0, (n_rows + 1) * 8, ctx->stream));
    return;
  }
  DevBuf<uint32_t> keys(ctx, n), perm(ctx, n);
  NPCG_CUDA(cudaMemcpyAsync(keys.get(), rowkey, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  iota_u32(ctx, perm.get(), n);
  radix_sort_u32(ctx, keys.get(), perm.get(), n,
                 std::max(1, bits_for(static_cast<uint64_t>(n_rows > 0 ? n_rows - 1 : 0))));
  // row_ptr[r] = first position of key >= r in the sorted keys (no atomics)
  launch(ctx, "row_bounds", k_row_bounds, dim3(static_cast<unsigned>(ceil_div(n + 1, 256))),
         dim3(256), 0, static_cast<const uint32_t*>(keys.get()), n, n_rows, out->row_ptr.get());
  launch(ctx, "gather_csr", k_gather3, dim3(static_cast<unsigned>(ceil_div(n, 256))), dim3(256),
         0, static_cast<const uint32_t*>(perm.get()), n, col, k, static_cast<const uint32_t*>(nullptr),
         out->col.get(), out->k.get(), static_cast<uint32_t*>(nullptr));
}

void csr_from_triplets(npcg_context* ctx, const npcg_triplets* T, bool transpose, int64_t n_rows,
                       CsrPlan* out) {
  csr_build(ctx, transpose ? T->j : T->i, transpose ? T->i : T->j, T->k, T->size, n_rows, out);
}

// Same-cloud handles: the radius relation is symmetric (d2 is computed from
// coordinate differences whose negation is exact, and the probe covers the same
// 27 cells), so row j of the transposed structure lists exactly row j's
// neighbours, i ascending: the forward arrays themselves.  Only the cells
// differ (k belongs to the pair (i, j): j relative to centre i), found by a
// binary search of j in forward row i.  A warp per row, rows in spatial order
// (neighbouring rows share most of their rows i: L2 hits).
__global__ void k_tcsr_cells(const int64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                             const uint32_t* __restrict__ kk, const uint32_t* __restrict__ perm,
                             int64_t n, uint32_t* __restrict__ out_k, int* __restrict__ missing) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const uint32_t j = perm[w];
  const int64_t e0 = row_ptr[j], e1 = row_ptr[j + 1];
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const uint32_t i = col[e];
    int64_t lo = row_ptr[i], hi = row_ptr[i + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (col[mid] < j) lo = mid + 1;
      else hi = mid;
    }
    if (lo < row_ptr[i + 1] && col[lo] == j) out_k[e] = kk[lo];
    else *missing = 1;
  }
}

static bool tcsr_sort_forced() {
  const char* e = std::getenv("NPCG_TCSR_SORT");  // (A/B and tests: the radix-sort build)
  return e && std::strcmp(e, "1") == 0;
}

void build_tcsr(npcg_context* ctx, npcg_neighbors* nb) {
  if (nb->tcsr) return;
  auto p = std::make_unique<CsrPlan>();
  if (nb->same_cloud && !nb->degraded && nb->t > 0 && !tcsr_sort_forced()) {
    const int64_t n = nb->n_out, nnz = nb->n_pairs;
    p->n_rows = n;
    p->nnz = nnz;
    p->row_ptr.alloc(ctx, n + 1);
    p->col.alloc(ctx, nnz);
    p->k.alloc(ctx, nnz);
    NPCG_CUDA(cudaMemcpyAsync(p->row_ptr.get(), nb->row_ptr.get(), (n + 1) * 8, cudaMemcpyDeviceToDevice,
                              ctx->stream));
    if (nnz) {
      NPCG_CUDA(cudaMemcpyAsync(p->col.get(), nb->col_j.get(), nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      DevBuf<int> missing(ctx, 1);
      NPCG_CUDA(cudaMemsetAsync(missing.get(), 0, 4, ctx->stream));
      launch(ctx, "tcsr_cells", k_tcsr_cells, dim3(static_cast<unsigned>(ceil_div(n * 32, 256))), dim3(256), 0,
             static_cast<const int64_t*>(nb->row_ptr.get()), static_cast<const uint32_t*>(nb->col_j.get()),
             static_cast<const uint32_t*>(nb->col_k.get()), static_cast<const uint32_t*>(nb->perm_out.get()), n,
             p->k.get(), missing.get());
      if (std::getenv("NPCG_PLAN_DEBUG")) {  // (the relation is symmetric by construction: checked on request)
        int h = 0;
        NPCG_CUDA(cudaMemcpyAsync(&h, missing.get(), 4, cudaMemcpyDeviceToHost, ctx->stream));
        NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (h) fail(NPCG_ERR_STATE, "transposed structure: asymmetric same-cloud neighbor relation");
      }
    }
    nb->tcsr = std::move(p);
    return;
  }
  DevBuf<uint32_t> ei(ctx, nb->n_pairs);
  if (nb->n_pairs) expand_rows_u32(ctx, nb->row_ptr.get(), nb->n_out, ei.get());
  // stable by j over the (i, j)-ordered list -> rows over j with i ascending
  csr_build(ctx, nb->col_j.get(), ei.get(), nb->col_k.get(), nb->n_pairs, nb->n_in, p.get());
  nb->tcsr = std::move(p);
}

static void cells_build(npcg_context* ctx, const uint32_t* i, const uint32_t* j,
                        const uint32_t* k, int64_t n, int64_t n_kernels, CellPlan* out) {
  out->n_kernels = n_kernels;
  out->nnz = n;
  out->k_ptr.alloc(ctx, n_kernels + 1);
  out->i.alloc(ctx, n);
  out->j.alloc(ctx, n);
  out->k_ptr_host.assign(n_kernels + 1, 0);
  if (n == 0) {
    NPCG_CUDA(cudaMemsetAsync(out->k_ptr.get(), 0, (n_kernels + 1) * 8, ctx->stream));
    return;
  }
  DevBuf<uint32_t> keys(ctx, n), perm(ctx, n);
  NPCG_CUDA(cudaMemcpyAsync(keys.get(), k, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  iota_u32(ctx, perm.get(), n);
  radix_sort_u32(ctx, keys.get(), perm.get(), n,
                 std::max(1, bits_for(static_cast<uint64_t>(n_kernels - 1))));
  // k_ptr from the sorted cells (no atomics on the K counters)
  launch(ctx, "row_bounds", k_row_bounds, dim3(static_cast<unsigned>(ceil_div(n + 1, 256))),
         dim3(256), 0, static_cast<const uint32_t*>(keys.get()), n, n_kernels, out->k_ptr.get());
  NPCG_CUDA(cudaMemcpyAsync(out->k_ptr_host.data(), out->k_ptr.get(), (n_kernels + 1) * 8,
                            cudaMemcpyDeviceToHost, ctx->stream));
  launch(ctx, "gather_cells", k_gather3, dim3(static_cast<unsigned>(ceil_div(n, 256))),
         dim3(256), 0, static_cast<const uint32_t*>(perm.get()), n, i, j,
         static_cast<const uint32_t*>(nullptr), out->i.get(), out->j.get(),
         static_cast<uint32_t*>(nullptr));
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void build_cells(npcg_context* ctx, npcg_neighbors* nb) {
  if (nb->cells) return;
  auto p = std::make_unique<CellPlan>();
  DevBuf<uint32_t> ei(ctx, nb->n_pairs);
  if (nb->n_pairs) expand_rows_u32(ctx, nb->row_ptr.get(), nb->n_out, ei.get());
  cells_build(ctx, ei.get(), nb->col_j.get(), nb->col_k.get(), nb->n_pairs, nb->n_kernels, p.get());
  nb->cells = std::move(p);
}

void cells_from_triplets(npcg_context* ctx, const npcg_triplets* T, int64_t n_kernels,
                         CellPlan* out) {
  cells_build(ctx, T->i, T->j, T->k, T->size, n_kernels, out);
}

}  // namespace npcg
