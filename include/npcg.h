/*
 * npcg.h -- C ABI of the B200-native point-centric convolution library
 * (libnpcg.so).  PointCNN++ (arXiv 2511.23227) hot path: neighbor build,
 * kernel-cell assignment, MVMR forward / input-gradient and VVOR
 * weight-gradient, re-designed for sm_100a.
 *
 * Each entry point replaces one function of the reference C++ API
 * (paths relative to /root/reference/proj/core/include/npconv/):
 *
 *   npcg_radius_search            spatial.hpp:39-40   radius_search
 *   npcg_build_triplets_native    triplets.hpp:56-57  build_triplets_native
 *                                  (+ triplets.hpp:48-49 local_voxel_kernel_index, fused)
 *   npcg_kernel_index             triplets.hpp:48-49  local_voxel_kernel_index (batched)
 *   npcg_sort_triplets            triplets.hpp:78     sort_triplets
 *   npcg_choose_sort_axis         triplets.hpp:82     choose_sort_axis
 *   npcg_mvmr                     engine.hpp:66-69    mvmr
 *   npcg_mvmr_transposed          engine.hpp:73-76    mvmr_transposed
 *   npcg_vvor                     vvor.hpp:85-88      vvor
 *   npcg_conv_forward             conv_op.hpp:129-175 PointConvOp::forward (cache hit)
 *   npcg_conv_backward            conv_op.hpp:177-203 PointConvOp::backward
 *   npcg_voxel_downsample         spatial.hpp:47-48   voxel_downsample
 *   npcg_build_triplets_degraded  triplets.hpp:63-76  build_triplets_degraded
 *   npcg_neighbors_export_sites   conv_op.hpp:56-57   snapped_cloud / site_map
 *   npcg_allreduce_dw             SURVEY.md §8(b,e): the one multi-GPU exchange
 *                                  (no reference counterpart: the reference is
 *                                  single-process; dW is a sum, vvor.hpp:79-84)
 *
 * Conventions
 *  - All tensor / index arrays are DEVICE pointers on the context's device.
 *    Calls are asynchronous and ordered on the context's CUDA stream, except
 *    where a count must be returned to the host (documented per call); those
 *    synchronise the stream.  Batch offsets are small HOST arrays (validated
 *    on the host exactly like make_point_cloud, point_cloud.cpp:20-36).
 *  - Layouts are the reference's: features (N, G, C) row-major
 *    (tensors.hpp:14-16); weights (K, G, C_in, C_out) (tensors.hpp:64-66);
 *    weight gradient (K, G, C_out, C_in) (vvor.hpp:12-16); triplets SoA u32.
 *  - Outputs are caller-owned and fully overwritten (the reference returns
 *    fresh zero-initialised containers: tensors.hpp:25, engine.cpp:303).
 *  - Errors never cross the ABI as exceptions: every npc:: error class maps
 *    1:1 to a status code below; npcg_last_error() returns the message.
 *    Validation happens before any compute, as in the reference.
 *  - No CPU fallback exists: every compute entry point runs CUDA kernels for
 *    sm_100a; without a usable device the context cannot be created.
 */
#ifndef NPCG_H_
#define NPCG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NPCG_API_VERSION 1

/* Status codes: 1..9 mirror the npc:: error hierarchy (errors.hpp:10-67). */
typedef enum npcg_status {
  NPCG_OK = 0,
  NPCG_ERR_OFFSET = 1,      /* npc::OffsetError    */
  NPCG_ERR_NONFINITE = 2,   /* npc::NonFiniteError */
  NPCG_ERR_SHAPE = 3,       /* npc::ShapeError     */
  NPCG_ERR_RADIUS = 4,      /* npc::RadiusError    */
  NPCG_ERR_VOXEL = 5,       /* npc::VoxelError     */
  NPCG_ERR_INDEX = 6,       /* npc::IndexError     */
  NPCG_ERR_DOMAIN = 7,      /* npc::DomainError    */
  NPCG_ERR_STATE = 8,       /* npc::StateError     */
  NPCG_ERR_IO = 9,          /* npc::IOError        */
  NPCG_ERR_CUDA = 10,       /* CUDA runtime / launch failure */
  NPCG_ERR_OOM = 11,        /* device allocation failed */
  NPCG_ERR_INVALID = 12,    /* null handle / pointer, bad enum */
  NPCG_ERR_UNSUPPORTED = 13 /* e.g. bf16 math requested for fp64 data */
} npcg_status;

typedef enum npcg_dtype { NPCG_F32 = 0, NPCG_F64 = 1 } npcg_dtype;

/* triplets.hpp:15 SortAxis */
typedef enum npcg_sort_axis {
  NPCG_SORT_NONE = 0,
  NPCG_SORT_BY_I = 1,
  NPCG_SORT_BY_J = 2,
  NPCG_SORT_BY_K = 3
} npcg_sort_axis;

/* Arithmetic of the MVMR / VVOR engines.  The reference computes in the API
 * dtype (fp32 / fp64) and pins fp32 results at rel <= 1e-5 against an fp64
 * oracle (acceptance.cpp:39); AUTO keeps that contract, BF16 is an explicit
 * opt-in with its own (looser) bound. */
typedef enum npcg_math {
  NPCG_MATH_AUTO = 0,  /* fp32 contract (rel <= 1e-5): F32 tensors run on the split tensor-core
                          path (F32TC) where it applies (G=1, K<=128, C_in and C_out multiples of
                          16 up to 256), everything else (fp64, G>1, other widths) on EXACT */
  NPCG_MATH_EXACT = 1, /* CUDA cores in the API dtype (fp32 / fp64 FMA, fp32 accumulate for F32) */
  NPCG_MATH_BF16 = 2,  /* opt-in: tcgen05 tensor cores, bf16 operands, fp32 accumulate (F32 API
                          only; C_in and C_out multiples of 16 up to 256, zero-padded inside);
                          rel ~2e-3, bound 1e-2 */
  NPCG_MATH_F32TC = 3  /* tcgen05 with split operands: every fp32 operand, scaled by a power of
                          two, x s = hi + lo 2^-11 (two fp16), products hi*hi + hi*lo + lo*hi
                          (+ lo*lo for the weight gradient), fp32 accumulation in short chains;
                          rel ~1e-6 (bound 1e-5, the reference's fp32 bound).  C_in, C_out
                          multiples of 16 up to 256 (wider than 128: 128-column halves) */
} npcg_math;

/* npcg_exec_config.flags */
#define NPCG_FLAG_FIN_UNCHANGED 1 /* npcg_conv_backward: `fin` is the same, unmodified buffer the
                                     last npcg_conv_forward on this handle read (the operator's
                                     saved input, conv_op.hpp:138), so the forward's device image
                                     of it may be reused instead of re-converting it */

/* engine.hpp:22-29 ExecConfig.  L / b_out / b_in / workers are validated like
 * the reference (ShapeError when < 1 / < 0) and otherwise only hints: the GPU
 * engines choose their own tiling.  The GPU engines are always deterministic
 * (fixed-order reductions, no floating-point atomics), so `deterministic` is
 * satisfied for both values. */
typedef struct npcg_exec_config {
  int64_t L;
  int64_t b_out;
  int64_t b_in;
  int32_t executor;      /* 0 naive, 1 grouped (engine.hpp:11) */
  int32_t deterministic; /* engine.hpp:27 */
  int32_t workers;       /* engine.hpp:28 */
  int32_t math;          /* npcg_math */
  int32_t flags;         /* NPCG_FLAG_* */
  int32_t reserved;
} npcg_exec_config;

/* point_cloud.hpp:18-50 PointCloud.  xyz: DEVICE (n_points, 3) float64 AoS;
 * batch_offsets: HOST int64[n_batches + 1], [0, ..., n_points]. */
typedef struct npcg_cloud {
  const double* xyz;
  const int64_t* batch_offsets;
  int64_t n_points;
  int64_t n_batches;
} npcg_cloud;

/* triplets.hpp:20-30 TripletList (DEVICE arrays). */
typedef struct npcg_triplets {
  const uint32_t* i;
  const uint32_t* j;
  const uint32_t* k;
  int64_t size;
  int64_t n_out;
  int64_t n_in;
  int64_t n_kernels;
  int32_t sort_axis;
} npcg_triplets;

typedef struct npcg_context npcg_context;     /* device, stream, scratch, profiler */
typedef struct npcg_comm npcg_comm;           /* NCCL communicator (dW all-reduce) */
typedef struct npcg_neighbors npcg_neighbors; /* device-resident neighbor structure */

/* ---- context ------------------------------------------------------------ */
int npcg_api_version(void);
const char* npcg_status_string(npcg_status s);
/* stream: a cudaStream_t (NULL = legacy default stream of `device`). */
npcg_status npcg_context_create(int device, void* stream, npcg_context** out);
npcg_status npcg_context_destroy(npcg_context* ctx);
npcg_status npcg_context_set_stream(npcg_context* ctx, void* stream);
npcg_status npcg_context_synchronize(npcg_context* ctx);
/* Message of the last failing call on this context ("" if none). */
const char* npcg_last_error(const npcg_context* ctx);

/* ---- instrumentation (SURVEY.md §5 tracing) ------------------------------
 * Launch counter: every kernel the library launches increments it.
 * Profiler: when enabled, each launch is bracketed by CUDA events on the
 * context stream; npcg_profile_query sums the durations of launches whose
 * kernel name contains `name_substr` (synchronises the stream). */
npcg_status npcg_launch_count(const npcg_context* ctx, int64_t* count);
npcg_status npcg_profile_enable(npcg_context* ctx, int enable);
npcg_status npcg_profile_reset(npcg_context* ctx);
npcg_status npcg_profile_query(npcg_context* ctx, const char* name_substr, int64_t* launches,
                               double* total_ms);
/* Writes "name\tlaunches\ttotal_ms\n" lines for all profiled kernels. */
npcg_status npcg_profile_dump(npcg_context* ctx, char* buf, size_t buf_len);
/* Device bytes currently / at peak allocated by this context and its handles. */
npcg_status npcg_memory_stats(const npcg_context* ctx, int64_t* current_bytes,
                              int64_t* peak_bytes);
npcg_status npcg_memory_reset_peak(npcg_context* ctx);

/* ---- geometry: neighbor build + kernel-cell assignment ------------------- */
/* spatial.hpp:39-40.  All (i, j) with |targets[j] - queries[i]|_2 <= radius in
 * the same batch, ordered by (i, j).  Bit-exact with the reference: cell edge =
 * radius, 27-cell probe, d2 = fma(dz,dz,fma(dx,dx,dy*dy)) accepted iff
 * radius*radius >= d2 (spatial.cpp:20-92).  Synchronises (returns a count).
 * Errors: RADIUS (radius <= 0), SHAPE (batch counts differ), OFFSET, NONFINITE. */
npcg_status npcg_radius_search(npcg_context* ctx, const npcg_cloud* queries,
                               const npcg_cloud* targets, double radius,
                               npcg_neighbors** out);

/* triplets.hpp:56-57.  radius_search(out_cloud, in_cloud) + per-pair
 * local_voxel_kernel_index (fused into the fill pass, triplets.cpp:42-51).
 * Errors as radius_search, plus SHAPE for t even or < 1. */
npcg_status npcg_build_triplets_native(npcg_context* ctx, const npcg_cloud* out_cloud,
                                       const npcg_cloud* in_cloud, double radius, int64_t t,
                                       npcg_neighbors** out);

/* triplets.hpp:63-76 build_triplets_degraded (ConvMode::degraded).  Sites =
 * voxel_downsample(in_cloud, voxel_size) snapped to voxel centres; triplets
 * (site, neighbor site, k) for the occupied voxels within (t-1)/2 voxels, in
 * the reference's build order (export with NPCG_SORT_NONE).  The handle's
 * clouds are the sites (n_out = n_in = sites); npcg_conv_forward / backward
 * on it gather the in_cloud rows through kept_index and scatter the input
 * gradient back (conv_op.hpp:133-158, 193-202).  Errors: SHAPE (t), VOXEL. */
npcg_status npcg_build_triplets_degraded(npcg_context* ctx, const npcg_cloud* in_cloud,
                                         double voxel_size, int64_t t, npcg_neighbors** out);
/* Degraded handles only (else STATE): site count, original point count, batches. */
npcg_status npcg_neighbors_sites(const npcg_neighbors* nb, int64_t* n_sites, int64_t* n_fine,
                                 int64_t* n_batches);
/* conv_op.hpp:56-57 snapped_cloud() / site_map(): snapped_xyz (n_sites, 3)
 * float64, kept (n_sites) and parent (n_fine) int64 DEVICE; site_offsets HOST
 * int64[n_batches + 1].  Any output may be NULL.  STATE on a native handle. */
npcg_status npcg_neighbors_export_sites(npcg_context* ctx, const npcg_neighbors* nb,
                                        double* snapped_xyz, int64_t* kept, int64_t* parent,
                                        int64_t* site_offsets);

npcg_status npcg_neighbors_destroy(npcg_neighbors* nb);
npcg_status npcg_neighbors_size(const npcg_neighbors* nb, int64_t* n_pairs);
/* n_kernels = t^3 (1 for a plain radius_search handle). */
npcg_status npcg_neighbors_info(const npcg_neighbors* nb, int64_t* n_out, int64_t* n_in,
                                int64_t* n_kernels, double* radius);
/* NeighborList (spatial.hpp:14-20): int64 out_index / in_index, (i, j) order. */
npcg_status npcg_neighbors_export_pairs(npcg_context* ctx, const npcg_neighbors* nb,
                                        int64_t* out_index, int64_t* in_index);
/* TripletList in the given order: NONE = build order (i, j) -- identical to
 * build_triplets_native; BY_K / BY_I / BY_J -- identical to
 * sort_triplets(build_triplets_native(...), axis) (stable). */
npcg_status npcg_neighbors_export_triplets(npcg_context* ctx, const npcg_neighbors* nb,
                                           int32_t axis, uint32_t* i, uint32_t* j,
                                           uint32_t* k);

/* triplets.hpp:48-49, batched: k[p] = local_voxel_kernel_index(centers[p],
 * neighbors[p], radius, t) with the exact fp64 recipe.  centers / neighbors
 * are DEVICE (n, 3) float64.  Errors: SHAPE (t), RADIUS. */
npcg_status npcg_kernel_index(npcg_context* ctx, const double* centers, const double* neighbors,
                              int64_t n, double radius, int64_t t, int64_t* k);

/* triplets.hpp:78: stable counting sort of `in` by axis into (oi, oj, ok)
 * (device, may not alias the inputs). */
npcg_status npcg_sort_triplets(npcg_context* ctx, const npcg_triplets* in, int32_t axis,
                               uint32_t* oi, uint32_t* oj, uint32_t* ok);
/* triplets.hpp:82 (pure host function). */
int32_t npcg_choose_sort_axis(int64_t n_out, int64_t n_in, int64_t n_kernels);

/* ---- MVMR / VVOR engines over a raw TripletList --------------------------- */
/* engine.hpp:66-69: out (n_out, G, C_out) = sum over triplets of W[k]^T fin[j]
 * into row i.  w (t^3, G, C_in, C_out); fin (n_fin, G, C_in).
 * Errors (engine.cpp:284-292, 448-453): SHAPE, INDEX. */
npcg_status npcg_mvmr(npcg_context* ctx, npcg_dtype dtype, const void* w, int64_t t,
                      int64_t groups, int64_t c_in, int64_t c_out, const void* fin,
                      int64_t n_fin, const npcg_triplets* triplets, int64_t n_out,
                      const npcg_exec_config* cfg, void* out);
/* engine.hpp:73-76: out (n_in, G, C_in) = sum of W[k] gout[i] into row j.
 * gout (n_gout, G, C_out).  No transposed weight copy is materialised. */
npcg_status npcg_mvmr_transposed(npcg_context* ctx, npcg_dtype dtype, const void* w, int64_t t,
                                 int64_t groups, int64_t c_in, int64_t c_out, const void* gout,
                                 int64_t n_gout, const npcg_triplets* triplets, int64_t n_in,
                                 const npcg_exec_config* cfg, void* out);
/* vvor.hpp:85-88: grad (n_kernels, G, C_out, C_in) = sum of gout[i] (x) fin[j]
 * into cell k.  Errors (vvor.cpp:106-123): SHAPE, INDEX. */
npcg_status npcg_vvor(npcg_context* ctx, npcg_dtype dtype, const void* gout, int64_t n_gout,
                      const void* fin, int64_t n_fin, int64_t groups, int64_t c_in,
                      int64_t c_out, const npcg_triplets* triplets, int64_t n_kernels,
                      const npcg_exec_config* cfg, void* grad);
/* The same three engines under the names of SURVEY.md §8(b)'s export list
 * (identical arguments and behaviour). */
npcg_status npcg_mvmr_fwd(npcg_context* ctx, npcg_dtype dtype, const void* w, int64_t t,
                          int64_t groups, int64_t c_in, int64_t c_out, const void* fin,
                          int64_t n_fin, const npcg_triplets* triplets, int64_t n_out,
                          const npcg_exec_config* cfg, void* out);
npcg_status npcg_mvmr_dgrad(npcg_context* ctx, npcg_dtype dtype, const void* w, int64_t t,
                            int64_t groups, int64_t c_in, int64_t c_out, const void* gout,
                            int64_t n_gout, const npcg_triplets* triplets, int64_t n_in,
                            const npcg_exec_config* cfg, void* out);
npcg_status npcg_vvor_wgrad(npcg_context* ctx, npcg_dtype dtype, const void* gout, int64_t n_gout,
                            const void* fin, int64_t n_fin, int64_t groups, int64_t c_in,
                            int64_t c_out, const npcg_triplets* triplets, int64_t n_kernels,
                            const npcg_exec_config* cfg, void* grad);

/* ---- operator path (PointConvOp with a cached neighbor structure) --------- */
/* conv_op.hpp:129-175 forward over a triplet handle (the PointConvOp cache,
 * conv_op.hpp:106-127).  fin (n_in, G, C_in) -> fout (n_out, G, C_out). */
npcg_status npcg_conv_forward(npcg_context* ctx, npcg_neighbors* nb, npcg_dtype dtype,
                              const void* w, int64_t groups, int64_t c_in, int64_t c_out,
                              const void* fin, const npcg_exec_config* cfg, void* fout);
/* conv_op.hpp:177-203 backward: grad_in = mvmr_transposed, grad_w = vvor.
 * Either output may be NULL to skip it.  `fin` is the operator's saved input
 * (PointConvOp copies it at forward, conv_op.hpp:138).  With
 * cfg->flags & NPCG_FLAG_FIN_UNCHANGED the tensor-core image the last forward
 * on this handle made of `fin` is reused (the caller guarantees it is the same
 * unmodified buffer); otherwise `fin` is read again.  On a degraded handle the
 * site rows are gathered again from `fin` (ShapeError if the operator's
 * widths differ from the forward's when `fin` is NULL). */
npcg_status npcg_conv_backward(npcg_context* ctx, npcg_neighbors* nb, npcg_dtype dtype,
                               const void* w, int64_t groups, int64_t c_in, int64_t c_out,
                               const void* fin, const void* gout, const npcg_exec_config* cfg,
                               void* grad_in, void* grad_w);
/* Builds (and caches in the handle) the compute plans the engines use, so
 * that the first forward / backward does not pay for them.  Optional. */
npcg_status npcg_neighbors_prepare(npcg_context* ctx, npcg_neighbors* nb, int32_t math);
/* Tensor-core tile-plan statistics (instrumentation; builds the plans): for
 * the forward, input-gradient and weight-gradient plans, four values each --
 * [super-tiles over all planning levels, rows beyond the capacity of 8-row
 *  tiles (served by the exact engine), max halo rows, mean halo rows x 100].
 * stats: HOST int64[12]. */
npcg_status npcg_neighbors_plan_stats(npcg_context* ctx, npcg_neighbors* nb, int64_t* stats);
/* Debug instrumentation: runs one tensor-core forward with per-stage pipeline
 * event clocks recorded for CTA 0; trace: HOST int64[512 x 8] (SM clock64 of
 * descriptor issue / arrival, A-slot free, aggregation done, MMA start / issue,
 * W arrival per stage).  Synchronises. */
npcg_status npcg_debug_trace_forward(npcg_context* ctx, npcg_neighbors* nb, const float* w,
                                     const float* fin, float* fout, int64_t* trace);

/* ---- strided path ------------------------------- */
/* spatial.hpp:47-48 voxel_downsample.  kept (n_points) / parent (n_points)
 * int64 DEVICE; out_offsets HOST int64[n_batches+1]; *n_kept set on return
 * (synchronises).  Errors: VOXEL (voxel <= 0). */
npcg_status npcg_voxel_downsample(npcg_context* ctx, const npcg_cloud* cloud, double voxel,
                                  int64_t* kept, int64_t* parent, int64_t* out_offsets,
                                  int64_t* n_kept);

/* spatial.hpp:52-54 upsample (spatial.cpp:154-169): fine (n_fine, width)
 * row m = coarse row parent[m]; parent: DEVICE int64[n_fine] (the map's
 * parent_of), coarse: DEVICE (n_coarse, width) of `dtype`.
 * Errors: SHAPE (width < 1), INDEX (a parent outside [0, n_coarse)). */
npcg_status npcg_upsample(npcg_context* ctx, npcg_dtype dtype, const int64_t* parent,
                          int64_t n_fine, const void* coarse, int64_t n_coarse, int64_t width,
                          void* fine);

/* ---- synthetic inputs (host) ---------------------------------------------
 * The reference core's seeded generators (synthetic.hpp:12-40,
 * tensors.hpp:142-150) over std::mt19937_64 (random.hpp:14-26), writing HOST
 * buffers: xyz (n, 3) float64; features (n, groups, channels) and weights
 * (t^3, groups, c_in, c_out) of `dtype`.  Errors: SHAPE, DOMAIN (extent <= 0). */
npcg_status npcg_gen_uniform_cube(int64_t n, double extent, uint64_t seed, double* xyz);
npcg_status npcg_gen_features(int64_t n, int64_t groups, int64_t channels, uint64_t seed,
                              npcg_dtype dtype, void* out);
npcg_status npcg_make_weights(int64_t t, int64_t groups, int64_t c_in, int64_t c_out,
                              uint64_t seed, npcg_dtype dtype, void* out);

/* ---- multi-GPU: dW all-reduce over NCCL -------------------
 * Whole point clouds are sharded per GPU; the weight gradient is the one
 * exchange: sum over ranks, in place, on the context stream.  NCCL is loaded
 * at first use (libnccl.so.2; the one a PyTorch process already has).
 * npcg_comm_unique_id: rank 0 creates the id (HOST bytes), the caller
 * broadcasts it (e.g. torch.distributed), every rank calls npcg_comm_create
 * (collective; synchronises).  NPCG_ERR_UNSUPPORTED when NCCL is absent. */
#define NPCG_COMM_ID_BYTES 128
npcg_status npcg_comm_unique_id(uint8_t* id);
npcg_status npcg_comm_create(npcg_context* ctx, int nranks, int rank, const uint8_t* id,
                             npcg_comm** out);
npcg_status npcg_comm_destroy(npcg_comm* comm);
/* dw: DEVICE (K, G, C_out, C_in) weight gradient, count elements, summed over
 * ranks in place (asynchronous, stream-ordered). */
npcg_status npcg_allreduce_dw(npcg_context* ctx, npcg_comm* comm, npcg_dtype dtype, void* dw,
                              int64_t count);

#ifdef __cplusplus
}
#endif
#endif /* NPCG_H_ */
