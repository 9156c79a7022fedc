// neighbors.cuh -- the device-resident neighbor structure (npcg_neighbors)
// and the compute plans derived from it.
//
// Layout in HBM:
//   row_ptr  int64[n_out+1]   CSR over output points i
//   col_j    u32[|T|]         neighbor j, ascending within a row  -> (i, j) order
//   col_k    u32[|T|]         kernel cell of (i, j)  (absent for radius_search)
//   perm_out / perm_in u32    spatial (batch, Morton) order of each cloud
// Plans (built lazily, cached in the handle = the PointConvOp triplet cache):
//   T-CSR    rows = input points j, entries (i, k) in (j, i) order  -> dgrad
//   cells    entries in (k, i, j) order + k_ptr[K+1]                -> wgrad, by_k export
//   tiles    tcgen05 tile plans (conv_tc.cu)
#pragma once

#include <memory>

#include "npcg_internal.cuh"

namespace npcg {

// CSR view used by the SIMT engines: rows -> (col, k) entries.
struct CsrView {
  const int64_t* row_ptr = nullptr;
  const uint32_t* col = nullptr;
  const uint32_t* k = nullptr;
  int64_t n_rows = 0;
  int64_t nnz = 0;
};

// Per-cell entry list (k-major): entries of cell k are [k_ptr[k], k_ptr[k+1]).
struct CellView {
  const int64_t* k_ptr = nullptr;  // host-visible copy lives in CellPlan
  const uint32_t* i = nullptr;
  const uint32_t* j = nullptr;
  int64_t n_kernels = 0;
  int64_t nnz = 0;
};

struct CsrPlan {
  DevBuf<int64_t> row_ptr;
  DevBuf<uint32_t> col;
  DevBuf<uint32_t> k;
  int64_t n_rows = 0, nnz = 0;
  CsrView view() const { return {row_ptr.get(), col.get(), k.get(), n_rows, nnz}; }
};

struct CellPlan {
  DevBuf<int64_t> k_ptr;
  std::vector<int64_t> k_ptr_host;
  DevBuf<uint32_t> i, j;
  int64_t n_kernels = 0, nnz = 0;
  CellView view() const { return {k_ptr.get(), i.get(), j.get(), n_kernels, nnz}; }
};

struct TcPlan;  // conv_tc.cu
void destroy_tc_plan(TcPlan* p);
struct TcPlanDeleter {
  void operator()(TcPlan* p) const { destroy_tc_plan(p); }
};

}  // namespace npcg

struct npcg_neighbors {
  // the stream of the last call that used the handle: destroy synchronises it
  // before the stream-ordered frees of the cached buffers (which are ordered
  // on the streams they were allocated on)
  cudaStream_t last_stream = nullptr;
  bool used = false;
  int device = 0;
  int64_t n_out = 0, n_in = 0;
  // batch offsets of the output / input clouds (the spatial orders perm_out /
  // perm_in are batch-major, so batch b occupies permuted rows [off[b], off[b+1]))
  std::vector<int64_t> out_off, in_off;
  int64_t t = 0;          // 0: plain radius_search handle (no kernel cells)
  int64_t n_kernels = 1;  // t^3
  double radius = 0.0;
  int64_t n_pairs = 0;
  npcg::DevBuf<int64_t> row_ptr;  // n_out + 1
  npcg::DevBuf<uint32_t> col_j;   // (i, j) order
  npcg::DevBuf<uint32_t> col_k;
  npcg::DevBuf<uint32_t> perm_out, perm_in;  // spatial order of each cloud (may alias: same cloud)
  bool same_cloud = false;
  // degraded mode (triplets.cpp:78-133): the handle's clouds are the snapped
  // sites; conv calls gather / scatter the n_fine original rows through kept
  bool degraded = false;
  int64_t n_fine = 0;
  npcg::DevBuf<double> site_xyz;       // (n_sites, 3) voxel centres
  npcg::DevBuf<int64_t> kept, parent;  // DownsampleMap: kept_index (n_sites), parent_of (n_fine)
  std::vector<int64_t> site_offsets;   // host, n_batches + 1
  npcg::DevBuf<uint8_t> site_fin;      // engine-facing rows saved by the last forward
  int32_t site_fin_dtype = -1;
  int64_t site_fin_width = 0;          // bytes per saved site row
  // cached plans
  std::unique_ptr<npcg::CsrPlan> tcsr;   // transposed CSR (rows = input points)
  std::unique_ptr<npcg::CellPlan> cells; // (k, i, j)
  std::unique_ptr<npcg::TcPlan, npcg::TcPlanDeleter> tc;
};

namespace npcg {

void validate_cloud(npcg_context* ctx, const npcg_cloud* c, const char* what);
// (batch, Morton code of the `edge` cell) order of a cloud -> perm
void spatial_order(npcg_context* ctx, const double* xyz, const uint32_t* bid, int64_t n,
                   int64_t n_batches, double edge, DevBuf<uint32_t>& perm);
void batch_ids_of(npcg_context* ctx, const npcg_cloud* c, DevBuf<uint32_t>& bid);
// Degraded build (triplets.cpp:78-133) into nb; t and voxel validated by the caller.
void build_degraded(npcg_context* ctx, const npcg_cloud* in_cloud, double voxel, int64_t t,
                    npcg_neighbors* nb);
void build_neighbors(npcg_context* ctx, const npcg_cloud* out_cloud, const npcg_cloud* in_cloud,
                     double radius, int64_t t, npcg_neighbors* nb);
// Expand CSR rows into an explicit row-index array (u32 or i64).
void expand_rows_u32(npcg_context* ctx, const int64_t* row_ptr, int64_t n_rows, uint32_t* out);
void expand_rows_i64(npcg_context* ctx, const int64_t* row_ptr, int64_t n_rows, int64_t* out);
// Stable sort of a triplet list by one key array; writes the permuted
// (i, j, k) into the outputs.  key_range = number of distinct key values.
void sort_triplets_by(npcg_context* ctx, const uint32_t* i, const uint32_t* j, const uint32_t* k,
                      int64_t n, int axis, int64_t key_range, uint32_t* oi, uint32_t* oj,
                      uint32_t* ok);
// Build plans.
void build_tcsr(npcg_context* ctx, npcg_neighbors* nb);
void build_cells(npcg_context* ctx, npcg_neighbors* nb);
// CSR (by i) of an arbitrary triplet list, entries in stable input order; also
// verifies index bounds (IndexError).  `transpose` builds rows over j instead.
void csr_from_triplets(npcg_context* ctx, const npcg_triplets* T, bool transpose,
                       int64_t n_rows, CsrPlan* out);
void cells_from_triplets(npcg_context* ctx, const npcg_triplets* T, int64_t n_kernels,
                         CellPlan* out);
// Device-side index bound check: returns true if any v[p] >= bound.
bool any_out_of_range(npcg_context* ctx, const uint32_t* v, int64_t n, int64_t bound);

}  // namespace npcg
