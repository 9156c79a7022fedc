// conv.cuh -- engine entry points shared by the C ABI (api.cu).
#pragma once

#include "neighbors.cuh"

namespace npcg {

// ---- exact engines (conv_simt.cu) -----------------------------------------
template <typename T>
void mvmr_rows(npcg_context* ctx, const CsrView& csr, const T* w, const T* fin, int G, int cin,
               int cout, T* out, int64_t n_kernels = 0);  // n_kernels > 0: W may be staged in smem
void mvmr_rows_subset_f32(npcg_context* ctx, const CsrView& csr, const uint32_t* perm,
                          const uint32_t* list, int64_t n_list, const float* w, const float* fin,
                          int cin, int cout, float* out);
template <typename T>
void transpose_w(npcg_context* ctx, const T* w, int64_t KG, int cin, int cout, T* wt);
template <typename T>
void vvor_cells(npcg_context* ctx, const CellPlan& cells, const T* gout, const T* fin, int G,
                int cin, int cout, T* grad);

// ---- tensor-core engines (conv_tc.cu) --------------------------------------
// Operand arithmetic of the tcgen05 path: bf16 operands (opt-in, rel ~2e-3),
// or split operands (x = hi + lo, two bf16 each; products hi*hi + hi*lo + lo*hi,
// fp32 accumulate; rel ~4e-6, inside the reference's fp32 bound of 1e-5).
enum class TcMode { none = 0, bf16 = 1, split = 2 };
// True when the tcgen05 path handles this shape in `mode`: G = 1, K <= 128
// (t <= 5), C_in and C_out multiples of 16 in [64, cmax] (automatic choice) or
// [16, cmax] (forced), cmax = 256 (bf16) / 128 (split); widths are zero-padded
// to 64 / 128 / 256 inside.
bool tc_supported(int64_t G, int64_t cin, int64_t cout, int64_t n_kernels, TcMode mode,
                  bool forced);
// Forward / input-gradient / weight-gradient over a neighbor handle on the
// tensor cores.  Builds and caches the tile plans.  fin_unchanged: `fin` is
// the buffer the last forward on this handle converted, unmodified (its device
// image is reused).
void tc_forward(npcg_context* ctx, npcg_neighbors* nb, TcMode mode, const float* w,
                const float* fin, float* fout, int cin, int cout);
void tc_backward(npcg_context* ctx, npcg_neighbors* nb, TcMode mode, const float* w,
                 const float* fin, const float* gout, float* grad_in, float* grad_w, int cin,
                 int cout, bool fin_unchanged);
void tc_prepare(npcg_context* ctx, npcg_neighbors* nb, TcMode mode);
void tc_plan_stats(npcg_context* ctx, npcg_neighbors* nb, int64_t* out12);
void tc_trace_forward(npcg_context* ctx, npcg_neighbors* nb, const float* w, const float* fin,
                      float* fout, int64_t* trace_host);

}  // namespace npcg
