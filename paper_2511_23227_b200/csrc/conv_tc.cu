// conv_tc.cu -- tcgen05 / TMEM engines for the point-centric convolution
// (bf16 operands, fp32 accumulate), G = 1, C_in, C_out in {64, 128, 256},
// K = t^3 <= 32.
//
// Formulation (output-stationary cell aggregation):
//     F_out[i] = sum_k W_k^T A_k[i],   A_k[i] = sum_{j in N_k(i)} F_in[j]
// Rows are processed in spatial (Morton) order in 128-row sub-tiles grouped
// into super-tiles (2 x 128 rows when 64 channels are written, 1 x 128
// otherwise).  Per super-tile the union of all neighbor rows (the halo,
// ~2.9x the rows) is loaded into shared memory once per 64-channel chunk;
// every A_k is then aggregated from shared memory (fp32 accumulate via
// FHADD.BF16, rounded once) into a SWIZZLE_128B K-major tile and multiplied on
// the tensor core against W_k (M128 x N{64,128,256} x K16 UMMAs), which is
// loaded once per super-tile, chunk and cell.  Accumulators live in TMEM
// (double-buffered); one epilogue store per output value, no atomics.
// Dense or strided neighborhoods are re-tiled by the planner (128..8-row
// tiles, then rank-split records accumulated in TMEM; see TcDirPlan).
//
//   forward   : rows = output points, gathered features = F_in, B = W_k
//   dgrad     : rows = input points (transposed CSR), features = G_out, B = W_k^T
//   wgrad     : rows = output points, A_k^T (MN-major, two (cell, C_in chunk)
//               tiles stacked to M = 128) x dense G_out tile (MN-major) into
//               per-pair TMEM accumulators; per-CTA partials reduced in a
//               fixed order.
//
// Warp roles (fwd / dgrad kernel, 736 threads):
//   warps 0-3   epilogue (TMEM lane quadrant = warp id) + L2 halo prefetch
//   warp 4      producer: stage-descriptor bulk copies
//   warp 5      MMA issuer (one elected lane) + TMEM allocator
//   warps 6-21  aggregation (4 groups x 4 warps; quarter-warp per row)
//   warp 22     producer: W_k bulk copies
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "conv.cuh"
#include "tc_common.cuh"

namespace npcg {
using namespace tc;

constexpr int TM = 128;
constexpr int CH = 64;
constexpr int KMAX = 128;   // kernel cells (t^3 <= 125: t = 1, 3, 5)
constexpr int G_KMAX = 32;  // the gather engine's planner keeps per-cell arrays in static smem
constexpr int MAXE_ST = 16384;         // entries per super-tile the planner sorts in smem
// (128-row super-tiles: half, so more planner CTAs fit an SM)
__host__ __device__ constexpr int maxe_of(int st) { return st == 1 ? MAXE_ST / 2 : MAXE_ST; }
// A (sub-tile, cell) descriptor block: u32 item[128] | u16 entry[E].  Its
// first BLOCK_MAX_BYTES (items + up to 512 entries) are staged in a shared-
// memory slot; the entries of larger blocks are read from L2 (global).
constexpr int SLOT_ENTRIES = 512;
constexpr int BLOCK_MAX_BYTES = 512 + 2 * SLOT_ENTRIES;
constexpr int MAX_BLOCK_ENTRIES = 8192;  // planner cap per block
constexpr uint32_t kOverflow = 0xFFFFFFFFu;
constexpr bool kSplitReady = true;
// Descriptor blocks are 16-byte aligned and addressed in 16-byte units (u32:
// 64 GB of blocks per plan, ~400M points at ~160 B per point).
__host__ __device__ __forceinline__ uint64_t blk_bytes(uint32_t units) {
  return static_cast<uint64_t>(units) << 4;
}
constexpr uint32_t SUP_FIRST = 1u << 8, SUP_LAST = 1u << 9;  // record flags in sup[].y

// A direction plan: super-tiles of 1..st sub-tiles sharing one shared-memory
// halo.  Level 0 tiles the permuted rows into 128-row sub-tiles, st per
// super-tile; a super-tile beyond the capacities (halo > hcap rows, > 512
// entries in a (sub-tile, cell) block, > 254 entries of one row in one cell,
// > MAXE_ST entries) is re-planned at the next level as single sub-tiles of
// half as many rows (128, 64, ..., 8), so dense or strided neighborhoods stay
// on the tensor cores with partially filled tiles; only rows that fail at
// 8-row tiles go to the exact engine.  Failed super-tiles stay in the arrays
// with halo_len = kOverflow (skipped by the kernels).
struct TcDirPlan {
  int st = 3;
  int hcap = 1280;
  int64_t n_rows = 0, n_cols = 0;
  int n_sub = 0, n_super = 0, K = 0;  // n_sub = sub-tiles over all levels
  int levels = 0;
  bool big_blocks = false;    // some descriptor block exceeds its shared-memory slot
  DevBuf<uint2> sup;          // n_super records {first sub-tile, sub-tiles | SUP_FIRST | SUP_LAST}
  DevBuf<uint32_t> item_start;  // n_items + 1 (records of an item share rows, accumulate)
  int n_items = 0;
  DevBuf<uint2> tiles;        // n_sub {first permuted row, rows (<= 128)}
  DevBuf<uint32_t> halo;      // n_super * hcap permuted source row of each halo row
  DevBuf<uint32_t> halo_len;  // n_super (kOverflow marks a super-tile the planner rejected)
  DevBuf<uint32_t> blk_off;   // n_sub*K (+1) offsets of the stage-descriptor blocks, in 16-byte units
  DevBuf<uint8_t> blocks;
  int n_overflow = 0;
  int max_halo = 0;
  double mean_halo = 0.0;
  DevBuf<uint32_t> spill_rows;  // permuted positions of rows in overflow super-tiles
  int64_t n_spill = 0;
  std::vector<unsigned long long> k_count;  // entries per kernel cell (host)
};

struct GatherPlan;
struct GatherPlanDeleter {
  void operator()(GatherPlan* p) const;
};
struct TcPlan {
  std::unique_ptr<TcDirPlan> fwd, bwd;  // wgrad reuses the forward plan
  std::unique_ptr<TcDirPlan> fwd1, bwd1;  // 128-row super-tiles for wide (C > 64) passes
  std::unique_ptr<GatherPlan, GatherPlanDeleter> gfwd, gbwd;  // gather-engine plans
  DevBuf<uint32_t> inv_perm_out, inv_perm_in;
  DevBuf<__nv_bfloat16> feat_in;   // bf16 F_in in perm_in order
  const void* saved_fin = nullptr;  // fin whose image feat_in holds (set by the forward)
  int saved_c = 0;                  // and its channel count
  bool saved_split = false;         // and its kind (bf16 image or split image)
  DevBuf<uint32_t> amax;            // split path: max |x| bits of [F_in, W, G_out, W] (scales)
  DevBuf<uint32_t> bf_flags;        // fused backward: per (item, quadrant) "half 0 stored" flags
  uint32_t bf_gen = 0;              // and the value of the last launch
  DevBuf<__nv_bfloat16> feat_out;  // bf16 G_out in perm_out order
  DevBuf<uint8_t> wpack;           // K x nci images of C x 128 B, SW128 K-major B operand
  DevBuf<float> partial;           // wgrad per-CTA partials
};

void destroy_tc_plan(TcPlan* p);

// Channel widths run on the tensor cores padded to 64 / 128 / 256 (zero
// channels in the bf16 images and packed weights; outputs written unpadded).
// The automatic choice keeps narrow layers (C < 64, where the contraction is
// not dense enough to pay for the padding) on the CUDA-core engines;
// math = bf16 forces the tensor cores for any multiple of 16 up to 256.
static bool tc_width(int64_t c, int64_t cmax, bool forced) {
  return c >= (forced ? 16 : 64) && c <= cmax && c % 16 == 0;
}
static int tc_pad(int c) { return c <= 64 ? 64 : c <= 128 ? 128 : 256; }
bool tc_supported(int64_t G, int64_t cin, int64_t cout, int64_t K, TcMode mode, bool forced) {
  if (mode == TcMode::none) return false;
  if (mode == TcMode::split && !kSplitReady) return false;
  const int64_t cmax = 256;  // (split: passes wider than 128 run in 128-column halves)
  return G == 1 && tc_width(cin, cmax, forced) && tc_width(cout, cmax, forced) && K >= 1 &&
         K <= KMAX;
}

// ===========================================================================
// planner
// ===========================================================================
__global__ void k_inverse_perm(const uint32_t* __restrict__ perm, int64_t n,
                               uint32_t* __restrict__ inv) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n) inv[perm[p]] = static_cast<uint32_t>(p);
}

__host__ __device__ __forceinline__ uint32_t item_encode(uint32_t r, uint32_t count, uint32_t eo) {
  return (8u * r + (r & 7u)) | (count << 10) | (eo << 18);
}
__device__ __forceinline__ uint32_t item_count(uint32_t it) { return (it >> 10) & 255u; }
__device__ __forceinline__ uint32_t item_eo(uint32_t it) { return it >> 18; }
// byte offset of the item's row, 16-byte chunk `l8x16` (= (lane & 7) << 4), in
// a SWIZZLE_128B K-major tile
__device__ __forceinline__ uint32_t item_sw128(uint32_t it, uint32_t l8x16) {
  return ((it << 4) & 0x3FF0u) ^ l8x16;
}

// Position of the p-th item (count-sorted order) in the block: quad q = p / 4
// goes to aggregation warp q % 4 as its quad q / 4; a warp's items are stored
// [sub-row][quad], so a lane's eight items are 32 contiguous bytes and the
// quads' first items (their largest counts) are the warp's first eight.
__host__ __device__ __forceinline__ int item_slot(int p) {
  return ((p >> 2) & 3) * 32 + (p & 3) * 8 + (p >> 4);
}

// Entry filter of a plan record: only the entries whose permuted column lies
// in [clo, chi) (a halo segment) and, among those, whose rank (order among
// the row's entries of that cell, CSR order) lies in [rlo, rhi).  Records
// that split one tile's entries this way form an item; the kernels
// accumulate its records in TMEM.
constexpr int MAXSEG = 16;  // halo segments per record at most
struct EntryFilter {
  uint32_t rlo, rhi, clo, chi;
  __host__ __device__ static EntryFilter from(uint4 v) { return {v.x, v.y, v.z, v.w}; }
  __device__ __forceinline__ bool all() const {
    return rlo == 0 && rhi == 0xFFFFFFFFu && clo == 0 && chi == 0xFFFFFFFFu;
  }
};
__host__ __device__ inline uint4 no_filter() { return make_uint4(0, 0xFFFFFFFFu, 0, 0xFFFFFFFFu); }

// Per sub-tile: entries per (sub-tile, cell) block -> block byte sizes; flags
// sub-tiles whose blocks exceed the stage-descriptor slot or whose per-(row,
// cell) counts exceed the 8-bit item field; reports the largest per-(row,
// cell) count (unfiltered), which sizes rank-split records.
__global__ void __launch_bounds__(TM) k_plan_counts(const int64_t* __restrict__ row_ptr,
                                                    const uint32_t* __restrict__ kk,
                                                    const uint32_t* __restrict__ col,
                                                    const uint32_t* __restrict__ inv_perm_cols,
                                                    const uint32_t* __restrict__ perm_rows,
                                                    const uint2* __restrict__ tiles,
                                                    const uint4* __restrict__ tfilter, int K,
                                                    uint32_t* __restrict__ blk_size,
                                                    uint32_t* __restrict__ sub_bad,
                                                    uint32_t* __restrict__ tile_maxc,
                                                    uint32_t* __restrict__ max_blk) {
  __shared__ uint32_t cnt[KMAX];
  extern __shared__ uint16_t pc_dyn[];  // rc[TM][K]: all entries per (row, cell); inc[TM][K]: filtered
  uint16_t* rc = pc_dyn;
  uint16_t* inc = pc_dyn + TM * K;
  __shared__ int bad;
  __shared__ uint32_t s_maxc;
  const int r = threadIdx.x;
  if (r < KMAX) cnt[r] = 0;
  if (r == 0) {
    bad = 0;
    s_maxc = 0;
  }
  for (int k = 0; k < K; ++k) rc[r * K + k] = inc[r * K + k] = 0;
  __syncthreads();
  const uint2 tl = tiles[blockIdx.x];
  const EntryFilter f = EntryFilter::from(tfilter[blockIdx.x]);
  const bool colf = !(f.clo == 0 && f.chi == 0xFFFFFFFFu);
  if (f.all()) {
    // no filter: every entry counts; a warp walks a row's entries in parallel
    // (the row / cell counts are u16 pairs updated with 32-bit atomics)
    const int lane = r & 31, warp = r >> 5;
    for (int rr = warp; rr < static_cast<int>(tl.y); rr += TM / 32) {
      const uint32_t i = perm_rows[tl.x + rr];
      const int64_t e0 = row_ptr[i], e1 = row_ptr[i + 1];
      for (int64_t e = e0 + lane; e < e1; e += 32) {
        const uint32_t k = kk[e];
        const int idx = rr * K + static_cast<int>(k);
        atomicAdd(reinterpret_cast<unsigned*>(rc) + (idx >> 1), 1u << (16 * (idx & 1)));
        atomicAdd(&cnt[k], 1u);
      }
    }
    __syncthreads();
    for (int k = 0; k < K; ++k) inc[r * K + k] = rc[r * K + k];
  } else if (static_cast<uint32_t>(r) < tl.y) {
    const uint32_t i = perm_rows[tl.x + r];
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      if (colf) {
        const uint32_t pj = inv_perm_cols[col[e]];
        if (pj < f.clo || pj >= f.chi) continue;
      }
      const uint32_t k = kk[e];
      const uint32_t rank = rc[r * K + k];
      if (rank < 0xFFFFu) rc[r * K + k] = static_cast<uint16_t>(rank + 1);
      if (rank >= f.rlo && rank < f.rhi) {
        atomicAdd(&cnt[k], 1u);
        inc[r * K + k]++;
      }
    }
  }
  uint32_t mx = 0;
  for (int k = 0; k < K; ++k) {
    if (inc[r * K + k] > 254) bad = 1;
    mx = max(mx, static_cast<uint32_t>(rc[r * K + k]));
  }
  atomicMax(&s_maxc, mx);
  __syncthreads();
  if (r < K) {  // K <= KMAX = TM
    const uint32_t E = cnt[r];
    if (E > MAX_BLOCK_ENTRIES) bad = 1;
    const uint32_t bytes = 512u + ((2u * E + 15u) / 16u) * 16u;
    blk_size[static_cast<int64_t>(blockIdx.x) * K + r] = bytes >> 4;
    atomicMax(max_blk, bytes);
  }
  __syncthreads();
  if (r == 0) {
    sub_bad[blockIdx.x] = bad;
    tile_maxc[blockIdx.x] = s_maxc;
  }
}

// Entries of one row passing a filter, in CSR order: fn(e, k).
template <typename F>
__device__ __forceinline__ void for_row_entries(const int64_t* row_ptr, const uint32_t* kk,
                                                const uint32_t* col, const uint32_t* inv_perm_cols,
                                                uint32_t row, const EntryFilter& f, F&& fn) {
  const int64_t e0 = row_ptr[row], e1 = row_ptr[row + 1];
  if (f.all()) {
    for (int64_t e = e0; e < e1; ++e) fn(e, static_cast<int>(kk[e]));
    return;
  }
  const bool colf = !(f.clo == 0 && f.chi == 0xFFFFFFFFu);
  uint16_t seen[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) seen[k] = 0;
  for (int64_t e = e0; e < e1; ++e) {
    if (colf) {
      const uint32_t pj = inv_perm_cols[col[e]];
      if (pj < f.clo || pj >= f.chi) continue;
    }
    const int k = static_cast<int>(kk[e]);
    const uint32_t rank = seen[k]++;
    if (rank >= f.rlo && rank < f.rhi) fn(e, k);
  }
}

// Lockstep branchless searches for U keys at once (the same trip count for
// every key, so their shared-memory loads are in flight together): the last
// index i in [0, n) with a[i] <= key[u] (a sorted ascending, a[0] <= key).
template <int U, typename T, typename K>
__device__ __forceinline__ void last_le(const T* a, int n, const K (&key)[U], int (&out)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) out[u] = 0;
  while (n > 1) {
    const int half = n >> 1;
#pragma unroll
    for (int u = 0; u < U; ++u) out[u] = static_cast<K>(a[out[u] + half]) <= key[u] ? out[u] + half : out[u];
    n -= half;
  }
}

// Per super-tile: halo (sorted unique permuted neighbor rows), per-(sub-tile,
// cell) item lists (rows ordered by entry count, descending) and u16 halo
// indices of the entries.  Block layout: u32 item[128] | u16 entry[E] (pad 16 B)
//   item = rs | count << 10 | x << 18   (count <= 254, x < 16384): x is the
//   entry offset, or, in a quad whose rows have at most one entry, the row's
//   one entry itself (its halo index)
//   rs = 8 r + (r & 7): rs << 4 is row r's byte offset in a SWIZZLE_128B tile
//   before the lane's 16-byte chunk is XOR-ed in
__global__ void __launch_bounds__(512) k_plan_super(
    const int64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
    const uint32_t* __restrict__ kk, const uint32_t* __restrict__ perm_rows,
    const uint32_t* __restrict__ inv_perm_cols, const uint2* __restrict__ sup,
    const uint2* __restrict__ tiles, const uint4* __restrict__ tfilter, int K, int st, int hcap,
    const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ sub_bad,
    uint32_t* __restrict__ halo_out,
    uint32_t* __restrict__ halo_len, uint32_t* __restrict__ seg,
    uint8_t* __restrict__ blocks, int packed, unsigned long long* __restrict__ pdbg) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int maxe = maxe_of(st);
  uint32_t* buf = reinterpret_cast<uint32_t*>(sm);                          // maxe
  uint16_t* cnt = reinterpret_cast<uint16_t*>(buf + maxe);                  // st*K*TM
  uint16_t* eoff = cnt + st * K * TM;                                        // st*K*TM
  int* rowoff = reinterpret_cast<int*>(eoff + st * K * TM);                  // st*TM + 1
  __shared__ int s_total, s_bad, s_H;
  // packed (plain records, column ids < 2^25): phase 2 keeps each entry as
  // (permuted column << 7 | cell) in buf, phase 6 reads them back from there
  // (no second pass over global memory); the halo goes to hal[]
  __shared__ int64_t rowe0[512];
  __shared__ uint32_t hal[1024];
  __shared__ uint64_t s_boff[2 * KMAX];
  __shared__ int wsum[16];

  const int s = blockIdx.x;
  if (pdbg && threadIdx.x == 0) pdbg[s * 8 + 6] = clock64();
  const int sub0 = static_cast<int>(sup[s].x);
  const int nsub = static_cast<int>(sup[s].y & 0xFFu);
  const int R = nsub * TM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_bad = 0;
    for (int g = 0; g < nsub; ++g) s_bad |= sub_bad[sub0 + g];
  }
  for (int x = tid; x < st * K * TM; x += blockDim.x) cnt[x] = 0;
  __syncthreads();
  if (s_bad) {
    if (tid == 0) {
      halo_len[s] = kOverflow;
      seg[static_cast<int64_t>(s) * (MAXSEG + 1)] = 0;
    }
    return;
  }
  // 1. row lengths -> offsets (block scan over R <= 512 rows)
  int len = 0;
  uint32_t row_i = 0;
  EntryFilter filt = EntryFilter::from(no_filter());
  if (tid < R) {
    const uint2 tl = tiles[sub0 + tid / TM];
    filt = EntryFilter::from(tfilter[sub0 + tid / TM]);
    if (static_cast<uint32_t>(tid % TM) < tl.y) {
      row_i = perm_rows[tl.x + tid % TM];
      rowe0[tid] = row_ptr[row_i];
      if (filt.all()) len = static_cast<int>(row_ptr[row_i + 1] - rowe0[tid]);
      else for_row_entries(row_ptr, kk, col, inv_perm_cols, row_i, filt, [&](int64_t, int) { ++len; });
    }
  }
  int incl = len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < 16; ++w) {
      const int v = wsum[w];
      wsum[w] = acc;
      acc += v;
    }
    s_total = acc;
  }
  __syncthreads();
  const int my_off = incl - len + wsum[warp];
  if (tid < R) rowoff[tid] = my_off;
  if (tid == 0) rowoff[R] = s_total;
  const int E = s_total;
  // records without entry filters (all but the rank / halo-segment splits):
  // the per-entry passes run warp-cooperatively, a row's entries in parallel
  __shared__ int s_plain;
  if (tid == 0) {
    int pl = 1;
    for (int g = 0; g < nsub; ++g) pl &= EntryFilter::from(tfilter[sub0 + g]).all() ? 1 : 0;
    s_plain = pl;
  }
  const int nwarps = static_cast<int>(blockDim.x) >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  if (E > maxe) {
    if (tid == 0) {
      halo_len[s] = kOverflow;
      seg[static_cast<int64_t>(s) * (MAXSEG + 1)] = 0;
    }
    return;
  }
  if (pdbg && tid == 0) pdbg[s * 8 + 0] = clock64();  // (planner profile: phase clocks)
  // 2. permuted neighbor ids + per-(sub, cell, row) counts
  __syncthreads();
  const bool plain = s_plain != 0;
  const bool pk = plain && packed != 0;
  if (pk) {
    // flattened over the super-tile's entries, four per thread in flight
    // warp-contiguous chunks of 32 entries (coalesced CSR reads), four chunks
    // per warp in flight; a lane's row from its chunk's first row (searched in
    // lockstep) and a short forward step
    for (int cb0 = 32 * warp; cb0 < E; cb0 += 4 * 32 * nwarps) {
      int cbs[4], r0[4], rr[4];
      int64_t e[4];
      uint32_t c[4], k[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) cbs[u] = min(cb0 + u * 32 * nwarps, E - 1);
      last_le<4>(rowoff, R, cbs, r0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = cb0 + u * 32 * nwarps + lane;
        rr[u] = r0[u];
        e[u] = -1;
        if (x < E) {
          while (rowoff[rr[u] + 1] <= x) ++rr[u];
          e[u] = rowe0[rr[u]] + (x - rowoff[rr[u]]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (e[u] >= 0) {
          c[u] = col[e[u]];
          k[u] = kk[e[u]];
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (e[u] >= 0) c[u] = inv_perm_cols[c[u]];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (e[u] >= 0) {
          const int g = rr[u] / TM, r = rr[u] % TM;
          buf[cb0 + u * 32 * nwarps + lane] = (c[u] << 7) | k[u];
          const int idx = (g * K + static_cast<int>(k[u])) * TM + r;
          atomicAdd(reinterpret_cast<unsigned*>(cnt) + (idx >> 1), 1u << (16 * (idx & 1)));
        }
    }
  } else if (plain) {
    for (int rr = warp; rr < R; rr += nwarps) {
      const int g = rr / TM, r = rr % TM;
      const int off = rowoff[rr], n = rowoff[rr + 1] - off;
      if (n == 0) continue;
      const int64_t e0 = row_ptr[perm_rows[tiles[sub0 + g].x + r]];
      for (int b = lane; b < n; b += 32) {
        const int64_t e = e0 + b;
        const int idx = (g * K + static_cast<int>(kk[e])) * TM + r;
        buf[off + b] = inv_perm_cols[col[e]];
        atomicAdd(reinterpret_cast<unsigned*>(cnt) + (idx >> 1), 1u << (16 * (idx & 1)));
      }
    }
  } else if (tid < R && len > 0) {
    const int g = tid / TM, r = tid % TM;
    int q = 0;
    for_row_entries(row_ptr, kk, col, inv_perm_cols, row_i, filt, [&](int64_t e, int k) {
      buf[my_off + q++] = inv_perm_cols[col[e]];
      cnt[(g * K + k) * TM + r]++;
    });
  }
  __syncthreads();
  // bitonic sort of buf[0, P) (P a power of two, padded with 0xFFFFFFFF)
  auto bitonic = [&](uint32_t* v, int P) {
    for (int size = 2; size <= P; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int x = tid; x < (P >> 1); x += blockDim.x) {
          const int lo = ((x & ~(stride - 1)) << 1) | (x & (stride - 1));  // (stride: a power of two)
          const int hi = lo + stride;
          const bool up = (lo & size) == 0;
          const uint32_t a = v[lo], b = v[hi];
          if ((a > b) == up) {
            v[lo] = b;
            v[hi] = a;
          }
        }
        __syncthreads();
      }
    }
  };
  if (pdbg && tid == 0) pdbg[s * 8 + 1] = clock64();
  // 3. the distinct rows, sorted, into buf[0, H).  Fast path: a shared hash
  //    set of the entries' rows; when at most HS_MAX rows are distinct (every
  //    super-tile whose halo can fit), only those are sorted.  Otherwise all
  //    entries are sorted and compacted.
  constexpr int HS_SIZE = 2048, HS_MAX = 1024;  // (inserts stop past HS_MAX: <= 1536 used)
  __shared__ uint32_t hset[HS_SIZE];
  __shared__ int s_n, s_c;
  for (int x = tid; x < HS_SIZE; x += blockDim.x) hset[x] = 0xFFFFFFFFu;
  if (tid == 0) s_n = s_c = 0;
  __syncthreads();
  for (int x = tid; x < E; x += blockDim.x) {
    if (*reinterpret_cast<volatile int*>(&s_n) > HS_MAX) break;
    const uint32_t v = pk ? buf[x] >> 7 : buf[x];
    uint32_t h = (v * 2654435761u) >> 21;
    while (true) {
      const uint32_t old = atomicCAS(&hset[h], 0xFFFFFFFFu, v);
      if (old == 0xFFFFFFFFu) {
        atomicAdd(&s_n, 1);
        break;
      }
      if (old == v) break;
      h = (h + 1) & (HS_SIZE - 1);
    }
  }
  __syncthreads();
  // the halo (sorted distinct rows): hal[] on the hash path (buf keeps the
  // entries), buf itself on the full-sort path (whose halo never fits)
  uint32_t* halo = buf;
  if (s_n <= HS_MAX) {
    halo = hal;
    for (int x = tid; x < HS_SIZE; x += blockDim.x) {
      const uint32_t v = hset[x];
      if (v != 0xFFFFFFFFu) hal[atomicAdd(&s_c, 1)] = v;
    }
    __syncthreads();
    const int Hn = s_n;
    int P = 1;
    while (P < Hn) P <<= 1;
    for (int x = Hn + tid; x < P; x += blockDim.x) hal[x] = 0xFFFFFFFFu;
    __syncthreads();
    bitonic(hal, P);
    if (tid == 0) s_H = Hn;
    __syncthreads();
  } else {
    if (pk) {
      for (int x = tid; x < E; x += blockDim.x) buf[x] >>= 7;
      __syncthreads();
    }
    int P = 1;
    while (P < E) P <<= 1;
    for (int x = E + tid; x < P; x += blockDim.x) buf[x] = 0xFFFFFFFFu;
    __syncthreads();
    bitonic(buf, P);
    // unique (compaction in place, chunked per thread)
    const int per = (P + blockDim.x - 1) / blockDim.x;
    const int c0 = tid * per, c1 = min(P, c0 + per);
    int local = 0;
    for (int x = c0; x < c1; ++x) {
      const uint32_t v = buf[x];
      if (v != 0xFFFFFFFFu && (x == 0 || buf[x - 1] != v)) ++local;
    }
    int li = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, li, o);
      if (lane >= o) li += n;
    }
    __syncthreads();
    if (lane == 31) wsum[warp] = li;
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int w = 0; w < 16; ++w) {
        const int v = wsum[w];
        wsum[w] = acc;
        acc += v;
      }
      s_H = acc;
    }
    __syncthreads();
    // gather my unique values into registers-by-chunk, then write compacted
    int w0 = li - local + wsum[warp];
    uint32_t vals[32];
    int nv = 0;
    for (int x = c0; x < c1 && nv < 32; ++x) {
      const uint32_t v = buf[x];
      if (v != 0xFFFFFFFFu && (x == 0 || buf[x - 1] != v)) vals[nv++] = v;
    }
    __syncthreads();
    for (int q = 0; q < nv; ++q) buf[w0 + q] = vals[q];
    __syncthreads();
  }
  const int H = s_H;
  const bool over = H > hcap;
  if (!over)
    for (int x = tid; x < H; x += blockDim.x) halo_out[static_cast<int64_t>(s) * hcap + x] = halo[x];
  __syncthreads();
  if (over) {
    // beyond the halo cap: report the split of the halo into <= hcap-row
    // segments (column ranges) so the host can plan the rows as one item of
    // segment records instead of smaller tiles
    if (tid == 0) {
      halo_len[s] = kOverflow;
      const int nseg = (H + hcap - 1) / hcap;
      uint32_t* sg = seg + static_cast<int64_t>(s) * (MAXSEG + 1);
      sg[0] = nseg <= MAXSEG ? static_cast<uint32_t>(nseg) : 0u;
      if (nseg <= MAXSEG)
        for (int q = 1; q < nseg; ++q) sg[q] = halo[static_cast<int64_t>(q) * H / nseg];
    }
    return;
  }
  if (pdbg && tid == 0) pdbg[s * 8 + 2] = clock64();
  // 5. items per (sub, cell) block: rows by count descending (stable in r)
  const unsigned lt = (1u << lane) - 1u;
  for (int b = warp; b < nsub * K; b += blockDim.x / 32) {
    const int g = b / K, k = b % K;
    const uint64_t boff = blk_bytes(blk_off[static_cast<int64_t>(sub0 + g) * K + k]);
    uint32_t* items = reinterpret_cast<uint32_t*>(blocks + boff);
    int pos = 0, ebase = 0;
    int vmax = 0;
    for (int ch = 0; ch < TM / 32; ++ch) vmax = max(vmax, static_cast<int>(cnt[(g * K + k) * TM + ch * 32 + lane]));
    vmax = __reduce_max_sync(0xffffffffu, vmax);
    for (int v = vmax; v >= 0; --v) {
      for (int ch = 0; ch < TM / 32; ++ch) {
        const int r = ch * 32 + lane;
        const int c = cnt[(g * K + k) * TM + r];
        const unsigned m = __ballot_sync(0xffffffffu, c == v);
        if (c == v) {
          const int before = __popc(m & lt);
          const int eo = ebase + v * before;
          items[item_slot(pos + before)] = item_encode(static_cast<uint32_t>(r),
                                                       static_cast<uint32_t>(c),
                                                       static_cast<uint32_t>(eo));
          eoff[(g * K + k) * TM + r] = static_cast<uint16_t>(eo);
        }
        pos += __popc(m);
        ebase += v * __popc(m);
      }
    }
  }
  __syncthreads();
  for (int x = tid; x < st * K * TM; x += blockDim.x) cnt[x] = 0;
  for (int x = tid; x < nsub * K; x += blockDim.x)
    s_boff[x] = blk_bytes(blk_off[static_cast<int64_t>(sub0 + x / K) * K + x % K]);
  __syncthreads();
  if (pdbg && tid == 0) pdbg[s * 8 + 3] = clock64();
  // 6. entries: halo index of each neighbor, written at its item's offset
  //    (in CSR order within each (row, cell))
  if (pk) {
    // warp-contiguous chunks of 32 entries (all reads from shared memory, two
    // chunks per warp with their searches in lockstep): the rank of an entry
    // within its (row, cell) -- CSR order -- is its rank among the chunk's
    // entries of the same (row, cell) plus the row's entries of that cell
    // before the chunk
    for (int cb0 = 32 * warp; cb0 < E; cb0 += 2 * 32 * nwarps) {
      int cbs[2], r0[2], rr[2], hx[2];
      uint32_t v[2], pj[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) cbs[u] = min(cb0 + u * 32 * nwarps, E - 1);
      last_le<2>(rowoff, R, cbs, r0);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int x = min(cb0 + u * 32 * nwarps + lane, E - 1);
        rr[u] = r0[u];
        while (rowoff[rr[u] + 1] <= x) ++rr[u];
        v[u] = buf[x];
        pj[u] = v[u] >> 7;
      }
      last_le<2>(hal, H, pj, hx);  // the entries' halo indices (their rows are in the halo)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int cb = cb0 + u * 32 * nwarps, x = cb + lane;
        const bool act = x < E;
        const uint32_t k = v[u] & 127u;
        const unsigned same = __match_any_sync(0xffffffffu, act ? static_cast<int>(rr[u] * 128 + k) : -1);
        if (!act) continue;
        int rank = __popc(same & lt_mask);
        for (int y = rowoff[rr[u]]; y < cb; ++y) rank += (buf[y] & 127u) == k;
        const int g = rr[u] / TM, r = rr[u] % TM;
        const int idx = (g * K + static_cast<int>(k)) * TM + r;
        reinterpret_cast<uint16_t*>(blocks + s_boff[g * K + k] + 512)[eoff[idx] + rank] =
            static_cast<uint16_t>(hx[u]);
      }
    }
  } else if (plain) {
    for (int rr = warp; rr < R; rr += nwarps) {
      const int g = rr / TM, r = rr % TM;
      const int n = rowoff[rr + 1] - rowoff[rr];
      if (n == 0) continue;
      const int64_t e0 = row_ptr[perm_rows[tiles[sub0 + g].x + r]];
      for (int b = 0; b < n; b += 32) {
        const bool act = b + lane < n;
        int k = -1, lo = 0;
        if (act) {
          const int64_t e = e0 + b + lane;
          k = static_cast<int>(kk[e]);
          const uint32_t pj = inv_perm_cols[col[e]];
          int hi = H;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (halo[mid] < pj) lo = mid + 1;
            else hi = mid;
          }
        }
        const unsigned same = __match_any_sync(0xffffffffu, k);
        const int rank = __popc(same & lt_mask);
        const int idx = (g * K + (act ? k : 0)) * TM + r;
        if (act) {
          const int pos = eoff[idx] + cnt[idx] + rank;
          const uint64_t boff = blk_bytes(blk_off[static_cast<int64_t>(sub0 + g) * K + k]);
          reinterpret_cast<uint16_t*>(blocks + boff + 512)[pos] = static_cast<uint16_t>(lo);
        }
        __syncwarp();
        if (act && rank == __popc(same) - 1) cnt[idx] = static_cast<uint16_t>(cnt[idx] + __popc(same));
        __syncwarp();
      }
    }
  } else if (tid < R && len > 0) {
    const int g = tid / TM, r = tid % TM;
    for_row_entries(row_ptr, kk, col, inv_perm_cols, row_i, filt, [&](int64_t e, int k) {
      const uint32_t pj = inv_perm_cols[col[e]];
      int lo = 0, hi = H;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (halo[mid] < pj) lo = mid + 1;
        else hi = mid;
      }
      const int idx = (g * K + k) * TM + r;
      const int pos = eoff[idx] + cnt[idx]++;
      const uint64_t boff = blk_bytes(blk_off[static_cast<int64_t>(sub0 + g) * K + k]);
      reinterpret_cast<uint16_t*>(blocks + boff + 512)[pos] = static_cast<uint16_t>(lo);
    });
  }
  __syncthreads();
  if (pdbg && tid == 0) pdbg[s * 8 + 4] = clock64();
  // 7. in quads whose rows have at most one entry (the copy pass), a row's
  //    item carries its entry's halo index instead of the entry offset
  for (int b = warp; b < nsub * K; b += blockDim.x / 32) {
    const uint64_t boff = blk_bytes(blk_off[static_cast<int64_t>(sub0 + b / K) * K + b % K]);
    uint32_t* items = reinterpret_cast<uint32_t*>(blocks + boff);
    const uint16_t* ents = reinterpret_cast<const uint16_t*>(blocks + boff + 512);
    for (int p = lane; p < TM; p += 32) {
      const uint32_t first = items[item_slot(p & ~3)];  // the quad's largest count
      const uint32_t it = items[item_slot(p)];
      if (((first >> 10) & 255u) <= 1u && ((it >> 10) & 255u) == 1u)
        items[item_slot(p)] = (it & 0x3FFFFu) | (static_cast<uint32_t>(ents[it >> 18]) << 18);
    }
  }
  if (tid == 0) halo_len[s] = static_cast<uint32_t>(H);
  if (pdbg) {
    __syncthreads();
    if (tid == 0) pdbg[s * 8 + 5] = clock64();
  }
}

__global__ void k_add_u32(uint32_t* __restrict__ p, int64_t n, uint32_t add) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x < n) p[x] += add;
}

// One planning level over a host list of super-tiles (tiles in level-local
// numbering).  Results stay in the level's own buffers until concatenation.
struct PlanLevel {
  int kind = 0;                 // 0 plain super-tiles, 1 rank-split items, 2 halo-segment items
  std::vector<uint2> sup, tiles;
  std::vector<uint4> tfilter;   // per tile entry filter {rank lo, hi, column lo, hi}
  std::vector<uint32_t> nom;    // per tile nominal rows (128, 64, ..., 8)
  std::vector<uint32_t> maxc;   // per tile largest (row, cell) entry count
  std::vector<uint32_t> seg;    // per record: halo segments and their column boundaries
  DevBuf<uint32_t> halo, halo_len, blk_off;
  DevBuf<uint8_t> blocks;
  uint32_t block_units = 0;     // descriptor blocks, 16-byte units
  uint32_t max_blk = 0;      // largest descriptor block (bytes)
  std::vector<uint32_t> hl;  // halo_len on the host
};

static void plan_level(npcg_context* ctx, PlanLevel& L, const int64_t* row_ptr, const uint32_t* col,
                       const uint32_t* kk, const uint32_t* perm_rows, const uint32_t* inv_perm_cols,
                       int K, int st, int hcap, bool packed) {
  const int ns = static_cast<int>(L.sup.size()), nt = static_cast<int>(L.tiles.size());
  static const bool hprof = std::getenv("NPCG_PLAN_PROFILE") != nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  auto hms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count(); };
  double tm[6] = {0, 0, 0, 0, 0, 0};
  if (L.tfilter.empty()) L.tfilter.assign(nt, no_filter());
  DevBuf<uint2> d_sup(ctx, ns), d_tiles(ctx, nt);
  DevBuf<uint4> d_filt(ctx, nt);
  DevBuf<uint32_t> d_seg(ctx, static_cast<int64_t>(ns) * (MAXSEG + 1));
  DevBuf<uint32_t> d_maxc(ctx, nt), d_maxblk(ctx, 1);
  NPCG_CUDA(cudaMemsetAsync(d_maxblk.get(), 0, 4, ctx->stream));
  // (records write only their used segment bounds; the whole array is read back)
  NPCG_CUDA(cudaMemsetAsync(d_seg.get(), 0, static_cast<size_t>(ns) * (MAXSEG + 1) * 4, ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(d_sup.get(), L.sup.data(), ns * sizeof(uint2), cudaMemcpyHostToDevice,
                            ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(d_tiles.get(), L.tiles.data(), nt * sizeof(uint2),
                            cudaMemcpyHostToDevice, ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(d_filt.get(), L.tfilter.data(), nt * sizeof(uint4),
                            cudaMemcpyHostToDevice, ctx->stream));
  const int64_t nblk = static_cast<int64_t>(nt) * K;
  DevBuf<uint32_t> blk_size(ctx, nblk + 1), sub_bad(ctx, nt);
  NPCG_CUDA(cudaMemsetAsync(blk_size.get() + nblk, 0, 4, ctx->stream));
  const size_t pc_smem = 2u * TM * static_cast<size_t>(K) * sizeof(uint16_t);
  NPCG_CUDA(cudaFuncSetAttribute(k_plan_counts, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(pc_smem)));
  launch(ctx, "plan_counts", k_plan_counts, dim3(nt), dim3(TM), pc_smem, row_ptr, kk, col, inv_perm_cols,
         perm_rows, static_cast<const uint2*>(d_tiles.get()), static_cast<const uint4*>(d_filt.get()), K,
         blk_size.get(), sub_bad.get(), d_maxc.get(), d_maxblk.get());
  L.blk_off.alloc(ctx, nblk + 1);
  if (hprof) tm[0] = hms();
  exclusive_scan_u32(ctx, blk_size.get(), L.blk_off.get(), nblk + 1, &L.block_units);
  if (hprof) tm[1] = hms();
  L.blocks.alloc(ctx, static_cast<int64_t>(blk_bytes(L.block_units)));
  L.halo.alloc(ctx, static_cast<int64_t>(ns) * hcap);
  L.halo_len.alloc(ctx, ns);
  const size_t smem = maxe_of(st) * 4 + 2 * static_cast<size_t>(st) * K * TM * 2 + (st * TM + 1) * 4;
  // NPCG_PLAN_PROFILE=1: per-phase clocks of k_plan_super (stderr, mean over records)
  static const bool prof = std::getenv("NPCG_PLAN_PROFILE") != nullptr;
  DevBuf<unsigned long long> pdbg;
  if (prof) {
    pdbg.alloc(ctx, static_cast<int64_t>(ns) * 8);
    NPCG_CUDA(cudaMemsetAsync(pdbg.get(), 0, static_cast<size_t>(ns) * 64, ctx->stream));
  }
  NPCG_CUDA(cudaFuncSetAttribute(k_plan_super, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  if (hprof) tm[2] = hms();
  launch(ctx, "plan_super", k_plan_super, dim3(ns), dim3(512), smem, row_ptr, col, kk, perm_rows,
         inv_perm_cols, static_cast<const uint2*>(d_sup.get()),
         static_cast<const uint2*>(d_tiles.get()), static_cast<const uint4*>(d_filt.get()), K, st,
         hcap,
         static_cast<const uint32_t*>(L.blk_off.get()), static_cast<const uint32_t*>(sub_bad.get()),
         L.halo.get(), L.halo_len.get(), d_seg.get(), L.blocks.get(), packed ? 1 : 0, pdbg.get());
  L.hl.resize(ns);
  L.maxc.resize(nt);
  NPCG_CUDA(cudaMemcpyAsync(L.hl.data(), L.halo_len.get(), ns * 4, cudaMemcpyDeviceToHost,
                            ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(L.maxc.data(), d_maxc.get(), nt * 4, cudaMemcpyDeviceToHost,
                            ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(&L.max_blk, d_maxblk.get(), 4, cudaMemcpyDeviceToHost, ctx->stream));
  L.seg.resize(static_cast<size_t>(ns) * (MAXSEG + 1));
  NPCG_CUDA(cudaMemcpyAsync(L.seg.data(), d_seg.get(), L.seg.size() * 4, cudaMemcpyDeviceToHost,
                            ctx->stream));
  if (hprof) tm[3] = hms();
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hprof)
    std::fprintf(stderr, "[npcg plan host] level: counts issued %.3f, scan synced %.3f, super issued %.3f, "
                 "readback issued %.3f, synced %.3f ms\n", tm[0], tm[1], tm[2], tm[3], hms());
  if (prof && ns) {
    std::vector<unsigned long long> h(static_cast<size_t>(ns) * 8);
    NPCG_CUDA(cudaMemcpy(h.data(), pdbg.get(), h.size() * 8, cudaMemcpyDeviceToHost));
    double acc[6] = {0, 0, 0, 0, 0, 0};
    int m = 0;
    for (int x = 0; x < ns; ++x) {
      const unsigned long long* c = &h[static_cast<size_t>(x) * 8];
      if (!c[5] || !c[6]) continue;  // (overflowed records return early)
      const unsigned long long v[6] = {c[6], c[0], c[1], c[2], c[3], c[4]};
      for (int q = 0; q < 5; ++q) acc[q] += static_cast<double>(v[q + 1] - v[q]);
      acc[5] += static_cast<double>(c[5] - c[4]);
      ++m;
    }
    std::fprintf(stderr, "[npcg plan profile] st %d records %d (complete %d), mean cycles: rows %.0f ids %.0f "
                 "halo %.0f items %.0f entries %.0f copyfix %.0f\n", st, ns, m, acc[0] / m, acc[1] / m,
                 acc[2] / m, acc[3] / m, acc[4] / m, acc[5] / m);
  }
}

// entries per kernel cell: shared-memory histogram of the structure's cells
__global__ void k_cell_hist(const int64_t* __restrict__ row_ptr, int64_t n_rows,
                            const uint32_t* __restrict__ kk, int K, unsigned long long* __restrict__ out) {
  __shared__ unsigned int h[KMAX];
  for (int x = threadIdx.x; x < K; x += blockDim.x) h[x] = 0;
  __syncthreads();
  const int64_t n = row_ptr[n_rows];
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&h[kk[e]], 1u);
  __syncthreads();
  for (int x = threadIdx.x; x < K; x += blockDim.x)
    if (h[x]) atomicAdd(&out[x], static_cast<unsigned long long>(h[x]));
}

static std::unique_ptr<TcDirPlan> build_dir_plan(npcg_context* ctx, const int64_t* row_ptr,
                                                 const uint32_t* col, const uint32_t* kk,
                                                 int64_t n_rows, int64_t n_cols,
                                                 const uint32_t* perm_rows,
                                                 const uint32_t* inv_perm_cols,
                                                 const std::vector<int64_t>& row_batches, int K,
                                                 int st, int hcap) {
  auto P = std::make_unique<TcDirPlan>();
  static const bool hprof = std::getenv("NPCG_PLAN_PROFILE") != nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  auto hms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count(); };
  P->st = st;
  P->hcap = hcap;
  P->n_rows = n_rows;
  P->n_cols = n_cols;
  P->K = K;
  if (n_rows == 0) return P;
  // level 0: 128-row sub-tiles, st per super-tile.  Tiles never cross a
  // batch boundary (the rows are batch-major), so a scene of a jagged batch
  // is tiled -- and computed, bit for bit -- exactly as the scene alone.
  std::vector<PlanLevel> lv(1);
  {
    std::vector<int64_t> bo = row_batches;
    if (bo.size() < 2 || bo.front() != 0 || bo.back() != n_rows) bo = {0, n_rows};
    for (size_t b = 0; b + 1 < bo.size(); ++b) {
      const int t0 = static_cast<int>(lv[0].tiles.size());
      for (int64_t p = bo[b]; p < bo[b + 1]; p += TM) {
        lv[0].tiles.push_back(make_uint2(static_cast<uint32_t>(p),
                                         static_cast<uint32_t>(std::min<int64_t>(TM, bo[b + 1] - p))));
        lv[0].nom.push_back(TM);
      }
      const int nt = static_cast<int>(lv[0].tiles.size());
      for (int t = t0; t < nt; t += st) lv[0].sup.push_back(make_uint2(t, std::min(st, nt - t)));
    }
  }
  // Planning levels form a worklist.  A plain super-tile beyond capacity
  // becomes, when only its halo is too large, one item of halo-segment
  // records (same rows, each record the entries of one column range of the
  // halo, <= hcap rows each); otherwise its rows are re-tiled as single
  // sub-tiles of half as many rows (128 after a multi-tile super-tile, 64,
  // ..., 8).  An 8-row tile that still fails becomes an item of rank-split
  // records (entries of rank [qQ, (q+1)Q) per (row, cell)), re-split with a
  // smaller Q down to the Q that always fits (8 rows x K cells x Q <= hcap);
  // only an item failing at that Q goes to the exact engine.
  std::vector<uint32_t> spill;
  const uint32_t q_safe = std::max<uint32_t>(1, static_cast<uint32_t>(hcap) / (8u * K));
  const uint32_t q_first = std::max<uint32_t>(q_safe, 64);
  auto push_rank_item = [](PlanLevel& nx, uint2 tile, uint32_t maxc, uint32_t Q) {
    const uint32_t nq = std::max<uint32_t>(1, (maxc + Q - 1) / Q);
    for (uint32_t q = 0; q < nq; ++q) {
      const uint32_t fl = (q == 0 ? SUP_FIRST : 0u) | (q + 1 == nq ? SUP_LAST : 0u);
      nx.sup.push_back(make_uint2(static_cast<uint32_t>(nx.tiles.size()), 1u | fl));
      nx.tiles.push_back(tile);
      nx.nom.push_back(8);
      nx.tfilter.push_back(make_uint4(q * Q, (q + 1) * Q, 0, 0xFFFFFFFFu));
    }
  };
  // mark the records [x, y) of a level overflowed (also on the device)
  auto drop = [&](PlanLevel& L, size_t x, size_t y) {
    for (size_t z = x; z < y; ++z) L.hl[z] = kOverflow;
    std::vector<uint32_t> ov(y - x, kOverflow);
    NPCG_CUDA(cudaMemcpyAsync(L.halo_len.get() + x, ov.data(), ov.size() * 4,
                              cudaMemcpyHostToDevice, ctx->stream));
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  };
  for (size_t li = 0; li < lv.size(); ++li) {
    // entries packed as (column << 7 | cell) in the planner's smem when they fit
    if (hprof) std::fprintf(stderr, "[npcg plan host] %.3f ms: level %zu start\n", hms(), li);
    plan_level(ctx, lv[li], row_ptr, col, kk, perm_rows, inv_perm_cols, K, st, hcap,
               n_cols <= (int64_t(1) << 25) && K <= 128);
    if (hprof) std::fprintf(stderr, "[npcg plan host] %.3f ms: level %zu planned\n", hms(), li);
    PlanLevel seg_items, halves, ranks;
    seg_items.kind = 2;
    ranks.kind = 1;
    PlanLevel& L = lv[li];
    // rows of a failed record / item -> smaller tiles (or rank items below 8 rows)
    auto retile = [&](uint32_t a, uint32_t b, uint32_t sz, uint32_t maxc) {
      if (sz < 8) {
        push_rank_item(ranks, make_uint2(a, b - a), maxc, q_first);
        return;
      }
      for (uint32_t p = a; p < b; p += sz) {
        halves.sup.push_back(make_uint2(static_cast<uint32_t>(halves.tiles.size()), 1));
        halves.tiles.push_back(make_uint2(p, std::min(sz, b - p)));
        halves.nom.push_back(sz);
      }
    };
    for (size_t x = 0; x < L.sup.size();) {
      size_t y = x + 1;  // records of one item
      if (L.kind != 0)
        while (y < L.sup.size() && !(L.sup[y].y & SUP_FIRST)) ++y;
      bool bad = false;
      for (size_t z = x; z < y; ++z) bad |= L.hl[z] == kOverflow;
      if (!bad) {
        x = y;
        continue;
      }
      const uint2 sp = L.sup[x];
      const uint32_t nsub = sp.y & 0xFFu;
      const uint32_t a = L.tiles[sp.x].x;
      const uint2 last = L.tiles[sp.x + nsub - 1];
      const uint32_t b = last.x + last.y;
      uint32_t maxc = 0;
      for (uint32_t t = sp.x; t < sp.x + nsub; ++t) maxc = std::max(maxc, L.maxc[t]);
      const uint32_t nom = L.nom[sp.x];
      if (L.kind == 0) {
        const uint32_t* sg = &L.seg[x * (MAXSEG + 1)];
        // halo too large only: a super-tile of several sub-tiles is re-tiled
        // first (halves: half the stages of segment records, and planned on
        // the plain path); a single tile becomes one item of segment records
        if (sg[0] >= 2 && (nsub == 1 || std::getenv("NPCG_PLAN_SEGMENTS_FIRST"))) {
          const uint32_t nseg = sg[0];
          for (uint32_t q = 0; q < nseg; ++q) {
            const uint32_t fl = (q == 0 ? SUP_FIRST : 0u) | (q + 1 == nseg ? SUP_LAST : 0u);
            seg_items.sup.push_back(make_uint2(static_cast<uint32_t>(seg_items.tiles.size()), nsub | fl));
            for (uint32_t t = sp.x; t < sp.x + nsub; ++t) {
              seg_items.tiles.push_back(L.tiles[t]);
              seg_items.nom.push_back(L.nom[t]);
              seg_items.tfilter.push_back(make_uint4(0, 0xFFFFFFFFu, q == 0 ? 0u : sg[q],
                                                     q + 1 == nseg ? 0xFFFFFFFFu : sg[q + 1]));
            }
          }
        } else {
          retile(a, b, nsub > 1 ? nom : nom / 2, maxc);
        }
      } else if (L.kind == 2) {
        drop(L, x, y);
        retile(a, b, nsub > 1 ? nom : nom / 2, maxc);
      } else {  // rank item: re-split with a smaller step, else the exact engine
        const uint32_t q_now = L.tfilter[sp.x].y - L.tfilter[sp.x].x;
        const uint32_t q_next = q_now > q_safe ? std::max(q_safe, q_now / 4) : 0;
        drop(L, x, y);
        if (q_next) push_rank_item(ranks, make_uint2(a, b - a), maxc, q_next);
        else
          for (uint32_t p = a; p < b; ++p) spill.push_back(p);
      }
      x = y;
    }
    for (PlanLevel* nx : {&seg_items, &halves, &ranks})
      if (!nx->sup.empty()) lv.push_back(std::move(*nx));
  }
  P->levels = static_cast<int>(lv.size());
  for (const PlanLevel& L : lv) P->big_blocks |= L.max_blk > static_cast<uint32_t>(BLOCK_MAX_BYTES);
  if (std::getenv("NPCG_PLAN_DEBUG")) {  // planner instrumentation (stderr)
    std::fprintf(stderr, "[npcg plan] rows %lld st %d hcap %d:", static_cast<long long>(n_rows), st, hcap);
    for (size_t li = 0; li < lv.size(); ++li) {
      size_t bad = 0;
      for (uint32_t h : lv[li].hl) bad += h == kOverflow;
      std::fprintf(stderr, " L%zu%s %zu recs (%zu tiles of %u rows) %zu failed;", li,
                   lv[li].kind == 1 ? "(rank)" : lv[li].kind == 2 ? "(seg)" : "", lv[li].sup.size(),
                   lv[li].tiles.size(), lv[li].nom.empty() ? 0u : lv[li].nom[0], bad);
    }
    std::fprintf(stderr, " spill rows %zu\n", spill.size());
  }
  if (lv.size() == 1) {  // one level: adopt its buffers as they are
    PlanLevel& L = lv[0];
    P->n_super = static_cast<int>(L.sup.size());
    P->n_sub = static_cast<int>(L.tiles.size());
    P->halo = std::move(L.halo);
    P->halo_len = std::move(L.halo_len);
    P->blk_off = std::move(L.blk_off);
    P->blocks = std::move(L.blocks);
    std::vector<uint2> sup_all(L.sup.size());
    std::vector<uint32_t> items(L.sup.size() + 1);
    double sum = 0;
    for (size_t x = 0; x < L.sup.size(); ++x) {
      sup_all[x] = make_uint2(L.sup[x].x, (L.sup[x].y & 0xFFu) | SUP_FIRST | SUP_LAST);
      items[x] = static_cast<uint32_t>(x);
      if (L.hl[x] == kOverflow) {
        P->n_overflow++;
      } else {
        P->max_halo = std::max<int>(P->max_halo, static_cast<int>(L.hl[x]));
        sum += L.hl[x];
      }
    }
    items[L.sup.size()] = static_cast<uint32_t>(L.sup.size());
    P->n_items = static_cast<int>(L.sup.size());
    P->item_start.alloc(ctx, items.size());
    P->sup.alloc(ctx, P->n_super);
    P->tiles.alloc(ctx, P->n_sub);
    NPCG_CUDA(cudaMemcpyAsync(P->item_start.get(), items.data(), items.size() * 4,
                              cudaMemcpyHostToDevice, ctx->stream));
    NPCG_CUDA(cudaMemcpyAsync(P->sup.get(), sup_all.data(), sup_all.size() * sizeof(uint2),
                              cudaMemcpyHostToDevice, ctx->stream));
    NPCG_CUDA(cudaMemcpyAsync(P->tiles.get(), L.tiles.data(), L.tiles.size() * sizeof(uint2),
                              cudaMemcpyHostToDevice, ctx->stream));
    const int ok = P->n_super - P->n_overflow;
    P->mean_halo = ok ? sum / ok : 0.0;
    NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
    return P;
  }
  // concatenate the levels
  int64_t ns = 0, nt = 0, bytes = 0;
  for (auto& L : lv) {
    ns += L.sup.size();
    nt += L.tiles.size();
    bytes += static_cast<int64_t>(blk_bytes(L.block_units));
  }
  P->n_super = static_cast<int>(ns);
  P->n_sub = static_cast<int>(nt);
  P->halo.alloc(ctx, ns * hcap);
  P->halo_len.alloc(ctx, ns);
  P->blk_off.alloc(ctx, nt * K + 1);
  P->blocks.alloc(ctx, bytes);
  std::vector<uint2> sup_all, tiles_all;
  int64_t s0 = 0, t0 = 0, b0 = 0;
  double sum = 0;
  std::vector<uint32_t> items;
  for (size_t li = 0; li < lv.size(); ++li) {
    PlanLevel& L = lv[li];
    const int64_t lns = L.sup.size(), lnt = L.tiles.size();
    for (const uint2& sp : L.sup) {
      // plain super-tiles are single-record items
      const uint32_t fl = L.kind != 0 ? (sp.y & (SUP_FIRST | SUP_LAST)) : (SUP_FIRST | SUP_LAST);
      if (fl & SUP_FIRST) items.push_back(static_cast<uint32_t>(sup_all.size()));
      sup_all.push_back(make_uint2(sp.x + static_cast<uint32_t>(t0), (sp.y & 0xFFu) | fl));
    }
    tiles_all.insert(tiles_all.end(), L.tiles.begin(), L.tiles.end());
    NPCG_CUDA(cudaMemcpyAsync(P->halo.get() + s0 * hcap, L.halo.get(), lns * hcap * 4,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    NPCG_CUDA(cudaMemcpyAsync(P->halo_len.get() + s0, L.halo_len.get(), lns * 4,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    NPCG_CUDA(cudaMemcpyAsync(P->blk_off.get() + t0 * K, L.blk_off.get(), (lnt * K + 1) * 4,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    if (b0)
      launch(ctx, "plan_rebase", k_add_u32, dim3(static_cast<unsigned>(ceil_div(lnt * K + 1, 256))),
             dim3(256), 0, P->blk_off.get() + t0 * K, lnt * K + 1, static_cast<uint32_t>(b0 >> 4));
    if (L.block_units)
      NPCG_CUDA(cudaMemcpyAsync(P->blocks.get() + b0, L.blocks.get(), blk_bytes(L.block_units),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    for (uint32_t h : L.hl) {
      if (h == kOverflow) {
        P->n_overflow++;
      } else {
        P->max_halo = std::max<int>(P->max_halo, static_cast<int>(h));
        sum += h;
      }
    }
    s0 += lns;
    t0 += lnt;
    b0 += static_cast<int64_t>(blk_bytes(L.block_units));
  }
  if (bytes >= (int64_t(1) << 36)) fail(NPCG_ERR_UNSUPPORTED, "tile plan exceeds 64 GB of descriptors");
  items.push_back(static_cast<uint32_t>(ns));
  P->n_items = static_cast<int>(items.size()) - 1;
  P->item_start.alloc(ctx, items.size());
  NPCG_CUDA(cudaMemcpyAsync(P->item_start.get(), items.data(), items.size() * 4,
                            cudaMemcpyHostToDevice, ctx->stream));
  P->sup.alloc(ctx, ns);
  P->tiles.alloc(ctx, nt);
  NPCG_CUDA(cudaMemcpyAsync(P->sup.get(), sup_all.data(), ns * sizeof(uint2), cudaMemcpyHostToDevice,
                            ctx->stream));
  NPCG_CUDA(cudaMemcpyAsync(P->tiles.get(), tiles_all.data(), nt * sizeof(uint2),
                            cudaMemcpyHostToDevice, ctx->stream));
  const int ok = P->n_super - P->n_overflow;
  P->mean_halo = ok ? sum / ok : 0.0;
  P->n_spill = static_cast<int64_t>(spill.size());
  if (P->n_spill) {
    P->spill_rows.alloc(ctx, P->n_spill);
    NPCG_CUDA(cudaMemcpyAsync(P->spill_rows.get(), spill.data(), spill.size() * 4,
                              cudaMemcpyHostToDevice, ctx->stream));
  }
  // per-cell entry counts (the weight gradient balances its cell runs on them)
  DevBuf<unsigned long long> kc(ctx, K);
  NPCG_CUDA(cudaMemsetAsync(kc.get(), 0, K * 8, ctx->stream));
  launch(ctx, "plan_cell_hist", k_cell_hist, dim3(static_cast<unsigned>(ctx->num_sms * 4)), dim3(256), 0,
         row_ptr, n_rows, kk, K, kc.get());
  P->k_count.assign(K, 0);
  NPCG_CUDA(cudaMemcpyAsync(P->k_count.data(), kc.get(), K * 8, cudaMemcpyDeviceToHost, ctx->stream));
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
  if (hprof) std::fprintf(stderr, "[npcg plan host] %.3f ms: plan done (%d records)\n", hms(), P->n_super);
  return P;
}

// ===========================================================================
// operand preparation
// ===========================================================================
// dst[p][c] = bf16(src[perm[p]][c]) for c < C, 0 for C <= c < CP (C % 8 == 0),
// 8 channels per thread.
__global__ void k_to_bf16_perm(const float* __restrict__ src, const uint32_t* __restrict__ perm,
                               int64_t n, int C, int CP, __nv_bfloat16* __restrict__ dst) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int qn = CP >> 3;
  if (x >= n * qn) return;
  const int64_t p = x / qn;
  const int q = static_cast<int>(x % qn);
  if (q * 8 >= C) {
    reinterpret_cast<uint4*>(dst + p * CP)[q] = make_uint4(0, 0, 0, 0);
    return;
  }
  const float4* s = reinterpret_cast<const float4*>(src + static_cast<int64_t>(perm[p]) * C + q * 8);
  const float4 a = __ldg(s), b = __ldg(s + 1);
  uint4 o;
  o.x = pack_bf16x2(a.x, a.y);
  o.y = pack_bf16x2(a.z, a.w);
  o.z = pack_bf16x2(b.x, b.y);
  o.w = pack_bf16x2(b.z, b.w);
  reinterpret_cast<uint4*>(dst + p * CP)[q] = o;
}

// ---- split operands of the fp32-contract path ---------------------------
// A tensor x is scaled by a power of two s (max |x| s < 2^7, exact) and each
// y = x s is split into two fp16 halves, y = hi + lo 2^-11 with hi = fp16(y),
// lo = fp16((y - hi) 2^11): 22 significand bits (fp32 has 24), both halves in
// range for sums of up to 254 rows (the planner's per-(row, cell) cap).
// max |x| of a tensor, as the bits of a non-negative float (atomicMax on the
// bit pattern orders like the value)
__global__ void k_absmax(const float* __restrict__ x, int64_t n, uint32_t* __restrict__ out) {
  uint32_t m = 0;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = max(m, __float_as_uint(fabsf(x[p])));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}
// s = 2^(7 - e) for max = f 2^e (f in [0.5, 1)): max s < 128; 1 when max = 0
__host__ __device__ __forceinline__ float split_scale(uint32_t max_bits) {
  if (max_bits == 0 || max_bits >= 0x7F800000u) return 1.f;
  const int e = static_cast<int>((max_bits >> 23) & 0xFF) - 126;  // max < 2^e (normal inputs)
  const int k = 7 - (e < -100 ? -100 : e);
  return ldexpf(1.f, k > 100 ? 100 : k);
}
__device__ __forceinline__ void split_f16(float y, float& hi, float& lo) {
  hi = __half2float(__float2half_rn(y));
  lo = (y - hi) * 2048.f;
}

// Split image: row p = for each chunk of 32 channels [hi(32) | lo(32)] in
// fp16 (128 bytes) of y = x s; channels C <= c < CP zero.  8 channels per thread.
__global__ void k_to_split_perm(const float* __restrict__ src, const uint32_t* __restrict__ perm,
                                int64_t n, int C, int CP, const uint32_t* __restrict__ amax,
                                __half* __restrict__ dst) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int qn = CP >> 3;
  if (x >= n * qn) return;
  const int64_t p = x / qn;
  const int q = static_cast<int>(x % qn);  // channels 8q .. 8q+7
  uint4 h = make_uint4(0, 0, 0, 0), l = make_uint4(0, 0, 0, 0);
  if (q * 8 < C) {
    const float sc = split_scale(*amax);
    const float4* s = reinterpret_cast<const float4*>(src + static_cast<int64_t>(perm[p]) * C + q * 8);
    const float4 a = __ldg(s), b = __ldg(s + 1);
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    float hv[8], lv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split_f16(v[i] * sc, hv[i], lv[i]);
    h = make_uint4(pack_f16x2(hv[0], hv[1]), pack_f16x2(hv[2], hv[3]), pack_f16x2(hv[4], hv[5]),
                   pack_f16x2(hv[6], hv[7]));
    l = make_uint4(pack_f16x2(lv[0], lv[1]), pack_f16x2(lv[2], lv[3]), pack_f16x2(lv[4], lv[5]),
                   pack_f16x2(lv[6], lv[7]));
  }
  uint4* row = reinterpret_cast<uint4*>(dst + p * 2 * CP);  // 16-byte units, 8 per 32-channel chunk
  const int chunk = q >> 2, sub = q & 3;
  row[chunk * 8 + sub] = h;
  row[chunk * 8 + 4 + sub] = l;
}

// Split B images (SW128 K-major, fp16) per (cell, 32-wide chunk r0 of the
// reduction dim), of W s_w = Wh + Wl 2^-11:
//   image 1 (main)  K 0..31 = Wh[r0 + kk], K 32..63 = 0 (only its first 32 K are read)
//   image 2 (corr)  K 0..31 = Wl[r0 + kk], K 32..63 = Wh[r0 + kk - 32]
// so that the tile [Ah | Al] gives main = Ah Wh and corr = Ah Wl + Al Wh.
// transpose as k_pack_w.
// Only B rows [n0, n0 + N) are packed (a 128-column half of a wider pass).
__global__ void k_pack_w_split(const float* __restrict__ w, int K, int cin, int cout, int N, int nchunk,
                               int n0, bool transpose, const uint32_t* __restrict__ amax,
                               uint8_t* __restrict__ out) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= static_cast<int64_t>(K) * cin * cout) return;
  const int k = static_cast<int>(x / (cin * cout)), rem = static_cast<int>(x % (cin * cout));
  const int c = rem / cout, m = rem % cout;  // W[k][c][m]
  const int n = (transpose ? c : m) - n0, r = transpose ? m : c;
  if (n < 0 || n >= N) return;
  const int64_t img = (static_cast<int64_t>(k) * nchunk + r / 32) * 2;  // two images per chunk
  float hi, lo;
  split_f16(w[x] * split_scale(*amax), hi, lo);
  uint8_t* i1 = out + img * N * 128;
  uint8_t* i2 = i1 + N * 128;
  reinterpret_cast<__half*>(i1 + sw128_off(n, r % 32))[0] = __float2half_rn(hi);
  reinterpret_cast<__half*>(i2 + sw128_off(n, r % 32))[0] = __float2half_rn(lo);
  reinterpret_cast<__half*>(i2 + sw128_off(n, 32 + r % 32))[0] = __float2half_rn(hi);
}

// B operand images (SW128 K-major), one per (cell, 64-wide chunk of the
// reduction dim), N x 128 B each.  transpose=false: N = C_out rows, reduction
// over C_in (forward); transpose=true: N = C_in rows, reduction over C_out (dgrad).
__global__ void k_pack_w(const float* __restrict__ w, int K, int cin, int cout, int cinp,
                         int coutp, bool transpose, uint8_t* __restrict__ out) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= static_cast<int64_t>(K) * cin * cout) return;
  const int k = static_cast<int>(x / (cin * cout)), rem = static_cast<int>(x % (cin * cout));
  const int c = rem / cout, m = rem % cout;  // W[k][c][m]
  const int n = transpose ? c : m, r = transpose ? m : c;  // B row, reduction index
  const int N = transpose ? cinp : coutp, nchunk = (transpose ? coutp : cinp) / CH;
  const int64_t img = static_cast<int64_t>(k) * nchunk + r / CH;
  reinterpret_cast<__nv_bfloat16*>(out + img * N * 128 + sw128_off(n, r % CH))[0] =
      __float2bfloat16_rn(w[x]);
}

// ===========================================================================
// forward / dgrad kernel
// ===========================================================================
struct FwdArgs {
  const uint32_t* halo;
  const uint32_t* halo_len;
  const uint32_t* blk_off;
  const uint8_t* blocks;
  const uint32_t* perm_rows;
  const uint2* sup;           // per record {first sub-tile, sub-tiles | SUP_FIRST | SUP_LAST}
  const uint2* tiles;         // per sub-tile {first permuted row, rows}
  const uint32_t* item_start; // n_items + 1: records [item_start[w], item_start[w + 1]) share rows
  int n_items;
  int64_t n_rows;
  int n_sub, n_super, st, hcap, K;
  int nci;                    // 64-channel chunks of the gathered features
  const __nv_bfloat16* feat;  // bf16 (n_cols, 64 nci), permuted
  const uint8_t* wpack;       // (K x nci) images of NOUT x 128 B
  float* out;                 // (n_rows, ncols), original order
  int ncols;                  // channels written per row (<= NOUT; the rest is padding)
  int out_stride, out_col0;   // output row stride and first written column (128-column halves)
  long long* trace;           // debug: per-stage event clocks of CTA 0 (traced variant only)
  const uint32_t* amax;       // SPLIT: max |x| bits of the gathered tensor and of W (scales)
};
constexpr int TRACE_STAGES = 512;
constexpr int TRACE_EV = 16;  // 0 d_issue, 1 d_full, 2 a_empty, 3 agg_done, 4 mma_start, 5 mma_issued, 6 w_full,
                              // 7 grp_done, 8 cell top, 10 fence done, 11 mma block done, 12 cell end
__device__ __forceinline__ void trace_ev(long long* tr, uint32_t stage, int ev) {
  if (tr && blockIdx.x == 0 && stage < TRACE_STAGES) tr[stage * TRACE_EV + ev] = clock64();
}
// the latest of several warps' clocks (ev 7: the group's last aggregation warp done)
__device__ __forceinline__ void trace_max(long long* tr, uint32_t stage, int ev) {
  if (tr && blockIdx.x == 0 && stage < TRACE_STAGES)
    atomicMax(reinterpret_cast<unsigned long long*>(tr) + stage * TRACE_EV + ev,
              static_cast<unsigned long long>(clock64()));
}

constexpr int FWD_AGG_WARP0 = 6;
constexpr int FWD_AGG_WARPS = 16;
constexpr int AGG_GROUPS = 4;                           // stage s is aggregated by group s % 4
constexpr int AGG_GROUP_WARPS = FWD_AGG_WARPS / AGG_GROUPS;
constexpr int FWD_W_WARP = FWD_AGG_WARP0 + FWD_AGG_WARPS;
constexpr int FWD_THREADS = 32 * (FWD_W_WARP + 1);
constexpr int FWD_ST = 2, FWD_HCAP = 928;  // 256-row super-tiles, halo <= 928 rows (116 KB)
#ifndef FWD_NMAIN
#define FWD_NMAIN 3  // split path: main accumulator sets (A/B)
#endif
constexpr int NSA = 4;  // A stages (16 KB)
constexpr int NSW = 3;  // W stages (NOUT x 128 B; 2 for NOUT = 256)
constexpr int NSD = 8;  // stage-descriptor slots (a multiple of AGG_GROUPS)
// per-CTA smem words: a super-tile's block offsets (st * K + 1 <= 2 * KMAX + 1)
// followed by the descriptor slots' sources (<= 2 * WG_NSD)
constexpr int OFFS_DSRC = 2 * KMAX + 4;
constexpr int OFFS_WORDS = OFFS_DSRC + 8;
// Wide outputs (NOUT = channels the pass writes): the W stages grow to
// NOUT x 128 B (two stages, six descriptor slots); NOUT = 128 keeps the
// 256-row super-tiles (TMEM 2 x 2 x 128 columns), NOUT = 256 uses 128-row
// super-tiles (TMEM 2 x 256 columns) with a smaller halo.
constexpr int FWD_HCAP1 = 672;  // halo rows of 128-row tiles (what fits beside 256-wide W stages)
// SPLIT (fp32-contract path): every stage multiplies the split A tile
// [Ah | Al] (32 input channels) by two W images -- [Wh; Wh] over the full K =
// 64 (Ah Wh + Al Wh) and [Wl; 0] over its first 32 K (Ah Wl) -- so a W stage
// is two NOUT x 128 B images; NOUT = 128 runs on 128-row super-tiles (the
// wide plan) to make room for them.
template <int NOUT, bool SPLIT = false>
struct FwdCfg {
  static constexpr int nsw = (NOUT == 64 && !SPLIT) ? NSW : 2;
  // descriptor slots: a multiple of the aggregation groups, so a slot is
  // always consumed by the same group (a waiter can then never be two
  // barrier phases ahead, which a parity wait cannot tell apart)
  static constexpr int nsd = NSD;
  static constexpr uint32_t wimg = NOUT * 128;              // one W image
  static constexpr uint32_t wbytes = (SPLIT ? 2 : 1) * wimg;  // a W stage
  static constexpr int st = (NOUT == 64 || (NOUT == 128 && !SPLIT)) ? FWD_ST : 1;
  static constexpr int acc_cols = st * NOUT;  // one accumulator set
  // SPLIT: NMAIN main accumulator sets (hi x hi, cells alternating: short
  // truncating chains, summed in fp32 round-to-nearest by the epilogue) and one
  // correction set, single-buffered; bf16: one set, double-buffered
  static constexpr int nmain = SPLIT ? FWD_NMAIN : 1;
  static constexpr int bsets = SPLIT ? nmain + 1 : 1;       // accumulator sets per buffer
  static constexpr int nbuf = 2 * bsets * acc_cols <= 512 ? 2 : 1;
  static constexpr int nsets = nbuf * bsets;
  static constexpr uint32_t bstride = bsets * acc_cols;     // TMEM columns per buffer
  static constexpr uint32_t tmem_cols = nsets * acc_cols <= 256 ? 256 : 512;
  static_assert(nsets * acc_cols <= 512, "TMEM");
  // the halo row list staged in smem by the descriptor producer (room only
  // beside the 64-column W stages)
  static constexpr bool hidx = NOUT == 64 && !SPLIT;
};

struct FwdSmem {
  uint32_t halo, a, w, d, bar, tmem_slot, offs, hidx;
  size_t total;
};
template <int NOUT, bool SPLIT = false>
__host__ __device__ constexpr FwdSmem fwd_smem_layout(int hcap) {
  using Cfg = FwdCfg<NOUT, SPLIT>;
  FwdSmem L{};
  uint32_t o = 0;
  L.halo = o;
  o += hcap * 128;
  o = (o + 1023) & ~1023u;
  L.a = o;
  o += NSA * 16384;
  L.w = o;
  o += Cfg::nsw * Cfg::wbytes;
  L.d = o;
  o += Cfg::nsd * BLOCK_MAX_BYTES;
  o = (o + 7) & ~7u;
  L.bar = o;
  o += 48 * 8;
  L.tmem_slot = o;
  o += 16;
  L.offs = o;
  o += OFFS_WORDS * 4;  // block offsets of the super-tile, then the slot sources
  o = (o + 15) & ~15u;
  L.hidx = o;           // the record's halo row list (bulk-copied ahead by the descriptor producer)
  if (Cfg::hidx) o += ((hcap * 4 + 15) & ~15);
  L.total = o + 1024;   // alignment slack
  return L;
}

static_assert(NSD % AGG_GROUPS == 0, "descriptor slots per group");
static_assert(fwd_smem_layout<64>(FWD_HCAP).total <= 232448, "smem");
static_assert(fwd_smem_layout<128>(FWD_HCAP).total <= 232448, "smem");
static_assert(fwd_smem_layout<256>(FWD_HCAP1).total <= 232448, "smem");
static_assert(fwd_smem_layout<64, true>(FWD_HCAP).total <= 232448, "smem");
static_assert(fwd_smem_layout<128, true>(FWD_HCAP1).total <= 232448, "smem");

// Warm L2 with a super-tile's halo rows: one prefetch.global.L2 per 128-byte
// row, row indices loaded in batches of 8 per lane before the prefetches.
template <int NT>
__device__ __forceinline__ void prefetch_halo_l2(const uint32_t* rows, uint32_t H,
                                                 const __nv_bfloat16* feat, int t,
                                                 int64_t stride = CH, int nchunk = 1) {
  for (uint32_t h0 = 0; h0 < H; h0 += 8 * NT) {
    uint32_t r[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const uint32_t h = h0 + x * NT + t;
      r[x] = h < H ? rows[h] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int x = 0; x < 8; ++x)
      if (r[x] != 0xFFFFFFFFu)
        for (int c = 0; c < nchunk; ++c)  // 64-channel chunks of the row
          asm volatile("prefetch.global.L2 [%0];" ::"l"(feat + static_cast<int64_t>(r[x]) * stride + c * CH));
  }
}
// Cooperative halo load by the aggregation warps: 16-byte cp.async per lane,
// 8 lanes per 128-byte row (coalesced within runs of consecutive rows).
// The row indices of a batch are loaded first (independent loads in flight),
// then the batch's copies are issued.
template <int NT, bool SMEM_ROWS = false>
__device__ __forceinline__ void coop_load_halo(const uint32_t* rows, uint32_t H,
                                               const __nv_bfloat16* feat, uint32_t s_halo,
                                               int t, int64_t stride = CH) {
  constexpr uint32_t STEP = NT / 8, B = 8;
  const uint32_t q = static_cast<uint32_t>(t & 7);
  const uint8_t* base = reinterpret_cast<const uint8_t*>(feat) + q * 16u;
  for (uint32_t h0 = static_cast<uint32_t>(t) >> 3; h0 < H; h0 += B * STEP) {
    uint32_t r[B];
#pragma unroll
    for (uint32_t x = 0; x < B; ++x) {
      const uint32_t h = h0 + x * STEP;
      r[x] = h < H ? (SMEM_ROWS ? rows[h] : __ldg(rows + h)) : 0u;
    }
#pragma unroll
    for (uint32_t x = 0; x < B; ++x) {
      const uint32_t h = h0 + x * STEP;
      if (h < H) cp_async16(s_halo + h * 128u + q * 16u, base + static_cast<int64_t>(r[x]) * stride * 2);
    }
  }
  cp_async_wait_all();
}
// Entries of a staged block are in the slot, or in global memory (L2) when
// the block did not fit (src = its byte offset, kFitsSlot when it fit).  The
// L2 variant is an out-of-line call, keeping the hot loop's code compact.
constexpr uint32_t kFitsSlot = 0xFFFFFFFFu;

// barrier indices
enum : int {
  B_HALO_FULL = 0,
  B_HALO_EMPTY = 1,
  B_A_FULL = 2,              // NSA
  B_A_EMPTY = B_A_FULL + NSA,
  B_W_FULL = B_A_EMPTY + NSA,  // NSW
  B_W_EMPTY = B_W_FULL + NSW,
  B_D_FULL = B_W_EMPTY + NSW,  // NSD
  B_D_EMPTY = B_D_FULL + NSD,
  B_T_FULL = B_D_EMPTY + NSD,  // 2
  B_T_EMPTY = B_T_FULL + 2,
  B_COUNT = B_T_EMPTY + 2
};
static_assert(B_COUNT <= 48, "barrier region");

// One pipeline stage of the aggregation: the 128 rows of a sub-tile for one
// kernel cell.  Warp `aw` of NW handles quads aw, aw+NW, ... (4 rows, a
// quarter-warp per 128-byte row).  Items are rows sorted by entry count
// (descending), so quads are mostly count-uniform: count 0 -> zero row,
// count 1 -> exact bf16 copy of the halo row, count >= 2 -> fp32 sum
// (FHADD.BF16) rounded once to bf16.  All loads of the warp's quads are issued
// before their uses (ILP), stores go to the SW128 K-major A tile.
// wait_slot() is called once, before the first store into the A slot, so the
// item / halo loads of the copy pass overlap the wait for the slot.
// SPLIT (the fp32-contract path): the halo rows are split images, each
// 128-byte row = [hi(32 channels) | lo(32 channels)] in fp16 of the scaled
// value y = x s = hi + lo 2^-11 (split_f16); lanes 0-3 of a row hold hi
// parts, lanes 4-7 the lo parts of the same channels.  Count-1 rows copy the
// pair unchanged; rows of >= 2 entries sum hi and lo in fp32 per lane, form
// the total hi_sum + lo_sum 2^-11 on both partner lanes (lane ^ 4, the same
// expression: bitwise equal) and split it again.
template <int NW, bool SPLIT = false, typename WaitSlot>
__device__ __forceinline__ void aggregate_stage(const uint8_t* blk, const uint16_t* ents,
                                                uint32_t s_halo, uint32_t s_A, int wig, int lane,
                                                WaitSlot&& wait_slot) {
  static_assert(NW == 4, "item layout (item_slot) is for four warps per A tile");
  constexpr int NQ = (TM / 4) / NW;  // quads per warp, round-robin over count-sorted items
  const uint32_t* items = reinterpret_cast<const uint32_t*>(blk);
  const int sub_l = lane >> 3;
  const uint32_t l8x16 = static_cast<uint32_t>(lane & 7) << 4;
  uint32_t it[NQ], cm[NQ];
  {  // a lane's eight items (two 16-byte loads); the quads' first items
     // (count-sorted: their largest counts) by broadcast loads
    const uint4* iv = reinterpret_cast<const uint4*>(items + wig * 32 + sub_l * 8);
    const uint4* fv = reinterpret_cast<const uint4*>(items + wig * 32);
    const uint4 a0 = iv[0], a1 = iv[1], f0 = fv[0], f1 = fv[1];
    it[0] = a0.x; it[1] = a0.y; it[2] = a0.z; it[3] = a0.w;
    it[4] = a1.x; it[5] = a1.y; it[6] = a1.z; it[7] = a1.w;
    cm[0] = item_count(f0.x); cm[1] = item_count(f0.y); cm[2] = item_count(f0.z);
    cm[3] = item_count(f0.w); cm[4] = item_count(f1.x); cm[5] = item_count(f1.y);
    cm[6] = item_count(f1.z); cm[7] = item_count(f1.w);
  }
  // pass 1: quads whose rows have at most one entry: zero rows / exact bf16 copies
  uint4 v[NQ];
#pragma unroll
  for (int qi = 0; qi < NQ; ++qi) {
    v[qi] = make_uint4(0, 0, 0, 0);
    if (cm[qi] <= 1u && item_count(it[qi]) == 1u)  // copy quads: x = the halo index
      v[qi] = lds128(s_halo + item_eo(it[qi]) * 128u + l8x16);
  }
  wait_slot();
#pragma unroll
  for (int qi = 0; qi < NQ; ++qi) {
    if (cm[qi] <= 1u) {
      sts128(s_A + item_sw128(it[qi], l8x16), v[qi]);
    }
  }
  // pass 2: quads with a row of >= 2 entries: fp32 sums rounded once to bf16
#pragma unroll
  for (int qi = 0; qi < NQ; ++qi) {
    if (cm[qi] >= 2u) {
      const uint32_t c = item_count(it[qi]), eo = item_eo(it[qi]);
      if (!SPLIT && cm[qi] == 2u) {  // at most two entries per row: one packed bf16x2 add
        uint4 w0 = make_uint4(0, 0, 0, 0), w1 = make_uint4(0, 0, 0, 0);
        if (c > 0u) w0 = lds128(s_halo + static_cast<uint32_t>(ents[eo]) * 128u + l8x16);
        if (c > 1u) w1 = lds128(s_halo + static_cast<uint32_t>(ents[eo + 1]) * 128u + l8x16);
        uint4 o;
        o.x = add_bf16x2_rn(w0.x, w1.x);
        o.y = add_bf16x2_rn(w0.y, w1.y);
        o.z = add_bf16x2_rn(w0.z, w1.z);
        o.w = add_bf16x2_rn(w0.w, w1.w);
        sts128(s_A + item_sw128(it[qi], l8x16), o);
        continue;
      }
      float acc[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) acc[x] = 0.f;
      for (uint32_t e = 0; e < cm[qi]; e += 2) {
        uint4 w0 = make_uint4(0, 0, 0, 0), w1 = make_uint4(0, 0, 0, 0);
        if (e < c) w0 = lds128(s_halo + static_cast<uint32_t>(ents[eo + e]) * 128u + l8x16);
        if (e + 1 < c) w1 = lds128(s_halo + static_cast<uint32_t>(ents[eo + e + 1]) * 128u + l8x16);
        if constexpr (SPLIT) {
          acc_f16x2(acc[0], acc[1], w0.x);
          acc_f16x2(acc[2], acc[3], w0.y);
          acc_f16x2(acc[4], acc[5], w0.z);
          acc_f16x2(acc[6], acc[7], w0.w);
          acc_f16x2(acc[0], acc[1], w1.x);
          acc_f16x2(acc[2], acc[3], w1.y);
          acc_f16x2(acc[4], acc[5], w1.z);
          acc_f16x2(acc[6], acc[7], w1.w);
        } else {
          acc_bf16x2(acc[0], acc[1], w0.x);
          acc_bf16x2(acc[2], acc[3], w0.y);
          acc_bf16x2(acc[4], acc[5], w0.z);
          acc_bf16x2(acc[6], acc[7], w0.w);
          acc_bf16x2(acc[0], acc[1], w1.x);
          acc_bf16x2(acc[2], acc[3], w1.y);
          acc_bf16x2(acc[4], acc[5], w1.z);
          acc_bf16x2(acc[6], acc[7], w1.w);
        }
      }
      uint4 o;
      if constexpr (SPLIT) {
        const bool lo_lane = (lane & 4) != 0;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const float other = __shfl_xor_sync(0xffffffffu, acc[x], 4);
          // y = hi_sum + lo_sum 2^-11 (the same expression on both lanes)
          const float y = lo_lane ? fmaf(acc[x], 0x1p-11f, other) : fmaf(other, 0x1p-11f, acc[x]);
          const float hi = __half2float(__float2half_rn(y));
          acc[x] = lo_lane ? (y - hi) * 2048.f : hi;
        }
        o.x = pack_f16x2(acc[0], acc[1]);
        o.y = pack_f16x2(acc[2], acc[3]);
        o.z = pack_f16x2(acc[4], acc[5]);
        o.w = pack_f16x2(acc[6], acc[7]);
      } else {
        o.x = pack_bf16x2(acc[0], acc[1]);
        o.y = pack_bf16x2(acc[2], acc[3]);
        o.z = pack_bf16x2(acc[4], acc[5]);
        o.w = pack_bf16x2(acc[6], acc[7]);
      }
      sts128(s_A + item_sw128(it[qi], l8x16), o);
    }
  }
}
template <int NW, bool SPLIT = false>
__device__ __noinline__ void aggregate_stage_l2(const uint8_t* blk, const uint16_t* ents,
                                                uint32_t s_halo, uint32_t s_A, int wig, int lane) {
  aggregate_stage<NW, SPLIT>(blk, ents, s_halo, s_A, wig, lane, [] {});
}

// Input channels come in a.nci chunks of 64: each super-tile runs the cells
// once per chunk (the halo reloaded with that chunk's 128-byte row slices),
// all accumulating into the same TMEM accumulators; W_k is packed per (cell,
// chunk) as an NOUT x 64 image.
// BIG: the plan has descriptor blocks beyond the shared-memory slot (their
// entries are read from L2); plans without them run the leaner variant.
// SPLIT: the fp32-contract path (chunks of 32 split channels, two W images).
template <int NOUT, bool BIG, bool TRACE = false, bool SPLIT = false>
__global__ void __launch_bounds__(FWD_THREADS, 1) k_conv_fwd_tc(FwdArgs a) {
  // pipeline event clocks only in the traced debug variant (the checks cost
  // issue slots in the product kernel)
  auto tev = [&](uint32_t stage, int ev) {
    if constexpr (TRACE) trace_ev(a.trace, stage, ev);
  };
  using Cfg = FwdCfg<NOUT, SPLIT>;
  constexpr int NSWt = Cfg::nsw, NSDt = Cfg::nsd;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const FwdSmem L = fwd_smem_layout<NOUT, SPLIT>(a.hcap);
  const int nci = a.nci;
  // SPLIT: main accumulators actually used (a record has K * nci stages)
  const int nmain = SPLIT ? min(Cfg::nmain, a.K * nci) : 1;
  const int64_t fstride = static_cast<int64_t>(nci) * CH;
  const uint32_t s_halo = base + L.halo, s_a = base + L.a, s_w = base + L.w, s_d = base + L.d;
  const uint32_t s_hidx = base + L.hidx;
  const uint32_t s_bar = base + L.bar;
  auto bar = [&](int i) { return s_bar + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + L.tmem_slot);
  const uint8_t* g_d = gbase + L.d;
  uint32_t* dsrc = reinterpret_cast<uint32_t*>(gbase + L.offs) + OFFS_DSRC;  // per descriptor slot

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar(B_HALO_FULL), 1);
    mbar_init(bar(B_HALO_EMPTY), FWD_AGG_WARPS);
    for (int i = 0; i < NSA; ++i) {
      mbar_init(bar(B_A_FULL + i), AGG_GROUP_WARPS);
      mbar_init(bar(B_A_EMPTY + i), 1);
    }
    for (int i = 0; i < NSWt; ++i) {
      mbar_init(bar(B_W_FULL + i), 1);
      mbar_init(bar(B_W_EMPTY + i), 1);
    }
    for (int i = 0; i < NSDt; ++i) {
      mbar_init(bar(B_D_FULL + i), 1);
      mbar_init(bar(B_D_EMPTY + i), AGG_GROUP_WARPS);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(B_T_FULL + i), 1);
      mbar_init(bar(B_T_EMPTY + i), 4);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<Cfg::tmem_cols>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int K = a.K;

  if (warp == 4) {
    // ------------------------ producer: halo + descriptors -----------------
    uint32_t* offs = reinterpret_cast<uint32_t*>(gbase + L.offs);
    uint32_t d_it = 0, h_it = 0;
    for (int w = blockIdx.x; w < a.n_items; w += gridDim.x)
    for (int s = static_cast<int>(a.item_start[w]); s < static_cast<int>(a.item_start[w + 1]); ++s) {
      const uint2 sp = a.sup[s];
      const int nsub = static_cast<int>(sp.y & 0xFFu);
      if (a.halo_len[s] == kOverflow) continue;
      if (Cfg::hidx && lane == 0) {  // the record's halo row list into shared memory (agg warps release it)
        const uint32_t hb = (a.halo_len[s] * 4u + 15u) & ~15u;
        mbar_wait(bar(B_HALO_EMPTY), (h_it & 1) ^ 1);
        mbar_expect_tx(bar(B_HALO_FULL), hb);
        if (hb) bulk_g2s(s_hidx, a.halo + static_cast<int64_t>(s) * a.hcap, hb, bar(B_HALO_FULL));  // (H = 0: arrival alone)
      }
      ++h_it;
      // stage this super-tile's descriptor offsets in smem
      const int64_t ob = static_cast<int64_t>(sp.x) * K;
      for (int x = lane; x <= nsub * K; x += 32) offs[x] = a.blk_off[ob + x];
      __syncwarp();
      for (int c = 0; c < nci; ++c)
      for (int k = 0; k < K; ++k) {
        for (int g = 0; g < nsub; ++g) {
          if (lane == 0) {
            const uint32_t ds = d_it % NSDt;
            mbar_wait(bar(B_D_EMPTY + ds), ((d_it / NSDt) & 1) ^ 1);
            const uint32_t o0 = offs[g * K + k], o1 = offs[g * K + k + 1];
            const uint32_t nb = min((o1 - o0) << 4, static_cast<uint32_t>(BLOCK_MAX_BYTES));
            if (BIG) dsrc[ds] = (o1 - o0) << 4 > static_cast<uint32_t>(BLOCK_MAX_BYTES) ? o0 : kFitsSlot;
            mbar_expect_tx(bar(B_D_FULL + ds), nb);
            bulk_g2s(s_d + ds * BLOCK_MAX_BYTES, a.blocks + blk_bytes(o0), nb, bar(B_D_FULL + ds));
            tev(d_it, 0);
          }
          ++d_it;
        }
      }
      __syncwarp();
    }
  } else if (warp == FWD_W_WARP) {
    // ------------------------ producer: W_k per super-tile and cell ---------
    if (lane == 0) {
      uint32_t w_it = 0;
      for (int w = blockIdx.x; w < a.n_items; w += gridDim.x)
    for (int s = static_cast<int>(a.item_start[w]); s < static_cast<int>(a.item_start[w + 1]); ++s) {
        if (a.halo_len[s] == kOverflow) continue;
        for (int c = 0; c < nci; ++c)
        for (int k = 0; k < K; ++k) {
          const uint32_t ws = w_it % NSWt;
          mbar_wait_sleep(bar(B_W_EMPTY + ws), ((w_it / NSWt) & 1) ^ 1);
          mbar_expect_tx(bar(B_W_FULL + ws), Cfg::wbytes);
          bulk_g2s(s_w + ws * Cfg::wbytes,
                   a.wpack + (static_cast<int64_t>(k) * nci + c) * Cfg::wbytes, Cfg::wbytes,
                   bar(B_W_FULL + ws));
          ++w_it;
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------ MMA issuer -----------------------------
    // The whole warp runs the loop converged (warp-uniform descriptors); one
    // elected lane issues tcgen05.mma / commit.
    constexpr uint32_t idesc = SPLIT ? idesc_f16(128, NOUT, false, false) : idesc_bf16(128, NOUT, false, false);
    constexpr uint32_t NB = Cfg::nbuf;
    const uint64_t a_desc0 = sdesc_sw128(s_a, 16, 1024), b_desc0 = sdesc_sw128(s_w, 16, 1024);
    uint32_t w_it = 0, a_it = 0, t_it = 0;
    // The epilogue warps block on named barrier 2 + (tile & 1) (no polling);
    // the tile's accumulator is handed over once its T_FULL commit landed,
    // checked after the first cell of the next tile has been issued.
    bool pending = false;
    uint32_t pend_t = 0;
    auto release_epilogue = [&]() {
      mbar_wait(bar(B_T_FULL + (pend_t % NB)), (pend_t / NB) & 1);
      named_bar_arrive(2 + (pend_t % NB), 32 * 5);
      pending = false;
    };
    for (int w = blockIdx.x; w < a.n_items; w += gridDim.x)
    for (int s = static_cast<int>(a.item_start[w]); s < static_cast<int>(a.item_start[w + 1]); ++s) {
      const uint2 sp = a.sup[s];
      const int nsub = static_cast<int>(sp.y & 0xFFu);
      if (a.halo_len[s] == kOverflow) continue;
      const bool first = (sp.y & SUP_FIRST) != 0, last = (sp.y & SUP_LAST) != 0;
      const uint32_t ab = t_it % NB;
      if (first) mbar_wait(bar(B_T_EMPTY + ab), ((t_it / NB) & 1) ^ 1);
      tc_fence_after();
      for (int c = 0; c < nci; ++c)
      for (int k = 0; k < K; ++k) {
        if (lane == 0) tev(a_it, 8);
        if (pending && (c > 0 || k == 1 || !first)) release_epilogue();
        const uint32_t ws = w_it % NSWt;
        mbar_wait(bar(B_W_FULL + ws), (w_it / NSWt) & 1);
        if (lane == 0) tev(a_it, 6);
        // The sub-tiles' stages of cell k feed different accumulators, so
        // whichever is aggregated first is issued first (each accumulator
        // still sums its cells in plan order: deterministic).
        auto issue = [&](int g) {
          const uint32_t st = a_it + static_cast<uint32_t>(g);
          const uint32_t as = st % NSA;
          if (lane == 0) tev(st, 4);
          tc_fence_after();
          if (lane == 0) tev(st, 10);
          // descriptor start-address field is in 16-byte units
          const uint64_t ad = a_desc0 + ((as * 16384u) >> 4);
          const uint64_t bd = b_desc0 + ((ws * Cfg::wbytes) >> 4);
          if constexpr (SPLIT) {
            // main: Ah (tile K 0..31) x Wh into set q % nmain; corr: [Ah | Al]
            // x [Wl; Wh] into the last set.  Each set is initialised by its
            // first MMA of the item (first record).
            const int q = c * K + k;
            const int pm = q % nmain;
            const uint32_t dm = tmem + ab * Cfg::bstride + pm * Cfg::acc_cols + g * NOUT;
            const uint32_t dc = tmem + ab * Cfg::bstride + Cfg::nmain * Cfg::acc_cols + g * NOUT;
            const uint64_t bd2 = bd + (Cfg::wimg >> 4);
            if (elect_one()) {
#pragma unroll
              for (int ks = 0; ks < 2; ++ks)
                umma_bf16(dm, ad + 2u * ks, bd + 2u * ks, idesc, (!first || q >= nmain || ks > 0) ? 1u : 0u);
#pragma unroll
              for (int ks = 0; ks < 4; ++ks)
                umma_bf16(dc, ad + 2u * ks, bd2 + 2u * ks, idesc, (!first || q > 0 || ks > 0) ? 1u : 0u);
              umma_commit(bar(B_A_EMPTY + as));
            }
          } else {
            const uint32_t d = tmem + ab * Cfg::acc_cols + g * NOUT;
            if (elect_one()) {
#pragma unroll
              for (int ks = 0; ks < 4; ++ks)
                umma_bf16(d, ad + 2u * ks, bd + 2u * ks, idesc,
                          (!first || c > 0 || k > 0 || ks > 0) ? 1u : 0u);
              tev(st, 11);
              umma_commit(bar(B_A_EMPTY + as));
            }
          }
          __syncwarp();
          if (lane == 0) tev(st, 5);
        };
        if (nsub == 2) {
          uint32_t todo = 3u;
          while (todo) {
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              const uint32_t st = a_it + static_cast<uint32_t>(g);
              if ((todo >> g) & 1u)
                if (__any_sync(0xffffffffu, mbar_test(bar(B_A_FULL + st % NSA), (st / NSA) & 1))) {
                  issue(g);
                  todo &= ~(1u << g);
                }
            }
          }
        } else {
          for (int g = 0; g < nsub; ++g) {
            const uint32_t st = a_it + static_cast<uint32_t>(g);
            mbar_wait(bar(B_A_FULL + st % NSA), (st / NSA) & 1);
            issue(g);
          }
        }
        a_it += static_cast<uint32_t>(nsub);
        if (elect_one()) umma_commit(bar(B_W_EMPTY + ws));
        __syncwarp();
        if (lane == 0) tev(a_it - nsub, 12);
        ++w_it;
      }
      if (!last) continue;  // the next record of this item accumulates on
      if (elect_one()) umma_commit(bar(B_T_FULL + ab));
      __syncwarp();
      if (pending) release_epilogue();  // K == 1
      pending = true;
      pend_t = t_it;
      ++t_it;
      // single-buffered sets: the next item's first MMA waits for this epilogue
      if (NB == 1) release_epilogue();
    }
    if (pending) release_epilogue();
  } else if (warp >= FWD_AGG_WARP0) {
    // ------------------------------ aggregation ----------------------------
    const int aw = warp - FWD_AGG_WARP0;
    const int grp = aw / AGG_GROUP_WARPS, wig = aw % AGG_GROUP_WARPS;
    uint32_t a_it = 0;  // pipeline position of the current (record, chunk)'s first stage
    uint32_t h_it = 0;
    const uint32_t* hidx = reinterpret_cast<const uint32_t*>(gbase + L.hidx);
    for (int w = blockIdx.x; w < a.n_items; w += gridDim.x)
    for (int s = static_cast<int>(a.item_start[w]); s < static_cast<int>(a.item_start[w + 1]); ++s) {
      const uint2 sp = a.sup[s];
      const int nsub = static_cast<int>(sp.y & 0xFFu);
      const uint32_t H = a.halo_len[s];
      if (H == kOverflow) continue;
      for (int c = 0; c < nci; ++c) {
      named_bar_sync(1, 32 * FWD_AGG_WARPS);  // all aggregation warps done with the previous halo
      if (Cfg::hidx) {
        if (c == 0) mbar_wait(bar(B_HALO_FULL), h_it & 1);  // the record's row list is in smem
        coop_load_halo<32 * FWD_AGG_WARPS, true>(hidx, H, a.feat + c * CH, s_halo, 32 * aw + lane, fstride);
      } else {
        coop_load_halo<32 * FWD_AGG_WARPS>(a.halo + static_cast<int64_t>(s) * a.hcap, H, a.feat + c * CH,
                                           s_halo, 32 * aw + lane, fstride);
      }
      if (Cfg::hidx && c == nci - 1) {  // (all chunks loaded: the producer may fetch the next list)
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(B_HALO_EMPTY));
        ++h_it;
      }
      named_bar_sync(1, 32 * FWD_AGG_WARPS);
      // this group's stages of the (record, chunk): every AGG_GROUPS-th one
      // (stage index = pipeline position; slot / parity derive from it)
      const uint32_t n_st = static_cast<uint32_t>(K * nsub);
      const uint32_t first = a_it + ((static_cast<uint32_t>(grp) - a_it) & (AGG_GROUPS - 1));
      for (uint32_t j = first; j < a_it + n_st; j += AGG_GROUPS) {
        const uint32_t ds = j % NSDt, as = j % NSA;
        mbar_wait(bar(B_D_FULL + ds), (j / NSDt) & 1);
        if (wig == 0 && lane == 0) tev(j, 1);
        const uint8_t* slot = g_d + ds * BLOCK_MAX_BYTES;
        const uint32_t src = BIG ? dsrc[ds] : kFitsSlot;
        auto wait_a = [&] {
          mbar_wait(bar(B_A_EMPTY + as), ((j / NSA) & 1) ^ 1);
          if (wig == 0 && lane == 0) tev(j, 2);
        };
        if (src == kFitsSlot) {  // (separate instantiations keep shared-memory loads)
          aggregate_stage<AGG_GROUP_WARPS, SPLIT>(slot, reinterpret_cast<const uint16_t*>(slot + 512),
                                                  s_halo, s_a + as * 16384u, wig, lane, wait_a);
        } else {
          wait_a();
          aggregate_stage_l2<AGG_GROUP_WARPS, SPLIT>(
              slot, reinterpret_cast<const uint16_t*>(a.blocks + blk_bytes(src) + 512), s_halo,
              s_a + as * 16384u, wig, lane);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (wig == 0 && lane == 0) tev(j, 3);
        if constexpr (TRACE) if (lane == 0) trace_max(a.trace, j, 7);
        if (lane == 0) {
          mbar_arrive(bar(B_A_FULL + as));
          mbar_arrive(bar(B_D_EMPTY + ds));
        }
      }
      a_it += n_st;
      }
    }
  } else {
    // ------------------------------ epilogue (warps 0-3) -------------------
    const int e = warp;
    uint32_t t_it = 0;
    // SPLIT: 1 / (s_feat s_w) (exact powers of two)
    const float inv_scale = SPLIT ? 1.f / (split_scale(a.amax[0]) * split_scale(a.amax[1])) : 1.f;
    for (int w = blockIdx.x; w < a.n_items; w += gridDim.x) {
      const int s = static_cast<int>(a.item_start[w + 1]) - 1;  // last record: the rows
      const uint2 sp = a.sup[s];
      const int nsub = static_cast<int>(sp.y & 0xFFu);
      if (a.halo_len[s] == kOverflow) continue;
      const uint32_t ab = t_it % Cfg::nbuf;
      {  // warm L2 with the next item's halo while this one is aggregated
        const int s_next = w + static_cast<int>(gridDim.x) < a.n_items
                               ? static_cast<int>(a.item_start[w + gridDim.x]) : a.n_super;
        if (s_next < a.n_super && a.halo_len[s_next] != kOverflow)
          prefetch_halo_l2<128>(a.halo + static_cast<int64_t>(s_next) * a.hcap,
                                a.halo_len[s_next], a.feat, 32 * e + lane, fstride, nci);
      }
      named_bar_sync(2 + ab, 32 * 5);  // released by the MMA warp once T_FULL(tile) landed
      tc_fence_after();
      for (int g = 0; g < nsub; ++g) {
        const uint32_t t0 = tmem + (static_cast<uint32_t>(32 * e) << 16) + ab * Cfg::bstride + g * NOUT;
        const uint2 tl = a.tiles[sp.x + g];
        const int64_t row = static_cast<int64_t>(tl.x) + 32 * e + lane;
        float4* o = static_cast<uint32_t>(32 * e + lane) < tl.y
                        ? reinterpret_cast<float4*>(a.out + static_cast<int64_t>(a.perm_rows[row]) * a.out_stride +
                                                    a.out_col0)
                        : nullptr;
#pragma unroll 4
        for (int q = 0; q < NOUT / 16; ++q) {
          if (q * 16 >= a.ncols) break;
          uint32_t v[16];
          tmem_ld16(t0 + 16 * q, v);
          tmem_ld_wait();
          if constexpr (SPLIT) {
            // y = ((main_0 + main_1) + main_2) + corr 2^-11, all fp32 round-to-
            // nearest, then the exact power-of-two unscaling
            float f[16];
#pragma unroll
            for (int x = 0; x < 16; ++x) f[x] = __uint_as_float(v[x]);
            for (int pm = 1; pm < nmain; ++pm) {
              tmem_ld16(t0 + pm * Cfg::acc_cols + 16 * q, v);
              tmem_ld_wait();
#pragma unroll
              for (int x = 0; x < 16; ++x) f[x] += __uint_as_float(v[x]);
            }
            tmem_ld16(t0 + Cfg::nmain * Cfg::acc_cols + 16 * q, v);
            tmem_ld_wait();
#pragma unroll
            for (int x = 0; x < 16; ++x) v[x] = __float_as_uint(fmaf(__uint_as_float(v[x]), 0x1p-11f, f[x]) * inv_scale);
          }
          if (o)
#pragma unroll
            for (int x = 0; x < 4; ++x)
              o[q * 4 + x] = make_float4(__uint_as_float(v[4 * x]), __uint_as_float(v[4 * x + 1]),
                                         __uint_as_float(v[4 * x + 2]), __uint_as_float(v[4 * x + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(B_T_EMPTY + ab));
      ++t_it;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_free<Cfg::tmem_cols>(tmem);
}

// ===========================================================================
// weight-gradient kernel over the forward plan's super-tiles
//   D_pair[(2 cells x 64 c_in) x NOUT c_out] += A_pair^T (MN-major) x G_tile (MN-major)
// Work items are (cell, 64-wide C_in chunk) A tiles; blockIdx.y selects a
// chunk and a run of 2 x WgCfg::pairs cells, whose pair accumulators stay in
// TMEM for the whole sweep (NOUT columns each).
// ===========================================================================
struct WgArgs {
  const uint32_t* halo;
  const uint32_t* halo_len;
  const uint32_t* blk_off;
  const uint8_t* blocks;
  const uint2* sup;            // per super-tile {first sub-tile, sub-tiles}
  const uint2* tiles;          // per sub-tile {first permuted row, rows}
  int64_t n_rows;
  int n_sub, n_super, st, hcap, K;  // the forward plan's super-tiles (st sub-tiles share a halo)
  int nci, gpc;                // C_in chunks; cell groups per chunk (blockIdx.y = c * gpc + group)
  const __nv_bfloat16* feat;   // bf16 F_in (n_cols, 64 nci), permuted
  const __nv_bfloat16* dense;  // bf16 G_out (n_rows, NOUT), permuted (row = sub-tile order)
  int dense_stride;            // elements per dense row (NOUT, or the whole width for a half)
  float* partial;              // [gridDim.x][K][64 nci c][NOUT m]
  uint8_t korder[KMAX];        // run slot -> kernel cell (runs of 2 x pairs slots, load-balanced)
  int seg;                     // SPLIT: super-tiles per accumulation segment (bounded chains)
};

constexpr int WG_THREADS = 32 * (FWD_AGG_WARP0 + FWD_AGG_WARPS);
constexpr int WG_PAIRS = 7;      // cell pairs per CTA (cell group = 14 cells)
constexpr int WG_NSA = 2;        // A pair stages (32 KB)
constexpr int WG_NSD = 4;        // descriptor slots (2 blocks each; a multiple of WG_GROUPS)
constexpr int WG_NSG = 2;        // dense G sub-tile slots (NOUT x 256 B; 1 for NOUT >= 128;
                                 // at 256 as two 64-row halves with their own barriers)
constexpr int WG_GROUPS = 2;     // stage (cell pair) s is aggregated by warp group s % 2

template <int NOUT>
struct WgCfg {
  static constexpr int pairs = NOUT == 64 ? WG_PAIRS : 512 / NOUT;  // TMEM: pairs x NOUT columns
  static constexpr int nsg = NOUT == 64 ? WG_NSG : 1;
  static constexpr int nsd = WG_NSD;
  static constexpr uint32_t gbytes = NOUT * 256;  // 128 rows x NOUT bf16, 64-column blocks
};
struct WgSmem {
  uint32_t halo, a, gt, d, bar, tmem_slot, offs;
  size_t total;
};
template <int NOUT>
__host__ __device__ constexpr WgSmem wg_smem_layout(int hcap) {
  WgSmem L{};
  uint32_t o = 0;
  L.halo = o;
  o += hcap * 128;
  o = (o + 1023) & ~1023u;
  L.a = o;
  o += WG_NSA * 32768;
  L.gt = o;
  o += WgCfg<NOUT>::nsg * WgCfg<NOUT>::gbytes;
  L.d = o;
  o += WgCfg<NOUT>::nsd * 2 * BLOCK_MAX_BYTES;
  o = (o + 7) & ~7u;
  L.bar = o;
  o += 24 * 8;
  L.tmem_slot = o;
  o += 16;
  L.offs = o;
  o += OFFS_WORDS * 4;  // block offsets of the super-tile, then the slot sources
  L.total = o + 1024;
  return L;
}

enum : int {
  W_HALO_FULL = 0,
  W_HALO_EMPTY = 1,
  W_A_FULL = 2,                    // WG_NSA
  W_A_EMPTY = W_A_FULL + WG_NSA,   // WG_NSA
  W_D_FULL = W_A_EMPTY + WG_NSA,   // WG_NSD
  W_D_EMPTY = W_D_FULL + WG_NSD,   // WG_NSD
  W_G_FULL = W_D_EMPTY + WG_NSD,   // WG_NSG
  W_G_EMPTY = W_G_FULL + WG_NSG,   // WG_NSG
  W_DONE = W_G_EMPTY + WG_NSG,
  W_SEG_FULL = W_DONE + 1,   // SPLIT: a segment's MMAs completed
  W_SEG_EMPTY = W_SEG_FULL + 1,  // SPLIT: its accumulators were flushed
  W_COUNT = W_SEG_EMPTY + 1
};
static_assert(W_COUNT <= 24, "wgrad barrier region");

static_assert(WG_NSD % WG_GROUPS == 0, "descriptor slots per group");
static_assert(wg_smem_layout<64>(FWD_HCAP).total <= 232448, "smem");
static_assert(wg_smem_layout<128>(FWD_HCAP).total <= 232448, "smem");
static_assert(wg_smem_layout<256>(FWD_HCAP1).total <= 232448, "smem");

// SPLIT (fp32-contract path): A tiles from the split F_in image (32 channels
// per chunk as [hi | lo], so an A_k^T pair is [Ah; Al] x 2 cells) against the
// split G_out image ([Gh | Gl] per 32 channels, NOUT = 2 x C_out): the four
// products (Ah+Al)^T (Gh+Gl) land in separate accumulator quadrants and the
// reduction adds them.
template <int NOUT, bool BIG, bool SPLIT = false>
__global__ void __launch_bounds__(WG_THREADS, 1) k_conv_wgrad_tc(WgArgs a) {
  using Cfg = WgCfg<NOUT>;
  constexpr int NP = Cfg::pairs, NSG = Cfg::nsg, WNSD = Cfg::nsd;
  // NOUT = 256 (one G slot, two pairs = the two A slots): the slot's 64-row
  // halves (MMA k-steps 0-3 / 4-7; loader warps 0-1 / 2-3) are filled and
  // released separately, so the next sub-tile's first half loads while the
  // MMAs consume the second (NOUT = 128 has four pairs for two A slots)
  constexpr bool GH = NOUT == 256;
  static_assert(!GH || (NSG == 1 && NP <= WG_NSA), "G halves: every pair's A slot held across both halves");
  constexpr uint32_t GB = Cfg::gbytes;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const WgSmem L = wg_smem_layout<NOUT>(a.hcap);
  const uint32_t s_halo = base + L.halo, s_a = base + L.a, s_g = base + L.gt, s_d = base + L.d;
  const uint32_t s_bar = base + L.bar;
  auto bar = [&](int i) { return s_bar + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + L.tmem_slot);
  const uint8_t* g_d = gbase + L.d;
  uint32_t* dsrc = reinterpret_cast<uint32_t*>(gbase + L.offs) + OFFS_DSRC;  // per descriptor half-slot

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K;
  const int chunk = blockIdx.y / a.gpc;      // C_in chunk
  const int k_begin = (blockIdx.y % a.gpc) * 2 * NP;  // first cell of this CTA
  const int n_pairs = max(0, min(NP, (K - k_begin + 1) / 2));
  const int64_t fstride = static_cast<int64_t>(a.nci) * CH;
  if (threadIdx.x == 0) {
    mbar_init(bar(W_HALO_FULL), 1);
    mbar_init(bar(W_HALO_EMPTY), FWD_AGG_WARPS);
    for (int i = 0; i < WG_NSA; ++i) {
      mbar_init(bar(W_A_FULL + i), FWD_AGG_WARPS / WG_GROUPS);
      mbar_init(bar(W_A_EMPTY + i), 1);
    }
    for (int i = 0; i < WNSD; ++i) {
      mbar_init(bar(W_D_FULL + i), 1);
      mbar_init(bar(W_D_EMPTY + i), FWD_AGG_WARPS / WG_GROUPS);
    }
    for (int i = 0; i < WG_NSG; ++i) {
      mbar_init(bar(W_G_FULL + i), GH ? 2 : 4);
      mbar_init(bar(W_G_EMPTY + i), 1);
    }
    mbar_init(bar(W_DONE), 1);
    mbar_init(bar(W_SEG_FULL), 1);
    mbar_init(bar(W_SEG_EMPTY), 4);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // producer: halo + descriptor blocks (two cells per stage)
    uint32_t* offs = reinterpret_cast<uint32_t*>(gbase + L.offs);
    uint32_t d_it = 0;
    for (int s = blockIdx.x; s < a.n_super; s += gridDim.x) {
      if (a.halo_len[s] == kOverflow) continue;
      const uint2 sp = a.sup[s];
      const int nsub = static_cast<int>(sp.y & 0xFFu);
      for (int x = lane; x <= nsub * K; x += 32)
        offs[x] = a.blk_off[static_cast<int64_t>(sp.x) * K + x];
      __syncwarp();
      for (int g = 0; g < nsub; ++g)
      for (int p = 0; p < n_pairs; ++p) {
        if (lane == 0) {
          const uint32_t ds = d_it % WNSD;
          mbar_wait(bar(W_D_EMPTY + ds), ((d_it / WNSD) & 1) ^ 1);
          const int ka = g * K + a.korder[k_begin + 2 * p];
          const bool two = k_begin + 2 * p + 1 < K;
          const int kb = two ? g * K + a.korder[k_begin + 2 * p + 1] : ka;
          const uint32_t o0 = offs[ka], e0 = offs[ka + 1];
          const uint32_t o1 = offs[kb], e1 = two ? offs[kb + 1] : o1;
          const uint32_t n0 = min((e0 - o0) << 4, static_cast<uint32_t>(BLOCK_MAX_BYTES));
          const uint32_t n1 = min((e1 - o1) << 4, static_cast<uint32_t>(BLOCK_MAX_BYTES));
          if (BIG) {
            dsrc[2 * ds] = (e0 - o0) << 4 > static_cast<uint32_t>(BLOCK_MAX_BYTES) ? o0 : kFitsSlot;
            dsrc[2 * ds + 1] = (e1 - o1) << 4 > static_cast<uint32_t>(BLOCK_MAX_BYTES) ? o1 : kFitsSlot;
          }
          mbar_expect_tx(bar(W_D_FULL + ds), n0 + n1);
          bulk_g2s(s_d + ds * 2 * BLOCK_MAX_BYTES, a.blocks + blk_bytes(o0), n0, bar(W_D_FULL + ds));
          if (n1)
            bulk_g2s(s_d + ds * 2 * BLOCK_MAX_BYTES + BLOCK_MAX_BYTES, a.blocks + blk_bytes(o1), n1,
                     bar(W_D_FULL + ds));
        }
        ++d_it;
      }
      __syncwarp();
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idesc = SPLIT ? idesc_f16(128, NOUT, true, true) : idesc_bf16(128, NOUT, true, true);
      uint32_t a_it = 0, g_it = 0;
      bool first = true;
      int in_seg = 0;        // SPLIT: super-tiles in the current accumulation segment
      uint32_t seg_it = 0;
      for (int s = blockIdx.x; s < a.n_super; s += gridDim.x) {
        if (a.halo_len[s] == kOverflow) continue;
        const uint2 sp = a.sup[s];
        const int nsub = static_cast<int>(sp.y & 0xFFu);
        if (SPLIT && in_seg == a.seg) {
          // the tensor core's fp32 accumulation truncates: a segment's sums
          // are handed to the epilogue warps (fp32 round-to-nearest adds into
          // the CTA's partial) and the accumulators restart
          umma_commit(bar(W_SEG_FULL));
          mbar_wait(bar(W_SEG_EMPTY), seg_it & 1);
          tc_fence_after();
          ++seg_it;
          in_seg = 0;
          first = true;
        }
        ++in_seg;
        for (int g = 0; g < nsub; ++g) {
        if (GH) {
          for (int h = 0; h < 2; ++h) {
            mbar_wait(bar(W_G_FULL + h), g_it & 1);
            tc_fence_after();
            for (int p = 0; p < n_pairs; ++p) {
              const uint32_t as = (a_it + p) % WG_NSA;
              if (h == 0) {
                mbar_wait(bar(W_A_FULL + as), ((a_it + p) / WG_NSA) & 1);
                tc_fence_after();
              }
              const uint32_t d = tmem + p * NOUT;
#pragma unroll
              for (int ks = 4 * h; ks < 4 * h + 4; ++ks) {
                const uint64_t ad = sdesc_sw128(s_a + as * 32768u + 2048u * ks, 16384, 1024);
                const uint64_t bd = sdesc_sw128(s_g + 2048u * ks, 16384, 1024);
                umma_bf16(d, ad, bd, idesc, (first && ks == 0) ? 0u : 1u);
              }
              if (h == 1) umma_commit(bar(W_A_EMPTY + as));
            }
            umma_commit(bar(W_G_EMPTY + h));
          }
          a_it += n_pairs;
          first = false;
          ++g_it;
          continue;
        }
        const uint32_t gs = g_it % NSG;
        mbar_wait(bar(W_G_FULL + gs), (g_it / NSG) & 1);
        for (int p = 0; p < n_pairs; ++p) {
          const uint32_t as = a_it % WG_NSA;
          mbar_wait(bar(W_A_FULL + as), (a_it / WG_NSA) & 1);
          tc_fence_after();
          const uint32_t d = tmem + p * NOUT;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            // K = points: 16 rows per step (2 x 8-row groups of 1024 B)
            const uint64_t ad = sdesc_sw128(s_a + as * 32768u + 2048u * ks, 16384, 1024);
            const uint64_t bd = sdesc_sw128(s_g + gs * GB + 2048u * ks, 16384, 1024);
            umma_bf16(d, ad, bd, idesc, (first && ks == 0) ? 0u : 1u);
          }
          umma_commit(bar(W_A_EMPTY + as));
          ++a_it;
        }
        first = false;
        umma_commit(bar(W_G_EMPTY + gs));
        ++g_it;
        }
      }
      umma_commit(bar(W_DONE));
    }
    __syncwarp();
  } else if (warp >= FWD_AGG_WARP0) {
    const int aw = warp - FWD_AGG_WARP0;
    const int grp = aw / (FWD_AGG_WARPS / WG_GROUPS), wig = aw % (FWD_AGG_WARPS / WG_GROUPS);
    uint32_t a_it = 0, d_it = 0;
    for (int s = blockIdx.x; s < a.n_super; s += gridDim.x) {
      const uint32_t H = a.halo_len[s];
      if (H == kOverflow) continue;
      const uint2 sp = a.sup[s];
      const int nsub = static_cast<int>(sp.y & 0xFFu);
      named_bar_sync(1, 32 * FWD_AGG_WARPS);
      coop_load_halo<32 * FWD_AGG_WARPS>(a.halo + static_cast<int64_t>(s) * a.hcap, H,
                                         a.feat + chunk * CH, s_halo, 32 * aw + lane, fstride);
      named_bar_sync(1, 32 * FWD_AGG_WARPS);
      for (int g = 0; g < nsub; ++g)
      for (int p = 0; p < n_pairs; ++p) {
        if (static_cast<int>(a_it % WG_GROUPS) == grp) {
          const uint32_t ds = d_it % WNSD, as = a_it % WG_NSA;
          mbar_wait(bar(W_D_FULL + ds), (d_it / WNSD) & 1);
          const int ncell = (k_begin + 2 * p + 1 < K) ? 2 : 1;
          bool waited = false;
          auto wait_a = [&] {
            if (!waited) mbar_wait(bar(W_A_EMPTY + as), ((a_it / WG_NSA) & 1) ^ 1);
            waited = true;
          };
          // the group's warps split in two teams, one per cell of the pair
          constexpr int TW = FWD_AGG_WARPS / WG_GROUPS / 2;
          const int half = wig / TW, wq = wig % TW;
          if (half < ncell) {
            const uint8_t* slot = g_d + ds * 2 * BLOCK_MAX_BYTES + half * BLOCK_MAX_BYTES;
            const uint32_t src = BIG ? dsrc[2 * ds + half] : kFitsSlot;
            if (src == kFitsSlot)
              aggregate_stage<TW, SPLIT>(slot, reinterpret_cast<const uint16_t*>(slot + 512), s_halo,
                                         s_a + as * 32768u + half * 16384u, wq, lane, wait_a);
            else if ((wait_a(), true))
              aggregate_stage_l2<TW, SPLIT>(
                  slot, reinterpret_cast<const uint16_t*>(a.blocks + blk_bytes(src) + 512), s_halo,
                  s_a + as * 32768u + half * 16384u, wq, lane);
          } else {
            wait_a();
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(bar(W_A_FULL + as));
            mbar_arrive(bar(W_D_EMPTY + ds));
          }
        }
        ++a_it;
        ++d_it;
      }
    }
  } else {
    // warps 0-3: dense G tile loader during the sweep, epilogue at the end
    // (SPLIT: also at every segment end), TMEM lanes 32e..32e+31 of each pair
    // accumulator -> the CTA's partial (SPLIT: added, fp32 round-to-nearest)
    const int e = warp;
    auto flush = [&](bool add) {
      tc_fence_after();
      for (int p = 0; p < n_pairs; ++p) {
        const uint32_t t0 = tmem + (static_cast<uint32_t>(32 * e) << 16) + p * NOUT;
        const int ks = k_begin + 2 * p + (e >> 1);
        const int k = ks < K ? a.korder[ks] : K;
        const int c = chunk * CH + 32 * (e & 1) + lane;
        float4* o = k < K ? reinterpret_cast<float4*>(
                                a.partial + ((static_cast<int64_t>(blockIdx.x) * K + k) * fstride + c) * NOUT)
                          : nullptr;
#pragma unroll 4
        for (int q = 0; q < NOUT / 16; ++q) {
          uint32_t v[16];
          tmem_ld16(t0 + 16 * q, v);
          tmem_ld_wait();
          if (o)
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              float4 r = make_float4(__uint_as_float(v[4 * x]), __uint_as_float(v[4 * x + 1]),
                                     __uint_as_float(v[4 * x + 2]), __uint_as_float(v[4 * x + 3]));
              if (add) {
                const float4 b = o[q * 4 + x];
                r.x += b.x;
                r.y += b.y;
                r.z += b.z;
                r.w += b.w;
              }
              o[q * 4 + x] = r;
            }
        }
      }
      tc_fence_before();
    };
    uint32_t g_it = 0;
    int in_seg = 0;
    uint32_t seg_it = 0;
    for (int s = blockIdx.x; s < a.n_super; s += gridDim.x) {
      if (a.halo_len[s] == kOverflow) continue;
      const uint2 sp = a.sup[s];
      const int nsub = static_cast<int>(sp.y & 0xFFu);
      if (SPLIT && in_seg == a.seg) {  // mirror of the MMA warp's segment
        mbar_wait(bar(W_SEG_FULL), seg_it & 1);
        flush(true);
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(W_SEG_EMPTY));
        ++seg_it;
        in_seg = 0;
      }
      ++in_seg;
      {
        const int s_next = s + gridDim.x;
        if (s_next < a.n_super && a.halo_len[s_next] != kOverflow)
          prefetch_halo_l2<128>(a.halo + static_cast<int64_t>(s_next) * a.hcap,
                                a.halo_len[s_next], a.feat + chunk * CH, 32 * warp + lane, fstride);
      }
      for (int g = 0; g < nsub; ++g) {
        const uint32_t gs = g_it % NSG, gu = GH ? (warp >> 1) : gs;  // barrier unit
        // a single G slot (NOUT >= 128) puts this wait on the MMA's critical path
        if (NSG == 1)
          mbar_wait(bar(W_G_EMPTY + gu), (g_it & 1) ^ 1);
        else
          mbar_wait_sleep(bar(W_G_EMPTY + gs), ((g_it / NSG) & 1) ^ 1);
        // 128 rows x NOUT/64 blocks x 8 chunks of 16 B; warp e copies rows 32e..32e+31
        // with cp.async (all of a lane's copies in flight; rows past the tile zero-filled)
        const uint32_t gt = s_g + gs * GB;
        const uint2 tl = a.tiles[sp.x + g];
#pragma unroll 8
        for (int x = lane; x < 32 * 8 * (NOUT / 64); x += 32) {
          const int j = x >> 8, r = 32 * warp + ((x >> 3) & 31), q = x & 7;
          const bool in = static_cast<uint32_t>(r) < tl.y;
          const int64_t row = static_cast<int64_t>(tl.x) + (in ? r : 0);
          cp_async16_zfill(gt + j * 16384 + r * 128 + (((q ^ (r & 7)) & 7) << 4),
                           reinterpret_cast<const uint4*>(a.dense + row * a.dense_stride) + j * 8 + q, in ? 16u : 0u);
        }
        cp_async_wait_all();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(W_G_FULL + gu));
        ++g_it;
      }
    }
    // epilogue: the last (or only) segment
    mbar_wait_sleep(bar(W_DONE), 0);
    if (g_it > 0) flush(SPLIT);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_free<512>(tmem);
}

// grad_w[k][m][c] = sum over CTAs x (fixed order) of partial[x][k][c][m]
__global__ void k_wgrad_reduce(const float* __restrict__ partial, int n_part, int K, int cin,
                               int cout, int cinp, int coutp, float* __restrict__ grad_w) {
  // thread = (k, c, m) with m fastest: the partial reads are coalesced (the
  // large side); the transposed grad_w stores are the small side
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(K) * cin * cout) return;
  const int k = static_cast<int>(idx / (cin * cout)), c = static_cast<int>((idx / cout) % cin),
            m = static_cast<int>(idx % cout);
  float s = 0.f;
  for (int x = 0; x < n_part; ++x)
    s += partial[((static_cast<int64_t>(x) * K + k) * cinp + c) * coutp + m];
  grad_w[(static_cast<int64_t>(k) * cout + m) * cin + c] = s;
}

// Split variant: partial[x][k][c'][m'] over split channels (c' = 64 (c / 32) +
// c % 32 for the hi half, + 32 for the scaled lo half; same for m');
// grad_w[k][m][c] = [sum over CTAs (fixed order) of hh + (hl + lh) 2^-11 +
// ll 2^-22] / (s_F s_G).
// (m0, cout_all: this partial holds output channels [m0, m0 + cout) of cout_all)
__global__ void k_wgrad_reduce_split(const float* __restrict__ partial, int n_part, int K, int cin,
                                     int cout, int cinp2, int coutp2, const uint32_t* __restrict__ amax_f,
                                     const uint32_t* __restrict__ amax_g, float* __restrict__ grad_w,
                                     int m0, int cout_all) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(K) * cin * cout) return;
  const int k = static_cast<int>(idx / (cin * cout)), c = static_cast<int>((idx / cout) % cin),
            m = static_cast<int>(idx % cout);
  const int ch = 64 * (c >> 5) + (c & 31), mh = 64 * (m >> 5) + (m & 31);
  float hh = 0.f, cr = 0.f, ll = 0.f;
  for (int x = 0; x < n_part; ++x) {
    const float* b = partial + (static_cast<int64_t>(x) * K + k) * cinp2 * coutp2;
    const float* rh = b + static_cast<int64_t>(ch) * coutp2;
    const float* rl = rh + 32 * coutp2;
    hh += rh[mh];
    cr += rh[mh + 32] + rl[mh];
    ll += rl[mh + 32];
  }
  const float inv = 1.f / (split_scale(*amax_f) * split_scale(*amax_g));
  grad_w[(static_cast<int64_t>(k) * cout_all + m0 + m) * cin + c] =
      (hh + fmaf(ll, 0x1p-11f, cr) * 0x1p-11f) * inv;
}

// ===========================================================================
// fused backward (bf16 operands, C_in, C_out <= 64, K = 27): the input
// gradient and the weight gradient from ONE aggregation pass.  Over the
// transposed plan (rows = input points j, 128-row super-tiles),
//     B_k[j] = sum_{i : (i, j, k)} G_out[i]
// is aggregated once per (tile, cell) and feeds both
//     grad_in[j] += B_k[j] W_k^T          (M128 N64 K64 into a TMEM accumulator)
//     dW_k       += B_k^T F_in[tile]      (vvor.hpp:79-84: two cells' A slots
//                                          stacked to M = 128 as an MN-major A
//                                          operand, the tile's dense F_in rows as
//                                          the MN-major B operand, K = 128 rows)
// (the weight-gradient MMA is M = 64: its accumulator takes lanes 0-15 of each
// 32-lane TMEM quadrant, or lanes 16-31 with a lane offset of 16 in the D
// address -- tools/micro/mma_m64.cu -- so two cells share 64 columns and every
// stage's MMAs release its A slot at once).  dW of 27 cells (442 KB fp32)
// exceeds one SM's TMEM, so the two CTAs of a cluster take the same
// super-tiles and half of the cells each (14 / 13); each keeps 7 column blocks
// of two cells (448 columns) + the 64-column input-gradient accumulator.
// The two halves' input-gradient sums meet in global memory: grad_in is zeroed
// and each CTA adds its sum once with red.global.add.v4.f32 (0 + a + b equals
// 0 + b + a in fp32: deterministic).  (BF_FLAGS=1: the half-0 CTA stores its
// sum and publishes a per-(item, quadrant) flag, the half-1 CTA adds after
// seeing it -- no zero fill, but measured slower: the halves wait on each
// other.)  Per-pair dW partials are reduced in a fixed order.
// ===========================================================================
constexpr int BF_STAGES = 14;      // at most this many stages (cells) per record and CTA
constexpr uint8_t BF_ZERO = 0xFF;  // no cell (the 13-cell half's 14th entry)
constexpr int NSF = 2;             // F tiles (16 KB: 128 rows x 64 channels, SW128)
// Slot counts of the fused kernel (the M = 64 weight-gradient MMAs need no
// slot pairing; -DBF_NSA_=.. etc. for A/B builds).
#ifndef BF_NSA_
#define BF_NSA_ 4
#endif
#ifndef BF_NSW_
#define BF_NSW_ 3
#endif
#ifndef BF_NSD_
#define BF_NSD_ 8
#endif
constexpr int BF_NSA = BF_NSA_, BF_NSW = BF_NSW_, BF_NSD = BF_NSD_;
#ifndef BF_FLAGS
#define BF_FLAGS 0  // 1: half 0 stores, half 1 adds after its flag (A/B: slower); 0: grad_in zeroed, both add
#endif
static_assert(BF_NSD % AGG_GROUPS == 0, "descriptor slots per group");
enum : int {
  BB_HALO_FULL = 0,
  BB_HALO_EMPTY = 1,
  BB_A_FULL = 2,
  BB_A_EMPTY = BB_A_FULL + BF_NSA,
  BB_W_FULL = BB_A_EMPTY + BF_NSA,
  BB_W_EMPTY = BB_W_FULL + BF_NSW,
  BB_D_FULL = BB_W_EMPTY + BF_NSW,
  BB_D_EMPTY = BB_D_FULL + BF_NSD,
  BB_T_FULL = BB_D_EMPTY + BF_NSD,
  BB_T_EMPTY = BB_T_FULL + 1,
  BB_F_FULL = BB_T_EMPTY + 1,
  BB_F_EMPTY = BB_F_FULL + NSF,
  BB_MMA_DONE = BB_F_EMPTY + NSF,
  BB_COUNT = BB_MMA_DONE + 1
};
static_assert(BB_COUNT <= 48, "barrier region");

struct BfArgs {
  const uint32_t* halo;
  const uint32_t* halo_len;
  const uint32_t* blk_off;
  const uint8_t* blocks;
  const uint32_t* perm_rows;  // perm_in: permuted row -> input point
  const uint2* sup;
  const uint2* tiles;
  const uint32_t* item_start;
  int n_items, hcap, K;
  const __nv_bfloat16* feat;  // bf16 G_out image (perm_out order): the gathered rows
  const __nv_bfloat16* fimg;  // bf16 F_in image (perm_in order): the tiles' dense rows
  const uint8_t* wpack;       // K images of W_k^T (64 x 128 B)
  float* gin;                 // (n_in, cin) original order
  int gin_cols;               // cin
  uint32_t* item_flag;        // [n_items][4]: the half-0 CTA stored the item's rows (quadrant e)
  uint32_t gen;               // this launch's flag value (flags are never reset)
  float* partial;             // [pairs][K][64 m][64 c]
  long long* prof;            // NPCG_BF_PROFILE: per CTA {halo-boundary clocks, aggregation-loop clocks}
  uint8_t cells[2 * BF_STAGES];  // per half: stage -> cell (BF_ZERO: none)
};

struct BfSmem {
  uint32_t halo, a, w, d, f, bar, tmem_slot, offs, hidx;
  size_t total;
};
__host__ __device__ constexpr BfSmem bf_smem_layout(int hcap) {
  BfSmem L{};
  uint32_t o = 0;
  L.halo = o;
  o += hcap * 128;
  o = (o + 1023) & ~1023u;
  L.a = o;
  o += BF_NSA * 16384;
  L.f = o;
  o += NSF * 16384;
  L.w = o;
  o += BF_NSW * 8192;
  L.d = o;
  o += BF_NSD * BLOCK_MAX_BYTES;
  o = (o + 7) & ~7u;
  L.bar = o;
  o += 48 * 8;
  L.tmem_slot = o;
  o += 16;
  L.offs = o;
  o += OFFS_WORDS * 4;
  o = (o + 15) & ~15u;
  L.hidx = o;  // the record's halo row list (bulk-copied ahead by the descriptor producer)
  o += ((hcap * 4 + 15) & ~15);
  L.total = o + 1024;
  return L;
}
static_assert(bf_smem_layout(FWD_HCAP1).total <= 232448, "smem");

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <bool BIG>
__global__ void __launch_bounds__(FWD_THREADS, 1) k_conv_bwd_fused(BfArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const BfSmem L = bf_smem_layout(a.hcap);
  const uint32_t s_halo = base + L.halo, s_a = base + L.a, s_w = base + L.w, s_d = base + L.d,
                 s_f = base + L.f, s_hidx = base + L.hidx;
  const uint32_t s_bar = base + L.bar;
  auto bar = [&](int i) { return s_bar + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + L.tmem_slot);
  const uint8_t* g_d = gbase + L.d;
  uint32_t* dsrc = reinterpret_cast<uint32_t*>(gbase + L.offs) + OFFS_DSRC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = static_cast<int>(cluster_ctarank());
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const uint8_t* cells = a.cells + half * BF_STAGES;
  int nst = 0;  // stages per record of this half
  while (nst < BF_STAGES && cells[nst] != BF_ZERO) ++nst;
  const int K = a.K;
  if (threadIdx.x == 0) {
    mbar_init(bar(BB_HALO_FULL), 1);
    mbar_init(bar(BB_HALO_EMPTY), FWD_AGG_WARPS);
    for (int i = 0; i < BF_NSA; ++i) {
      mbar_init(bar(BB_A_FULL + i), AGG_GROUP_WARPS);
      mbar_init(bar(BB_A_EMPTY + i), 1);
    }
    for (int i = 0; i < BF_NSW; ++i) {
      mbar_init(bar(BB_W_FULL + i), 1);
      mbar_init(bar(BB_W_EMPTY + i), 1);
    }
    for (int i = 0; i < BF_NSD; ++i) {
      mbar_init(bar(BB_D_FULL + i), 1);
      mbar_init(bar(BB_D_EMPTY + i), AGG_GROUP_WARPS);
    }
    mbar_init(bar(BB_T_FULL), 1);
    mbar_init(bar(BB_T_EMPTY), 4);
    for (int i = 0; i < NSF; ++i) {
      mbar_init(bar(BB_F_FULL + i), 4);
      mbar_init(bar(BB_F_EMPTY + i), 1);
    }
    mbar_init(bar(BB_MMA_DONE), 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ------------------------ producer: stage descriptors ---------------------
    uint32_t* offs = reinterpret_cast<uint32_t*>(gbase + L.offs);
    uint32_t d_it = 0, h_it = 0;
    for (int w = pair; w < a.n_items; w += npairs)
      for (int s = static_cast<int>(a.item_start[w]); s < static_cast<int>(a.item_start[w + 1]); ++s) {
        if (a.halo_len[s] == kOverflow) continue;
        if (lane == 0) {  // the record's halo row list into shared memory (agg warps release it)
          const uint32_t hb = (a.halo_len[s] * 4u + 15u) & ~15u;
          mbar_wait(bar(BB_HALO_EMPTY), (h_it & 1) ^ 1);
          mbar_expect_tx(bar(BB_HALO_FULL), hb);
          if (hb) bulk_g2s(s_hidx, a.halo + static_cast<int64_t>(s) * a.hcap, hb, bar(BB_HALO_FULL));
        }
        ++h_it;
        const uint2 sp = a.sup[s];
        const int64_t ob = static_cast<int64_t>(sp.x) * K;
        for (int x = lane; x <= K; x += 32) offs[x] = a.blk_off[ob + x];
        __syncwarp();
        for (int ci = 0; ci < nst; ++ci) {
          if (lane == 0) {
            const uint32_t ds = d_it % BF_NSD;
            mbar_wait(bar(BB_D_EMPTY + ds), ((d_it / BF_NSD) & 1) ^ 1);
            const int k = cells[ci];
            const uint32_t o0 = offs[k], o1 = offs[k + 1];
            const uint32_t nb = min((o1 - o0) << 4, static_cast<uint32_t>(BLOCK_MAX_BYTES));
            if (BIG) dsrc[ds] = (o1 - o0) << 4 > static_cast<uint32_t>(BLOCK_MAX_BYTES) ? o0 : kFitsSlot;
            mbar_expect_tx(bar(BB_D_FULL + ds), nb);
            bulk_g2s(s_d + ds * BLOCK_MAX_BYTES, a.blocks + blk_bytes(o0), nb, bar(BB_D_FULL + ds));
          }
          ++d_it;
        }
        __syncwarp();
      }
  } else if (warp == FWD_W_WARP) {
    // ------------------------ producer: W_k^T per record and stage ------------
    if (lane == 0) {
      uint32_t w_it = 0;
      for (int w = pair; w < a.n_items; w += npairs)
        for (int s = static_cast<int>(a.item_start[w]); s < static_cast<int>(a.item_start[w + 1]); ++s) {
          if (a.halo_len[s] == kOverflow) continue;
          for (int ci = 0; ci < nst; ++ci) {
            const int k = cells[ci];
            const uint32_t ws = w_it % BF_NSW;
            mbar_wait_sleep(bar(BB_W_EMPTY + ws), ((w_it / BF_NSW) & 1) ^ 1);
            mbar_expect_tx(bar(BB_W_FULL + ws), 8192u);
            bulk_g2s(s_w + ws * 8192u, a.wpack + static_cast<int64_t>(k) * 8192, 8192u, bar(BB_W_FULL + ws));
            ++w_it;
          }
        }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------ MMA issuer --------------------------------
    constexpr uint32_t idesc_d = idesc_bf16(128, 64, false, false);  // B_k x W_k^T
    constexpr uint32_t idesc_w = idesc_bf16(64, 64, true, true);     // B_k^T x F (M = 64)
    const uint64_t a_desc0 = sdesc_sw128(s_a, 16, 1024), b_desc0 = sdesc_sw128(s_w, 16, 1024);
    uint32_t w_it = 0, a_it = 0, t_it = 0, f_it = 0;
    bool dw_fresh = true;  // the pair accumulators' first MMA (per CTA)
    for (int w = pair; w < a.n_items; w += npairs)
      for (int s = static_cast<int>(a.item_start[w]); s < static_cast<int>(a.item_start[w + 1]); ++s) {
        const uint2 sp = a.sup[s];
        if (a.halo_len[s] == kOverflow) continue;
        const bool first = (sp.y & SUP_FIRST) != 0, last = (sp.y & SUP_LAST) != 0;
        // single-buffered input-gradient accumulator: the previous item drained
        if (first) mbar_wait(bar(BB_T_EMPTY), (t_it & 1) ^ 1);
        const uint32_t fs = f_it % NSF;
        mbar_wait(bar(BB_F_FULL + fs), (f_it / NSF) & 1);
        tc_fence_after();
        for (int ci = 0; ci < nst; ++ci) {
          const uint32_t ws = w_it % BF_NSW;
          mbar_wait(bar(BB_W_FULL + ws), (w_it / BF_NSW) & 1);
          const uint32_t st = a_it + static_cast<uint32_t>(ci);
          const uint32_t as = st % BF_NSA;
          mbar_wait(bar(BB_A_FULL + as), (st / BF_NSA) & 1);
          tc_fence_after();
          const uint64_t ad = a_desc0 + ((as * 16384u) >> 4);
          const uint64_t bd = b_desc0 + ((ws * 8192u) >> 4);
          // cell stage ci: column block ci / 2, lanes 0-15 / 16-31 of each quadrant
          const uint32_t dw = tmem + 64u + 64u * static_cast<uint32_t>(ci >> 1) + ((ci & 1) ? (16u << 16) : 0u);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              umma_bf16(tmem, ad + 2u * ks, bd + 2u * ks, idesc_d, (!first || ci > 0 || ks > 0) ? 1u : 0u);
            umma_commit(bar(BB_W_EMPTY + ws));
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {  // K = tile rows, 16 per step
              const uint64_t ada = sdesc_sw128(s_a + as * 16384u + 2048u * ks, 16384, 1024);
              const uint64_t bdf = sdesc_sw128(s_f + fs * 16384u + 2048u * ks, 16384, 1024);
              umma_bf16(dw, ada, bdf, idesc_w, (dw_fresh && ks == 0) ? 0u : 1u);
            }
            umma_commit(bar(BB_A_EMPTY + as));
          }
          __syncwarp();
          ++w_it;
        }
        a_it += static_cast<uint32_t>(nst);
        dw_fresh = false;
        if (elect_one()) umma_commit(bar(BB_F_EMPTY + fs));
        __syncwarp();
        ++f_it;
        if (!last) continue;
        if (elect_one()) umma_commit(bar(BB_T_FULL));
        __syncwarp();
        mbar_wait(bar(BB_T_FULL), t_it & 1);
        named_bar_arrive(2, 32 * 5);  // hand the accumulator to the epilogue
        ++t_it;
      }
    if (elect_one()) umma_commit(bar(BB_MMA_DONE));
    __syncwarp();
  } else if (warp >= FWD_AGG_WARP0) {
    // ------------------------------ aggregation --------------------------------
    const int aw = warp - FWD_AGG_WARP0;
    const int grp = aw / AGG_GROUP_WARPS, wig = aw % AGG_GROUP_WARPS;
    uint32_t a_it = 0, h_it = 0;
    long long p_bnd = 0, p_wait = 0, p_t0 = a.prof ? clock64() : 0;
    for (int w = pair; w < a.n_items; w += npairs)
      for (int s = static_cast<int>(a.item_start[w]); s < static_cast<int>(a.item_start[w + 1]); ++s) {
        const uint32_t H = a.halo_len[s];
        if (H == kOverflow) continue;
        const long long p_b0 = a.prof ? clock64() : 0;
        named_bar_sync(1, 32 * FWD_AGG_WARPS);
        if (a.prof) p_wait += clock64() - p_b0;
        mbar_wait(bar(BB_HALO_FULL), h_it & 1);  // the record's row list is in smem
        coop_load_halo<32 * FWD_AGG_WARPS, true>(reinterpret_cast<const uint32_t*>(gbase + L.hidx), H, a.feat,
                                                 s_halo, 32 * aw + lane, CH);
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(BB_HALO_EMPTY));
        ++h_it;
        named_bar_sync(1, 32 * FWD_AGG_WARPS);
        if (a.prof) p_bnd += clock64() - p_b0;
        const uint32_t first = a_it + ((static_cast<uint32_t>(grp) - a_it) & (AGG_GROUPS - 1));
        for (uint32_t j = first; j < a_it + static_cast<uint32_t>(nst); j += AGG_GROUPS) {
          const uint32_t ds = j % BF_NSD, as = j % BF_NSA;
          mbar_wait(bar(BB_D_FULL + ds), (j / BF_NSD) & 1);
          auto wait_a = [&] { mbar_wait(bar(BB_A_EMPTY + as), ((j / BF_NSA) & 1) ^ 1); };
          const uint8_t* slot = g_d + ds * BLOCK_MAX_BYTES;
          const uint32_t src = BIG ? dsrc[ds] : kFitsSlot;
          if (src == kFitsSlot) {
            aggregate_stage<AGG_GROUP_WARPS>(slot, reinterpret_cast<const uint16_t*>(slot + 512), s_halo,
                                             s_a + as * 16384u, wig, lane, wait_a);
          } else {
            wait_a();
            aggregate_stage_l2<AGG_GROUP_WARPS>(
                slot, reinterpret_cast<const uint16_t*>(a.blocks + blk_bytes(src) + 512), s_halo,
                s_a + as * 16384u, wig, lane);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(bar(BB_A_FULL + as));
            mbar_arrive(bar(BB_D_EMPTY + ds));
          }
        }
        a_it += static_cast<uint32_t>(nst);
      }
    if (a.prof && aw == 0 && lane == 0) {
      a.prof[3 * blockIdx.x] = p_bnd;
      a.prof[3 * blockIdx.x + 1] = clock64() - p_t0;
      a.prof[3 * blockIdx.x + 2] = p_wait;
    }
  } else {
    // ----------------- warps 0-3: F tiles, input-gradient drains, dW dump -------
    const int e = warp;
    uint32_t f_it = 0;
    int pend_s = -1;  // the item (its last record) whose accumulator is to be drained next
    auto load_f = [&](int s) {
      const uint32_t fs = f_it % NSF;
      mbar_wait(bar(BB_F_EMPTY + fs), ((f_it / NSF) & 1) ^ 1);
      const uint2 tl = a.tiles[a.sup[s].x];
      const uint32_t ft = s_f + fs * 16384u;
#pragma unroll 8
      for (int x = lane; x < 32 * 8; x += 32) {  // rows 32e..32e+31, 8 chunks of 16 B
        const int r = 32 * e + (x >> 3), q = x & 7;
        const bool in = static_cast<uint32_t>(r) < tl.y;
        const int64_t row = static_cast<int64_t>(tl.x) + (in ? r : 0);
        cp_async16_zfill(ft + r * 128 + (((q ^ (r & 7)) & 7) << 4),
                         reinterpret_cast<const uint4*>(a.fimg + row * CH) + q, in ? 16u : 0u);
      }
      cp_async_wait_all();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(BB_F_FULL + fs));
      ++f_it;
    };
    auto drain = [&](int s, int w) {
      named_bar_sync(2, 32 * 5);  // released by the MMA warp once the item's T_FULL landed
      tc_fence_after();
      const uint2 tl = a.tiles[a.sup[s].x];
      const uint32_t t0 = tmem + (static_cast<uint32_t>(32 * e) << 16);
      const bool in = static_cast<uint32_t>(32 * e + lane) < tl.y;
      float4* o = in ? reinterpret_cast<float4*>(
                           a.gin + static_cast<int64_t>(a.perm_rows[static_cast<int64_t>(tl.x) + 32 * e + lane]) *
                                       a.gin_cols)
                     : nullptr;
      uint32_t* flag = BF_FLAGS ? a.item_flag + static_cast<int64_t>(w) * 4 + e : nullptr;
      uint32_t v[4][16];
#pragma unroll
      for (int q = 0; q < 4; ++q) tmem_ld16(t0 + 16 * q, v[q]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(BB_T_EMPTY));  // the accumulator is free again
      if (BF_FLAGS && half == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (o && q * 16 < a.gin_cols)
#pragma unroll
            for (int x = 0; x < 4; ++x)
              o[q * 4 + x] = make_float4(__uint_as_float(v[q][4 * x]), __uint_as_float(v[q][4 * x + 1]),
                                         __uint_as_float(v[q][4 * x + 2]), __uint_as_float(v[q][4 * x + 3]));
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(a.gen) : "memory");
        }
      } else {
        if (BF_FLAGS && lane == 0) {
          uint32_t f = 0;
          while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(flag) : "memory");
            if (f == a.gen) break;
            __nanosleep(64);
          }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (o && q * 16 < a.gin_cols)
#pragma unroll
            for (int x = 0; x < 4; ++x)
              asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(o + q * 4 + x),
                           "f"(__uint_as_float(v[q][4 * x])), "f"(__uint_as_float(v[q][4 * x + 1])),
                           "f"(__uint_as_float(v[q][4 * x + 2])), "f"(__uint_as_float(v[q][4 * x + 3]))
                           : "memory");
      }
    };
    int pend_w = -1;
    for (int w = pair; w < a.n_items; w += npairs) {
      {  // warm L2 with the next item's halo while this one is aggregated
        const int s_next = w + npairs < a.n_items ? static_cast<int>(a.item_start[w + npairs]) : -1;
        if (s_next >= 0 && a.halo_len[s_next] != kOverflow)
          prefetch_halo_l2<128>(a.halo + static_cast<int64_t>(s_next) * a.hcap, a.halo_len[s_next], a.feat,
                                32 * e + lane, CH, 1);
      }
      int nrec = 0, last_s = -1;
      for (int s = static_cast<int>(a.item_start[w]); s < static_cast<int>(a.item_start[w + 1]); ++s) {
        if (a.halo_len[s] == kOverflow) continue;
        if (nrec == 2 && pend_s >= 0) {  // free the accumulator before the F ring blocks
          drain(pend_s, pend_w);
          pend_s = -1;
        }
        load_f(s);
        ++nrec;
        last_s = s;
      }
      if (last_s < 0) continue;
      if (pend_s >= 0) drain(pend_s, pend_w);
      pend_s = last_s;
      pend_w = w;
    }
    if (pend_s >= 0) drain(pend_s, pend_w);
    // dW: column block b holds cell stages 2b (lanes 0-15 of each quadrant) and
    // 2b + 1 (lanes 16-31); quadrant e holds rows m = 16e .. 16e + 15
    mbar_wait_sleep(bar(BB_MMA_DONE), 0);
    tc_fence_after();
    const bool none = f_it == 0;  // no records at all: the accumulators were never written
    for (int b = 0; b < BF_STAGES / 2; ++b) {
      const int ci = 2 * b + (lane >> 4);
      const int k = cells[ci];  // (ci < BF_STAGES)
      const int m = 16 * e + (lane & 15);
      float4* o = k != BF_ZERO
                      ? reinterpret_cast<float4*>(a.partial + ((static_cast<int64_t>(pair) * K + k) * 64 + m) * 64)
                      : nullptr;
      const uint32_t t0 = tmem + (static_cast<uint32_t>(32 * e) << 16) + 64u + 64u * b;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t v[16];
        tmem_ld16(t0 + 16 * q, v);
        tmem_ld_wait();
        if (o)
#pragma unroll
          for (int x = 0; x < 4; ++x)
            o[q * 4 + x] = none ? make_float4(0.f, 0.f, 0.f, 0.f)
                                : make_float4(__uint_as_float(v[4 * x]), __uint_as_float(v[4 * x + 1]),
                                              __uint_as_float(v[4 * x + 2]), __uint_as_float(v[4 * x + 3]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_free<512>(tmem);
}

// grad_w[k][m][c] = sum over pairs (fixed order) of partial[x][k][m][c] (64 x 64 padded)
__global__ void k_wgrad_reduce_mc(const float* __restrict__ partial, int n_part, int K, int cin, int cout,
                                  float* __restrict__ grad_w) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(K) * cin * cout) return;
  const int k = static_cast<int>(idx / (cin * cout)), m = static_cast<int>((idx / cin) % cout),
            c = static_cast<int>(idx % cin);
  float s = 0.f;
  for (int x = 0; x < n_part; ++x) s += partial[((static_cast<int64_t>(x) * K + k) * 64 + m) * 64 + c];
  grad_w[idx] = s;
}

// ===========================================================================
// gather engine (forward / dgrad): A tiles assembled by TMA tile::gather4
// ===========================================================================
// A stage (128-row sub-tile t, cell k) needs A_k[r] = sum of the bf16 feature
// rows of row r's neighbors in cell k.  Instead of staging a halo and summing
// on the SM, one producer lane issues 32 cp.async.bulk.tensor.tile::gather4
// per stage: 4 arbitrary 128-byte rows each, written straight into the
// SWIZZLE_128B K-major A tile (the swizzle comes from the tensor map).  Row r
// receives its FIRST neighbor (or an out-of-bounds coordinate -> a zero row);
// the remaining neighbors of rows with >= 2 entries ("extras", ~40 rows per
// stage) are gathered the same way into an extras tile, and fixup warps add
// them to their rows in fp32, in CSR order, rounding once (the numerics of
// the halo engine's emulation, exactly).  No halo: shared memory holds 5 A +
// 5 extras stages instead, so the gathers of several stages are in flight.
//
// Stage descriptor (per (sub-tile, cell), 16-byte aligned):
//   u32 hdr[4] = {nfix, E, 0, 0} | u32 src[128] | u32 ext[E] | u32 fix[nfix]
//   src[r] = bf16 feature row of row r's first entry or 0xFFFFFFFF (zero row)
//   fix    = r | (count - 1) << 7 | ext_offset << 12
constexpr uint32_t kOOB = 0xFFFFFFFFu;
constexpr int G_XCAP = 128;   // extras rows gathered per stage (more -> read from L2)
constexpr int G_NSA = 5;      // A + extras stages
constexpr int G_NSW = 3;      // W stages
constexpr int G_NSD = 8;      // descriptor stages
constexpr int G_DWORDS = 512;           // E + nfix per stage (more -> exact engine)
constexpr int G_DCAP = 528 + 4 * G_DWORDS;
constexpr int G_ST = 2;       // sub-tiles per super-tile (W_k loaded once per super-tile)
constexpr int G_LOAD_WARPS = 8;   // cp.async gather warps (warps 7 ..)
constexpr int G_FIX_WARP0 = 7 + G_LOAD_WARPS;
constexpr int G_FIX_GROUPS = 2;   // fixup groups alternate stages
constexpr int G_FIX_GW = 4;       // warps per fixup group
constexpr int G_FIX_WARPS = G_FIX_GROUPS * G_FIX_GW;
constexpr int G_THREADS = 32 * (G_FIX_WARP0 + G_FIX_WARPS);

struct GatherPlan {
  int64_t n_rows = 0;
  int n_sub = 0, n_super = 0, K = 0;
  DevBuf<uint32_t> blk_off;    // n_sub * K + 1
  DevBuf<uint8_t> blocks;
  DevBuf<uint32_t> super_bad;  // per super-tile: rows served by the exact engine
  DevBuf<uint32_t> spill_rows;
  int64_t n_spill = 0;
  int n_overflow = 0;
};

// Per 128-row sub-tile (one thread per row): block sizes (COUNT) or contents (FILL).
template <bool FILL>
__global__ void __launch_bounds__(TM) k_gplan(const int64_t* __restrict__ row_ptr,
                                              const uint32_t* __restrict__ col,
                                              const uint32_t* __restrict__ kk,
                                              const uint32_t* __restrict__ perm_rows,
                                              const uint32_t* __restrict__ inv_perm_cols,
                                              int64_t n_rows, int K,
                                              const uint32_t* __restrict__ blk_off,
                                              uint32_t* __restrict__ blk_size,
                                              uint32_t* __restrict__ sub_bad,
                                              uint8_t* __restrict__ blocks) {
  __shared__ uint8_t cnt[G_KMAX][TM], run[G_KMAX][TM];
  __shared__ uint16_t fpos[G_KMAX][TM], xpos[G_KMAX][TM];
  __shared__ int nfix_k[G_KMAX], next_k[G_KMAX], wsum[2][4], bad;
  const int r = threadIdx.x, lane = r & 31, warp = r >> 5;
  const int sub = blockIdx.x;
  for (int k = 0; k < G_KMAX; ++k) {
    cnt[k][r] = 0;
    run[k][r] = 0;
  }
  if (r == 0) bad = 0;
  __syncthreads();
  const int64_t p = static_cast<int64_t>(sub) * TM + r;
  uint32_t row_i = 0;
  int64_t e0 = 0, e1 = 0;
  if (p < n_rows) {
    row_i = perm_rows[p];
    e0 = row_ptr[row_i];
    e1 = row_ptr[row_i + 1];
    for (int64_t e = e0; e < e1; ++e) {
      const uint32_t k = kk[e];
      if (cnt[k][r] < 255) cnt[k][r]++;
    }
  }
  for (int k = 0; k < K; ++k) {
    const int c = cnt[k][r];
    if (c > 32) bad = 1;
    const int nf = c >= 2, ne = c > 1 ? c - 1 : 0;
    int inf = nf, ine = ne;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, inf, o), b = __shfl_up_sync(0xffffffffu, ine, o);
      if (lane >= o) {
        inf += a;
        ine += b;
      }
    }
    if (lane == 31) {
      wsum[0][warp] = inf;
      wsum[1][warp] = ine;
    }
    __syncthreads();
    int bf = 0, be = 0, tf = 0, te = 0;
    for (int w = 0; w < 4; ++w) {
      if (w < warp) {
        bf += wsum[0][w];
        be += wsum[1][w];
      }
      tf += wsum[0][w];
      te += wsum[1][w];
    }
    fpos[k][r] = static_cast<uint16_t>(bf + inf - nf);
    xpos[k][r] = static_cast<uint16_t>(be + ine - ne);
    if (r == 0) {
      nfix_k[k] = tf;
      next_k[k] = te;
    }
    __syncthreads();
  }
  if (!FILL) {
    if (r < K) {
      if (nfix_k[r] + next_k[r] > G_DWORDS) bad = 1;
      blk_size[static_cast<int64_t>(sub) * K + r] =
          (528u + 4u * static_cast<uint32_t>(nfix_k[r] + next_k[r]) + 15u) >> 4;
    }
    __syncthreads();
    if (r == 0) sub_bad[sub] = bad;
    return;
  }
  // FILL: header, zero rows, entries in CSR order, fixup items
  for (int k = 0; k < K; ++k) {
    uint8_t* b = blocks + blk_bytes(blk_off[static_cast<int64_t>(sub) * K + k]);
    if (r == 0) {
      reinterpret_cast<uint32_t*>(b)[0] = static_cast<uint32_t>(nfix_k[k]);
      reinterpret_cast<uint32_t*>(b)[1] = static_cast<uint32_t>(next_k[k]);
      reinterpret_cast<uint32_t*>(b)[2] = 0;
      reinterpret_cast<uint32_t*>(b)[3] = 0;
    }
    const int c = cnt[k][r];
    if (c == 0) reinterpret_cast<uint32_t*>(b + 16)[r] = kOOB;
    if (c >= 2)
      reinterpret_cast<uint32_t*>(b + 528 + 4 * next_k[k])[fpos[k][r]] =
          static_cast<uint32_t>(r) | (static_cast<uint32_t>(c - 1) << 7) |
          (static_cast<uint32_t>(xpos[k][r]) << 12);
  }
  for (int64_t e = e0; e < e1; ++e) {
    const int k = static_cast<int>(kk[e]);
    const uint32_t v = inv_perm_cols[col[e]];
    uint8_t* b = blocks + blk_bytes(blk_off[static_cast<int64_t>(sub) * K + k]);
    const int n = run[k][r]++;
    if (n == 0) reinterpret_cast<uint32_t*>(b + 16)[r] = v;
    else reinterpret_cast<uint32_t*>(b + 528)[xpos[k][r] + n - 1] = v;
  }
}

static std::unique_ptr<GatherPlan> build_gather_plan(npcg_context* ctx, const int64_t* row_ptr,
                                                     const uint32_t* col, const uint32_t* kk,
                                                     int64_t n_rows, const uint32_t* perm_rows,
                                                     const uint32_t* inv_perm_cols, int K) {
  auto P = std::make_unique<GatherPlan>();
  P->n_rows = n_rows;
  P->K = K;
  P->n_sub = static_cast<int>(ceil_div(n_rows, TM));
  P->n_super = static_cast<int>(ceil_div(P->n_sub, G_ST));
  if (P->n_sub == 0) return P;
  const int64_t nblk = static_cast<int64_t>(P->n_sub) * K;
  DevBuf<uint32_t> blk_size(ctx, nblk + 1), sub_bad(ctx, P->n_sub);
  NPCG_CUDA(cudaMemsetAsync(blk_size.get() + nblk, 0, 4, ctx->stream));
  launch(ctx, "gplan_count", k_gplan<false>, dim3(P->n_sub), dim3(TM), 0, row_ptr, col, kk,
         perm_rows, inv_perm_cols, n_rows, K, static_cast<const uint32_t*>(nullptr),
         blk_size.get(), sub_bad.get(), static_cast<uint8_t*>(nullptr));
  P->blk_off.alloc(ctx, nblk + 1);
  uint32_t total = 0;
  exclusive_scan_u32(ctx, blk_size.get(), P->blk_off.get(), nblk + 1, &total);
  P->blocks.alloc(ctx, static_cast<int64_t>(blk_bytes(total)));
  launch(ctx, "gplan_fill", k_gplan<true>, dim3(P->n_sub), dim3(TM), 0, row_ptr, col, kk,
         perm_rows, inv_perm_cols, n_rows, K, static_cast<const uint32_t*>(P->blk_off.get()),
         static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), P->blocks.get());
  std::vector<uint32_t> sb(P->n_sub);
  NPCG_CUDA(cudaMemcpyAsync(sb.data(), sub_bad.get(), sb.size() * 4, cudaMemcpyDeviceToHost,
                            ctx->stream));
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<uint32_t> bad(P->n_super, 0);
  for (int s = 0; s < P->n_sub; ++s) bad[s / G_ST] |= sb[s];
  std::vector<uint32_t> rows;
  for (int S = 0; S < P->n_super; ++S)
    if (bad[S]) {
      P->n_overflow++;
      for (int64_t q = static_cast<int64_t>(S) * G_ST * TM;
           q < std::min<int64_t>(n_rows, static_cast<int64_t>(S + 1) * G_ST * TM); ++q)
        rows.push_back(static_cast<uint32_t>(q));
    }
  P->super_bad.alloc(ctx, P->n_super);
  NPCG_CUDA(cudaMemcpyAsync(P->super_bad.get(), bad.data(), bad.size() * 4, cudaMemcpyHostToDevice,
                            ctx->stream));
  P->n_spill = static_cast<int64_t>(rows.size());
  if (P->n_spill) {
    P->spill_rows.alloc(ctx, P->n_spill);
    NPCG_CUDA(cudaMemcpyAsync(P->spill_rows.get(), rows.data(), rows.size() * 4,
                              cudaMemcpyHostToDevice, ctx->stream));
  }
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
  return P;
}

struct GArgs {
  const uint32_t* blk_off;
  const uint8_t* blocks;
  const uint32_t* super_bad;
  const uint32_t* perm_rows;
  int64_t n_rows;
  int n_sub, n_super, K;
  const __nv_bfloat16* feat;  // bf16 (n_cols, 64), permuted
  const uint8_t* wpack;       // K x 8 KB
  float* out;
  long long* trace;
};

struct GSmem {
  uint32_t a, x, w, d, bar, tmem_slot, offs;
  size_t total;
};
__host__ __device__ inline GSmem g_smem_layout() {
  GSmem L{};
  uint32_t o = 0;
  L.a = o;
  o += G_NSA * 16384;
  L.x = o;
  o += G_NSA * G_XCAP * 128;
  L.w = o;
  o += G_NSW * 8192;
  L.d = o;
  o += G_NSD * G_DCAP;
  o = (o + 7) & ~7u;
  L.bar = o;
  o += 48 * 8;
  L.tmem_slot = o;
  o += 16;
  L.offs = o;
  o += (G_ST * G_KMAX + 1) * 4;
  L.total = o + 1024;
  return L;
}
enum : int {
  G_A_FULL = 0,                   // G_NSA: gathers landed (tx)
  G_A_READY = G_A_FULL + G_NSA,   // G_NSA: fixups done
  G_A_EMPTY = G_A_READY + G_NSA,  // G_NSA: MMA done reading
  G_W_FULL = G_A_EMPTY + G_NSA,   // G_NSW
  G_W_EMPTY = G_W_FULL + G_NSW,
  G_D_FULL = G_W_EMPTY + G_NSW,   // G_NSD
  G_D_EMPTY = G_D_FULL + G_NSD,
  G_T_FULL = G_D_EMPTY + G_NSD,   // 2
  G_T_EMPTY = G_T_FULL + 2,
  G_COUNT = G_T_EMPTY + 2
};
static_assert(G_COUNT <= 48, "gather barrier region");

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, uint4 rows,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(rows.x), "r"(rows.y), "r"(rows.z),
      "r"(rows.w), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(G_THREADS, 1)
    k_conv_gather(const __grid_constant__ CUtensorMap tmap, GArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const GSmem L = g_smem_layout();
  const uint32_t s_a = base + L.a, s_x = base + L.x, s_w = base + L.w, s_d = base + L.d;
  const uint32_t s_bar = base + L.bar;
  auto bar = [&](int i) { return s_bar + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + L.tmem_slot);
  const uint8_t* g_d = gbase + L.d;
  const uint8_t* g_x = gbase + L.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K;
  if (threadIdx.x == 0) {
    for (int i = 0; i < G_NSA; ++i) {
      mbar_init(bar(G_A_FULL + i), 32 * G_LOAD_WARPS);  // one cp.async arrive per loader thread
      mbar_init(bar(G_A_READY + i), G_FIX_GW);
      mbar_init(bar(G_A_EMPTY + i), 1);
    }
    for (int i = 0; i < G_NSW; ++i) {
      mbar_init(bar(G_W_FULL + i), 1);
      mbar_init(bar(G_W_EMPTY + i), 1);
    }
    for (int i = 0; i < G_NSD; ++i) {
      mbar_init(bar(G_D_FULL + i), 1);
      mbar_init(bar(G_D_EMPTY + i), G_LOAD_WARPS + G_FIX_GW);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(G_T_FULL + i), 1);
      mbar_init(bar(G_T_EMPTY + i), 4);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<256>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto nsub_of = [&](int S) { return min(G_ST, a.n_sub - S * G_ST); };

  if (warp == 4) {
    // ---- descriptor producer: bulk copies into the D ring --------------------
    uint32_t* offs = reinterpret_cast<uint32_t*>(gbase + L.offs);
    uint32_t d_it = 0;
    for (int S = blockIdx.x; S < a.n_super; S += gridDim.x) {
      if (a.super_bad[S]) continue;
      const int nsub = nsub_of(S);
      for (int x = lane; x <= nsub * K; x += 32)
        offs[x] = a.blk_off[static_cast<int64_t>(S) * G_ST * K + x];
      __syncwarp();
      for (int k = 0; k < K; ++k)
        for (int g = 0; g < nsub; ++g) {
          if (lane == 0) {
            const uint32_t ds = d_it % G_NSD;
            mbar_wait(bar(G_D_EMPTY + ds), ((d_it / G_NSD) & 1) ^ 1);
            const uint32_t o0 = offs[g * K + k], o1 = offs[g * K + k + 1];
            mbar_expect_tx(bar(G_D_FULL + ds), (o1 - o0) << 4);
            bulk_g2s(s_d + ds * G_DCAP, a.blocks + blk_bytes(o0), (o1 - o0) << 4, bar(G_D_FULL + ds));
          }
          ++d_it;
        }
      __syncwarp();
    }
  } else if (warp >= 7 && warp < G_FIX_WARP0) {
    // ---- loaders: cp.async (16 B per lane, 4 rows per warp instruction) of
    // every row's first neighbor into the swizzled A tile (zero-fill for
    // rows without neighbors) and of up to G_XCAP extras into the X tile;
    // the A_FULL mbarrier tracks their completion (arrive.noinc) -----------
    const int lw = warp - 7;
    const uint32_t q = static_cast<uint32_t>(lane & 7), rq = static_cast<uint32_t>(lane >> 3);
    constexpr int RI = TM / (4 * G_LOAD_WARPS);  // row iterations per loader warp
    uint32_t dsto[RI];                           // swizzled destination of this lane's chunks
#pragma unroll
    for (int i = 0; i < RI; ++i) {
      const uint32_t r = static_cast<uint32_t>(lw * 4 * RI + i * 4) + rq;
      dsto[i] = r * 128u + ((q ^ (r & 7u)) << 4);
    }
    const uint8_t* fbase = reinterpret_cast<const uint8_t*>(a.feat) + q * 16u;
    uint32_t it = 0;
    for (int S = blockIdx.x; S < a.n_super; S += gridDim.x) {
      if (a.super_bad[S]) continue;
      const int nsub = nsub_of(S);
      for (int k = 0; k < K; ++k)
        for (int g = 0; g < nsub; ++g, ++it) {
          const uint32_t ds = it % G_NSD, as = it % G_NSA;
          mbar_wait(bar(G_D_FULL + ds), (it / G_NSD) & 1);
          mbar_wait(bar(G_A_EMPTY + as), ((it / G_NSA) & 1) ^ 1);
          if (lw == 0 && lane == 0) trace_ev(a.trace, it, 0);
          const uint8_t* blk = g_d + ds * G_DCAP;
          const uint32_t E = reinterpret_cast<const uint32_t*>(blk)[1];
          const uint32_t ex = min(E, static_cast<uint32_t>(G_XCAP));
          const uint32_t* src = reinterpret_cast<const uint32_t*>(blk + 16) + lw * 4 * RI + rq;
          const uint32_t* ext = reinterpret_cast<const uint32_t*>(blk + 528);
          const uint32_t sa = s_a + as * 16384u, sx = s_x + as * (G_XCAP * 128u);
          uint32_t v[RI];
#pragma unroll
          for (int i = 0; i < RI; ++i) v[i] = src[i * 4];
#pragma unroll
          for (int i = 0; i < RI; ++i)
            cp_async16_zfill(sa + dsto[i], fbase + static_cast<uint64_t>(v[i] == kOOB ? 0u : v[i]) * 128u,
                             v[i] == kOOB ? 0u : 16u);
          for (uint32_t x = static_cast<uint32_t>(lw * 4) + rq; x < ex; x += 4 * G_LOAD_WARPS)
            cp_async16_zfill(sx + x * 128u + ((q ^ (x & 7u)) << 4),
                             fbase + static_cast<uint64_t>(ext[x]) * 128u, 16u);
          cp_async_mbar_arrive_noinc(bar(G_A_FULL + as));
          __syncwarp();
          if (lw == 0 && lane == 0) trace_ev(a.trace, it, 1);
          if (lane == 0) mbar_arrive(bar(G_D_EMPTY + ds));
        }
    }
  } else if (warp == 6) {
    // ---- W_k producer ------------------------------------------------------------
    if (lane == 0) {
      uint32_t w_it = 0;
      for (int S = blockIdx.x; S < a.n_super; S += gridDim.x) {
        if (a.super_bad[S]) continue;
        for (int k = 0; k < K; ++k, ++w_it) {
          const uint32_t ws = w_it % G_NSW;
          mbar_wait_sleep(bar(G_W_EMPTY + ws), ((w_it / G_NSW) & 1) ^ 1);
          mbar_expect_tx(bar(G_W_FULL + ws), 8192u);
          bulk_g2s(s_w + ws * 8192u, a.wpack + static_cast<int64_t>(k) * 8192, 8192u,
                   bar(G_W_FULL + ws));
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ---- MMA issuer (as the halo engine) -------------------------------------------
    constexpr uint32_t idesc = idesc_bf16(128, 64, false, false);
    const uint64_t a_desc0 = sdesc_sw128(s_a, 16, 1024), b_desc0 = sdesc_sw128(s_w, 16, 1024);
    uint32_t w_it = 0, it = 0, t_it = 0;
    bool pending = false;
    uint32_t pend_t = 0;
    auto release_epilogue = [&]() {
      mbar_wait(bar(G_T_FULL + (pend_t & 1)), (pend_t >> 1) & 1);
      named_bar_arrive(2 + (pend_t & 1), 32 * 5);
      pending = false;
    };
    for (int S = blockIdx.x; S < a.n_super; S += gridDim.x) {
      if (a.super_bad[S]) continue;
      const int nsub = nsub_of(S);
      const uint32_t ab = t_it & 1;
      mbar_wait(bar(G_T_EMPTY + ab), ((t_it >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int k = 0; k < K; ++k) {
        if (pending && k == 1) release_epilogue();
        const uint32_t ws = w_it % G_NSW;
        mbar_wait(bar(G_W_FULL + ws), (w_it / G_NSW) & 1);
        for (int g = 0; g < nsub; ++g, ++it) {
          const uint32_t as = it % G_NSA;
          mbar_wait(bar(G_A_READY + as), (it / G_NSA) & 1);
          if (lane == 0) trace_ev(a.trace, it, 4);
          tc_fence_after();
          const uint32_t d = tmem + ab * (G_ST * 64) + g * 64;
          const uint64_t ad = a_desc0 + ((as * 16384u) >> 4);
          const uint64_t bd = b_desc0 + ((ws * 8192u) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              umma_bf16(d, ad + 2u * ks, bd + 2u * ks, idesc, (k > 0 || ks > 0) ? 1u : 0u);
            umma_commit(bar(G_A_EMPTY + as));
          }
          __syncwarp();
          if (lane == 0) trace_ev(a.trace, it, 5);
        }
        if (elect_one()) umma_commit(bar(G_W_EMPTY + ws));
        __syncwarp();
        ++w_it;
      }
      if (elect_one()) umma_commit(bar(G_T_FULL + ab));
      __syncwarp();
      if (pending) release_epilogue();
      pending = true;
      pend_t = t_it;
      ++t_it;
    }
    if (pending) release_epilogue();
  } else if (warp >= G_FIX_WARP0) {
    // ---- fixups: rows of >= 2 entries, fp32 sum (CSR order) rounded once ---------
    // quarter-warp per row: lane group q8 = lane / 8 of warp fw handles rows
    // fw * 4 + q8, + 32, ...; each lane one 16-byte chunk (8 channels)
    const int fw = (warp - G_FIX_WARP0) % G_FIX_GW, fg = (warp - G_FIX_WARP0) / G_FIX_GW;
    const uint32_t q = static_cast<uint32_t>(lane & 7);
    uint32_t it = 0;
    for (int S = blockIdx.x; S < a.n_super; S += gridDim.x) {
      if (a.super_bad[S]) continue;
      const int nsub = nsub_of(S);
      for (int k = 0; k < K; ++k)
        for (int g = 0; g < nsub; ++g, ++it) {
          if (static_cast<int>(it % G_FIX_GROUPS) != fg) continue;
          const uint32_t ds = it % G_NSD, as = it % G_NSA;
          mbar_wait(bar(G_D_FULL + ds), (it / G_NSD) & 1);
          const uint8_t* blk = g_d + ds * G_DCAP;
          const uint32_t nfix = reinterpret_cast<const uint32_t*>(blk)[0];
          const uint32_t E = reinterpret_cast<const uint32_t*>(blk)[1];
          const uint32_t* ext = reinterpret_cast<const uint32_t*>(blk + 528);
          const uint32_t* fix = ext + E;
          mbar_wait(bar(G_A_FULL + as), (it / G_NSA) & 1);
          if (fw == 0 && lane == 0) trace_ev(a.trace, it, 2);
          const uint32_t sa = s_a + as * 16384u;
          const uint8_t* gx = g_x + as * (G_XCAP * 128u);
          for (uint32_t f = static_cast<uint32_t>(fw * 4 + (lane >> 3)); f < nfix; f += G_FIX_GW * 4) {
            const uint32_t item = fix[f];
            const uint32_t r = item & 127u, c1 = (item >> 7) & 31u, xo = item >> 12;
            const uint32_t ra = sa + r * 128u + ((q ^ (r & 7u)) << 4);
            float acc[8];
            const uint4 v0 = lds128(ra);
#pragma unroll
            for (int x = 0; x < 8; ++x) acc[x] = 0.f;
            acc_bf16x2(acc[0], acc[1], v0.x);
            acc_bf16x2(acc[2], acc[3], v0.y);
            acc_bf16x2(acc[4], acc[5], v0.z);
            acc_bf16x2(acc[6], acc[7], v0.w);
            for (uint32_t e = 0; e < c1; ++e) {
              const uint32_t xr = xo + e;
              uint4 w;
              if (xr < static_cast<uint32_t>(G_XCAP))
                w = *reinterpret_cast<const uint4*>(gx + xr * 128u + ((q ^ (xr & 7u)) << 4));
              else
                w = __ldg(reinterpret_cast<const uint4*>(a.feat + static_cast<int64_t>(ext[xr]) * CH) + q);
              acc_bf16x2(acc[0], acc[1], w.x);
              acc_bf16x2(acc[2], acc[3], w.y);
              acc_bf16x2(acc[4], acc[5], w.z);
              acc_bf16x2(acc[6], acc[7], w.w);
            }
            uint4 o;
            o.x = pack_bf16x2(acc[0], acc[1]);
            o.y = pack_bf16x2(acc[2], acc[3]);
            o.z = pack_bf16x2(acc[4], acc[5]);
            o.w = pack_bf16x2(acc[6], acc[7]);
            sts128(ra, o);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (fw == 0 && lane == 0) trace_ev(a.trace, it, 3);
          if (lane == 0) {
            mbar_arrive(bar(G_A_READY + as));
            mbar_arrive(bar(G_D_EMPTY + ds));
          }
        }
    }
  } else {
    // ---- epilogue (warps 0-3): TMEM -> output rows --------------------------------
    const int e = warp;
    uint32_t t_it = 0;
    for (int S = blockIdx.x; S < a.n_super; S += gridDim.x) {
      if (a.super_bad[S]) continue;
      const int nsub = nsub_of(S);
      const uint32_t ab = t_it & 1;
      named_bar_sync(2 + ab, 32 * 5);
      tc_fence_after();
      for (int g = 0; g < nsub; ++g) {
        const uint32_t t0 = tmem + (static_cast<uint32_t>(32 * e) << 16) + ab * (G_ST * 64) + g * 64;
        const int64_t row = (static_cast<int64_t>(S) * G_ST + g) * TM + 32 * e + lane;
        float4* o = row < a.n_rows
                        ? reinterpret_cast<float4*>(a.out + static_cast<int64_t>(a.perm_rows[row]) * CH)
                        : nullptr;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          uint32_t v[16];
          tmem_ld16(t0 + 16 * qq, v);
          tmem_ld_wait();
          if (o)
#pragma unroll
            for (int x = 0; x < 4; ++x)
              o[qq * 4 + x] = make_float4(__uint_as_float(v[4 * x]), __uint_as_float(v[4 * x + 1]),
                                          __uint_as_float(v[4 * x + 2]), __uint_as_float(v[4 * x + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(G_T_EMPTY + ab));
      ++t_it;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_free<256>(tmem);
}

// Tensor map of a bf16 (rows, 64) feature matrix for tile::gather4: box 64 x 1,
// SWIZZLE_128B (matches the A tile layout), out-of-bounds rows read as zeros.
static CUtensorMap feature_tmap(const __nv_bfloat16* feat, int64_t rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(CH), static_cast<cuuint64_t>(std::max<int64_t>(rows, 1))};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(CH) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(CH), 1};
  const cuuint32_t estr[2] = {1, 1};
  // the driver entry point is resolved through the runtime, so libnpcg.so does
  // not link libcuda (it loads on GPU-less hosts)
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    NPCG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) fail(NPCG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const CUresult r = encode(
      &m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(feat), dims, strides, box,
      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(NPCG_ERR_CUDA, "cuTensorMapEncodeTiled failed for the feature map");
  return m;
}

static void run_gather_kernel(npcg_context* ctx, GatherPlan* P, const __nv_bfloat16* feat,
                              int64_t n_cols, const uint8_t* wpack, const uint32_t* perm_rows,
                              float* out, const char* name, long long* trace = nullptr) {
  if (P->n_super == 0 || P->n_overflow == P->n_super) return;
  GArgs a{};
  a.blk_off = P->blk_off.get();
  a.blocks = P->blocks.get();
  a.super_bad = P->super_bad.get();
  a.perm_rows = perm_rows;
  a.n_rows = P->n_rows;
  a.n_sub = P->n_sub;
  a.n_super = P->n_super;
  a.K = P->K;
  a.feat = feat;
  a.wpack = wpack;
  a.out = out;
  a.trace = trace;
  const CUtensorMap tmap = feature_tmap(feat, n_cols);
  const GSmem L = g_smem_layout();
  NPCG_CUDA(cudaFuncSetAttribute(k_conv_gather, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(L.total)));
  const int grid = std::min(P->n_super, ctx->num_sms);
  launch(ctx, name, k_conv_gather, dim3(grid), dim3(G_THREADS), L.total, tmap, a);
}

// ===========================================================================
// host drivers
// ===========================================================================

static TcPlan* get_plan(npcg_context* ctx, npcg_neighbors* nb) {
  if (!nb->tc) {
    auto* p = new TcPlan();
    nb->tc.reset(p);
    p->inv_perm_out.alloc(ctx, nb->n_out);
    p->inv_perm_in.alloc(ctx, nb->n_in);
    if (nb->n_out)
      launch(ctx, "inverse_perm", k_inverse_perm, dim3(static_cast<unsigned>(ceil_div(nb->n_out, 256))),
             dim3(256), 0, static_cast<const uint32_t*>(nb->perm_out.get()), nb->n_out,
             p->inv_perm_out.get());
    if (nb->n_in)
      launch(ctx, "inverse_perm", k_inverse_perm, dim3(static_cast<unsigned>(ceil_div(nb->n_in, 256))),
             dim3(256), 0, static_cast<const uint32_t*>(nb->perm_in.get()), nb->n_in,
             p->inv_perm_in.get());
  }
  return nb->tc.get();
}

static void wgrad_cell_order(const TcDirPlan* P, int K, int np, int gpc, uint8_t* korder);

// wide = the pass writes 256 channels: 128-row super-tiles (st = 1); 64- and
// 128-channel passes share the 256-row plan
static TcDirPlan* plan_fwd(npcg_context* ctx, npcg_neighbors* nb, bool wide = false) {
  TcPlan* p = get_plan(ctx, nb);
  auto& slot = wide ? p->fwd1 : p->fwd;
  if (!slot)
    slot = build_dir_plan(ctx, nb->row_ptr.get(), nb->col_j.get(), nb->col_k.get(), nb->n_out,
                          nb->n_in, nb->perm_out.get(), p->inv_perm_in.get(), nb->out_off,
                          static_cast<int>(nb->n_kernels), wide ? 1 : FWD_ST,
                          wide ? FWD_HCAP1 : FWD_HCAP);
  return slot.get();
}
static TcDirPlan* plan_bwd(npcg_context* ctx, npcg_neighbors* nb, bool wide = false) {
  TcPlan* p = get_plan(ctx, nb);
  auto& slot = wide ? p->bwd1 : p->bwd;
  if (!slot) {
    build_tcsr(ctx, nb);
    slot = build_dir_plan(ctx, nb->tcsr->row_ptr.get(), nb->tcsr->col.get(), nb->tcsr->k.get(),
                          nb->n_in, nb->n_out, nb->perm_in.get(), p->inv_perm_out.get(), nb->in_off,
                          static_cast<int>(nb->n_kernels), wide ? 1 : FWD_ST,
                          wide ? FWD_HCAP1 : FWD_HCAP);
  }
  return slot.get();
}

static bool use_gather_engine_env();
// Split weight gradient: super-tiles per TMEM accumulation segment (each
// segment's chain of truncating fp32 accumulations is bounded: 2 sub-tiles x
// 8 MMAs x seg), NPCG_SPLIT_SEG overrides (read once per process).
static int split_segment() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("NPCG_SPLIT_SEG");
    v = e ? std::max(1, std::atoi(e)) : 4;
  }
  return v;
}
static bool use_gather_engine(int64_t K) { return use_gather_engine_env() && K <= G_KMAX; }
static GatherPlan* gplan_fwd(npcg_context* ctx, npcg_neighbors* nb);
static GatherPlan* gplan_bwd(npcg_context* ctx, npcg_neighbors* nb);

static bool fused_bwd_enabled();
// The plans a 64-channel layer's forward + backward use in `mode`: the
// forward plan, and the transposed plan of the fused backward (bf16, K = 27:
// 128-row super-tiles) or of the separate dgrad.
void tc_prepare(npcg_context* ctx, npcg_neighbors* nb, TcMode mode) {
  if (use_gather_engine(nb->n_kernels)) {
    gplan_fwd(ctx, nb);
    gplan_bwd(ctx, nb);
  }
  plan_fwd(ctx, nb);
  const bool fused = mode == TcMode::bf16 && nb->n_kernels == 27 && fused_bwd_enabled() &&
                     !use_gather_engine(nb->n_kernels);
  plan_bwd(ctx, nb, fused);
}

// bf16 image of C-channel rows, padded with zero channels to CP = tc_pad(C)
static void convert(npcg_context* ctx, const float* src, const uint32_t* perm, int64_t n,
                    DevBuf<__nv_bfloat16>& dst, int C = CH) {
  const int CP = tc_pad(C);
  if (dst.size() < n * CP) dst.alloc(ctx, n * CP);
  if (n == 0) return;
  launch(ctx, "to_bf16_perm", k_to_bf16_perm, dim3(static_cast<unsigned>(ceil_div(n * (CP / 8), 256))),
         dim3(256), 0, src, perm, n, C, CP, dst.get());
}

// max |x| of a tensor into a scale slot (split path)
static uint32_t* amax_slot(npcg_context* ctx, TcPlan* p, int slot) {
  if (p->amax.size() < 4) p->amax.alloc(ctx, 4);
  return p->amax.get() + slot;
}
static void absmax(npcg_context* ctx, const float* x, int64_t n, uint32_t* slot) {
  NPCG_CUDA(cudaMemsetAsync(slot, 0, 4, ctx->stream));
  if (n == 0) return;
  launch(ctx, "absmax", k_absmax,
         dim3(static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 4 * ctx->num_sms))), dim3(256), 0,
         x, n, slot);
}

// split image (fp32-contract path): 2 x CP fp16 per row, scaled by the slot's scale
static void convert_split(npcg_context* ctx, const float* src, const uint32_t* perm, int64_t n,
                          DevBuf<__nv_bfloat16>& dst, int C, uint32_t* slot) {
  const int CP = tc_pad(C);
  absmax(ctx, src, n * C, slot);
  if (dst.size() < n * 2 * CP) dst.alloc(ctx, n * 2 * CP);
  if (n == 0) return;
  launch(ctx, "to_split_perm", k_to_split_perm, dim3(static_cast<unsigned>(ceil_div(n * (CP / 8), 256))),
         dim3(256), 0, src, perm, n, C, CP, static_cast<const uint32_t*>(slot),
         reinterpret_cast<__half*>(dst.get()));
}

// Written channels [n0, n0 + nn) of the pass (C_out forward, C_in dgrad);
// the scale slot is filled from the whole tensor when n0 == 0.
static void pack_w_split(npcg_context* ctx, TcPlan* p, const float* w, int K, bool transpose,
                         int cin, int cout, uint32_t* slot, int n0 = 0, int nn = -1) {
  if (nn < 0) nn = transpose ? cin : cout;
  const int N = tc_pad(nn), R = tc_pad(transpose ? cout : cin);
  const int64_t n = static_cast<int64_t>(K) * cin * cout;
  const int64_t bytes = static_cast<int64_t>(K) * R * N * 2 * 2 * 2;  // 2 images, K 64 per 32
  if (n0 == 0) absmax(ctx, w, n, slot);
  if (p->wpack.size() < bytes) p->wpack.alloc(ctx, bytes);
  NPCG_CUDA(cudaMemsetAsync(p->wpack.get(), 0, bytes, ctx->stream));
  launch(ctx, "pack_w_split", k_pack_w_split, dim3(static_cast<unsigned>(ceil_div(n, 256))), dim3(256),
         0, w, K, cin, cout, N, R / 32, n0, transpose, static_cast<const uint32_t*>(slot), p->wpack.get());
}

static void pack_w(npcg_context* ctx, TcPlan* p, const float* w, int K, bool transpose,
                   int cin = CH, int cout = CH) {
  const int cinp = tc_pad(cin), coutp = tc_pad(cout);
  const int64_t n = static_cast<int64_t>(K) * cin * cout;
  const int64_t bytes = static_cast<int64_t>(K) * cinp * coutp * 2;
  if (p->wpack.size() < bytes) p->wpack.alloc(ctx, bytes);
  if (cinp != cin || coutp != cout)
    NPCG_CUDA(cudaMemsetAsync(p->wpack.get(), 0, bytes, ctx->stream));
  launch(ctx, "pack_w", k_pack_w, dim3(static_cast<unsigned>(ceil_div(n, 256))), dim3(256), 0, w,
         K, cin, cout, cinp, coutp, transpose, p->wpack.get());
}

template <int NOUT, bool SPLIT = false>
static void launch_fwd(npcg_context* ctx, const FwdArgs& a, int hcap, int grid, const char* name,
                       bool big) {
  const FwdSmem L = fwd_smem_layout<NOUT, SPLIT>(hcap);
  if (a.trace && (NOUT != 64 || SPLIT)) fail(NPCG_ERR_UNSUPPORTED, "trace: 64-channel bf16 passes only");
  auto kern = big ? k_conv_fwd_tc<NOUT, true, false, SPLIT> : k_conv_fwd_tc<NOUT, false, false, SPLIT>;
  if constexpr (NOUT == 64 && !SPLIT)
    if (a.trace) kern = big ? k_conv_fwd_tc<64, true, true> : k_conv_fwd_tc<64, false, true>;
  NPCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(L.total)));
  launch(ctx, name, kern, dim3(grid), dim3(FWD_THREADS), L.total, a);
}

// One gather-side pass (forward or dgrad): cin_g gathered channels -> nout
// written channels per row.
static void run_fwd_kernel(npcg_context* ctx, TcDirPlan* P, const __nv_bfloat16* feat,
                           const uint8_t* wpack, const uint32_t* perm_rows, float* out,
                           const char* name, long long* trace = nullptr, int cin_g = CH,
                           int nout = CH, bool split = false, const uint32_t* amax = nullptr,
                           int col0 = 0, int out_stride = -1) {
  // cin_g / nout: real gathered / written channels; the kernel runs padded
  // (split: chunks of 32 real channels, each a 64-wide [hi | lo] bf16 slice)
  const int ncols = nout;
  cin_g = tc_pad(cin_g);
  nout = tc_pad(nout);
  if (P->n_super == 0) return;
  FwdArgs a{};
  a.halo = P->halo.get();
  a.halo_len = P->halo_len.get();
  a.blk_off = P->blk_off.get();
  a.blocks = P->blocks.get();
  a.perm_rows = perm_rows;
  a.sup = P->sup.get();
  a.tiles = P->tiles.get();
  a.item_start = P->item_start.get();
  a.n_items = P->n_items;
  a.n_rows = P->n_rows;
  a.n_sub = P->n_sub;
  a.n_super = P->n_super;
  a.st = P->st;
  a.hcap = P->hcap;
  a.K = P->K;
  a.nci = split ? cin_g / 32 : cin_g / CH;
  a.feat = feat;
  a.wpack = wpack;
  a.out = out;
  a.ncols = ncols;
  a.out_stride = out_stride < 0 ? ncols : out_stride;
  a.out_col0 = col0;
  a.trace = trace;
  a.amax = amax;
  const int grid = std::min(P->n_super, ctx->num_sms);
  if (split) {
    if (nout == 64) launch_fwd<64, true>(ctx, a, P->hcap, grid, name, P->big_blocks);
    else if (nout == 128) launch_fwd<128, true>(ctx, a, P->hcap, grid, name, P->big_blocks);
    else fail(NPCG_ERR_UNSUPPORTED, "split tensor-core path: at most 128 written channels");
    return;
  }
  if (nout == 64) launch_fwd<64>(ctx, a, P->hcap, grid, name, P->big_blocks);
  else if (nout == 128) launch_fwd<128>(ctx, a, P->hcap, grid, name, P->big_blocks);
  else launch_fwd<256>(ctx, a, P->hcap, grid, name, P->big_blocks);
}


void GatherPlanDeleter::operator()(GatherPlan* p) const { delete p; }
void destroy_tc_plan(TcPlan* p) { delete p; }

// Forward / dgrad engine: "halo" (shared-memory halo + SM aggregation, the
// default: 0.85 ms per 1M-point pass) or "gather" (A tiles gathered from L2
// by cp.async, fixups on the SM: 0.99 ms; profiles/r1_pipeline_experiments.md).
// NPCG_TC_ENGINE=gather selects the latter (read once per process).
static bool use_gather_engine_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("NPCG_TC_ENGINE");
    v = (e && std::strcmp(e, "gather") == 0) ? 1 : 0;
  }
  return v == 1;
}
static GatherPlan* gplan_fwd(npcg_context* ctx, npcg_neighbors* nb) {
  TcPlan* p = get_plan(ctx, nb);
  if (!p->gfwd)
    p->gfwd.reset(build_gather_plan(ctx, nb->row_ptr.get(), nb->col_j.get(), nb->col_k.get(),
                                    nb->n_out, nb->perm_out.get(), p->inv_perm_in.get(),
                                    static_cast<int>(nb->n_kernels)).release());
  return p->gfwd.get();
}
static GatherPlan* gplan_bwd(npcg_context* ctx, npcg_neighbors* nb) {
  TcPlan* p = get_plan(ctx, nb);
  if (!p->gbwd) {
    build_tcsr(ctx, nb);
    p->gbwd.reset(build_gather_plan(ctx, nb->tcsr->row_ptr.get(), nb->tcsr->col.get(),
                                    nb->tcsr->k.get(), nb->n_in, nb->perm_in.get(),
                                    p->inv_perm_out.get(), static_cast<int>(nb->n_kernels))
                      .release());
  }
  return p->gbwd.get();
}

// The forward's device image of fin (bf16 or split), kept for the backward.
static void input_image(npcg_context* ctx, npcg_neighbors* nb, TcPlan* p, const float* fin, int cin,
                        bool split) {
  if (split) convert_split(ctx, fin, nb->perm_in.get(), nb->n_in, p->feat_in, cin, amax_slot(ctx, p, 0));
  else convert(ctx, fin, nb->perm_in.get(), nb->n_in, p->feat_in, cin);
  p->saved_fin = fin;  // PointConvOp saves its input (conv_op.hpp:138)
  p->saved_c = cin;
  p->saved_split = split;
}

// Plans: 256-row super-tiles unless the pass writes more than 128 channels
// (bf16) / more than 64 (split: its W stages are twice as large).
static bool wide_pass(int written, bool split) { return tc_pad(written) > (split ? CH : 2 * CH); }

// A split (fp32-contract) gather pass: the split kernels hold at most 128
// written channels in TMEM (3 main + 1 correction accumulator sets), so a
// wider pass runs as 128-column halves, each with its own W images and the
// output row stride of the whole width.  transpose: the dgrad pass (gathers
// C_out, writes C_in).
static void split_passes(npcg_context* ctx, TcPlan* p, TcDirPlan* P, const float* w, bool transpose,
                         int cin, int cout, const __nv_bfloat16* feat, const uint32_t* perm_rows,
                         float* out, const char* name, uint32_t* amax_feat, uint32_t* amax_w) {
  const int gathered = transpose ? cout : cin, written = transpose ? cin : cout;
  for (int n0 = 0; n0 < written; n0 += 128) {
    const int nn = std::min(128, written - n0);
    pack_w_split(ctx, p, w, P->K, transpose, cin, cout, amax_w, n0, nn);
    run_fwd_kernel(ctx, P, feat, p->wpack.get(), perm_rows, out, name, nullptr, gathered, nn, true, amax_feat,
                   n0, written);
  }
}

void tc_forward(npcg_context* ctx, npcg_neighbors* nb, TcMode mode, const float* w,
                const float* fin, float* fout, int cin, int cout) {
  const bool split = mode == TcMode::split;
  if (!split && use_gather_engine(nb->n_kernels) && cin == CH && cout == CH) {
    GatherPlan* G = gplan_fwd(ctx, nb);
    TcPlan* p = nb->tc.get();
    if (G->n_overflow < G->n_super) {
      convert(ctx, fin, nb->perm_in.get(), nb->n_in, p->feat_in);
      p->saved_fin = fin;  // PointConvOp saves its input at forward (conv_op.hpp:138)
      p->saved_c = CH;
      pack_w(ctx, p, w, G->K, false);
      run_gather_kernel(ctx, G, p->feat_in.get(), nb->n_in, p->wpack.get(), nb->perm_out.get(),
                        fout, "conv_fwd_tc");
    }
    const CsrView v{nb->row_ptr.get(), nb->col_j.get(), nb->col_k.get(), nb->n_out, nb->n_pairs};
    mvmr_rows_subset_f32(ctx, v, nb->perm_out.get(), G->spill_rows.get(), G->n_spill, w, fin, CH,
                         CH, fout);
    return;
  }
  TcDirPlan* P = plan_fwd(ctx, nb, wide_pass(cout, split));
  TcPlan* p = nb->tc.get();
  if (P->n_overflow < P->n_super) {
    input_image(ctx, nb, p, fin, cin, split);
    if (split) {
      split_passes(ctx, p, P, w, false, cin, cout, p->feat_in.get(), nb->perm_out.get(), fout,
                   "conv_fwd_tc_split", amax_slot(ctx, p, 0), amax_slot(ctx, p, 1));
    } else {
      pack_w(ctx, p, w, P->K, false, cin, cout);
      run_fwd_kernel(ctx, P, p->feat_in.get(), p->wpack.get(), nb->perm_out.get(), fout, "conv_fwd_tc",
                     nullptr, cin, cout);
    }
  }
  // rows of super-tiles beyond the tile capacities: exact engine on those rows only
  const CsrView v{nb->row_ptr.get(), nb->col_j.get(), nb->col_k.get(), nb->n_out, nb->n_pairs};
  mvmr_rows_subset_f32(ctx, v, nb->perm_out.get(), P->spill_rows.get(), P->n_spill, w, fin, cin,
                       cout, fout);
}

__global__ void k_add_inplace(float* __restrict__ a, const float* __restrict__ b, int64_t n) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x < n) a[x] += b[x];
}

// Exact weight gradient of the rows of overflow tiles (vvor over that subset).
__global__ void k_gather_rows_triplets(const int64_t* __restrict__ row_ptr,
                                       const uint32_t* __restrict__ col,
                                       const uint32_t* __restrict__ kk,
                                       const uint32_t* __restrict__ perm,
                                       const uint32_t* __restrict__ list, int64_t n_list,
                                       const int64_t* __restrict__ off, uint32_t* __restrict__ oi,
                                       uint32_t* __restrict__ oj, uint32_t* __restrict__ ok) {
  const int64_t x = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (x >= n_list) return;
  const uint32_t row = perm[list[x]];
  const int64_t s = row_ptr[row], n = row_ptr[row + 1] - s;
  for (int64_t q = lane; q < n; q += 32) {
    oi[off[x] + q] = row;
    oj[off[x] + q] = col[s + q];
    ok[off[x] + q] = kk[s + q];
  }
}
__global__ void k_row_lens(const int64_t* __restrict__ row_ptr, const uint32_t* __restrict__ perm,
                           const uint32_t* __restrict__ list, int64_t n_list,
                           int64_t* __restrict__ len) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x < n_list) {
    const uint32_t row = perm[list[x]];
    len[x] = row_ptr[row + 1] - row_ptr[row];
  }
}

template <int NOUT, bool SPLIT = false>
static void launch_wgrad(npcg_context* ctx, const WgArgs& a, int hcap, dim3 grid, bool big) {
  const WgSmem L = wg_smem_layout<NOUT>(hcap);
  auto kern = big ? k_conv_wgrad_tc<NOUT, true, SPLIT> : k_conv_wgrad_tc<NOUT, false, SPLIT>;
  NPCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(L.total)));
  launch(ctx, SPLIT ? "conv_wgrad_tc_split" : "conv_wgrad_tc", kern, grid, dim3(WG_THREADS), L.total,
         a);
}

// Exact weight gradient of the rows a plan left to the exact engine (vvor
// over their triplets).  transposed: the plan's rows are input points j (the
// fused backward's plan over the transposed structure).
static void wgrad_spill(npcg_context* ctx, npcg_neighbors* nb, TcDirPlan* P, const float* fin,
                        const float* gout, float* grad_w, bool accumulate, int cin, int cout,
                        bool transposed = false) {
  const int K = static_cast<int>(nb->n_kernels);
  const int64_t* rp = transposed ? nb->tcsr->row_ptr.get() : nb->row_ptr.get();
  const uint32_t* cc = transposed ? nb->tcsr->col.get() : nb->col_j.get();
  const uint32_t* ck = transposed ? nb->tcsr->k.get() : nb->col_k.get();
  const uint32_t* perm = transposed ? nb->perm_in.get() : nb->perm_out.get();
  DevBuf<int64_t> len(ctx, P->n_spill + 1), off(ctx, P->n_spill + 1);
  NPCG_CUDA(cudaMemsetAsync(len.get(), 0, (P->n_spill + 1) * 8, ctx->stream));
  launch(ctx, "spill_lens", k_row_lens, dim3(static_cast<unsigned>(ceil_div(P->n_spill, 256))),
         dim3(256), 0, rp, perm, static_cast<const uint32_t*>(P->spill_rows.get()), P->n_spill, len.get());
  int64_t total = 0;
  exclusive_scan_i64(ctx, len.get(), off.get(), P->n_spill + 1, &total);
  DevBuf<uint32_t> ti(ctx, total), tj(ctx, total), tk(ctx, total);
  // (row, col, k) -> (i, j, k), rows are j when transposed
  launch(ctx, "spill_gather", k_gather_rows_triplets,
         dim3(static_cast<unsigned>(ceil_div(P->n_spill * 32, 256))), dim3(256), 0, rp, cc, ck, perm,
         static_cast<const uint32_t*>(P->spill_rows.get()), P->n_spill,
         static_cast<const int64_t*>(off.get()), transposed ? tj.get() : ti.get(),
         transposed ? ti.get() : tj.get(), tk.get());
  npcg_triplets T{ti.get(), tj.get(), tk.get(), total, nb->n_out, nb->n_in, K, 0};
  CellPlan cells;
  cells_from_triplets(ctx, &T, K, &cells);
  if (!accumulate) {
    vvor_cells<float>(ctx, cells, gout, fin, 1, cin, cout, grad_w);
    return;
  }
  const int64_t nw = static_cast<int64_t>(K) * cin * cout;
  DevBuf<float> tmp(ctx, nw);
  vvor_cells<float>(ctx, cells, gout, fin, 1, cin, cout, tmp.get());
  launch(ctx, "add_inplace", k_add_inplace, dim3(static_cast<unsigned>(ceil_div(nw, 256))),
         dim3(256), 0, grad_w, static_cast<const float*>(tmp.get()), nw);
}

// The fused backward (one aggregation for dgrad + wgrad) serves the bf16
// path at K = 27, C_in, C_out <= 64; NPCG_FUSED_BWD=0 disables it (A/B).
static bool fused_bwd_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("NPCG_FUSED_BWD");
    v = (e && std::strcmp(e, "0") == 0) ? 0 : 1;
  }
  return v == 1;
}

static void run_fused_backward(npcg_context* ctx, npcg_neighbors* nb, TcPlan* p, TcDirPlan* P,
                               float* grad_in, float* grad_w, int cin, int cout) {
  const int K = static_cast<int>(nb->n_kernels);
  const int npairs = std::max(1, std::min(P->n_items, ctx->num_sms / 2));
  const int64_t need = static_cast<int64_t>(npairs) * K * 64 * 64;
  if (p->partial.size() < need) p->partial.alloc(ctx, need);
  if (!BF_FLAGS) NPCG_CUDA(cudaMemsetAsync(grad_in, 0, nb->n_in * cin * sizeof(float), ctx->stream));
  if (BF_FLAGS) {
    if (p->bf_flags.size() < static_cast<int64_t>(P->n_items) * 4) {
      p->bf_flags.alloc(ctx, static_cast<int64_t>(P->n_items) * 4);
      NPCG_CUDA(cudaMemsetAsync(p->bf_flags.get(), 0, P->n_items * 16, ctx->stream));
      p->bf_gen = 0;
    }
    if (++p->bf_gen == 0) {  // wrapped: flags of a previous launch could match
      NPCG_CUDA(cudaMemsetAsync(p->bf_flags.get(), 0, p->bf_flags.size() * 4, ctx->stream));
      p->bf_gen = 1;
    }
  }
  BfArgs a{};
  a.item_flag = p->bf_flags.get();
  a.gen = p->bf_gen;
  a.halo = P->halo.get();
  a.halo_len = P->halo_len.get();
  a.blk_off = P->blk_off.get();
  a.blocks = P->blocks.get();
  a.perm_rows = nb->perm_in.get();
  a.sup = P->sup.get();
  a.tiles = P->tiles.get();
  a.item_start = P->item_start.get();
  a.n_items = P->n_items;
  a.hcap = P->hcap;
  a.K = K;
  a.feat = p->feat_out.get();
  a.fimg = p->feat_in.get();
  a.wpack = p->wpack.get();
  a.gin = grad_in;
  a.gin_cols = cin;
  a.partial = p->partial.get();
  // the two halves of the cells, load-balanced like the weight gradient's runs
  // (7 pairs each); the 13-cell half is padded with a zero stage
  uint8_t korder[KMAX];
  wgrad_cell_order(P, K, BF_STAGES / 2, 2, korder);
  for (int x = 0; x < 2 * BF_STAGES; ++x) a.cells[x] = x < K ? korder[x] : BF_ZERO;
  const BfSmem L = bf_smem_layout(P->hcap);
  auto kern = P->big_blocks ? k_conv_bwd_fused<true> : k_conv_bwd_fused<false>;
  NPCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(L.total)));
  static const bool bprof = std::getenv("NPCG_BF_PROFILE") != nullptr;
  DevBuf<long long> prof;
  if (bprof) {
    prof.alloc(ctx, 6 * npairs);
    NPCG_CUDA(cudaMemsetAsync(prof.get(), 0, 48 * npairs, ctx->stream));
    a.prof = prof.get();
  }
  launch_cluster(ctx, "conv_bwd_fused", kern, dim3(2 * npairs), dim3(FWD_THREADS), L.total, 2, a);
  if (bprof) {  // (debug: synchronises)
    std::vector<long long> h(6 * npairs);
    NPCG_CUDA(cudaMemcpy(h.data(), prof.get(), h.size() * 8, cudaMemcpyDeviceToHost));
    double bnd = 0, tot = 0, wt = 0;
    for (int x = 0; x < 2 * npairs; ++x) {
      bnd += static_cast<double>(h[3 * x]);
      tot += static_cast<double>(h[3 * x + 1]);
      wt += static_cast<double>(h[3 * x + 2]);
    }
    std::fprintf(stderr, "[npcg fused profile] halo boundaries %.1f %% of the aggregation loop (of which %.1f %% "
                 "waiting for the last group of the record; %.0f clocks per CTA)\n",
                 100.0 * bnd / std::max(tot, 1.0), 100.0 * wt / std::max(tot, 1.0), tot / (2 * npairs));
  }
  const int64_t nw = static_cast<int64_t>(K) * cin * cout;
  launch(ctx, "wgrad_reduce", k_wgrad_reduce_mc, dim3(static_cast<unsigned>(ceil_div(nw, 256))), dim3(256),
         0, static_cast<const float*>(p->partial.get()), npairs, K, cin, cout, grad_w);
}

void tc_backward(npcg_context* ctx, npcg_neighbors* nb, TcMode mode, const float* w,
                 const float* fin, const float* gout, float* grad_in, float* grad_w, int cin,
                 int cout, bool fin_unchanged) {
  const bool split = mode == TcMode::split;
  TcPlan* p = get_plan(ctx, nb);
  const int K = static_cast<int>(nb->n_kernels);
  bool g_converted = false;
  auto g_image = [&] {
    if (split) convert_split(ctx, gout, nb->perm_out.get(), nb->n_out, p->feat_out, cout, amax_slot(ctx, p, 2));
    else convert(ctx, gout, nb->perm_out.get(), nb->n_out, p->feat_out, cout);
    g_converted = true;
  };
  if (!split && grad_in && grad_w && K == 27 && tc_pad(cin) == CH && tc_pad(cout) == CH &&
      fused_bwd_enabled() && !use_gather_engine(nb->n_kernels)) {
    // one aggregation pass feeds both gradients (over 128-row super-tiles)
    TcDirPlan* P = plan_bwd(ctx, nb, true);
    if (!fin_unchanged || fin != p->saved_fin || cin != p->saved_c || p->saved_split)
      input_image(ctx, nb, p, fin, cin, false);
    g_image();
    pack_w(ctx, p, w, K, true, cin, cout);
    if (P->n_overflow < P->n_super) {
      run_fused_backward(ctx, nb, p, P, grad_in, grad_w, cin, cout);
    } else {
      NPCG_CUDA(cudaMemsetAsync(grad_w, 0, static_cast<int64_t>(K) * cin * cout * 4, ctx->stream));
    }
    if (P->n_spill) {  // rows beyond the tile capacities: exact engines on those rows
      DevBuf<float> wt(ctx, static_cast<int64_t>(K) * cin * cout);
      transpose_w<float>(ctx, w, K, cin, cout, wt.get());
      mvmr_rows_subset_f32(ctx, nb->tcsr->view(), nb->perm_in.get(), P->spill_rows.get(), P->n_spill,
                           wt.get(), gout, cout, cin, grad_in);
      wgrad_spill(ctx, nb, P, fin, gout, grad_w, true, cin, cout, true);
    }
    return;
  }
  if (grad_in && !split && use_gather_engine(nb->n_kernels) && cin == CH && cout == CH) {
    GatherPlan* G = gplan_bwd(ctx, nb);
    if (G->n_overflow < G->n_super) {
      convert(ctx, gout, nb->perm_out.get(), nb->n_out, p->feat_out);
      g_converted = true;
      pack_w(ctx, p, w, K, true);
      run_gather_kernel(ctx, G, p->feat_out.get(), nb->n_out, p->wpack.get(), nb->perm_in.get(),
                        grad_in, "conv_dgrad_tc");
    }
    if (G->n_spill) {
      DevBuf<float> wt(ctx, static_cast<int64_t>(K) * CH * CH);
      transpose_w<float>(ctx, w, K, CH, CH, wt.get());
      mvmr_rows_subset_f32(ctx, nb->tcsr->view(), nb->perm_in.get(), G->spill_rows.get(),
                           G->n_spill, wt.get(), gout, CH, CH, grad_in);
    }
  } else if (grad_in) {
    TcDirPlan* P = plan_bwd(ctx, nb, wide_pass(cin, split));
    if (P->n_overflow < P->n_super) {
      g_image();
      if (split) {
        split_passes(ctx, p, P, w, true, cin, cout, p->feat_out.get(), nb->perm_in.get(), grad_in,
                     "conv_dgrad_tc_split", amax_slot(ctx, p, 2), amax_slot(ctx, p, 3));
      } else {
        pack_w(ctx, p, w, K, true, cin, cout);
        run_fwd_kernel(ctx, P, p->feat_out.get(), p->wpack.get(), nb->perm_in.get(), grad_in,
                       "conv_dgrad_tc", nullptr, cout, cin);
      }
    }
    if (P->n_spill) {
      DevBuf<float> wt(ctx, static_cast<int64_t>(K) * cin * cout);
      transpose_w<float>(ctx, w, K, cin, cout, wt.get());
      mvmr_rows_subset_f32(ctx, nb->tcsr->view(), nb->perm_in.get(), P->spill_rows.get(),
                           P->n_spill, wt.get(), gout, cout, cin, grad_in);
    }
  }
  if (grad_w) {
    // same rows and gathers as the forward (split: the pass writes 2 x C_out columns)
    TcDirPlan* P = plan_fwd(ctx, nb, wide_pass(cout, split));
    if (P->n_overflow == P->n_super) {
      wgrad_spill(ctx, nb, P, fin, gout, grad_w, false, cin, cout);
      return;
    }
    // the bf16 input image made by the forward on this handle is reused when
    // the caller vouches that the backward's input is that same, unmodified
    // buffer (NPCG_FLAG_FIN_UNCHANGED: the operator's saved copy)
    if (!fin_unchanged || fin != p->saved_fin || cin != p->saved_c || split != p->saved_split)
      input_image(ctx, nb, p, fin, cin, split);
    if (!g_converted) g_image();
    const int cinp = tc_pad(cin), coutp = tc_pad(cout);
    // split: chunks of 32 real input channels, 2 x C_out accumulator columns;
    // C_out > 128 runs as 128-channel halves of the G image (the kernel holds
    // at most 256 accumulator columns)
    const int nci = split ? cinp / 32 : cinp / CH;
    for (int m0 = 0; m0 < cout; m0 += split ? 128 : cout) {
      const int mc = split ? std::min(128, cout - m0) : cout;  // output channels of this pass
      const int mcp = tc_pad(mc);
      const int nw = split ? 2 * mcp : coutp;  // accumulator columns (the kernel's NOUT)
      const int np = nw == 64 ? WgCfg<64>::pairs : nw == 128 ? WgCfg<128>::pairs : WgCfg<256>::pairs;
      const int gpc = (K + 2 * np - 1) / (2 * np);  // cell groups per C_in chunk
      const int groups = nci * gpc;
      // one CTA per SM in total over (super-tile slices x groups)
      const int gx = std::max(1, std::min(P->n_super, ctx->num_sms / groups));
      const int64_t need = static_cast<int64_t>(gx) * K * nci * CH * nw;
      if (p->partial.size() < need) p->partial.alloc(ctx, need);
      NPCG_CUDA(cudaMemsetAsync(p->partial.get(), 0, need * 4, ctx->stream));
      WgArgs a{};
      a.halo = P->halo.get();
      a.halo_len = P->halo_len.get();
      a.blk_off = P->blk_off.get();
      a.blocks = P->blocks.get();
      a.sup = P->sup.get();
      a.tiles = P->tiles.get();
      a.n_rows = P->n_rows;
      a.n_sub = P->n_sub;
      a.n_super = P->n_super;
      a.st = P->st;
      a.hcap = P->hcap;
      a.K = K;
      a.nci = nci;
      a.gpc = gpc;
      a.feat = p->feat_in.get();
      a.dense = p->feat_out.get() + (split ? 2 * m0 : 0);
      a.dense_stride = split ? 2 * coutp : coutp;
      a.partial = p->partial.get();
      a.seg = split_segment();
      wgrad_cell_order(P, K, np, gpc, a.korder);
      const dim3 grid(gx, groups);
      const int64_t nwt = static_cast<int64_t>(K) * cin * mc;
      if (split) {
        if (nw == 128) launch_wgrad<128, true>(ctx, a, P->hcap, grid, P->big_blocks);
        else launch_wgrad<256, true>(ctx, a, P->hcap, grid, P->big_blocks);
        launch(ctx, "wgrad_reduce", k_wgrad_reduce_split, dim3(static_cast<unsigned>(ceil_div(nwt, 256))),
               dim3(256), 0, static_cast<const float*>(p->partial.get()), gx, K, cin, mc, 2 * cinp, nw,
               static_cast<const uint32_t*>(amax_slot(ctx, p, 0)),
               static_cast<const uint32_t*>(amax_slot(ctx, p, 2)), grad_w, m0, cout);
      } else {
        if (coutp == 64) launch_wgrad<64>(ctx, a, P->hcap, grid, P->big_blocks);
        else if (coutp == 128) launch_wgrad<128>(ctx, a, P->hcap, grid, P->big_blocks);
        else launch_wgrad<256>(ctx, a, P->hcap, grid, P->big_blocks);
        launch(ctx, "wgrad_reduce", k_wgrad_reduce, dim3(static_cast<unsigned>(ceil_div(nwt, 256))),
               dim3(256), 0, static_cast<const float*>(p->partial.get()), gx, K, cin, cout, cinp, coutp,
               grad_w);
      }
    }
    if (P->n_spill) wgrad_spill(ctx, nb, P, fin, gout, grad_w, true, cin, cout);
  }
}

// Cell runs of the weight gradient: gpc runs of 2 x np slots (the last one
// short), each run swept by its own CTAs over every super-tile, so a run's
// time follows the entries of its cells -- uneven by ~15 % with index-order
// runs (the centre and face cells are the dense ones).  Cells go to runs by
// longest-processing-time greedy on (entries + a per-row cost), and within a
// run in descending order so the two cells of a pair (aggregated side by
// side) have similar loads.  Each cell's sum keeps its order (same CTAs, same
// super-tiles), so the result does not depend on the assignment.
static void wgrad_cell_order(const TcDirPlan* P, int K, int np, int gpc, uint8_t* korder) {
  std::vector<double> cost(K, 1.0);
  if (static_cast<int>(P->k_count.size()) == K)
    for (int k = 0; k < K; ++k) cost[k] = static_cast<double>(P->k_count[k]) + 0.5 * P->n_rows;
  std::vector<int> by(K);
  for (int k = 0; k < K; ++k) by[k] = k;
  std::stable_sort(by.begin(), by.end(), [&](int x, int y) { return cost[x] > cost[y]; });
  std::vector<std::vector<int>> run(gpc);
  std::vector<double> load(gpc, 0.0);
  for (int k : by) {
    int best = -1;
    for (int r = 0; r < gpc; ++r) {
      const int cap = std::min(2 * np, K - r * 2 * np);
      if (static_cast<int>(run[r].size()) < cap && (best < 0 || load[r] < load[best])) best = r;
    }
    run[best].push_back(k);  // cells arrive in descending cost: each run stays sorted
    load[best] += cost[k];
  }
  for (int r = 0; r < gpc; ++r)
    for (size_t x = 0; x < run[r].size(); ++x) korder[r * 2 * np + x] = static_cast<uint8_t>(run[r][x]);
}

// Debug: one traced forward; trace_host receives TRACE_STAGES x TRACE_EV clocks.
void tc_trace_forward(npcg_context* ctx, npcg_neighbors* nb, const float* w, const float* fin,
                      float* fout, int64_t* trace_host) {
  TcPlan* p = get_plan(ctx, nb);
  DevBuf<long long> tr(ctx, TRACE_STAGES * TRACE_EV);
  NPCG_CUDA(cudaMemsetAsync(tr.get(), 0, TRACE_STAGES * TRACE_EV * 8, ctx->stream));
  if (use_gather_engine(nb->n_kernels)) {
    GatherPlan* G = gplan_fwd(ctx, nb);
    convert(ctx, fin, nb->perm_in.get(), nb->n_in, p->feat_in);
    p->saved_fin = fin;
    p->saved_c = CH;
    pack_w(ctx, p, w, G->K, false);
    run_gather_kernel(ctx, G, p->feat_in.get(), nb->n_in, p->wpack.get(), nb->perm_out.get(), fout,
                      "conv_fwd_tc_traced", tr.get());
  } else {
    TcDirPlan* P = plan_fwd(ctx, nb);
    convert(ctx, fin, nb->perm_in.get(), nb->n_in, p->feat_in);
    p->saved_fin = fin;
    p->saved_c = CH;
    pack_w(ctx, p, w, P->K, false);
    run_fwd_kernel(ctx, P, p->feat_in.get(), p->wpack.get(), nb->perm_out.get(), fout,
                   "conv_fwd_tc_traced", tr.get());
  }
  NPCG_CUDA(cudaMemcpyAsync(trace_host, tr.get(), TRACE_STAGES * TRACE_EV * 8,
                            cudaMemcpyDeviceToHost, ctx->stream));
  NPCG_CUDA(cudaStreamSynchronize(ctx->stream));
}

// plan statistics for the bench / tests: [n_super, n_overflow, max_halo, mean_halo*100] x 3 dirs
void tc_plan_stats(npcg_context* ctx, npcg_neighbors* nb, int64_t* out12) {
  // the plans of the 64-channel bf16 passes: forward, and dgrad / wgrad (the
  // fused backward's 128-row transposed plan at K = 27, else the transposed
  // plan of the dgrad and the forward plan of the wgrad)
  tc_prepare(ctx, nb, TcMode::bf16);
  TcPlan* p = nb->tc.get();
  const bool fused = p->bwd1 && nb->n_kernels == 27 && fused_bwd_enabled();
  const TcDirPlan* ds[3] = {p->fwd.get(), fused ? p->bwd1.get() : p->bwd.get(),
                            fused ? p->bwd1.get() : p->fwd.get()};  // wgrad runs on the forward plan
  for (int i = 0; i < 3; ++i) {
    out12[4 * i + 0] = ds[i]->n_super;
    out12[4 * i + 1] = ds[i]->n_spill;
    out12[4 * i + 2] = ds[i]->max_halo;
    out12[4 * i + 3] = static_cast<int64_t>(ds[i]->mean_halo * 100);
  }
}

}  // namespace npcg
