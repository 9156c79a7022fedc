// Microbenchmark: TMA tile::gather4 (sm_100a) of arbitrary 128-byte rows of a
// bf16 (n x 64) matrix into consecutive shared-memory rows, the halo-load
// shape of the conv kernels.  Checks the bytes, then times H-row halo loads
// (gather4 issued by one warp, complete_tx on one mbarrier) against the
// 16-byte cp.async loop of coop_load_halo.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o gather4 gather4.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, int c0, int r0, int r1, int r2,
                                        int r3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}

// mode 0: gather4 by warp 0 (lanes issue 4 rows each), 1: cp.async by all threads
__global__ void k_halo(const __grid_constant__ CUtensorMap map, const __nv_bfloat16* feat, const uint32_t* rows,
                       int H, int reps, int mode, uint8_t* out, long long* clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s = smem_u32(sm);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (mode == 0) {
      if (threadIdx.x < 32) {
        if (threadIdx.x == 0) mbar_expect_tx(smem_u32(&bar), static_cast<uint32_t>(H) * 128u);
        __syncwarp();
        for (int q = threadIdx.x; 4 * q < H; q += 32) {
          int r[4];
          for (int u = 0; u < 4; ++u) r[u] = 4 * q + u < H ? static_cast<int>(rows[4 * q + u]) : static_cast<int>(rows[H - 1]);
          // (a partial last group re-reads row H-1 into padding rows: expect_tx counts whole groups)
          gather4(s + 4 * q * 128u, &map, 0, r[0], r[1], r[2], r[3], smem_u32(&bar));
        }
      }
      mbar_wait(smem_u32(&bar), rep & 1);
    } else {
      const uint32_t q = threadIdx.x & 7;
      for (uint32_t h = threadIdx.x >> 3; h < static_cast<uint32_t>(H); h += blockDim.x >> 3)
        cp_async16(s + h * 128u + q * 16u, reinterpret_cast<const uint8_t*>(feat) + static_cast<int64_t>(rows[h]) * 128 + q * 16);
      cp_async_wait_all();
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  if (blockIdx.x == 0)
    for (int x = threadIdx.x; x < H * 128; x += blockDim.x) out[x] = sm[x];
}

int main() {
  const int n = 1 << 20, H = 752, reps = 50;
  std::vector<uint16_t> h(static_cast<size_t>(n) * 64);
  for (size_t x = 0; x < h.size(); ++x) h[x] = static_cast<uint16_t>(x * 2654435761u >> 7);
  std::mt19937 rng(5);
  std::vector<uint32_t> rows(H);
  uint32_t base = 1000;
  for (int x = 0; x < H; ++x) {  // sorted, with runs (like a halo)
    base += 1 + (rng() % 5 == 0 ? rng() % 300 : 0);
    rows[x] = base % n;
  }
  __nv_bfloat16* d;
  uint32_t* drows;
  uint8_t* dout;
  long long* dclk;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&drows, H * 4);
  cudaMalloc(&dout, H * 128);
  cudaMalloc(&dclk, 148 * 8);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(drows, rows.data(), H * 4, cudaMemcpyHostToDevice);
  CUtensorMap map;
  const cuuint64_t gdim[2] = {64, static_cast<cuuint64_t>(n)};
  const cuuint64_t gstride[1] = {128};
  const cuuint32_t box[2] = {64, 1};
  const cuuint32_t es[2] = {1, 1};
  CUresult cr = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, gdim, gstride, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("encode: %d\n", static_cast<int>(cr));
  const int smem = (H + 4) * 128;
  cudaFuncSetAttribute(k_halo, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dout, 0, H * 128);
    k_halo<<<148, 512, smem>>>(map, d, drows, H, reps, mode, dout, dclk);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint8_t> o(H * 128);
    std::vector<long long> clk(148);
    cudaMemcpy(o.data(), dout, o.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(clk.data(), dclk, 148 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int x = 0; x < H; ++x)
      for (int c = 0; c < 64; ++c) {
        uint16_t v;
        std::memcpy(&v, &o[x * 128 + 2 * c], 2);
        bad += v != h[static_cast<size_t>(rows[x]) * 64 + c];
      }
    std::sort(clk.begin(), clk.end());
    std::printf("%s: %s, wrong values %d, cycles per %d-row halo load: median %.0f (max %.0f)\n",
                mode == 0 ? "gather4 " : "cp.async", cudaGetErrorString(e), bad, H, clk[74] / double(reps),
                clk[147] / double(reps));
  }
  return 0;
}
