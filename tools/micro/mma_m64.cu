// Microbenchmark: where an M = 64 tcgen05.mma (cta_group::1, kind::f16)
// accumulator lives in TMEM, and whether two M = 64 accumulators can share
// columns through a lane offset in the D address.  D[m][n] = m + 1 (A column
// 0 = m + 1, B column 0 = 1); prints the lane -> value map.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mma_m64 mma_m64.cu
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;

__global__ void k_m64(const uint8_t* a_img, const uint8_t* b_img, uint32_t lane_off, int two,
                      float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s = (smem_u32(sm) + 1023u) & ~1023u;
  uint8_t* g = sm + (s - smem_u32(sm));
  for (int x = threadIdx.x; x < 16384 + 8192; x += blockDim.x) g[x] = x < 16384 ? a_img[x] : b_img[x - 16384];
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<64>(smem_u32(&slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // zero the accumulator columns first (every lane) so untouched lanes read 0
  {
    const int w = threadIdx.x >> 5;
    uint32_t z[16];
    for (int x = 0; x < 16; ++x) z[x] = 0;
    for (int q = 0; q < 4; ++q)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
              tmem + (static_cast<uint32_t>(32 * w) << 16) + 16 * q),
          "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]), "r"(z[8]),
          "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t idesc = idesc_bf16(64, 64, false, false);
  if (threadIdx.x < 32) {
    if (elect_one()) {
      const uint64_t ad = sdesc_sw128(s, 16, 1024), bd = sdesc_sw128(s + 16384, 16, 1024);
      umma_bf16(tmem + (lane_off << 16), ad, bd, idesc, 1u);
      if (two) umma_bf16(tmem, ad + (8192 >> 4), bd, idesc, 1u);  // rows 64..127 of the A image
      umma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int q = 0; q < 4; ++q) {
    uint32_t v[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(32 * w) << 16) + 16 * q, v);
    tmem_ld_wait();
    for (int x = 0; x < 16; ++x) out[(32 * w + l) * 64 + 16 * q + x] = __uint_as_float(v[x]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_free<64>(tmem);
}

static uint16_t bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return static_cast<uint16_t>((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}
static size_t sw(int row, int col) { return row * 128 + ((((col >> 3) ^ (row & 7)) & 7) << 4) + ((col & 7) << 1); }

int main() {
  std::vector<uint8_t> ai(16384, 0), bi(8192, 0);
  for (int r = 0; r < 128; ++r) {
    const uint16_t h = bf(static_cast<float>(r + 1));
    std::memcpy(&ai[sw(r, 0)], &h, 2);
  }
  for (int n = 0; n < 64; ++n) {
    const uint16_t h = bf(1.f + n / 64.f);  // column n scaled: value = (m + 1) (1 + n / 64)
    std::memcpy(&bi[sw(n, 0)], &h, 2);
  }
  uint8_t *da, *db;
  float* dout;
  cudaMalloc(&da, ai.size());
  cudaMalloc(&db, bi.size());
  cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(da, ai.data(), ai.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, bi.data(), bi.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_m64, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 8192 + 1024);
  std::vector<float> out(128 * 64);
  for (uint32_t off : {0u, 16u, 32u, 64u}) {
    for (int two = 0; two < 2; ++two) {
      if (two && off == 0) continue;
      cudaMemset(dout, 0xFF, 128 * 64 * 4);
      k_m64<<<1, 128, 16384 + 8192 + 1024>>>(da, db, off, two, dout);
      const cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
      std::printf("lane offset %u%s: %s\n  lane: value(col 0) / value(col 63)\n", off,
                  two ? " + a second M=64 MMA (rows 64..127) at offset 0" : "", cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
      for (int lane = 0; lane < 128; ++lane)
        if (out[lane * 64] != 0.f)
          std::printf("  %3d: %7.2f / %7.2f\n", lane, out[lane * 64], out[lane * 64 + 63]);
    }
  }
  return 0;
}
