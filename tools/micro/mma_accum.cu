// Microbenchmark: the rounding of tcgen05.mma (kind::f16, bf16 in, fp32
// accumulate) when one TMEM accumulator sums a long chain of K=16 MMAs.
// Compares the hardware result, bit for bit, with fp32 emulations of
// D = round(D + sum of the 16 exact products) under round-to-nearest and
// round-toward-zero, and reports the error growth against the exact (fp64)
// sum.  Decides how long an accumulation chain the fp32-contract path may
// keep in TMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mma_accum mma_accum.cu
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;

constexpr int NT = 4;  // A tiles (128 x 64 bf16, SW128 K-major)

__global__ void k_chain(const uint8_t* a_img, const uint8_t* b_img, int steps, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s = (smem_u32(sm) + 1023u) & ~1023u;
  uint8_t* g = sm + (s - smem_u32(sm));
  for (int x = threadIdx.x; x < NT * 16384 + 8192; x += blockDim.x)
    g[x] = x < NT * 16384 ? a_img[x] : b_img[x - NT * 16384];
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
  constexpr uint32_t idesc = idesc_bf16(128, 64, false, false);
  if (threadIdx.x < 32) {
    if (elect_one()) {
      for (int st = 0; st < steps; ++st) {
        const int t = st % NT, ks = (st / NT) % 4;
        const uint64_t ad = sdesc_sw128(s + t * 16384, 16, 1024) + 2u * ks;
        const uint64_t bd = sdesc_sw128(s + NT * 16384, 16, 1024) + 2u * ks;
        umma_bf16(tmem, ad, bd, idesc, st > 0 ? 1u : 0u);
      }
      umma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // lane = row, 64 columns
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

static uint16_t bf(float f) {  // RN to bf16 bits
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return static_cast<uint16_t>(u >> 16);
}
static float fbf(uint16_t h) {
  uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
static size_t sw(int row, int col) {
  return row * 128 + ((((col >> 3) ^ (row & 7)) & 7) << 4) + ((col & 7) << 1);
}
static float rz(double x) {  // round toward zero to fp32
  float f = static_cast<float>(x);
  if (std::fabs(static_cast<double>(f)) > std::fabs(x)) f = std::nextafter(f, 0.0f);
  return f;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? std::atoi(argv[1]) : 0;  // 0 random, 1 mixed-sign biased
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<uint16_t> A(NT * 128 * 64), B(64 * 64);
  std::vector<uint8_t> ai(NT * 16384), bi(8192);
  for (int t = 0; t < NT; ++t)
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 64; ++c) {
        const double v = mode == 1 ? 0.5 + 0.5 * U(rng) : U(rng);
        const uint16_t h = bf(static_cast<float>(v));
        A[(t * 128 + r) * 64 + c] = h;
        std::memcpy(&ai[t * 16384 + sw(r, c)], &h, 2);
      }
  for (int n = 0; n < 64; ++n)
    for (int c = 0; c < 64; ++c) {
      const uint16_t h = bf(static_cast<float>(U(rng)));
      B[n * 64 + c] = h;
      std::memcpy(&bi[sw(n, c)], &h, 2);
    }
  uint8_t *da, *db;
  float* dout;
  cudaMalloc(&da, ai.size());
  cudaMalloc(&db, bi.size());
  cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(da, ai.data(), ai.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, bi.data(), bi.size(), cudaMemcpyHostToDevice);
  const size_t smem = NT * 16384 + 8192 + 1024;
  cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  std::vector<float> out(128 * 64);
  for (int steps : {1, 4, 16, 64, 256, 1024, 4096}) {
    k_chain<<<1, 128, smem>>>(da, db, steps, dout);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    int eq_rn = 0, eq_rz = 0;
    double err = 0, err_rn = 0, err_rz = 0, mag = 0;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < 64; ++n) {
        double ex = 0;
        float drn = 0, drz = 0;
        for (int st = 0; st < steps; ++st) {
          const int t = st % NT, ks = (st / NT) % 4;
          double p = 0;
          for (int k = 0; k < 16; ++k)
            p += static_cast<double>(fbf(A[(t * 128 + r) * 64 + 16 * ks + k])) *
                 fbf(B[n * 64 + 16 * ks + k]);
          ex += p;
          drn = static_cast<float>(static_cast<double>(drn) + p);
          drz = rz(static_cast<double>(drz) + p);
        }
        const float g = out[r * 64 + n];
        eq_rn += g == drn;
        eq_rz += g == drz;
        err = std::max(err, std::fabs(g - ex));
        err_rn = std::max(err_rn, std::fabs(drn - ex));
        err_rz = std::max(err_rz, std::fabs(drz - ex));
        mag = std::max(mag, std::fabs(ex));
      }
    std::printf("mode %d steps %5d: bit-equal RN-emul %5d / 8192, RZ-emul %5d / 8192; rel err hw %.2e  "
                "RN %.2e  RZ %.2e  (%s)\n",
                mode, steps, eq_rn, eq_rz, err / mag, err_rn / mag, err_rz / mag,
                cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
