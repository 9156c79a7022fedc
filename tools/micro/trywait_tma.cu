// try_wait probe count while other warps generate async traffic: bulk copies
// completing on another mbarrier (mode 1) or tcgen05 MMAs + commits (mode 2).
#include <cstdio>
#include <cstdint>
#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;
__global__ void k(long long* out, const uint8_t* g, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t b, c;
  __shared__ int stop;
  __shared__ uint32_t slot;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&b), 1); mbar_init(smem_u32(&c), 1); stop = 0; fence_barrier_init(); }
  if (w == 2) tmem_alloc<128>(smem_u32(&slot));
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (w == 1 && mode == 3) {
  } else if (w == 1) {
    const long long t0 = clock64();
    while (clock64() - t0 < 200000) {}
    if (l == 0) mbar_arrive(smem_u32(&b));
  } else if (w == 0) {
    long long probes = 0;
    const long long t0 = clock64();
    while (!mbar_try_wait(smem_u32(&b), 0)) ++probes;
    if (l == 0) { out[0] = probes; atomicExch(&stop, 1); if (mode == 3) out[1] = clock64() - t0; }
  } else if (w == 2 && mode == 3) {
    constexpr uint32_t idesc = idesc_bf16(128, 64, false, false);
    const uint64_t ad = sdesc_sw128(smem_u32(sm), 16, 1024), bd = sdesc_sw128(smem_u32(sm) + 16384, 16, 1024);
    if (elect_one()) {
      for (int st = 0; st < 1000; ++st) for (int ks = 0; ks < 4; ++ks) umma_bf16(slot, ad + 2 * ks, bd + 2 * ks, idesc, 1);
      umma_commit(smem_u32(&b));
    }
    __syncwarp();
    if (l == 0) out[1] = 1000;
  } else if (w == 2 && mode == 1) {
    uint32_t ph = 0; long long n = 0;
    while (!*(volatile int*)&stop) {
      if (l == 0) { mbar_expect_tx(smem_u32(&c), 4096); bulk_g2s(smem_u32(sm), g, 4096, smem_u32(&c)); }
      __syncwarp();
      while (!mbar_try_wait(smem_u32(&c), ph)) {}
      ph ^= 1; ++n;
    }
    if (l == 0) out[1] = n;
  } else if (w == 2 && mode == 2) {
    uint32_t ph = 0; long long n = 0;
    constexpr uint32_t idesc = idesc_bf16(128, 64, false, false);
    const uint64_t ad = sdesc_sw128(smem_u32(sm), 16, 1024), bd = sdesc_sw128(smem_u32(sm) + 16384, 16, 1024);
    while (!*(volatile int*)&stop) {
      if (elect_one()) { for (int ks = 0; ks < 4; ++ks) umma_bf16(slot, ad + 2 * ks, bd + 2 * ks, idesc, 1); umma_commit(smem_u32(&c)); }
      __syncwarp();
      while (!mbar_try_wait(smem_u32(&c), ph)) {}
      ph ^= 1; ++n;
    }
    if (l == 0) out[1] = n;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (w == 2) tmem_free<128>(slot);
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  uint8_t* g; cudaMalloc(&g, 1 << 20); cudaMemset(g, 0, 1 << 20);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(d, 0, 16);
    k<<<1, 96, 64 * 1024>>>(d, g, mode);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): waiter probes %lld over 200K cycles; background ops %lld  %s\n", mode, mode == 0 ? "idle" : mode == 1 ? "bulk copies" : mode == 2 ? "tcgen05 mma+commit" : "wait on a commit barrier behind 1000 MMA stages", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
