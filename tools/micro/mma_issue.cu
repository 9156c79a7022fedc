// Microbenchmark: issue rate of tcgen05.mma (bf16, SS, cta_group::1) from one
// elected lane, per "stage" of 4 MMAs (K = 64) + commits, with operands
// already in smem; shapes M128 x N{64,128,256} (the conv kernels' M128 N64
// stage) and M64 x N{64,128,256} (the transposed form D^T = W^T A^T, N = the
// tile rows).  Prints cycles per stage and MACs per cycle.
#include <cstdio>
#include <cstdint>
#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;

template <int NCOMMIT, int N, int M = 128>
__global__ void k(long long* out, int stages) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[4];
  const uint32_t s = smem_u32(sm);
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bars[i]), 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<256>(smem_u32(&slot));
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = idesc_bf16(M, N, false, false);
  const uint64_t ad = sdesc_sw128(s, 16, 1024), bd = sdesc_sw128(s + 65536, 16, 1024);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {
    t0 = clock64();
    for (int st = 0; st < stages; ++st) {
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) umma_bf16(tmem, ad + 2u * ks + (st & 3) * 1024, bd + 2u * ks, idesc, 1u);
#pragma unroll
        for (int c = 0; c < NCOMMIT; ++c) umma_commit(smem_u32(&bars[c]));
      }
      __syncwarp();
    }
    t1 = clock64();
    // wait for completion of the last commit
    if (NCOMMIT > 0) mbar_wait(smem_u32(&bars[0]), (stages - 1) & 1);
    const long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_free<256>(tmem);
}

int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  const int stages = 4096;
  auto run = [&](auto kern, const char* name, double macs = 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    kern<<<1, 128, 100 * 1024>>>(d, stages);
    kern<<<1, 128, 100 * 1024>>>(d, stages);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-28s issue %.1f cyc/stage, complete %.1f cyc/stage, %.0f MAC/clk  (%s)\n", name, (double)h[0] / stages,
           (double)h[1] / stages, macs / ((double)h[1] / stages), cudaGetErrorString(cudaGetLastError()));
  };
  const double m16 = 4.0 * 16;  // K per stage
  run(k<1, 64>, "4xM128N64K16 + 1 commit", m16 * 128 * 64);
  run(k<2, 64>, "4xM128N64K16 + 2 commits", m16 * 128 * 64);
  run(k<3, 64>, "4xM128N64K16 + 3 commits", m16 * 128 * 64);
  run(k<1, 128>, "4xM128N128K16 + 1 commit", m16 * 128 * 128);
  run(k<1, 256>, "4xM128N256K16 + 1 commit", m16 * 128 * 256);
  run(k<1, 64, 64>, "4xM64N64K16 + 1 commit", m16 * 64 * 64);
  run(k<1, 128, 64>, "4xM64N128K16 + 1 commit", m16 * 64 * 128);
  run(k<1, 256, 64>, "4xM64N256K16 + 1 commit", m16 * 64 * 256);
  return 0;
}
