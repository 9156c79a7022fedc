// Microbenchmark: tcgen05.mma.cta_group::2 (an SM pair, M = 256 split 128
// rows per CTA, B split N/2 per CTA) vs cta_group::1, bf16 SS, stages of
// 4 x K16 + one commit, issued by one elected lane of the pair's leader CTA.
// Prints cycles per stage and MACs per clock per SM.  Every wait is bounded
// (a spin limit), so a wrong encoding reports an error instead of hanging.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mma_2sm mma_2sm.cu
#include <cstdint>
#include <cstdio>

#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ bool bounded_wait(uint32_t bar, uint32_t parity) {
  for (long i = 0; i < (1l << 24); ++i)
    if (mbar_try_wait(bar, parity)) return true;
  return false;
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) k_2sm(long long* out, int stages) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s = smem_u32(sm);
  const uint32_t rank = ctarank();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  // M = 256 (the pair), N per the instruction; each CTA holds its 128 A rows and N/2 B rows
  constexpr uint32_t idesc = idesc_bf16(256, N, false, false);
  const uint64_t ad = sdesc_sw128(s, 16, 1024), bd = sdesc_sw128(s + 65536, 16, 1024);
  long long t0 = 0, t1 = 0;
  bool ok = true;
  if (rank == 0 && threadIdx.x < 32) {
    t0 = clock64();
    for (int st = 0; st < stages; ++st) {
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(ad + 2u * ks + (st & 3) * 1024), "l"(bd + 2u * ks), "r"(idesc), "r"(1u)
              : "memory");
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"(static_cast<uint16_t>(3))
            : "memory");
      }
      __syncwarp();
    }
    t1 = clock64();
  }
  // both CTAs: the last stage's commit arrives on each CTA's barrier
  if (threadIdx.x < 32) ok = bounded_wait(smem_u32(&bar), (stages - 1) & 1);
  const long long t2 = clock64();
  if (threadIdx.x == 0 && rank == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t0;
    out[2] = ok ? 1 : 0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 32);
  long long h[3] = {0, 0, 0};
  const int stages = 4096;
  auto run = [&](auto kern, const char* name, double macs_per_sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaMemset(d, 0, 32);
    kern<<<2, 128, 100 * 1024>>>(d, stages);
    kern<<<2, 128, 100 * 1024>>>(d, stages);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    std::printf("%-34s issue %.1f cyc/stage, complete %.1f cyc/stage, %.0f MAC/clk per SM, waits %s (%s)\n", name,
                (double)h[0] / stages, (double)h[1] / stages, macs_per_sm / ((double)h[1] / stages),
                h[2] ? "ok" : "TIMED OUT", cudaGetErrorString(e));
    return e == cudaSuccess;
  };
  const double k64 = 4.0 * 16;
  if (!run(k_2sm<64>, "2SM 4xM256N64K16 + 1 commit", k64 * 128 * 64)) return 1;
  run(k_2sm<128>, "2SM 4xM256N128K16 + 1 commit", k64 * 128 * 128);
  run(k_2sm<256>, "2SM 4xM256N256K16 + 1 commit", k64 * 128 * 256);
  return 0;
}
