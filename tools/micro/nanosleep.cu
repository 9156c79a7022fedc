// Does __nanosleep actually suspend a warp on sm_100 while other warps of the
// CTA churn mbarriers?  Warp 0 sleeps N times for `ns`; warps 1..7 either idle
// or arrive on a private mbarrier in a loop.
#include <cstdio>
#include <cstdint>
#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;
__global__ void k(long long* out, uint32_t ns, int churn, int iters) {
  __shared__ __align__(8) uint64_t b[8];
  __shared__ int stop;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(smem_u32(&b[i]), 1); stop = 0; fence_barrier_init(); }
  __syncthreads();
  if (w == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) __nanosleep(ns);
    long long t1 = clock64();
    if (l == 0) { out[0] = t1 - t0; atomicExch(&stop, 1); }
  } else if (churn) {
    uint32_t ph = 0;
    while (!*(volatile int*)&stop) {
      if (l == 0) mbar_arrive(smem_u32(&b[w]));
      mbar_wait(smem_u32(&b[w]), ph); ph ^= 1;
    }
  }
}
int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  for (int churn = 0; churn < 2; ++churn)
    for (uint32_t ns : {100u, 1000u, 10000u}) {
      k<<<1, 256>>>(d, ns, churn, 200);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("churn=%d nanosleep(%u ns) x200: %.1f cycles/iter  (%.2f ns at 1.9GHz)  %s\n", churn, ns, h / 200.0, h / 200.0 / 1.9, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
