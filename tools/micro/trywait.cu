// How long does one mbarrier.try_wait probe block, and does a nanosleep
// backoff loop on an mbarrier really sleep?  Warp 1 completes barrier b after
// `delay` cycles; warp 0 waits with (a) a bare try_wait loop, (b) try_wait +
// nanosleep backoff, (c) test_wait + nanosleep; we count probes.
#include <cstdio>
#include <cstdint>
#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;
__global__ void k(long long* out, int mode, long long delay, int churn) {
  __shared__ __align__(8) uint64_t b, cb[8];
  __shared__ int stop;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&b), 1); for (int i = 0; i < 8; ++i) mbar_init(smem_u32(&cb[i]), 1); stop = 0; fence_barrier_init(); }
  __syncthreads();
  if (w == 1) {
    const long long t0 = clock64();
    while (clock64() - t0 < delay) {}
    if (l == 0) mbar_arrive(smem_u32(&b));
  } else if (w == 0) {
    const long long t0 = clock64();
    long long probes = 0;
    uint32_t ns = 32;
    if (mode == 0) {
      while (!mbar_try_wait(smem_u32(&b), 0)) ++probes;
    } else if (mode == 1) {
      while (!mbar_try_wait(smem_u32(&b), 0)) { ++probes; __nanosleep(ns); if (ns < 1024) ns <<= 1; }
    } else {
      while (!mbar_test_wait(smem_u32(&b), 0)) { ++probes; __nanosleep(ns); if (ns < 1024) ns <<= 1; }
    }
    if (l == 0) { out[0] = clock64() - t0; out[1] = probes; atomicExch(&stop, 1); }
  } else if (churn) {
    uint32_t ph = 0;
    while (!*(volatile int*)&stop) {
      if (l == 0) mbar_arrive(smem_u32(&cb[w]));
      while (!mbar_test_wait(smem_u32(&cb[w]), ph)) {}
      ph ^= 1;
      const long long t = clock64(); while (clock64() - t < 200) {}
    }
  }
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  const char* names[] = {"try_wait spin", "try_wait+sleep", "test_wait+sleep"};
  for (int churn = 0; churn < 2; ++churn)
  for (int mode = 0; mode < 3; ++mode)
    for (long long delay : {20000ll, 200000ll}) {
      k<<<1, churn ? 256 : 64>>>(d, mode, delay, churn);
      printf("churn=%d ", churn);
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%-16s delay %7lld cyc: waited %7lld cyc, %6lld probes (%.0f cyc/probe) %s\n", names[mode], delay, h[0], h[1], h[1] ? (double)h[0] / h[1] : 0.0, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
