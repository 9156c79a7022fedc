// N warps wait (bare try_wait loop) on one mbarrier completed after `delay`
// cycles by the last warp; report average probes per waiting warp.
#include <cstdio>
#include <cstdint>
#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;
__global__ void k(long long* out, int nwait, long long delay, int distinct) {
  __shared__ __align__(8) uint64_t b[32];
  __shared__ unsigned long long probes_sum;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < 32; ++i) mbar_init(smem_u32(&b[i]), distinct == 2 ? 40 : 1); probes_sum = 0; fence_barrier_init(); }
  __syncthreads();
  if (w == nwait) {
    const long long t0 = clock64();
    while (clock64() - t0 < delay) {}
    if (distinct == 2) {  // 40 partial arrivals, one every 5K cycles
      for (int a = 0; a < 40; ++a) { const long long t = clock64(); while (clock64() - t < 5000) {} if (l == 0) mbar_arrive(smem_u32(&b[0])); }
    } else if (l == 0) for (int i = 0; i < 32; ++i) mbar_arrive(smem_u32(&b[i]));
  } else if (w < nwait) {
    long long probes = 0;
    const uint32_t bb = smem_u32(&b[distinct == 1 ? w : 0]);
    while (!mbar_try_wait(bb, 0)) ++probes;
    if (l == 0) atomicAdd(&probes_sum, (unsigned long long)probes);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[0] = probes_sum;
}
int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  for (int distinct = 0; distinct < 3; ++distinct)
    for (int nw : {1, 8}) {
      k<<<1, 32 * (nw + 1)>>>(d, nw, 200000, distinct);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%s barriers, %2d waiting warps, 200K-cycle wait: %.1f probes/warp %s\n", distinct == 2 ? "partial-arrivals" : distinct ? "distinct" : "shared  ", nw, (double)h / nw, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
