// Microbenchmark: throughput of small cp.async.bulk copies (TMA engine) vs
// LDG+STS copies, per SM, from an L2-resident buffer.  Guides the halo /
// descriptor loading design of conv_tc.cu.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2511_23227_b200/csrc/tc_common.cuh"
using namespace npcg::tc;

__global__ void k_bulk(const uint8_t* src, size_t src_bytes, int size, int copies, int reps, long long* cyc) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = smem_u32(&bar);
  if (threadIdx.x == 0) { mbar_init(b, 1); fence_barrier_init(); }
  __syncthreads();
  long long t0 = clock64();
  uint32_t ph = 0;
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) mbar_expect_tx(b, size * copies);
    __syncwarp();
    for (int c = threadIdx.x; c < copies; c += 32) {
      size_t off = ((size_t)(blockIdx.x * 7919 + c * 104729 + r * 31) * 128) % (src_bytes - size);
      off &= ~(size_t)127;
      bulk_g2s(smem_u32(sm) + (c * size) % (64 * 1024), src + off, size, b);
    }
    mbar_wait(b, ph); ph ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ldst(const uint8_t* src, size_t src_bytes, int size, int copies, int reps, long long* cyc) {
  extern __shared__ __align__(128) uint8_t sm[];
  long long t0 = clock64();
  const int chunks = size / 16;
  for (int r = 0; r < reps; ++r) {
    for (int x = threadIdx.x; x < copies * chunks; x += blockDim.x) {
      int c = x / chunks, q = x % chunks;
      size_t off = ((size_t)(blockIdx.x * 7919 + c * 104729 + r * 31) * 128) % (src_bytes - size);
      off &= ~(size_t)127;
      uint4 v = *reinterpret_cast<const uint4*>(src + off + q * 16);
      *reinterpret_cast<uint4*>(sm + ((c * size) % (64 * 1024)) + q * 16) = v;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  size_t bytes = 64ull << 20;  // 64 MB: L2-resident after warm-up
  uint8_t* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  long long* cyc; cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k_ldst, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  long long h[148];
  int sizes[] = {128, 512, 1536, 8192};
  for (int s : sizes) {
    int copies = (s >= 8192) ? 8 : (s >= 1536 ? 32 : 128);
    int reps = 50;
    k_bulk<<<148, 32, 65536>>>(src, bytes, s, copies, reps, cyc);
    cudaDeviceSynchronize();
    k_bulk<<<148, 32, 65536>>>(src, bytes, s, copies, reps, cyc);
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("bulk  size %5d copies/batch %3d: %8.1f cycles/batch, %6.1f cyc/copy, %6.1f B/cyc/SM\n", s, copies, c / reps, c / reps / copies, (double)s * copies * reps / c);
    for (int thr : {128, 512}) {
      k_ldst<<<148, thr, 65536>>>(src, bytes, s, copies, reps, cyc);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
      c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
      printf("ldst%3d size %5d copies/batch %3d: %8.1f cycles/batch, %6.1f cyc/copy, %6.1f B/cyc/SM\n", thr, s, copies, c / reps, c / reps / copies, (double)s * copies * reps / c);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
