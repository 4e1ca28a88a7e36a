// Microbenchmark: TMEM read bandwidth per SM with tcgen05.ld.32x32b.{x32,x64} from W warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2602_21247_b200/csrc tools/micro/tmem_bw.cu -o /tmp/tmem_bw
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace pipnn;

template <int X>
__global__ void tmem_read(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t taddr_sh;
  const int warp = threadIdx.x / 32;
  if (warp == 0) ptx::tmem_alloc(&taddr_sh, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = taddr_sh;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t col = (uint32_t)(((warp >> 2) * X + i * X * 4) & 511);
    if (X == 64) {
      uint32_t v[64];
      ptx::tmem_ld64(tmem + lane_base + col, v);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 64; ++j) acc ^= v[j];
    } else {
      uint32_t v[32];
      ptx::tmem_ld32(tmem + lane_base + col, v);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= v[j];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 4096;
  for (int W : {4, 8, 12, 16}) {
    for (int X : {32, 64}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (X == 32) tmem_read<32><<<148, W * 32>>>(iters, cyc, sink);
        else tmem_read<64><<<148, W * 32>>>(iters, cyc, sink);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double mean = 0;
      for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
      const double bytes = (double)W * 32 * X * 4 * iters;
      printf("W=%2d x%d: %.0f cycles, %.1f B/cycle/SM, %.1f cycles per 128x128 fp32 tile\n", W, X, mean,
             bytes / mean, 65536.0 / (bytes / mean));
    }
  }
  return 0;
}
