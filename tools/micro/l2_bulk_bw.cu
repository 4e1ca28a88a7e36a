// Microbenchmark: L2 -> SMEM bandwidth of 1-D cp.async.bulk (the leaf kernel's B-tile stream), persistent grid
// of one CTA per SM, one producer thread per "pipeline" keeping NS chunks of CH bytes in flight from a buffer
// of BUF bytes (L2-resident when BUF < 126 MB). Prints bytes/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2602_21247_b200/csrc tools/micro/l2_bulk_bw.cu -o /tmp/l2bw
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "ptx.cuh"
using namespace pipnn;

__device__ __forceinline__ bool test_wait(uint32_t a, uint32_t par) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(a), "r"(par) : "memory");
  return ok != 0;
}
__device__ int g_mode;
__device__ __forceinline__ bool wait_mode(uint64_t* bar, uint32_t par, int* err) {
  const int mode = g_mode;
  (void)mode;
  while (!test_wait(ptx::smem_u32(bar), par)) {}
  return true;
}
__global__ void bw(const uint8_t* src, size_t buf, int ch, int ns, int iters, int pipes, int* err) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[8][16];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0)
    for (int p = 0; p < 8; ++p)
      for (int s = 0; s < 16; ++s) ptx::mbar_init(&full[p][s], 1);
  ptx::fence_mbar_init();
  __syncthreads();
  // mode 0: pipe p = warp p, lane 0; mode 1: pipe p = warp 0, lane p
  const int pid = g_mode == 0 ? w : lane;
  if ((g_mode == 0 ? (w < pipes && lane == 0) : (w == 0 && lane < pipes))) {
    const int w = pid;
    uint8_t* ring = sm + (size_t)w * ns * ch;
    const size_t nch = buf / ch;
    uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x * 2 + w + 1);
    for (int i = 0; i < iters + ns; ++i) {
      const int s = i % ns;
      if (i >= ns) {
        if (!wait_mode(&full[w][s], ((i / ns) - 1) & 1, err)) return;
      }
      if (i < iters) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const size_t c = (x >> 20) & (nch - 1);  // nch is a power of two
        ptx::mbar_arrive_expect_tx(&full[w][s], ch);
        ptx::bulk_g2s(ring + (size_t)s * ch, src + c * ch, ch, &full[w][s]);
      }
    }
  }
}

int main(int argc, char** argv) {
  const size_t buf = (size_t)(argc > 1 ? atol(argv[1]) : 64) << 20;
  uint8_t* d;
  int* err;
  cudaMalloc(&d, buf);
  cudaMemset(d, 1, buf);
  cudaMalloc(&err, 4);
  cudaMemset(err, 0, 4);
  int nsm = 148;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode)
  for (int pipes : {1, 2, 4, 8})
    for (int ch : {4096, 16384})
      for (int ns : {2, 8}) {
        cudaMemcpyToSymbol(g_mode, &mode, 4);
        const int smem = pipes * ns * ch;
        if (smem > 200 * 1024) continue;
        cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int iters = (int)((256ll << 20) / ch);
        bw<<<nsm, 256, smem>>>(d, buf, ch, ns, iters / 8, pipes, err);
        cudaEventRecord(a);
        bw<<<nsm, 256, smem>>>(d, buf, ch, ns, iters, pipes, err);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)nsm * pipes * iters * ch;
        printf("mode %d buf %4zu MB pipes %d chunk %6d stages %d: %7.1f GB/s (%.1f KB in flight/SM)\n", mode, buf >> 20, pipes, ch, ns,
               bytes / ms / 1e6, pipes * ns * ch / 1024.0);
      }
  int h = 0;
  cudaMemcpy(&h, err, 4, cudaMemcpyDeviceToHost);
  printf("err %d %s\n", h, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
