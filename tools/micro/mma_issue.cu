// Microbenchmark: tcgen05.mma issue cost in the leaf kernel's style (converged warp, elected lane, uniform
// descriptors), tiles of 5 MMAs (K = 160 B u8) with a commit per tile; one or two issuing warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_21247_b200/csrc tools/micro/mma_issue.cu
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace pipnn;

__global__ void mma_issue(int tiles, int nwarps, int N, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_sh;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (warp == 0) ptx::tmem_alloc(&taddr_sh, 512);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar[0], 1); ptx::mbar_init(&bar[1], 1); ptx::fence_mbar_init(); }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = taddr_sh;
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const uint64_t a_desc = ptx::smem_desc_kmajor_noswz(ptx::smem_u32(sm + warp * 16384), 2048, 128);
    const uint64_t b_desc0 = ptx::smem_desc_kmajor_noswz(ptx::smem_u32(sm + 32768), 2048, 128);
    const uint32_t idesc = ptx::idesc_u8_s32(128, N);
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dtm = tmem + warp * 256 + (t & 1) * 128;
      const uint64_t b_desc = b_desc0 + (uint64_t)((t & 3) * 8 * 128 / 4);
      if (ptx::elect_one()) {
        for (int kc = 0; kc < 10; kc += 2) {
          ptx::mma_i8(dtm, a_desc + (uint64_t)(kc * 128), b_desc + (uint64_t)(kc * 128), idesc, kc > 0);
        }
        ptx::mma_commit(&bar[warp]);
      }
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::mma_commit(&bar[warp]);
    __syncwarp();
    // wait for the last commit: the number of commits is tiles + 1 -> phase parity of completion
    ptx::mbar_wait(&bar[warp], (uint32_t)(tiles & 1), nullptr, 0);
    if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 2 + warp] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 2 * 8);
  cudaFuncSetAttribute(mma_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int tiles = 4000;
  for (int nw : {1, 2, 1, 2})
    for (int N : {128}) {
      for (int rep = 0; rep < 2; ++rep) mma_issue<<<148, 64, 65536>>>(tiles, nw, N, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[296];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 148; ++i) for (int w = 0; w < nw; ++w) mx += h[2 * i + w] / (148.0 * nw);
      printf("warps=%d N=%d: %.1f cycles per tile per warp (5 MMAs), %.1f per MMA per SM\n", nw, N, mx / tiles,
             mx / tiles / 5 / nw);
    }
  return 0;
}
