// Microbenchmark: tcgen05.mma issue rate from SMEM operands, by layout (SWIZZLE_NONE block-major as in the
// leaf kernel vs SWIZZLE_128B) and N. One CTA per SM, one issuing thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_21247_b200/csrc tools/micro/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace pipnn;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                       // LBO (ignored for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO = 8 rows x 128 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

template <bool U8>
__global__ void mma_rate(int iters, int N, int layout, unsigned long long* cyc, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_sh;
  __shared__ __align__(8) uint64_t bar, bar2[2];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = (mode & 8) ? 0u : (mode & 16) ? 0x80808080u : i * 2654435761u;
  if (warp == 0) ptx::tmem_alloc(&taddr_sh, 512);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::mbar_init(&bar2[0], 1); ptx::mbar_init(&bar2[1], 1); ptx::fence_mbar_init(); }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = taddr_sh;
  // mode bit 1: commit to an mbarrier after every 4 MMAs (+ fence after); bit 2: two issuing warps (0 and 1)
  const bool two = (mode & 2) != 0;
  if (threadIdx.x == 0 || (two && threadIdx.x == 32)) {
    const int who = threadIdx.x >> 5;
    const uint32_t a0 = ptx::smem_u32(sm), b0 = ptx::smem_u32(sm + 32768);
    const uint32_t idesc = U8 ? ptx::idesc_u8_s32(128, N) : ptx::idesc_bf16_f32(128, N);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      for (int kc = 0; kc < 4; ++kc) {  // K = 128 bytes per row: 4 MMAs of 32 B
        uint64_t ad, bd;
        // mode bit 4: B from 4 different 16 KB tiles in turn (fresh operand data every tile, like a ring)
        const uint32_t boff = (mode & 4) ? (uint32_t)((i & 1) * 16384) : 0u;
        const uint32_t aoff = (mode & 4) ? (uint32_t)(((i >> 1) & 1) * 16384) : 0u;
        if (layout == 0) {
          ad = ptx::smem_desc_kmajor_noswz(a0 + aoff + kc * 2 * 2048, 2048, 128);
          bd = ptx::smem_desc_kmajor_noswz(b0 + boff + kc * 2 * 2048, 2048, 128);
        } else {
          ad = desc_sw128(a0 + aoff + kc * 32);
          bd = desc_sw128(b0 + boff + kc * 32);
        }
        const uint32_t d = tmem + (two ? who * 256 + (i & 1) * 128 : (i & 1) * 256);
        if (U8) ptx::mma_i8(d, ad, bd, idesc, kc > 0);
        else ptx::mma_bf16(d, ad, bd, idesc, kc > 0);
      }
      if (mode & 1) {
        ptx::mma_commit(&bar2[who]);
        ptx::tc_fence_after();
      }
    }
    ptx::mma_commit(&bar);
    if (who == 0) {
      ptx::mbar_wait(&bar, 0, nullptr, 0);
      const unsigned long long t1 = clock64();
      cyc[blockIdx.x] = t1 - t0;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 20000;
  cudaFuncSetAttribute(mma_rate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  cudaFuncSetAttribute(mma_rate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  for (int u8 = 1; u8 >= 1; --u8)
    for (int layout = 0; layout < 1; ++layout)
      for (int N : {128, 128, 256, 128, 64, 128, 256, 128}) for (int mode : {0}) {
        if (N > 128 && (mode & 4)) continue;
        for (int rep = 0; rep < 2; ++rep) {
          if (u8) mma_rate<true><<<148, 128, 98304>>>(iters, N, layout, cyc, mode);
          else mma_rate<false><<<148, 128, 98304>>>(iters, N, layout, cyc, mode);
        }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long h[148];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double mean = 0;
        for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
        const double per = mean / (iters * 4.0 * ((mode & 2) ? 2 : 1));
        const double ops = 2.0 * 128 * N * (u8 ? 32 : 16);
        printf("%s layout=%s N=%3d mode=%d: %.1f cycles per MMA, %.0f ops/cycle/SM\n", u8 ? "i8  " : "bf16",
               layout ? "sw128" : "none ", N, mode, per, ops / per);
      }
  return 0;
}
