// tc_probe.cu — standalone sm_100a probe for the tcgen05 building blocks used by the leaf/partition
// distance kernel: (1) correctness of the K-major SWIZZLE_NONE tile layout + descriptors for
// kind::i8 (u8 x u8 -> s32) and kind::f16 (bf16 x bf16 -> f32), loaded with 1-D bulk copies;
// (2) raw MMA issue throughput of that layout on all SMs (M=128, N=128 and N=256).
//
// Tile layout in global and shared memory ("tiled rows"): a block of R rows x Kb bytes is stored as
//   [kc = 0..Kb/16) [row = 0..R) [16 bytes]
// so an 8-row core matrix is 128 contiguous bytes, SBO = 128 B, LBO = R*16 B.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>
#include <cuda_bf16.h>
#include "../paper_2602_21247_b200/csrc/ptx.cuh"

using namespace pipnn::ptx;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <bool kU8>
__global__ void __launch_bounds__(128, 1) probe_gemm(const uint8_t* A, const uint8_t* B, int Kb, int N, int32_t* C, int* err) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * Kb;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_load, 128 * Kb + N * Kb);
    bulk_g2s(sA, A, 128 * Kb, &bar_load);
    bulk_g2s(sB, B, N * Kb, &bar_load);
  }
  mbar_wait(&bar_load, 0, err, 1);
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = kU8 ? idesc_u8_s32(128, N) : idesc_bf16_f32(128, N);
    for (int kk = 0; kk < Kb / 32; ++kk) {
      uint64_t ad = smem_desc_kmajor_noswz(smem_u32(sA + kk * 2 * 128 * 16), 128 * 16, 128);
      uint64_t bd = smem_desc_kmajor_noswz(smem_u32(sB + kk * 2 * N * 16), N * 16, 128);
      if (kU8) mma_i8(tbase, ad, bd, idesc, kk > 0);
      else mma_bf16(tbase, ad, bd, idesc, kk > 0);
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0, err, 2);
  tc_fence_after();
  const int row = threadIdx.x;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 32 && c0 + j < N; ++j) C[row * N + c0 + j] = (int32_t)v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

// Throughput: every CTA issues `reps` passes of Kb/32 MMAs (M=128, N) over resident tiles.
template <bool kU8>
__global__ void __launch_bounds__(128, 1) probe_tput(int Kb, int N, int reps, int* err, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * Kb;
  for (int i = threadIdx.x; i < (128 + N) * Kb / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x01010101u * (i & 3);
  fence_proxy_async_smem();
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar_mma, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t idesc = kU8 ? idesc_u8_s32(128, N) : idesc_bf16_f32(128, N);
    for (int r = 0; r < reps; ++r)
      for (int kk = 0; kk < Kb / 32; ++kk) {
        uint64_t ad = smem_desc_kmajor_noswz(smem_u32(sA + kk * 2 * 128 * 16), 128 * 16, 128);
        uint64_t bd = smem_desc_kmajor_noswz(smem_u32(sB + kk * 2 * N * 16), N * 16, 128);
        if (kU8) mma_i8(tbase + (r & 1) * 256, ad, bd, idesc, kk > 0);
        else mma_bf16(tbase + (r & 1) * 256, ad, bd, idesc, kk > 0);
      }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0, err, 3);
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cycles, (unsigned long long)(t1 - t0));
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); u += 0x7FFF + ((u >> 16) & 1); return (uint16_t)(u >> 16); }
static float bf2f(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }

// pack row-major [R][Kb bytes] into tiled [Kb/16][R][16]
static void tile(const uint8_t* src, int R, int Kb, uint8_t* dst) {
  for (int r = 0; r < R; ++r)
    for (int kc = 0; kc < Kb / 16; ++kc) memcpy(dst + ((size_t)kc * R + r) * 16, src + (size_t)r * Kb + kc * 16, 16);
}

template <bool kU8>
static int run_gemm(int K, int N) {
  const int esz = kU8 ? 1 : 2, Kb = K * esz;
  std::vector<uint8_t> a(128 * Kb), b(N * Kb), at(128 * Kb), bt(N * Kb);
  srand(1234 + K + N);
  std::vector<double> af(128 * K), bf(N * K);
  for (int i = 0; i < 128 * K; ++i) {
    if (kU8) { a[i] = rand() & 255; af[i] = a[i]; }
    else { float f = (rand() % 2001 - 1000) / 250.0f; uint16_t h = f2bf(f); memcpy(&a[2 * i], &h, 2); af[i] = bf2f(h); }
  }
  for (int i = 0; i < N * K; ++i) {
    if (kU8) { b[i] = rand() & 255; bf[i] = b[i]; }
    else { float f = (rand() % 2001 - 1000) / 250.0f; uint16_t h = f2bf(f); memcpy(&b[2 * i], &h, 2); bf[i] = bf2f(h); }
  }
  tile(a.data(), 128, Kb, at.data());
  tile(b.data(), N, Kb, bt.data());
  uint8_t *dA, *dB; int32_t* dC; int* derr;
  CK(cudaMalloc(&dA, at.size())); CK(cudaMalloc(&dB, bt.size())); CK(cudaMalloc(&dC, 128 * N * 4)); CK(cudaMalloc(&derr, 4));
  CK(cudaMemcpy(dA, at.data(), at.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, bt.data(), bt.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(derr, 0, 4)); CK(cudaMemset(dC, 0xFF, 128 * N * 4));
  int smem = (128 + N) * Kb;
  CK(cudaFuncSetAttribute(probe_gemm<kU8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe_gemm<kU8><<<1, 128, smem>>>(dA, dB, Kb, N, dC, derr);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  int herr; CK(cudaMemcpy(&herr, derr, 4, cudaMemcpyDeviceToHost));
  std::vector<int32_t> c(128 * N);
  CK(cudaMemcpy(c.data(), dC, c.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0; double maxrel = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      double ref = 0, mag = 0; for (int k = 0; k < K; ++k) { ref += af[i * K + k] * bf[j * K + k]; mag += fabs(af[i * K + k] * bf[j * K + k]); }
      if (kU8) { if ((int64_t)ref != c[i * N + j]) { if (bad < 5) printf("  mismatch (%d,%d) got %d want %lld\n", i, j, c[i * N + j], (long long)ref); ++bad; } }
      else { float g; memcpy(&g, &c[i * N + j], 4); double rel = fabs(g - ref) / (mag + 1e-30); if (rel > maxrel) maxrel = rel; if (rel > 1e-5) { if (bad < 5) printf("  mismatch (%d,%d) got %g want %g\n", i, j, g, ref); ++bad; } }
    }
  printf("gemm %s K=%d N=%d: err_flag=%d mismatches=%ld maxrel=%.3g -> %s\n", kU8 ? "u8" : "bf16", K, N, herr, bad, maxrel, (bad == 0 && herr == 0) ? "PASS" : "FAIL");
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(derr);
  return (bad == 0 && herr == 0) ? 0 : 1;
}

template <bool kU8>
static void run_tput(int K, int N, int reps) {
  const int esz = kU8 ? 1 : 2, Kb = K * esz;
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  int smem = (128 + N) * Kb;
  CK(cudaFuncSetAttribute(probe_tput<kU8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int* derr; unsigned long long* dcyc; CK(cudaMalloc(&derr, 4)); CK(cudaMalloc(&dcyc, 8));
  CK(cudaMemset(derr, 0, 4)); CK(cudaMemset(dcyc, 0, 8));
  probe_tput<kU8><<<nsm, 128, smem>>>(Kb, N, 4, derr, dcyc);  // warm
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(dcyc, 0, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe_tput<kU8><<<nsm, 128, smem>>>(Kb, N, reps, derr, dcyc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; int herr;
  CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(&herr, derr, 4, cudaMemcpyDeviceToHost));
  double ops = 2.0 * 128 * N * K * (double)reps * nsm;
  double cyc_per_mma = (double)cyc / nsm / ((double)reps * (Kb / 32));
  printf("tput %s K=%d N=%d reps=%d: %.3f ms  %.1f T%s/s  cycles/MMA=%.1f (floor 128xN/256=%.1f) err=%d\n", kU8 ? "u8" : "bf16", K, N, reps, ms,
         ops / ms / 1e9, kU8 ? "OP" : "FLOP", cyc_per_mma, 128.0 * N / 256.0, herr);
  cudaFree(derr); cudaFree(dcyc);
}

int main() {
  int fails = 0;
  fails += run_gemm<true>(128, 128);
  fails += run_gemm<true>(128, 48);
  fails += run_gemm<true>(96, 256);
  fails += run_gemm<false>(96, 128);
  fails += run_gemm<false>(208, 64);
  fails += run_gemm<false>(128, 256);
  if (fails) { printf("PROBE FAIL %d\n", fails); return 1; }
  run_tput<true>(128, 128, 20000);
  run_tput<true>(128, 256, 10000);
  run_tput<false>(128, 128, 20000);
  run_tput<false>(128, 256, 10000);
  run_tput<false>(208, 128, 10000);
  printf("PROBE OK\n");
  return 0;
}
