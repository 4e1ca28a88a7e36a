// Microbenchmark: issue rate of 1-D cp.async.bulk from one thread with no waits in between (copies of CH bytes
// from an L2-resident buffer into NB distinct SMEM slots with their own mbarriers; the thread waits once at the
// end), and the completion -> waiter wake-up path: cycles per copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2602_21247_b200/csrc tools/micro/bulk_issue.cu -o /tmp/bi
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace pipnn;

__global__ void issue(const uint8_t* src, int ch, int nb, int rounds, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[32];
  if (threadIdx.x == 0) {
    for (int i = 0; i < nb; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t_issue = 0, t_total = 0;
  for (int r = 0; r < rounds; ++r) {
    const unsigned long long t0 = clock64();
    for (int i = 0; i < nb; ++i) {
      ptx::mbar_arrive_expect_tx(&bar[i], ch);
      ptx::bulk_g2s(sm + (size_t)i * ch, src + ((size_t)(blockIdx.x * 64 + r * nb + i) % 4096) * ch, ch, &bar[i]);
    }
    const unsigned long long t1 = clock64();
    for (int i = 0; i < nb; ++i) ptx::mbar_wait(&bar[i], r & 1, nullptr, 0);
    const unsigned long long t2 = clock64();
    t_issue += t1 - t0;
    t_total += t2 - t0;
  }
  out[blockIdx.x * 2] = t_issue;
  out[blockIdx.x * 2 + 1] = t_total;
}

int main() {
  uint8_t* d;
  cudaMalloc(&d, 64 << 20);
  cudaMemset(d, 1, 64 << 20);
  unsigned long long* o;
  cudaMalloc(&o, 148 * 16);
  for (int ch : {4096, 16384})
    for (int nb : {1, 4, 8}) {
      const int smem = ch * nb;
      if (smem > 200 * 1024) continue;
      cudaFuncSetAttribute(issue, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int rounds = 200;
      issue<<<148, 32, smem>>>(d, ch, nb, rounds, o);
      cudaDeviceSynchronize();
      unsigned long long h[296];
      cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
      double ti = 0, tt = 0;
      for (int b = 0; b < 148; ++b) { ti += h[2 * b]; tt += h[2 * b + 1]; }
      ti /= 148.0 * rounds; tt /= 148.0 * rounds;
      printf("chunk %6d, %d copies per round: issue %.0f cycles, issue+complete %.0f cycles per round (%.0f per copy)\n",
             ch, nb, ti, tt, tt / nb);
    }
  return 0;
}
