// final_prune.cu — final RobustPrune of every reservoir and the CSR write-out (§4.3, P:568-570;
// Alg. 2 P:227-248 in its lazy form P:938-942), one warp per point:
//   1. candidates = the reservoir's ids; D(u, v) recomputed at path precision: exact integers for
//      uint8 (|a-b| per byte + dp4a), fp32 on bf16-rounded coordinates for float (direct form);
//   2. bitonic sort by (D, v) — the total order of DESIGN.md R4;
//   3. lazy scan: admit c unless an admitted y has alpha_num*D(y,c) < alpha_den*D(u,c); stop at R.
//      For <= 64 candidates the candidate Gram D(v_i, v_j) is computed once into SMEM (lane per pair);
//      larger lists compute D(y, c) on demand (lane per admitted y).
// Then row_ptr = exclusive scan of the degrees and a coalesced copy into col_idx.
#include <cub/cub.cuh>

#include "internal.h"

namespace pipnn {

constexpr int kFpGram = 64;

template <bool U8, bool MIPS>
__device__ __forceinline__ float row_dist(const void* __restrict__ Xv, int64_t ld, int d, uint32_t a, uint32_t b) {
  if (U8) {
    const uint8_t* ra = (const uint8_t*)Xv + (int64_t)a * ld;
    const uint8_t* rb = (const uint8_t*)Xv + (int64_t)b * ld;
    uint32_t acc = 0;
    if (((d | ld) & 3) == 0) {
      const uint32_t* wa = (const uint32_t*)ra;
      const uint32_t* wb = (const uint32_t*)rb;
      for (int w = 0; w < (d >> 2); ++w) {
        const uint32_t df = __vabsdiffu4(__ldg(wa + w), __ldg(wb + w));
        acc = __dp4a(df, df, acc);
      }
    } else {
      for (int j = 0; j < d; ++j) {
        const int t = (int)ra[j] - (int)rb[j];
        acc += (uint32_t)(t * t);
      }
    }
    return (float)acc;  // exact: < 2^24 for d <= 512... integer value carried as float
  } else {
    const float* ra = (const float*)Xv + (int64_t)a * ld;
    const float* rb = (const float*)Xv + (int64_t)b * ld;
    float acc = 0.0f;
    for (int j = 0; j < d; ++j) {
      const float x = __uint_as_float((uint32_t)f32_to_bf16_rne(__ldg(ra + j)) << 16);
      const float y = __uint_as_float((uint32_t)f32_to_bf16_rne(__ldg(rb + j)) << 16);
      if (MIPS) acc = fmaf(x, y, acc);
      else acc = fmaf(x - y, x - y, acc);
    }
    return MIPS ? -acc : acc;
  }
}

__device__ __forceinline__ uint32_t f_ord(float f) {
  const uint32_t b = __float_as_uint(f + 0.0f);
  return b ^ ((b & 0x80000000u) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float f_unord(uint32_t o) {
  return __uint_as_float(o ^ ((o & 0x80000000u) ? 0x80000000u : 0xFFFFFFFFu));
}

__device__ __forceinline__ void warp_sort_u64(uint64_t* a, int P, int lane) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t x = a[i], y = a[ixj];
          if ((x > y) == ((i & k) == 0)) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncwarp();
    }
}

// alpha test on (integer-valued for u8) distances: alpha_num * D(y,c) < alpha_den * D(u,c)
template <bool U8>
__device__ __forceinline__ bool prunes(float Dyc, float Duc, int an, int ad) {
  if (U8) return (int64_t)an * (int64_t)Dyc < (int64_t)ad * (int64_t)Duc;
  return (float)an * Dyc < (float)ad * Duc;
}

template <bool U8, bool MIPS>
__global__ void __launch_bounds__(128) final_prune_kernel(const void* __restrict__ Xv, int64_t n, int d, int64_t ld,
                                                          int l_max, int cap, const uint64_t* __restrict__ slots,
                                                          const uint32_t* __restrict__ count, int R, int an, int ad,
                                                          int final_prune, uint32_t* __restrict__ nbr_tmp,
                                                          uint32_t* __restrict__ deg) {
  extern __shared__ uint64_t fsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* keys = fsm + (size_t)warp * cap;
  float* gram = reinterpret_cast<float*>(fsm + 4 * (size_t)cap) + (size_t)warp * kFpGram * kFpGram;
  __shared__ int16_t adm[4][256];
  for (int64_t u = blockIdx.x * 4 + warp; u < n; u += (int64_t)gridDim.x * 4) {
    const int c = (int)count[u];
    const uint64_t* res = slots + u * (int64_t)l_max;
    uint32_t* out = nbr_tmp + u * (int64_t)R;
    if (c == 0) {
      if (lane == 0) deg[u] = 0;
      continue;
    }
    const int P = [&] { int p = 32; while (p < c) p <<= 1; return p; }();
    if (!final_prune) {
      // the R nearest reservoir entries by (bf16 dist, id)
      for (int t = lane; t < P; t += 32) keys[t] = t < c ? (res[t] & 0xFFFFFFFFFFFFull) : ~0ull;
      __syncwarp();
      warp_sort_u64(keys, P, lane);
      const int dg = min(c, R);
      for (int t = lane; t < dg; t += 32) out[t] = (uint32_t)(keys[t] & 0xFFFFFFFFu);
      if (lane == 0) deg[u] = (uint32_t)dg;
      __syncwarp();
      continue;
    }
    for (int t = lane; t < P; t += 32) {
      uint64_t key = ~0ull;
      if (t < c) {
        const uint32_t v = (uint32_t)(res[t] & 0xFFFFFFFFu);
        const float D = row_dist<U8, MIPS>(Xv, ld, d, (uint32_t)u, v);
        const uint32_t o = U8 ? (uint32_t)D : f_ord(D);
        key = ((uint64_t)o << 32) | v;
      }
      keys[t] = key;
    }
    __syncwarp();
    warp_sort_u64(keys, P, lane);
    const bool use_gram = c <= kFpGram;
    if (use_gram) {
      const int npairs = c * (c - 1) / 2;
      for (int p = lane; p < npairs; p += 32) {
        // p -> (i, j), i < j, row-major over the strict upper triangle
        int i = 0, rem = p;
        while (rem >= c - 1 - i) {
          rem -= c - 1 - i;
          ++i;
        }
        const int j = i + 1 + rem;
        const float D = row_dist<U8, MIPS>(Xv, ld, d, (uint32_t)(keys[i] & 0xFFFFFFFFu), (uint32_t)(keys[j] & 0xFFFFFFFFu));
        gram[i * kFpGram + j] = D;
        gram[j * kFpGram + i] = D;
      }
      __syncwarp();
    }
    int na = 0;
    for (int i = 0; i < c && na < R; ++i) {
      const uint64_t ki = keys[i];
      const uint32_t vi = (uint32_t)(ki & 0xFFFFFFFFu);
      const float Dui = U8 ? (float)(uint32_t)(ki >> 32) : f_unord((uint32_t)(ki >> 32));
      bool pr = false;
      for (int a0 = 0; a0 < na && !pr; a0 += 32) {
        bool mine = false;
        if (a0 + lane < na) {
          const int y = adm[warp][a0 + lane];
          const float Dyi = use_gram ? gram[y * kFpGram + i]
                                     : row_dist<U8, MIPS>(Xv, ld, d, (uint32_t)(keys[y] & 0xFFFFFFFFu), vi);
          mine = prunes<U8>(Dyi, Dui, an, ad);
        }
        pr = __any_sync(0xffffffffu, mine);
      }
      if (!pr) {
        if (lane == 0) {
          adm[warp][na] = (int16_t)i;
          out[na] = vi;
        }
        ++na;
        __syncwarp();
      }
    }
    if (lane == 0) deg[u] = (uint32_t)na;
    __syncwarp();
  }
}

__global__ void csr_copy_kernel(int64_t n, int R, const uint32_t* __restrict__ nbr_tmp, const uint32_t* __restrict__ deg,
                                const uint64_t* __restrict__ row_ptr, uint32_t* __restrict__ col_idx) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; u < n;
       u += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const uint32_t dg = deg[u];
    const uint64_t o = row_ptr[u];
    for (uint32_t t = lane; t < dg; t += 32) col_idx[o + t] = nbr_tmp[u * (int64_t)R + t];
  }
}

pipnn_status final_prune_impl(const pipnn_points* X, int l_max, const uint64_t* slots, const uint32_t* count,
                              const pipnn_prune_params* p, uint64_t* row_ptr, uint32_t* col_idx, Arena& ar,
                              const Ctx& c) {
  const int64_t n = X->n;
  const int R = p->R;
  uint32_t* nbr_tmp = ar.take<uint32_t>((size_t)n * R);
  uint32_t* deg = ar.take<uint32_t>(n + 1);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (const uint32_t*)nullptr, (uint64_t*)nullptr, (int)(n + 1));
  void* tmp = ar.take<uint8_t>(tmp_bytes);
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (final_prune)");
  if (R > 256) return fail(PIPNN_EUNSUPPORTED, "R > 256");
  int cap = 32;
  while (cap < l_max) cap <<= 1;
  const int smem = 4 * cap * 8 + 4 * kFpGram * kFpGram * 4;
  const int64_t blocks = std::min<int64_t>(ceil_div(n, 4), (int64_t)num_sms() * 32);
  const bool u8 = X->dtype == PIPNN_U8, mips = X->metric == PIPNN_MIPS;
  PIPNN_CUDA(cudaMemsetAsync(deg + n, 0, sizeof(uint32_t), c.st));
#define FP_LAUNCH(U, M)                                                                                           \
  do {                                                                                                            \
    PIPNN_CUDA(cudaFuncSetAttribute(final_prune_kernel<U, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    final_prune_kernel<U, M><<<(unsigned)blocks, 128, smem, c.st>>>(X->data, n, X->d, X->ld, l_max, cap, slots,   \
                                                                   count, R, p->alpha_num, p->alpha_den,          \
                                                                   p->final_prune, nbr_tmp, deg);                 \
  } while (0)
  if (u8) FP_LAUNCH(true, false);
  else if (mips) FP_LAUNCH(false, true);
  else FP_LAUNCH(false, false);
#undef FP_LAUNCH
  PIPNN_LAUNCHED("final_prune_kernel", c.st);
  PIPNN_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, deg, row_ptr, (int)(n + 1), c.st));
  csr_copy_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 8), num_sms() * 32), 256, 0, c.st>>>(n, R, nbr_tmp, deg,
                                                                                                 row_ptr, col_idx);
  PIPNN_LAUNCHED("csr_copy_kernel", c.st);
  return PIPNN_OK;
}

}  // namespace pipnn
