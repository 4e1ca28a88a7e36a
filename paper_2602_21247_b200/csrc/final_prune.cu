// final_prune.cu — final RobustPrune of every reservoir and the CSR write-out (§4.3, P:568-570;
// Alg. 2 P:227-248 in its lazy form P:938-942), one warp per point:
//   1. candidates = the reservoir's ids; their vectors (and u's) are staged in shared memory with coalesced
//      row loads (float rows as bf16, the path precision of DESIGN.md R19/R24), row stride padded by one
//      word so lane-per-candidate reads are bank-conflict free;
//   2. D(u, v) recomputed at path precision: exact integers for uint8 (|a-b| per byte + dp4a),
//      fp32 on bf16 coordinates for float (direct form); bitonic sort by (D, v) (R4);
//   3. the candidate Gram D(v_i, v_j) (lane per pair, from SMEM), then the lazy scan: admit c unless an
//      admitted y has alpha_num*D(y,c) < alpha_den*D(u,c); stop at R (the lanes test the admitted set).
//   Reservoirs with more than kFpStage candidates take a slow path (warp-cooperative distances from HBM).
// Then row_ptr = exclusive scan of the degrees and a coalesced copy into col_idx.
#include <cub/cub.cuh>

#include "internal.h"

namespace pipnn {

constexpr int kFpStage = 48;  // candidates staged in SMEM (Gram path)

__device__ __forceinline__ uint32_t f_ord(float f) {
  const uint32_t b = __float_as_uint(f + 0.0f);
  return b ^ ((b & 0x80000000u) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float f_unord(uint32_t o) {
  return __uint_as_float(o ^ ((o & 0x80000000u) ? 0x80000000u : 0xFFFFFFFFu));
}

// distance between two staged rows (nw 32-bit words each)
template <bool U8, bool MIPS>
__device__ __forceinline__ float srow_dist(const uint32_t* a, const uint32_t* b, int nw) {
  if (U8) {
    uint32_t acc = 0;
    for (int w = 0; w < nw; ++w) {
      const uint32_t df = __vabsdiffu4(a[w], b[w]);
      acc = __dp4a(df, df, acc);
    }
    return (float)acc;  // exact integer (< 2^24 for d <= 512... d*255^2)
  } else {
    float acc = 0.0f;
    for (int w = 0; w < nw; ++w) {
      const uint32_t x = a[w], y = b[w];
      const float x0 = __uint_as_float(x << 16), x1 = __uint_as_float(x & 0xFFFF0000u);
      const float y0 = __uint_as_float(y << 16), y1 = __uint_as_float(y & 0xFFFF0000u);
      if (MIPS) {
        acc = fmaf(x0, y0, acc);
        acc = fmaf(x1, y1, acc);
      } else {
        acc = fmaf(x0 - y0, x0 - y0, acc);
        acc = fmaf(x1 - y1, x1 - y1, acc);
      }
    }
    return MIPS ? -acc : acc;
  }
}

// warp-cooperative distance of two rows straight from X (slow path)
template <bool U8, bool MIPS>
__device__ __forceinline__ float warp_row_dist(const void* Xv, int64_t ld, int d, uint32_t a, uint32_t b, int lane) {
  float acc = 0.0f;
  if (U8) {
    const uint8_t* ra = (const uint8_t*)Xv + (int64_t)a * ld;
    const uint8_t* rb = (const uint8_t*)Xv + (int64_t)b * ld;
    uint32_t s = 0;
    for (int j = lane; j < d; j += 32) {
      const int t = (int)ra[j] - (int)rb[j];
      s += (uint32_t)(t * t);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return (float)s;
  }
  const float* ra = (const float*)Xv + (int64_t)a * ld;
  const float* rb = (const float*)Xv + (int64_t)b * ld;
  for (int j = lane; j < d; j += 32) {
    const float x = __uint_as_float((uint32_t)f32_to_bf16_rne(ra[j]) << 16);
    const float y = __uint_as_float((uint32_t)f32_to_bf16_rne(rb[j]) << 16);
    acc = MIPS ? fmaf(x, y, acc) : fmaf(x - y, x - y, acc);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return MIPS ? -acc : acc;
}

// stage rows sids[0..c) into rows[r*sw], and sids[cap] (the point itself) into rows[cap*sw];
// flattened (row, word) index space, 16 independent loads in flight per lane.
template <bool U8>
__device__ __forceinline__ void stage_rows(const void* Xv, int64_t ld, int d, const uint32_t* sids, int c, int cap,
                                           uint32_t* rows, int nw, int sw, int lane) {
  const int total = (c + 1) * nw;
  const bool fast = U8 ? (((d | ld) & 3) == 0) : true;
  for (int e0 = 0; e0 < total; e0 += 512) {
    uint32_t v[16];
    int dst[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int e = e0 + j * 32 + lane;
      dst[j] = -1;
      if (e < total) {
        const int r = e / nw, w = e - r * nw;
        const int rr = r < c ? r : cap;
        const uint32_t id = sids[rr];
        dst[j] = rr * sw + w;
        if (U8) {
          const uint8_t* row = (const uint8_t*)Xv + (int64_t)id * ld;
          if (fast) {
            v[j] = __ldg((const uint32_t*)row + w);
          } else {
            uint32_t x = 0;
            for (int t = 0; t < 4; ++t)
              if (4 * w + t < d) x |= (uint32_t)row[4 * w + t] << (8 * t);
            v[j] = x;
          }
        } else {
          const float* row = (const float*)Xv + (int64_t)id * ld;
          const float a = 2 * w < d ? __ldg(row + 2 * w) : 0.0f;
          const float b = 2 * w + 1 < d ? __ldg(row + 2 * w + 1) : 0.0f;
          v[j] = (uint32_t)f32_to_bf16_rne(a) | ((uint32_t)f32_to_bf16_rne(b) << 16);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (dst[j] >= 0) rows[dst[j]] = v[j];
  }
}

__device__ __forceinline__ void warp_sort_kv(uint64_t* a, uint16_t* v, int P, int lane) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t x = a[i], y = a[ixj];
          if ((x > y) == ((i & k) == 0)) {
            a[i] = y;
            a[ixj] = x;
            const uint16_t t = v[i];
            v[i] = v[ixj];
            v[ixj] = t;
          }
        }
      }
      __syncwarp();
    }
}

// alpha test: alpha_num * D(y,c) < alpha_den * D(u,c)  (integers exact for uint8)
template <bool U8>
__device__ __forceinline__ bool prunes(float Dyc, float Duc, int an, int ad) {
  if (U8) return (int64_t)an * (int64_t)Dyc < (int64_t)ad * (int64_t)Duc;
  return (float)an * Dyc < (float)ad * Duc;
}

struct FpLayout {
  int nw, stride_w, kcap;
  size_t rows_off, ids_off, keys_off, vals_off, gram_off, adm_off, per_warp;
};
__host__ __device__ inline FpLayout fp_layout(int d, bool u8, int l_max, int cap_rows) {
  FpLayout L;
  L.nw = u8 ? (d + 3) / 4 : (d + 1) / 2;
  L.stride_w = L.nw + 1;
  int kc = 32;
  while (kc < l_max) kc <<= 1;
  L.kcap = kc;
  size_t o = 0;
  L.rows_off = o;
  o += (size_t)(cap_rows + 1) * L.stride_w * 4;
  L.ids_off = o;
  o += (size_t)(cap_rows + 1) * 4;
  o = (o + 15) & ~(size_t)15;
  L.keys_off = o;
  o += (size_t)kc * 8;
  L.vals_off = o;
  o += (size_t)kc * 2;
  o = (o + 15) & ~(size_t)15;
  L.gram_off = o;
  o += (size_t)kFpStage * kFpStage * 4;
  L.adm_off = o;
  o += 256 * 2;
  L.per_warp = (o + 127) & ~(size_t)127;
  return L;
}

// Pass 0 (deferred == nullptr on input list): every point; reservoirs with more than kFpStage candidates
// are appended to `defer` and handled by pass 1, which stages up to l_max rows per warp (one warp per CTA)
// and runs the lazy scan from SMEM without a Gram.
template <bool U8, bool MIPS>
__global__ void final_prune_kernel(const void* __restrict__ Xv, int64_t n, int d, int64_t ld, int l_max,
                                   const uint64_t* __restrict__ slots, const uint32_t* __restrict__ count, int R,
                                   int an, int ad, int final_prune, uint32_t* __restrict__ nbr_tmp,
                                   uint32_t* __restrict__ deg, int cap_rows, const uint32_t* __restrict__ list,
                                   const uint32_t* __restrict__ list_n, uint32_t* __restrict__ defer,
                                   uint32_t* __restrict__ defer_n) {
  extern __shared__ __align__(16) uint8_t fsm[];
  const FpLayout Lo = fp_layout(d, U8, l_max, cap_rows);
  const int64_t n_iter = list ? (int64_t)*list_n : n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  uint8_t* base = fsm + (size_t)warp * Lo.per_warp;
  uint32_t* rows = (uint32_t*)(base + Lo.rows_off);
  uint64_t* keys = (uint64_t*)(base + Lo.keys_off);
  uint16_t* vals = (uint16_t*)(base + Lo.vals_off);
  float* gram = (float*)(base + Lo.gram_off);
  int16_t* adm = (int16_t*)(base + Lo.adm_off);
  uint32_t* sids = (uint32_t*)(base + Lo.ids_off);
  const int nw = Lo.nw, sw = Lo.stride_w;
  uint32_t* urow = rows + (size_t)cap_rows * sw;
  uint16_t* pairs = (uint16_t*)(fsm + (size_t)wpb * Lo.per_warp);  // (i, j) table, j-major: (0,1),(0,2),(1,2),..
  for (int p = threadIdx.x; p < kFpStage * (kFpStage - 1) / 2; p += blockDim.x) {
    int j = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)p)) * 0.5f);
    while (j * (j - 1) / 2 > p) --j;
    while ((j + 1) * j / 2 <= p) ++j;
    pairs[2 * p] = (uint16_t)(p - j * (j - 1) / 2);
    pairs[2 * p + 1] = (uint16_t)j;
  }
  __syncthreads();

  for (int64_t it = (int64_t)blockIdx.x * wpb + warp; it < n_iter; it += (int64_t)gridDim.x * wpb) {
    const int64_t u = list ? (int64_t)list[it] : it;
    const int c = (int)count[u];
    if (!list && final_prune && c > kFpStage) {  // deferred to pass 1
      if (lane == 0) defer[atomicAdd(defer_n, 1u)] = (uint32_t)u;
      continue;
    }
    const uint64_t* res = slots + u * (int64_t)l_max;
    uint32_t* out = nbr_tmp + u * (int64_t)R;
    if (c == 0) {
      if (lane == 0) deg[u] = 0;
      continue;
    }
    int P = 32;
    while (P < c) P <<= 1;
    if (!final_prune) {
      // the R nearest reservoir entries by (bf16 dist, id)
      for (int t = lane; t < P; t += 32) {
        keys[t] = t < c ? (res[t] & 0xFFFFFFFFFFFFull) : ~0ull;
        vals[t] = 0;
      }
      __syncwarp();
      warp_sort_kv(keys, vals, P, lane);
      const int dg = min(c, R);
      for (int t = lane; t < dg; t += 32) out[t] = (uint32_t)(keys[t] & 0xFFFFFFFFu);
      if (lane == 0) deg[u] = (uint32_t)dg;
      __syncwarp();
      continue;
    }
    const bool staged = c <= cap_rows;
    if (staged) {
      // rows 0..c-1 = candidates, row cap_rows = u; many independent loads in flight per lane
      for (int t = lane; t < c; t += 32) sids[t] = (uint32_t)(res[t] & 0xFFFFFFFFu);
      if (lane == 0) sids[cap_rows] = (uint32_t)u;
      __syncwarp();
      stage_rows<U8>(Xv, ld, d, sids, c, cap_rows, rows, nw, sw, lane);
      __syncwarp();
      for (int t = lane; t < P; t += 32) {
        uint64_t key = ~0ull;
        if (t < c) {
          const uint32_t v = (uint32_t)(res[t] & 0xFFFFFFFFu);
          const float D = srow_dist<U8, MIPS>(urow, rows + (size_t)t * sw, nw);
          key = ((uint64_t)(U8 ? (uint32_t)D : f_ord(D)) << 32) | v;
        }
        keys[t] = key;
        vals[t] = (uint16_t)t;
      }
    } else {
      for (int t = 0; t < P; ++t) {
        uint64_t key = ~0ull;
        if (t < c) {
          const uint32_t v = (uint32_t)(res[t] & 0xFFFFFFFFu);
          const float D = warp_row_dist<U8, MIPS>(Xv, ld, d, (uint32_t)u, v, lane);
          key = ((uint64_t)(U8 ? (uint32_t)D : f_ord(D)) << 32) | v;
        }
        if (lane == 0) {
          keys[t] = key;
          vals[t] = 0;
        }
      }
    }
    __syncwarp();
    warp_sort_kv(keys, vals, P, lane);
    const bool use_gram = c <= kFpStage;
    if (use_gram) {
      // Gram over sorted positions, lane per pair (i < j); pairs with j < c are a prefix of the table
      const int npairs = c * (c - 1) / 2;
      for (int p = lane; p < npairs; p += 32) {
        const int i = pairs[2 * p], j = pairs[2 * p + 1];
        const float D = srow_dist<U8, MIPS>(rows + (size_t)vals[i] * sw, rows + (size_t)vals[j] * sw, nw);
        gram[i * kFpStage + j] = D;
        gram[j * kFpStage + i] = D;
      }
      __syncwarp();
    }
    int na = 0;
    for (int i = 0; i < c && na < R; ++i) {
      const uint64_t ki = keys[i];
      const uint32_t vi = (uint32_t)(ki & 0xFFFFFFFFu);
      const float Dui = U8 ? (float)(uint32_t)(ki >> 32) : f_unord((uint32_t)(ki >> 32));
      bool pr = false;
      if (use_gram) {
        for (int a0 = 0; a0 < na && !pr; a0 += 32) {
          bool mine = false;
          if (a0 + lane < na) mine = prunes<U8>(gram[adm[a0 + lane] * kFpStage + i], Dui, an, ad);
          pr = __any_sync(0xffffffffu, mine);
        }
      } else if (staged) {
        // lane per admitted y, distances from the staged rows
        const uint32_t* ri = rows + (size_t)vals[i] * sw;
        for (int a0 = 0; a0 < na && !pr; a0 += 32) {
          bool mine = false;
          if (a0 + lane < na)
            mine = prunes<U8>(srow_dist<U8, MIPS>(rows + (size_t)vals[adm[a0 + lane]] * sw, ri, nw), Dui, an, ad);
          pr = __any_sync(0xffffffffu, mine);
        }
      } else {
        for (int a = 0; a < na && !pr; ++a) {
          const float Dyi = warp_row_dist<U8, MIPS>(Xv, ld, d, (uint32_t)(keys[adm[a]] & 0xFFFFFFFFu), vi, lane);
          pr = prunes<U8>(Dyi, Dui, an, ad);
        }
      }
      if (!pr) {
        if (lane == 0) {
          adm[na] = (int16_t)i;
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
  uint32_t* defer = ar.take<uint32_t>(n);
  uint32_t* defer_n = ar.take<uint32_t>(1);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (const uint32_t*)nullptr, (uint64_t*)nullptr, (int)(n + 1));
  void* tmp = ar.take<uint8_t>(tmp_bytes);
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (final_prune)");
  if (R > 256) return fail(PIPNN_EUNSUPPORTED, "R > 256");
  const bool u8 = X->dtype == PIPNN_U8, mips = X->metric == PIPNN_MIPS;
  // pass 0: many warps, <= kFpStage staged candidates (Gram); pass 1: one warp per CTA, up to l_max rows
  const FpLayout L0 = fp_layout(X->d, u8, l_max, kFpStage);
  int wpb = 8;
  while (wpb > 1 && (size_t)wpb * L0.per_warp > 96 * 1024) wpb >>= 1;
  const size_t pair_bytes = (size_t)kFpStage * (kFpStage - 1) * 2;  // u16 (i, j) pairs
  const int smem0 = (int)(wpb * L0.per_warp + pair_bytes);
  int cap1 = l_max;
  FpLayout L1 = fp_layout(X->d, u8, l_max, cap1);
  while (cap1 > kFpStage && L1.per_warp + pair_bytes > 200 * 1024) L1 = fp_layout(X->d, u8, l_max, cap1 -= 16);
  const int smem1 = (int)(L1.per_warp + pair_bytes);
  const int64_t blocks = std::min<int64_t>(ceil_div(n, wpb), (int64_t)num_sms() * 16);
  PIPNN_CUDA(cudaMemsetAsync(deg + n, 0, sizeof(uint32_t), c.st));
  PIPNN_CUDA(cudaMemsetAsync(defer_n, 0, sizeof(uint32_t), c.st));
#define FP_LAUNCH(U, M)                                                                                            \
  do {                                                                                                             \
    auto* fn = final_prune_kernel<U, M>;                                                                           \
    PIPNN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, std::max(smem0, smem1)));      \
    fn<<<(unsigned)blocks, 32 * wpb, smem0, c.st>>>(X->data, n, X->d, X->ld, l_max, slots, count, R, p->alpha_num,  \
                                                    p->alpha_den, p->final_prune, nbr_tmp, deg, kFpStage, nullptr,  \
                                                    nullptr, defer, defer_n);                                       \
    PIPNN_LAUNCHED("final_prune_kernel", c.st);                                                                    \
    fn<<<(unsigned)(num_sms() * 2), 32, smem1, c.st>>>(X->data, n, X->d, X->ld, l_max, slots, count, R,            \
                                                      p->alpha_num, p->alpha_den, p->final_prune, nbr_tmp, deg,     \
                                                      cap1, defer, defer_n, nullptr, nullptr);                      \
    PIPNN_LAUNCHED("final_prune_kernel(deferred)", c.st);                                                          \
  } while (0)
  if (u8) FP_LAUNCH(true, false);
  else if (mips) FP_LAUNCH(false, true);
  else FP_LAUNCH(false, false);
#undef FP_LAUNCH
  PIPNN_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, deg, row_ptr, (int)(n + 1), c.st));
  csr_copy_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 8), num_sms() * 32), 256, 0, c.st>>>(n, R, nbr_tmp, deg,
                                                                                                 row_ptr, col_idx);
  PIPNN_LAUNCHED("csr_copy_kernel", c.st);
  return PIPNN_OK;
}

}  // namespace pipnn
