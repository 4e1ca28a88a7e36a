// final_prune.cu — final RobustPrune of every reservoir and the CSR write-out (§4.3, P:568-570;
// Alg. 2 P:227-248 in its lazy form P:938-942). Per point u:
//   1. rows = u and its c reservoir candidates, staged in shared memory (uint8 bytes, or the bf16 RNE
//      coordinates of float rows: the path precision of DESIGN.md R19/R24);
//   2. the (c+1)x(c+1) Gram on the tensor cores with warp-level MMAs (u8 x u8 -> s32, exact; bf16 -> f32);
//      D(r,s) = G_rr + G_ss - 2 G_rs (L2), -G_rs (MIPS);
//   3. prune bitmasks (alpha_num*D'(y,c) < alpha_den*D'(u,c)) and the (D(u,.), id) order (R4), where
//      D' = D for L2 and the angular dissimilarity 1 - G_rs / sqrt(G_rr G_ss) for MIPS (R22);
//   4. the lazy scan: admit c unless an admitted earlier y prunes it; stop at R.
// Tiers by reservoir occupancy, each a kernel shaped for its size:
//   <= 31 candidates : one warp per point — fp_gram_kernel (uint8: Gram in SMEM, fixpoint over ballots) or
//                      fp_warp_kernel (float: Gram in registers, masks from the MMA fragments, warp bitonic
//                      sort, sequential scan over shuffles);
//   <= 63, <= 127,   : fp_band_kernel (a warp per 16-row Gram band, masks from the fragments and the
//   <= 191             candidates' ranks in the band warps, a scan warp that resolves 32-candidate batches
//                      as ballot fixpoints while the band warps start the next point);
//   larger           : the generic final_prune_kernel.
// final_prune = 0 (keep the R nearest reservoir entries) uses the generic kernel.
// Then row_ptr = exclusive scan of the degrees and a coalesced copy into col_idx.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

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

// MIPS prune dissimilarity (R22): 1 - <a,b> inv(a) inv(b), inv = 1/||.|| (0 for a zero vector, so
// cos = 0 and the dissimilarity is 1, as in the oracle)
__device__ __forceinline__ float inv_norm(float nn) { return nn > 0.0f ? 1.0f / sqrtf(nn) : 0.0f; }
__device__ __forceinline__ float ang_d(float dot, float ia, float ib) { return 1.0f - dot * ia * ib; }

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

// the prune dissimilarity D' of two staged rows (D itself for L2; angular for MIPS, R22)
template <bool U8, bool MIPS>
__device__ __forceinline__ float srow_pd(const uint32_t* a, const uint32_t* b, int nw) {
  if (!MIPS) return srow_dist<U8, MIPS>(a, b, nw);
  const float ab = -srow_dist<U8, MIPS>(a, b, nw), aa = -srow_dist<U8, MIPS>(a, a, nw),
              bb = -srow_dist<U8, MIPS>(b, b, nw);
  return ang_d(ab, inv_norm(aa), inv_norm(bb));
}
template <bool U8, bool MIPS>
__device__ __forceinline__ float warp_row_pd(const void* Xv, int64_t ld, int d, uint32_t a, uint32_t b, int lane) {
  if (!MIPS) return warp_row_dist<U8, MIPS>(Xv, ld, d, a, b, lane);
  const float ab = -warp_row_dist<U8, MIPS>(Xv, ld, d, a, b, lane), aa = -warp_row_dist<U8, MIPS>(Xv, ld, d, a, a, lane),
              bb = -warp_row_dist<U8, MIPS>(Xv, ld, d, b, b, lane);
  return ang_d(ab, inv_norm(aa), inv_norm(bb));
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
        const float D = srow_pd<U8, MIPS>(rows + (size_t)vals[i] * sw, rows + (size_t)vals[j] * sw, nw);
        gram[i * kFpStage + j] = D;
        gram[j * kFpStage + i] = D;
      }
      __syncwarp();
    }
    int na = 0;
    for (int i = 0; i < c && na < R; ++i) {
      const uint64_t ki = keys[i];
      const uint32_t vi = (uint32_t)(ki & 0xFFFFFFFFu);
      float Dui = U8 ? (float)(uint32_t)(ki >> 32) : f_unord((uint32_t)(ki >> 32));
      if (MIPS)  // the prune test's D'(u, i)
        Dui = (use_gram || staged) ? srow_pd<U8, MIPS>(urow, rows + (size_t)vals[i] * sw, nw)
                                   : warp_row_pd<U8, MIPS>(Xv, ld, d, (uint32_t)u, vi, lane);
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
            mine = prunes<U8>(srow_pd<U8, MIPS>(rows + (size_t)vals[adm[a0 + lane]] * sw, ri, nw), Dui, an, ad);
          pr = __any_sync(0xffffffffu, mine);
        }
      } else {
        for (int a = 0; a < na && !pr; ++a) {
          const float Dyi = warp_row_pd<U8, MIPS>(Xv, ld, d, (uint32_t)(keys[adm[a]] & 0xFFFFFFFFu), vi, lane);
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

// ------------------------------------------------------------------ Gram path (tensor cores, warp per point)
// Rows 0..c of a per-warp SMEM tile hold u (row 0) and its c reservoir candidates (rows 1..c), as u8 bytes or
// bf16 coordinates, zero-padded to Kb bytes and to a multiple of 16 rows; the row pitch is Kb + 16 bytes so
// the mma.sync fragment loads (8 rows x 4 consecutive words per instruction) are bank-conflict free. The
// Gram G = V V^T comes from warp-level MMAs (m16n8k32 u8 x u8 -> s32, exact; m16n8k16 bf16 x bf16 -> f32),
// then D(r, s) = G_rr + G_ss - 2 G_rs (L2; clamped at 0 for float) or -G_rs (MIPS) in place.
// Both fragment layouts address the same bytes: one K-step = 32 bytes of every row.
template <bool U8>
__device__ __forceinline__ void mma_16x8(int32_t (&acc)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  if (U8) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x4_s(uint32_t (&r)[4], uint32_t saddr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr));
}
// No "memory" clobber: a clobber in the staging loops makes the compiler reload every kernel parameter per
// copy (the C4 warp tier spent a third of its instructions there). Ordering against the tile's other SMEM
// accesses comes from cp_async_fence() before a staging loop and cp_async_wait_all() after it.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16_s(uint32_t dst_smem, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst_smem), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_fence() { asm volatile("" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// Per-warp SMEM: a row tile of CP rows x (<= 128 B of K), the Gram [CP][CP+1], norms and ids. K is processed
// in chunks of 128 B (one chunk for uint8 d <= 128), so the tile size does not grow with d.
struct GpLayout {
  int Kb, Kc, pitch;  // bytes of a staged row (multiple of 32), bytes per K-chunk (<= 128), SMEM row pitch (Kc+16)
  size_t rows_off, g_off, nrm_off, ids_off, per_warp;
};
__host__ __device__ inline GpLayout gp_layout(int d, bool u8, int CP) {
  GpLayout L;
  L.Kb = u8 ? (d + 31) / 32 * 32 : (d + 15) / 16 * 32;
  L.Kc = L.Kb < 128 ? L.Kb : 128;
  L.pitch = L.Kc + 16;
  size_t o = 0;
  L.rows_off = o;
  o += (size_t)CP * L.pitch;
  L.g_off = o;
  o += (size_t)CP * (CP + 4) * 4;  // Gram row stride CP + 4 words (see fp_gram_kernel)
  L.nrm_off = o;
  o += (size_t)CP * 4;
  L.ids_off = o;
  o += (size_t)CP * 4;
  L.per_warp = (o + 127) & ~(size_t)127;
  return L;
}

// Stage bytes [kc0, kc0 + Kc) of rows ids[0..nr) into the tile as 16-B chunks (u8 bytes / bf16 coordinates);
// bytes beyond the row and rows nr..nrp-1 are zero. Lane -> (row rr of a pass, chunk ch) is fixed.
template <bool U8>
__device__ __forceinline__ void gp_stage(const void* __restrict__ Xv, int64_t ld, int d, const uint32_t* ids, int nr,
                                         int nrp, uint8_t* rows, const GpLayout& L, int lane, int src_bf16, int kc0) {
  const int cpr = L.Kc >> 4;  // 16-B chunks per row and K-chunk (<= 8)
  const int rpp = 32 / cpr;   // rows per pass
  const int rr = lane / cpr, ch = lane - rr * cpr;
  const bool act = rr < rpp;
  const int cb = kc0 + ch * 16;  // byte offset of this lane's chunk in the staged row
  const bool fast = U8 ? ((d & 15) == 0 && (ld & 15) == 0) : ((d & 7) == 0 && (ld & 3) == 0);
  if ((U8 && fast) || (!U8 && src_bf16)) {
    // cp.async straight into the tile (16 B per lane, zero fill beyond the row and for padding rows); uint8
    // rows of ld bytes, or the bf16 copy's rows of ld elements (zero padded, ld a multiple of 8)
    const int64_t rb = U8 ? ld : 2 * ld;
    const int lim = U8 ? d : (int)(2 * ld);
    cp_async_fence();
    if (act) {
      // branch-free per row: padding rows (r >= nr) re-address the last real row with a zero-byte source
      const bool col_on = cb < lim;
      const uint8_t* xb = (const uint8_t*)Xv + (col_on ? cb : 0);
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(rows + (size_t)rr * L.pitch + ch * 16);
      const uint32_t dstep = (uint32_t)(rpp * L.pitch);
      for (int r = rr; r < nrp; r += rpp, dst += dstep)
        cp_async16_s(dst, xb + (int64_t)ids[min(r, nr - 1)] * rb, (col_on && r < nr) ? 16u : 0u);
    }
    cp_async_wait_all();
    return;
  }
  for (int r0 = 0; r0 < nrp; r0 += 8 * rpp) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int r = r0 + j * rpp + rr;
      v[j] = make_uint4(0u, 0u, 0u, 0u);
      if (act && r < nr) {
        const int64_t id = ids[r];
        if (U8) {
          const uint8_t* src = (const uint8_t*)Xv + id * ld;
          uint32_t w[4] = {0u, 0u, 0u, 0u};
          for (int t = 0; t < 16; ++t)
            if (cb + t < d) w[t >> 2] |= (uint32_t)src[cb + t] << (8 * (t & 3));
          v[j] = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
          const float* src = (const float*)Xv + id * ld;
          const int e0 = cb >> 1;  // first coordinate of the chunk
          float f[8];
          if (fast && e0 < d) {
            const float4 a = __ldg((const float4*)(src + e0));
            const float4 b = __ldg((const float4*)(src + e0 + 4));
            f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
          } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) f[t] = (e0 + t < d) ? __ldg(src + e0 + t) : 0.0f;
          }
          uint32_t w[4];
#pragma unroll
          for (int t = 0; t < 4; ++t)
            w[t] = (uint32_t)f32_to_bf16_rne(f[2 * t]) | ((uint32_t)f32_to_bf16_rne(f[2 * t + 1]) << 16);
          v[j] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int r = r0 + j * rpp + rr;
      if (act && r < nrp) *(uint4*)(rows + (size_t)r * L.pitch + ch * 16) = v[j];
    }
  }
}

// Pass over points (list == nullptr: all points) whose reservoir fits CP-1 candidates; larger ones are
// appended to `defer` for the next tier. final_prune == 1 only (the R-nearest variant uses the generic kernel).
// Per point (one warp): stage rows (u, candidates) -> Gram G on the tensor cores -> lane per candidate i:
// bitmasks P_i (y precedes i in the (D(u,.), id) order) and M_i (y precedes i and an*D(y,i) < ad*D(u,i)) ->
// the lazy scan of P:938-942 (admit i unless an admitted y prunes it) solved as a fixpoint over ballots, no
// sort: the admission order is the (D, id) order, so an admitted i lands at rank popc(admitted & P_i).
template <bool U8, bool MIPS, int CP>
__global__ void __launch_bounds__(256, CP == 32 ? 3 : 1) fp_gram_kernel(const void* __restrict__ Xv, int64_t n, int d, int64_t ld,
                                                      int l_max, const uint64_t* __restrict__ slots,
                                                      const uint32_t* __restrict__ count, int R, int an, int ad,
                                                      uint32_t* __restrict__ nbr_tmp, uint32_t* __restrict__ deg,
                                                      const uint32_t* __restrict__ list,
                                                      const uint32_t* __restrict__ list_n,
                                                      uint32_t* __restrict__ defer, uint32_t* __restrict__ defer_n,
                                                      int src_bf16) {
  using DT = typename std::conditional<U8, int32_t, float>::type;
  static_assert(U8 && !MIPS, "the Gram-in-SMEM warp tier serves uint8 (L2) only; float uses fp_warp_kernel");
  constexpr int E = CP / 32;  // sorted candidates per lane; also the bitmask words per candidate
  extern __shared__ __align__(16) uint8_t gsm[];
  const GpLayout L = gp_layout(d, U8, CP);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  uint8_t* base = gsm + (size_t)warp * L.per_warp;
  uint8_t* rows = base + L.rows_off;
  DT* G = (DT*)(base + L.g_off);  // [CP][CP + 4] Gram
  DT* nrm = (DT*)(base + L.nrm_off);
  uint32_t* ids = (uint32_t*)(base + L.ids_off);
  // Row stride = 4 mod 32 words and the accumulator fragments stored transposed (the Gram is symmetric): element
  // (r, s) of a fragment goes to G[s][r], word (2 t4 + e) DS + g + const = 8 t4 + g + const mod 32 — all 32 lanes
  // of a store on distinct banks (stride CP + 1 with the direct store was a 4-way conflict, 25% of the kernel's
  // shared-memory wavefronts, and the kernel is bound by that pipe: l1tex data-pipe 70% busy).
  const int DS = CP + 4;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t n_iter = list ? (int64_t)*list_n : n;

  for (int64_t it = (int64_t)blockIdx.x * wpb + warp; it < n_iter; it += (int64_t)gridDim.x * wpb) {
    const int64_t u = list ? (int64_t)list[it] : it;
    const int c = (int)count[u];
    if (c > CP - 1) {
      if (lane == 0) defer[atomicAdd(defer_n, 1u)] = (uint32_t)u;
      continue;
    }
    uint32_t* out = nbr_tmp + u * (int64_t)R;
    if (c == 0) {
      if (lane == 0) deg[u] = 0;
      continue;
    }
    const uint64_t* res = slots + u * (int64_t)l_max;
    const int nr = c + 1, nrp = (nr + 15) & ~15;
    for (int t = lane; t < nr; t += 32) ids[t] = t == 0 ? (uint32_t)u : (uint32_t)(res[t - 1] & 0xFFFFFFFFu);
    __syncwarp();
    // ---- Gram on tensor cores, K in chunks of <= 128 B staged per chunk: 16-row blocks x 16-row (two 8-row)
    // blocks, 32-byte K-steps; fragments by ldmatrix (matrix m of x4 = rows +8*(m&1), bytes +16*(m>>1): exactly
    // the a0..a3 / b0,b1 register layout); partial sums of later chunks are added to G in SMEM
    const int nb16 = nrp >> 4;
    const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lcol = (lane >> 4) * 16;
    for (int kc0 = 0; kc0 < L.Kb; kc0 += L.Kc) {
      const int kcn = min(L.Kc, L.Kb - kc0);
      __syncwarp();
      gp_stage<U8>(Xv, ld, d, ids, nr, nrp, rows, L, lane, src_bf16, kc0);
      __syncwarp();
      for (int bi = 0; bi < nb16; ++bi) {
        int32_t acc[CP / 8][4];
#pragma unroll
        for (int bj = 0; bj < CP / 8; ++bj) acc[bj][0] = acc[bj][1] = acc[bj][2] = acc[bj][3] = 0;
        const uint8_t* ra = rows + (size_t)(bi * 16 + lrow) * L.pitch + lcol;
        for (int kb = 0; kb < kcn; kb += 32) {
          uint32_t a[4];
          ldsm_x4(a, ra + kb);
#pragma unroll
          for (int bj2 = 0; bj2 < CP / 16; ++bj2) {
            if (bj2 < nb16) {
              uint32_t bb[4];
              ldsm_x4(bb, rows + (size_t)(bj2 * 16 + lrow) * L.pitch + lcol + kb);
              const uint32_t b0[2] = {bb[0], bb[2]}, b1[2] = {bb[1], bb[3]};
              mma_16x8<U8>(acc[2 * bj2], a, b0);
              mma_16x8<U8>(acc[2 * bj2 + 1], a, b1);
            }
          }
        }
#pragma unroll
        for (int bj = 0; bj < CP / 8; ++bj) {
          if (bj < 2 * nb16) {
            const int r = bi * 16 + g, s = bj * 8 + 2 * t4;
            DT* d0 = G + (size_t)s * DS + r;  // (r, s), (r + 8, s) -> G[s][r], G[s][r + 8]
            DT* d1 = d0 + DS;                 // (r, s + 1), (r + 8, s + 1)
            if (U8) {
              if (kc0 == 0) {
                d0[0] = acc[bj][0]; d1[0] = acc[bj][1]; d0[8] = acc[bj][2]; d1[8] = acc[bj][3];
              } else {
                d0[0] += acc[bj][0]; d1[0] += acc[bj][1]; d0[8] += acc[bj][2]; d1[8] += acc[bj][3];
              }
            } else {
              if (kc0 == 0) {
                d0[0] = __int_as_float(acc[bj][0]); d1[0] = __int_as_float(acc[bj][1]);
                d0[8] = __int_as_float(acc[bj][2]); d1[8] = __int_as_float(acc[bj][3]);
              } else {
                d0[0] += __int_as_float(acc[bj][0]); d1[0] += __int_as_float(acc[bj][1]);
                d0[8] += __int_as_float(acc[bj][2]); d1[8] += __int_as_float(acc[bj][3]);
              }
            }
          }
        }
      }
    }
    __syncwarp();
    for (int r = lane; r < nr; r += 32) nrm[r] = MIPS ? (DT)0 : G[(size_t)r * DS + r];
    __syncwarp();
    // D(r, s) from the Gram: L2 n_r + n_s - 2 G_rs (float: clamped at 0), MIPS -G_rs
    auto Dof = [&](int r, int s, DT nr_, DT ns_) -> DT {
      const DT gg = G[(size_t)r * DS + s];
      if (MIPS) return -gg;
      if (U8) return nr_ + ns_ - 2 * gg;
      return fmaxf(nr_ + ns_ - 2.0f * gg, 0.0f);
    };
    const DT n0 = nrm[0];
    // ---- lane-per-candidate (E per lane): position i = 32 e + lane is candidate row i + 1, key (D(u,v), v)
    uint64_t key[E];
    DT ni[E];
    uint32_t thr_i[E];  // uint8: ad * D(u, v) (exact in 32 bits: D < 2^25, alpha terms <= 127)
    float thr_f[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = e * 32 + lane;
      key[e] = ~0ull;
      ni[e] = 0;
      thr_i[e] = 0;
      thr_f[e] = 0.0f;
      if (i < c) {
        ni[e] = nrm[i + 1];
        const DT Du = Dof(0, i + 1, n0, ni[e]);
        key[e] = ((uint64_t)(U8 ? (uint32_t)Du : f_ord((float)Du)) << 32) | ids[i + 1];
        if (U8) thr_i[e] = (uint32_t)ad * (uint32_t)Du;
        else thr_f[e] = (float)ad * (float)Du;
      }
    }
    // ---- precedence and prune masks, bit y of word w <-> position 32 w + b:
    //   P_i: y precedes i in the (D(u,.), id) order;  M_i: y precedes i and an*D(y,i) < ad*D(u,i)
    uint32_t Pm[E][E], M[E][E];
#pragma unroll
    for (int e = 0; e < E; ++e)
#pragma unroll
      for (int w = 0; w < E; ++w) Pm[e][w] = M[e][w] = 0u;
    // Fast path (one word per lane, d <= 256): the masks over k32 = 32 D(u, i) + i (D < 2^24), which is the
    // (D, id) order unless two candidates share D (checked below; then the general loop). y precedes i iff
    // k32_y - k32_i < 0, and y prunes i iff an (n_y + n_i - 2 G_yi) - ad D(u, i) < 0 (|.| < 2^31 for d <= 256);
    // both bits enter their masks by a funnel shift of the difference's sign (y descending, so bit y lands at
    // position y), M = P & (prune bits).
    bool fast = false;
    if (E == 1 && U8 && d <= 256) {
      const bool vi = lane < c;
      const uint32_t du = (uint32_t)(key[0] >> 32);
      const int32_t k32 = vi ? (int32_t)((du << 5) | (uint32_t)lane) : 0x7FFFFFFF;
      const int32_t ani = an * (int32_t)ni[0];
      const int32_t ci = ani - (int32_t)thr_i[0];
      const int32_t an2 = -2 * an;
      const DT* gcol = G + lane + 1;
      uint32_t P = 0u, Q = 0u;
      for (int y = c - 1; y >= 0; --y) {
        const int32_t ky = __shfl_sync(0xffffffffu, k32, y);
        const int32_t ay = __shfl_sync(0xffffffffu, ani, y);
        const int32_t gy = (int32_t)gcol[(size_t)(y + 1) * DS];
        P = __funnelshift_l((uint32_t)(ky - k32), P, 1);
        Q = __funnelshift_l((uint32_t)(gy * an2 + (ay + ci)), Q, 1);
      }
      // D ties: neighbours in the k32 order (rank = popc(P)) with the same D; G row 0 (D(u, .) is in the keys
      // already) is the scratch
      uint32_t* sc = reinterpret_cast<uint32_t*>(G);
      const int rk = __popc(P);
      __syncwarp();
      if (vi) sc[rk] = du;
      __syncwarp();
      const bool tie = vi && rk + 1 < c && sc[rk + 1] == du;
      fast = __ballot_sync(0xffffffffu, tie) == 0u;
      if (fast) {
        Pm[0][0] = P;
        M[0][0] = P & Q;
      }
    }
#pragma unroll
    for (int wy = 0; wy < (fast ? 0 : E); ++wy) {
      const int ylim = min(32, c - 32 * wy);
      for (int b = 0; b < ylim; ++b) {
        const int y = 32 * wy + b;
        const uint64_t ky = __shfl_sync(0xffffffffu, key[wy], b);
        const DT ny = nrm[y + 1];
        const uint32_t bit = 1u << b;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const bool prec = ky < key[e];
          const DT Dyi = Dof(y + 1, e * 32 + lane + 1, ny, ni[e]);
          bool p;
          if (U8) p = (uint32_t)an * (uint32_t)Dyi < thr_i[e];
          else p = (float)an * (float)Dyi < thr_f[e];
          if (prec) {
            Pm[e][wy] |= bit;
            if (p) M[e][wy] |= bit;
          }
        }
      }
    }
    // ---- lazy RobustPrune as a fixpoint: i is admitted iff no admitted y in M_i. Decided lanes never change;
    // each round decides at least the earliest undecided position, so <= c rounds (typically 2-4).
    uint32_t KA[E], KR[E];  // admitted / rejected positions (warp-uniform)
#pragma unroll
    for (int w = 0; w < E; ++w) {
      const int valid = min(32, max(0, c - 32 * w));
      KA[w] = 0u;
      KR[w] = valid == 32 ? 0u : ~((1u << valid) - 1u);  // positions >= c count as rejected
    }
    for (int round = 0; round < c; ++round) {
      bool undecided_any = false;
      uint32_t adm[E], rej[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const bool undecided = !((KA[e] | KR[e]) >> lane & 1u);
        bool hit = false, open = false;
#pragma unroll
        for (int w = 0; w < E; ++w) {
          hit |= (M[e][w] & KA[w]) != 0u;
          open |= (M[e][w] & ~KR[w]) != 0u;
        }
        adm[e] = __ballot_sync(0xffffffffu, undecided && !hit && !open);
        rej[e] = __ballot_sync(0xffffffffu, undecided && hit);
      }
#pragma unroll
      for (int w = 0; w < E; ++w) {
        KA[w] |= adm[w];
        KR[w] |= rej[w];
        undecided_any |= (KA[w] | KR[w]) != 0xFFFFFFFFu;
      }
      if (!undecided_any) break;
    }
    // ---- output: the first R admitted positions in (D(u,.), id) order ("stop at R")
    int na = 0;
#pragma unroll
    for (int w = 0; w < E; ++w) na += __popc(KA[w]);
    na = min(na, R);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (KA[e] >> lane & 1u) {
        int rank = 0;
#pragma unroll
        for (int w = 0; w < E; ++w) rank += __popc(KA[w] & Pm[e][w]);
        if (rank < R) out[rank] = (uint32_t)(key[e] & 0xFFFFFFFFu);
      }
    }
    if (lane == 0) deg[u] = (uint32_t)na;
    __syncwarp();
  }
}

// ------------------------------------------------------------------ cooperative tiers (CP = 64, 128)
// Staging by a group of nt threads (thread t of the group): the same chunk layout as gp_stage.
template <bool U8>
__device__ __forceinline__ void gp_stage_group(const void* __restrict__ Xv, int64_t ld, int d, const uint32_t* ids,
                                               int nr, int nrp, uint8_t* rows, const GpLayout& L, int t, int nt,
                                               int src_bf16, int kc0) {
  const int cpr = L.Kc >> 4;
  const int rpp = nt / cpr;
  const int rr = t / cpr, ch = t - rr * cpr;
  const bool act = rr < rpp;
  const int cb = kc0 + ch * 16;
  const bool fast = U8 ? ((d & 15) == 0 && (ld & 15) == 0) : ((d & 7) == 0 && (ld & 3) == 0);
  if ((U8 && fast) || (!U8 && src_bf16)) {
    const int64_t rb = U8 ? ld : 2 * ld;
    const int lim = U8 ? d : (int)(2 * ld);
    cp_async_fence();
    if (act) {
      // branch-free per row: padding rows (r >= nr) re-address the last real row with a zero-byte source
      const bool col_on = cb < lim;
      const uint8_t* xb = (const uint8_t*)Xv + (col_on ? cb : 0);
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(rows + (size_t)rr * L.pitch + ch * 16);
      const uint32_t dstep = (uint32_t)(rpp * L.pitch);
      for (int r = rr; r < nrp; r += rpp, dst += dstep)
        cp_async16_s(dst, xb + (int64_t)ids[min(r, nr - 1)] * rb, (col_on && r < nr) ? 16u : 0u);
    }
    cp_async_wait_all();
    return;
  }
  if (!act) return;
  for (int r = rr; r < nrp; r += rpp) {
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (r < nr) {
      const int64_t id = ids[r];
      if (U8) {
        const uint8_t* src = (const uint8_t*)Xv + id * ld;
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        for (int q = 0; q < 16; ++q)
          if (cb + q < d) w[q >> 2] |= (uint32_t)src[cb + q] << (8 * (q & 3));
        v = make_uint4(w[0], w[1], w[2], w[3]);
      } else {
        const float* src = (const float*)Xv + id * ld;
        const int e0 = cb >> 1;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float a = e0 + 2 * q < d ? __ldg(src + e0 + 2 * q) : 0.0f;
          const float b = e0 + 2 * q + 1 < d ? __ldg(src + e0 + 2 * q + 1) : 0.0f;
          w[q] = (uint32_t)f32_to_bf16_rne(a) | ((uint32_t)f32_to_bf16_rne(b) << 16);
        }
        v = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    *(uint4*)(rows + (size_t)r * L.pitch + ch * 16) = v;
  }
}

// ------------------------------------------------------------------ warp tier (<= 31 candidates)
// One warp per point, everything in registers but the staged rows: lane t <-> Gram index t (0 = u, 1..c the
// candidates). The 32x32 Gram (two 16-row bands x four 8-column blocks of mma.sync fragments) stays in the
// accumulators; each thread forms the prune bits an*D(y,r) < ad*D(u,r) of its four rows r, ORs them over the
// quad, and lane i collects its row M_i with one shuffle per (band, half). Lanes rank their candidates by
// (D(u,.), id) and the lazy scan resolves the single batch in sorted order over ballots.
struct WarpLayout {
  int Kb, pitch;
  size_t per_warp;
};
__host__ __device__ inline WarpLayout warp_layout(int d, bool u8) {
  WarpLayout L;
  L.Kb = u8 ? (d + 31) / 32 * 32 : (d + 15) / 16 * 32;
  L.pitch = L.Kb + 16;
  L.per_warp = ((size_t)32 * L.pitch + 2 * 32 * 4 + 32 * 4 + 127) & ~(size_t)127;  // rows | nrm, g0 | perm
  return L;
}

template <bool U8, bool MIPS>
__global__ void __launch_bounds__(256, 3) fp_warp_kernel(const void* __restrict__ Xv, int64_t n, int d, int64_t ld,
                                                        int l_max, const uint64_t* __restrict__ slots,
                                                        const uint32_t* __restrict__ count, int R, int an, int ad,
                                                        uint32_t* __restrict__ nbr_tmp, uint32_t* __restrict__ deg,
                                                        const uint32_t* __restrict__ list,
                                                        const uint32_t* __restrict__ list_n,
                                                        uint32_t* __restrict__ defer, uint32_t* __restrict__ defer_n,
                                                        int src_bf16) {
  using DT = typename std::conditional<U8, int32_t, float>::type;
  extern __shared__ __align__(16) uint8_t wsm[];
  const WarpLayout WL = warp_layout(d, U8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  uint8_t* rows = wsm + (size_t)warp * WL.per_warp;
  DT* nrm = (DT*)(rows + (size_t)32 * WL.pitch);
  DT* g0 = nrm + 32;
  uint32_t* perm = (uint32_t*)(g0 + 32);
  const int g = lane >> 2, t4 = lane & 3;
  const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lcol = (lane >> 4) * 16;
  const int cpr = WL.Kb >> 4;  // 16-B chunks per staged row (<= 32)
  const int rpp = 32 / cpr, rr = lane / cpr, ch = lane - (lane / cpr) * cpr;
  const bool act_stage = rr < rpp;
  const bool fast = U8 ? ((d & 15) == 0 && (ld & 15) == 0) : (src_bf16 != 0);
  const int64_t rowbytes = U8 ? ld : (src_bf16 ? 2 * ld : 4 * ld);
  const int lim = U8 ? d : (src_bf16 ? (int)(2 * ld) : 2 * d);  // staged bytes that come from the source row
  // D (the order key) and D' (the prune test); norms are squared norms for L2, inverse norms for MIPS
  auto Dof = [](DT gg, DT na_, DT nb_) -> DT {
    if (MIPS) return -gg;
    if (U8) return na_ + nb_ - 2 * gg;
    return fmaxf(na_ + nb_ - 2.0f * gg, 0.0f);
  };
  auto Dpr = [&](DT gg, DT na_, DT nb_) -> DT {
    if (MIPS) return (DT)ang_d((float)gg, (float)na_, (float)nb_);
    return Dof(gg, na_, nb_);
  };
  auto val = [](int32_t x) -> DT {
    if (U8) return (DT)x;
    return (DT)__int_as_float(x);
  };
  const int64_t n_iter = list ? (int64_t)*list_n : n;
  for (int64_t it = (int64_t)blockIdx.x * wpb + warp; it < n_iter; it += (int64_t)gridDim.x * wpb) {
    const int64_t u = list ? (int64_t)list[it] : it;
    const int c = (int)count[u];
    if (c > 31) {
      if (lane == 0) defer[atomicAdd(defer_n, 1u)] = (uint32_t)u;
      continue;
    }
    if (c == 0) {
      if (lane == 0) deg[u] = 0;
      continue;
    }
    const int nr = c + 1, nrp = (nr + 15) & ~15;
    const uint32_t my_id = lane == 0 ? (uint32_t)u : (lane <= c ? (uint32_t)(slots[u * (int64_t)l_max + lane - 1] & 0xFFFFFFFFu) : 0u);
    // ---- stage rows 0..nrp-1 (zero beyond nr and beyond the source row), 16-B chunks; lane -> (row rr of
    // a pass of rpp rows, chunk ch) fixed
    __syncwarp();
    if (fast) {
      const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(rows + (size_t)rr * WL.pitch + ch * 16);
      const uint32_t dstep = (uint32_t)(rpp * WL.pitch);
      const bool col_on = act_stage && ch * 16 < lim;
      // the lane's source base: its chunk, or (chunk beyond the row) the row start with a zero-byte copy;
      // rows >= nr read id 0 (lanes > c hold 0) with a zero-byte copy, so every address is a valid row
      const uint8_t* src0 = (const uint8_t*)Xv + (col_on ? ch * 16 : 0);
      uint32_t rb32;  // row stride < 2^32 B; rid * rb32 widened in one IMAD (opaque: kept in a register, not
                      // re-derived from the kernel parameters in every iteration)
      asm("mov.b32 %0, %1;" : "=r"(rb32) : "r"((uint32_t)rowbytes));
      uint32_t dst = dst0;
      cp_async_fence();
      for (int r = rr; r - rr < nrp; r += rpp, dst += dstep) {
        const uint32_t rid = __shfl_sync(0xffffffffu, my_id, r & 31);
        if (act_stage && r < nrp) {
          const uint8_t* src = src0 + (uint64_t)rid * rb32;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                       "r"(col_on && r < nr ? 16u : 0u));
        }
      }
    } else {
      for (int r0 = 0; r0 < nrp; r0 += rpp) {
        const int r = r0 + rr;
        const uint32_t rid = __shfl_sync(0xffffffffu, my_id, r & 31);
        if (act_stage && r < nrp) {
          const int cb = ch * 16;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (r < nr && cb < lim) {
            if (U8) {
              const uint8_t* src = (const uint8_t*)Xv + (int64_t)rid * ld;
              uint32_t w[4] = {0u, 0u, 0u, 0u};
              for (int t = 0; t < 16; ++t)
                if (cb + t < d) w[t >> 2] |= (uint32_t)src[cb + t] << (8 * (t & 3));
              v = make_uint4(w[0], w[1], w[2], w[3]);
            } else {
              const float* src = (const float*)Xv + (int64_t)rid * ld;
              const int e0 = cb >> 1;
              uint32_t w[4];
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float a = e0 + 2 * t < d ? __ldg(src + e0 + 2 * t) : 0.0f;
                const float b = e0 + 2 * t + 1 < d ? __ldg(src + e0 + 2 * t + 1) : 0.0f;
                w[t] = (uint32_t)f32_to_bf16_rne(a) | ((uint32_t)f32_to_bf16_rne(b) << 16);
              }
              v = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
          *(uint4*)(rows + (size_t)r * WL.pitch + cb) = v;
        }
      }
    }
    if (fast) cp_async_wait_all();
    __syncwarp();
    // ---- Gram: bands b = 0 (rows 0-15) and 1 (rows 16-31, when nrp = 32), column blocks of 8
    const bool two = nrp > 16;
    int32_t acc[2][4][4];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int bj = 0; bj < 4; ++bj) acc[b][bj][0] = acc[b][bj][1] = acc[b][bj][2] = acc[b][bj][3] = 0;
    {
      const uint32_t r0a = (uint32_t)__cvta_generic_to_shared(rows + (size_t)lrow * WL.pitch + lcol);
      const uint32_t bstep = 16u * (uint32_t)WL.pitch;
      if (two) {
        for (int kb = 0; kb < WL.Kb; kb += 32) {
          uint32_t a0[4], a1[4], b0r[4], b1r[4];
          ldsm_x4_s(a0, r0a + kb);
          ldsm_x4_s(a1, r0a + bstep + kb);
          b0r[0] = a0[0]; b0r[1] = a0[1]; b0r[2] = a0[2]; b0r[3] = a0[3];  // rows 0-15 as B
          b1r[0] = a1[0]; b1r[1] = a1[1]; b1r[2] = a1[2]; b1r[3] = a1[3];  // rows 16-31 as B
          const uint32_t c0[2] = {b0r[0], b0r[2]}, c1[2] = {b0r[1], b0r[3]};
          const uint32_t c2[2] = {b1r[0], b1r[2]}, c3[2] = {b1r[1], b1r[3]};
          mma_16x8<U8>(acc[0][0], a0, c0);
          mma_16x8<U8>(acc[0][1], a0, c1);
          mma_16x8<U8>(acc[0][2], a0, c2);
          mma_16x8<U8>(acc[0][3], a0, c3);
          mma_16x8<U8>(acc[1][0], a1, c0);
          mma_16x8<U8>(acc[1][1], a1, c1);
          mma_16x8<U8>(acc[1][2], a1, c2);
          mma_16x8<U8>(acc[1][3], a1, c3);
        }
      } else {
        for (int kb = 0; kb < WL.Kb; kb += 32) {
          uint32_t a0[4];
          ldsm_x4_s(a0, r0a + kb);
          const uint32_t c0[2] = {a0[0], a0[2]}, c1[2] = {a0[1], a0[3]};
          mma_16x8<U8>(acc[0][0], a0, c0);
          mma_16x8<U8>(acc[0][1], a0, c1);
        }
      }
    }
    // ---- norms (the Gram diagonal; row r = 16b + 8h + g sits at column block 2b + h, offset g) and row 0
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (2 * t4 + e == g) nrm[16 * b + 8 * h + g] = val(acc[b][2 * b + h][2 * h + e]);
    if (g == 0) {
#pragma unroll
      for (int bj = 0; bj < 4; ++bj) {
        g0[8 * bj + 2 * t4] = val(acc[0][bj][0]);
        g0[8 * bj + 2 * t4 + 1] = val(acc[0][bj][1]);
      }
    }
    __syncwarp();
    // ---- lane i: key (D(u,i), id) and threshold ad*D(u,i)
    const DT n_me = MIPS ? (DT)inv_norm((float)nrm[lane]) : nrm[lane];
    const DT n_u = MIPS ? (DT)inv_norm((float)nrm[0]) : nrm[0];
    const DT Du = Dof(g0[lane], n_u, n_me);
    const bool cand_ok = lane >= 1 && lane <= c;
    const uint64_t key = cand_ok ? (((uint64_t)(U8 ? (uint32_t)Du : f_ord((float)Du)) << 32) | my_id) : ~0ull;
    DT thr_me;
    if (U8) thr_me = (DT)((uint32_t)ad * (uint32_t)Du);
    else thr_me = (DT)((float)ad * (float)Dpr(g0[lane], n_u, n_me));
    // ---- prune bits of rows r = 16b + 8h + g, columns y = 8bj + 2t4 + e
    DT nyv[4][2];
#pragma unroll
    for (int bj = 0; bj < 4; ++bj)
#pragma unroll
      for (int e = 0; e < 2; ++e) nyv[bj][e] = __shfl_sync(0xffffffffu, n_me, 8 * bj + 2 * t4 + e);
    const uint32_t ymask = ((c >= 31) ? 0xFFFFFFFFu : ((2u << c) - 1u)) & ~1u;  // candidates 1..c
    uint32_t mrow[2][2] = {{0u, 0u}, {0u, 0u}};
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (b == 1 && !two) break;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 16 * b + 8 * h + g;
        const DT nr_ = __shfl_sync(0xffffffffu, n_me, r);
        const DT th = __shfl_sync(0xffffffffu, thr_me, r);
        uint32_t w = 0u;
#pragma unroll
        for (int bj = 0; bj < 4; ++bj) {
          if (bj >= 2 && !two) break;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const DT D = Dpr(val(acc[b][bj][2 * h + e]), nr_, nyv[bj][e]);
            bool pr;
            if (U8) pr = (uint32_t)an * (uint32_t)D < (uint32_t)th;
            else pr = (float)an * (float)D < (float)th;
            w |= (pr ? 1u : 0u) << (8 * bj + 2 * t4 + e);
          }
        }
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        mrow[b][h] = w & ymask & ~(1u << r);
      }
    }
    // lane i <- M_i from the quad holding row i (b = i >> 4, h = (i >> 3) & 1, g = i & 7)
    uint32_t Mi = 0u;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t v = __shfl_sync(0xffffffffu, mrow[b][h], 4 * (lane & 7));
        if ((lane >> 4) == b && ((lane >> 3) & 1) == h) Mi = v;
      }
    // ---- bitonic sort of (key, Gram index) over the warp: lane k ends with the k-th candidate (keys are
    // distinct; non-candidates carry ~0 and sort last)
    uint64_t sk = key;
    int i = lane;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const uint64_t ok = __shfl_xor_sync(0xffffffffu, sk, stride);
        const int oi = __shfl_xor_sync(0xffffffffu, i, stride);
        const bool up = (lane & size) == 0;           // ascending block
        const bool lower = (lane & stride) == 0;      // this lane keeps the smaller of the pair when up
        const bool take = (lower == up) ? (ok < sk) : (ok > sk);
        if (take) {
          sk = ok;
          i = oi;
        }
      }
    }
    // ---- lazy scan in sorted order: lane k holds the k-th candidate's Gram index and prune mask; the
    // admitted set (Gram-index bits) is updated once per step
    const bool inb = lane < c;
    const uint32_t Mk = __shfl_sync(0xffffffffu, Mi, i);
    uint32_t adm = 0u, admS = 0u;
    for (int k = 0; k < c; ++k) {
      const uint32_t mk = __shfl_sync(0xffffffffu, Mk, k);
      const int ik = __shfl_sync(0xffffffffu, i, k);
      if ((mk & adm) == 0u) {
        adm |= 1u << ik;
        admS |= 1u << k;
      }
    }
    const uint32_t id_i = __shfl_sync(0xffffffffu, my_id, i);
    const int pos = __popc(admS & ((1u << lane) - 1u));
    if (((admS >> lane) & 1u) && pos < R) nbr_tmp[u * (int64_t)R + pos] = id_i;
    if (lane == 0) deg[u] = (uint32_t)min(__popc(admS), R);
  }
}

// ------------------------------------------------------------------ band tiers (CP = 64, 128, 192)
// One point per CTA pass: CP/16 "band" warps and one "scan" warp. Band warp b owns the 16-row band b of the
// (c+1)x(c+1) Gram, whole rows staged once (no K chunks, so the accumulators stay in registers and the Gram
// never goes to SMEM). From its fragments each thread forms the prune bits of its two rows r
// (an*D(y,r) < ad*D(u,r), every y: in the scan only earlier y can act) and ORs them over the quad into 32-bit
// words M[r]. The scan warp ranks the candidates by (D(u,.), id) and runs the lazy scan 32
// candidates at a time (a lane per candidate, pruned by the admitted set A or by an earlier admitted candidate
// of its batch, resolved over ballots) while the band warps already work on the next point: ids, keys and M
// are double buffered and handed over with named barriers (READY[b]: band -> scan, FREE[b]: scan -> band).
struct BandLayout {
  int Kb, pitch;
  size_t rows_off, m_off, key_off, nrm_off, g0_off, thr_off, ids_off, perm_off, bytes;
};
__host__ __device__ inline BandLayout band_layout(int d, bool u8, int CP) {
  BandLayout L;
  L.Kb = u8 ? (d + 31) / 32 * 32 : (d + 15) / 16 * 32;
  L.pitch = L.Kb + 16;  // odd multiple of 16 B: conflict-free ldmatrix rows
  size_t o = 0;
  L.rows_off = o;
  o += (size_t)CP * L.pitch;
  L.m_off = o;  // [2][CP][CP/32]
  o += (size_t)2 * CP * (CP / 32) * 4;
  L.key_off = o;  // [2][CP]
  o += (size_t)2 * CP * 8;
  L.nrm_off = o;
  o += (size_t)CP * 4;
  L.g0_off = o;
  o += (size_t)CP * 4;
  L.thr_off = o;
  o += (size_t)CP * 4;
  L.ids_off = o;  // [2][CP]
  o += (size_t)2 * CP * 4;
  L.perm_off = o;  // [2][CP]
  o += (size_t)2 * CP * 4;
  L.bytes = (o + 127) & ~(size_t)127;
  return L;
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <bool U8, bool MIPS, int CP>
__global__ void __launch_bounds__(2 * CP + 32, CP <= 64 ? 4 : (CP <= 128 ? 2 : 1)) fp_band_kernel(const void* __restrict__ Xv, int64_t n, int d, int64_t ld,
                                                       int l_max, const uint64_t* __restrict__ slots,
                                                       const uint32_t* __restrict__ count, int R, int an, int ad,
                                                       uint32_t* __restrict__ nbr_tmp, uint32_t* __restrict__ deg,
                                                       const uint32_t* __restrict__ list,
                                                       const uint32_t* __restrict__ list_n,
                                                       uint32_t* __restrict__ defer, uint32_t* __restrict__ defer_n,
                                                       int src_bf16) {
  using DT = typename std::conditional<U8, int32_t, float>::type;
  constexpr int NW = CP / 16;  // band warps
  constexpr int NB_T = 32 * NW;  // band threads
  constexpr int W = CP / 32;   // mask words per row
  constexpr int NB = CP / 8;   // 8-column fragments per band
  constexpr int kBarBand = 1, kBarReady = 2, kBarFree = 4;  // named barriers (0 = __syncthreads)
  extern __shared__ __align__(16) uint8_t bsm[];
  const BandLayout BL = band_layout(d, U8, CP);
  GpLayout L;  // full-row staging view for gp_stage_group
  L.Kb = BL.Kb;
  L.Kc = BL.Kb;
  L.pitch = BL.pitch;
  uint8_t* rows = bsm + BL.rows_off;
  uint32_t* Mb = (uint32_t*)(bsm + BL.m_off);
  uint64_t* skeyb = (uint64_t*)(bsm + BL.key_off);
  DT* nrm = (DT*)(bsm + BL.nrm_off);
  DT* g0 = (DT*)(bsm + BL.g0_off);
  DT* thr = (DT*)(bsm + BL.thr_off);
  uint32_t* idsb = (uint32_t*)(bsm + BL.ids_off);
  uint32_t* permb = (uint32_t*)(bsm + BL.perm_off);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n_iter = list ? (int64_t)*list_n : n;
  int p = 0;  // points handed over so far (buffer = p & 1)
  if (warp < NW) {
    // ================================================================ band warps
    const int g = lane >> 2, t4 = lane & 3;
    const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lcol = (lane >> 4) * 16;
    // D (order key) and D' (prune test); nrm holds squared norms (L2) or inverse norms (MIPS)
    auto Dof = [](DT gg, DT na_, DT nb_) -> DT {
      if (MIPS) return -gg;
      if (U8) return na_ + nb_ - 2 * gg;
      return fmaxf(na_ + nb_ - 2.0f * gg, 0.0f);
    };
    auto Dpr = [&](DT gg, DT na_, DT nb_) -> DT {
      if (MIPS) return (DT)ang_d((float)gg, (float)na_, (float)nb_);
      return Dof(gg, na_, nb_);
    };
    auto val = [](int32_t x) -> DT {
      if (U8) return (DT)x;
      return (DT)__int_as_float(x);
    };
    for (int64_t it = blockIdx.x; it < n_iter; it += gridDim.x) {
      const int64_t u = list ? (int64_t)list[it] : it;
      const int c = (int)count[u];
      if (c > CP - 1) {
        if (tid == 0) defer[atomicAdd(defer_n, 1u)] = (uint32_t)u;
        continue;
      }
      if (c == 0) {
        if (tid == 0) deg[u] = 0;
        continue;
      }
      const int bsel = p & 1;
      uint32_t* ids = idsb + bsel * CP;
      uint32_t* M = Mb + bsel * CP * W;
      uint64_t* skey = skeyb + bsel * CP;
      uint32_t* perm = permb + bsel * CP;
      if (p >= 2) named_sync(kBarFree + bsel, NB_T + 32);  // the scan of point p-2 released this buffer
      const uint64_t* res = slots + u * (int64_t)l_max;
      const int nr = c + 1, nrp = (nr + 15) & ~15;
      named_sync(kBarBand, NB_T);  // the previous point's rows / nrm / g0 / thr are no longer read
      for (int t = tid; t < nr; t += NB_T) ids[t] = t == 0 ? (uint32_t)u : (uint32_t)(res[t - 1] & 0xFFFFFFFFu);
      named_sync(kBarBand, NB_T);
      gp_stage_group<U8>(Xv, ld, d, ids, nr, nrp, rows, L, tid, NB_T, src_bf16, 0);
      named_sync(kBarBand, NB_T);
      // ---- Gram band of this warp (rows 16*warp .. +15), every column block (rows beyond nrp hold stale
      // bytes; their columns are never read), K = the whole row
      const bool act = warp * 16 < nrp;
      int32_t acc[NB][4];
#pragma unroll
      for (int bj = 0; bj < NB; ++bj) acc[bj][0] = acc[bj][1] = acc[bj][2] = acc[bj][3] = 0;
      if (act) {
        const uint32_t ra = (uint32_t)__cvta_generic_to_shared(rows + (size_t)(warp * 16 + lrow) * L.pitch + lcol);
        const uint32_t rb = (uint32_t)__cvta_generic_to_shared(rows + (size_t)lrow * L.pitch + lcol);
        const uint32_t bstep = 16u * (uint32_t)L.pitch;
        for (int kb = 0; kb < L.Kb; kb += 32) {
          uint32_t a[4];
          ldsm_x4_s(a, ra + kb);
#pragma unroll
          for (int bj2 = 0; bj2 < CP / 16; ++bj2) {
            uint32_t bb[4];
            ldsm_x4_s(bb, rb + bj2 * bstep + kb);
            const uint32_t b0[2] = {bb[0], bb[2]}, b1[2] = {bb[1], bb[3]};
            mma_16x8<U8>(acc[2 * bj2], a, b0);
            mma_16x8<U8>(acc[2 * bj2 + 1], a, b1);
          }
        }
      }
      const int r0 = warp * 16 + g, r1 = r0 + 8;
      // ---- row 0 of the Gram (u against every candidate) and the squared norms (from the staged rows)
      if (warp == 0 && g == 0) {
#pragma unroll
        for (int bj = 0; bj < NB; ++bj) {
          g0[bj * 8 + 2 * t4] = val(acc[bj][0]);
          g0[bj * 8 + 2 * t4 + 1] = val(acc[bj][1]);
        }
      }
      {
        for (int r = tid; r < nr; r += NB_T) {
          const uint4* rw = reinterpret_cast<const uint4*>(rows + (size_t)r * L.pitch);
          int32_t si = 0;
          float sf = 0.0f;
          for (int q = 0; q < (L.Kb >> 4); ++q) {
            const uint4 v4 = rw[q];
            const uint32_t wv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (U8) {
                si = (int32_t)__dp4a(wv[e], wv[e], (uint32_t)si);
              } else {
                const float lo = __uint_as_float(wv[e] << 16), hi = __uint_as_float(wv[e] & 0xFFFF0000u);
                sf = fmaf(lo, lo, sf);
                sf = fmaf(hi, hi, sf);
              }
            }
          }
          if (U8) nrm[r] = (DT)si;
          else nrm[r] = MIPS ? (DT)inv_norm(sf) : (DT)sf;
        }
      }
      named_sync(kBarBand, NB_T);
      // ---- keys (D(u,y), id) and thresholds ad*D(u,y) of the candidates y = 1..c
      for (int y = tid + 1; y <= c; y += NB_T) {
        const DT ny = nrm[y];
        const DT Du = Dof(g0[y], nrm[0], ny);
        skey[y] = ((uint64_t)(U8 ? (uint32_t)Du : f_ord((float)Du)) << 32) | ids[y];
        if (U8) thr[y] = (DT)((uint32_t)ad * (uint32_t)Du);
        else thr[y] = (DT)((float)ad * (float)Dpr(g0[y], nrm[0], ny));
      }
      named_sync(kBarBand, NB_T);
      // ---- prune bits of rows r0, r1 (Gram indices; candidates are 1..c), OR-reduced over the quad
      if (act) {
        const DT n0 = r0 > c ? (DT)0 : nrm[r0], n1 = r1 > c ? (DT)0 : nrm[r1];
        const DT th0 = (r0 >= 1 && r0 <= c) ? thr[r0] : (DT)0, th1 = (r1 >= 1 && r1 <= c) ? thr[r1] : (DT)0;
        uint32_t w0[W], w1[W];
#pragma unroll
        for (int k = 0; k < W; ++k) w0[k] = w1[k] = 0u;
#pragma unroll
        for (int bj = 0; bj < NB; ++bj) {
          if (bj * 8 < nrp) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int y = bj * 8 + 2 * t4 + e;
              if (y >= 1 && y <= c) {
                const DT ny = nrm[y];
                const DT D0 = Dpr(val(acc[bj][e]), n0, ny), D1 = Dpr(val(acc[bj][2 + e]), n1, ny);
                bool p0, p1;
                if (U8) {
                  p0 = (uint32_t)an * (uint32_t)D0 < (uint32_t)th0;
                  p1 = (uint32_t)an * (uint32_t)D1 < (uint32_t)th1;
                } else {
                  p0 = (float)an * (float)D0 < (float)th0;
                  p1 = (float)an * (float)D1 < (float)th1;
                }
                const uint32_t bit = 1u << ((bj & 3) * 8 + 2 * t4 + e);
                if (p0 && y != r0) w0[bj >> 2] |= bit;
                if (p1 && y != r1) w1[bj >> 2] |= bit;
              }
            }
          }
        }
#pragma unroll
        for (int k = 0; k < W; ++k) {
          w0[k] |= __shfl_xor_sync(0xffffffffu, w0[k], 1);
          w0[k] |= __shfl_xor_sync(0xffffffffu, w0[k], 2);
          w1[k] |= __shfl_xor_sync(0xffffffffu, w1[k], 1);
          w1[k] |= __shfl_xor_sync(0xffffffffu, w1[k], 2);
        }
        if (t4 == 0) {
#pragma unroll
          for (int k = 0; k < W; ++k) {
            if (r0 <= c) M[r0 * W + k] = w0[k];
            if (r1 <= c) M[r1 * W + k] = w1[k];
          }
        }
      }
      // ---- rank of every candidate in the (D(u,.), id) order (keys are distinct: ids are), a thread per
      // candidate (done here, in parallel, rather than in the scan warp, which bounds the tier)
      for (int y = tid + 1; y <= c; y += NB_T) {
        const uint64_t ky = skey[y];
        int rank = 0;
        for (int z = 1; z <= c; ++z) rank += skey[z] < ky ? 1 : 0;
        perm[rank] = (uint32_t)y;
      }
      __threadfence_block();
      named_arrive(kBarReady + bsel, NB_T + 32);  // ids, keys, M and the ranks of point p are complete
      ++p;
    }
  } else {
    // ================================================================ scan warp
    for (int64_t it = blockIdx.x; it < n_iter; it += gridDim.x) {
      const int64_t u = list ? (int64_t)list[it] : it;
      const int c = (int)count[u];
      if (c > CP - 1 || c == 0) continue;
      const int bsel = p & 1;
      const uint32_t* ids = idsb + bsel * CP;
      const uint32_t* M = Mb + bsel * CP * W;
      const uint32_t* perm = permb + bsel * CP;
      named_sync(kBarReady + bsel, NB_T + 32);
      // ---- lazy scan, 32 candidates per step
      uint32_t* out = nbr_tmp + u * (int64_t)R;
      uint32_t A[W];
#pragma unroll
      for (int k = 0; k < W; ++k) A[k] = 0u;
      int na = 0;
      for (int b0 = 0; b0 < c && na < R; b0 += 32) {
        const bool inb = b0 + lane < c;
        const int i = inb ? (int)perm[b0 + lane] : 0;
        const uint32_t* Mi = M + i * W;
        bool hitA = false;
#pragma unroll
        for (int k = 0; k < W; ++k) hitA |= ((inb ? Mi[k] : 0u) & A[k]) != 0u;
        // intra-batch pruners: bit k = candidate at batch position k (< lane) prunes me
        uint32_t intra = 0u;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const int ik = __shfl_sync(0xffffffffu, i, k);
          if (k < lane && inb && ((Mi[ik >> 5] >> (ik & 31)) & 1u)) intra |= 1u << k;
        }
        const uint32_t cand = __ballot_sync(0xffffffffu, inb && !hitA);
        // the batch's sequential scan (admit k unless an admitted earlier candidate prunes it) as a fixpoint
        // over ballots: a lane is admitted once all its in-batch pruners are rejected, rejected once one is
        // admitted; the earliest undecided lane always decides, typically 2-4 rounds instead of 32 steps
        uint32_t adm = 0u, rej = ~cand;
        while ((adm | rej) != 0xFFFFFFFFu) {
          const bool undecided = !(((adm | rej) >> lane) & 1u);
          const bool hit = (intra & adm) != 0u, open = (intra & ~rej) != 0u;
          const uint32_t a = __ballot_sync(0xffffffffu, undecided && !hit && !open);
          const uint32_t r = __ballot_sync(0xffffffffu, undecided && hit);
          adm |= a;
          rej |= r;
        }
        const bool me = (adm >> lane) & 1u;
        const int pos = na + __popc(adm & ((1u << lane) - 1u));
        if (me && pos < R) out[pos] = ids[i];
        na += __popc(adm);
#pragma unroll
        for (int k = 0; k < W; ++k)
          A[k] |= __reduce_or_sync(0xffffffffu, (me && (i >> 5) == k) ? (1u << (i & 31)) : 0u);
      }
      if (lane == 0) deg[u] = (uint32_t)min(na, R);
      __syncwarp();
      named_arrive(kBarFree + bsel, NB_T + 32);  // buffer bsel may be refilled (point p + 2)
      ++p;
    }
  }
}

__global__ void csr_copy_kernel(int64_t n, int R, const uint32_t* __restrict__ nbr_tmp, const uint32_t* __restrict__ deg,
                                const uint64_t* __restrict__ row_ptr, uint32_t* __restrict__ col_idx) {
  // a warp per 32 consecutive points: their degrees and offsets in one coalesced load each, then the rows in
  // groups of 4 points with all loads of a group in flight before its stores (latency-bound otherwise)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunk = (n + 31) >> 5;
  for (int64_t ch = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; ch < nchunk;
       ch += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t u0 = ch << 5;
    const int64_t ul = u0 + lane;
    const uint32_t dgl = ul < n ? deg[ul] : 0u;
    const uint64_t ol = ul < n ? row_ptr[ul] : 0ull;
    if (R <= 32) {
      // one entry per lane and row: all 32 rows' loads in flight, then the 32 stores
      uint32_t v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const uint32_t dq = __shfl_sync(0xffffffffu, dgl, q);
        v[q] = (uint32_t)lane < dq ? nbr_tmp[(u0 + q) * (int64_t)R + lane] : 0u;
      }
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const uint32_t dq = __shfl_sync(0xffffffffu, dgl, q);
        const uint64_t oq = __shfl_sync(0xffffffffu, ol, q);
        if ((uint32_t)lane < dq) col_idx[oq + lane] = v[q];
      }
      continue;
    }
    for (int j0 = 0; j0 < 32; j0 += 4) {
      uint32_t v[4][2];
      uint32_t dgs[4];
      uint64_t os[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        dgs[q] = __shfl_sync(0xffffffffu, dgl, j0 + q);
        os[q] = __shfl_sync(0xffffffffu, ol, j0 + q);
        const uint32_t* src = nbr_tmp + (u0 + j0 + q) * (int64_t)R;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t t = lane + 32 * h;
          v[q][h] = t < dgs[q] ? src[t] : 0u;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t t = lane + 32 * h;
          if (t < dgs[q]) col_idx[os[q] + t] = v[q][h];
        }
      }
      // rows longer than 64 entries (R > 64)
      for (int q = 0; q < 4; ++q)
        for (uint32_t t = 64 + lane; t < dgs[q]; t += 32)
          col_idx[os[q] + t] = nbr_tmp[(u0 + j0 + q) * (int64_t)R + t];
    }
  }
}

// Processing order of the final prune in pipnn_build: every point once, at its first instance in leaf order,
// so the warps of an SM at any moment gather candidate rows of the same few leaves (L2 reuse).
__global__ void first_instance_kernel(const uint32_t* __restrict__ leaf_ids, int64_t I, uint32_t* __restrict__ first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x)
    atomicMin(&first[leaf_ids[i]], (uint32_t)i);
}
__global__ void first_flag_kernel(const uint32_t* __restrict__ leaf_ids, int64_t I, const uint32_t* __restrict__ first,
                                  uint8_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = first[leaf_ids[i]] == (uint32_t)i;
}

pipnn_status leaf_order(const uint32_t* leaf_ids, int64_t n_inst, int64_t n, uint32_t* order, uint32_t* order_n,
                        Arena& ar, const Ctx& c) {
  uint32_t* first = ar.take<uint32_t>(n);
  uint8_t* flag = ar.take<uint8_t>(std::max<int64_t>(1, n_inst));
  size_t tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, leaf_ids, flag, order, order_n, (int)std::max<int64_t>(1, n_inst));
  void* tmp = ar.take<uint8_t>(tb);
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (leaf_order)");
  PIPNN_CUDA(kmemset(first, 0xFF, (size_t)n * sizeof(uint32_t), c.st));
  const int64_t g = std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_inst, 256), num_sms() * 32));
  first_instance_kernel<<<(unsigned)g, 256, 0, c.st>>>(leaf_ids, n_inst, first);
  PIPNN_LAUNCHED("first_instance_kernel", c.st);
  first_flag_kernel<<<(unsigned)g, 256, 0, c.st>>>(leaf_ids, n_inst, first, flag);
  PIPNN_LAUNCHED("first_flag_kernel", c.st);
  PIPNN_CUDA(cub::DeviceSelect::Flagged(tmp, tb, leaf_ids, flag, order, order_n, (int)n_inst, c.st));
  return PIPNN_OK;
}

pipnn_status final_prune_impl(const pipnn_points* X, int l_max, const uint64_t* slots, const uint32_t* count,
                              const pipnn_prune_params* p, uint64_t* row_ptr, uint32_t* col_idx, Arena& ar,
                              const Ctx& c, const uint32_t* order, const uint32_t* order_n, const pipnn_points* Xb) {
  const int64_t n = X->n;
  const pipnn_points* Xg = Xb ? Xb : X;  // rows the Gram path reads (the bf16 copy of float data when given)
  const int src_bf16 = Xg->dtype == kDtypeBf16 ? 1 : 0;
  const int R = p->R;
  uint32_t* nbr_tmp = ar.take<uint32_t>((size_t)n * R);
  uint32_t* deg = ar.take<uint32_t>(n + 1);
  uint32_t* defer = ar.take<uint32_t>((size_t)4 * n);
  uint32_t* defer_n = ar.take<uint32_t>(5);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (const uint32_t*)nullptr, (uint64_t*)nullptr, (int)(n + 1));
  void* tmp = ar.take<uint8_t>(tmp_bytes);
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (final_prune)");
  if (R > 256) return fail(PIPNN_EUNSUPPORTED, "R > 256");
  const bool u8 = X->dtype == PIPNN_U8, mips = X->metric == PIPNN_MIPS;
  PIPNN_CUDA(kmemset(deg + n, 0, sizeof(uint32_t), c.st));
  PIPNN_CUDA(kmemset(defer_n, 0, 5 * sizeof(uint32_t), c.st));
  const size_t pair_bytes = (size_t)kFpStage * (kFpStage - 1) * 2;  // u16 (i, j) pairs of the generic kernel
  int cap1 = l_max;
  FpLayout L1 = fp_layout(X->d, u8, l_max, cap1);
  while (cap1 > kFpStage && L1.per_warp + pair_bytes > 200 * 1024) L1 = fp_layout(X->d, u8, l_max, cap1 -= 16);
  const int smem1 = (int)(L1.per_warp + pair_bytes);
  if (p->final_prune) {
    // tiers of the Gram path: <= 31, <= 63, <= 127 candidates; anything larger -> generic kernel
    const uint32_t* in_list = order;  // nullptr: points in id order
    const uint32_t* in_n = order_n;
    bool first_tier = true;
    static const bool warp_u8 = std::getenv("PIPNN_FP_WARP_U8") != nullptr;  // experiment hook, read once
#define GP_TIER(U, M, CPV, T)                                                                                      \
  do {                                                                                                             \
    const GpLayout GL = gp_layout(X->d, U, CPV);                                                                   \
    int w = (int)std::min<size_t>(8, (200 * 1024) / GL.per_warp);                                                  \
    if (w < 1) return fail(PIPNN_EUNSUPPORTED, "final prune: row too large for the Gram tile");                   \
    const int sm = (int)(w * GL.per_warp);                                                                         \
    auto* fn = fp_gram_kernel<U, M, CPV>;                                                                          \
    PIPNN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));                         \
    const int64_t blocks = first_tier ? std::min<int64_t>(ceil_div(n, w), num_sms() * 32) : (int64_t)num_sms() * 4; \
    first_tier = false;                                                                                            \
    fn<<<(unsigned)blocks, 32 * w, sm, c.st>>>(Xg->data, n, X->d, Xg->ld, l_max, slots, count, R, p->alpha_num,    \
                                               p->alpha_den, nbr_tmp, deg, in_list, in_n, defer + (T) * n,        \
                                               defer_n + (T), src_bf16);                                           \
    PIPNN_LAUNCHED("fp_gram_kernel", c.st);                                                                        \
    in_list = defer + (T) * n;                                                                                     \
    in_n = defer_n + (T);                                                                                          \
  } while (0)
#define GP_BAND(U, M, CPV, T)                                                                                      \
  do {                                                                                                             \
    const BandLayout BL = band_layout(X->d, U, CPV);                                                               \
    const int sm = (int)BL.bytes;                                                                                  \
    auto* fn = fp_band_kernel<U, M, CPV>;                                                                          \
    PIPNN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));                         \
    const int per_sm = std::max(1, std::min(2048 / (2 * CPV + 32), (int)((227 * 1024) / (sm + 1024))));            \
    fn<<<(unsigned)(num_sms() * per_sm), 2 * CPV + 32, sm, c.st>>>(Xg->data, n, X->d, Xg->ld, l_max, slots, count, R, \
                                                              p->alpha_num, p->alpha_den, nbr_tmp, deg, in_list,    \
                                                              in_n, defer + (T) * n, defer_n + (T), src_bf16);      \
    PIPNN_LAUNCHED("fp_band_kernel", c.st);                                                                        \
    in_list = defer + (T) * n;                                                                                     \
    in_n = defer_n + (T);                                                                                          \
  } while (0)
#define GP_WARP(U, M)                                                                                              \
  do {                                                                                                             \
    const WarpLayout WL = warp_layout(X->d, U);                                                                    \
    int w = (int)std::min<size_t>(8, (200 * 1024) / WL.per_warp);                                                  \
    if (w < 1) return fail(PIPNN_EUNSUPPORTED, "final prune: row too large for the warp tile");                   \
    const int sm = (int)(w * WL.per_warp);                                                                         \
    auto* fn = fp_warp_kernel<U, M>;                                                                               \
    PIPNN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));                         \
    const int64_t blocks = std::min<int64_t>(ceil_div(n, w), num_sms() * 32);                                      \
    first_tier = false;                                                                                            \
    fn<<<(unsigned)blocks, 32 * w, sm, c.st>>>(Xg->data, n, X->d, Xg->ld, l_max, slots, count, R, p->alpha_num,    \
                                               p->alpha_den, nbr_tmp, deg, in_list, in_n, defer, defer_n,          \
                                               src_bf16);                                                          \
    PIPNN_LAUNCHED("fp_warp_kernel", c.st);                                                                        \
    in_list = defer;                                                                                               \
    in_n = defer_n;                                                                                                \
  } while (0)
#define GP_ALL(U, M)                                                                                               \
  do {                                                                                                             \
    if (U && !warp_u8) GP_TIER(true, false, 32, 0); else GP_WARP(U, M);                                            \
    if (l_max > 31) GP_BAND(U, M, 64, 1);                                                                          \
    if (l_max > 63) GP_BAND(U, M, 128, 2);                                                                         \
    if (l_max > 127 && band_layout(X->d, U, 192).bytes <= 200 * 1024) GP_BAND(U, M, 192, 3);                       \
    if (l_max > (band_layout(X->d, U, 192).bytes <= 200 * 1024 ? 191 : 127)) {                                     \
      auto* fn = final_prune_kernel<U, M>;                                                                         \
      PIPNN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1));                    \
      fn<<<(unsigned)(num_sms() * 2), 32, smem1, c.st>>>(X->data, n, X->d, X->ld, l_max, slots, count, R,          \
                                                        p->alpha_num, p->alpha_den, 1, nbr_tmp, deg, cap1, in_list, \
                                                        in_n, nullptr, nullptr);                                    \
      PIPNN_LAUNCHED("final_prune_kernel(generic)", c.st);                                                         \
    }                                                                                                              \
  } while (0)
    if (u8) GP_ALL(true, false);
    else if (mips) GP_ALL(false, true);
    else GP_ALL(false, false);
    static const bool dbg_timing = [] {
      const char* e = std::getenv("PIPNN_DEBUG_TIMING");
      return e && e[0] == '1';
    }();
    if (dbg_timing) {  // tier sizes (points with <= 31 / <= 63 / <= 127 / more candidates)
      uint32_t hd[4] = {0, 0, 0, 0};
      PIPNN_CUDA(cudaMemcpyAsync(hd, defer_n, sizeof(hd), cudaMemcpyDeviceToHost, c.st));
      PIPNN_CUDA(cudaStreamSynchronize(c.st));
      std::fprintf(stderr, "[pipnn] final prune tiers: <=31 %lld, <=63 %u, <=127 %u, >127 %u\n",
                   (long long)(n - hd[0]), hd[0] - hd[1], hd[1] - hd[2], hd[2]);
    }
#undef GP_ALL
#undef GP_BAND
#undef GP_WARP
#undef GP_TIER
  } else {
    // final_prune = 0: the R nearest reservoir entries, generic kernel
    const FpLayout L0 = fp_layout(X->d, u8, l_max, kFpStage);
    int wpb = 8;
    while (wpb > 1 && (size_t)wpb * L0.per_warp > 96 * 1024) wpb >>= 1;
    const int smem0 = (int)(wpb * L0.per_warp + pair_bytes);
    const int64_t blocks = std::min<int64_t>(ceil_div(n, wpb), (int64_t)num_sms() * 16);
#define FP_LAUNCH(U, M)                                                                                            \
  do {                                                                                                             \
    auto* fn = final_prune_kernel<U, M>;                                                                           \
    PIPNN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, std::max(smem0, smem1)));      \
    fn<<<(unsigned)blocks, 32 * wpb, smem0, c.st>>>(X->data, n, X->d, X->ld, l_max, slots, count, R, p->alpha_num,  \
                                                    p->alpha_den, 0, nbr_tmp, deg, kFpStage, nullptr, nullptr,      \
                                                    nullptr, nullptr);                                              \
    PIPNN_LAUNCHED("final_prune_kernel", c.st);                                                                    \
  } while (0)
    if (u8) FP_LAUNCH(true, false);
    else if (mips) FP_LAUNCH(false, true);
    else FP_LAUNCH(false, false);
#undef FP_LAUNCH
  }
  PIPNN_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, deg, row_ptr, (int)(n + 1), c.st));
  csr_copy_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), num_sms() * 16), 256, 0, c.st>>>(n, R, nbr_tmp, deg,
                                                                                                 row_ptr, col_idx);
  PIPNN_LAUNCHED("csr_copy_kernel", c.st);
  return PIPNN_OK;
}

}  // namespace pipnn
