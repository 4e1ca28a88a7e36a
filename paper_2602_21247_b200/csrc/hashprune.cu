// hashprune.cu — HashPrune reservoirs (§3, Alg. 3) on the GPU.
//
// Alg. 3 is sequential per point, but its result is history independent (proof P:1125-1129):
// the final reservoir of u is the l_max nearest (by (bf16 dist, id), R4/R5) of the per-hash-
// bucket minima of everything ever streamed to u. Applied to "old reservoir U new batch" this is exactly
// what Alg. 3 returns after streaming the batch into the old reservoir, so the kernel below
//   (1) groups a batch of directed edges by owner (counting sort: histogram -> scan -> scatter; the order
//       inside an owner's segment is irrelevant and left to the atomics), and
//   (2) merges each owner's segment into its reservoir with one warp: bitonic-sort the u64 slot keys
//       hash<<48 | okey(bf16 D)<<32 | id, keep the first key of every hash run (the bucket minimum), and if
//       more than l_max buckets survive keep the l_max smallest by (okey, id); write back sorted by hash.
// Segments longer than the warp's SMEM capacity are merged in chunks (exact by the same lemma).
#include <cub/cub.cuh>

#include "internal.h"

namespace pipnn {

// residual hash h_u(v): bit i = [S(v)_i >= S(u)_i] (Eq. 1 via sketches)
template <typename ST>
__device__ __forceinline__ uint32_t residual_hash(const ST* __restrict__ S, int m, uint32_t u, uint32_t v) {
  const ST* su = S + (int64_t)u * m;
  const ST* sv = S + (int64_t)v * m;
  uint32_t h = 0;
  for (int i = 0; i < m; ++i) h |= (uint32_t)(sv[i] >= su[i]) << i;
  return h;
}

template <typename ST>
__device__ __forceinline__ uint64_t slot_key(const ST* S, int m, uint32_t owner, uint32_t cand, float D) {
  const uint64_t h = residual_hash<ST>(S, m, owner, cand);
  return (h << 48) | ((uint64_t)dist_order_key(D) << 32) | (uint64_t)cand;
}

// ------------------------------------------------------------------ grouping of explicit edge batches
__global__ void hp_hist_kernel(const uint32_t* __restrict__ owner, int64_t E, uint32_t* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[owner[e]], 1u);
}

template <typename ST>
__global__ void hp_scatter_kernel(const uint32_t* __restrict__ owner, const uint32_t* __restrict__ cand,
                                  const float* __restrict__ dist, int64_t E, const ST* __restrict__ S, int m,
                                  const uint64_t* __restrict__ start, uint32_t* __restrict__ cursor,
                                  uint64_t* __restrict__ keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = owner[e];
    const uint64_t pos = start[u] + atomicAdd(&cursor[u], 1u);
    keys[pos] = slot_key<ST>(S, m, u, cand[e], dist[e]);
  }
}

// ------------------------------------------------------------------ grouping of candidate lists (build path)
// Instance i holds point p = leaf_ids[i] and its picks nbr[i*k + t] with D = dist[i*k + t]. Every valid pick
// q yields the forward edge p -> q (owner p) and the reverse edge q -> p (owner q), both carrying D (P:565,
// P:914; each directed edge goes to its source's reservoir).
__global__ void hp_hist_lists_kernel(const uint32_t* __restrict__ leaf_ids, int64_t I, int k,
                                     const uint32_t* __restrict__ nbr, uint32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = leaf_ids[i];
    uint32_t nv = 0;
    for (int t = 0; t < k; ++t) {
      const uint32_t q = nbr[i * k + t];
      if (q == 0xFFFFFFFFu) break;
      ++nv;
      atomicAdd(&cnt[q], 1u);
    }
    if (nv) atomicAdd(&cnt[p], nv);
  }
}

template <typename ST>
__global__ void hp_scatter_lists_kernel(const uint32_t* __restrict__ leaf_ids, int64_t I, int k,
                                        const uint32_t* __restrict__ nbr, const float* __restrict__ dist,
                                        const ST* __restrict__ S, int m, const uint64_t* __restrict__ start,
                                        uint32_t* __restrict__ cursor, uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = leaf_ids[i];
    uint32_t nv = 0;
    for (int t = 0; t < k; ++t)
      if (nbr[i * k + t] != 0xFFFFFFFFu) ++nv;
    if (!nv) continue;
    uint64_t fwd = start[p] + atomicAdd(&cursor[p], nv);
    for (int t = 0; t < (int)nv; ++t) {
      const uint32_t q = nbr[i * k + t];
      const float D = dist[i * k + t];
      keys[fwd + t] = slot_key<ST>(S, m, p, q, D);
      const uint64_t rev = start[q] + atomicAdd(&cursor[q], 1u);
      keys[rev] = slot_key<ST>(S, m, q, p, D);
    }
  }
}

// ------------------------------------------------------------------ per-owner merge (warp per owner)
__device__ __forceinline__ void warp_bitonic_sort(uint64_t* a, int P, int lane) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t x = a[i], y = a[ixj];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncwarp();
    }
}

__device__ __forceinline__ int pow2_at_least(int x) {
  int p = 32;
  while (p < x) p <<= 1;
  return p;
}

// keys sorted by (hash, okey, id) in buf[0..total): keep the first of each hash run -> out, returns count
__device__ __forceinline__ int warp_bucket_minima(const uint64_t* buf, int total, uint64_t* out, int lane) {
  int base = 0;
  for (int i0 = 0; i0 < total; i0 += 32) {
    const int i = i0 + lane;
    bool keep = false;
    uint64_t x = 0;
    if (i < total) {
      x = buf[i];
      keep = (i == 0) || ((buf[i - 1] >> 48) != (x >> 48));
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) out[base + __popc(bal & ((1u << lane) - 1u))] = x;
    base += __popc(bal);
  }
  __syncwarp();
  return base;
}

__global__ void __launch_bounds__(128) hp_merge_kernel(int64_t n, int l_max, int cap, const uint64_t* __restrict__ start,
                                                       const uint64_t* __restrict__ keys, uint64_t* __restrict__ slots,
                                                       uint32_t* __restrict__ count) {
  extern __shared__ uint64_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* buf = sm + (size_t)warp * 2 * cap;
  uint64_t* tmp = buf + cap;
  const int64_t wstride = (int64_t)gridDim.x * 4;
  for (int64_t u = blockIdx.x * 4 + warp; u < n; u += wstride) {
    const uint64_t s0 = start[u], s1 = start[u + 1];
    if (s0 == s1) continue;
    int c = (int)count[u];
    uint64_t* res = slots + u * (int64_t)l_max;
    for (int t = lane; t < c; t += 32) buf[t] = res[t];
    uint64_t e = s0;
    while (e < s1) {
      const uint64_t rem = s1 - e, room = (uint64_t)(cap - c);
      const int chunk = (int)(rem < room ? rem : room);
      for (int t = lane; t < chunk; t += 32) buf[c + t] = keys[e + t];
      const int total = c + chunk;
      const int P = pow2_at_least(total);
      for (int t = total + lane; t < P; t += 32) buf[t] = ~0ull;
      __syncwarp();
      warp_bitonic_sort(buf, P, lane);
      int B = warp_bucket_minima(buf, total, tmp, lane);
      if (B > l_max) {
        // keep the l_max smallest by (okey, id): sort by (low 48 bits, hash), truncate, re-sort by hash
        const int PB = pow2_at_least(B);
        for (int t = lane; t < PB; t += 32) {
          const uint64_t x = t < B ? tmp[t] : ~0ull;
          tmp[t] = t < B ? ((x << 16) | (x >> 48)) : ~0ull;
        }
        __syncwarp();
        warp_bitonic_sort(tmp, PB, lane);
        const int PL = pow2_at_least(l_max);
        for (int t = lane; t < PL; t += 32) {
          const uint64_t x = tmp[t];
          tmp[t] = t < l_max ? ((x >> 16) | (x << 48)) : ~0ull;
        }
        __syncwarp();
        warp_bitonic_sort(tmp, PL, lane);
        B = l_max;
      }
      for (int t = lane; t < B; t += 32) buf[t] = tmp[t];
      __syncwarp();
      c = B;
      e += chunk;
    }
    for (int t = lane; t < c; t += 32) res[t] = buf[t];
    if (lane == 0) count[u] = (uint32_t)c;
  }
}

static int merge_cap(int l_max) {
  int cap = 512;
  while (cap < 2 * l_max) cap <<= 1;
  return cap;
}

static pipnn_status launch_merge(int64_t n, int l_max, const uint64_t* start, const uint64_t* keys, uint64_t* slots,
                                 uint32_t* count, const Ctx& c) {
  const int cap = merge_cap(l_max);
  const int smem = 4 * 2 * cap * (int)sizeof(uint64_t);
  PIPNN_CUDA(cudaFuncSetAttribute(hp_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int64_t blocks = std::min<int64_t>(ceil_div(n, 4), (int64_t)num_sms() * 16);
  hp_merge_kernel<<<(unsigned)blocks, 128, smem, c.st>>>(n, l_max, cap, start, keys, slots, count);
  PIPNN_LAUNCHED("hp_merge_kernel", c.st);
  return PIPNN_OK;
}

// cnt[n] (u32) -> start[n+1] (u64) exclusive scan; cursor zeroed.
struct Grouping {
  uint32_t* cnt;
  uint64_t* start;
  uint32_t* cursor;
  void* tmp;
  size_t tmp_bytes;
};

static Grouping take_grouping(int64_t n, Arena& ar) {
  Grouping g{};
  g.cnt = ar.take<uint32_t>(n + 1);
  g.start = ar.take<uint64_t>(n + 1);
  g.cursor = ar.take<uint32_t>(n);
  cub::DeviceScan::ExclusiveSum(nullptr, g.tmp_bytes, (const uint32_t*)nullptr, (uint64_t*)nullptr, (int)(n + 1));
  g.tmp = ar.take<uint8_t>(g.tmp_bytes);
  return g;
}

static int64_t grid_for(int64_t work) { return std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), num_sms() * 32)); }

pipnn_status hashprune_impl(int m, int l_max, int64_t n, const void* sketch, bool sk_int, uint64_t* slots,
                            uint32_t* count, const uint32_t* owner, const uint32_t* cand, const float* dist,
                            int64_t n_edges, Arena& ar, const Ctx& c) {
  Grouping g = take_grouping(n, ar);
  uint64_t* keys = ar.take<uint64_t>(std::max<int64_t>(1, n_edges));
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (hashprune)");
  if (n_edges == 0) return PIPNN_OK;
  PIPNN_CUDA(cudaMemsetAsync(g.cnt, 0, (n + 1) * sizeof(uint32_t), c.st));
  PIPNN_CUDA(cudaMemsetAsync(g.cursor, 0, n * sizeof(uint32_t), c.st));
  hp_hist_kernel<<<(unsigned)grid_for(n_edges), 256, 0, c.st>>>(owner, n_edges, g.cnt);
  PIPNN_LAUNCHED("hp_hist_kernel", c.st);
  PIPNN_CUDA(cub::DeviceScan::ExclusiveSum(g.tmp, g.tmp_bytes, g.cnt, g.start, (int)(n + 1), c.st));
  if (sk_int)
    hp_scatter_kernel<int32_t><<<(unsigned)grid_for(n_edges), 256, 0, c.st>>>(
        owner, cand, dist, n_edges, (const int32_t*)sketch, m, g.start, g.cursor, keys);
  else
    hp_scatter_kernel<float><<<(unsigned)grid_for(n_edges), 256, 0, c.st>>>(owner, cand, dist, n_edges,
                                                                             (const float*)sketch, m, g.start,
                                                                             g.cursor, keys);
  PIPNN_LAUNCHED("hp_scatter_kernel", c.st);
  return launch_merge(n, l_max, g.start, keys, slots, count, c);
}

pipnn_status hashprune_from_lists(int m, int l_max, int64_t n, const void* sketch, bool sk_int, uint64_t* slots,
                                  uint32_t* count, const uint32_t* leaf_ids, int64_t n_inst, int k,
                                  const uint32_t* nbr, const float* dist, int64_t* n_edges_dev, Arena& ar,
                                  const Ctx& c) {
  Grouping g = take_grouping(n, ar);
  uint64_t* keys = ar.take<uint64_t>(std::max<int64_t>(1, 2 * n_inst * k));
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (hashprune)");
  PIPNN_CUDA(cudaMemsetAsync(g.cnt, 0, (n + 1) * sizeof(uint32_t), c.st));
  PIPNN_CUDA(cudaMemsetAsync(g.cursor, 0, n * sizeof(uint32_t), c.st));
  if (n_inst > 0) {
    hp_hist_lists_kernel<<<(unsigned)grid_for(n_inst), 256, 0, c.st>>>(leaf_ids, n_inst, k, nbr, g.cnt);
    PIPNN_LAUNCHED("hp_hist_lists_kernel", c.st);
  }
  PIPNN_CUDA(cub::DeviceScan::ExclusiveSum(g.tmp, g.tmp_bytes, g.cnt, g.start, (int)(n + 1), c.st));
  if (n_edges_dev)
    PIPNN_CUDA(cudaMemcpyAsync(n_edges_dev, g.start + n, sizeof(int64_t), cudaMemcpyDeviceToDevice, c.st));
  if (n_inst == 0) return PIPNN_OK;
  if (sk_int)
    hp_scatter_lists_kernel<int32_t><<<(unsigned)grid_for(n_inst), 256, 0, c.st>>>(
        leaf_ids, n_inst, k, nbr, dist, (const int32_t*)sketch, m, g.start, g.cursor, keys);
  else
    hp_scatter_lists_kernel<float><<<(unsigned)grid_for(n_inst), 256, 0, c.st>>>(
        leaf_ids, n_inst, k, nbr, dist, (const float*)sketch, m, g.start, g.cursor, keys);
  PIPNN_LAUNCHED("hp_scatter_lists_kernel", c.st);
  return launch_merge(n, l_max, g.start, keys, slots, count, c);
}

}  // namespace pipnn
