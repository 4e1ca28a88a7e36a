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

#include <cstdio>
#include <cstdlib>
#include <vector>
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
  PIPNN_CUDA(kmemset(g.cnt, 0, (n + 1) * sizeof(uint32_t), c.st));
  PIPNN_CUDA(kmemset(g.cursor, 0, n * sizeof(uint32_t), c.st));
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

// ================================================================== instance-major build path (overlap-heavy builds)
// The round-1/2 leaf-local grouping kept for builds whose points sit in many leaves (the owner-major path below
// overflows every reservoir row there: fanout [10, 3] has ~30 instances per point and ~480 keys per owner):
// forward keys at the picking instance, reverse keys grouped by owner instance inside the emitting leaf's block,
// a point -> instance index, and a merge per owner over its instances' segments (a warp; a CTA table for hubs).
namespace im {
// ------------------------------------------------------------------ build path: leaf-local edge grouping
// Every edge a leaf emits has its owner inside that leaf (p -> q with owner p, q -> p with
// owner q, both members of the leaf). So the edges are grouped per leaf in shared memory, without any
// global sort: forward keys go to fwd[i*k + t] (instance i = p's position in leaf_ids), reverse keys of
// owner instance j are laid out contiguously in rev[] inside the leaf's own block [off_b*k, off_{b+1}*k)
// (the leaf emits as many reverse as forward edges), with rev_start[j] / rev_cnt[j]. The residual hashes
// (Eq. 1 via sketches) of both directions come from the leaf members' sketches staged in SMEM.
template <typename ST>
__device__ __forceinline__ ST bitcast_st(int x);
template <>
__device__ __forceinline__ int32_t bitcast_st<int32_t>(int x) { return x; }
template <>
__device__ __forceinline__ float bitcast_st<float>(int x) { return __int_as_float(x); }

template <typename ST, int NT>
__global__ void __launch_bounds__(NT) hp_emit_kernel(const int64_t* __restrict__ leaf_off, const uint32_t* __restrict__ leaf_ids,
                                                      int k, const uint16_t* __restrict__ cols,
                                                      const float* __restrict__ dist, const ST* __restrict__ S, int m,
                                                      int stage_sk, uint64_t* __restrict__ fwd, uint64_t* __restrict__ rev,
                                                      uint32_t* __restrict__ rev_start, uint32_t* __restrict__ rev_cnt,
                                                      uint2* __restrict__ rev_meta, int64_t* __restrict__ n_edges) {
  extern __shared__ __align__(16) uint8_t esm[];
  __shared__ uint32_t tot_sh;
  __shared__ uint32_t part[NT];
  const int64_t b = blockIdx.x;
  const int64_t o0 = leaf_off[b];
  const int s = (int)(leaf_off[b + 1] - o0);
  const int ms = m | 1;             // SMEM sketch row stride (odd: conflict-free row-per-thread reads)
  uint32_t* ids = (uint32_t*)esm;   // [s]
  uint32_t* rc = ids + s;           // [s] reverse in-degree, then cursor
  uint32_t* rs = rc + s;            // [s] exclusive scan of rc
  ST* sk = (ST*)(rs + s);           // [s][ms] when staged
  if (threadIdx.x == 0) tot_sh = 0;
  for (int j = threadIdx.x; j < s; j += blockDim.x) {
    const uint32_t id = leaf_ids[o0 + j];
    ids[j] = id;
    rc[j] = 0;
    if (stage_sk) {
      const ST* src = S + (int64_t)id * m;
      if ((m & 3) == 0) {  // rows of m 4-byte values are 16-B aligned: m / 4 vector loads
        int4 w[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * t < m) w[t] = __ldg(reinterpret_cast<const int4*>(src) + t);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * t < m) {
            ST* d = sk + j * ms + 4 * t;
            d[0] = bitcast_st<ST>(w[t].x);
            d[1] = bitcast_st<ST>(w[t].y);
            d[2] = bitcast_st<ST>(w[t].z);
            d[3] = bitcast_st<ST>(w[t].w);
          }
      } else {
        ST v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t < m) v[t] = src[t];  // independent loads, all in flight
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t < m) sk[j * ms + t] = v[t];
      }
    }
  }
  __syncthreads();
  const uint16_t* cl = cols + o0 * k;
  // A reverse edge q -> p (carrying D(p, q)) is dropped when q's own pick list already holds p with the same D
  // bit for bit: q's forward edge q -> p is then the identical key (same bucket h_q(p), same dist, same id),
  // and a duplicate insert is idempotent (Alg. 3). Mutual picks are common, so this halves many merges.
  const float* dl = dist + o0 * k;
  uint16_t* dup = (uint16_t*)(sk + (stage_sk ? s * ms : 0));  // [s] bit t: pick t's reverse edge is a duplicate
  auto mutual = [&](int p_local, int q_local, float Dpq) -> bool {
    int hit = -1;
    if (k == 8) {  // one 16-B load of q's picks
      const uint4 v = *reinterpret_cast<const uint4*>(cl + q_local * 8);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if ((w[j] & 0xFFFFu) == (uint32_t)p_local) hit = 2 * j;
        if ((w[j] >> 16) == (uint32_t)p_local) hit = 2 * j + 1;
      }
    } else {
      for (int t = 0; t < k; ++t)
        if (cl[q_local * k + t] == (uint16_t)p_local) hit = t;
    }
    return hit >= 0 && __float_as_uint(dl[q_local * k + hit]) == __float_as_uint(Dpq);
  };
  __shared__ uint32_t picks_sh;
  if (threadIdx.x == 0) picks_sh = 0;
  __syncthreads();
  // pass A: reverse in-degree of every member (thread per instance; the k picks of an instance in one go)
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    uint16_t q[16];
    float D[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (t < k) {
        q[t] = cl[i * k + t];
        D[t] = dl[i * k + t];
      }
    uint32_t np = 0, dm = 0;
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (t < k && q[t] != 0xFFFFu) {
        ++np;
        if (mutual(i, q[t], D[t])) dm |= 1u << t;
        else atomicAdd(&rc[q[t]], 1u);
      }
    dup[i] = (uint16_t)dm;
    if (np) atomicAdd(&picks_sh, np);
  }
  __syncthreads();
  // exclusive scan of rc (block-wide, thread-serial chunks + warp scan of chunk sums)
  {
    const int per = (s + blockDim.x - 1) / blockDim.x;
    const int j0 = threadIdx.x * per, j1 = min(s, j0 + per);
    uint32_t sum = 0;
    for (int j = j0; j < j1; ++j) sum += rc[j];
    part[threadIdx.x] = sum;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t run = 0;
      for (int w0 = 0; w0 < (int)blockDim.x; w0 += 32) {
        uint32_t v = part[w0 + threadIdx.x], x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if ((int)threadIdx.x >= o) x += y;
        }
        part[w0 + threadIdx.x] = run + x - v;
        run += __shfl_sync(0xffffffffu, x, 31);
      }
      if (threadIdx.x == 0) tot_sh = run;
    }
    __syncthreads();
    uint32_t acc = part[threadIdx.x];
    for (int j = j0; j < j1; ++j) {
      rs[j] = acc;
      acc += rc[j];
    }
  }
  __syncthreads();
  const uint64_t rbase = (uint64_t)o0 * k;
  for (int j = threadIdx.x; j < s; j += blockDim.x) {
    rev_start[o0 + j] = (uint32_t)(rbase + rs[j]);  // absolute offset into rev (I*k < 2^32, checked on the host)
    rev_cnt[o0 + j] = rc[j];
    rev_meta[o0 + j] = make_uint2((uint32_t)(rbase + rs[j]), rc[j]);  // both in one 8-B load for the merge
    rc[j] = 0;
  }
  __syncthreads();
  // pass B: both directions of every pick (thread per instance)
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    uint16_t q[16];
    float D[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (t < k) {
        q[t] = cl[i * k + t];
        D[t] = dist[(o0 + i) * k + t];
      }
    const uint32_t pid = ids[i];
    const uint32_t dm = dup[i];
    ST sp[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (t < m) sp[t] = stage_sk ? sk[i * ms + t] : S[(int64_t)pid * m + t];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      if (t >= k) break;
      uint64_t kf = ~0ull;
      if (q[t] != 0xFFFFu) {
        const int qq = q[t];
        const uint32_t qid = ids[qq];
        uint32_t hf = 0, hr = 0;
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          if (h < m) {
            const ST a = sp[h], c = stage_sk ? sk[qq * ms + h] : S[(int64_t)qid * m + h];
            hf |= (uint32_t)(c >= a) << h;  // h_p(q): bit h = [S(q)_h >= S(p)_h]
            hr |= (uint32_t)(a >= c) << h;  // h_q(p)
          }
        }
        const uint64_t dk = (uint64_t)dist_order_key(D[t]) << 32;
        kf = ((uint64_t)hf << 48) | dk | qid;
        if (!((dm >> t) & 1u)) {
          const uint32_t pos = rs[qq] + atomicAdd(&rc[qq], 1u);
          rev[rbase + pos] = ((uint64_t)hr << 48) | dk | pid;
        }
      }
      fwd[(o0 + i) * k + t] = kf;
    }
  }
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)n_edges, 2ull * picks_sh);  // streamed edges: both directions
}

// point -> instances (inverse of leaf_ids): counting sort; the order inside a point's list is irrelevant.
__global__ void hp_inv_hist_kernel(const uint32_t* __restrict__ leaf_ids, int64_t I, uint32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[leaf_ids[i]], 1u);
}
__global__ void hp_inv_fill_kernel(const uint32_t* __restrict__ leaf_ids, int64_t I, const uint64_t* __restrict__ start,
                                   uint32_t* __restrict__ cursor, uint32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = leaf_ids[i];
    inv[start[p] + atomicAdd(&cursor[p], 1u)] = (uint32_t)i;
  }
}

// Register bitonic sort of E*32 u64 keys across a warp, ascending; element i = e*32 + lane.
template <int E>
__device__ __forceinline__ void warp_sort_regs(uint64_t (&k)[E], int lane) {
#pragma unroll
  for (int kk = 2; kk <= 32 * E; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int f = e ^ (j >> 5);
          if (f > e) {
            const bool up = ((e * 32 + lane) & kk) == 0;
            const uint64_t a = k[e], c = k[f];
            const bool sw = (a > c) == up;
            k[e] = sw ? c : a;
            k[f] = sw ? a : c;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t o = __shfl_xor_sync(0xffffffffu, k[e], j);
          const bool lower = (lane & j) == 0;
          const bool up = ((e * 32 + lane) & kk) == 0;
          const uint64_t mn = o < k[e] ? o : k[e], mx = o < k[e] ? k[e] : o;
          k[e] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

// The keys streamed to owner u, addressed by a flat index: its reservoir (c keys), then for each of its
// instances the k forward keys and the rev_cnt reverse keys. Forward keys of missing picks are ~0.
struct OwnerKeys {
  const uint64_t* res;
  int c, k;
  const uint32_t* inst;  // the owner's instance ids
  int ninst;
  const uint64_t* fwd;
  const uint64_t* rev;
  const uint32_t* rev_start;
  const uint32_t* rev_cnt;
  __device__ __forceinline__ uint64_t get(int idx) const {
    if (idx < c) return res[idx];
    idx -= c;
    for (int t = 0; t < ninst; ++t) {
      const uint32_t i = inst[t];
      if (idx < k) return fwd[(int64_t)i * k + idx];
      idx -= k;
      const int rcn = (int)rev_cnt[i];
      if (idx < rcn) return rev[(uint64_t)rev_start[i] + idx];
      idx -= rcn;
    }
    return ~0ull;
  }
};

// Fast merge: one warp per owner, all of its keys (reservoir + new, <= 32*E) in registers: bitonic sort,
// keep the first key of every hash run (bucket minimum, Alg. 3's collision rule), write back sorted by hash.
// Returns false (nothing written) when more than l_max buckets survive.
template <int E>
__device__ __forceinline__ bool merge_owner_regs(int lane, int T, int c, int k, const uint64_t* res_in,
                                                 const uint32_t* sinst, const uint32_t* sbeg, const uint32_t* srs,
                                                 int ni, const uint64_t* __restrict__ fwd,
                                                 const uint64_t* __restrict__ rev, int l_max, uint64_t* res,
                                                 int& B_out) {
  uint64_t key[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    int idx = e * 32 + lane;
    uint64_t v = ~0ull;
    if (idx < T) {
      if (idx < c) {
        v = res_in[idx];
      } else {
        idx -= c;
        int j = 0;
        while (j + 1 < ni && (int)sbeg[j + 1] <= idx) ++j;  // segment j: k forward then rev keys of instance j
        const int o = idx - (int)sbeg[j];
        const uint32_t i = sinst[j];
        v = o < k ? fwd[(int64_t)i * k + o] : rev[(uint64_t)srs[j] + (o - k)];
      }
    }
    key[e] = v;
  }
  warp_sort_regs<E>(key, lane);
  bool keep[E];
  int B = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint64_t up = __shfl_up_sync(0xffffffffu, key[e], 1);
    const uint64_t last = __shfl_sync(0xffffffffu, key[e > 0 ? e - 1 : 0], 31);  // element 32e - 1
    const uint64_t prev = lane > 0 ? up : last;
    const bool first = (e == 0 && lane == 0) || ((prev >> 48) != (key[e] >> 48));
    keep[e] = key[e] != ~0ull && first;
    B += __popc(__ballot_sync(0xffffffffu, keep[e]));
  }
  if (B > l_max) return false;
  int base = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t bal = __ballot_sync(0xffffffffu, keep[e]);
    if (keep[e]) res[base + __popc(bal & ((1u << lane) - 1u))] = key[e];
    base += __popc(bal);
  }
  B_out = B;
  return true;
}

// One warp per owner: the owner's instance table (instance id, first flat index of its keys) in SMEM, then
// the register merge with 32 (common: 2 k f keys), 64 or 128 slots. Owners with more keys, more instances than
// lanes, or more than l_max buckets go to the generic merge.
__global__ void __launch_bounds__(256) hp_merge_inst_kernel(int64_t n, int l_max, int k, const uint64_t* __restrict__ inv_start,
                                                            const uint32_t* __restrict__ inv, const uint64_t* __restrict__ fwd,
                                                            const uint64_t* __restrict__ rev,
                                                            const uint2* __restrict__ rev_meta,
                                                            uint64_t* __restrict__ slots, uint32_t* __restrict__ count,
                                                            uint32_t* __restrict__ defer, uint32_t* __restrict__ defer_n) {
  __shared__ uint32_t s_inst[8][32], s_beg[8][32], s_rs[8][32];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = wid; u < n; u += nw) {
    const uint64_t i0 = inv_start[u];
    const int ni = (int)(inv_start[u + 1] - i0);
    if (ni == 0) continue;
    if (ni > 32) {
      if (lane == 0) defer[atomicAdd(defer_n, 1u)] = (uint32_t)u;
      continue;
    }
    const int c = (int)count[u];
    int sz = 0;
    uint32_t inst = 0, rs0 = 0;
    if (lane < ni) {
      inst = inv[i0 + lane];
      const uint2 mt = rev_meta[inst];  // (rev start, rev count) in one load
      rs0 = mt.x;
      sz = k + (int)mt.y;
    }
    int x = sz;  // inclusive prefix over the instance segments
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const int T = c + __shfl_sync(0xffffffffu, x, 31);
    if (T > 128) {
      if (lane == 0) defer[atomicAdd(defer_n, 1u)] = (uint32_t)u;
      continue;
    }
    __syncwarp();
    s_inst[wl][lane] = inst;
    s_beg[wl][lane] = (uint32_t)(x - sz);
    s_rs[wl][lane] = rs0;
    __syncwarp();
    uint64_t* res = slots + u * (int64_t)l_max;
    int B = 0;
    bool ok;
    if (T <= 32) ok = merge_owner_regs<1>(lane, T, c, k, res, s_inst[wl], s_beg[wl], s_rs[wl], ni, fwd, rev, l_max, res, B);
    else if (T <= 64) ok = merge_owner_regs<2>(lane, T, c, k, res, s_inst[wl], s_beg[wl], s_rs[wl], ni, fwd, rev, l_max, res, B);
    else ok = merge_owner_regs<4>(lane, T, c, k, res, s_inst[wl], s_beg[wl], s_rs[wl], ni, fwd, rev, l_max, res, B);
    if (!ok) {
      if (lane == 0) defer[atomicAdd(defer_n, 1u)] = (uint32_t)u;
      continue;
    }
    if (lane == 0) count[u] = (uint32_t)B;
  }
}

// Block (256 threads) sum and exclusive scan of one int per thread; s8 = 8 ints of SMEM.
__device__ __forceinline__ int block256_sum(int x, int* s8) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (lane == 0) s8[w] = x;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += s8[i];
  __syncthreads();
  return t;
}
__device__ __forceinline__ int block256_excl(int x, int* s8) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s8[w] = inc;
  __syncthreads();
  int off = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) off += i < w ? s8[i] : 0;
  __syncthreads();
  return off + inc - x;
}

// Table merge for the deferred owners (hubs, evictions; m <= 12): one CTA per owner, a 2^m-entry SMEM table
// indexed by the hash. Every key (reservoir + new) goes in with a 64-bit atomicMin on its bucket — the bucket
// minimum of Alg. 3's collision rule, in any order. The occupied buckets, read back in table order, are
// sorted by hash; when more than l_max survive, the l_max-th smallest 48-bit (dist16 | id32) value is found by
// an MSB-first bisection with block-wide counts (values are distinct: one bucket per id) and only the entries
// at or below it are kept (the eviction rule's end state).
__global__ void __launch_bounds__(256) hp_merge_table_kernel(int m, int l_max, int k, const uint64_t* __restrict__ inv_start,
                                                             const uint32_t* __restrict__ inv,
                                                             const uint64_t* __restrict__ fwd,
                                                             const uint64_t* __restrict__ rev,
                                                             const uint32_t* __restrict__ rev_start,
                                                             const uint32_t* __restrict__ rev_cnt,
                                                             uint64_t* __restrict__ slots, uint32_t* __restrict__ count,
                                                             const uint32_t* __restrict__ list,
                                                             const uint32_t* __restrict__ list_n) {
  extern __shared__ uint64_t tbl[];  // [2^m]
  __shared__ int s8[8];
  __shared__ uint32_t s_hist[256];
  __shared__ uint32_t s_sel;
  __shared__ uint32_t s_inst[256], s_rs[256];
  __shared__ int s_off[257];
  const int NB = 1 << m, tid = threadIdx.x;
  const int64_t nl = *list_n;
  constexpr uint64_t kLow48 = 0xFFFFFFFFFFFFull;
  for (int64_t it = blockIdx.x; it < nl; it += gridDim.x) {
    const int64_t u = list[it];
    uint64_t* res = slots + u * (int64_t)l_max;
    const int c = (int)count[u];
    const uint64_t i0 = inv_start[u], i1 = inv_start[u + 1];
    // table size: 2^m slots indexed by the hash, or — for an owner whose keys all fit one staging round — the
    // power of two >= 2 x its key count (>= 256), probed linearly from hash & (S - 1): fewer slots to clear
    // and read back. (The build's reservoirs are read as sets; only the hash-indexed table keeps hash order.)
    int S = NB;
    bool staged = false;
    auto stage = [&](uint64_t q0) -> int {  // instances q0.. (<= 256): ids, reverse starts, key offsets
      const int ni = (int)(i1 - q0 < 256 ? i1 - q0 : 256);
      int sz = 0;
      if (tid < ni) {
        const uint32_t i = inv[q0 + tid];
        s_inst[tid] = i;
        s_rs[tid] = rev_start[i];
        sz = k + (int)rev_cnt[i];
      }
      const int off = block256_excl(sz, s8);  // (its barriers also publish s_inst / s_rs)
      if (tid < ni) s_off[tid] = off;
      if (tid == ni - 1) s_off[ni] = off + sz;
      __syncthreads();
      return ni;
    };
    __syncthreads();  // the previous owner's table and staging arrays are no longer read
    int ni0 = 0;
    if (i1 - i0 <= 256) {
      ni0 = i1 > i0 ? stage(i0) : 0;
      staged = true;
      const int T = c + (ni0 ? s_off[ni0] : 0);
      while (S > 256 && S >= 4 * T) S >>= 1;
    }
    const bool direct = S == NB;
    for (int t = tid; t < S; t += 256) tbl[t] = ~0ull;
    __syncthreads();
    auto put = [&](uint64_t key) {
      const uint32_t h = (uint32_t)(key >> 48);
      if (direct) {
        atomicMin((unsigned long long*)&tbl[h], (unsigned long long)key);
        return;
      }
      uint32_t sl = h & (uint32_t)(S - 1);
      while (true) {
        unsigned long long cur = *(volatile unsigned long long*)&tbl[sl];
        if (cur == ~0ull) {
          cur = atomicCAS((unsigned long long*)&tbl[sl], ~0ull, (unsigned long long)key);
          if (cur == ~0ull) return;
        }
        if ((uint32_t)(cur >> 48) == h) {
          atomicMin((unsigned long long*)&tbl[sl], (unsigned long long)key);
          return;
        }
        sl = (sl + 1) & (uint32_t)(S - 1);
      }
    };
    for (int t = tid; t < c; t += 256) put(res[t]);
    // the owner's instances, 256 at a time, their keys as one flat index space (a thread per key, segment by
    // binary search)
    for (uint64_t q0 = i0; q0 < i1; q0 += 256) {
      const int ni = staged ? ni0 : stage(q0);
      staged = false;
      const int tot = s_off[ni];
      for (int f = tid; f < tot; f += 256) {
        int lo = 0, hi = ni - 1;  // the segment holding flat index f: largest t with s_off[t] <= f
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_off[mid] <= f) lo = mid;
          else hi = mid - 1;
        }
        const int j = f - s_off[lo];
        const uint32_t i = s_inst[lo];
        const uint64_t key = j < k ? fwd[(int64_t)i * k + j] : rev[(uint64_t)s_rs[lo] + (j - k)];
        if (key != ~0ull) put(key);
      }
      __syncthreads();
    }
    uint64_t v[16];
    int cnt = 0;
    const int per = (S + 255) / 256;  // table entries per thread (<= 16; contiguous chunk)
    const int b0 = tid * per;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      v[e] = (e < per && b0 + e < S) ? tbl[b0 + e] : ~0ull;
      cnt += v[e] != ~0ull ? 1 : 0;
    }
    const int total = block256_sum(cnt, s8);
    uint64_t thr48 = kLow48;
    if (total > l_max) {
      // radix select, 8-bit digits MSB first: the bucket of the need-th smallest among the values that share
      // the prefix decided so far (6 rounds of a 256-bin SMEM histogram + scan)
      uint32_t* hist = s_hist;
      uint64_t prefix = 0;
      int need = l_max;
      for (int sh = 40; sh >= 0; sh -= 8) {
        hist[tid] = 0u;
        __syncthreads();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const uint64_t x = v[e] & kLow48;
          if (v[e] != ~0ull && (sh == 40 || (x >> (sh + 8)) == (prefix >> (sh + 8))))
            atomicAdd(&hist[(x >> sh) & 0xFF], 1u);
        }
        __syncthreads();
        const int hb = (int)hist[tid];
        const int below = block256_excl(hb, s8);  // values with this prefix and a smaller digit
        if (below < need && need <= below + hb) s_sel = (uint32_t)((tid << 16) | (uint32_t)(need - below));
        __syncthreads();
        const uint32_t sel = s_sel;
        prefix |= (uint64_t)(sel >> 16) << sh;
        need = (int)(sel & 0xFFFFu);
      }
      thr48 = prefix;
    }
    int kc = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) kc += (v[e] != ~0ull && (v[e] & kLow48) <= thr48) ? 1 : 0;
    int o = block256_excl(kc, s8);
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (v[e] != ~0ull && (v[e] & kLow48) <= thr48) res[o++] = v[e];
    if (tid == 255) count[u] = (uint32_t)o;
  }
}

// Generic merge for the deferred owners: the chunked SMEM algorithm of hp_merge_kernel over OwnerKeys.
__global__ void __launch_bounds__(128) hp_merge_inst_generic_kernel(int l_max, int cap, int k,
                                                                    const uint64_t* __restrict__ inv_start,
                                                                    const uint32_t* __restrict__ inv,
                                                                    const uint64_t* __restrict__ fwd,
                                                                    const uint64_t* __restrict__ rev,
                                                                    const uint32_t* __restrict__ rev_start,
                                                                    const uint32_t* __restrict__ rev_cnt,
                                                                    uint64_t* __restrict__ slots, uint32_t* __restrict__ count,
                                                                    const uint32_t* __restrict__ list,
                                                                    const uint32_t* __restrict__ list_n) {
  extern __shared__ uint64_t gm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* buf = gm + (size_t)warp * 2 * cap;
  uint64_t* tmp = buf + cap;
  const int64_t nl = *list_n;
  for (int64_t it = blockIdx.x * 4 + warp; it < nl; it += (int64_t)gridDim.x * 4) {
    const int64_t u = list[it];
    const uint64_t i0 = inv_start[u];
    const int ni = (int)(inv_start[u + 1] - i0);
    uint64_t* res = slots + u * (int64_t)l_max;
    int c = (int)count[u];
    int total_new = 0;
    for (int t = lane; t < ni; t += 32) total_new += k + (int)rev_cnt[inv[i0 + t]];
#pragma unroll
    for (int o = 16; o; o >>= 1) total_new += __shfl_xor_sync(0xffffffffu, total_new, o);
    OwnerKeys ok{res, 0, k, inv + i0, ni, fwd, rev, rev_start, rev_cnt};
    for (int t = lane; t < c; t += 32) buf[t] = res[t];
    int e = 0;
    while (e < total_new) {
      const int chunk = min(total_new - e, cap - c);
      for (int t = lane; t < chunk; t += 32) buf[c + t] = ok.get(e + t);
      const int total = c + chunk;
      const int P = pow2_at_least(total);
      for (int t = total + lane; t < P; t += 32) buf[t] = ~0ull;
      __syncwarp();
      warp_bitonic_sort(buf, P, lane);
      // drop ~0 keys (missing picks) before taking bucket minima
      int tv = total;
      while (tv > 0 && buf[tv - 1] == ~0ull) --tv;
      int B = warp_bucket_minima(buf, tv, tmp, lane);
      if (B > l_max) {
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

pipnn_status from_leaves(int m, int l_max, int64_t n, const void* sketch, bool sk_int, uint64_t* slots,
                                   uint32_t* count, const int64_t* leaf_off, int64_t n_leaves, const uint32_t* leaf_ids,
                                   int64_t n_inst, int k, const uint16_t* cols, const float* dist, int max_leaf,
                                   int64_t* n_edges_dev, Arena& ar, const Ctx& c) {
  const int64_t P = std::max<int64_t>(1, n_inst * k);
  uint64_t* fwd = ar.take<uint64_t>(P);
  uint64_t* rev = ar.take<uint64_t>(P);
  uint32_t* rev_start = ar.take<uint32_t>(std::max<int64_t>(1, n_inst));
  uint32_t* rev_cnt = ar.take<uint32_t>(std::max<int64_t>(1, n_inst));
  uint2* rev_meta = ar.take<uint2>(std::max<int64_t>(1, n_inst));
  Grouping g = take_grouping(n, ar);  // point -> instances
  uint32_t* inv = ar.take<uint32_t>(std::max<int64_t>(1, n_inst));
  uint32_t* defer = ar.take<uint32_t>(n);
  uint32_t* defer_n = ar.take<uint32_t>(1);
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (hashprune)");
  if (P >= ((int64_t)1 << 32)) return fail(PIPNN_EUNSUPPORTED, "hashprune: more than 2^32 picks in one wave");
  PIPNN_CUDA(kmemset(n_edges_dev, 0, sizeof(int64_t), c.st));
  if (n_inst == 0 || n_leaves == 0) return PIPNN_OK;
  // (1) leaf-local emission of both edge directions; members' sketches staged in SMEM (C5's 2048-member leaves:
  // 106 KB of sketches, so a CTA of 1024 threads per leaf there instead of 256)
  max_leaf = std::max(1, std::min(max_leaf, 4096));
  const size_t sk_bytes = (size_t)max_leaf * (m | 1) * 4;
  const int stage_sk = (size_t)max_leaf * 14 + sk_bytes <= 200 * 1024 ? 1 : 0;
  const int smem = (int)((size_t)max_leaf * 14 + (stage_sk ? sk_bytes : 0));
  const bool big = max_leaf > 1024;
#define HP_EMIT(ST, NTH)                                                                                          \
  do {                                                                                                            \
    PIPNN_CUDA(cudaFuncSetAttribute(hp_emit_kernel<ST, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    hp_emit_kernel<ST, NTH><<<(unsigned)n_leaves, NTH, smem, c.st>>>(leaf_off, leaf_ids, k, cols, dist,           \
                                                                   (const ST*)sketch, m, stage_sk, fwd, rev,       \
                                                                   rev_start, rev_cnt, rev_meta, n_edges_dev);    \
  } while (0)
  if (sk_int) {
    if (big) HP_EMIT(int32_t, 1024); else HP_EMIT(int32_t, 256);
  } else {
    if (big) HP_EMIT(float, 1024); else HP_EMIT(float, 256);
  }
#undef HP_EMIT
  PIPNN_LAUNCHED("hp_emit_kernel", c.st);
  // (2) point -> instances
  PIPNN_CUDA(kmemset(g.cnt, 0, (n + 1) * sizeof(uint32_t), c.st));
  PIPNN_CUDA(kmemset(g.cursor, 0, n * sizeof(uint32_t), c.st));
  hp_inv_hist_kernel<<<(unsigned)grid_for(n_inst), 256, 0, c.st>>>(leaf_ids, n_inst, g.cnt);
  PIPNN_LAUNCHED("hp_inv_hist_kernel", c.st);
  PIPNN_CUDA(cub::DeviceScan::ExclusiveSum(g.tmp, g.tmp_bytes, g.cnt, g.start, (int)(n + 1), c.st));
  hp_inv_fill_kernel<<<(unsigned)grid_for(n_inst), 256, 0, c.st>>>(leaf_ids, n_inst, g.start, g.cursor, inv);
  PIPNN_LAUNCHED("hp_inv_fill_kernel", c.st);
  // (3) merge per owner (register path), deferred owners through the generic chunked path
  PIPNN_CUDA(kmemset(defer_n, 0, sizeof(uint32_t), c.st));
  const int64_t blocks = std::min<int64_t>(ceil_div(n, 8), (int64_t)num_sms() * 32);
  // (measured: the sort-free set merge below, match_any / SMEM-table buckets, was slower than the register
  // bitonic merge: C5 44.0 vs 31.9 ms, C2 0.90 vs 0.55 ms — the merge is bound by its dependent gathers)
  hp_merge_inst_kernel<<<(unsigned)blocks, 256, 0, c.st>>>(n, l_max, k, g.start, inv, fwd, rev, rev_meta, slots,
                                                               count, defer, defer_n);
  PIPNN_LAUNCHED("hp_merge_inst_kernel", c.st);
  if (m <= 12) {
    const int tsm = (int)((size_t)8 << m);
    PIPNN_CUDA(cudaFuncSetAttribute(hp_merge_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tsm));
    hp_merge_table_kernel<<<(unsigned)(num_sms() * 6), 256, tsm, c.st>>>(m, l_max, k, g.start, inv, fwd, rev, rev_start,
                                                                          rev_cnt, slots, count, defer, defer_n);
    PIPNN_LAUNCHED("hp_merge_table_kernel", c.st);
  } else {
    const int cap = merge_cap(l_max);
    const int gsm = 4 * 2 * cap * (int)sizeof(uint64_t);
    PIPNN_CUDA(cudaFuncSetAttribute(hp_merge_inst_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gsm));
    hp_merge_inst_generic_kernel<<<(unsigned)(num_sms() * 4), 128, gsm, c.st>>>(l_max, cap, k, g.start, inv, fwd, rev,
                                                                                rev_start, rev_cnt, slots, count, defer,
                                                                                defer_n);
    PIPNN_LAUNCHED("hp_merge_inst_generic_kernel", c.st);
  }
  static const bool dbg_timing = [] {
    const char* e = std::getenv("PIPNN_DEBUG_TIMING");
    return e && e[0] == '1';
  }();
  if (dbg_timing) {
    uint32_t hd = 0;
    PIPNN_CUDA(cudaMemcpyAsync(&hd, defer_n, sizeof(hd), cudaMemcpyDeviceToHost, c.st));
    PIPNN_CUDA(cudaStreamSynchronize(c.st));
    std::vector<uint32_t> dl(hd);
    std::vector<uint64_t> st(n + 1);
    if (hd) PIPNN_CUDA(cudaMemcpy(dl.data(), defer, hd * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    PIPNN_CUDA(cudaMemcpy(st.data(), g.start, (n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> rc(n_inst), ivv(n_inst);
    PIPNN_CUDA(cudaMemcpy(rc.data(), rev_cnt, n_inst * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    PIPNN_CUDA(cudaMemcpy(ivv.data(), inv, n_inst * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    int64_t tsum = 0, tmax = 0;
    for (uint32_t u : dl) {
      int64_t T = 0;
      for (uint64_t j = st[u]; j < st[u + 1]; ++j) T += k + rc[ivv[j]];
      tsum += T;
      tmax = std::max(tmax, T);
    }
    std::fprintf(stderr, "[pipnn] hashprune: %u owners deferred to the generic merge, keys mean %.0f max %lld\n", hd,
                 hd ? (double)tsum / hd : 0.0, (long long)tmax);
  }
  return PIPNN_OK;
}

}  // namespace im

// ------------------------------------------------------------------ build path: owner-major emission
// Every edge a leaf emits has its owner inside that leaf (p -> q with owner p, q -> p with owner
// q, both members of the leaf). Each owner instance (p in leaf b) counts its keys — its valid picks plus the
// reverse edges the other members send it — and claims a run of that many positions in p's own reservoir row
// slots[p, .] with one atomicAdd on count[p] (count starts at 0); the CTA then writes the keys there. A
// point's keys from all of its leaves so end up contiguous in its row, and the merge reads one contiguous row
// per owner (no point -> instance index, no scattered per-instance segments). An instance whose run would
// pass l_max writes its keys to an overflow buffer instead and links a record (owner, base, key offset, count)
// into its owner's list; owners whose count exceeds l_max are merged by the deferred kernels. The merge
// computes the history-independent closed form of Alg. 3, so neither the claim order
// nor the order inside a row matters; inside the build a reservoir is a set (the final prune orders it).
template <typename ST>
__device__ __forceinline__ ST bitcast_st(int x);
template <>
__device__ __forceinline__ int32_t bitcast_st<int32_t>(int x) { return x; }
template <>
__device__ __forceinline__ float bitcast_st<float>(int x) { return __int_as_float(x); }

struct HpOverflow {
  uint64_t* keys;              // overflow keys
  unsigned long long* keys_n;  // keys used
  unsigned long long keys_cap;
  uint4* rec;                  // (owner, base, key offset, key count) of every overflowing instance
  uint32_t* rec_next;          // next record of the same owner (~0 ends)
  uint32_t* rec_n;
  uint32_t rec_cap;
  uint32_t* head;              // [n] first record of the owner (~0: none)
};

constexpr uint64_t kDstNone = ~0ull;
constexpr uint64_t kDstOvf = 1ull << 63;

// SMEM bytes per leaf member of hp_emit_kernel (without the staged sketches): destination (8), id (4), reverse
// count / cursor (4), duplicate mask (2), valid picks (1).
constexpr int kEmitBytesPerMember = 19;

template <typename ST, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) hp_emit_kernel(const int64_t* __restrict__ leaf_off, const uint32_t* __restrict__ leaf_ids,
                                                      int k, const uint16_t* __restrict__ cols,
                                                      const float* __restrict__ dist, const ST* __restrict__ S, int m,
                                                      int stage_sk, int l_max, uint64_t* __restrict__ slots,
                                                      uint32_t* __restrict__ count, HpOverflow ov,
                                                      int64_t* __restrict__ n_edges, int* __restrict__ err,
                                                      int s_lo, int s_hi) {
  extern __shared__ __align__(16) uint8_t esm[];
  __shared__ uint32_t picks_sh;
  const int64_t b = blockIdx.x;
  const int64_t o0 = leaf_off[b];
  const int s = (int)(leaf_off[b + 1] - o0);
  if (s <= s_lo || s > s_hi) return;  // size class of this launch: leaves of s_lo < s <= s_hi members
  const int ms = m | 1;                          // SMEM sketch row stride (odd: conflict-free row-per-thread reads)
  uint64_t* dst = (uint64_t*)esm;                // [s] where the instance's keys go (slots index | kDstOvf + offset)
  uint32_t* ids = (uint32_t*)(dst + s);          // [s]
  uint32_t* rc = ids + s;                        // [s] reverse in-degree, then cursor
  ST* sk = (ST*)(rc + s);                        // [s][ms] when staged
  uint16_t* dup = (uint16_t*)(sk + (stage_sk ? s * ms : 0));  // [s] bit t: pick t's reverse edge is a duplicate
  uint8_t* nv = (uint8_t*)(dup + s);             // [s] valid picks of the instance
  if (threadIdx.x == 0) picks_sh = 0;
  for (int j = threadIdx.x; j < s; j += blockDim.x) {
    const uint32_t id = leaf_ids[o0 + j];
    ids[j] = id;
    rc[j] = 0;
    if (stage_sk) {
      const ST* src = S + (int64_t)id * m;
      if ((m & 3) == 0) {  // rows of m 4-byte values are 16-B aligned: m / 4 vector loads
        int4 w[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * t < m) w[t] = __ldg(reinterpret_cast<const int4*>(src) + t);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * t < m) {
            ST* d = sk + j * ms + 4 * t;
            d[0] = bitcast_st<ST>(w[t].x);
            d[1] = bitcast_st<ST>(w[t].y);
            d[2] = bitcast_st<ST>(w[t].z);
            d[3] = bitcast_st<ST>(w[t].w);
          }
      } else {
        ST v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t < m) v[t] = src[t];  // independent loads, all in flight
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t < m) sk[j * ms + t] = v[t];
      }
    }
  }
  __syncthreads();
  const uint16_t* cl = cols + o0 * k;
  const float* dl = dist + o0 * k;
  // A reverse edge q -> p (carrying D(p, q)) is dropped when q's own pick list already holds p with the same D
  // bit for bit: q's forward edge q -> p is then the identical key (same bucket h_q(p), same dist, same id),
  // and a duplicate insert is idempotent (Alg. 3). Mutual picks are common, so this shortens many rows.
  auto mutual = [&](int p_local, int q_local, float Dpq) -> bool {
    int hit = -1;
    if (k == 8) {  // one 16-B load of q's picks
      const uint4 v = *reinterpret_cast<const uint4*>(cl + q_local * 8);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if ((w[j] & 0xFFFFu) == (uint32_t)p_local) hit = 2 * j;
        if ((w[j] >> 16) == (uint32_t)p_local) hit = 2 * j + 1;
      }
    } else {
      for (int t = 0; t < k; ++t)
        if (cl[q_local * k + t] == (uint16_t)p_local) hit = t;
    }
    return hit >= 0 && __float_as_uint(dl[q_local * k + hit]) == __float_as_uint(Dpq);
  };
  // pass A: valid picks and reverse in-degree of every member (thread per instance)
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    uint16_t q[16];
    float D[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (t < k) {
        q[t] = cl[i * k + t];
        D[t] = dl[i * k + t];
      }
    uint32_t np = 0, dm = 0;
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (t < k && q[t] != 0xFFFFu) {
        ++np;
        if (mutual(i, q[t], D[t])) dm |= 1u << t;
        else atomicAdd(&rc[q[t]], 1u);
      }
    dup[i] = (uint16_t)dm;
    nv[i] = (uint8_t)np;
    if (np) atomicAdd(&picks_sh, np);
  }
  __syncthreads();
  // claim: each instance's run of keys in its owner's row (or in the overflow buffer)
  for (int j = threadIdx.x; j < s; j += blockDim.x) {
    const uint32_t tot = nv[j] + rc[j];
    rc[j] = 0;
    uint64_t d = kDstNone;
    if (tot) {
      const uint32_t p = ids[j];
      const uint32_t base = atomicAdd(&count[p], tot);
      if ((uint64_t)base + tot <= (uint64_t)l_max) {
        d = (uint64_t)p * (uint64_t)l_max + base;
      } else {
        const unsigned long long off = atomicAdd(ov.keys_n, (unsigned long long)tot);
        const uint32_t r = atomicAdd(ov.rec_n, 1u);
        if (off + tot > ov.keys_cap || r >= ov.rec_cap) {
          atomicCAS(err, 0, (int)DERR_CAPACITY);
        } else {
          ov.rec[r] = make_uint4(p, base, (uint32_t)off, tot);
          ov.rec_next[r] = atomicExch(&ov.head[p], r);
          d = kDstOvf | off;
        }
      }
    }
    dst[j] = d;
  }
  __syncthreads();
  auto put = [&](uint64_t d, uint32_t idx, uint64_t key) {
    if (d == kDstNone) return;
    if (d & kDstOvf) ov.keys[(d & ~kDstOvf) + idx] = key;
    else slots[d + idx] = key;
  };
  // pass B: both directions of every pick (thread per instance): forward keys first in the owner's run, the
  // reverse keys after them (cursor per owner member)
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    uint16_t q[16];
    float D[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (t < k) {
        q[t] = cl[i * k + t];
        D[t] = dl[i * k + t];
      }
    const uint32_t pid = ids[i];
    const uint32_t dm = dup[i];
    const uint64_t di = dst[i];
    ST sp[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (t < m) sp[t] = stage_sk ? sk[i * ms + t] : S[(int64_t)pid * m + t];
    uint32_t f = 0;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      if (t >= k) break;
      if (q[t] == 0xFFFFu) continue;
      const int qq = q[t];
      const uint32_t qid = ids[qq];
      uint32_t hf = 0, hr = 0;
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        if (h < m) {
          const ST a = sp[h], c = stage_sk ? sk[qq * ms + h] : S[(int64_t)qid * m + h];
          hf |= (uint32_t)(c >= a) << h;  // h_p(q): bit h = [S(q)_h >= S(p)_h]
          hr |= (uint32_t)(a >= c) << h;  // h_q(p)
        }
      }
      const uint64_t dk = (uint64_t)dist_order_key(D[t]) << 32;
      put(di, f++, ((uint64_t)hf << 48) | dk | qid);
      if (!((dm >> t) & 1u)) {
        const uint32_t pos = (uint32_t)nv[qq] + atomicAdd(&rc[qq], 1u);
        put(dst[qq], pos, ((uint64_t)hr << 48) | dk | pid);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)n_edges, 2ull * picks_sh);  // streamed edges: both directions
}

// Register bitonic sort of E*32 u64 keys across a warp, ascending; element i = e*32 + lane.
template <int E>
__device__ __forceinline__ void warp_sort_regs(uint64_t (&k)[E], int lane) {
#pragma unroll
  for (int kk = 2; kk <= 32 * E; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int f = e ^ (j >> 5);
          if (f > e) {
            const bool up = ((e * 32 + lane) & kk) == 0;
            const uint64_t a = k[e], c = k[f];
            const bool sw = (a > c) == up;
            k[e] = sw ? c : a;
            k[f] = sw ? a : c;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t o = __shfl_xor_sync(0xffffffffu, k[e], j);
          const bool lower = (lane & j) == 0;
          const bool up = ((e * 32 + lane) & kk) == 0;
          const uint64_t mn = o < k[e] ? o : k[e], mx = o < k[e] ? k[e] : o;
          k[e] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

// The same network with the stage loops kept rolled (only the per-register work unrolled): a fraction of the code
// size, for kernels whose instruction fetch would otherwise thrash (hp_defer_sort_kernel: 84% "no instruction"
// stalls with the fully unrolled E = 4/8/16 networks).
template <int E>
__device__ __forceinline__ void warp_sort_regs_rolled(uint64_t (&k)[E], int lane) {
#pragma unroll 1
  for (int kk = 2; kk <= 32 * E; kk <<= 1) {
#pragma unroll 1
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int js = j >> 5;  // register distance (1, 2, 4, 8)
#pragma unroll
        for (int e = 0; e < E; ++e) {
          // partner e ^ js, handled by the lower of the two
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            if ((1 << b) < E && js == (1 << b) && !(e & (1 << b))) {
              const int f = e | (1 << b);
              const bool up = ((e * 32 + lane) & kk) == 0;
              const uint64_t a = k[e], c = k[f];
              const bool sw = (a > c) == up;
              k[e] = sw ? c : a;
              k[f] = sw ? a : c;
            }
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t o = __shfl_xor_sync(0xffffffffu, k[e], j);
          const bool lower = (lane & j) == 0;
          const bool up = ((e * 32 + lane) & kk) == 0;
          const uint64_t mn = o < k[e] ? o : k[e], mx = o < k[e] ? k[e] : o;
          k[e] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

// The keys streamed to owner u, addressed by a flat index: its reservoir (c keys), then for each of its

// Merge of a row of c <= 32 keys (one per lane, lane < c): keep the minimum of every hash bucket (Alg. 3's
// collision rule; identical keys — the same edge from two leaves — keep one), compacted to the row's front.
// Returns the number kept (<= c <= l_max: no eviction).
__device__ __forceinline__ int merge_row32(uint64_t* res, int c, int lane, uint64_t key) {
  const bool valid = lane < c;
  const uint32_t mv = valid ? (uint32_t)(key >> 48) : (0x10000u + (uint32_t)lane);
  const uint32_t grp = __match_any_sync(0xffffffffu, mv);
  uint32_t rem = grp & ~(1u << lane);
  const int R = __reduce_max_sync(0xffffffffu, (uint32_t)__popc(rem));
  bool keep = valid;
  for (int r = 0; r < R; ++r) {  // the r-th other key of the bucket (uniform trip count)
    const int j = rem ? __ffs(rem) - 1 : lane;
    rem &= rem - 1;
    const uint64_t kj = __shfl_sync(0xffffffffu, key, j);
    if (j != lane && (kj < key || (kj == key && j < lane))) keep = false;
  }
  const uint32_t bal = __ballot_sync(0xffffffffu, keep);
  if (keep) res[__popc(bal & ((1u << lane) - 1u))] = key;
  return __popc(bal);
}

// The same for 32 < c <= 32 E keys: register bitonic sort, the first key of every hash run.
template <int E>
__device__ __forceinline__ int merge_row_regs(uint64_t* res, int c, int lane) {
  uint64_t key[E];
#pragma unroll
  for (int e = 0; e < E; ++e) key[e] = e * 32 + lane < c ? res[e * 32 + lane] : ~0ull;
  warp_sort_regs<E>(key, lane);
  bool keep[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint64_t up = __shfl_up_sync(0xffffffffu, key[e], 1);
    const uint64_t last = __shfl_sync(0xffffffffu, key[e > 0 ? e - 1 : 0], 31);  // element 32e - 1
    const uint64_t prev = lane > 0 ? up : last;
    const bool first = (e == 0 && lane == 0) || ((prev >> 48) != (key[e] >> 48));
    keep[e] = key[e] != ~0ull && first;
  }
  int base = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t bal = __ballot_sync(0xffffffffu, keep[e]);
    if (keep[e]) res[base + __popc(bal & ((1u << lane) - 1u))] = key[e];
    base += __popc(bal);
  }
  return base;
}

// Row merge: a warp per 32 consecutive owners (their counts in one coalesced load), each owner's row merged
// in place. Owners with more than min(l_max, 128) keys go to the deferred list (their count stays raw).
__global__ void __launch_bounds__(256) hp_merge_rows_kernel(int64_t n, int l_max, uint64_t* __restrict__ slots,
                                                            uint32_t* __restrict__ count, uint32_t* __restrict__ defer,
                                                            uint32_t* __restrict__ defer_n) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int cmax = l_max < 128 ? l_max : 128;
  for (int64_t u0 = wid * 32; u0 < n; u0 += nw * 32) {
    const int64_t u = u0 + lane;
    const uint32_t cl = u < n ? count[u] : 0u;
    uint32_t outc = cl;
    const uint32_t big = __ballot_sync(0xffffffffu, cl > (uint32_t)cmax);
    if (big & (1u << lane)) defer[atomicAdd(defer_n, 1u)] = (uint32_t)u;
    uint32_t todo = __ballot_sync(0xffffffffu, cl > 0u) & ~big;
    // the next owner's row (one key per lane, rows of <= 32 keys) is loaded while the current one merges
    // (C5 row merge 14.8 -> 12.9 ms; up to 4 keys per lane for rows of <= 128: 13.1 ms)
    auto first_keys = [&](int j) -> uint64_t {
      if (j < 0) return ~0ull;
      const int c = (int)__shfl_sync(0xffffffffu, cl, j);
      return (c <= 32 && lane < c) ? slots[(u0 + j) * (int64_t)l_max + lane] : ~0ull;
    };
    int jn = todo ? __ffs(todo) - 1 : -1;
    uint64_t kn = first_keys(jn);
    while (todo) {
      const int j = jn;
      const uint64_t key = kn;
      todo &= todo - 1;
      jn = todo ? __ffs(todo) - 1 : -1;
      kn = first_keys(jn);
      const int c = (int)__shfl_sync(0xffffffffu, cl, j);
      uint64_t* res = slots + (u0 + j) * (int64_t)l_max;
      int B;
      if (c <= 32) B = merge_row32(res, c, lane, key);
      else if (c <= 64) B = merge_row_regs<2>(res, c, lane);
      else B = merge_row_regs<4>(res, c, lane);
      if (lane == j) outc = (uint32_t)B;
    }
    if (u < n && outc != cl) count[u] = outc;
  }
}

// Block (256 threads) sum and exclusive scan of one int per thread; s8 = 8 ints of SMEM.
__device__ __forceinline__ int block256_sum(int x, int* s8) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (lane == 0) s8[w] = x;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += s8[i];
  __syncthreads();
  return t;
}
__device__ __forceinline__ int block256_excl(int x, int* s8) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s8[w] = inc;
  __syncthreads();
  int off = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) off += i < w ? s8[i] : 0;
  __syncthreads();
  return off + inc - x;
}

// The deferred owner's key sources: the front of its row (the runs that fit: every instance whose run passed
// l_max claimed a later position than every run that fit, so the fitted runs are exactly [0, min base of the
// owner's overflow records)), then each overflow record's keys.
__device__ __forceinline__ uint32_t row_prefix(uint32_t c, const HpOverflow& ov, uint32_t u) {
  uint32_t pre = c;
  for (uint32_t r = ov.head[u]; r != ~0u; r = ov.rec_next[r]) pre = min(pre, ov.rec[r].y);
  return pre;
}

// Sort merge for the deferred owners with at most 32 E_MAX keys (nearly all of them): a warp per owner. Its keys (row
// front, then the overflow records) are staged in the warp's SMEM buffer and sorted in registers (bitonic, u64
// hash | okey | id); the first key of every hash run is the bucket minimum. When more than l_max buckets remain, the
// run heads are rotated to (okey | id | hash), sorted again, and the l_max smallest kept — the eviction rule's end
// state ((okey, id) is distinct per bucket: a candidate's hash is a function of the pair). Owners with
// more keys go to `big` for the table kernel.
template <int E>
__device__ __forceinline__ void defer_sort_owner(const uint64_t* buf, int total, int l_max, uint64_t* res,
                                                 uint32_t* cnt_u, int lane) {
  uint64_t key[E];
#pragma unroll
  for (int e = 0; e < E; ++e) key[e] = e * 32 + lane < total ? buf[e * 32 + lane] : ~0ull;
  warp_sort_regs_rolled<E>(key, lane);
  bool keep[E];
  int nh = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint64_t up = __shfl_up_sync(0xffffffffu, key[e], 1);
    const uint64_t last = __shfl_sync(0xffffffffu, key[e > 0 ? e - 1 : 0], 31);  // element 32e - 1
    const uint64_t prev = lane > 0 ? up : last;
    const bool first = (e == 0 && lane == 0) || ((prev >> 48) != (key[e] >> 48));
    keep[e] = key[e] != ~0ull && first;
    nh += __popc(__ballot_sync(0xffffffffu, keep[e]));
  }
  if (nh <= l_max) {
    int base = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t bal = __ballot_sync(0xffffffffu, keep[e]);
      if (keep[e]) res[base + __popc(bal & ((1u << lane) - 1u))] = key[e];
      base += __popc(bal);
    }
    if (lane == 0) *cnt_u = (uint32_t)base;
    return;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) key[e] = keep[e] ? ((key[e] << 16) | (key[e] >> 48)) : ~0ull;
  warp_sort_regs_rolled<E>(key, lane);
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (e * 32 + lane < l_max) res[e * 32 + lane] = (key[e] >> 16) | (key[e] << 48);
  if (lane == 0) *cnt_u = (uint32_t)l_max;
}
constexpr int kDeferSortMax = 512;  // keys per owner of the sort merge (E = 16)
constexpr int kDeferRecs = 64;      // overflow records per owner of the sort merge
__global__ void __launch_bounds__(128) hp_defer_sort_kernel(int l_max, uint64_t* __restrict__ slots,
                                                            uint32_t* __restrict__ count, HpOverflow ov,
                                                            const uint32_t* __restrict__ list,
                                                            const uint32_t* __restrict__ list_n,
                                                            uint32_t* __restrict__ big, uint32_t* __restrict__ big_n) {
  __shared__ uint64_t sbuf[4][kDeferSortMax];
  __shared__ uint2 srec[4][kDeferRecs];  // the owner's overflow records (key offset, key count), in list order
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t* buf = sbuf[w];
  uint2* recs = srec[w];
  const int64_t nl = *list_n;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nl; it += nw) {
    const uint32_t u = list[it];
    uint64_t* res = slots + (int64_t)u * l_max;
    // one walk of the record list (a dependent chain: overlap-heavy builds link ~20 records per owner), the
    // records kept in SMEM so that their keys then load in parallel
    uint32_t pre = count[u], novf = 0;
    int nrec = 0;
    for (uint32_t r = ov.head[u]; r != ~0u; r = ov.rec_next[r]) {
      const uint4 rc = ov.rec[r];
      pre = min(pre, rc.y);
      novf += rc.w;
      if (lane == 0 && nrec < kDeferRecs) recs[nrec] = make_uint2(rc.z, rc.w);
      ++nrec;
    }
    const int total = (int)(pre + novf);
    if (total > kDeferSortMax || nrec > kDeferRecs) {
      if (lane == 0) big[atomicAdd(big_n, 1u)] = u;
      continue;
    }
    __syncwarp();
    for (int i = lane; i < (int)pre; i += 32) buf[i] = res[i];
    int off = (int)pre;
    for (int q = 0; q < nrec; ++q) {
      const uint2 rc = recs[q];
      for (int t = lane; t < (int)rc.y; t += 32) buf[off + t] = ov.keys[(uint64_t)rc.x + t];
      off += (int)rc.y;
    }
    __syncwarp();
    if (total <= 128) defer_sort_owner<4>(buf, total, l_max, res, count + u, lane);
    else defer_sort_owner<16>(buf, total, l_max, res, count + u, lane);
  }
}

// Table merge for the deferred owners (hubs, evictions; m <= 12): one CTA per owner, a 2^m-entry SMEM table
// indexed by the hash. Every key goes in with a 64-bit atomicMin on its bucket — the bucket minimum of Alg. 3's
// collision rule, in any order. When more than l_max buckets are occupied, the l_max-th smallest 48-bit
// (dist16 | id32) value is found by an MSB-first radix select with block-wide counts (values are distinct: one
// bucket per id) and only the entries at or below it are kept (the eviction rule's end state).
__global__ void __launch_bounds__(256) hp_defer_table_kernel(int m, int l_max, uint64_t* __restrict__ slots,
                                                             uint32_t* __restrict__ count, HpOverflow ov,
                                                             const uint32_t* __restrict__ list,
                                                             const uint32_t* __restrict__ list_n) {
  extern __shared__ uint64_t tbl[];  // [2^m]
  __shared__ int s8[8];
  __shared__ uint32_t s_hist[256];
  __shared__ uint32_t s_sel;
  const int NB = 1 << m, tid = threadIdx.x;
  const int64_t nl = *list_n;
  constexpr uint64_t kLow48 = 0xFFFFFFFFFFFFull;
  for (int64_t it = blockIdx.x; it < nl; it += gridDim.x) {
    const uint32_t u = list[it];
    uint64_t* res = slots + (int64_t)u * l_max;
    const uint32_t pre = row_prefix(count[u], ov, u);
    __syncthreads();  // the previous owner's table is no longer read
    for (int t = tid; t < NB; t += 256) tbl[t] = ~0ull;
    __syncthreads();
    auto put = [&](uint64_t key) { atomicMin((unsigned long long*)&tbl[key >> 48], (unsigned long long)key); };
    for (uint32_t t = tid; t < pre; t += 256) put(res[t]);
    for (uint32_t r = ov.head[u]; r != ~0u; r = ov.rec_next[r]) {
      const uint4 rc = ov.rec[r];
      for (uint32_t t = tid; t < rc.w; t += 256) put(ov.keys[(uint64_t)rc.z + t]);
    }
    __syncthreads();
    uint64_t v[16];
    int cnt = 0;
    const int per = (NB + 255) / 256;  // table entries per thread (<= 16; contiguous chunk)
    const int b0 = tid * per;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      v[e] = (e < per && b0 + e < NB) ? tbl[b0 + e] : ~0ull;
      cnt += v[e] != ~0ull ? 1 : 0;
    }
    const int total = block256_sum(cnt, s8);
    uint64_t thr48 = kLow48;
    if (total > l_max) {
      // radix select, 8-bit digits MSB first: the bucket of the need-th smallest among the values that share
      // the prefix decided so far (6 rounds of a 256-bin SMEM histogram + scan)
      uint32_t* hist = s_hist;
      uint64_t prefix = 0;
      int need = l_max;
      for (int sh = 40; sh >= 0; sh -= 8) {
        hist[tid] = 0u;
        __syncthreads();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const uint64_t x = v[e] & kLow48;
          if (v[e] != ~0ull && (sh == 40 || (x >> (sh + 8)) == (prefix >> (sh + 8))))
            atomicAdd(&hist[(x >> sh) & 0xFF], 1u);
        }
        __syncthreads();
        const int hb = (int)hist[tid];
        const int below = block256_excl(hb, s8);  // values with this prefix and a smaller digit
        if (below < need && need <= below + hb) s_sel = (uint32_t)((tid << 16) | (uint32_t)(need - below));
        __syncthreads();
        const uint32_t sel = s_sel;
        prefix |= (uint64_t)(sel >> 16) << sh;
        need = (int)(sel & 0xFFFFu);
      }
      thr48 = prefix;
    }
    int kc = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) kc += (v[e] != ~0ull && (v[e] & kLow48) <= thr48) ? 1 : 0;
    int o = block256_excl(kc, s8);
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (v[e] != ~0ull && (v[e] & kLow48) <= thr48) res[o++] = v[e];
    if (tid == 255) count[u] = (uint32_t)o;
  }
}

// Generic merge for the deferred owners (any m): a warp per owner, the chunked SMEM algorithm of hp_merge_kernel
// over the owner's sources (row front, then the overflow records).
__global__ void __launch_bounds__(128) hp_defer_generic_kernel(int l_max, int cap, uint64_t* __restrict__ slots,
                                                               uint32_t* __restrict__ count, HpOverflow ov,
                                                               const uint32_t* __restrict__ list,
                                                               const uint32_t* __restrict__ list_n) {
  extern __shared__ uint64_t gm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* buf = gm + (size_t)warp * 2 * cap;
  uint64_t* tmp = buf + cap;
  const int64_t nl = *list_n;
  for (int64_t it = blockIdx.x * 4 + warp; it < nl; it += (int64_t)gridDim.x * 4) {
    const uint32_t u = list[it];
    uint64_t* res = slots + (int64_t)u * l_max;
    const uint32_t pre = row_prefix(count[u], ov, u);
    int c = 0;
    auto absorb = [&](const uint64_t* src, int len) {
      int e = 0;
      while (e < len) {
        const int chunk = min(len - e, cap - c);
        for (int t = lane; t < chunk; t += 32) buf[c + t] = src[e + t];
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
    };
    absorb(res, (int)pre);
    for (uint32_t r = ov.head[u]; r != ~0u; r = ov.rec_next[r]) {
      const uint4 rc = ov.rec[r];
      absorb(ov.keys + rc.z, (int)rc.w);
    }
    for (int t = lane; t < c; t += 32) res[t] = buf[t];
    if (lane == 0) count[u] = (uint32_t)c;
  }
}

pipnn_status hashprune_from_leaves(int m, int l_max, int64_t n, const void* sketch, bool sk_int, uint64_t* slots,
                                   uint32_t* count, const int64_t* leaf_off, int64_t n_leaves, const uint32_t* leaf_ids,
                                   int64_t n_inst, int k, const uint16_t* cols, const float* dist, int max_leaf,
                                   int64_t* n_edges_dev, Arena& ar, const Ctx& c, int inst_per_point) {
  // more than 4 leaf instances per point (wide overlap, e.g. fanout [10, 3]: 30): the instance-major path
  // (fanout [10, 3] at 1M points: HashPrune 25.6 vs 44 ms owner-major); C5 (2 per point): owner-major (56 vs 74 ms)
  static const int im_min = [] {  // experiment hook (read once): instances per point from which im is used
    const char* e = std::getenv("PIPNN_HP_IM_MIN");
    return e ? std::atoi(e) : 5;
  }();
  if (inst_per_point >= im_min)
    return im::from_leaves(m, l_max, n, sketch, sk_int, slots, count, leaf_off, n_leaves, leaf_ids, n_inst, k, cols,
                           dist, max_leaf, n_edges_dev, ar, c);
  // overflow capacity: every key of the wave (at most 2 k per instance) — never exceeded
  const int64_t P = std::max<int64_t>(1, 2 * n_inst * k);
  HpOverflow ov{};
  ov.keys = ar.take<uint64_t>(P);
  ov.keys_cap = (unsigned long long)P;
  ov.rec = ar.take<uint4>(std::max<int64_t>(1, n_inst));
  ov.rec_next = ar.take<uint32_t>(std::max<int64_t>(1, n_inst));
  ov.rec_cap = (uint32_t)std::min<int64_t>(std::max<int64_t>(1, n_inst), 0xFFFFFFFFll);
  ov.head = ar.take<uint32_t>(std::max<int64_t>(1, n));
  uint32_t* counters = ar.take<uint32_t>(6);  // keys_n (u64), rec_n, defer_n, big_n
  uint32_t* defer = ar.take<uint32_t>(std::max<int64_t>(1, n));
  uint32_t* defer_big = ar.take<uint32_t>(std::max<int64_t>(1, n));
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (hashprune)");
  if (P >= ((int64_t)1 << 32)) return fail(PIPNN_EUNSUPPORTED, "hashprune: more than 2^32 edge keys in one wave");
  ov.keys_n = reinterpret_cast<unsigned long long*>(counters);
  ov.rec_n = counters + 2;
  uint32_t* defer_n = counters + 3;
  PIPNN_CUDA(kmemset(n_edges_dev, 0, sizeof(int64_t), c.st));
  if (n_inst == 0 || n_leaves == 0) return PIPNN_OK;
  PIPNN_CUDA(kmemset(counters, 0, 6 * sizeof(uint32_t), c.st));
  PIPNN_CUDA(kmemset(ov.head, 0xFF, (size_t)n * sizeof(uint32_t), c.st));
  // (1) leaf-local emission of both edge directions into the owners' rows; members' sketches staged in SMEM
  // (C5's 2048-member leaves: 106 KB of sketches, so a CTA of 1024 threads per leaf there instead of 256)
  max_leaf = std::max(1, std::min(max_leaf, 4096));
  const size_t sk_bytes = (size_t)max_leaf * (m | 1) * 4;
  const size_t mem_bytes = (size_t)max_leaf * kEmitBytesPerMember;
  const int stage_sk = mem_bytes + sk_bytes <= 200 * 1024 ? 1 : 0;
  const int smem = (int)(mem_bytes + (stage_sk ? sk_bytes : 0));
  const bool big = max_leaf > 1024;
  // Leaves above 1024 members take 1024-thread CTAs (one per SM: 145 KB of SMEM at 2048 members); with such
  // leaves present the smaller ones go in a launch of their own with 512-thread CTAs and SMEM for 1024 members
  // (two per SM, so one CTA's barriers and claim latencies overlap the other's work). Both launches span all
  // leaves; a CTA whose leaf is not of the launch's size class exits at once.
  const int smem_half = (int)((size_t)1024 * kEmitBytesPerMember + (stage_sk ? (size_t)1024 * (m | 1) * 4 : 0));
#define HP_EMIT(ST, NTH, MINB, SM, LO, HI)                                                                        \
  do {                                                                                                            \
    PIPNN_CUDA(cudaFuncSetAttribute(hp_emit_kernel<ST, NTH, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM)); \
    hp_emit_kernel<ST, NTH, MINB><<<(unsigned)n_leaves, NTH, SM, c.st>>>(leaf_off, leaf_ids, k, cols, dist,       \
                                                                 (const ST*)sketch, m, stage_sk, l_max, slots,     \
                                                                 count, ov, n_edges_dev, c.err, LO, HI);           \
  } while (0)
#define HP_EMIT_BIG(ST)                                     \
  do {                                                      \
    HP_EMIT(ST, 512, 2, smem_half, 0, 1024);                \
    HP_EMIT(ST, 1024, 1, smem, 1024, 1 << 30);              \
  } while (0)
  if (sk_int) {
    if (big) HP_EMIT_BIG(int32_t);
    else HP_EMIT(int32_t, 256, 1, smem, 0, 1 << 30);
  } else {
    if (big) HP_EMIT_BIG(float);
    else HP_EMIT(float, 256, 1, smem, 0, 1 << 30);
  }
#undef HP_EMIT_BIG
#undef HP_EMIT
  PIPNN_LAUNCHED("hp_emit_kernel", c.st);
  // (2) row merge per owner; owners with long rows (hubs, overflow) through the deferred kernels
  const int64_t blocks = std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 16);
  hp_merge_rows_kernel<<<(unsigned)std::max<int64_t>(1, blocks), 256, 0, c.st>>>(n, l_max, slots, count, defer, defer_n);
  PIPNN_LAUNCHED("hp_merge_rows_kernel", c.st);
  if (m <= 12) {
    // most deferred owners by the warp sort merge, the ones with more than kDeferSortMax keys by the table kernel
    hp_defer_sort_kernel<<<(unsigned)(num_sms() * 8), 128, 0, c.st>>>(l_max, slots, count, ov, defer, defer_n,
                                                                     defer_big, defer_n + 1);
    PIPNN_LAUNCHED("hp_defer_sort_kernel", c.st);
    const int tsm = (int)((size_t)8 << m);
    PIPNN_CUDA(cudaFuncSetAttribute(hp_defer_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tsm));
    hp_defer_table_kernel<<<(unsigned)(num_sms() * 6), 256, tsm, c.st>>>(m, l_max, slots, count, ov, defer_big,
                                                                       defer_n + 1);
    PIPNN_LAUNCHED("hp_defer_table_kernel", c.st);
  } else {
    const int cap = merge_cap(l_max);
    const int gsm = 4 * 2 * cap * (int)sizeof(uint64_t);
    PIPNN_CUDA(cudaFuncSetAttribute(hp_defer_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gsm));
    hp_defer_generic_kernel<<<(unsigned)(num_sms() * 4), 128, gsm, c.st>>>(l_max, cap, slots, count, ov, defer,
                                                                          defer_n);
    PIPNN_LAUNCHED("hp_defer_generic_kernel", c.st);
  }
  static const bool dbg_timing = [] {
    const char* e = std::getenv("PIPNN_DEBUG_TIMING");
    return e && e[0] == '1';
  }();
  if (dbg_timing) {
    uint32_t hc[6] = {0, 0, 0, 0, 0, 0};
    PIPNN_CUDA(cudaMemcpyAsync(hc, counters, sizeof(hc), cudaMemcpyDeviceToHost, c.st));
    PIPNN_CUDA(cudaStreamSynchronize(c.st));
    std::fprintf(stderr, "[pipnn] hashprune: %u owners deferred (%u to the table merge), %u overflow records, %llu overflow keys\n", hc[3], hc[4],
                 hc[2], (unsigned long long)hc[0] | ((unsigned long long)hc[1] << 32));
  }
  return PIPNN_OK;
}

}  // namespace pipnn
