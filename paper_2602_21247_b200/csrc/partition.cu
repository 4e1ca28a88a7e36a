// partition.cu — Randomized Ball Carving with fanout and merging (§4.1, Alg. 5) as a
// level-synchronous GPU loop. The recursion of Alg. 5 is breadth-first here: all open subproblems of one
// depth are processed together, which is equivalent because every subproblem is carved independently
// from its own key (docs/DETERMINISM.md). Per level:
//   1. leaders: the l_g members with the smallest mix(K_g, id) (line 2, "SampleLeaders"): a threshold
//      filter keeps ~4 l_g + 64 candidates per subproblem in a segment of capacity 8 l_g + 256, a
//      (segmented) sort orders them, the first l_g are sorted by id. mix(K, .) is injective, so the selection
//      is exact; if any subproblem's filter kept more than its capacity or fewer than l_g candidates, the
//      level is redone without the filter.
//   2. nearest leaders (lines 5-9): members and leaders are gathered into the tiled MMA layout and the
//      dist_topk kernel (tcgen05, the same kernel as the leaf pick) returns each member's f_g nearest
//      leaders by (D, leader id) — leaders are in ascending id order, so "smaller column" = "smaller id".
//   3. group-by: the distance kernel writes (child, id) pairs in member order and the child histogram;
//      a stable radix sort by child -> every child ascending.
//   4. one device->host copy of the child sizes and leader ids (the level's only synchronisation); the
//      host applies the merge rule of small
//      siblings (line 10, R15), the base case, the degenerate-input guard, and schedules
//      (a) leaf jobs (plain copies, or sorted + deduplicated unions for merged groups) and
//      (b) the next level's subproblems (children larger than C_max, key mix(K_g, l + 1)).
// At the end, leaf sizes -> exclusive scan -> leaf_off, and the staged leaves are compacted into leaf_ids.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cub/cub.cuh>
#include <map>
#include <thread>
#include <vector>

#include "internal.h"

namespace pipnn {

struct PGroup {       // device view of an open subproblem at the current level
  uint64_t key;       // K_g
  uint64_t thr;       // leader-priority filter threshold
  int64_t off;        // members: mem[off .. off+size)
  int64_t cbase;      // compacted member index of its first member
  int64_t size;
  int64_t cand_off;   // candidate buffer offset
  int64_t lead_off;   // leader buffer offset (= child base)
  int64_t pair_off;   // (member, slot) pair offset
  int32_t l, f;
  int32_t cap;        // candidate segment capacity
  int32_t pad_;
};

struct LeafPart {
  int64_t src;  // offset into the level's child-id buffer
  int32_t len;
  int32_t pad_;
};
struct LeafJob {
  int64_t dst;      // staging offset
  int64_t leaf;     // leaf index
  int32_t part0, nparts;
};

// ------------------------------------------------------------------ kernels
__global__ void iota_reps_kernel(uint32_t* __restrict__ out, int64_t n, int reps) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * reps; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (uint32_t)(e % n);
}

__device__ __forceinline__ int find_group(const int64_t* __restrict__ cbase, int G, int64_t e) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cbase[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Leader candidates: members whose priority mix(K_g, id) is below the group's filter threshold, scattered into
// the group's candidate segment [cand_off, cand_off + cap) (the rest of the segment stays ~0 and sorts last).
// A group whose filter kept more than cap or fewer than l candidates raises *redo (the level is then redone
// without the filter, exactly).
__global__ void prio_kernel(const PGroup* __restrict__ gs, const int64_t* __restrict__ cbase, int G, int64_t M,
                            const uint32_t* __restrict__ mem, uint32_t* __restrict__ cnt, uint64_t* __restrict__ ck,
                            uint32_t* __restrict__ cv, int* __restrict__ redo) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M; e += (int64_t)gridDim.x * blockDim.x) {
    const int g = find_group(cbase, G, e);
    const PGroup& p = gs[g];
    const uint32_t id = mem[p.off + (e - p.cbase)];
    const uint64_t pri = mix64(p.key, id);
    if (pri < p.thr || p.thr == ~0ull) {
      const uint32_t slot = atomicAdd(&cnt[g], 1u);
      if (slot < (uint32_t)p.cap) {
        ck[p.cand_off + slot] = pri;
        cv[p.cand_off + slot] = id;
      } else {
        *redo = 1;
      }
    }
  }
}

__global__ void prio_check_kernel(const PGroup* __restrict__ gs, int G, const uint32_t* __restrict__ cnt,
                                  int* __restrict__ redo) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < G && cnt[g] < (uint32_t)gs[g].l) *redo = 1;
}

__global__ void init_ctr_kernel(unsigned long long* ctr, unsigned long long stage0, int* max_depth) {
  if (threadIdx.x == 0) {
    ctr[0] = 0ull;     // device-carved leaves
    ctr[1] = stage0;   // their staging cursor (second half of the staging area)
    *max_depth = 0;
  }
}

__global__ void iota_kernel(uint32_t* __restrict__ out, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (uint32_t)e;
}

// The level's work items (one per 128-row block of every group's members, resp. leaders): CTA g writes
// its group's items at its offsets (host prefix sums over the groups; the item lists themselves never pass the host).
__global__ void level_items_kernel(const int64_t* __restrict__ offA, const int64_t* __restrict__ offB, int G,
                                   WorkItem* __restrict__ itA, WorkItem* __restrict__ itB,
                                   const int64_t* __restrict__ offP, WorkItem* __restrict__ itP) {
  const int g = blockIdx.x;
  if (g >= G) return;
  const int64_t a0 = offA[g], a1 = offA[g + 1], b0 = offB[g], b1 = offB[g + 1];
  for (int64_t i = a0 + threadIdx.x; i < a1; i += blockDim.x) itA[i] = WorkItem{g, (int32_t)(i - a0)};
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) itB[i] = WorkItem{g, (int32_t)(i - b0)};
  if (itP) {  // pair items (blocks 2i, 2i + 1) for dist_topk_uf2_kernel's static schedule
    const int64_t p0 = offP[g], p1 = offP[g + 1];
    for (int64_t i = p0 + threadIdx.x; i < p1; i += blockDim.x) itP[i] = WorkItem{g, (int32_t)(2 * (i - p0))};
  }
}

// Leaders of every group (Alg. 5 line 3, R12): the l_g candidates of smallest priority, then by id. One
// CTA (1024 threads) per group over its candidate segment (cap entries; unfilled slots hold key ~0; real keys are
// distinct: mix(K, .) is injective):
//   * cap <= 2048: the segment bitonic-sorted by key in SMEM, the first l_g ids taken;
//   * larger: an MSB-first radix select, 12 bits per pass: a SMEM histogram of the digit of every key under the
//     current prefix, the bin holding the l_g-th key found by a block scan; keys in smaller bins are taken, the
//     boundary bin becomes the prefix, until it holds <= 2048 keys, which are bitonic-sorted and the rest taken;
// then the l_g ids are bitonic-sorted ascending and written to lead_sorted.
constexpr int kLeadSortMax = 1 << 20;  // segments above this use the library sort (redo_unfiltered only)
constexpr int kLeadSmall = 2048;
__device__ __forceinline__ int next_pow2_dev(int x) { return x <= 1 ? 1 : 1 << (32 - __clz(x - 1)); }
template <typename K, typename V>
__device__ void block_bitonic(K* k, V* v, int N) {  // ascending by k, N a power of two, all threads of the block
  for (int size = 2; size <= N; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (N >> 1); i += blockDim.x) {
        const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const K a = k[lo], b = k[hi];
        if ((a > b) == up) {
          k[lo] = b;
          k[hi] = a;
          if (v) {
            const V t = v[lo];
            v[lo] = v[hi];
            v[hi] = t;
          }
        }
      }
      __syncthreads();
    }
}
// SMEM: keys [kLeadSmall] u64 | ids [kLeadSmall] u32 | hist [4096] u32 | warp sums [32] | sel [l_max] u32 | scalars
__global__ void __launch_bounds__(1024) leaders_kernel(const PGroup* __restrict__ gs, int G, const uint64_t* __restrict__ ck,
                                                       const uint32_t* __restrict__ cv, uint32_t* __restrict__ lead_sorted) {
  extern __shared__ __align__(16) uint64_t lsm[];
  __shared__ int nsel_sh, bin_sh, below_sh, nb_sh;
  const int g = blockIdx.x;
  if (g >= G) return;
  const PGroup p = gs[g];
  const int cap = p.cap, l = p.l, tid = threadIdx.x, nt = blockDim.x;
  uint64_t* k = lsm;
  uint32_t* v = reinterpret_cast<uint32_t*>(k + kLeadSmall);
  uint32_t* hist = v + kLeadSmall;
  uint32_t* wsum = hist + 4096;
  uint32_t* sel = wsum + 32;  // [next_pow2(l)]
  const uint64_t* key = ck + p.cand_off;
  const uint32_t* id = cv + p.cand_off;
  if (tid == 0) nsel_sh = 0;
  __syncthreads();
  int need = l;  // still to select, all from keys under the prefix
  uint64_t prefix = 0;
  int pbits = 0;  // bits of the prefix (keys with key >> (64 - pbits) == prefix are "under" it)
  bool small = cap <= kLeadSmall;
  while (!small) {
    const int shift = 64 - pbits - 12;  // digit = bits [shift, shift + 12) (the last pass: 4 bits, shift 0)
    const int sh = shift < 0 ? 0 : shift;
    const uint32_t dmask = shift < 0 ? 0xFu : 0xFFFu;
    for (int i = tid; i < 4096; i += nt) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < cap; i += nt) {
      const uint64_t x = key[i];
      if (pbits == 0 || (x >> (64 - pbits)) == prefix) atomicAdd(&hist[(x >> sh) & dmask], 1u);
    }
    __syncthreads();
    // block exclusive scan of the 4096 bins (4 per thread), then the bin b with below(b) < need <= below(b + 1)
    uint32_t h4[4], s = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      h4[t] = hist[4 * tid + t];
      s += h4[t];
    }
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if ((tid & 31) >= o) inc += y;
    }
    if ((tid & 31) == 31) wsum[tid >> 5] = inc;
    __syncthreads();
    if (tid < 32) {
      uint32_t w = wsum[tid], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (tid >= o) wi += y;
      }
      wsum[tid] = wi - w;  // exclusive warp offsets
    }
    __syncthreads();
    uint32_t run = wsum[tid >> 5] + inc - s;  // exclusive prefix of this thread's first bin
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (run < (uint32_t)need && run + h4[t] >= (uint32_t)need) {
        bin_sh = 4 * tid + t;
        below_sh = (int)run;
        nb_sh = (int)h4[t];
      }
      run += h4[t];
    }
    __syncthreads();
    const int b = bin_sh, below = below_sh, nb = nb_sh;
    // take every key under the prefix whose digit is below b
    for (int i = tid; i < cap; i += nt) {
      const uint64_t x = key[i];
      if ((pbits == 0 || (x >> (64 - pbits)) == prefix) && (int)((x >> sh) & dmask) < b)
        sel[atomicAdd(&nsel_sh, 1)] = id[i];
    }
    need -= below;
    prefix = (prefix << (shift < 0 ? 4 : 12)) | (uint64_t)b;
    pbits += shift < 0 ? 4 : 12;
    __syncthreads();
    if (nb <= kLeadSmall || pbits >= 64) {
      // the boundary bin: its keys into the small buffer
      if (tid == 0) bin_sh = 0;
      __syncthreads();
      for (int i = tid; i < cap; i += nt) {
        const uint64_t x = key[i];
        if ((x >> (64 - pbits)) == prefix || pbits >= 64 && x == prefix) {
          const int j = atomicAdd(&bin_sh, 1);
          if (j < kLeadSmall) {
            k[j] = x;
            v[j] = id[i];
          }
        }
      }
      __syncthreads();
      small = true;
    }
  }
  // sort the small set by key and take its first `need`
  const int ns = cap <= kLeadSmall ? cap : min(bin_sh, kLeadSmall);
  const int N = next_pow2_dev(ns < 2 ? 2 : ns);
  if (cap <= kLeadSmall)
    for (int i = tid; i < N; i += nt) {
      k[i] = i < cap ? key[i] : ~0ull;
      v[i] = i < cap ? id[i] : 0u;
    }
  else
    for (int i = ns + tid; i < N; i += nt) k[i] = ~0ull;
  __syncthreads();
  block_bitonic<uint64_t, uint32_t>(k, v, N);
  const int base = nsel_sh;
  for (int j = tid; j < need; j += nt) sel[base + j] = v[j];
  __syncthreads();
  // the l leaders ascending by id
  const int N2 = next_pow2_dev(l < 2 ? 2 : l);
  for (int i = l + tid; i < N2; i += nt) sel[i] = 0xFFFFFFFFu;
  __syncthreads();
  block_bitonic<uint32_t, uint32_t>(sel, nullptr, N2);
  for (int j = tid; j < l; j += nt) lead_sorted[p.lead_off + j] = sel[j];
}

// first l_g sorted candidates -> leaders (then sorted by id with a segmented sort)
__global__ void take_leaders_kernel(const PGroup* __restrict__ gs, int G, const uint32_t* __restrict__ cv_sorted,
                                    uint32_t* __restrict__ lead) {
  const int g = blockIdx.x;
  if (g >= G) return;
  const PGroup& p = gs[g];
  for (int j = threadIdx.x; j < p.l; j += blockDim.x) lead[p.lead_off + j] = cv_sorted[p.cand_off + j];
}

// One CTA per leaf job: a plain copy, or the sorted, deduplicated union of several sibling groups.
__global__ void __launch_bounds__(256) leaf_job_kernel(const LeafJob* __restrict__ jobs, int nj,
                                                       const LeafPart* __restrict__ parts,
                                                       const uint32_t* __restrict__ src, uint32_t* __restrict__ staging,
                                                       int64_t* __restrict__ leaf_size) {
  __shared__ uint32_t a[4096];
  __shared__ int total_sh;
  const int j = blockIdx.x;
  if (j >= nj) return;
  const LeafJob J = jobs[j];
  if (J.nparts == 1) {
    const LeafPart P = parts[J.part0];
    for (int i = threadIdx.x; i < P.len; i += blockDim.x) staging[J.dst + i] = src[P.src + i];
    if (threadIdx.x == 0) leaf_size[J.leaf] = P.len;
    return;
  }
  int total = 0;
  for (int q = 0; q < J.nparts; ++q) {
    const LeafPart P = parts[J.part0 + q];
    for (int i = threadIdx.x; i < P.len; i += blockDim.x) a[total + i] = src[P.src + i];
    total += P.len;
  }
  int Pn = 32;
  while (Pn < total) Pn <<= 1;
  for (int i = total + threadIdx.x; i < Pn; i += blockDim.x) a[i] = 0xFFFFFFFFu;
  __syncthreads();
  for (int k = 2; k <= Pn; k <<= 1)
    for (int s = k >> 1; s > 0; s >>= 1) {
      for (int i = threadIdx.x; i < Pn; i += blockDim.x) {
        const int ixj = i ^ s;
        if (ixj > i) {
          const uint32_t x = a[i], y = a[ixj];
          if ((x > y) == ((i & k) == 0)) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x < 32) {  // warp 0: ordered compaction of first occurrences
    const int lane = threadIdx.x;
    int base = 0;
    for (int i0 = 0; i0 < total; i0 += 32) {
      const int i = i0 + lane;
      const bool keep = i < total && (i == 0 || a[i] != a[i - 1]);
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) staging[J.dst + base + __popc(bal & ((1u << lane) - 1u))] = a[i];
      base += __popc(bal);
    }
    if (lane == 0) total_sh = base;
  }
  __syncthreads();
  if (threadIdx.x == 0) leaf_size[J.leaf] = total_sh;
}

__global__ void leaf_compact_kernel(int64_t nl, const int64_t* __restrict__ leaf_dst, const int64_t* __restrict__ off,
                                    const uint32_t* __restrict__ staging, uint32_t* __restrict__ out) {
  for (int64_t b = blockIdx.x; b < nl; b += gridDim.x) {
    const int64_t s = off[b], len = off[b + 1] - s, d = leaf_dst[b];
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) out[s + i] = staging[d + i];
  }
}

// Host -> device copies of the per-depth plan go through pinned staging memory: a copy from pageable memory
// synchronises the stream first, which would serialise the host planning with every kernel of the level.
// Two thread-local arenas: one for the level's plan (reused after the level's synchronisation), one for the
// leaf jobs (reused after the next level's synchronisation). Growing synchronises the stream first.
struct PinnedArena {
  uint8_t* base = nullptr;
  size_t cap = 0, used = 0;
  ~PinnedArena() {
    if (base) cudaFreeHost(base);
  }
  std::vector<KCopyDesc> pend;  // staged copies not yet launched (flush: one kernel for all of them)
  cudaError_t grow(size_t need, cudaStream_t st) {
    cudaError_t e = flush(st);  // the pending copies read the old block: launch them first
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);  // every pending copy from this arena has completed
    if (e != cudaSuccess) return e;
    if (base) cudaFreeHost(base);
    base = nullptr;
    cap = std::max<size_t>(2 * cap, std::max<size_t>(need, (size_t)1 << 20));
    used = 0;
    e = cudaHostAlloc((void**)&base, cap, cudaHostAllocMapped);  // read by the copy kernel
    if (e != cudaSuccess) {
      base = nullptr;
      cap = 0;
    }
    return e;
  }
  uint8_t* stage(const void* src, size_t bytes, cudaStream_t st, cudaError_t& e) {
    e = cudaSuccess;
    const size_t need = (used + bytes + 255) & ~(size_t)255;
    if (need > cap && (e = grow(need, st)) != cudaSuccess) return nullptr;
    uint8_t* p = base + used;
    used = (used + bytes + 255) & ~(size_t)255;
    if (src) std::memcpy(p, src, bytes);
    return p;
  }
  // Stage src and queue its copy to dst; it runs at the next flush (call flush before the first kernel
  // that reads dst).
  cudaError_t copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return cudaSuccess;
    cudaError_t e;
    uint8_t* p = stage(src, bytes, st, e);
    if (!p) return e;
    pend.push_back(KCopyDesc{dst, p, (unsigned long long)bytes});
    return cudaSuccess;
  }
  cudaError_t flush(cudaStream_t st) {
    if (pend.empty()) return cudaSuccess;
    const size_t nb = pend.size() * sizeof(KCopyDesc);
    std::vector<KCopyDesc> d;
    d.swap(pend);
    const size_t need = (used + nb + 255) & ~(size_t)255;
    if (need > cap) {  // no room for the descriptors: launch the copies one by one (rare)
      for (const KCopyDesc& x : d) {
        cudaError_t e = kcopy(x.dst, x.src, x.bytes, st);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    }
    uint8_t* p = base + used;
    used = need;
    std::memcpy(p, d.data(), nb);
    return kcopy_batch(reinterpret_cast<const KCopyDesc*>(p), (int)d.size(), st);
  }
  void reset() { used = 0; pend.clear(); }
};
static thread_local PinnedArena g_pin_level, g_pin_jobs;

// The level synchronisation's event (per thread and device, created once; no timing).
static cudaEvent_t level_sync_event() {
  static thread_local std::map<int, cudaEvent_t> evs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  auto it = evs.find(dev);
  if (it != evs.end()) return it->second;
  cudaEvent_t e = nullptr;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
  evs[dev] = e;
  return e;
}

// ------------------------------------------------------------------ host helpers
static int64_t leaders_of(int64_t sz, const pipnn_partition_params* p) {
  int64_t l = ((int64_t)p->p_samp_num * sz + p->p_samp_den - 1) / p->p_samp_den;
  l = std::max<int64_t>(l, 2);
  l = std::min<int64_t>(l, p->leader_cap);
  return std::min<int64_t>(l, sz);
}

static int64_t prod_fan(const pipnn_partition_params* p) {
  int64_t f = 1;
  for (int i = 0; i < p->n_fanout; ++i) f *= p->fanout[i];
  return f * p->replicas;
}

struct HGroup {  // host view of an open subproblem
  int64_t off, size;
  uint64_t key;
};

// Merge plan of one parent's children (R15) — same rule as the oracle, re-implemented.
struct HMerge {
  std::vector<int> big;
  std::vector<std::vector<int>> bins;
  std::vector<int> leftover;
  int absorb = -1;
};
static HMerge merge_plan(const std::vector<int64_t>& sz, const std::vector<std::pair<uint64_t, uint32_t>>& key,
                         int64_t c_min, int64_t c_max) {
  HMerge m;
  std::vector<int> small;
  for (int j = 0; j < (int)sz.size(); ++j) {
    if (sz[j] == 0) continue;
    if (sz[j] < c_min) small.push_back(j);
    else m.big.push_back(j);
  }
  std::sort(small.begin(), small.end(), [&](int a, int b) { return key[a] < key[b]; });
  std::vector<int> cur;
  int64_t sum = 0;
  for (int j : small) {
    cur.push_back(j);
    sum += sz[j];
    if (sum >= c_min) {
      m.bins.push_back(cur);
      cur.clear();
      sum = 0;
    }
  }
  if (!cur.empty()) {
    if (!m.bins.empty()) {
      m.bins[0].insert(m.bins[0].end(), cur.begin(), cur.end());
    } else {
      for (int j : m.big) {
        if (sz[j] + sum > c_max) continue;
        if (m.absorb < 0 || sz[j] < sz[m.absorb] || (sz[j] == sz[m.absorb] && key[j] < key[m.absorb])) m.absorb = j;
      }
      if (m.absorb < 0) m.bins.push_back(cur);
      else m.leftover = cur;
    }
  }
  return m;
}

struct PartCaps {
  int64_t L;        // instances bound n * prod(fanout) * replicas
  int64_t G;        // open groups per level
  int64_t C;        // children (leaders) per level
  int64_t J;        // leaf jobs / parts per level
  int64_t rowsA;    // tiled member rows
  int64_t rowsB;    // tiled leader rows
  int64_t leaves;   // total leaves
};
static PartCaps caps_of(const pipnn_points* X, const pipnn_partition_params* p) {
  PartCaps c;
  c.L = X->n * prod_fan(p);
  c.G = c.L / (p->c_max + 1) + p->replicas + 1;
  c.C = c.L * p->p_samp_num / p->p_samp_den + 2 * c.G + 16;
  c.C = std::min<int64_t>(c.C, c.G * p->leader_cap + 16);
  c.J = c.C + 2 * c.L / std::max(1, p->c_max) + c.G + 16;
  c.rowsA = c.L + 128 * c.G;
  c.rowsB = c.C + 128 * c.G;
  c.leaves = c.L + 1;
  return c;
}

static int bits_for(int64_t v) {
  int b = 1;
  while (((int64_t)1 << b) <= v) ++b;
  return b;
}

// CUB temporary bytes of every sort/scan of the partition at these capacities. The size queries cost tens of
// microseconds of host time at the start of each build (GPU idle), so they are cached per thread.
static size_t partition_cub_bytes(const PartCaps& cp) {
  static thread_local std::map<std::array<int64_t, 4>, size_t> cache;
  const std::array<int64_t, 4> key{cp.L, cp.G, cp.C, cp.leaves};
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  cub::DeviceSegmentedSort::SortPairs(nullptr, t1, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                      (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)std::min<int64_t>(cp.L, INT32_MAX),
                                      (int)cp.G, (const int64_t*)nullptr, (const int64_t*)nullptr);
  cub::DeviceSegmentedSort::SortKeys(nullptr, t2, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)cp.C, (int)cp.G,
                                     (const int64_t*)nullptr, (const int64_t*)nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, t3, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)std::min<int64_t>(cp.L, INT32_MAX));
  cub::DeviceScan::ExclusiveSum(nullptr, t4, (const int64_t*)nullptr, (int64_t*)nullptr, (int)cp.leaves);
  size_t t5 = 0, t6 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t5, (const uint64_t*)nullptr, (uint64_t*)nullptr, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)std::min<int64_t>(cp.L, INT32_MAX), 0, 64);
  cub::DeviceRadixSort::SortKeys(nullptr, t6, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)cp.C, 0, 32);
  const size_t bytes = std::max(std::max(std::max(t1, t2), std::max(t3, t4)), std::max(t5, t6));
  cache[key] = bytes;
  return bytes;
}

static pipnn_status partition_body(const pipnn_points* X, const pipnn_partition_params* p, int64_t* leaf_off,
                                   int64_t leaf_off_cap, uint32_t* leaf_ids, int64_t leaf_ids_cap, int64_t* n_leaves_h,
                                   int64_t* n_inst_h, int* depth_h, Arena& ar, const Ctx& c);

// The level plans are staged in thread-local mapped pinned buffers (g_pin_level, g_pin_jobs, pinned_scratch)
// that copy kernels read asynchronously; a successful call ends with its caller's synchronisation, and a
// failing one synchronises here, so no copy is still reading them when the next call resets them.
pipnn_status partition_impl(const pipnn_points* X, const pipnn_partition_params* p, int64_t* leaf_off,
                            int64_t leaf_off_cap, uint32_t* leaf_ids, int64_t leaf_ids_cap, int64_t* n_leaves_h,
                            int64_t* n_inst_h, int* depth_h, Arena& ar, const Ctx& c) {
  const pipnn_status s = partition_body(X, p, leaf_off, leaf_off_cap, leaf_ids, leaf_ids_cap, n_leaves_h, n_inst_h,
                                        depth_h, ar, c);
  if (s != PIPNN_OK && !ar.measuring()) cudaStreamSynchronize(c.st);
  return s;
}

static pipnn_status partition_body(const pipnn_points* X, const pipnn_partition_params* p, int64_t* leaf_off,
                                   int64_t leaf_off_cap, uint32_t* leaf_ids, int64_t leaf_ids_cap, int64_t* n_leaves_h,
                                   int64_t* n_inst_h, int* depth_h, Arena& ar, const Ctx& c) {
  const PartCaps cp = caps_of(X, p);
  const int Kb = tiled_row_bytes(X);
  int fmax = 1;
  for (int i = 0; i < p->n_fanout; ++i) fmax = std::max(fmax, p->fanout[i]);
  // ---- workspace
  uint32_t* memA = ar.take<uint32_t>(cp.L);
  uint32_t* memB = ar.take<uint32_t>(cp.L);
  uint32_t* staging = ar.take<uint32_t>(2 * cp.L);  // [0, L): host-staged leaves, [L, 2L): device subtrees
  int64_t* leaf_size = ar.take<int64_t>(cp.leaves + 1);
  int64_t* leaf_dst = ar.take<int64_t>(cp.leaves);
  int64_t* dev_leaf_size = ar.take<int64_t>(cp.leaves);
  int64_t* dev_leaf_dst = ar.take<int64_t>(cp.leaves);
  uint8_t* dev_groups = ar.take<uint8_t>((size_t)cp.G * subtree_group_bytes());
  unsigned long long* dev_ctr = ar.take<unsigned long long>(4);  // [0] leaves, [1] staging cursor
  int64_t* d_poff = ar.take<int64_t>(cp.G + 1);                   // pair-item offsets per group (packed pass)
  WorkItem* itP = ar.take<WorkItem>(cp.rowsA / 256 + cp.G + 1);    // pair items (packed pass on dist_topk_uf2)
  int64_t* n_pairs = ar.take<int64_t>(1);
  int* dev_work = ar.take<int>(2);                                 // [0] group counter, [1] max depth
  PGroup* d_groups = ar.take<PGroup>(cp.G);
  int64_t* d_cbase = ar.take<int64_t>(cp.G);
  uint32_t* d_cnt = ar.take<uint32_t>(cp.G);
  int64_t* d_cand_seg = ar.take<int64_t>(cp.G + 1);
  int64_t* d_lead_seg = ar.take<int64_t>(cp.G + 1);
  uint64_t* ck = ar.take<uint64_t>(cp.L);
  uint32_t* cv = ar.take<uint32_t>(cp.L);
  uint64_t* ck2 = ar.take<uint64_t>(cp.L);
  uint32_t* cv2 = ar.take<uint32_t>(cp.L);
  uint32_t* lead = ar.take<uint32_t>(cp.C);
  uint32_t* lead_sorted = ar.take<uint32_t>(cp.C);
  uint32_t* ccnt = ar.take<uint32_t>(cp.C);
  uint8_t* TA = ar.take<uint8_t>((size_t)cp.rowsA * Kb);
  int32_t* nA = ar.take<int32_t>(cp.rowsA);
  uint8_t* TB = ar.take<uint8_t>((size_t)cp.rowsB * Kb);
  int32_t* nB = ar.take<int32_t>(cp.rowsB);
  TileSeg* tsA = ar.take<TileSeg>(cp.G);
  TileSeg* tsB = ar.take<TileSeg>(cp.G);
  DistSeg* dsegs = ar.take<DistSeg>(cp.G);
  WorkItem* itA = ar.take<WorkItem>(cp.rowsA / 128 + 1);
  WorkItem* itB = ar.take<WorkItem>(cp.rowsB / 128 + 1);
  int64_t* d_itoff = ar.take<int64_t>(2 * (cp.G + 1));
  int64_t* n_it = ar.take<int64_t>(2);
  uint32_t* pk = ar.take<uint32_t>(cp.L);
  uint32_t* iota = ar.take<uint32_t>(cp.C);
  int* d_redo = ar.take<int>(1);
  uint32_t* pk2 = ar.take<uint32_t>(cp.L);
  LeafJob* d_jobs = ar.take<LeafJob>(cp.J);
  LeafPart* d_parts = ar.take<LeafPart>(cp.J);
  const size_t cub_bytes = partition_cub_bytes(cp);
  void* cub_tmp = ar.take<uint8_t>(cub_bytes);
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (partition)");
  if (leaf_ids_cap < cp.L || leaf_off_cap < cp.L + 1) return fail(PIPNN_ECAPACITY, "leaf capacities too small");

  const int64_t n = X->n;
  const int reps = p->replicas;
  const cudaStream_t st = c.st;
  // level 0: one subproblem per replica, members 0..n-1 each
  iota_reps_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n * reps, 256), num_sms() * 64), 256, 0, st>>>(memA, n, reps);
  PIPNN_LAUNCHED("iota_reps_kernel", st);
  iota_kernel<<<(unsigned)std::min<int64_t>(ceil_div(cp.C, 256), num_sms() * 16), 256, 0, st>>>(iota, cp.C);
  PIPNN_LAUNCHED("iota_kernel", st);
  init_ctr_kernel<<<1, 32, 0, st>>>(dev_ctr, (unsigned long long)cp.L, dev_work + 1);
  PIPNN_LAUNCHED("init_ctr_kernel", st);
  // subproblems below depth 0 that one CTA can carve completely go to the device subtree kernel
  static const bool use_subtree = [] {
    const char* e = std::getenv("PIPNN_NO_SUBTREE");
    return !(e && e[0] == '1');
  }();
  // from depth 1 on, one CTA carves a whole subtree (no host round trip per depth); C2: 3.01 vs 3.11 ms,
  // C3: 1.82 vs 3.34 ms partition (B200). PIPNN_SUBTREE_DEPTH moves the first device depth (experiments).
  static const int subtree_min_depth = [] {
    const char* e = std::getenv("PIPNN_SUBTREE_DEPTH");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  struct DevGroup {
    int64_t off;
    int32_t size, depth;
    uint64_t key;
  };
  static_assert(sizeof(DevGroup) == 24, "StGroup layout");
  std::vector<HGroup> open;
  uint32_t* mem = memA;
  uint32_t* nxt = memB;
  int64_t n_leaves = 0, staged = 0;
  int depth = 0;
  // Host plan buffers keep their capacity across levels and calls (thread-local): fresh multi-MB vectors per
  // level cost ~4 ms of page faults at C5 depth 1 (99k children), with the GPU idle behind the read-back.
  // (bound to local references: the planning threads must see the calling thread's vectors)
  static thread_local std::vector<LeafJob> tl_jobs;
  static thread_local std::vector<LeafPart> tl_parts;
  static thread_local std::vector<int64_t> tl_leaf_dst, tl_coff;
  static thread_local std::vector<uint32_t> tl_hccnt, tl_hlead;
  std::vector<LeafJob>& jobs = tl_jobs;
  std::vector<LeafPart>& parts = tl_parts;
  std::vector<int64_t>&h_leaf_dst = tl_leaf_dst, &coff = tl_coff;
  std::vector<uint32_t>&hccnt = tl_hccnt, &hlead = tl_hlead;
  jobs.clear();
  parts.clear();
  h_leaf_dst.clear();

  auto flush_jobs = [&](const uint32_t* src) -> pipnn_status {
    if (jobs.empty()) return PIPNN_OK;
    if ((int64_t)jobs.size() > cp.J || (int64_t)parts.size() > cp.J) return fail(PIPNN_ECAPACITY, "partition: job capacity");
    g_pin_jobs.reset();  // its previous copies completed at the last synchronisation
    PIPNN_CUDA(g_pin_jobs.copy(d_jobs, jobs.data(), jobs.size() * sizeof(LeafJob), st));
    PIPNN_CUDA(g_pin_jobs.copy(d_parts, parts.data(), parts.size() * sizeof(LeafPart), st));
    PIPNN_CUDA(g_pin_jobs.flush(st));
    leaf_job_kernel<<<(unsigned)jobs.size(), 256, 0, st>>>(d_jobs, (int)jobs.size(), d_parts, src, staging, leaf_size);
    PIPNN_LAUNCHED("leaf_job_kernel", st);
    // (host->device copies from pageable memory have consumed jobs/parts when they return)
    jobs.clear();
    parts.clear();
    return PIPNN_OK;
  };
  auto add_leaf = [&](std::initializer_list<LeafPart> ps, int64_t upper) {
    LeafJob J;
    J.dst = staged;
    J.leaf = n_leaves;
    J.part0 = (int32_t)parts.size();
    J.nparts = (int32_t)ps.size();
    for (const LeafPart& q : ps) parts.push_back(q);
    jobs.push_back(J);
    h_leaf_dst.push_back(staged);
    staged += upper;
    ++n_leaves;
  };

  for (int r = 0; r < reps; ++r) {
    if (n <= p->c_max) add_leaf({LeafPart{(int64_t)r * n, (int32_t)n, 0}}, n);  // line 1: base case
    else open.push_back(HGroup{(int64_t)r * n, n, mix64(mix64(p->seed, kDomPart), (uint64_t)r)});
  }
  PIPNN_TRY(flush_jobs(memA));

  static const bool dbg_timing = [] {
    const char* e = std::getenv("PIPNN_DEBUG_TIMING");
    return e && e[0] == '1';
  }();
  auto wall = [] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  // Device subtrees of level L run after level L + 1's kernels and read-back are enqueued: the host waits on an
  // event behind the read-back, so the subtree kernel overlaps the host's planning of level L + 1. Stream order
  // keeps their member buffer intact (level L + 1 writes the other buffer; level L + 2 is enqueued after it).
  struct PendingSubtree {
    bool on = false;
    int ng = 0;
    const uint32_t* mem = nullptr;
  } pend;
  auto launch_pending = [&]() -> pipnn_status {
    if (!pend.on) return PIPNN_OK;
    pend.on = false;
    PIPNN_CUDA(kmemset(dev_work, 0, sizeof(int), st));
    return subtree_launch(X, p, dev_groups, pend.ng, pend.mem, staging, 2 * cp.L, dev_ctr + 1, dev_leaf_dst,
                          dev_leaf_size, cp.leaves, dev_ctr, dev_work, c.err, dev_work + 1, st);
  };
  cudaEvent_t ev_sync = level_sync_event();
  if (!ev_sync) return fail(PIPNN_ECUDA, "partition: sync event");
  while (!open.empty()) {
    const int G = (int)open.size();
    if (G > cp.G) return fail(PIPNN_ECAPACITY, "partition: open-group capacity");
    const double t_level0 = dbg_timing ? wall() : 0.0;
    double t_sync0 = 0.0, t_sync1 = 0.0;
    // ---- host plan of the level
    std::vector<PGroup> hg(G);
    std::vector<int64_t> cb(G);
    int64_t M = 0, C = 0, Q = 0;
    int fmax_l = 1;
    for (int g = 0; g < G; ++g) {
      PGroup& q = hg[g];
      q.key = open[g].key;
      q.off = open[g].off;
      q.size = open[g].size;
      q.cbase = M;
      cb[g] = M;
      q.l = (int32_t)leaders_of(q.size, p);
      const int fan = depth < p->n_fanout ? p->fanout[depth] : 1;
      q.f = std::min(fan, q.l);
      fmax_l = std::max(fmax_l, q.f);
      q.lead_off = C;
      q.pair_off = Q;
      // filter threshold: expected 4 l + 64 candidates; no filter when that is most of the group
      const double want = 4.0 * q.l + 64.0;
      if (want >= 0.5 * (double)q.size) q.thr = ~0ull;
      else q.thr = (uint64_t)(want / (double)q.size * 18446744073709551615.0);
      M += q.size;
      C += q.l;
      Q += q.size * q.f;
    }
    if (C > cp.C || Q > cp.L || M > cp.L) return fail(PIPNN_ECAPACITY, "partition: level capacity");
    (void)fmax;
    // ---- 1. leaders: capacity-bounded filter by priority, sort each group's candidates by (priority, id)
    // [the candidate keys are distinct: mix(K, .) is injective], first l_g, then sorted by id. A group whose
    // filter kept more than its capacity or fewer than l_g candidates makes the whole level run again
    // without the filter (checked at the level's single host synchronisation below).
    std::vector<int64_t> cand_seg(G + 1, 0), lead_seg(G + 1, 0);
    bool redo_unfiltered = false;
  level_again:
    g_pin_level.reset();  // the previous level's (or attempt's) copies completed at its synchronisation
    for (int g = 0; g < G; ++g) {
      PGroup& q = hg[g];
      if (redo_unfiltered) q.thr = ~0ull;
      const int64_t cap = q.thr == ~0ull ? q.size : std::min<int64_t>(q.size, 8 * (int64_t)q.l + 256);
      q.cap = (int32_t)cap;
      q.cand_off = cand_seg[g];
      cand_seg[g + 1] = cand_seg[g] + cap;
      lead_seg[g + 1] = lead_seg[g] + q.l;
    }
    const int64_t NC = cand_seg[G];
    PIPNN_CUDA(g_pin_level.copy(d_groups, hg.data(), G * sizeof(PGroup), st));
    PIPNN_CUDA(g_pin_level.copy(d_cbase, cb.data(), G * sizeof(int64_t), st));
    PIPNN_CUDA(g_pin_level.copy(d_cand_seg, cand_seg.data(), (G + 1) * sizeof(int64_t), st));
    PIPNN_CUDA(g_pin_level.copy(d_lead_seg, lead_seg.data(), (G + 1) * sizeof(int64_t), st));
    PIPNN_CUDA(g_pin_level.flush(st));
    PIPNN_CUDA(kmemset(d_cnt, 0, G * sizeof(uint32_t), st));
    PIPNN_CUDA(kmemset(d_redo, 0, sizeof(int), st));
    PIPNN_CUDA(kmemset(ck, 0xFF, NC * sizeof(uint64_t), st));
    prio_kernel<<<(unsigned)std::min<int64_t>(ceil_div(M, 256), num_sms() * 64), 256, 0, st>>>(
        d_groups, d_cbase, G, M, mem, d_cnt, ck, cv, d_redo);
    PIPNN_LAUNCHED("prio_kernel", st);
    prio_check_kernel<<<(unsigned)ceil_div(G, 256), 256, 0, st>>>(d_groups, G, d_cnt, d_redo);
    PIPNN_LAUNCHED("prio_check_kernel", st);
    const double t_prio = dbg_timing ? wall() : 0.0;
    size_t tb = cub_bytes;
    int max_cap = 0;
    for (int g = 0; g < G; ++g) max_cap = std::max(max_cap, hg[g].cap);
    if (max_cap <= kLeadSortMax) {
      // hand-written: one CTA per group (the common case; no library sort, no host synchronisation)
      int max_l = 2;
      for (int g = 0; g < G; ++g) max_l = std::max(max_l, hg[g].l);
      int np = 2;
      while (np < max_l) np <<= 1;
      const int smem = kLeadSmall * 12 + 4096 * 4 + 32 * 4 + np * 4;
      if (smem > 200 * 1024) return fail(PIPNN_EUNSUPPORTED, "partition: leader count too large");
      PIPNN_CUDA(cudaFuncSetAttribute(leaders_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      leaders_kernel<<<G, 1024, smem, st>>>(d_groups, G, ck, cv, lead_sorted);
      PIPNN_LAUNCHED("leaders_kernel", st);
    } else if (G == 1) {
      // (a group whose filter was dropped, redo_unfiltered: every member is a candidate)
      PIPNN_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, ck, ck2, cv, cv2, (int)NC, 0, 64, st));
    } else {
      PIPNN_CUDA(cub::DeviceSegmentedSort::SortPairs(cub_tmp, tb, ck, ck2, cv, cv2, (int)NC, G, d_cand_seg,
                                                     d_cand_seg + 1, st));
    }
    if (max_cap > kLeadSortMax) {
      take_leaders_kernel<<<G, 128, 0, st>>>(d_groups, G, cv2, lead);
      PIPNN_LAUNCHED("take_leaders_kernel", st);
      tb = cub_bytes;
      if (G == 1) {
        PIPNN_CUDA(cub::DeviceRadixSort::SortKeys(cub_tmp, tb, lead, lead_sorted, (int)C, 0, 32, st));
      } else {
        PIPNN_CUDA(cub::DeviceSegmentedSort::SortKeys(cub_tmp, tb, lead, lead_sorted, (int)C, G, d_lead_seg,
                                                      d_lead_seg + 1, st));
      }
    }
    const double t_leaders = dbg_timing ? wall() : 0.0;
    // ---- 2. nearest f_g leaders of every member (tcgen05 distance tiles + top-f), written directly as
    // (child = lead_off + leader index, member id) pairs with the child histogram
    std::vector<TileSeg> hA(G), hB(G);
    std::vector<DistSeg> hD(G);
    std::vector<int64_t> hOffA(G + 1), hOffB(G + 1);  // item offsets: one item per 128-row block
    std::vector<int64_t> hOffP(G + 1);                 // pair-item offsets: one per two 128-row blocks
    int64_t posA = 0, posB = 0, nP = 0;
    for (int g = 0; g < G; ++g) {
      const PGroup& q = hg[g];
      TileSeg a{q.off, posA, (int32_t)round_up(q.size, 128), (int32_t)q.size};
      TileSeg b{q.lead_off, posB, (int32_t)round_up(q.l, 128), q.l};
      hOffA[g] = posA / 128;
      hOffB[g] = posB / 128;
      hOffP[g] = nP;
      nP += (a.pad / 128 + 1) / 2;
      posA += a.pad;
      posB += b.pad;
      hA[g] = a;
      hB[g] = b;
      DistSeg d;
      d.a = a;
      d.b = b;
      d.out_off = q.pair_off;
      d.k = q.f;
      d.self = 0;
      d.ostride = q.f;
      d.pad_ = 0;
      hD[g] = d;
    }
    if (posA > cp.rowsA || posB > cp.rowsB) return fail(PIPNN_ECAPACITY, "partition: tiled capacity");
    const int64_t nItA = posA / 128, nItB = posB / 128;
    hOffA[G] = nItA;
    hOffB[G] = nItB;
    hOffP[G] = nP;
    const int64_t nits[2] = {nItA, nItB};
    PIPNN_CUDA(g_pin_level.copy(tsA, hA.data(), G * sizeof(TileSeg), st));
    PIPNN_CUDA(g_pin_level.copy(tsB, hB.data(), G * sizeof(TileSeg), st));
    PIPNN_CUDA(g_pin_level.copy(dsegs, hD.data(), G * sizeof(DistSeg), st));
    PIPNN_CUDA(g_pin_level.copy(d_itoff, hOffA.data(), (G + 1) * sizeof(int64_t), st));
    PIPNN_CUDA(g_pin_level.copy(d_itoff + (G + 1), hOffB.data(), (G + 1) * sizeof(int64_t), st));
    PIPNN_CUDA(g_pin_level.copy(n_it, nits, 2 * sizeof(int64_t), st));
    PIPNN_CUDA(g_pin_level.flush(st));
    // uint8 with fanout <= 2 at this level: leader norms in the packed form of the single-pass top-2
    static const bool no_packed = std::getenv("PIPNN_NO_PACKED") != nullptr;  // experiment hook
    const int packed = X->dtype == PIPNN_U8 && fmax_l <= 2 && !no_packed ? 1 : 0;
    const bool pairs = packed && dt_packed_pairs(Kb);  // the packed pass runs on dist_topk_uf2_kernel (pair items)
    if (pairs) {
      PIPNN_CUDA(g_pin_level.copy(d_poff, hOffP.data(), (G + 1) * sizeof(int64_t), st));
      PIPNN_CUDA(g_pin_level.copy(n_pairs, &nP, sizeof(int64_t), st));
      PIPNN_CUDA(g_pin_level.flush(st));
    }
    level_items_kernel<<<G, 256, 0, st>>>(d_itoff, d_itoff + (G + 1), G, itA, itB, pairs ? d_poff : nullptr,
                                          pairs ? itP : nullptr);
    PIPNN_LAUNCHED("level_items_kernel", st);
    const double t_plan2 = dbg_timing ? wall() : 0.0;
    PIPNN_TRY(gather_tiled(X, mem, tsA, itA, n_it, nItA, TA, nA, c));
    PIPNN_TRY(gather_tiled(X, lead_sorted, tsB, itB, n_it + 1, nItB, TB, nB, c, 0, packed));
    const double t_gather = dbg_timing ? wall() : 0.0;
    PIPNN_CUDA(kmemset(ccnt, 0, C * sizeof(uint32_t), st));
    DistTopkArgs da{};
    da.Ta = TA;
    da.Tb = TB;
    da.na = nA;
    da.nb = nB;
    da.Kb = Kb;
    da.segs = dsegs;
    da.items = itA;
    da.n_items = n_it;
    da.col_ids = iota;   // leader index j of group g -> child id lead_off + j
    da.out_idx = pk;
    da.out_dist = nullptr;
    da.row_ids = mem;    // member ids
    da.out_rowid = cv2;
    da.out_cnt = ccnt;
    da.packed = packed;
    da.err = c.err;
    if (pairs) {
      // dist_topk_uf2_kernel over the pair items, static round-robin schedule (a device claim per item measured
      // slower here: the packed epilogue is light, so the claim latency is exposed)
      da.items = itP;
      da.n_items = n_pairs;
      da.pairs = 1;
    }
    PIPNN_TRY(launch_dist_topk(da, X->dtype == PIPNN_U8, X->metric == PIPNN_MIPS, fmax_l, st));
    const double t_dist = dbg_timing ? wall() : 0.0;
    // ---- 3. group-by: stable radix sort of the (child, id) pairs, in member order -> every child ascending
    tb = cub_bytes;
    PIPNN_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, pk, pk2, cv2, nxt, (int)Q, 0, bits_for(C), st));
    // ---- 4. host merge plan (the level's one synchronisation)
    // (pinned read-back: the three copies stay asynchronous, one synchronisation)
    // one batched read-back (child counts, sorted leaders, redo flag) into pinned scratch; its descriptors
    // sit behind the data in the same mapped buffer
    const size_t hb_data = ((2 * C + 1) * sizeof(uint32_t) + 15) & ~(size_t)15;
    uint8_t* hraw = pinned_scratch(hb_data + 3 * sizeof(KCopyDesc));
    if (!hraw) return fail(PIPNN_ECUDA, "pinned host scratch");
    uint32_t* hbuf = reinterpret_cast<uint32_t*>(hraw);
    KCopyDesc* hd = reinterpret_cast<KCopyDesc*>(hraw + hb_data);
    hd[0] = KCopyDesc{hbuf, ccnt, (unsigned long long)(C * sizeof(uint32_t))};
    hd[1] = KCopyDesc{hbuf + C, lead_sorted, (unsigned long long)(C * sizeof(uint32_t))};
    hd[2] = KCopyDesc{hbuf + 2 * C, d_redo, (unsigned long long)sizeof(int)};
    PIPNN_CUDA(kcopy_batch(hd, 3, st));
    PIPNN_CUDA(cudaEventRecord(ev_sync, st));
    PIPNN_TRY(launch_pending());  // the previous level's device subtrees (see PendingSubtree)
    // the caller's independent work (pipnn_build: sketches), once, behind the read-back of the level with the
    // longest host plan, so that it fills the GPU's idle time there: depth 0 (<= leader_cap children), or depth 1
    // when that level is expected to have many more children (C5: ~98k, 2.7 ms of planning with the GPU otherwise
    // idle; C2: ~4k, where depth 0 measured better). A partition that ends first leaves it to the caller.
    const bool side_later = depth == 0 && (double)Q * (double)p->p_samp_num / (double)std::max<int64_t>(1, p->p_samp_den) >= 32768.0;
    if (!side_later && c.side_work && *c.side_work) {
      std::function<pipnn_status()> fn;
      fn.swap(*c.side_work);
      PIPNN_TRY(fn());
    }
    if (dbg_timing) t_sync0 = wall();
    PIPNN_CUDA(cudaEventSynchronize(ev_sync));
    if (dbg_timing) t_sync1 = wall();
    hccnt.assign(hbuf, hbuf + C);
    hlead.assign(hbuf + C, hbuf + 2 * C);
    const int hredo = (int)hbuf[2 * C];
    if (hredo) {
      if (redo_unfiltered) return fail(PIPNN_ECUDA, "partition: leader selection failed without filter");
      redo_unfiltered = true;  // exceedingly rare: every member becomes a leader candidate
      goto level_again;
    }
    coff.assign(C + 1, 0);
    for (int64_t j = 0; j < C; ++j) coff[j + 1] = coff[j] + hccnt[j];
    std::vector<HGroup> next;
    // The groups' merge plans are independent: levels with many groups (C5 depth 1: 990 groups, ~100 children
    // each, 4.3 ms on one core with the GPU idle behind the read-back) plan them on a few host threads; the
    // leaves, jobs and next-level groups are then emitted in group order as before.
    const double t_copy = dbg_timing ? wall() : 0.0;
    std::vector<HMerge> plans(G);
    std::atomic<int> next_g{0};
    auto plan_groups = [&]() {  // groups are claimed from a counter: any number of started threads completes them
      std::vector<int64_t> sz;
      std::vector<std::pair<uint64_t, uint32_t>> mk;
      for (int g; (g = next_g.fetch_add(1, std::memory_order_relaxed)) < G;) {
        const PGroup& q = hg[g];
        sz.resize(q.l);
        mk.resize(q.l);
        const uint64_t KM = q.key ^ kDomMerge;
        for (int j = 0; j < q.l; ++j) {
          sz[j] = hccnt[q.lead_off + j];
          const uint32_t lid = hlead[q.lead_off + j];
          mk[j] = {mix64(KM, lid), lid};
        }
        plans[g] = merge_plan(sz, mk, p->c_min, p->c_max);
      }
    };
    {
      const int hw = (int)std::thread::hardware_concurrency();
      const int nt = std::max(1, std::min({8, hw > 1 ? hw - 1 : 1, G / 64}));
      std::vector<std::thread> th;
      for (int t = 1; t < nt; ++t) {
        try {
          th.emplace_back(plan_groups);
        } catch (...) {  // no thread available: the calling thread plans the rest
          break;
        }
      }
      plan_groups();
      for (auto& t : th) t.join();
    }
    const double t_planned = dbg_timing ? wall() : 0.0;
    for (int g = 0; g < G; ++g) {
      const PGroup& q = hg[g];
      const HMerge& mp = plans[g];
      auto sz = [&](int j) -> int64_t { return hccnt[q.lead_off + j]; };
      auto part_of = [&](int j) { return LeafPart{coff[q.lead_off + j], (int32_t)sz(j), 0}; };
      for (int j : mp.big) {
        if (j == mp.absorb) {
          int64_t upper = sz(j);
          LeafJob J;
          J.dst = staged;
          J.leaf = n_leaves;
          J.part0 = (int32_t)parts.size();
          J.nparts = 1 + (int32_t)mp.leftover.size();
          parts.push_back(part_of(j));
          for (int s : mp.leftover) {
            parts.push_back(part_of(s));
            upper += sz(s);
          }
          jobs.push_back(J);
          h_leaf_dst.push_back(staged);
          staged += upper;
          ++n_leaves;
          continue;
        }
        if (sz(j) <= p->c_max) {
          add_leaf({part_of(j)}, sz(j));
        } else if (sz(j) == q.size || depth + 1 >= 64) {
          // degenerate-input guard: ceil(|g|/C_max) near-equal chunks by ascending id
          const int64_t nc = ceil_div(sz(j), p->c_max);
          for (int64_t t = 0; t < nc; ++t) {
            const int64_t lo = t * sz(j) / nc, hi = (t + 1) * sz(j) / nc;
            add_leaf({LeafPart{coff[q.lead_off + j] + lo, (int32_t)(hi - lo), 0}}, hi - lo);
          }
        } else {
          next.push_back(HGroup{coff[q.lead_off + j], sz(j), mix64(q.key, (uint64_t)hlead[q.lead_off + j] + 1)});
        }
      }
      for (auto& bin : mp.bins) {
        LeafJob J;
        J.dst = staged;
        J.leaf = n_leaves;
        J.part0 = (int32_t)parts.size();
        J.nparts = (int32_t)bin.size();
        int64_t upper = 0;
        for (int s : bin) {
          parts.push_back(part_of(s));
          upper += sz(s);
        }
        jobs.push_back(J);
        h_leaf_dst.push_back(staged);
        staged += upper;
        ++n_leaves;
      }
    }
    if (staged > cp.L || n_leaves > cp.leaves - 1) return fail(PIPNN_ECAPACITY, "partition: leaf capacity");
    const double t_merge = dbg_timing ? wall() : 0.0;
    PIPNN_TRY(flush_jobs(nxt));
    const double t_flush = dbg_timing ? wall() : 0.0;
    if (use_subtree && !next.empty() && depth + 1 >= subtree_min_depth) {
      std::vector<DevGroup> dg;
      std::vector<HGroup> keep;
      for (const HGroup& h : next) {
        if (subtree_fits(X, p, h.size, depth + 1)) dg.push_back(DevGroup{h.off, (int32_t)h.size, depth + 1, h.key});
        else keep.push_back(h);
      }
      if (!dg.empty()) {
        // largest subproblems first (the CTAs take groups in this order): the longest serial subtrees start early
        std::stable_sort(dg.begin(), dg.end(), [](const DevGroup& a, const DevGroup& b) { return a.size > b.size; });
        // the members live in `nxt`, which the level after next overwrites: stream order runs this first
        PIPNN_CUDA(g_pin_jobs.copy(dev_groups, dg.data(), dg.size() * sizeof(DevGroup), st));
        PIPNN_CUDA(g_pin_jobs.flush(st));
        pend.on = true;  // launched behind the next level's read-back (or after the loop)
        pend.ng = (int)dg.size();
        pend.mem = nxt;
        next.swap(keep);
      }
    }
    if (dbg_timing)
      std::fprintf(stderr, "[pipnn] depth %d: groups %d members %lld | enqueue %.0f us (prio %.0f leaders %.0f plan %.0f gather %.0f dist %.0f sort %.0f), wait %.0f us, host plan %.0f us (merge %.0f = copy %.0f + plans %.0f + emit, jobs %.0f)\n",
                   depth, G, (long long)M, t_sync0 - t_level0, t_prio - t_level0, t_leaders - t_prio, t_plan2 - t_leaders,
                   t_gather - t_plan2, t_dist - t_gather, t_sync0 - t_dist, t_sync1 - t_sync0, wall() - t_sync1,
                   t_merge - t_sync1, t_copy - t_sync1, t_planned - t_copy, t_flush - t_merge);
    // next level: subproblems live in `nxt`; ping-pong the member buffers
    open.swap(next);
    std::swap(mem, nxt);
    ++depth;
  }
  PIPNN_TRY(launch_pending());
  // ---- leaves carved on the device follow the host's leaves
  g_pin_level.reset();
  PIPNN_CUDA(g_pin_level.copy(leaf_dst, h_leaf_dst.data(), n_leaves * sizeof(int64_t), st));
  PIPNN_CUDA(g_pin_level.flush(st));
  {
    unsigned long long* hb = reinterpret_cast<unsigned long long*>(pinned_scratch(3 * sizeof(unsigned long long)));
    if (!hb) return fail(PIPNN_ECUDA, "pinned host scratch");
    hb[2] = 0;
    PIPNN_CUDA(kcopy(hb, dev_ctr, 2 * sizeof(unsigned long long), st));
    PIPNN_CUDA(kcopy(&hb[2], dev_work + 1, sizeof(int), st));
    PIPNN_CUDA(cudaStreamSynchronize(st));
    const unsigned long long hc[2] = {hb[0], hb[1]};
    const int hdepth = (int)(hb[2] & 0xFFFFFFFFull);
    const int64_t nd = (int64_t)hc[0];
    if (n_leaves + nd > cp.leaves) return fail(PIPNN_ECAPACITY, "partition: leaf capacity (device subtrees)");
    if (nd > 0) {
      PIPNN_CUDA(kcopy(leaf_size + n_leaves, dev_leaf_size, nd * sizeof(int64_t), st));
      PIPNN_CUDA(kcopy(leaf_dst + n_leaves, dev_leaf_dst, nd * sizeof(int64_t), st));
      n_leaves += nd;
    }
    depth = std::max(depth, hdepth);
  }
  // ---- leaf_off = exclusive scan of the leaf sizes; compact the staged leaves into leaf_ids
  PIPNN_CUDA(kmemset(leaf_size + n_leaves, 0, sizeof(int64_t), st));
  size_t tb = cub_bytes;
  PIPNN_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, leaf_size, leaf_off, (int)(n_leaves + 1), st));
  if (n_leaves > 0) {
    leaf_compact_kernel<<<(unsigned)std::min<int64_t>(n_leaves, 65535), 256, 0, st>>>(n_leaves, leaf_dst, leaf_off,
                                                                                         staging, leaf_ids);
    PIPNN_LAUNCHED("leaf_compact_kernel", st);
  }
  *n_leaves_h = n_leaves;
  *depth_h = depth;
  if (c.defer_inst_count) {  // pipnn_build reads leaf_off (and with it the count) right after
    *n_inst_h = -1;
    return PIPNN_OK;
  }
  int64_t* hni = reinterpret_cast<int64_t*>(pinned_scratch(sizeof(int64_t)));
  if (!hni) return fail(PIPNN_ECUDA, "pinned host scratch");
  PIPNN_CUDA(kcopy(hni, leaf_off + n_leaves, sizeof(int64_t), st));
  PIPNN_CUDA(cudaStreamSynchronize(st));
  *n_inst_h = *hni;
  *depth_h = depth;
  return PIPNN_OK;
}

}  // namespace pipnn
