// partition_subtree.cu — Alg. 5 (Randomized Ball Carving) below depth 0, entirely on the device:
// one CTA carves one open subproblem and all of its descendants (depth-first, its own stack in SMEM) with
// the exact rules of the host level loop (partition.cu) and the oracle (R10-R16):
//   leaders     = the l members with the smallest (mix(K, id), id), l = min(cap, max(2, ceil(num |P| / den)), |P|),
//                 sorted by id (a priority-threshold filter keeps ~4 l + 64 candidates; selection by rank);
//   assignment  = each member's nearest leader by (D(x, l), leader id) — fanout 1 below depth 0 — with D the
//                 dataset's measure on the stored rows (uint8: exact integers; float: the bf16 copy, fp32);
//   group-by    = stable counting sort by leader (members stay ascending by id inside every child);
//   merge       = the sibling merge of small children (R15), the base case |child| <= C_max, the degenerate-
//                 input guard (R16), recursion into the other children with key mix(K, leader + 1).
// Merged leaves are the rank-merge of their sorted sibling runs. Leaves are written to the staging area at
// an atomic cursor (leaf order is unspecified; the leaf SET is the exact one). The host loop keeps depth 0 and any subproblem this kernel cannot hold (see subtree_fits).
#include <algorithm>
#include <cub/cub.cuh>

#include "internal.h"

namespace pipnn {

constexpr int kStThreads = 256;
constexpr int kStMaxMembers = 4096;   // ids per ping-pong buffer
constexpr int kStMaxLeaders = 64;
constexpr int kStMaxCand = 512;       // leader-priority candidates
constexpr int kStMaxStack = 256;
constexpr int kStUnion = 4096;        // a merged leaf (<= C_max <= 4096 ids)

struct StGroup {
  int64_t off;  // members mem[off .. off + size), ascending by id
  int32_t size, depth;
  uint64_t key;
};

struct StEntry {
  int32_t a, b;  // range in a ping-pong buffer
  int32_t buf, depth;
  uint64_t key;
};

struct SubtreeArgs {
  const void* X;
  int64_t ld;
  int d, u8, mips;
  int c_max, c_min, p_num, p_den, leader_cap;
  const StGroup* groups;
  int n_groups;
  const uint32_t* mem;
  uint32_t* staging;
  int64_t stage_cap;
  unsigned long long* stage_cursor;
  int64_t* leaf_dst;
  int64_t* leaf_size;
  int64_t leaf_cap;
  unsigned long long* leaf_count;
  int* work;
  int* err;
  int* max_depth;
  int64_t n;  // points (bounds checks)
};

__host__ __device__ inline int st_row_bytes(int d, bool u8) { return u8 ? (d + 15) / 16 * 16 : (d + 7) / 8 * 16; }

__host__ __device__ inline size_t st_smem_bytes(int d, bool u8) {
  return (size_t)2 * kStMaxMembers * 4                     // ping-pong member buffers
         + (size_t)kStMaxMembers                           // assignment (child index per member)
         + (size_t)kStMaxCand * 16                         // candidate (priority, id) + leader scratch
         + (size_t)kStMaxLeaders * st_row_bytes(d, u8)     // leader rows
         + (size_t)kStMaxStack * sizeof(StEntry)           // DFS stack
         + (size_t)kStMaxLeaders * (kStThreads / 32) * 4   // per-warp child counts
         + 8192;                                           // small arrays
}

// Merge-plan actions of one subproblem (thread 0 plans, the CTA executes)
constexpr int kActLeaf = 0;   // leaf = child range [x, y) of dst (a whole child or a guard chunk)
constexpr int kActUnion = 1;  // leaf = sorted union of the children in mask
constexpr int kStMaxAct = 160;

__global__ void __launch_bounds__(kStThreads, 2) subtree_kernel(const SubtreeArgs A) {
  extern __shared__ __align__(16) uint8_t ssm[];
  const bool u8 = A.u8 != 0, mips = A.mips != 0;
  const int rb = st_row_bytes(A.d, u8), nchunk = rb >> 4;
  const int64_t row_stride = u8 ? A.ld : 2 * A.ld;  // bytes
  uint32_t* bufs = (uint32_t*)ssm;                    // [2][kStMaxMembers]
  uint8_t* asg = (uint8_t*)(bufs + 2 * kStMaxMembers);
  uint64_t* ck = (uint64_t*)(asg + kStMaxMembers);
  uint32_t* cv = (uint32_t*)(ck + kStMaxCand);
  uint8_t* lrows = (uint8_t*)(cv + 2 * kStMaxCand);
  StEntry* stack = (StEntry*)(lrows + (size_t)kStMaxLeaders * rb);
  uint32_t* wcnt = (uint32_t*)(stack + kStMaxStack);            // [kStMaxLeaders][nwarps]
  uint32_t* lead = wcnt + kStMaxLeaders * (kStThreads / 32);    // [64] leader ids, ascending
  uint32_t* coff = lead + 64;                                   // [65] child offsets in dst
  int32_t* act_t = (int32_t*)(coff + 72);                       // [kStMaxAct]
  int32_t* act_x = act_t + kStMaxAct;
  int32_t* act_y = act_x + kStMaxAct;
  uint64_t* act_m = (uint64_t*)(act_y + kStMaxAct);             // union member children
  __shared__ int s_g, s_sp, s_ncand, s_nact, s_fail, s_usize;
  __shared__ StEntry s_cur;
  __shared__ unsigned long long s_dst;
  __shared__ int s_leaf_ok;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int nw = kStThreads / 32;

  for (;;) {
    __syncthreads();
    if (tid == 0) {
      s_g = atomicAdd(A.work, 1);
      s_fail = 0;
    }
    __syncthreads();
    const int gi = s_g;
    if (gi >= A.n_groups) break;
    const StGroup G = A.groups[gi];
    if (G.size > kStMaxMembers || G.size < 0) {  // never: the host checks subtree_fits
      if (tid == 0) atomicExch(A.err, 0x100 | DERR_CAPACITY);
      continue;
    }
    for (int i = tid; i < G.size; i += kStThreads) bufs[i] = A.mem[G.off + i];
    if (tid == 0) {
      stack[0] = StEntry{0, G.size, 0, G.depth, G.key};
      s_sp = 1;
    }
    __syncthreads();
    while (true) {
      __syncthreads();
      const bool stop = s_sp == 0 || s_fail;
      __syncthreads();  // every thread has read s_sp / s_fail before thread 0 pops (uniform exit)
      if (stop) break;
      if (tid == 0) s_cur = stack[--s_sp];
      __syncthreads();
      const StEntry E = s_cur;
      const int p = E.b - E.a;
      if (tid == 0) atomicMax(A.max_depth, E.depth + 1);
      const uint32_t* src = bufs + E.buf * kStMaxMembers + E.a;
      uint32_t* dst = bufs + (E.buf ^ 1) * kStMaxMembers + E.a;
      // ---- leaders: the l members with the smallest (mix(K, id), id), then sorted by id
      int l = (int)(((int64_t)A.p_num * p + A.p_den - 1) / A.p_den);
      l = min(min(max(l, 2), A.leader_cap), p);
      if (l > kStMaxLeaders) {  // the host only sends groups whose top level fits; children are smaller
        if (tid == 0) {
          atomicExch(A.err, DERR_CAPACITY);
          s_fail = 1;
        }
        continue;
      }
      const double want = 4.0 * l + 64.0;
      unsigned long long thr = want >= 0.5 * p ? ~0ull : (unsigned long long)(want / p * 18446744073709551615.0);
      int ncand = 0;
      for (int attempt = 0; attempt < 40; ++attempt) {
        if (tid == 0) s_ncand = 0;
        __syncthreads();
        for (int i = tid; i < p; i += kStThreads) {
          const uint32_t id = src[i];
          const uint64_t pri = mix64(E.key, id);
          if (thr == ~0ull || pri < thr) {
            const int slot = atomicAdd(&s_ncand, 1);
            if (slot < kStMaxCand) {
              ck[slot] = pri;
              cv[slot] = id;
            }
          }
        }
        __syncthreads();
        ncand = s_ncand;
        __syncthreads();
        if (ncand >= l && ncand <= kStMaxCand) break;
        if (ncand < l) thr = thr > (~0ull >> 1) ? ~0ull : (thr << 1) | 1ull;  // too few: widen
        else thr >>= 1;                                                     // too many: narrow
      }
      if (ncand < l || ncand > kStMaxCand) {
        if (tid == 0) {
          atomicExch(A.err, DERR_CAPACITY);
          s_fail = 1;
        }
        continue;
      }
      // rank selection (keys are distinct): candidate q is a leader iff fewer than l candidates precede it;
      // the leaders' ranks by id give their sorted position — two barriers, no sorting network
      for (int q = tid; q < ncand; q += kStThreads) {
        const uint64_t kq = ck[q];
        int r = 0;
        for (int t = 0; t < ncand; ++t) r += ck[t] < kq;
        if (r < l) cv[kStMaxCand + r] = cv[q];  // (second half of cv: the l leaders, by priority rank)
      }
      __syncthreads();
      if (tid < l) {
        const uint32_t me = cv[kStMaxCand + tid];
        int r = 0;
        for (int t = 0; t < l; ++t) r += cv[kStMaxCand + t] < me;
        lead[r] = me;
      }
      __syncthreads();
      if (tid < l && lead[tid] >= (uint64_t)A.n) {
        atomicExch(A.err, 0x200 | DERR_CAPACITY);
        s_fail = 1;
      }
      __syncthreads();
      if (s_fail) continue;
      for (int e = tid; e < l * nchunk; e += kStThreads) {
        const int j = e / nchunk, c = e - j * nchunk;
        ((uint4*)(lrows + (size_t)j * rb))[c] = __ldg((const uint4*)((const uint8_t*)A.X + (int64_t)lead[j] * row_stride) + c);
      }
      for (int e = tid; e < kStMaxLeaders * nw; e += kStThreads) wcnt[e] = 0;
      __syncthreads();
      // ---- nearest leader of every member by (D, leader id); warp w owns the contiguous slice [w0, w1)
      const int per_w = (p + nw - 1) / nw;
      const int w0 = min(p, warp * per_w), w1 = min(p, w0 + per_w);
      for (int i = w0 + lane; i < w1; i += 32) {
        const uint4* xr = (const uint4*)((const uint8_t*)A.X + (int64_t)src[i] * row_stride);
        int best = 0;
        // leaders in blocks of 8: every 16-B chunk of the member row is loaded once per block (all loads of
        // a block independent), 8 partial sums in registers; ties keep the smaller leader index (= id)
        uint32_t bdu = 0xFFFFFFFFu;
        float bdf = 0.0f;
        for (int j0 = 0; j0 < l; j0 += 8) {
          uint32_t au[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
          float af[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          // the member row in batches of 4 chunks, the batch's loads issued together (latency-bound otherwise)
          for (int c0 = 0; c0 < nchunk; c0 += 4) {
          uint4 xs[4];
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (c0 + t < nchunk) xs[t] = __ldg(xr + c0 + t);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            if (c0 + t >= nchunk) break;
            const int c = c0 + t;
            const uint4 x = xs[t];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              if (j0 + jj < l) {
                const uint4 y = ((const uint4*)(lrows + (size_t)(j0 + jj) * rb))[c];
                if (u8) {
                  uint32_t df = __vabsdiffu4(x.x, y.x);
                  au[jj] = __dp4a(df, df, au[jj]);
                  df = __vabsdiffu4(x.y, y.y);
                  au[jj] = __dp4a(df, df, au[jj]);
                  df = __vabsdiffu4(x.z, y.z);
                  au[jj] = __dp4a(df, df, au[jj]);
                  df = __vabsdiffu4(x.w, y.w);
                  au[jj] = __dp4a(df, df, au[jj]);
                } else {
                  const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, yw[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                  for (int t = 0; t < 4; ++t) {
                    const float x0 = __uint_as_float(xw[t] << 16), x1 = __uint_as_float(xw[t] & 0xFFFF0000u);
                    const float y0 = __uint_as_float(yw[t] << 16), y1 = __uint_as_float(yw[t] & 0xFFFF0000u);
                    if (mips) {
                      af[jj] = fmaf(x0, y0, af[jj]);
                      af[jj] = fmaf(x1, y1, af[jj]);
                    } else {
                      af[jj] = fmaf(x0 - y0, x0 - y0, af[jj]);
                      af[jj] = fmaf(x1 - y1, x1 - y1, af[jj]);
                    }
                  }
                }
              }
            }
          }
          }
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            if (j0 + jj >= l) break;
            if (u8) {
              if (au[jj] < bdu) {
                bdu = au[jj];
                best = j0 + jj;
              }
            } else {
              const float D = mips ? -af[jj] : af[jj];
              if (j0 + jj == 0 || D < bdf) {
                bdf = D;
                best = j0 + jj;
              }
            }
          }
        }
        asg[i] = (uint8_t)best;
        atomicAdd(&wcnt[best * nw + warp], 1u);
      }
      __syncthreads();
      if (tid == 0) {  // exclusive offsets, child-major then warp
        uint32_t run = 0;
        for (int j = 0; j < l; ++j) {
          coff[j] = run;
          for (int w = 0; w < nw; ++w) {
            const uint32_t cnt = wcnt[j * nw + w];
            wcnt[j * nw + w] = run;
            run += cnt;
          }
        }
        coff[l] = run;
      }
      __syncthreads();
      // ---- stable scatter (every warp walks its slice in order; members stay ascending inside a child)
      for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        const int ch = i < w1 ? (int)asg[i] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, ch);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        uint32_t pos = 0;
        if (ch >= 0) pos = wcnt[ch * nw + warp] + rank;
        __syncwarp();
        if (ch >= 0) {
          dst[pos] = src[i];
          if (rank == 0) wcnt[ch * nw + warp] += (uint32_t)__popc(peers);
        }
        __syncwarp();
      }
      __syncthreads();
      // ---- merge plan (thread 0): the same rule as partition.cu merge_plan / the oracle (R15)
      if (tid == 0) {
        int nact = 0;
        int small[kStMaxLeaders], ns = 0;
        uint64_t skey[kStMaxLeaders];
        const uint64_t KM = E.key ^ kDomMerge;
        for (int j = 0; j < l; ++j) {
          const int sz = (int)(coff[j + 1] - coff[j]);
          if (sz > 0 && sz < A.c_min) {
            const uint64_t kj = mix64(KM, lead[j]);
            int q = ns++;
            while (q > 0 && (skey[q - 1] > kj || (skey[q - 1] == kj && lead[small[q - 1]] > lead[j]))) {
              skey[q] = skey[q - 1];
              small[q] = small[q - 1];
              --q;
            }
            skey[q] = kj;
            small[q] = j;
          }
        }
        // bins of small children in key order, closed when their size sum reaches C_min
        uint64_t bins[kStMaxLeaders];
        int nb = 0;
        uint64_t cur = 0;
        int64_t sum = 0;
        for (int q = 0; q < ns; ++q) {
          const int j = small[q];
          cur |= 1ull << j;
          sum += coff[j + 1] - coff[j];
          if (sum >= A.c_min) {
            bins[nb++] = cur;
            cur = 0;
            sum = 0;
          }
        }
        int absorb = -1;
        uint64_t leftover = 0;
        if (cur) {
          if (nb > 0) {
            bins[0] |= cur;
          } else {
            for (int j = 0; j < l; ++j) {
              const int64_t sz = coff[j + 1] - coff[j];
              if (sz < A.c_min) continue;  // big children only
              if (sz + sum > A.c_max) continue;
              if (absorb < 0) {
                absorb = j;
                continue;
              }
              const int64_t sa = coff[absorb + 1] - coff[absorb];
              const uint64_t kj = mix64(KM, lead[j]), ka = mix64(KM, lead[absorb]);
              if (sz < sa || (sz == sa && (kj < ka || (kj == ka && lead[j] < lead[absorb])))) absorb = j;
            }
            if (absorb < 0) bins[nb++] = cur;
            else leftover = cur;
          }
        }
        for (int j = 0; j < l && !s_fail; ++j) {
          const int64_t sz = coff[j + 1] - coff[j];
          if (sz < A.c_min) continue;
          if (j == absorb) {
            act_t[nact] = kActUnion;
            act_m[nact++] = leftover | (1ull << j);
          } else if (sz <= A.c_max) {
            act_t[nact] = kActLeaf;
            act_x[nact] = (int)coff[j];
            act_y[nact++] = (int)coff[j + 1];
          } else if (sz == p || E.depth + 1 >= 64) {
            const int64_t nc = (sz + A.c_max - 1) / A.c_max;  // degenerate-input guard (R16)
            for (int64_t t = 0; t < nc; ++t) {
              if (nact >= kStMaxAct) break;
              act_t[nact] = kActLeaf;
              act_x[nact] = (int)(coff[j] + t * sz / nc);
              act_y[nact++] = (int)(coff[j] + (t + 1) * sz / nc);
            }
          } else {
            if (s_sp >= kStMaxStack) {
              atomicExch(A.err, DERR_CAPACITY);
              s_fail = 1;
              break;
            }
            stack[s_sp++] = StEntry{E.a + (int)coff[j], E.a + (int)coff[j + 1], E.buf ^ 1, E.depth + 1,
                                    mix64(E.key, (uint64_t)lead[j] + 1)};
          }
          if (nact >= kStMaxAct - kStMaxLeaders) {
            atomicExch(A.err, DERR_CAPACITY);
            s_fail = 1;
          }
        }
        for (int b = 0; b < nb; ++b) {
          act_t[nact] = kActUnion;
          act_m[nact++] = bins[b];
        }
        s_nact = nact;
      }
      __syncthreads();
      // ---- execute the leaf actions (merged leaves are built in the subproblem's source range, free now
      // that its members are scattered into dst; a merged leaf never holds more than the subproblem)
      uint32_t* uni = bufs + E.buf * kStMaxMembers + E.a;
      const int nact = s_nact;
      __syncthreads();  // every thread has read the action count
      for (int a = 0; a < nact; ++a) {
        int size = 0;
        if (act_t[a] == kActLeaf) {
          size = act_y[a] - act_x[a];
        } else {
          // concatenate the member children (disjoint: fanout 1), then sort ascending
          if (tid == 0) {
            int tot = 0;
            for (int j = 0; j < l; ++j)
              if (act_m[a] >> j & 1ull) tot += (int)(coff[j + 1] - coff[j]);
            s_usize = tot;
          }
          __syncthreads();
          size = s_usize;
          // merge of the sorted, disjoint child runs: output position of x from run r = its index in r +
          // the number of elements below x in every other run (binary searches), one barrier
          for (int j = 0; j < l; ++j) {
            if (!(act_m[a] >> j & 1ull)) continue;
            const int c0 = (int)coff[j], c1 = (int)coff[j + 1];
            for (int i = tid; i < c1 - c0; i += kStThreads) {
              const uint32_t x = dst[c0 + i];
              int pos = i;
              for (int q = 0; q < l; ++q) {
                if (q == j || !(act_m[a] >> q & 1ull)) continue;
                int lo = (int)coff[q], hi = (int)coff[q + 1];
                while (lo < hi) {
                  const int mid = (lo + hi) >> 1;
                  if (dst[mid] < x) lo = mid + 1;
                  else hi = mid;
                }
                pos += lo - (int)coff[q];
              }
              uni[pos] = x;
            }
          }
          __syncthreads();
        }
        if (tid == 0) {
          s_leaf_ok = 0;
          const unsigned long long d0 = atomicAdd(A.stage_cursor, (unsigned long long)size);
          const unsigned long long li = atomicAdd(A.leaf_count, 1ull);
          if ((int64_t)(d0 + size) <= A.stage_cap && (int64_t)li < A.leaf_cap) {
            A.leaf_dst[li] = (int64_t)d0;
            A.leaf_size[li] = size;
            s_dst = d0;
            s_leaf_ok = 1;
          } else {
            atomicExch(A.err, DERR_CAPACITY);
          }
        }
        __syncthreads();
        if (s_leaf_ok) {
          const uint32_t* from = act_t[a] == kActLeaf ? dst + act_x[a] : uni;
          for (int i = tid; i < size; i += kStThreads) {
            const uint32_t v = from[i];
            if (v >= (uint64_t)A.n) atomicExch(A.err, 0x300 | DERR_CAPACITY);
            A.staging[s_dst + i] = v;
          }
        }
        __syncthreads();
      }
      if (tid == 0) s_nact = 0;
    }
  }
}

// Device subtree carving of the host-selected subproblems (see subtree_fits). The leaf counter and the staging
// cursor continue from the host loop's values; leaves are appended at leaf_dst / leaf_size.
bool subtree_fits(const pipnn_points* X, const pipnn_partition_params* p, int64_t size, int depth) {
  if (size > kStMaxMembers) return false;
  const bool u8 = X->dtype == PIPNN_U8;
  if (!u8 && X->dtype != kDtypeBf16) return false;
  if (u8 && ((X->d & 15) || (X->ld & 15))) return false;
  // the subtree kernel computes member -> leader distances on CUDA cores: only for short rows (uint8 d <= 256,
  // bf16 d <= 128); longer rows (e.g. C4, d = 200 float) measured faster through the batched tcgen05 levels
  if (st_row_bytes(X->d, u8) > 256) return false;
  for (int t = depth; t < p->n_fanout; ++t)
    if (p->fanout[t] != 1) return false;  // fanout > 1 below depth 0: host loop
  int64_t l = ((int64_t)p->p_samp_num * size + p->p_samp_den - 1) / p->p_samp_den;
  l = std::min<int64_t>(std::min<int64_t>(std::max<int64_t>(l, 2), p->leader_cap), size);
  if (l > kStMaxLeaders) return false;
  if (p->c_max > kStUnion) return false;
  return true;
}

size_t subtree_smem(const pipnn_points* X) { return st_smem_bytes(X->d, X->dtype == PIPNN_U8); }

pipnn_status subtree_launch(const pipnn_points* X, const pipnn_partition_params* p, const void* groups, int n_groups,
                            const uint32_t* mem, uint32_t* staging, int64_t stage_cap, unsigned long long* stage_cursor,
                            int64_t* leaf_dst, int64_t* leaf_size, int64_t leaf_cap, unsigned long long* leaf_count,
                            int* work, int* err, int* max_depth, cudaStream_t st) {
  if (n_groups <= 0) return PIPNN_OK;
  SubtreeArgs a;
  a.X = X->data;
  a.ld = X->ld;
  a.d = X->d;
  a.u8 = X->dtype == PIPNN_U8;
  a.mips = X->metric == PIPNN_MIPS;
  a.c_max = p->c_max;
  a.c_min = p->c_min;
  a.p_num = p->p_samp_num;
  a.p_den = p->p_samp_den;
  a.leader_cap = p->leader_cap;
  a.groups = (const StGroup*)groups;
  a.n_groups = n_groups;
  a.mem = mem;
  a.staging = staging;
  a.stage_cap = stage_cap;
  a.stage_cursor = stage_cursor;
  a.leaf_dst = leaf_dst;
  a.leaf_size = leaf_size;
  a.leaf_cap = leaf_cap;
  a.leaf_count = leaf_count;
  a.work = work;
  a.err = err;
  a.max_depth = max_depth;
  a.n = X->n;
  const size_t smem = subtree_smem(X);
  PIPNN_CUDA(cudaFuncSetAttribute(subtree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  subtree_kernel<<<(unsigned)std::min(n_groups, 3 * num_sms()), kStThreads, smem, st>>>(a);
  PIPNN_LAUNCHED("subtree_kernel", st);
  return PIPNN_OK;
}

size_t subtree_group_bytes() { return sizeof(StGroup); }

}  // namespace pipnn
