// search.cu — batched greedy beam search over the built graph (Alg. 1 BeamSearch, P:176-207;
// SURVEY §8(f) NEXT-1), one warp per query:
//   beam B = the L best (D, id) seen so far, kept sorted in SMEM as 64-bit keys (ordered D << 32 | id), with a
//   visited flag each; visited set V = an open-addressing SMEM hash of the expanded points.
//   Repeat: expand the first unvisited element p of B (ballot over the flags); every out-neighbour v of p
//   (a lane each) is skipped if v is in V or in B — membership in B is a binary search for v's exact key, D
//   being a deterministic function of (q, v) — otherwise its key joins a candidate list; the candidates are
//   sorted in registers (warp bitonic) and merged into B (each lane computes its output positions by a
//   co-rank search), keeping the first L. Stop when every element of B is visited; answer = B's first k.
// Same rules as the oracle harness (oracle/pipnn_oracle.cpp or_beam_search): (D, id) beam order, only
// neighbours neither visited nor in the beam are added. uint8 distances are exact integers; float
// distances are fp32 from the fp32 rows (the oracle's are fp64, so float results agree up to near-ties).
#include <cstdint>

#include "internal.h"

namespace pipnn {

constexpr int kSrchWarps = 4;        // queries (warps) per CTA
constexpr int kSrchHash = 4096;      // visited-set slots per query (power of two)
constexpr int kSrchMaxL = 256;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t ord_key(int32_t d) { return (uint32_t)d ^ 0x80000000u; }
__device__ __forceinline__ uint32_t ord_key(float f) {
  const uint32_t b = __float_as_uint(f + 0.0f);
  return b ^ ((b & 0x80000000u) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float unord_f(uint32_t o) {
  return __uint_as_float(o ^ ((o & 0x80000000u) ? 0x80000000u : 0xFFFFFFFFu));
}
__device__ __forceinline__ uint32_t hslot(uint32_t v) { return (v * 2654435761u) >> (32 - 12); }

struct SrchSmem {
  uint64_t beam[2][kSrchMaxL];  // double-buffered sorted beam
  uint8_t vis[2][kSrchMaxL];
  uint64_t cand[256];
  uint32_t hash[kSrchHash];
};

// D(q, row v): uint8 exact squared L2; float squared L2 or -dot (MIPS) in fp32. q in SMEM (16-B chunks).
template <bool U8, bool MIPS>
__device__ __forceinline__ uint32_t row_key(const void* __restrict__ Xv, int64_t ld, int d, const uint4* q, uint32_t v,
                                            float* dout) {
  if (U8) {
    uint32_t acc = 0;
    if ((d & 15) || (ld & 15)) {  // unaligned rows: bytes
      const uint8_t* x = (const uint8_t*)Xv + (int64_t)v * ld;
      const uint8_t* qb = reinterpret_cast<const uint8_t*>(q);
      for (int j = 0; j < d; ++j) {
        const int t = (int)__ldg(x + j) - (int)qb[j];
        acc += (uint32_t)(t * t);
      }
      *dout = (float)acc;
      return ord_key((int32_t)acc);
    }
    const uint4* x = reinterpret_cast<const uint4*>((const uint8_t*)Xv + (int64_t)v * ld);
    for (int c = 0; c < d / 16; ++c) {
      const uint4 a = __ldg(x + c), b = q[c];
      const uint32_t a4[4] = {a.x, a.y, a.z, a.w}, b4[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t ad = __vabsdiffu4(a4[t], b4[t]);
        acc = __dp4a(ad, ad, acc);
      }
    }
    *dout = (float)acc;
    return ord_key((int32_t)acc);
  } else {
    const float* x = (const float*)Xv + (int64_t)v * ld;
    const float* qf = reinterpret_cast<const float*>(q);
    float acc = 0.0f;
    int j = 0;
    if (!(d & 3) && !(ld & 3)) {
      for (; j < d; j += 4) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(x + j));
        const float4 b = *reinterpret_cast<const float4*>(qf + j);
        if (MIPS) {
          acc = fmaf(a.x, b.x, acc); acc = fmaf(a.y, b.y, acc); acc = fmaf(a.z, b.z, acc); acc = fmaf(a.w, b.w, acc);
        } else {
          acc = fmaf(a.x - b.x, a.x - b.x, acc); acc = fmaf(a.y - b.y, a.y - b.y, acc);
          acc = fmaf(a.z - b.z, a.z - b.z, acc); acc = fmaf(a.w - b.w, a.w - b.w, acc);
        }
      }
    }
    for (; j < d; ++j) {
      const float a = __ldg(x + j), b = qf[j];
      if (MIPS) acc = fmaf(a, b, acc);
      else acc = fmaf(a - b, a - b, acc);
    }
    const float D = MIPS ? -acc : acc;
    *dout = D;
    return ord_key(D);
  }
}

template <bool U8, bool MIPS>
__global__ void __launch_bounds__(32 * kSrchWarps) search_kernel(const void* __restrict__ Xv, int64_t ld, int d,
                                                                 const uint64_t* __restrict__ row_ptr,
                                                                 const uint32_t* __restrict__ col_idx,
                                                                 const void* __restrict__ Q, int64_t ldq, int64_t nq,
                                                                 uint32_t entry, int L, int k, int excl,
                                                                 uint32_t* __restrict__ out_ids,
                                                                 float* __restrict__ out_dist,
                                                                 int64_t* __restrict__ n_cmps, int* err) {
  extern __shared__ __align__(16) uint8_t ssm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qbytes = U8 ? ((d + 15) & ~15) : ((4 * d + 15) & ~15);
  SrchSmem& S = *reinterpret_cast<SrchSmem*>(ssm + (size_t)warp * (sizeof(SrchSmem) + qbytes));
  uint4* qs = reinterpret_cast<uint4*>(ssm + (size_t)warp * (sizeof(SrchSmem) + qbytes) + sizeof(SrchSmem));
  int64_t cmps_local = 0;
  for (int64_t qi = (int64_t)blockIdx.x * kSrchWarps + warp; qi < nq; qi += (int64_t)gridDim.x * kSrchWarps) {
    // query row into SMEM (zero padded to 16 B), visited set cleared
    __syncwarp();
    for (int b = lane; b < qbytes / 4; b += 32) {
      uint32_t w = 0;
      if (U8) {
        const uint8_t* src = (const uint8_t*)Q + qi * ldq;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * b + t < d) w |= (uint32_t)src[4 * b + t] << (8 * t);
      } else {
        if (b < d) w = __float_as_uint(((const float*)Q)[qi * ldq + b]);
      }
      reinterpret_cast<uint32_t*>(qs)[b] = w;
    }
    for (int t = lane; t < kSrchHash; t += 32) S.hash[t] = kEmpty;
    __syncwarp();
    float De;
    const uint32_t ke = row_key<U8, MIPS>(Xv, ld, d, qs, entry, &De);
    int cur = 0, nb = 1;
    if (lane == 0) {
      S.beam[0][0] = ((uint64_t)ke << 32) | entry;
      S.vis[0][0] = 0;
    }
    int64_t cmps = 1;
    int n_vis = 0;
    __syncwarp();
    while (true) {
      // first unvisited element of the beam
      int pi = -1;
      for (int b0 = 0; b0 < nb && pi < 0; b0 += 32) {
        const bool un = b0 + lane < nb && !S.vis[cur][b0 + lane];
        const uint32_t bal = __ballot_sync(0xffffffffu, un);
        if (bal) pi = b0 + __ffs(bal) - 1;
      }
      if (pi < 0) break;
      const uint32_t p = (uint32_t)(S.beam[cur][pi] & 0xFFFFFFFFu);
      if (++n_vis > kSrchHash / 2) {  // visited set full: report instead of degrading silently
        if (lane == 0) atomicExch(err, DERR_CAPACITY | 0x400);
        break;
      }
      if (lane == 0) {
        S.vis[cur][pi] = 1;
        uint32_t h = hslot(p);
        while (S.hash[h] != kEmpty) h = (h + 1) & (kSrchHash - 1);
        S.hash[h] = p;
      }
      __syncwarp();
      const uint64_t r0 = row_ptr[p], r1 = row_ptr[p + 1];
      // the row in steps of <= 256 neighbours (S.cand's capacity), each merged into the beam before the next
      // is read: top-L composes, so this equals one merge of the whole row for any out-degree
      for (uint64_t q0 = r0; q0 < r1; q0 += 256) {
      const uint64_t q1 = min(r1, q0 + 256);
      int nc = 0;
      for (uint64_t e0 = q0; e0 < q1; e0 += 32) {
        const bool valid = e0 + lane < q1;
        const uint32_t v = valid ? col_idx[e0 + lane] : kEmpty;
        bool add = valid;
        if (add) {  // visited?
          uint32_t h = hslot(v);
          while (true) {
            const uint32_t s = S.hash[h];
            if (s == v) { add = false; break; }
            if (s == kEmpty) break;
            h = (h + 1) & (kSrchHash - 1);
          }
        }
        uint64_t key = ~0ull;
        if (add) {
          float Dv;
          key = ((uint64_t)row_key<U8, MIPS>(Xv, ld, d, qs, v, &Dv) << 32) | v;
          // in the beam? binary search for the exact key
          int lo = 0, hi = nb;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (S.beam[cur][mid] < key) lo = mid + 1;
            else hi = mid;
          }
          if (lo < nb && S.beam[cur][lo] == key) add = false;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, add);
        if (add) S.cand[nc + __popc(bal & ((1u << lane) - 1u))] = key;
        nc += __popc(bal);
      }
      cmps += nc;
      __syncwarp();
      if (nc == 0) continue;
      if (nc > 64) {  // high-degree point: SMEM bitonic sort of the candidates
        int P2 = 64;
        while (P2 < nc) P2 <<= 1;
        for (int t = nc + lane; t < P2; t += 32) S.cand[t] = ~0ull;
        __syncwarp();
        for (int size = 2; size <= P2; size <<= 1)
          for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < P2; t += 32) {
              const int o = t ^ stride;
              if (o > t) {
                const bool up = (t & size) == 0;
                const uint64_t a = S.cand[t], b = S.cand[o];
                if ((a > b) == up) {
                  S.cand[t] = b;
                  S.cand[o] = a;
                }
              }
            }
            __syncwarp();
          }
      } else {
      // sort the candidates (<= 64) in registers: two per lane, bitonic over 64
      uint64_t c0 = lane < nc ? S.cand[lane] : ~0ull, c1 = lane + 32 < nc ? S.cand[lane + 32] : ~0ull;
#pragma unroll
      for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          if (stride == 32) {
            const bool up = (lane & size) == 0;  // size == 64: ascending
            const uint64_t mn = c0 < c1 ? c0 : c1, mx = c0 < c1 ? c1 : c0;
            c0 = up ? mn : mx;
            c1 = up ? mx : mn;
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint64_t& c = h ? c1 : c0;
              const int idx = lane + 32 * h;
              const uint64_t o = __shfl_xor_sync(0xffffffffu, c, stride);
              const bool up = (idx & size) == 0, lower = (lane & stride) == 0;
              const uint64_t mn = o < c ? o : c, mx = o < c ? c : o;
              c = (lower == up) ? mn : mx;
            }
          }
        }
      }
      __syncwarp();
      S.cand[lane] = c0;
      S.cand[lane + 32] = c1;
      __syncwarp();
      }
      // merge beam (nb, flags) and candidates (nc, unvisited) -> first min(L, nb + nc) into the other buffer
      const int nt = min(L, nb + nc), nxt = cur ^ 1;
      for (int t = lane; t < nt; t += 32) {
        // co-rank: i from the beam, t - i from the candidates, beam first on equal keys (never equal: distinct)
        int lo = max(0, t + 1 - nc), hi = min(t + 1, nb);
        while (lo < hi) {  // the number of beam elements among the first t + 1
          const int i = (lo + hi) >> 1;
          // take i + 1 beam elements iff beam[i] < cand[t - i]
          const uint64_t a = S.beam[cur][i], b = (t - i) < nc ? S.cand[t - i] : ~0ull;
          if (a < b) lo = i + 1;
          else hi = i;
        }
        const int i = lo;  // beam elements among the first t + 1 outputs
        const int j = t + 1 - i;
        // output t is the larger of beam[i - 1] and cand[j - 1]
        const uint64_t a = i > 0 ? S.beam[cur][i - 1] : 0ull, b = j > 0 ? S.cand[j - 1] : 0ull;
        if (i > 0 && (j == 0 || a > b)) {
          S.beam[nxt][t] = a;
          S.vis[nxt][t] = S.vis[cur][i - 1];
        } else {
          S.beam[nxt][t] = b;
          S.vis[nxt][t] = 0;
        }
      }
      __syncwarp();
      cur = nxt;
      nb = nt;
      }
    }
    // answer: the beam's first k (excluding the query's own id for the k-NN-graph task)
    int pself = nb;
    if (excl) {
      for (int b0 = 0; b0 < nb; b0 += 32) {
        const bool me = b0 + lane < nb && (uint32_t)(S.beam[cur][b0 + lane] & 0xFFFFFFFFu) == (uint32_t)qi;
        const uint32_t bal = __ballot_sync(0xffffffffu, me);
        if (bal && pself == nb) pself = b0 + __ffs(bal) - 1;
      }
    }
    const int nav = nb - (pself < nb ? 1 : 0);
    for (int t = lane; t < k; t += 32) {
      const bool ok = t < nav;
      const int src = t + (t >= pself ? 1 : 0);
      const uint64_t key = ok ? S.beam[cur][src] : ~0ull;
      out_ids[qi * k + t] = ok ? (uint32_t)(key & 0xFFFFFFFFu) : kEmpty;
      if (out_dist) {
        float D = __int_as_float(0x7F800000);
        if (ok) {
          const uint32_t o = (uint32_t)(key >> 32);
          D = U8 ? (float)(int32_t)(o ^ 0x80000000u) : unord_f(o);
        }
        out_dist[qi * k + t] = D;
      }
    }
    cmps_local += cmps;
  }
  if (n_cmps && lane == 0) atomicAdd((unsigned long long*)n_cmps, (unsigned long long)cmps_local);
}

size_t search_smem_per_warp(const pipnn_points* X) {
  const int qbytes = X->dtype == PIPNN_U8 ? ((X->d + 15) & ~15) : ((4 * X->d + 15) & ~15);
  return sizeof(SrchSmem) + qbytes;
}

pipnn_status search_impl(const pipnn_points* X, const uint64_t* row_ptr, const uint32_t* col_idx, const void* Q,
                         int64_t ldq, int64_t nq, uint32_t entry, int L, int k, int excl, uint32_t* out_ids,
                         float* out_dist, int64_t* n_cmps_dev, const Ctx& c) {
  if (nq == 0) return PIPNN_OK;
  const size_t smem = kSrchWarps * search_smem_per_warp(X);
  const int64_t blocks = std::min<int64_t>(ceil_div(nq, kSrchWarps), (int64_t)num_sms() * 16);
#define SR_LAUNCH(U, M)                                                                                            \
  do {                                                                                                             \
    PIPNN_CUDA(cudaFuncSetAttribute(search_kernel<U, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    search_kernel<U, M><<<(unsigned)blocks, 32 * kSrchWarps, smem, c.st>>>(X->data, X->ld, X->d, row_ptr, col_idx,  \
                                                                          Q, ldq, nq, entry, L, k, excl, out_ids,   \
                                                                          out_dist, n_cmps_dev, c.err);             \
  } while (0)
  if (X->dtype == PIPNN_U8) SR_LAUNCH(true, false);
  else if (X->metric == PIPNN_MIPS) SR_LAUNCH(false, true);
  else SR_LAUNCH(false, false);
#undef SR_LAUNCH
  PIPNN_LAUNCHED("search_kernel", c.st);
  return PIPNN_OK;
}

}  // namespace pipnn
