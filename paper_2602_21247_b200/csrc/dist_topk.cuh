// dist_topk.cuh — the distance-tile kernel of the PiPNN build path (§4.2 "Leaf Building",
// P:558-565, and the nearest-leader step of Alg. 5): for every segment s (a leaf, or a
// partition subproblem against its leaders) and every row i of s, the k columns j with the smallest
//     D(i,j) = ||x_i||^2 + ||y_j||^2 - 2 x_i.y_j   (squared L2)      or   D(i,j) = -x_i.y_j   (MIPS)
// by (D, j), with j = i excluded when A and B are the same segment (self exclusion by id).
// Rows are ranked by a key that differs from D by a per-row constant:
//     uint8 L2 : key = ||y_j||^2 - 2 x_i.y_j                    (int32, exact)
//     float L2 : key = ||y_j||^2/2 - x_i.y_j  (= (D - ||x_i||^2)/2, computed by the MMA itself)
//     MIPS     : key = -x_i.y_j                                   (computed by the MMA itself)
// Output D = ||x_i||^2 + key (u8), max(0, ||x_i||^2 + 2 key) (float L2), key (MIPS).
//
// Blackwell mapping:
//   * persistent grid, one CTA per SM, 6 warps: warp 0 = bulk-copy producer, warp 1 = tcgen05.mma
//     issuer (+ TMEM owner), warps 2-5 = epilogue (warp w reads TMEM lanes 32*(w%4)..+31 = its rows);
//   * work item = (segment, 128-row block); the A block (128 rows x K) stays in SMEM for the item, B
//     column tiles of <= 256 rows (multiple of 32) stream through a 4-stage ring of 32 KB K-chunks;
//   * operands in the K-major SWIZZLE_NONE canonical layout, produced directly by the gather kernel
//     ("tiled rows": [K/16][rows][16 B] per segment), so each K-chunk plane is one contiguous bulk copy;
//   * uint8: tcgen05.mma kind::i8 (u8 x u8 -> s32, exact). float: kind::f16 (bf16 x bf16 -> f32) with the
//     B operand negated (instruction-descriptor bit) and one extra K-step that adds the column term
//     ||y||^2/2 (split over three bf16 values; padding rows carry +1e30): A-side ones come from a
//     constant SMEM tile, so the epilogue does no arithmetic per element — compare and (rarely) insert;
//   * accumulators: two 128x256 32-bit TMEM buffers (all 512 columns) so the MMA of tile t+1 overlaps
//     the epilogue of tile t; each row's running top-(k+1) lives in SMEM with its threshold in a register;
//     the distance tile is never written to memory.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>
#include "common.cuh"
#include "ptx.cuh"

namespace pipnn {

// A segment of gathered rows in a tiled buffer.
struct TileSeg {
  int64_t id_off;  // ids[id_off + i] is the point id of local row i
  int64_t pos;     // first row position in the tiled buffer / norm array (multiple of 128)
  int32_t pad;     // padded row count (multiple of 128): the plane stride of the [K/16][pad][16] layout
  int32_t rows;    // valid rows
};

struct DistSeg {
  TileSeg a;        // rows (queries of the row-wise top-k)
  TileSeg b;        // columns (candidates)
  int64_t out_off;  // output element offset of local row 0; row i writes [out_off + i*ostride, +ostride)
  int32_t k;        // picks per row (<= ostride); remaining slots of the row are padded
  int32_t self;     // 1: exclude column == row (A and B are the same segment)
  int32_t ostride;  // output slots per row
  int32_t pad_;
};

struct WorkItem {
  int32_t seg;
  int32_t rb;  // 128-row block index within the segment
};

struct DistTopkArgs {
  const uint8_t* Ta;
  const uint8_t* Tb;
  const void* na;  // per-position squared norms of A rows (int32 for uint8, float otherwise)
  const void* nb;  // per-position squared norms of B rows (uint8 only; padding rows hold kPadNormU8)
  int Kb;          // bytes per row in the tiled buffers (multiple of 32, <= 512), augment K-step included
  const DistSeg* segs;
  const WorkItem* items;
  const int64_t* n_items;  // device scalar
  const uint32_t* col_ids; // nullable: output id of column j = col_ids[b.id_off + j], else j
  uint32_t* out_idx;       // output picks (column ids), layout given by DistSeg::out_off / ostride
  float* out_dist;         // output D, same layout, nullable
  int* err;
};

constexpr int kDtMaxStages = 4;
constexpr int kDtStageBytes = 256 * 128;  // 256 rows x 128 B of K
constexpr int kDtThreads = 192;
constexpr int kTopkMax = 16;              // max entries of a row's running list (k+1 with self exclusion)
constexpr int kQCap = 64;                 // per-row candidate queue (SMEM) between drains
constexpr int32_t kPadNormU8 = 0x3FFFFFFF; // norm of a padding row: key far above any real key
constexpr float kPadKey = 1e30f;           // float: column term of a padding row

__host__ __device__ constexpr int dt_fixed_smem(int Kb) { return 128 * Kb + 4096 /*ones*/ + kQCap * 128 * 8 /*queues*/; }
__host__ __device__ constexpr int dt_stages(int Kb) {
  return (227 * 1024 - 2048 - dt_fixed_smem(Kb)) / kDtStageBytes >= kDtMaxStages
             ? kDtMaxStages
             : (227 * 1024 - 2048 - dt_fixed_smem(Kb)) / kDtStageBytes;
}
__host__ __device__ constexpr int dt_smem_bytes(int Kb) { return dt_fixed_smem(Kb) + dt_stages(Kb) * kDtStageBytes; }

// Register top-K list (sorted ascending by (key, col)); insert requires key < kk[K-1] for the runtime K.
template <typename KT, int KMAX>
__device__ __forceinline__ void topk_insert(KT (&kk)[KMAX], uint32_t (&ii)[KMAX], KT key, uint32_t col) {
#pragma unroll
  for (int t = KMAX - 1; t >= 0; --t) {
    if (t > 0 && key < kk[t - 1]) {
      kk[t] = kk[t - 1];
      ii[t] = ii[t - 1];
    } else if (key < kk[t]) {
      kk[t] = key;
      ii[t] = col;
    }
  }
}
template <typename KT, int KMAX>
__device__ __forceinline__ KT topk_kth(const KT (&kk)[KMAX], int K) {
  KT r = kk[0];
#pragma unroll
  for (int t = 1; t < KMAX; ++t)
    if (t == K - 1) r = kk[t];
  return r;
}

// Drain a row's SMEM candidate queue (stride 128 words) into its register list.
template <typename KT, int KMAX>
__device__ __forceinline__ void topk_drain(KT (&kk)[KMAX], uint32_t (&ii)[KMAX], KT& thr, int& qlen,
                                           const KT* qk, const uint32_t* qc, int K) {
  for (int e = 0; e < qlen; ++e) {
    const KT key = qk[e * 128];
    if (key < thr) {
      topk_insert<KT, KMAX>(kk, ii, key, qc[e * 128]);
      thr = topk_kth<KT, KMAX>(kk, K);
    }
  }
  qlen = 0;
}

template <bool U8, bool MIPS, int KMAX>
__global__ void __launch_bounds__(kDtThreads, 1) dist_topk_kernel(const DistTopkArgs args) {
  using KT = typename std::conditional<U8, int32_t, float>::type;
  constexpr bool kFold = !U8;  // float paths fold the column term into an augmented MMA K-step
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_a_full, bar_a_empty;
  __shared__ __align__(8) uint64_t bar_b_full[kDtMaxStages], bar_b_empty[kDtMaxStages];
  __shared__ __align__(8) uint64_t bar_acc_full[2], bar_acc_empty[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Kb = args.Kb;
  const int KC = Kb >> 4;                   // 16-B K planes per row (incl. the 2 augment planes for float)
  const int KCm = kFold ? KC - 2 : KC;      // planes of the coordinates themselves
  const int nchunks = (KC + 7) >> 3;
  const int NS = dt_stages(Kb);
  uint8_t* sA = smem;
  uint8_t* sOnes = smem + 128 * Kb;
  KT* q_key = reinterpret_cast<KT*>(sOnes + 4096);                  // [kQCap][128]
  uint32_t* q_col = reinterpret_cast<uint32_t*>(q_key + kQCap * 128);  // [kQCap][128]
  uint8_t* sB = reinterpret_cast<uint8_t*>(q_col + kQCap * 128);    // NS stages of 32 KB

  if (kFold) {
    // constant A-side augment tile, [2 planes][128 rows][16 B]: row = (1, 1, 1, 0, ...) in bf16
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
      const int plane = e >> 9, r = (e >> 2) & 127, w = e & 3;
      reinterpret_cast<uint32_t*>(sOnes)[(plane * 128 + r) * 4 + w] =
          (plane == 0 && w == 0) ? 0x3F803F80u : ((plane == 0 && w == 1) ? 0x00003F80u : 0u);
    }
    ptx::fence_proxy_async_smem();
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_a_full, 1);
    ptx::mbar_init(&bar_a_empty, 1);
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&bar_b_full[s], 1);
      ptx::mbar_init(&bar_b_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&bar_acc_full[b], 1);
      ptx::mbar_init(&bar_acc_empty[b], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(&tmem_base_sh, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int64_t n_items = *args.n_items;

  if (warp == 0) {
    // ------------------------------------------------------------ producer (one lane)
    if (lane == 0) [&]() {
      uint32_t g = 0;
      int64_t i = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x, ++i) {
        const WorkItem w = args.items[it];
        const DistSeg S = args.segs[w.seg];
        const int r0 = w.rb * 128;
        if (!ptx::mbar_wait(&bar_a_empty, (uint32_t)(i & 1) ^ 1u, args.err, DERR_WAIT_TIMEOUT)) return;
        ptx::mbar_arrive_expect_tx(&bar_a_full, 2048u * KCm);
        const uint8_t* srcA = args.Ta + S.a.pos * Kb + (int64_t)r0 * 16;
        for (int kc = 0; kc < KCm; ++kc)
          ptx::bulk_g2s(sA + kc * 2048, srcA + (int64_t)kc * S.a.pad * 16, 2048, &bar_a_full);
        const int ncols = S.b.rows;
        const uint8_t* baseB = args.Tb + S.b.pos * Kb;
        for (int c0 = 0; c0 < ncols; c0 += 256) {
          const int Nt = min(256, (ncols - c0 + 31) & ~31);
          for (int ch = 0; ch < nchunks; ++ch, ++g) {
            const int s = g % NS;
            const uint32_t ph = (g / NS) & 1;
            if (!ptx::mbar_wait(&bar_b_empty[s], ph ^ 1u, args.err, DERR_WAIT_TIMEOUT)) return;
            const int kc0 = ch * 8, kc1 = min(KC, kc0 + 8);
            ptx::mbar_arrive_expect_tx(&bar_b_full[s], (uint32_t)((kc1 - kc0) * Nt * 16));
            uint8_t* dst = sB + s * kDtStageBytes;
            for (int kc = kc0; kc < kc1; ++kc)
              ptx::bulk_g2s(dst + (kc - kc0) * Nt * 16, baseB + ((int64_t)kc * S.b.pad + c0) * 16, Nt * 16,
                            &bar_b_full[s]);
          }
        }
      }
    }();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (one lane)
    if (lane == 0) [&]() {
      uint32_t g = 0, tcount = 0;
      int64_t i = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x, ++i) {
        const WorkItem w = args.items[it];
        const int ncols = args.segs[w.seg].b.rows;
        if (!ptx::mbar_wait(&bar_a_full, (uint32_t)(i & 1), args.err, DERR_WAIT_TIMEOUT)) return;
        ptx::tc_fence_after();
        for (int c0 = 0; c0 < ncols; c0 += 256, ++tcount) {
          const int Nt = min(256, (ncols - c0 + 31) & ~31);
          const uint32_t buf = tcount & 1, use = tcount >> 1;
          if (!ptx::mbar_wait(&bar_acc_empty[buf], (use & 1) ^ 1u, args.err, DERR_WAIT_TIMEOUT)) return;
          ptx::tc_fence_after();
          // float: negate B (bit 14), so the accumulator is -x.y + (column term)
          const uint32_t idesc = U8 ? ptx::idesc_u8_s32(128, Nt) : (ptx::idesc_bf16_f32(128, Nt) | (1u << 14));
          const uint32_t dtm = tmem + buf * 256;
          for (int ch = 0; ch < nchunks; ++ch, ++g) {
            const int s = g % NS;
            const uint32_t ph = (g / NS) & 1;
            if (!ptx::mbar_wait(&bar_b_full[s], ph, args.err, DERR_WAIT_TIMEOUT)) return;
            ptx::tc_fence_after();
            const int kc0 = ch * 8, kc1 = min(KC, kc0 + 8);
            const uint8_t* sb = sB + s * kDtStageBytes;
            for (int kc = kc0; kc < kc1; kc += 2) {
              const uint8_t* a_src = (kFold && kc >= KCm) ? sOnes + (kc - KCm) * 2048 : sA + kc * 2048;
              const uint64_t ad = ptx::smem_desc_kmajor_noswz(ptx::smem_u32(a_src), 2048, 128);
              const uint64_t bd =
                  ptx::smem_desc_kmajor_noswz(ptx::smem_u32(sb + (kc - kc0) * Nt * 16), (uint32_t)Nt * 16, 128);
              const uint32_t acc = (ch > 0 || kc > kc0) ? 1u : 0u;
              if (U8) ptx::mma_i8(dtm, ad, bd, idesc, acc);
              else ptx::mma_bf16(dtm, ad, bd, idesc, acc);
            }
            ptx::mma_commit(&bar_b_empty[s]);
          }
          ptx::mma_commit(&bar_acc_full[buf]);
        }
        ptx::mma_commit(&bar_a_empty);
      }
    }();
  } else {
    // ------------------------------------------------------------ epilogue (4 warps, one row per thread)
    // Per element: (u8) key = ||y||^2 - 2 acc, then append to the row's SMEM queue iff key < thr
    // (predicated, no divergence). The queue is drained into the register top-K list — re-checking each
    // entry against the (meanwhile tighter) threshold — whenever any lane of the warp might overflow it,
    // while the list is not yet full, and at the end of the row. Appends happen in ascending column
    // order and insertion is strict, so equal keys keep the smaller column (= smaller id), exactly.
    [&]() {
      const int q = warp & 3;
      const int tid = q * 32 + lane;  // = row within the 128-row block = TMEM lane
      const KT kInf = U8 ? (KT)0x7FFFFFFF : (KT)__int_as_float(0x7F800000);
      KT* my_qk = q_key + tid;
      uint32_t* my_qc = q_col + tid;
      uint32_t tcount = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const WorkItem w = args.items[it];
        const DistSeg S = args.segs[w.seg];
        const int r0 = w.rb * 128;
        const int row = r0 + tid;
        const int K = S.k + (S.self ? 1 : 0);  // self exclusion: keep k+1, drop the row itself afterwards
        const int ncols = S.b.rows;
        KT kk[KMAX];
        uint32_t ii[KMAX];
#pragma unroll
        for (int t = 0; t < KMAX; ++t) {
          kk[t] = kInf;
          ii[t] = 0xFFFFFFFFu;
        }
        KT thr = kInf;
        int qlen = 0;
        const KT* nbp = U8 ? (const KT*)args.nb + S.b.pos : nullptr;
        for (int c0 = 0; c0 < ncols; c0 += 256, ++tcount) {
          const int Nt = min(256, (ncols - c0 + 31) & ~31);
          const uint32_t buf = tcount & 1, use = tcount >> 1;
          if (!ptx::mbar_wait(&bar_acc_full[buf], use & 1, args.err, DERR_WAIT_TIMEOUT)) return;
          ptx::tc_fence_after();
          const uint32_t taddr = tmem + buf * 256 + ((uint32_t)(q * 32) << 16);
          for (int j0 = 0; j0 < Nt; j0 += 32) {
            uint32_t v[32];
            ptx::tmem_ld32(taddr + j0, v);
            const int col0 = c0 + j0;
            int32_t nbv[32];
            if (U8) {
              const int4* p4 = reinterpret_cast<const int4*>(nbp + col0);
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int4 x = __ldg(p4 + u);
                nbv[4 * u + 0] = x.x;
                nbv[4 * u + 1] = x.y;
                nbv[4 * u + 2] = x.z;
                nbv[4 * u + 3] = x.w;
              }
            }
            ptx::tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              KT key;
              if (U8) key = nbv[jj] - 2 * (int32_t)v[jj];
              else key = __uint_as_float(v[jj]);
              if (key < thr) {
                my_qk[qlen * 128] = key;
                my_qc[qlen * 128] = (uint32_t)(col0 + jj);
                ++qlen;
              }
            }
            // warp-uniform drain decision: the queue could overflow on the next chunk, or the list is not
            // full yet (then every chunk drains, which also makes the threshold finite quickly)
            if (__any_sync(0xffffffffu, qlen > kQCap - 32 || (qlen > 0 && thr == kInf)))
              topk_drain<KT, KMAX>(kk, ii, thr, qlen, my_qk, my_qc, K);
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&bar_acc_empty[buf]);
        }
        topk_drain<KT, KMAX>(kk, ii, thr, qlen, my_qk, my_qc, K);
        if (row < S.a.rows) {
          const int64_t obase = S.out_off + (int64_t)row * S.ostride;
          KT na = 0;
          if (!MIPS) na = ((const KT*)args.na)[S.a.pos + row];
          int o = 0;
#pragma unroll
          for (int t = 0; t < KMAX; ++t) {
            const uint32_t col = ii[t];
            const bool take = t < K && o < S.k && col != 0xFFFFFFFFu && col < (uint32_t)ncols &&
                              !(S.self && col == (uint32_t)row);
            if (take) {
              const KT key = kk[t];
              float D;
              if (MIPS) D = (float)key;
              else if (U8) D = (float)(na + key);
              else D = fmaxf(fmaf(2.0f, (float)key, (float)na), 0.0f);
              args.out_idx[obase + o] = args.col_ids ? args.col_ids[S.b.id_off + col] : col;
              if (args.out_dist) args.out_dist[obase + o] = D;
              ++o;
            }
          }
          for (; o < S.ostride; ++o) {
            args.out_idx[obase + o] = 0xFFFFFFFFu;
            if (args.out_dist) args.out_dist[obase + o] = __int_as_float(0x7F800000);
          }
        }
      }
    }();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// Host launcher (dist_topk.cu): picks the instantiation for (dtype, metric).
pipnn_status launch_dist_topk(const DistTopkArgs& a, bool u8, bool mips, int kmax, cudaStream_t st);

}  // namespace pipnn
