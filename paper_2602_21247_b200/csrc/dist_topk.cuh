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
//   * persistent grid, one CTA per SM, 12 warps = two independent pipelines (producer warp g, tcgen05.mma
//     issuer warp 2+g, epilogue warpgroup g = warps 4+4g..7+4g). Work item = (segment, 128-row block); the
//     CTA's items alternate between the two pipelines, so each epilogue thread owns one row of its item for
//     the whole item (its running top-K never leaves registers, no cross-thread merge);
//   * a tile = 128 rows x <= 128 columns; each pipeline has two 128-column TMEM accumulators, so the MMA of
//     a warpgroup's next tile overlaps the epilogue of its current one, and the two pipelines hide each
//     other's latencies without waiting for each other;
//   * every K-chunk (<= 128 B of every row) of a tile's A rows and B rows arrives by 1-D bulk copies (cp.async.bulk, TMA engine) into a 4-stage SMEM ring with mbarrier
//     transaction counts; operands are in the K-major SWIZZLE_NONE canonical layout produced directly by
//     the gather kernel ("tiled rows": [K/16][rows][16 B] per segment), so each plane slice is one copy;
//   * uint8: tcgen05.mma kind::i8 (u8 x u8 -> s32, exact). float: kind::f16 (bf16 x bf16 -> f32) with the
//     B operand negated (instruction-descriptor bit) and one extra K-step that adds the column term
//     ||y||^2/2 (split over three bf16 values; padding rows carry +1e30): A-side ones come from a
//     constant SMEM tile, so the epilogue does no arithmetic per element;
//   * epilogue per 32-column chunk (tcgen05.ld 32x32b.x32, one row per thread): key, compare with the
//     row's threshold (the K-th best so far) into a 32-bit pass mask; if any lane passed, the keys are
//     staged in SMEM and the passing (key, column) pairs appended to the row's SMEM queue; the queue is
//     drained into the sorted register list (insertion) when it could overflow, while the list is not
//     full, and at the row's end. The distance tile is never written to memory.
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
  int32_t pad;     // padded row count (multiple of 128)
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
  uint32_t* out_idx;       // output picks (column ids), layout given by DistSeg::out_off / ostride; nullable
  uint16_t* out_col;       // nullable: the picks' local column indices (same layout; 0xFFFF = none)
  float* out_dist;         // output D, same layout, nullable
  const uint32_t* row_ids; // with out_rowid: id of local row i = row_ids[a.id_off + i]
  uint32_t* out_rowid;     // nullable: the row's id next to every output slot (same layout)
  uint32_t* out_cnt;       // nullable: out_cnt[pick id] += 1 for every valid pick (group-by histogram)
  int p1cap;               // max column tiles of the threshold pass (>= 1)
  int geo;                 // pipeline geometry request: 0 = default (dt_geom), else 16 * NA + planes per chunk
  int packed;              // uint8, K <= 2, no self exclusion (the partition): nb holds 32 ||y||^2 + (pos mod 32)
                           // and every tile goes through one packed pass (no threshold pass)
  int uf_aug;              // folded uint8 leaves (kernel template UF): augment planes per row (2 per 32-B K-step);
                           // na = per-position row base ||x||^2 + 2 R_x (int32), nb = parity bits of ||y||^2 (u32
                           // words, bit p & 31 of word p >> 5); see leaf.cu "folded uint8 rows"
  int dbg;                 // experiment hook (PIPNN_DEBUG_EPI): low bits 1 = epilogue skips all tile processing,
                           // 2 = skips pass 2; bit 64 = wait profile (pipnn_debug_dt_prof)
  int* err;
  // nullable: dynamic item scheduling — each pipeline's producer claims the next item with an atomicAdd on this
  // device counter (zeroed before the launch) and hands it to its MMA warp and epilogue warpgroup through an
  // SMEM ring; nullptr: the static round-robin order (item = CTA + (2 j + pipeline) * grid)
  unsigned long long* work;
  // dist_topk_uf2_kernel only: 1 = items are pair heads (blocks rb, rb + 1), scheduled statically (work == nullptr)
  int pairs;
};

constexpr int kDtItemRing = 8;  // claimed items in flight per pipeline (dynamic scheduling)
constexpr int kDtCopyLanes = 4;  // producer lanes issuing B-tile copies
constexpr int kDtMaxStages = 16;                    // B ring stages (both pipelines)
constexpr int kDtTileN = 128;                       // columns per tile (one TMEM accumulator)
constexpr int kDtThreads = 384;
constexpr int kTopkMax = 16;                        // max K (k, or the partition fanout)
constexpr int kQCap = 16;                           // per-row candidate queue (SMEM) between drains
constexpr int kStgPitch = 36;                       // words per row of the key staging tile
constexpr int32_t kPadNormU8 = 0x3FFFFFFF;          // norm of a padding row: key far above any real key
constexpr float kPadKey = 1e30f;                    // float: column term of a padding row

// dynamic SMEM: A block per warpgroup [2][NA][KCa planes][128 rows][16 B] | B ring [stages][ppc planes] |
//               key staging per warpgroup [128][kStgPitch] | queues key [kQCap][128] + col u16 [kQCap][128] |
//               A-side augment tile (2 planes)
constexpr int kDtStgBytes = 128 * kStgPitch * 4;
constexpr int kDtQBytes = kQCap * 128 * 6;
constexpr int kDtSmemBudget = 227 * 1024 - 1024;
// Plane geometry of a tiled buffer with Kb bytes per row: KCs planes per 128-row block (its stride), of which
// KCm hold coordinates (float: the last 2 are the augment step that folds the column term into the MMA);
// all KCs are multiplied, a tile's planes arriving in nchunks chunks of <= ppc planes.
struct DtGeom {
  int KCs, KCm, KCuse, nchunks, ppc, stage_bytes, KCa, NA, stages, smem;
};
// augp: augment planes at the end of every row (float: 2 = one bf16 K-step; folded uint8: 2 per 32-B K-step), whose
// A side comes from a constant SMEM tile instead of the A block.
__host__ __device__ inline DtGeom dt_geom(int Kb, int augp, int geo = 0) {
  DtGeom g;
  g.KCs = Kb / 16;
  g.KCm = g.KCs - augp;
  g.KCuse = g.KCs;
  const int ppc_req = geo & 15, na_req = geo >> 4;
  g.nchunks = ppc_req ? (g.KCuse + ppc_req - 1) / ppc_req
                      : (g.KCuse + 9) / 10;  // <= 10 planes (160 B of K) per chunk: one chunk per tile up to K = 160 B
  g.ppc = ((g.KCuse + g.nchunks - 1) / g.nchunks + 1) & ~1;
  g.stage_bytes = g.ppc * 2048;
  g.KCa = g.KCm;
  const int rest = 2 * kDtStgBytes + 2 * kDtQBytes + (augp > 2 ? augp : 2) * 2048;
  // 2 A slots per warpgroup (the next item's A block loads while the current item runs) when that still
  // leaves room for 4 B stages, else 1
  g.NA = 2 * 2 * g.KCa * 2048 + rest + 4 * g.stage_bytes <= kDtSmemBudget ? 2 : 1;
  if (na_req) g.NA = na_req;
  const int fixed = 2 * g.NA * g.KCa * 2048 + rest;
  g.stages = (kDtSmemBudget - fixed) / g.stage_bytes;
  if (g.stages > kDtMaxStages) g.stages = kDtMaxStages;
  g.stages &= ~1;
  g.smem = fixed + g.stages * g.stage_bytes;
  return g;
}

// Passes per item: 2 (threshold, then exact picks). A single exact pass through the queue (U = +inf; every
// key of the first chunk passes) measured slower even for the partition's K = 2 (C2: 3.08 vs 2.89 ms
// partition). Segments of <= 32 columns with K <= 4 and no self exclusion (the partition below depth 0: a
// handful of leaders) take a direct single pass instead: all 32 keys of the one chunk go through the
// branch-free (key, column) insertion network.
__host__ __device__ __forceinline__ bool dt_direct(int k, int ncols, int self) { return ncols <= 32 && k <= 4 && !self; }
// Tiles of the threshold pass: the first min(T, p1cap) column tiles (any column subset gives a valid bound).
__host__ __device__ __forceinline__ int dt_p1(int k, int ncols, int self, int p1cap) {
  const int T = (ncols + 127) / 128;
  return dt_direct(k, ncols, self) ? 0 : (T < p1cap ? T : p1cap);
}

// Sorted insertion into a register list (ascending; equal keys keep the earlier entry first).
// Precondition: key < kk[KMAX-1].
template <typename KT, int KMAX>
__device__ __forceinline__ void topk_insert(KT (&kk)[KMAX], uint16_t (&ii)[KMAX], KT key, uint32_t col) {
  bool lt[KMAX];
#pragma unroll
  for (int t = 0; t < KMAX; ++t) lt[t] = key < kk[t];
  // keys: kk'[t] = max(kk[t-1], min(kk[t], key)) (no NaN can occur). The equivalent nested select
  // lt[t-1] ? kk[t-1] : (lt[t] ? key : kk[t]) is miscompiled for float lists by nvcc 12.9 (sm_100a):
  // the last slot keeps its old value (reproduced with a 4-slot standalone kernel).
#pragma unroll
  for (int t = KMAX - 1; t > 0; --t) {
    if (std::is_same<KT, float>::value) kk[t] = (KT)fmaxf((float)kk[t - 1], fminf((float)kk[t], (float)key));
    else kk[t] = max(kk[t - 1], min(kk[t], key));
    ii[t] = lt[t - 1] ? ii[t - 1] : (lt[t] ? (uint16_t)col : ii[t]);
  }
  if (lt[0]) {
    kk[0] = key;
    ii[0] = (uint16_t)col;
  }
}

// Drain a row's SMEM queue (stride 128 entries) into its register list.
template <typename KT, int KMAX>
__device__ __forceinline__ void topk_drain(KT (&kk)[KMAX], uint16_t (&ii)[KMAX], int& qlen, const KT* qk,
                                           const uint16_t* qc) {
  for (int e = 0; e < qlen; ++e) {
    const KT key = qk[e * 128];
    if (key < kk[KMAX - 1]) topk_insert<KT, KMAX>(kk, ii, key, qc[e * 128]);
  }
  qlen = 0;
}

// Pipeline profile (experiment hook, PIPNN_DEBUG_EPI bit 64): clock64 cycles spent in each wait, per role,
// summed over the grid; read and cleared by pipnn_debug_dt_prof (dist_topk.cu).
static __device__ unsigned long long g_dt_prof[16];

// UF (uint8 leaves, L2): the "folded" uint8 rows of leaf.cu — s8 coordinates y - 128 and augment K-steps whose
// s8 digits against constant A-side weights add E_y = 128 sum(y) - ceil(||y||^2/2) (offset), so the int32
// accumulator is acc = x.y - ceil(||y||^2/2) + R_x (R_x per row): larger is nearer, no per-element norm term.
template <bool U8, bool MIPS, int KMAX, bool UF = false>
__global__ void __launch_bounds__(kDtThreads, 1) dist_topk_kernel(const DistTopkArgs args) {
  using KT = typename std::conditional<U8, int32_t, float>::type;
  constexpr bool kFold = !U8;  // float paths fold the column term into an augmented MMA K-step
  constexpr bool kAug = kFold || UF;
  static_assert(!UF || (U8 && !MIPS), "the folded path is uint8 L2");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_full[2][kDtMaxStages / 2], bar_empty[2][kDtMaxStages / 2];
  __shared__ __align__(8) uint64_t bar_a_full[2][2], bar_a_empty[2][2];  // [warpgroup][slot]
  __shared__ __align__(8) uint64_t bar_acc_full[4], bar_acc_empty[4];
  __shared__ __align__(8) uint64_t bar_it_full[2][kDtItemRing], bar_it_empty[2][kDtItemRing];
  __shared__ int64_t item_ring[2][kDtItemRing];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int augp = kFold ? 2 : (UF ? args.uf_aug : 0);
  const DtGeom GM = dt_geom(args.Kb, augp, args.geo);
  const int KCs = GM.KCs;                // planes per 128-row block of the tiled buffers (block stride)
  const int KCm = GM.KCm;                // planes of the coordinates themselves
  const int KCu = GM.KCuse;              // planes multiplied per tile (incl. the augment step when folded)
  const int nchunks = GM.nchunks;        // K-chunks of <= ppc planes per tile
  const int ppc = GM.ppc;
  const int SB = GM.stage_bytes;
  const int NS = GM.stages / 2;          // B stages per warpgroup pipeline
  const int KCa = GM.KCa;                // == KCm: the A planes held in SMEM
  const int NA = GM.NA;                  // A slots per warpgroup
  uint8_t* sA = smem;                    // [2 warpgroups][NA][KCa][128][16]
  uint8_t* ring = sA + 2 * NA * KCa * 2048;  // [2 warpgroups][NS][SB]
  uint8_t* stg_base = ring + GM.stages * SB;
  uint8_t* q_base = stg_base + 2 * kDtStgBytes;
  uint8_t* sOnes = q_base + 2 * kDtQBytes;  // [augp planes][128 rows][16 B] A-side augment

  if (kFold) {
    // constant A-side augment tile: row = (1, 1, 1, 0, ...) in bf16
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
      const int plane = e >> 9, w = e & 3;
      reinterpret_cast<uint32_t*>(sOnes)[e] =
          (plane == 0 && w == 0) ? 0x3F803F80u : ((plane == 0 && w == 1) ? 0x00003F80u : 0u);
    }
    ptx::fence_proxy_async_smem();
  }
  if (UF) {
    // constant A-side augment rows of the folded uint8 layout: s8 weights 127 for every entry but the last
    // (weight 1) of the last plane
    for (int e = threadIdx.x; e < augp * 512; e += blockDim.x) {
      const bool last = (e >> 9) == augp - 1 && (e & 3) == 3;
      reinterpret_cast<uint32_t*>(sOnes)[e] = last ? 0x017F7F7Fu : 0x7F7F7F7Fu;
    }
    ptx::fence_proxy_async_smem();
  }
  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g) {
      for (int s = 0; s < NS; ++s) {
        ptx::mbar_init(&bar_full[g][s], 1);
        ptx::mbar_init(&bar_empty[g][s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        ptx::mbar_init(&bar_a_full[g][a], 1);
        ptx::mbar_init(&bar_a_empty[g][a], 1);
      }
    }
    for (int b = 0; b < 4; ++b) {
      ptx::mbar_init(&bar_acc_full[b], 1);
      ptx::mbar_init(&bar_acc_empty[b], 4);
    }
    for (int g = 0; g < 2; ++g)
      for (int e = 0; e < kDtItemRing; ++e) {
        ptx::mbar_init(&bar_it_full[g][e], 1);
        ptx::mbar_init(&bar_it_empty[g][e], 5);  // the MMA warp + the 4 epilogue warps of the pipeline
      }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(&tmem_base_sh, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int64_t n_items = *args.n_items;
  const bool prof = (args.dbg & 64) != 0;
  const bool dyn = args.work != nullptr;
  // Item sequence of pipeline g: j-th item. Static: CTA + (2 j + g) * grid. Dynamic: claimed by the producer
  // (claim_item), read by the MMA warp and the epilogue warps (take_item); -1 ends the sequence.
  auto claim_item = [&](int g, uint32_t j) -> int64_t {  // producer (one lane)
    if (!dyn) {
      const int64_t it = (int64_t)blockIdx.x + (2 * (int64_t)j + g) * gridDim.x;
      return it < n_items ? it : -1;
    }
    const int e = (int)(j % kDtItemRing);
    if (!ptx::mbar_wait_hint(&bar_it_empty[g][e], ((j / kDtItemRing) & 1) ^ 1u, args.err, DERR_WAIT_TIMEOUT, 1000000u))
      return -1;
    const int64_t it = (int64_t)atomicAdd(args.work, 1ull);
    item_ring[g][e] = it < n_items ? it : -1;
    ptx::mbar_arrive(&bar_it_full[g][e]);  // (release: the ring entry is visible to the waiters)
    return it < n_items ? it : -1;
  };
  auto take_item = [&](int g, uint32_t j, bool arrive) -> int64_t {  // MMA warp / epilogue warps
    if (!dyn) {
      const int64_t it = (int64_t)blockIdx.x + (2 * (int64_t)j + g) * gridDim.x;
      return it < n_items ? it : -1;
    }
    const int e = (int)(j % kDtItemRing);
    if (!ptx::mbar_wait(&bar_it_full[g][e], (j / kDtItemRing) & 1, args.err, DERR_WAIT_TIMEOUT)) return -1;
    const int64_t it = *(volatile int64_t*)&item_ring[g][e];
    __syncwarp();
    if (arrive) ptx::mbar_arrive(&bar_it_empty[g][e]);
    return it;
  };
  unsigned long long pw[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const unsigned long long t_start = clock64();
  // Producer and MMA waits (slots < 8) park in hardware on a try_wait suspend-time hint instead of re-issuing
  // try_wait, which takes issue slots from the epilogue warps of the sub-partition (C2 leaf tiles -1%).
#define PWAIT(slot, bar, par, err, code)                                                  \
  [&]() {                                                                                 \
    const unsigned long long t0_ = prof ? clock64() : 0ull;                               \
    const bool ok_ = (slot) < 8 ? ptx::mbar_wait_hint((bar), (par), (err), (code), 1000000u)  \
                                : ptx::mbar_wait((bar), (par), (err), (code));                \
    if (prof) pw[slot] += clock64() - t0_;                                                \
    return ok_;                                                                           \
  }()

  // Two independent pipelines, one per epilogue warpgroup g: producer warp g, MMA warp 2 + g, TMEM
  // accumulators 2g and 2g + 1, its own A slots and B ring. Warpgroup g takes the CTA's items
  // it = blockIdx.x + (2 j + g) * gridDim.x; every item's column tiles are computed twice (pass 1: threshold,
  // pass 2: exact picks).
  if (warp < 2) {
    // ------------------------------------------------------------ producer of pipeline g
    // Lane 0 claims items and loads A blocks; the B-chunk copies are spread over kDtCopyLanes lanes (ring stage
    // s belongs to lane s % kDtCopyLanes): one thread's bulk copies complete one after another (~0.3-0.4 us each
    // on B200, tools/micro/l2_bulk_bw.cu), several lanes overlap them.
    const int g = warp;
    [&]() {
      uint32_t sg = 0, ia = 0;
      uint8_t* my_ring = ring + g * NS * SB;
      for (uint32_t jj = 0;; ++jj) {
        int64_t it = 0;
        if (lane == 0) it = claim_item(g, jj);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it < 0) break;
        const WorkItem w = args.items[it];
        const DistSeg S = args.segs[w.seg];
        const int T = (S.b.rows + kDtTileN - 1) / kDtTileN;
        bool ok = true;
        // the item's A block stays in SMEM for all of its tiles (both passes); block-major tiled layout:
        // 128-row block j of a segment = KC planes x 2 KB, contiguous
        {
          const int slot = (int)(ia % NA);
          const uint32_t ph = (ia / NA) & 1;
          ++ia;
          if (lane == 0) {
            ok = PWAIT(0, &bar_a_empty[g][slot], ph ^ 1u, args.err, DERR_WAIT_TIMEOUT);
            if (ok) {
              ptx::mbar_arrive_expect_tx(&bar_a_full[g][slot], (uint32_t)(KCa * 2048));
              ptx::bulk_g2s(sA + (g * NA + slot) * KCa * 2048,
                            args.Ta + (S.a.pos / 128 + w.rb) * (int64_t)KCs * 2048, KCa * 2048, &bar_a_full[g][slot]);
            }
          }
        }
        const int p1 = dt_p1(S.k, S.b.rows, S.self, args.p1cap);
        for (int t = 0; t < p1 + T; ++t) {
          const int c0 = (t < p1 ? t : t - p1) * kDtTileN;
          const uint8_t* srcB = args.Tb + (S.b.pos / 128 + c0 / 128) * (int64_t)KCs * 2048;
          for (int ch = 0; ch < nchunks; ++ch, ++sg) {
            // stage s is always filled by lane s % kDtCopyLanes, so each lane waits on its stages in order
            // (a parity wait can never be two phases behind)
            const int s = sg % NS;
            if (s % kDtCopyLanes != lane || !ok) continue;
            const uint32_t ph = (sg / NS) & 1;
            ok = PWAIT(1, &bar_empty[g][s], ph ^ 1u, args.err, DERR_WAIT_TIMEOUT);
            if (!ok) continue;
            const int kc0 = ch * ppc, kc1 = min(KCu, kc0 + ppc);
            ptx::mbar_arrive_expect_tx(&bar_full[g][s], (uint32_t)((kc1 - kc0) * 2048));
            ptx::bulk_g2s(my_ring + s * SB, srcB + (int64_t)kc0 * 2048, (kc1 - kc0) * 2048, &bar_full[g][s]);
          }
        }
        if (!__all_sync(0xffffffffu, ok)) return;
      }
      if (prof && lane == 0) {
        atomicAdd(&g_dt_prof[0], pw[0]);
        atomicAdd(&g_dt_prof[1], pw[1]);
        atomicAdd(&g_dt_prof[2], clock64() - t_start);
      }
    }();
  } else if (warp < 4) {
    // ------------------------------------------------------------ MMA issuer of pipeline g
    // The whole warp runs the loop (converged, so descriptors and counters stay warp-uniform and live in
    // uniform registers); one elected lane issues the tcgen05.mma / commit instructions. Descriptors of
    // consecutive 16-B K planes differ by 2048 B = 128 in the descriptor's address field.
    const int g = warp - 2;
    [&]() {
      uint32_t sg = 0, ia = 0, tc = 0;
      const uint32_t ring_u32 = ptx::smem_u32(ring + g * NS * SB);
      const uint64_t ones_desc = ptx::smem_desc_kmajor_noswz(ptx::smem_u32(sOnes), 2048, 128);
      for (uint32_t jj = 0;; ++jj) {
        const int64_t it = take_item(g, jj, lane == 0);
        if (it < 0) break;
        const unsigned long long ti0 = prof ? clock64() : 0ull;
        const WorkItem w = args.items[it];
        const DistSeg Sg = args.segs[w.seg];
        const int ncols = Sg.b.rows;
        const int T = (ncols + kDtTileN - 1) / kDtTileN;
        const int p1 = dt_p1(Sg.k, ncols, Sg.self, args.p1cap);
        const int NT = p1 + T;
        const int slot = (int)(ia % NA);
        if (prof) pw[7] += clock64() - ti0;
        if (!PWAIT(4, &bar_a_full[g][slot], (ia / NA) & 1, args.err, DERR_WAIT_TIMEOUT)) return;
        ++ia;
        const uint64_t a_desc = ptx::smem_desc_kmajor_noswz(ptx::smem_u32(sA + (g * NA + slot) * KCa * 2048), 2048, 128);
        for (int t = 0; t < NT; ++t, ++tc) {
          const int c0 = (t < p1 ? t : t - p1) * kDtTileN;
          const int Nt = min(kDtTileN, (ncols - c0 + 31) & ~31);
          const uint32_t buf = 2 * g + (tc & 1), use = tc >> 1;
          if (!PWAIT(5, &bar_acc_empty[buf], (use & 1) ^ 1u, args.err, DERR_WAIT_TIMEOUT)) return;
          const unsigned long long tt0 = prof ? clock64() : 0ull;
          const unsigned long long w6 = pw[6];
          ptx::tc_fence_after();
          // float: negate B (bit 14), so the accumulator is -x.y + (column term)
          // folded uint8: A and B signed (s8, bits 7 and 10)
          const uint32_t idesc = UF ? (ptx::idesc_u8_s32(128, Nt) | (1u << 7) | (1u << 10))
                                    : (U8 ? ptx::idesc_u8_s32(128, Nt) : (ptx::idesc_bf16_f32(128, Nt) | (1u << 14)));
          const uint32_t dtm = tmem + buf * kDtTileN;
          for (int ch = 0; ch < nchunks; ++ch, ++sg) {
            const int s = sg % NS;
            if (!PWAIT(6, &bar_full[g][s], (sg / NS) & 1, args.err, DERR_WAIT_TIMEOUT)) return;
            ptx::tc_fence_after();
            const int kc0 = ch * ppc, kc1 = min(KCu, kc0 + ppc);
            const uint64_t b_desc = ptx::smem_desc_kmajor_noswz(ring_u32 + s * SB, 2048, 128);
            const unsigned long long tm0 = prof ? clock64() : 0ull;
            if (ptx::elect_one()) {
              for (int kc = kc0; kc < kc1; kc += 2) {
                const bool augk = kAug && kc >= KCm;
                const uint64_t ad = augk ? ones_desc + (uint64_t)((kc - KCm) * 128) : a_desc + (uint64_t)(kc * 128);
                const uint64_t bd = b_desc + (uint64_t)((kc - kc0) * 128);
                const uint32_t acc = (ch > 0 || kc > kc0) ? 1u : 0u;
                if (U8) ptx::mma_i8(dtm, ad, bd, idesc, acc);
                else ptx::mma_bf16(dtm, ad, bd, idesc, acc);
              }
              ptx::mma_commit(&bar_empty[g][s]);
            }
            __syncwarp();
            if (prof) pw[2] += clock64() - tm0;
          }
          if (ptx::elect_one()) ptx::mma_commit(&bar_acc_full[buf]);
          __syncwarp();
          if (prof) pw[3] += clock64() - tt0 - (pw[6] - w6);
        }
        if (ptx::elect_one()) ptx::mma_commit(&bar_a_empty[g][slot]);  // the item's MMAs issued: free its A
        __syncwarp();
      }
      if (prof && lane == 0) {
        atomicAdd(&g_dt_prof[4], pw[4]);
        atomicAdd(&g_dt_prof[5], pw[5]);
        atomicAdd(&g_dt_prof[6], pw[6]);
        atomicAdd(&g_dt_prof[7], clock64() - t_start);
        atomicAdd(&g_dt_prof[12], pw[3]);
        atomicAdd(&g_dt_prof[14], pw[2]);
        atomicAdd(&g_dt_prof[13], pw[7]);
      }
    }();
  } else {
    // ------------------------------------------------------------ epilogue (2 warpgroups, one row per thread)
    // Pass 1 (threshold): the row's keys in groups of 16 consecutive columns; the K1 = K + self smallest group
    // minima (a sorted value list, min/max network, branch free) are K1 distinct elements, at most one of them
    // the row itself, so U = the K1-th smallest group minimum bounds the K-th smallest key from above.
    // Pass 2 (exact): the same tiles again; a key passes iff key <= U (until the exact list is full) or
    // key < the list's K-th key, so only ~K+2 elements per row reach the (key, column) insertion.
    // Passing keys are staged in SMEM and appended to the row's queue; the queue is drained into the sorted
    // register list when it could overflow and at the row's end. Columns arrive in ascending order and the
    // insertion is strict, so equal keys keep the smaller column (= smaller id).
    [&]() {
      const int ew = warp - 4;             // 0..7
      const int wg = ew >> 2;              // warpgroup = pipeline
      const int q = warp & 3;              // TMEM lane quadrant of this warp (hardware: warp id % 4)
      const int tid = q * 32 + lane;       // row within the 128-row block = TMEM lane
      const KT kInf = U8 ? (KT)0x7FFFFFFF : (KT)__int_as_float(0x7F800000);
      const KT kNegInf = U8 ? (KT)(-0x7FFFFFFF - 1) : (KT)__int_as_float(0xFF800000);
      constexpr int VK = KMAX + 1;         // value list of pass 1: K + self <= KMAX + 1
      uint32_t* stg = reinterpret_cast<uint32_t*>(stg_base + wg * kDtStgBytes) + tid * kStgPitch;
      KT* my_qk = reinterpret_cast<KT*>(q_base + wg * kDtQBytes) + tid;
      uint16_t* my_qc = reinterpret_cast<uint16_t*>(q_base + wg * kDtQBytes + kQCap * 128 * 4) + tid;
      uint32_t tcount = 0;
      for (uint32_t jj = 0;; ++jj) {
        const int64_t it = take_item(wg, jj, lane == 0);
        if (it < 0) break;
        const WorkItem w = args.items[it];
        const DistSeg S = args.segs[w.seg];
        const int r0 = w.rb * 128;
        const int row = r0 + tid;
        // the row's own norm, needed only at the output: loaded now, in flight during the tiles
        const KT na_row = (!MIPS && row < S.a.rows) ? ((const KT*)args.na)[S.a.pos + row] : (KT)0;
        const int K = S.k;
        const int K1 = K + (S.self ? 1 : 0);
        const int ncols = S.b.rows;
        const int T = (ncols + kDtTileN - 1) / kDtTileN;
        KT vk[VK];
#pragma unroll
        for (int t = 0; t < VK; ++t) vk[t] = t < VK - K1 ? kNegInf : kInf;
        // exact list of KMAX slots; the first KMAX-K hold -inf sentinels so that kk[KMAX-1] is the K-th best
        KT kk[KMAX];
        uint16_t ii[KMAX];
#pragma unroll
        for (int t = 0; t < KMAX; ++t) {
          kk[t] = t < KMAX - K ? kNegInf : kInf;
          ii[t] = 0xFFFFu;
        }
        KT U = kInf;
        int qlen = 0;
        const int diag_chunk = S.self ? (r0 + q * 32) : -1;  // column base of this warp's diagonal chunk
        const bool direct = KMAX <= 4 && dt_direct(K, ncols, S.self);
        // packed single pass (KMAX == 2, uint8): q_j = 32 key_j + (j mod 32) = nbp_j - 64 v_j is one IMAD and
        // orders the chunk's columns by (key, column) exactly (|32 key| < 2^30 for d <= 512); the chunk's two
        // smallest by a min/max network on column pairs, then inserted into the row's list
        const bool packedm = KMAX == 2 && U8 && args.packed;
        const int P1 = dt_p1(K, ncols, S.self, args.p1cap);  // tiles of pass 1 (none: direct single pass)
        for (int t2 = 0; t2 < P1 + T; ++t2, ++tcount) {
          const bool pass2 = t2 >= P1;
          const int c0 = (pass2 ? t2 - P1 : t2) * kDtTileN;
          const int Nt = min(kDtTileN, (ncols - c0 + 31) & ~31);
          const uint32_t buf = 2 * wg + (tcount & 1), use = tcount >> 1;
          if (!PWAIT(8, &bar_acc_full[buf], use & 1, args.err, DERR_WAIT_TIMEOUT)) return;
          ptx::tc_fence_after();
          const uint32_t taddr = tmem + buf * kDtTileN + ((uint32_t)(q * 32) << 16);
          if (t2 == P1 && P1 > 0) {
            U = vk[VK - 1];
            if (UF) {
              // vk holds negated group maxima of acc: -U is the K1-th largest, so acc >= -U passes (key_l <=
              // -2 (-U) exactly); no bound yet (fewer than K1 groups): everything passes
              U = U == kInf ? (KT)(1 << 30) : U;
            } else {
              if (U8 && U != kInf) U = U + 1;  // key <= U  <=>  key < U + 1
              if (!U8) U = (KT)nextafterf((float)U, __int_as_float(0x7F800000));
            }
          }
          if ((args.dbg & 15) == 1 || ((args.dbg & 15) == 2 && pass2)) {
          } else if (UF && !pass2) {
            // ---- folded uint8, pass 1: maxima of acc over groups of 16 columns (3-input max), negated into
            // the value list; padding columns (beyond ncols) never win
            for (int j0 = 0; j0 < Nt; j0 += 32) {
              const int valid = min(32, ncols - (c0 + j0));
              uint32_t v[32];
              ptx::tmem_ld32(taddr + j0, v);
              ptx::tmem_ld_wait();
              if (valid < 32) {
#pragma unroll
                for (int jj = 0; jj < 32; ++jj)
                  if (jj >= valid) v[jj] = 0x80000000u;
              }
#pragma unroll
              for (int gq = 0; gq < 2; ++gq) {
                const int32_t* w = reinterpret_cast<const int32_t*>(v) + 16 * gq;
                int32_t g = __vimax3_s32(w[0], w[1], w[2]);
                g = __vimax3_s32(g, w[3], w[4]);
                g = __vimax3_s32(g, w[5], w[6]);
                g = __vimax3_s32(g, w[7], w[8]);
                g = __vimax3_s32(g, w[9], w[10]);
                g = __vimax3_s32(g, w[11], w[12]);
                g = __vimax3_s32(g, w[13], w[14]);
                g = max(g, w[15]);
                const KT gm = (16 * gq < valid) ? (KT)(-g) : kInf;
#pragma unroll
                for (int t = VK - 1; t > 0; --t) vk[t] = max(vk[t - 1], min(vk[t], gm));
                vk[0] = min(vk[0], gm);
              }
            }
          } else if (UF) {
            // ---- folded uint8, pass 2: acc >= tau passes, tau = -U until the exact list is full, then
            // ceil((-kk - 1) / 2) for its K-th key kk (key_l = -2 acc - parity <= kk requires it: conservative,
            // the drain compares exactly); the funnel collects sign(acc - tau) (one IADD each), inverted per chunk
            for (int j0 = 0; j0 < Nt; j0 += 32) {
              const int col0 = c0 + j0;
              const int valid = min(32, ncols - col0);
              uint32_t v[32];
              ptx::tmem_ld32(taddr + j0, v);
              const int32_t kk8 = (int32_t)kk[KMAX - 1];
              const int32_t tau = kk8 != (int32_t)kInf ? ((-kk8) >> 1) : -(int32_t)U;
              ptx::tmem_ld_wait();
              uint32_t m8[4] = {0u, 0u, 0u, 0u};
#pragma unroll
              for (int jj = 7; jj >= 0; --jj) {
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) {
                  const int j = 8 * qd + jj;
                  m8[qd] = __funnelshift_l((uint32_t)((int32_t)v[j] - tau), m8[qd], 1);  // 1: acc < tau
                }
              }
              uint32_t mask = ~(m8[0] | (m8[1] << 8) | (m8[2] << 16) | (m8[3] << 24));
              if (valid < 32) mask &= (1u << valid) - 1u;
              if (col0 == diag_chunk) mask &= ~(1u << lane);  // self exclusion (by id: the diagonal element)
              if (__any_sync(0xffffffffu, mask != 0)) {
                if (__any_sync(0xffffffffu, qlen + __popc(mask) > kQCap)) topk_drain<KT, KMAX>(kk, ii, qlen, my_qk, my_qc);
                const uint32_t pbits = reinterpret_cast<const uint32_t*>(args.nb)[(S.b.pos + col0) >> 5];  // parities
#pragma unroll
                for (int u = 0; u < 8; ++u)
                  *reinterpret_cast<uint4*>(stg + 4 * u) = make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                __syncwarp();
                while (mask) {
                  const int jj = __ffs(mask) - 1;
                  mask &= mask - 1;
                  if (qlen == kQCap) topk_drain<KT, KMAX>(kk, ii, qlen, my_qk, my_qc);
                  my_qk[qlen * 128] = (KT)(-2 * reinterpret_cast<const int32_t*>(stg)[jj] - (int32_t)((pbits >> jj) & 1u));
                  my_qc[qlen * 128] = (uint16_t)(col0 + jj);
                  ++qlen;
                  if (prof) ++pw[2];
                }
                __syncwarp();
              }
            }
          } else if (packedm) {
            for (int j0 = 0; j0 < Nt; j0 += 32) {
              const int col0 = c0 + j0;
              int4 nb4[8];
              const int4* p4 = reinterpret_cast<const int4*>((const int32_t*)args.nb + S.b.pos + col0);
#pragma unroll
              for (int u = 0; u < 8; ++u) nb4[u] = __ldg(p4 + u);
              uint32_t v[32];
              ptx::tmem_ld32(taddr + j0, v);
              ptx::tmem_ld_wait();
              int32_t qv[32];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                qv[4 * u + 0] = nb4[u].x - 64 * (int32_t)v[4 * u + 0];
                qv[4 * u + 1] = nb4[u].y - 64 * (int32_t)v[4 * u + 1];
                qv[4 * u + 2] = nb4[u].z - 64 * (int32_t)v[4 * u + 2];
                qv[4 * u + 3] = nb4[u].w - 64 * (int32_t)v[4 * u + 3];
              }
              int32_t m1 = 0x7FFFFFFF, m2 = 0x7FFFFFFF;
              if (K == 1) {
#pragma unroll
                for (int jj = 0; jj < 32; jj += 2) m1 = min(m1, min(qv[jj], qv[jj + 1]));
              } else {
#pragma unroll
                for (int jj = 0; jj < 32; jj += 2) {
                  const int32_t a = min(qv[jj], qv[jj + 1]), b = max(qv[jj], qv[jj + 1]);
                  const int32_t t = max(m1, a);
                  m1 = min(m1, a);
                  m2 = __vimin3_s32(t, m2, b);  // second smallest of {m1, m2} u {a, b} (3-input min)
                }
              }
              // decode (key = q >> 5, exact: arithmetic shift) and insert; columns grow with the chunks, so
              // the strict insertion keeps the earlier column on equal keys
              const int32_t k1 = m1 >> 5, k2 = m2 >> 5;
              if (k1 < kk[KMAX - 1]) topk_insert<KT, KMAX>(kk, ii, (KT)k1, (uint32_t)(col0 + (m1 & 31)));
              if (K == 2 && k2 < kk[KMAX - 1]) topk_insert<KT, KMAX>(kk, ii, (KT)k2, (uint32_t)(col0 + (m2 & 31)));
            }
          } else if (direct) {
            // ---- direct single pass (one chunk of <= 32 columns, K <= 4): every key through the insertion
            // network (columns ascending, strict: ties keep the smaller column)
            int4 nb4[8];
            if (U8) {
              const int4* p4 = reinterpret_cast<const int4*>((const int32_t*)args.nb + S.b.pos + c0);
#pragma unroll
              for (int u = 0; u < 8; ++u) nb4[u] = __ldg(p4 + u);
            }
            uint32_t v[32];
            ptx::tmem_ld32(taddr, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              KT key;
              if (U8) {
                const int nbv = (jj & 3) == 0 ? nb4[jj >> 2].x : (jj & 3) == 1 ? nb4[jj >> 2].y
                                : (jj & 3) == 2 ? nb4[jj >> 2].z : nb4[jj >> 2].w;
                key = nbv - 2 * (int32_t)v[jj];
              } else {
                key = __uint_as_float(v[jj]);
              }
              if (key < kk[KMAX - 1]) topk_insert<KT, KMAX>(kk, ii, key, (uint32_t)(c0 + jj));
            }
          } else if (!pass2) {
            // ---- pass 1: group minima of 16 keys, inserted into the value list; uint8: 32 columns per TMEM
            // load (with the 32 column norms in 8 int4 registers), float: 64 (one load wait per 64 columns; the
            // tile's column count is a multiple of 32, the upper half of a 64-column load beyond Nt holds stale
            // values and is masked to +inf)
            constexpr int P1W = U8 ? 32 : 64;
            for (int j0 = 0; j0 < Nt; j0 += P1W) {
              const int col0 = c0 + j0;
              const int nw = min(P1W, Nt - j0);  // 32 or 64 (Nt is a multiple of 32)
              int4 nb4[8];
              if (U8) {
                const int4* p4 = reinterpret_cast<const int4*>((const int32_t*)args.nb + S.b.pos + col0);
#pragma unroll
                for (int u = 0; u < 8; ++u) nb4[u] = __ldg(p4 + u);
              }
              uint32_t v[P1W];
              if (P1W == 32) ptx::tmem_ld32(taddr + j0, *reinterpret_cast<uint32_t(*)[32]>(v));
              else ptx::tmem_ld64(taddr + j0, *reinterpret_cast<uint32_t(*)[64]>(v));
              ptx::tmem_ld_wait();
#pragma unroll
              for (int gq = 0; gq < P1W / 16; ++gq) {
                KT k16[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                  const int c = 16 * gq + jj;
                  if (U8) {
                    const int nbv = (c & 3) == 0 ? nb4[c >> 2].x : (c & 3) == 1 ? nb4[c >> 2].y
                                    : (c & 3) == 2 ? nb4[c >> 2].z : nb4[c >> 2].w;
                    k16[jj] = nbv - 2 * (int32_t)v[c];
                  } else {
                    k16[jj] = __uint_as_float(v[c]);
                  }
                }
                KT gm;
                if (U8) {
                  gm = min(min(min(k16[0], k16[1]), min(k16[2], k16[3])), min(min(k16[4], k16[5]), min(k16[6], k16[7])));
                  gm = min(gm, min(min(min(k16[8], k16[9]), min(k16[10], k16[11])),
                                   min(min(k16[12], k16[13]), min(k16[14], k16[15]))));
                } else {
                  gm = fminf(fminf(fminf(k16[0], k16[1]), fminf(k16[2], k16[3])),
                             fminf(fminf(k16[4], k16[5]), fminf(k16[6], k16[7])));
                  gm = fminf(gm, fminf(fminf(fminf(k16[8], k16[9]), fminf(k16[10], k16[11])),
                                       fminf(fminf(k16[12], k16[13]), fminf(k16[14], k16[15]))));
                }
                if (16 * gq >= nw) gm = kInf;  // (float: the upper 32 columns of a 64-column load beyond Nt)
#pragma unroll
                for (int t = VK - 1; t > 0; --t) {
                  if (U8) vk[t] = max(vk[t - 1], min(vk[t], gm));
                  else vk[t] = fmaxf(vk[t - 1], fminf(vk[t], gm));
                }
                if (U8) vk[0] = min(vk[0], gm);  // (no ?: — it would mix int and float types)
                else vk[0] = fminf(vk[0], gm);
              }
            }
          } else {
          for (int j0 = 0; j0 < Nt; j0 += 32) {
            const int col0 = c0 + j0;
            int4 nb4[8];
            if (U8) {
              // B column norms: 128 B per 32 columns, identical for all lanes (broadcast, L1/L2 resident)
              const int4* p4 = reinterpret_cast<const int4*>((const int32_t*)args.nb + S.b.pos + col0);
#pragma unroll
              for (int u = 0; u < 8; ++u) nb4[u] = __ldg(p4 + u);
            }
            uint32_t v[32];
            ptx::tmem_ld32(taddr + j0, v);
            ptx::tmem_ld_wait();
            // ---- pass 2: t_j = key_j - thr, its sign bit is the pass bit (key_j < thr). uint8: no overflow
            // (real keys lie in (-2^25, 2^25), padding keys are 0x3FFFFFFF, thr is a real key + 1 or 0x40000000);
            // float: the sign of a difference is exact. The mask is built with one funnel shift per element.
            const KT thr = kk[KMAX - 1] != kInf ? kk[KMAX - 1] : U;
            const KT thr_eff = U8 ? (thr == kInf ? (KT)0x40000000 : thr) : thr;
            // uint8: v becomes t = key - thr in place (the staged value); float: v keeps the key bits
            uint32_t mask = 0;
            if (U8) {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                v[4 * u + 0] = (uint32_t)((nb4[u].x - thr_eff) - 2 * (int32_t)v[4 * u + 0]);
                v[4 * u + 1] = (uint32_t)((nb4[u].y - thr_eff) - 2 * (int32_t)v[4 * u + 1]);
                v[4 * u + 2] = (uint32_t)((nb4[u].z - thr_eff) - 2 * (int32_t)v[4 * u + 2]);
                v[4 * u + 3] = (uint32_t)((nb4[u].w - thr_eff) - 2 * (int32_t)v[4 * u + 3]);
              }
            }
            // four independent funnel-shift chains of 8 bits each (a single 32-long chain is latency-bound)
            uint32_t m8[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int jj = 7; jj >= 0; --jj) {
#pragma unroll
              for (int qd = 0; qd < 4; ++qd) {
                const int j = 8 * qd + jj;
                const uint32_t bits = U8 ? v[j] : __float_as_uint(__uint_as_float(v[j]) - (float)thr_eff);
                m8[qd] = __funnelshift_l(bits, m8[qd], 1);  // (m << 1) | sign(t_j)
              }
            }
            mask = m8[0] | (m8[1] << 8) | (m8[2] << 16) | (m8[3] << 24);
            if (col0 == diag_chunk) mask &= ~(1u << lane);  // self exclusion (by id: the diagonal element)
            if (__any_sync(0xffffffffu, mask != 0)) {
              // room for this chunk's passes (a drain empties the queue; a chunk can still exceed kQCap)
              if (__any_sync(0xffffffffu, qlen + __popc(mask) > kQCap)) topk_drain<KT, KMAX>(kk, ii, qlen, my_qk, my_qc);
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                *reinterpret_cast<uint4*>(stg + 4 * u) = make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
              }
              __syncwarp();
              while (mask) {
                const int jj = __ffs(mask) - 1;
                mask &= mask - 1;
                if (qlen == kQCap) topk_drain<KT, KMAX>(kk, ii, qlen, my_qk, my_qc);  // (per lane) never overflow
                // uint8 stages t = key - thr (key = t + thr exactly); float stages the key itself
                my_qk[qlen * 128] = U8 ? (KT)(reinterpret_cast<const int32_t*>(stg)[jj] + (int32_t)thr_eff)
                                       : (KT)reinterpret_cast<const float*>(stg)[jj];
                my_qc[qlen * 128] = (uint16_t)(col0 + jj);
                ++qlen;
                if (prof) ++pw[2];
              }
              __syncwarp();
            }
          }
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&bar_acc_empty[buf]);
        }
        const unsigned long long t_out = prof ? clock64() : 0ull;
        if (prof) ++pw[3];  // items (rows) of this thread
        topk_drain<KT, KMAX>(kk, ii, qlen, my_qk, my_qc);
        bool vec_done = false;
        if (KMAX == 8 && row < S.a.rows && K == 8 && S.ostride == 8 && args.out_col && args.out_dist && !args.out_idx &&
            !args.out_cnt && !args.out_rowid) {
          // the build path's leaf picks (k = 8, every slot valid): the row's 8 columns (16 B) and distances (32 B) as
          // vector stores instead of 16 scalar stores at an 8-element stride
          bool allv = true;
#pragma unroll
          for (int t = 0; t < 8; ++t) allv &= ii[t] != 0xFFFFu && ii[t] < (uint32_t)ncols;
          if (allv) {
            const int64_t obase = S.out_off + (int64_t)row * 8;
            float Dv[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              if (MIPS) Dv[t] = (float)kk[t];
              else if (U8) Dv[t] = (float)(na_row + kk[t]);
              else Dv[t] = fmaxf(fmaf(2.0f, (float)kk[t], (float)na_row), 0.0f);
            }
            *reinterpret_cast<uint4*>(args.out_col + obase) =
                make_uint4((uint32_t)ii[0] | ((uint32_t)ii[1] << 16), (uint32_t)ii[2] | ((uint32_t)ii[3] << 16),
                           (uint32_t)ii[4] | ((uint32_t)ii[5] << 16), (uint32_t)ii[6] | ((uint32_t)ii[7] << 16));
            float4* dp = reinterpret_cast<float4*>(args.out_dist + obase);
            dp[0] = make_float4(Dv[0], Dv[1], Dv[2], Dv[3]);
            dp[1] = make_float4(Dv[4], Dv[5], Dv[6], Dv[7]);
            vec_done = true;
          }
        }
        if (row < S.a.rows && !vec_done) {
          const int64_t obase = S.out_off + (int64_t)row * S.ostride;
          const KT na = na_row;
          int o = 0;
#pragma unroll
          for (int t = 0; t < KMAX; ++t) {
            const uint32_t col = ii[t];
            const bool take = t >= KMAX - K && col != 0xFFFFu && col < (uint32_t)ncols;
            if (take) {
              const KT key = kk[t];
              float D;
              if (MIPS) D = (float)key;
              else if (U8) D = (float)(na + key);
              else D = fmaxf(fmaf(2.0f, (float)key, (float)na), 0.0f);
              // (the pick's id is needed only for out_idx / out_cnt: the build path writes local columns)
              const uint32_t pid = (args.out_idx || args.out_cnt) && args.col_ids ? args.col_ids[S.b.id_off + col] : col;
              if (args.out_idx) args.out_idx[obase + o] = pid;
              if (args.out_col) args.out_col[obase + o] = (uint16_t)col;
              if (args.out_dist) args.out_dist[obase + o] = D;
              if (args.out_cnt) atomicAdd(&args.out_cnt[pid], 1u);
              ++o;
            }
          }
          if (args.out_rowid) {
            const uint32_t rid = args.row_ids[S.a.id_off + row];
            for (int t = 0; t < S.ostride; ++t) args.out_rowid[obase + t] = rid;
          }
          for (; o < S.ostride; ++o) {
            if (args.out_idx) args.out_idx[obase + o] = 0xFFFFFFFFu;
            if (args.out_col) args.out_col[obase + o] = 0xFFFFu;
            if (args.out_dist) args.out_dist[obase + o] = __int_as_float(0x7F800000);
          }
        }
        if (prof) pw[9] += clock64() - t_out;
      }
      if (prof && tid == 0) {
        atomicAdd(&g_dt_prof[11], pw[9]);
        atomicAdd(&g_dt_prof[15], pw[2]);  // pass-2 candidates appended (this thread's rows)
        atomicAdd(&g_dt_prof[3], pw[3]);  // rows sampled
        atomicAdd(&g_dt_prof[8], pw[8]);
        atomicAdd(&g_dt_prof[9], clock64() - t_start);
        atomicAdd(&g_dt_prof[10], (unsigned long long)tcount);
      }
    }();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// Host launcher (dist_topk.cu): picks the instantiation for (dtype, metric, K).
pipnn_status launch_dist_topk(const DistTopkArgs& a, bool u8, bool mips, int kmax, cudaStream_t st);
// Whether the packed partition pass (uint8, K <= 2) runs on dist_topk_uf2_kernel, which then takes pair items
// (DistTopkArgs::pairs = 1) instead of block items.
bool dt_packed_pairs(int Kb);

}  // namespace pipnn
