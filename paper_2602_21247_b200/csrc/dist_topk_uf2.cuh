// dist_topk_uf2.cuh — the folded-uint8 leaf kernel with four epilogue warpgroups (§4.2 "Leaf Building",
// for every leaf and every member row, the k nearest other members by (D, id); the ranking and the
// folded layout are those of dist_topk.cuh, UF path, and of leaf.cu "folded uint8 rows").
//
// Why a second kernel (DESIGN.md §7 "K5, four epilogue warpgroups"): the UF path of dist_topk_kernel is bound by
// its epilogue's latencies with two epilogue warps per scheduler (ncu: issue slots ~49% busy; per-instruction
// samples spread over TMEM-load waits, the pass-2 filter chains and the divergent candidate loop). Here:
//   * a work item is a PAIR of 128-row blocks of one leaf (blocks rb, rb + 1; the odd-rb items of the block list
//     are skipped by the producer's claim), and both blocks multiply the same B tile: one B copy per tile for
//     256 rows (half the L2 -> SMEM traffic of the one-block item);
//   * 20 warps: producer warps 0, 1 and MMA-issuer warps 2, 3 of pipelines 0 and 1; epilogue warpgroups 0..3 =
//     warps 4..19, warpgroup 2p + b owning block b of pipeline p's item and TMEM accumulator 2p + b (128 columns
//     each, all 512 columns; one accumulator per warpgroup — the other three warpgroups hide its MMA round trip);
//     so four epilogue warps per scheduler instead of two;
//   * SMEM (d = 128: 24-KB tile stages, 16-KB A blocks) is bought by a compact A-side augment tile (8 identical
//     rows per plane, row-group stride 0 in the descriptor), an XOR-swizzled 16-KB key staging area per warpgroup
//     (no padding) and no candidate queue: passing keys go straight into the register list, so the pass-2
//     threshold tightens with every insertion.
// The picks are identical to dist_topk_kernel<U8=1, MIPS=0, KMAX, UF=1>: columns arrive in ascending order, the
// insertion is strict, so equal keys keep the smaller column (= smaller id inside a leaf).
// PK = the partition's packed single pass instead (uint8 rows against a group's leaders, K <= 2, no threshold pass,
// plain u8 x u8 MMA; the packed leader norms 32 ||l||^2 + (position mod 32) order a chunk by (key, column) — the
// packedm branch of dist_topk_kernel), identical to dist_topk_kernel<1, 0, 2, 0> with packed = 1.
#pragma once
#include "dist_topk.cuh"

namespace pipnn {

constexpr int kUf2Threads = 640;
constexpr int kUf2StgBytes = 128 * 32 * 4;  // per warpgroup: 32 staged words per row
constexpr int kUf2OnesBytes = 1024;         // compact augment tile: <= 8 planes x 128 B

struct Uf2Geom {
  int KCs, KCm, stage_bytes, NS, smem;
};
// Plane geometry (as dt_geom): KCs planes of 16 B per row (the block stride), KCm of them coordinates; a whole
// tile per ring stage; NS stages per pipeline.
__host__ __device__ inline Uf2Geom uf2_geom(int Kb, int augp) {
  Uf2Geom g;
  g.KCs = Kb / 16;
  g.KCm = g.KCs - augp;
  g.stage_bytes = g.KCs * 2048;
  const int fixed = 4 * g.KCm * 2048 + 4 * kUf2StgBytes + kUf2OnesBytes;
  g.NS = (kDtSmemBudget - 1024 - fixed) / (2 * g.stage_bytes);
  if (g.NS > 4) g.NS = 4;
  g.smem = fixed + 2 * g.NS * g.stage_bytes;
  return g;
}
// The kernel applies when both pipelines get >= 2 stages (folded rows: d <= 128 at 4 augment planes) and augp <= 8
// (folded rows) or augp == 0 (packed partition pass).
__host__ __device__ inline bool uf2_fits(int Kb, int augp, bool packed = false) {
  const Uf2Geom g = uf2_geom(Kb, augp);
  return (packed ? augp == 0 : (augp > 0 && augp <= 8)) && (g.KCs & 1) == 0 && g.NS >= 2;
}

template <int KMAX, bool PK = false>
__global__ void __launch_bounds__(kUf2Threads, 1) dist_topk_uf2_kernel(const DistTopkArgs args) {
  using KT = int32_t;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_full[2][4], bar_empty[2][4];
  __shared__ __align__(8) uint64_t bar_a_full[2], bar_a_empty[2];
  __shared__ __align__(8) uint64_t bar_acc_full[4], bar_acc_empty[4];
  __shared__ __align__(8) uint64_t bar_it_full[2][kDtItemRing], bar_it_empty[2][kDtItemRing];
  __shared__ int64_t item_ring[2][kDtItemRing];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int augp = args.uf_aug;
  const Uf2Geom GM = uf2_geom(args.Kb, augp);
  const int KCs = GM.KCs, KCm = GM.KCm, SB = GM.stage_bytes, NS = GM.NS;
  uint8_t* sA = smem;                                // [2 pipelines][2 blocks][KCm][128][16]
  uint8_t* ring = sA + 4 * KCm * 2048;               // [2 pipelines][NS][SB]
  uint8_t* stg_base = ring + 2 * NS * SB;            // [4 warpgroups][128 rows][32 words], 16-B units swizzled
  uint8_t* sOnes = stg_base + 4 * kUf2StgBytes;      // [augp planes][8 rows][16 B]

  // constant A-side augment rows (dist_topk.cuh, UF): s8 weight 127 everywhere but the last byte of the last
  // plane (weight 1); 8 rows per plane, all read for every 8-row group (descriptor row-group stride 0)
  for (int e = threadIdx.x; e < augp * 32; e += blockDim.x) {
    const bool last = (e >> 5) == augp - 1 && (e & 3) == 3;
    reinterpret_cast<uint32_t*>(sOnes)[e] = last ? 0x017F7F7Fu : 0x7F7F7F7Fu;
  }
  ptx::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int p = 0; p < 2; ++p) {
      for (int s = 0; s < NS; ++s) {
        ptx::mbar_init(&bar_full[p][s], 1);
        ptx::mbar_init(&bar_empty[p][s], 1);
      }
      ptx::mbar_init(&bar_a_full[p], 1);
      ptx::mbar_init(&bar_a_empty[p], 1);
      for (int e = 0; e < kDtItemRing; ++e) {
        ptx::mbar_init(&bar_it_full[p][e], 1);
        ptx::mbar_init(&bar_it_empty[p][e], 9);  // the MMA warp + the 8 epilogue warps of the pipeline
      }
    }
    for (int b = 0; b < 4; ++b) {
      ptx::mbar_init(&bar_acc_full[b], 1);
      ptx::mbar_init(&bar_acc_empty[b], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(&tmem_base_sh, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int64_t n_items = *args.n_items;

  // Item sequence of pipeline p (dynamic): the producer claims block items from the shared counter, skips the
  // odd blocks (each is the second block of its even predecessor's pair) and hands the pair to its MMA warp and
  // epilogue warpgroups through an SMEM ring; -1 ends the sequence.
  const bool dyn = args.work != nullptr;  // else: static round-robin over pair items (args.pairs)
  auto claim_item = [&](int p, uint32_t j) -> int64_t {  // producer (one lane)
    if (!dyn) {
      const int64_t it = (int64_t)blockIdx.x + (2 * (int64_t)j + p) * gridDim.x;
      return it < n_items ? it : -1;
    }
    const int e = (int)(j % kDtItemRing);
    if (!ptx::mbar_wait_hint(&bar_it_empty[p][e], ((j / kDtItemRing) & 1) ^ 1u, args.err, DERR_WAIT_TIMEOUT, 1000000u))
      return -1;
    int64_t it;
    for (;;) {
      it = (int64_t)atomicAdd(args.work, 1ull);
      if (it >= n_items || (args.items[it].rb & 1) == 0) break;
    }
    item_ring[p][e] = it < n_items ? it : -1;
    ptx::mbar_arrive(&bar_it_full[p][e]);
    return it < n_items ? it : -1;
  };
  auto take_item = [&](int p, uint32_t j, bool arrive) -> int64_t {  // MMA warp / epilogue warps
    if (!dyn) {
      const int64_t it = (int64_t)blockIdx.x + (2 * (int64_t)j + p) * gridDim.x;
      return it < n_items ? it : -1;
    }
    const int e = (int)(j % kDtItemRing);
    if (!ptx::mbar_wait(&bar_it_full[p][e], (j / kDtItemRing) & 1, args.err, DERR_WAIT_TIMEOUT)) return -1;
    const int64_t it = *(volatile int64_t*)&item_ring[p][e];
    __syncwarp();
    if (arrive) ptx::mbar_arrive(&bar_it_empty[p][e]);
    return it;
  };

  if (warp < 2) {
    // ------------------------------------------------------------ producer of pipeline p
    const int p = warp;
    uint32_t sg = 0, ia = 0;
    uint8_t* my_ring = ring + p * NS * SB;
    for (uint32_t jj = 0;; ++jj) {
      int64_t it = 0;
      if (lane == 0) it = claim_item(p, jj);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it < 0) break;
      const WorkItem w = args.items[it];
      const DistSeg S = args.segs[w.seg];
      const int T = (S.b.rows + kDtTileN - 1) / kDtTileN;
      const int nb = (w.rb + 1) * 128 < S.a.rows ? 2 : 1;
      bool ok = true;
      if (lane == 0) {
        ok = ptx::mbar_wait_hint(&bar_a_empty[p], (ia & 1) ^ 1u, args.err, DERR_WAIT_TIMEOUT, 1000000u);
        if (ok) {
          ptx::mbar_arrive_expect_tx(&bar_a_full[p], (uint32_t)(nb * KCm * 2048));
          for (int b = 0; b < nb; ++b)
            ptx::bulk_g2s(sA + (2 * p + b) * KCm * 2048, args.Ta + (S.a.pos / 128 + w.rb + b) * (int64_t)KCs * 2048,
                          KCm * 2048, &bar_a_full[p]);
        }
      }
      ++ia;
      const int p1 = dt_p1(S.k, S.b.rows, S.self, args.p1cap);
      for (int t = 0; t < p1 + T; ++t, ++sg) {
        const int s = sg % NS;
        if (s % kDtCopyLanes != lane || !ok) continue;
        const int c0 = (t < p1 ? t : t - p1) * kDtTileN;
        ok = ptx::mbar_wait_hint(&bar_empty[p][s], ((sg / NS) & 1) ^ 1u, args.err, DERR_WAIT_TIMEOUT, 1000000u);
        if (!ok) continue;
        ptx::mbar_arrive_expect_tx(&bar_full[p][s], (uint32_t)SB);
        ptx::bulk_g2s(my_ring + s * SB, args.Tb + (S.b.pos / 128 + c0 / 128) * (int64_t)KCs * 2048, SB, &bar_full[p][s]);
      }
      if (!__all_sync(0xffffffffu, ok)) break;
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ MMA issuer of pipeline p (converged warp)
    const int p = warp - 2;
    uint32_t sg = 0, ia = 0, tcb0 = 0, tcb1 = 0;
    const uint32_t ring_u32 = ptx::smem_u32(ring + p * NS * SB);
    const uint64_t ones_desc = ptx::smem_desc_kmajor_noswz(ptx::smem_u32(sOnes), 128, 0);
    const uint64_t a_desc0 = ptx::smem_desc_kmajor_noswz(ptx::smem_u32(sA + (2 * p) * KCm * 2048), 2048, 128);
    const uint64_t a_desc1 = ptx::smem_desc_kmajor_noswz(ptx::smem_u32(sA + (2 * p + 1) * KCm * 2048), 2048, 128);
    [&]() {
      for (uint32_t jj = 0;; ++jj) {
        const int64_t it = take_item(p, jj, lane == 0);
        if (it < 0) return;
        const WorkItem w = args.items[it];
        const DistSeg S = args.segs[w.seg];
        const int ncols = S.b.rows;
        const int T = (ncols + kDtTileN - 1) / kDtTileN;
        const int p1 = dt_p1(S.k, ncols, S.self, args.p1cap);
        const int nb = (w.rb + 1) * 128 < S.a.rows ? 2 : 1;
        if (!ptx::mbar_wait_hint(&bar_a_full[p], ia & 1, args.err, DERR_WAIT_TIMEOUT, 1000000u)) return;
        ++ia;
        for (int t = 0; t < p1 + T; ++t, ++sg) {
          const int c0 = (t < p1 ? t : t - p1) * kDtTileN;
          const int Nt = min(kDtTileN, (ncols - c0 + 31) & ~31);
          // folded rows: A and B signed (s8); packed partition pass: u8 x u8
          const uint32_t idesc = PK ? ptx::idesc_u8_s32(128, Nt) : (ptx::idesc_u8_s32(128, Nt) | (1u << 7) | (1u << 10));
          const int s = sg % NS;
          if (!ptx::mbar_wait_hint(&bar_full[p][s], (sg / NS) & 1, args.err, DERR_WAIT_TIMEOUT, 1000000u)) return;
          ptx::tc_fence_after();
          const uint64_t b_desc = ptx::smem_desc_kmajor_noswz(ring_u32 + s * SB, 2048, 128);
          for (int b = 0; b < nb; ++b) {
            const int acc = 2 * p + b;
            const uint32_t use = b ? tcb1++ : tcb0++;
            if (!ptx::mbar_wait_hint(&bar_acc_empty[acc], (use & 1) ^ 1u, args.err, DERR_WAIT_TIMEOUT, 1000000u)) return;
            ptx::tc_fence_after();
            const uint64_t a_desc = b ? a_desc1 : a_desc0;
            if (ptx::elect_one()) {
              for (int kc = 0; kc < KCs; kc += 2) {
                const uint64_t ad = kc >= KCm ? ones_desc + (uint64_t)((kc - KCm) * 8) : a_desc + (uint64_t)(kc * 128);
                ptx::mma_i8(tmem + acc * kDtTileN, ad, b_desc + (uint64_t)(kc * 128), idesc, kc > 0 ? 1u : 0u);
              }
              ptx::mma_commit(&bar_acc_full[acc]);
            }
            __syncwarp();
          }
          if (ptx::elect_one()) ptx::mma_commit(&bar_empty[p][s]);  // the stage's MMAs issued: free it
          __syncwarp();
        }
        if (ptx::elect_one()) ptx::mma_commit(&bar_a_empty[p]);  // the item's MMAs issued: free its A blocks
        __syncwarp();
      }
    }();
  } else {
    // ------------------------------------------------------------ epilogue warpgroup wg = 2p + b, one row per thread
    // Pass 1 (threshold) and pass 2 (exact) exactly as the UF path of dist_topk_kernel; pass 2 inserts every
    // passing key directly into the sorted register list (no SMEM queue), so its threshold is the list's current
    // K-th key as soon as the list is full.
    const int ew = warp - 4;
    const int wg = ew >> 2, p = wg >> 1, b = wg & 1;
    const int q = warp & 3;                 // TMEM lane quadrant (hardware: warp id % 4)
    const int tid = q * 32 + lane;          // row within the 128-row block = TMEM lane
    const KT kInf = (KT)0x7FFFFFFF;
    const KT kNegInf = (KT)(-0x7FFFFFFF - 1);
    constexpr int VK = KMAX + 1;
    uint32_t* stg = reinterpret_cast<uint32_t*>(stg_base + wg * kUf2StgBytes) + tid * 32;
    const int swz = tid & 7;
    uint32_t tcount = 0;
    const uint32_t tacc = tmem + wg * kDtTileN + ((uint32_t)(q * 32) << 16);
    [&]() {
    for (uint32_t jj = 0;; ++jj) {
      const int64_t it = take_item(p, jj, lane == 0);
      if (it < 0) break;
      const WorkItem w = args.items[it];
      const DistSeg S = args.segs[w.seg];
      const int r0 = (w.rb + b) * 128;
      if (r0 >= S.a.rows) continue;  // the pair's second block does not exist: no tiles for this warpgroup
      const int row = r0 + tid;
      const KT na_row = row < S.a.rows ? ((const KT*)args.na)[S.a.pos + row] : (KT)0;
      const int K = S.k;
      const int K1 = K + (S.self ? 1 : 0);
      const int ncols = S.b.rows;
      const int T = (ncols + kDtTileN - 1) / kDtTileN;
      KT vk[VK];
#pragma unroll
      for (int t = 0; t < VK; ++t) vk[t] = t < VK - K1 ? kNegInf : kInf;
      KT kk[KMAX];
      uint16_t ii[KMAX];
#pragma unroll
      for (int t = 0; t < KMAX; ++t) {
        kk[t] = t < KMAX - K ? kNegInf : kInf;
        ii[t] = 0xFFFFu;
      }
      KT U = kInf;
      const int diag_chunk = S.self ? (r0 + q * 32) : -1;
      const int P1 = dt_p1(K, ncols, S.self, args.p1cap);
      for (int t2 = 0; t2 < P1 + T; ++t2, ++tcount) {
        const bool pass2 = t2 >= P1;
        const int c0 = (pass2 ? t2 - P1 : t2) * kDtTileN;
        const int Nt = min(kDtTileN, (ncols - c0 + 31) & ~31);
        if (!ptx::mbar_wait(&bar_acc_full[wg], tcount & 1, args.err, DERR_WAIT_TIMEOUT)) return;
        ptx::tc_fence_after();
        if (t2 == P1 && P1 > 0) {
          U = vk[VK - 1];
          U = U == kInf ? (KT)(1 << 30) : U;  // fewer than K1 groups: everything passes
        }
        if (PK) {
          // packed single pass (K <= 2): q_j = 32 key_j + (j mod 32) = nbp_j - 64 v_j (one IMAD) orders the chunk's
          // columns by (key, column) exactly; its two smallest by a min/max network on column pairs, inserted
          for (int j0 = 0; j0 < Nt; j0 += 32) {
            const int col0 = c0 + j0;
            int4 nb4[8];
            const int4* p4 = reinterpret_cast<const int4*>((const int32_t*)args.nb + S.b.pos + col0);
#pragma unroll
            for (int u = 0; u < 8; ++u) nb4[u] = __ldg(p4 + u);
            uint32_t v[32];
            ptx::tmem_ld32(tacc + j0, v);
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
              for (int j = 0; j < 32; j += 2) m1 = min(m1, min(qv[j], qv[j + 1]));
            } else {
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const int32_t lo = min(qv[j], qv[j + 1]), hi = max(qv[j], qv[j + 1]);
                const int32_t t = max(m1, lo);
                m1 = min(m1, lo);
                m2 = __vimin3_s32(t, m2, hi);
              }
            }
            const int32_t k1 = m1 >> 5, k2 = m2 >> 5;
            if (k1 < kk[KMAX - 1]) topk_insert<KT, KMAX>(kk, ii, (KT)k1, (uint32_t)(col0 + (m1 & 31)));
            if (K == 2 && k2 < kk[KMAX - 1]) topk_insert<KT, KMAX>(kk, ii, (KT)k2, (uint32_t)(col0 + (m2 & 31)));
          }
        } else if (!pass2) {
          // maxima of acc over groups of 16 columns, negated into the value list; padding columns never win
          for (int j0 = 0; j0 < Nt; j0 += 32) {
            const int valid = min(32, ncols - (c0 + j0));
            uint32_t v[32];
            ptx::tmem_ld32(tacc + j0, v);
            ptx::tmem_ld_wait();
            if (valid < 32) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j >= valid) v[j] = 0x80000000u;
            }
#pragma unroll
            for (int gq = 0; gq < 2; ++gq) {
              const int32_t* wv = reinterpret_cast<const int32_t*>(v) + 16 * gq;
              int32_t g = __vimax3_s32(wv[0], wv[1], wv[2]);
              g = __vimax3_s32(g, wv[3], wv[4]);
              g = __vimax3_s32(g, wv[5], wv[6]);
              g = __vimax3_s32(g, wv[7], wv[8]);
              g = __vimax3_s32(g, wv[9], wv[10]);
              g = __vimax3_s32(g, wv[11], wv[12]);
              g = __vimax3_s32(g, wv[13], wv[14]);
              g = max(g, wv[15]);
              const KT gm = (16 * gq < valid) ? (KT)(-g) : kInf;
#pragma unroll
              for (int t = VK - 1; t > 0; --t) vk[t] = max(vk[t - 1], min(vk[t], gm));
              vk[0] = min(vk[0], gm);
            }
          }
        } else {
          // acc >= tau passes: tau = -U until the list is full, then floor(-kk / 2) of its K-th key kk (a
          // conservative bound; the insertion compares the exact key -2 acc - parity)
          for (int j0 = 0; j0 < Nt; j0 += 32) {
            const int col0 = c0 + j0;
            const int valid = min(32, ncols - col0);
            uint32_t v[32];
            ptx::tmem_ld32(tacc + j0, v);
            // the chunk's parity word, needed only when a lane passes: loaded here so that its latency overlaps the
            // TMEM load instead of sitting in the candidate path
            const uint32_t pbits = __ldg(reinterpret_cast<const uint32_t*>(args.nb) + ((S.b.pos + col0) >> 5));
            const int32_t kk8 = (int32_t)kk[KMAX - 1];
            const int32_t tau = kk8 != (int32_t)kInf ? ((-kk8) >> 1) : -(int32_t)U;
            ptx::tmem_ld_wait();
            uint32_t m8[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int j = 7; j >= 0; --j) {
#pragma unroll
              for (int qd = 0; qd < 4; ++qd) m8[qd] = __funnelshift_l((uint32_t)((int32_t)v[8 * qd + j] - tau), m8[qd], 1);
            }
            uint32_t mask = ~(m8[0] | (m8[1] << 8) | (m8[2] << 16) | (m8[3] << 24));
            if (valid < 32) mask &= (1u << valid) - 1u;
            if (col0 == diag_chunk) mask &= ~(1u << lane);  // self exclusion (the diagonal element)
            if (__any_sync(0xffffffffu, mask != 0)) {
              if (mask) {
#pragma unroll
                for (int u = 0; u < 8; ++u)
                  *reinterpret_cast<uint4*>(stg + 4 * (u ^ swz)) = make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                while (mask) {
                  const int j = __ffs(mask) - 1;
                  mask &= mask - 1;
                  const KT key = (KT)(-2 * (int32_t)stg[4 * ((j >> 2) ^ swz) + (j & 3)] - (int32_t)((pbits >> j) & 1u));
                  if (key < kk[KMAX - 1]) topk_insert<KT, KMAX>(kk, ii, key, (uint32_t)(col0 + j));
                }
              }
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&bar_acc_empty[wg]);
      }
      if (row >= S.a.rows) continue;
      bool vec_done = false;
      if (KMAX == 8 && K == 8 && S.ostride == 8 && args.out_col && args.out_dist && !args.out_idx && !args.out_cnt &&
          !args.out_rowid) {
        // the build path's picks (k = 8, every slot valid): 16-B column store + two 16-B distance stores
        bool allv = true;
#pragma unroll
        for (int t = 0; t < 8; ++t) allv &= ii[t] != 0xFFFFu && ii[t] < (uint32_t)ncols;
        if (allv) {
          const int64_t obase = S.out_off + (int64_t)row * 8;
          float Dv[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) Dv[t] = (float)(na_row + kk[t]);
          *reinterpret_cast<uint4*>(args.out_col + obase) =
              make_uint4((uint32_t)ii[0] | ((uint32_t)ii[1] << 16), (uint32_t)ii[2] | ((uint32_t)ii[3] << 16),
                         (uint32_t)ii[4] | ((uint32_t)ii[5] << 16), (uint32_t)ii[6] | ((uint32_t)ii[7] << 16));
          float4* dp = reinterpret_cast<float4*>(args.out_dist + obase);
          dp[0] = make_float4(Dv[0], Dv[1], Dv[2], Dv[3]);
          dp[1] = make_float4(Dv[4], Dv[5], Dv[6], Dv[7]);
          vec_done = true;
        }
      }
      if (!vec_done) {
        const int64_t obase = S.out_off + (int64_t)row * S.ostride;
        int o = 0;
#pragma unroll
        for (int t = 0; t < KMAX; ++t) {
          const uint32_t col = ii[t];
          if (t >= KMAX - K && col != 0xFFFFu && col < (uint32_t)ncols) {
            const float D = (float)(na_row + kk[t]);
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

}  // namespace pipnn
