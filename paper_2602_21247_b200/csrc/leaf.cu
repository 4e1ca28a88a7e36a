// leaf.cu — leaf gather into the tiled MMA layout (+ squared norms) and the leaf-pick driver
// (§4.2: all-pairs distances inside each leaf, then the bidirected k-NN pick).
#include <algorithm>
#include <cub/cub.cuh>

#include "internal.h"

namespace pipnn {

int tiled_row_bytes(const pipnn_points* X) {
  if (X->dtype == PIPNN_U8) return (int)round_up(X->d, 32);
  return (int)round_up(X->d, 16) * 2 + 32;  // bf16 coordinates + one augmented K-step (dist_topk.cuh)
}

// ------------------------------------------------------------------ gather
// One CTA of 4 warps per (segment, 128-row block); lane = row (warp w: rows 32w..32w+31 of the block). Each
// lane walks its row in 16-B chunks (fp32 -> bf16 RNE for float data; consecutive chunks of a row share L1
// sectors) and stores chunk kc of its row at plane kc of the block-major layout [K/16][128][16 B]: a warp's
// stores of one plane are 512 contiguous bytes. The row's squared norm accumulates in the lane (int32 exact
// for uint8, fp32 of the bf16 values for float). No shared memory, no block barrier.
// Float rows end with the 16-element augment K-step of dist_topk.cuh: (t_hi, t_mid, t_lo, 0...) with
// t = -||y||^2/2 (L2) or 0 (MIPS), split over three bf16 values; padding rows get t = -1e30 (u8 padding
// rows get the norm kPadNormU8 instead), so padded columns never enter a top-k.
template <int SRC>  // 0: uint8, 1: float32, 2: bf16 (kDtypeBf16)
__global__ void __launch_bounds__(128) gather_tiled_kernel(const void* __restrict__ Xv, int64_t ld, int d, int Kb,
                                                           int mips, const uint32_t* __restrict__ ids,
                                                           const TileSeg* __restrict__ segs,
                                                           const WorkItem* __restrict__ items,
                                                           const int64_t* __restrict__ n_items, uint8_t* __restrict__ T,
                                                           void* __restrict__ nrm, int* err, int packed) {
  constexpr bool U8 = SRC == 0;
  if ((int64_t)blockIdx.x >= *n_items) return;
  const WorkItem w = items[blockIdx.x];
  const TileSeg S = segs[w.seg];
  const int r = threadIdx.x;  // row within the 128-row block
  const int local = w.rb * 128 + r;
  const bool valid = local < S.rows;
  const int KC = Kb >> 4;
  const int ldm = U8 ? Kb : (Kb - 32) / 2;      // elements of the coordinate part (float: bf16 elements)
  const int ncc = U8 ? KC : (ldm >> 3);          // 16-B chunks holding coordinates
  uint8_t* dst = T + (S.pos / 128 + w.rb) * (int64_t)KC * 2048 + r * 16;
  const int64_t id = valid ? (ids ? (int64_t)ids[S.id_off + local] : (S.id_off + local)) : 0;
  int32_t ni = 0;
  float nf = 0.0f;
  bool bad = false;
  const bool vec = U8 ? ((d & 15) == 0 && (ld & 15) == 0) : ((d & 3) == 0 && (ld & 3) == 0);
#pragma unroll 4
  for (int kc = 0; kc < ncc; ++kc) {
    uint4 out = make_uint4(0u, 0u, 0u, 0u);
    if (valid) {
      if (U8) {
        const uint8_t* src = (const uint8_t*)Xv + id * ld;
        if (vec) {
          if (kc * 16 < d) out = __ldg((const uint4*)src + kc);
        } else {
          uint32_t wv[4] = {0u, 0u, 0u, 0u};
          for (int t = 0; t < 16; ++t)
            if (kc * 16 + t < d) wv[t >> 2] |= (uint32_t)src[kc * 16 + t] << (8 * (t & 3));
          out = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
        ni = (int32_t)__dp4a(out.x, out.x, (uint32_t)ni);
        ni = (int32_t)__dp4a(out.y, out.y, (uint32_t)ni);
        ni = (int32_t)__dp4a(out.z, out.z, (uint32_t)ni);
        ni = (int32_t)__dp4a(out.w, out.w, (uint32_t)ni);
      } else if (SRC == 2) {
        // bf16 rows zero padded to ld (a multiple of 8): 16-B chunks, norm of the bf16 values
        if (kc * 8 < ld) out = __ldg((const uint4*)((const uint16_t*)Xv + id * ld) + kc);
        const uint32_t wv[4] = {out.x, out.y, out.z, out.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float xl = __uint_as_float(wv[t] << 16), xh = __uint_as_float(wv[t] & 0xFFFF0000u);
          nf = fmaf(xl, xl, nf);
          nf = fmaf(xh, xh, nf);
        }
      } else {
        const float* src = (const float*)Xv + id * ld;
        float f[8];
        if (vec && kc * 8 + 8 <= d) {
          const float4 a = __ldg((const float4*)(src + kc * 8));
          const float4 b = __ldg((const float4*)(src + kc * 8 + 4));
          f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
        } else {
#pragma unroll
          for (int t = 0; t < 8; ++t) f[t] = kc * 8 + t < d ? __ldg(src + kc * 8 + t) : 0.0f;
        }
        uint32_t wv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint16_t lo = f32_to_bf16_rne(f[2 * t]), hi = f32_to_bf16_rne(f[2 * t + 1]);
          bad |= !isfinite(f[2 * t]) || !isfinite(f[2 * t + 1]);
          const float xl = __uint_as_float((uint32_t)lo << 16), xh = __uint_as_float((uint32_t)hi << 16);
          nf = fmaf(xl, xl, nf);
          nf = fmaf(xh, xh, nf);
          wv[t] = (uint32_t)lo | ((uint32_t)hi << 16);
        }
        out = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    }
    *(uint4*)(dst + (int64_t)kc * 2048) = out;
  }
  if (bad) atomicExch(err, DERR_NONFINITE);
  if (U8) {
    // packed (the partition's K <= 2 single pass, dist_topk.cuh): 32 ||y||^2 + (position mod 32)
    ((int32_t*)nrm)[S.pos + local] = valid ? (packed ? 32 * ni + ((S.pos + local) & 31) : ni) : kPadNormU8;
  } else {
    ((float*)nrm)[S.pos + local] = nf;
    const float t = valid ? (mips ? 0.0f : -0.5f * nf) : -kPadKey;
    const uint16_t hi = f32_to_bf16_rne(t);
    const float r1 = t - __uint_as_float((uint32_t)hi << 16);
    const uint16_t mid = f32_to_bf16_rne(r1);
    const float r2 = r1 - __uint_as_float((uint32_t)mid << 16);
    const uint16_t lo = f32_to_bf16_rne(r2);
    *(uint4*)(dst + (int64_t)ncc * 2048) = make_uint4((uint32_t)hi | ((uint32_t)mid << 16), (uint32_t)lo, 0u, 0u);
    *(uint4*)(dst + (int64_t)(ncc + 1) * 2048) = make_uint4(0u, 0u, 0u, 0u);
  }
}

pipnn_status gather_tiled(const pipnn_points* X, const uint32_t* ids, const TileSeg* segs, const WorkItem* items,
                          const int64_t* n_items, int64_t max_items, uint8_t* T, void* nrm, const Ctx& c, int Kb,
                          int packed) {
  if (max_items <= 0) return PIPNN_OK;
  if (Kb <= 0) Kb = tiled_row_bytes(X);
  const int64_t ld = X->ld;
#define GT_LAUNCH(SRC)                                                                                             \
  gather_tiled_kernel<SRC><<<(unsigned)max_items, 128, 0, c.st>>>(X->data, ld, X->d, Kb, X->metric == PIPNN_MIPS,   \
                                                                  ids, segs, items, n_items, T, nrm, c.err, packed)
  if (X->dtype == PIPNN_U8) GT_LAUNCH(0);
  else if (X->dtype == kDtypeBf16) GT_LAUNCH(2);
  else GT_LAUNCH(1);
#undef GT_LAUNCH
  PIPNN_LAUNCHED("gather_tiled_kernel", c.st);
  return PIPNN_OK;
}

// ------------------------------------------------------------------ CSR segments -> DistSegs + items
__global__ void csr_pad_kernel(const int64_t* __restrict__ off, int64_t ns, int64_t* __restrict__ blocks) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < ns) blocks[s] = (off[s + 1] - off[s] + 127) / 128;
}

__global__ void csr_fill_kernel(const int64_t* __restrict__ off, int64_t ns, const int64_t* __restrict__ blocks,
                                const int64_t* __restrict__ bpos, int k, int self, DistSeg* __restrict__ segs,
                                WorkItem* __restrict__ items, int64_t* __restrict__ n_items) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const int64_t nb = blocks[s], p = bpos[s];
  TileSeg t;
  t.id_off = off[s];
  t.pos = p * 128;
  t.pad = (int32_t)(nb * 128);
  t.rows = (int32_t)(off[s + 1] - off[s]);
  DistSeg d;
  d.a = t;
  d.b = t;
  d.out_off = off[s] * k;
  d.k = k;
  d.self = self;
  d.ostride = k;
  d.pad_ = 0;
  segs[s] = d;
  for (int64_t rb = 0; rb < nb; ++rb) items[p + rb] = WorkItem{(int32_t)s, (int32_t)rb};
  if (s == ns - 1) *n_items = p + nb;
}

pipnn_status csr_dist_segs(const int64_t* off, int64_t ns, int k, int self, DistSeg* segs, WorkItem* items,
                           int64_t* n_items, Arena& ar, const Ctx& c) {
  int64_t* blocks = ar.take<int64_t>(ns);
  int64_t* bpos = ar.take<int64_t>(ns);
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, blocks, bpos, (int)ns, c.st);
  void* tmpbuf = ar.take<uint8_t>(tmp);
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (csr_dist_segs)");
  if (ns == 0) {
    PIPNN_CUDA(kmemset(n_items, 0, sizeof(int64_t), c.st));
    return PIPNN_OK;
  }
  const int tb = 256;
  csr_pad_kernel<<<(unsigned)ceil_div(ns, tb), tb, 0, c.st>>>(off, ns, blocks);
  PIPNN_LAUNCHED("csr_pad_kernel", c.st);
  PIPNN_CUDA(cub::DeviceScan::ExclusiveSum(tmpbuf, tmp, blocks, bpos, (int)ns, c.st));
  csr_fill_kernel<<<(unsigned)ceil_div(ns, tb), tb, 0, c.st>>>(off, ns, blocks, bpos, k, self, segs, items, n_items);
  PIPNN_LAUNCHED("csr_fill_kernel", c.st);
  return PIPNN_OK;
}

// The gather's compact view of the leaf segments (a kernel rather than a strided copy-engine copy).
__global__ void tileseg_view_kernel(const DistSeg* __restrict__ segs, int64_t n, TileSeg* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = segs[i].a;
}

// ------------------------------------------------------------------ leaf pick
int64_t leaf_items_bound(int64_t n_leaves, int64_t n_inst) { return n_inst / 128 + n_leaves + 1; }

pipnn_status leaf_pick_impl(const pipnn_points* X, const int64_t* leaf_off, const uint32_t* leaf_ids, int64_t n_leaves,
                            int64_t n_inst, int k, uint32_t* nbr, float* dist, Arena& ar, const Ctx& c,
                            int64_t max_items, uint16_t* cols) {
  const int Kb = tiled_row_bytes(X);
  if (max_items <= 0) max_items = leaf_items_bound(n_leaves, n_inst);
  const int64_t seg_cap = std::min<int64_t>(n_leaves, max_items);
  const int64_t max_rows = max_items * 128;
  uint8_t* T = ar.take<uint8_t>((size_t)max_rows * Kb);
  void* nrm = ar.take<int32_t>(max_rows);
  DistSeg* segs = ar.take<DistSeg>(seg_cap);
  WorkItem* items = ar.take<WorkItem>(max_items);
  int64_t* n_items = ar.take<int64_t>(1);
  TileSeg* tsegs = ar.take<TileSeg>(seg_cap);  // compact TileSeg view (seg.a) for the gather kernel
  PIPNN_TRY(csr_dist_segs(leaf_off, seg_cap, k, 1, segs, items, n_items, ar, c));
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (leaf_pick)");
  if (n_leaves == 0 || n_inst == 0) return PIPNN_OK;
  tileseg_view_kernel<<<(unsigned)ceil_div(n_leaves, 256), 256, 0, c.st>>>(segs, n_leaves, tsegs);
  PIPNN_LAUNCHED("tileseg_view_kernel", c.st);
  PIPNN_TRY(gather_tiled(X, leaf_ids, tsegs, items, n_items, max_items, T, nrm, c, Kb));
  DistTopkArgs a{};
  a.Ta = T;
  a.Tb = T;
  a.na = nrm;
  a.nb = nrm;
  a.Kb = Kb;
  a.segs = segs;
  a.items = items;
  a.n_items = n_items;
  a.col_ids = leaf_ids;
  a.out_idx = nbr;
  a.out_col = cols;
  a.out_dist = dist;
  a.err = c.err;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c.tile_events) {
    e0 = pool_event(7 + 2 * c.tile_events->size());
    e1 = pool_event(8 + 2 * c.tile_events->size());
    if (!e0 || !e1) return fail(PIPNN_ECUDA, "timing event");
    PIPNN_CUDA(cudaEventRecord(e0, c.st));
  }
  PIPNN_TRY(launch_dist_topk(a, X->dtype == PIPNN_U8, X->metric == PIPNN_MIPS, k, c.st));
  if (c.tile_events) {
    PIPNN_CUDA(cudaEventRecord(e1, c.st));
    c.tile_events->push_back({e0, e1});
  }
  return PIPNN_OK;
}

}  // namespace pipnn
