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

// ------------------------------------------------------------------ folded uint8 rows (leaf self-join, L2)
// For uint8 L2 leaves the row is stored as s8 coordinates b = y - 128 (y ^ 0x80; zero beyond d) followed by
// augment K-steps of s8 digits g_e(y) that the MMA multiplies with constant A-side weights w_e (127 for every
// entry but the last, whose weight is 1; dist_topk.cuh UF), so that with A = B = the same rows
//   acc = sum_i (x_i - 128)(y_i - 128) + sum_e w_e g_e(y)
//       = x.y - 128 sum(x) - 128 sum(y) + 16384 d + (E_y - OFF),      E_y = 128 sum(y) - ceil(||y||^2 / 2)
//       = x.y - ceil(||y||^2 / 2) + R_x,                               R_x = 16384 d - 128 sum(x) - OFF.
// E_y = sum_i y_i (128 - y_i / 2) (+1/2 if ||y||^2 is odd) lies in [0, 8192 d]; OFF = 127 floor(8192 d / 254)
// centres it. With p_y = ||y||^2 mod 2, the key ||y||^2 - 2 x.y = 2 R_x - (2 acc + p_y): larger acc is nearer,
// exactly, and D(x, y) = (||x||^2 + 2 R_x) + key_l with key_l = -2 acc - p_y. Every partial sum is an exact
// integer (|acc| < 2^24). Per position the gather also writes base = ||x||^2 + 2 R_x (int32) and the parity
// bit p (u32 bit array).
int fold_aug_planes(int d) {
  const int F = 8192 * d / 254;
  for (int st = 1; st <= 8; ++st)
    if ((32 * st - 1) * 126 >= F + 2) return 2 * st;  // digits stay within [-128, 127]
  return 0;
}
int fold_row_bytes(int d) {
  const int ap = fold_aug_planes(d);
  const int kb = (int)round_up(d, 32) + 16 * ap;
  return (ap > 0 && kb <= 512) ? kb : 0;  // 0: no folded layout (the plain uint8 rows are used)
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
// SRC 0: uint8, 1: float32, 2: bf16 (kDtypeBf16), 3: uint8 folded (nrm = base, par = parity bits), 4: bf16 rows
// scalar-quantised per leaf (qstats, NEXT-2) into the folded uint8 layout
template <int SRC>
__global__ void __launch_bounds__(128) gather_tiled_kernel(const void* __restrict__ Xv, int64_t ld, int d, int Kb,
                                                           int mips, const uint32_t* __restrict__ ids,
                                                           const TileSeg* __restrict__ segs,
                                                           const WorkItem* __restrict__ items,
                                                           const int64_t* __restrict__ n_items, uint8_t* __restrict__ T,
                                                           void* __restrict__ nrm, int* err, int packed,
                                                           int augp, uint32_t* __restrict__ par,
                                                           const float* __restrict__ qstats) {
  constexpr bool U8 = SRC == 0 || SRC == 3 || SRC == 4;
  constexpr bool UF = SRC == 3 || SRC == 4;
  if ((int64_t)blockIdx.x >= *n_items) return;
  const WorkItem w = items[blockIdx.x];
  const TileSeg S = segs[w.seg];
  const int r = threadIdx.x;  // row within the 128-row block
  const int local = w.rb * 128 + r;
  const bool valid = local < S.rows;
  const int KC = Kb >> 4;
  const int ldm = U8 ? Kb - 16 * augp : (Kb - 32) / 2;  // elements of the coordinate part (float: bf16 elements)
  const int ncc = U8 ? (ldm >> 4) : (ldm >> 3);          // 16-B chunks holding coordinates
  uint8_t* dst = T + (S.pos / 128 + w.rb) * (int64_t)KC * 2048 + r * 16;
  const int64_t id = valid ? (ids ? (int64_t)ids[S.id_off + local] : (S.id_off + local)) : 0;
  int32_t ni = 0, sy = 0;
  float nf = 0.0f;
  bool bad = false;
  const bool vec = SRC == 4 ? true : (U8 ? ((d & 15) == 0 && (ld & 15) == 0) : ((d & 3) == 0 && (ld & 3) == 0));
  const float* qs = SRC == 4 ? qstats + (int64_t)w.seg * (d + 1) : nullptr;  // centre [d], inverse scale
  // uint8 rows of <= 128 B: every chunk of the row loaded before any is processed (8 loads in flight per lane)
  uint4 pre[8];
  const bool batch = (SRC == 0 || SRC == 3) && vec && ncc <= 8;
  if (batch) {
#pragma unroll
    for (int kc = 0; kc < 8; ++kc)
      pre[kc] = (valid && kc < ncc && kc * 16 < d) ? __ldg((const uint4*)((const uint8_t*)Xv + id * ld) + kc)
                                                   : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll 4
  for (int kc = 0; kc < ncc; ++kc) {
    uint4 out = make_uint4(0u, 0u, 0u, 0u);
    if (valid) {
      if (SRC == 4) {
        // y_j = clamp(rint((x_j - c_j) / s), -127, 127) + 128 of the bf16 coordinates (ld = bf16 row stride)
        const uint16_t* src = (const uint16_t*)Xv + id * ld;
        const float inv_s = qs[d];
        uint32_t wv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e0 = kc * 16 + 8 * h;
          uint4 raw = make_uint4(0u, 0u, 0u, 0u);
          if (e0 < d) raw = __ldg((const uint4*)(src + e0));  // rows zero padded to ld (a multiple of 8)
          const uint32_t rw[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int j = e0 + t;
            if (j < d) {
              const float x = __uint_as_float((t & 1) ? (rw[t >> 1] & 0xFFFF0000u) : (rw[t >> 1] << 16));
              const float qf = fminf(fmaxf(rintf((x - __ldg(qs + j)) * inv_s), -127.0f), 127.0f);
              wv[(8 * h + t) >> 2] |= (uint32_t)((int)qf + 128) << (8 * (t & 3));
            }
          }
        }
        out = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        ni = (int32_t)__dp4a(out.x, out.x, (uint32_t)ni);
        ni = (int32_t)__dp4a(out.y, out.y, (uint32_t)ni);
        ni = (int32_t)__dp4a(out.z, out.z, (uint32_t)ni);
        ni = (int32_t)__dp4a(out.w, out.w, (uint32_t)ni);
        sy = (int32_t)__dp4a(out.x, 0x01010101u, (uint32_t)sy);
        sy = (int32_t)__dp4a(out.y, 0x01010101u, (uint32_t)sy);
        sy = (int32_t)__dp4a(out.z, 0x01010101u, (uint32_t)sy);
        sy = (int32_t)__dp4a(out.w, 0x01010101u, (uint32_t)sy);
        const int nb = d - kc * 16;
        uint32_t xm[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int b = nb - 4 * t;
          xm[t] = b >= 4 ? 0x80808080u : (b <= 0 ? 0u : (0x80808080u >> (8 * (4 - b))));
        }
        out = make_uint4(out.x ^ xm[0], out.y ^ xm[1], out.z ^ xm[2], out.w ^ xm[3]);
      } else if (U8) {
        const uint8_t* src = (const uint8_t*)Xv + id * ld;
        if (batch) {
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t == kc) out = pre[t];
        } else if (vec) {
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
        if (UF) {
          sy = (int32_t)__dp4a(out.x, 0x01010101u, (uint32_t)sy);
          sy = (int32_t)__dp4a(out.y, 0x01010101u, (uint32_t)sy);
          sy = (int32_t)__dp4a(out.z, 0x01010101u, (uint32_t)sy);
          sy = (int32_t)__dp4a(out.w, 0x01010101u, (uint32_t)sy);
          // s8 coordinates y - 128 for the bytes inside the row, 0 beyond d
          const int nb = d - kc * 16;
          uint32_t xm[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int b = nb - 4 * t;
            xm[t] = b >= 4 ? 0x80808080u : (b <= 0 ? 0u : (0x80808080u >> (8 * (4 - b))));
          }
          out = make_uint4(out.x ^ xm[0], out.y ^ xm[1], out.z ^ xm[2], out.w ^ xm[3]);
        }
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
  if (UF) {
    // augment digits of E_y - OFF = 127 q + r: q split over the NE - 1 weight-127 entries, r on the weight-1 one
    const int NE = 16 * augp;
    const int32_t OFF = 127 * ((8192 * d) / 254);
    const int32_t E = 128 * sy - ((ni + 1) >> 1);
    const int32_t aug = E - OFF;
    const int32_t q = aug >= 0 ? aug / 127 : -((-aug + 126) / 127);  // floor division
    const int32_t rr = aug - 127 * q;
    const int32_t bq = q >= 0 ? q / (NE - 1) : -((-q + NE - 2) / (NE - 1));
    const int32_t rem = q - bq * (NE - 1);  // in [0, NE - 2]: the first rem digits get bq + 1
    for (int pl = 0; pl < augp; ++pl) {
      uint32_t wv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        uint32_t w = 0;
#pragma unroll
        for (int by = 0; by < 4; ++by) {
          const int e = pl * 16 + 4 * t + by;
          const int32_t g = !valid ? 0 : (e == NE - 1 ? rr : bq + (e < rem ? 1 : 0));
          w |= ((uint32_t)g & 0xFFu) << (8 * by);
        }
        wv[t] = w;
      }
      *(uint4*)(dst + (int64_t)(ncc + pl) * 2048) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
    const int32_t Rx = 16384 * d - 128 * sy - OFF;
    ((int32_t*)nrm)[S.pos + local] = valid ? ni + 2 * Rx : 0;
    const uint32_t pb = __ballot_sync(0xffffffffu, valid && (ni & 1));
    if ((threadIdx.x & 31) == 0) par[(S.pos + local) >> 5] = pb;  // rows 32w .. 32w + 31 of the block
  } else if (U8) {
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
                          int packed, int augp, uint32_t* par, const float* qstats) {
  if (max_items <= 0) return PIPNN_OK;
  if (Kb <= 0) Kb = tiled_row_bytes(X);
  const int64_t ld = X->ld;
#define GT_LAUNCH(SRC)                                                                                             \
  gather_tiled_kernel<SRC><<<(unsigned)max_items, 128, 0, c.st>>>(X->data, ld, X->d, Kb, X->metric == PIPNN_MIPS,   \
                                                                  ids, segs, items, n_items, T, nrm, c.err, packed, \
                                                                  augp, par, qstats)
  if (qstats) GT_LAUNCH(4);
  else if (X->dtype == PIPNN_U8 && augp > 0) GT_LAUNCH(3);
  else if (X->dtype == PIPNN_U8) GT_LAUNCH(0);
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
                                WorkItem* __restrict__ items, int64_t* __restrict__ n_items, int rebase) {
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
  d.out_off = (off[s] - (rebase ? off[0] : 0)) * k;  // rebase: outputs relative to the first segment
  d.k = k;
  d.self = self;
  d.ostride = k;
  d.pad_ = 0;
  segs[s] = d;
  for (int64_t rb = 0; rb < nb; ++rb) items[p + rb] = WorkItem{(int32_t)s, (int32_t)rb};
  if (s == ns - 1) *n_items = p + nb;
}

pipnn_status csr_dist_segs(const int64_t* off, int64_t ns, int k, int self, DistSeg* segs, WorkItem* items,
                           int64_t* n_items, Arena& ar, const Ctx& c, int rebase) {
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
  csr_fill_kernel<<<(unsigned)ceil_div(ns, tb), tb, 0, c.st>>>(off, ns, blocks, bpos, k, self, segs, items, n_items,
                                                                rebase);
  PIPNN_LAUNCHED("csr_fill_kernel", c.st);
  return PIPNN_OK;
}

// The gather's compact view of the leaf segments (a kernel rather than a strided copy-engine copy).
__global__ void tileseg_view_kernel(const DistSeg* __restrict__ segs, int64_t n, TileSeg* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = segs[i].a;
}

// ------------------------------------------------------------------ NEXT-2: scalar-quantised float leaves
static int kQuantExtra = [] {
  const char* e = std::getenv("PIPNN_QUANT_EXTRA");  // experiment hook (read once): extra quantised picks
  return e ? std::max(1, std::atoi(e)) : 4;
}();
// ("quantized GEMM operations"; float L2). Per leaf: centre c_j = (min_j + max_j)
// / 2 of the members' bf16 coordinates and one scale s = max_j (max_j - min_j) / 2 / 127; q = clamp(rint((x - c) /
// s), -127, 127) is stored as the folded uint8 row of y = q + 128 (gather_tiled_kernel<4>), so the int8 kernel ranks
// the leaf's pairs by ||q_x - q_y||^2 (a translation keeps L2 distances and the common s^2 keeps their order, up to
// the rounding of q). It keeps the k2 > k nearest by that; leaf_rerank_kernel recomputes their exact distances
// (fp32 on the bf16 rows) and keeps the k nearest by (D, id).
__global__ void __launch_bounds__(256) leaf_qstats_kernel(const uint16_t* __restrict__ Xb, int64_t ldb, int d,
                                                          const DistSeg* __restrict__ segs, int64_t ns,
                                                          const uint32_t* __restrict__ ids, float* __restrict__ stats) {
  // a warp per member row at a time (lane = 8 consecutive bf16 coordinates per 16-B chunk, chunks strided by 32),
  // per-lane min/max over the warp's rows, then combined over the 8 warps through SMEM
  __shared__ float smin[8][256], smax[8][256], sred[8];
  const int64_t sg = blockIdx.x;
  if (sg >= ns) return;
  const TileSeg A = segs[sg].a;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (d + 7) >> 3;  // <= 30 chunks of 8 (d <= 240)
  float mn[8], mx[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    mn[t] = 3.4e38f;
    mx[t] = -3.4e38f;
  }
  if (lane < nch) {
    for (int r = warp; r < A.rows; r += 8) {
      const uint4 v = __ldg((const uint4*)(Xb + (int64_t)__ldg(ids + A.id_off + r) * ldb) + lane);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float x = __uint_as_float((t & 1) ? (w[t >> 1] & 0xFFFF0000u) : (w[t >> 1] << 16));
        mn[t] = fminf(mn[t], x);
        mx[t] = fmaxf(mx[t], x);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if (lane * 8 + t < 256) {
      smin[warp][lane * 8 + t] = mn[t];
      smax[warp][lane * 8 + t] = mx[t];
    }
  }
  __syncthreads();
  float half = 0.0f;
  const int j = threadIdx.x;
  if (j < d) {
    float a = 3.4e38f, b = -3.4e38f;
    for (int w8 = 0; w8 < 8; ++w8) {
      a = fminf(a, smin[w8][j]);
      b = fmaxf(b, smax[w8][j]);
    }
    stats[sg * (d + 1) + j] = 0.5f * (a + b);
    half = 0.5f * (b - a);
  }
  for (int o = 16; o; o >>= 1) half = fmaxf(half, __shfl_xor_sync(0xffffffffu, half, o));
  if (lane == 0) sred[warp] = half;
  __syncthreads();
  if (threadIdx.x == 0) {
    float h = 0.0f;
    for (int w8 = 0; w8 < 8; ++w8) h = fmaxf(h, sred[w8]);
    stats[sg * (d + 1) + d] = h > 0.0f ? 127.0f / h : 1.0f;  // 1 / s
  }
}

// A half-warp per instance (16 lanes = up to 16 quantised picks; one CTA of 256 threads per 128-row item, 16
// instances per pass): lane e computes candidate e's exact D (direct form, fp32 on the bf16 rows), a 16-lane bitonic
// sort orders (D, column) — column order is id order inside a leaf — and lanes 0..k-1 write the k nearest in the
// output layout of the plain path.
__global__ void __launch_bounds__(256) leaf_rerank_kernel(const uint16_t* __restrict__ Xb, int64_t ldb, int d,
                                                          const DistSeg* __restrict__ segs,
                                                          const WorkItem* __restrict__ items,
                                                          const int64_t* __restrict__ n_items,
                                                          const int64_t* __restrict__ leaf_off,
                                                          const uint32_t* __restrict__ ids, int k2,
                                                          const uint16_t* __restrict__ qcols, int k,
                                                          uint32_t* __restrict__ out_idx, uint16_t* __restrict__ out_col,
                                                          float* __restrict__ out_dist) {
  if ((int64_t)blockIdx.x >= *n_items) return;
  const WorkItem w = items[blockIdx.x];
  const TileSeg A = segs[w.seg].a;
  const int e = threadIdx.x & 15, sub = threadIdx.x >> 4;  // lane in the half-warp, instance slot 0..15
  const int nch = (d + 7) >> 3;
  const int64_t off0 = leaf_off[0];
  for (int r0 = w.rb * 128; r0 < min(A.rows, w.rb * 128 + 128); r0 += 16) {
    const int r = r0 + sub;
    const bool row_ok = r < A.rows;
    const int64_t inst = A.id_off + r;
    uint32_t col = 0xFFFFu;
    float D = __int_as_float(0x7F800000);
    if (row_ok && e < k2) col = qcols[(inst - off0) * k2 + e];
    if (col != 0xFFFFu) {
      const uint16_t* xr = Xb + (int64_t)__ldg(ids + inst) * ldb;
      const uint16_t* yr = Xb + (int64_t)__ldg(ids + A.id_off + col) * ldb;
      float acc = 0.0f;
      for (int ch = 0; ch < nch; ++ch) {
        const uint4 a = __ldg((const uint4*)(xr + 8 * ch)), b = __ldg((const uint4*)(yr + 8 * ch));
        const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float d0 = __uint_as_float(av[q] << 16) - __uint_as_float(bv[q] << 16);
          const float d1 = __uint_as_float(av[q] & 0xFFFF0000u) - __uint_as_float(bv[q] & 0xFFFF0000u);
          acc = fmaf(d0, d0, acc);
          acc = fmaf(d1, d1, acc);
        }
      }
      D = acc;
    }
    // bitonic sort of the 16 (D, column) pairs of the half-warp, ascending (missing picks: +inf, 0xFFFF, last)
#pragma unroll
    for (int size = 2; size <= 16; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const float oD = __shfl_xor_sync(0xffffffffu, D, stride, 16);
        const uint32_t oc = __shfl_xor_sync(0xffffffffu, col, stride, 16);
        const bool other_less = oD < D || (oD == D && oc < col);
        const bool up = (e & size) == 0, lower = (e & stride) == 0;
        if ((lower == up) == other_less) {  // keep the smaller on the lower lane of an ascending pair
          D = oD;
          col = oc;
        }
      }
    }
    if (row_ok && e < k) {
      const bool ok = col != 0xFFFFu;
      if (out_idx) out_idx[inst * k + e] = ok ? ids[A.id_off + col] : 0xFFFFFFFFu;
      if (out_col) out_col[inst * k + e] = ok ? (uint16_t)col : (uint16_t)0xFFFFu;
      if (out_dist) out_dist[inst * k + e] = ok ? D : __int_as_float(0x7F800000);
    }
  }
}

// ------------------------------------------------------------------ leaf pick
int64_t leaf_items_bound(int64_t n_leaves, int64_t n_inst) { return n_inst / 128 + n_leaves + 1; }

int quant_pick_count(int k) { return std::min(16, k + kQuantExtra); }

pipnn_status leaf_pick_impl(const pipnn_points* X, const int64_t* leaf_off, const uint32_t* leaf_ids, int64_t n_leaves,
                            int64_t n_inst, int k, uint32_t* nbr, float* dist, Arena& ar, const Ctx& c,
                            int64_t max_items, uint16_t* cols, int quant) {
  const bool is_float = X->dtype != PIPNN_U8;
  // NEXT-2 (float L2): per-leaf scalar-quantised rows through the folded int8 kernel, then an exact re-rank
  const bool qmode = quant && is_float && X->metric == PIPNN_L2 && fold_row_bytes(X->d) > 0;
  if (quant && is_float && !qmode) return fail(PIPNN_EUNSUPPORTED, "quantised leaf pick: float L2 with d <= 352 only");
  // uint8 L2 leaves: the folded rows (exact int8 MMA that yields the ranking key directly); others: tiled rows
  const bool fold = (X->dtype == PIPNN_U8 && X->metric == PIPNN_L2 && fold_row_bytes(X->d) > 0) || qmode;
  const int Kb = fold ? fold_row_bytes(X->d) : tiled_row_bytes(X);
  const int augp = fold ? fold_aug_planes(X->d) : 0;
  const int kq = qmode ? quant_pick_count(k) : k;  // picks of the distance kernel
  if (max_items <= 0) max_items = leaf_items_bound(n_leaves, n_inst);
  const int64_t seg_cap = std::min<int64_t>(n_leaves, max_items);
  const int64_t max_rows = max_items * 128;
  uint8_t* T = ar.take<uint8_t>((size_t)max_rows * Kb);
  void* nrm = ar.take<int32_t>(max_rows);
  uint32_t* par = fold ? ar.take<uint32_t>(max_rows / 32 + 1) : nullptr;
  DistSeg* segs = ar.take<DistSeg>(seg_cap);
  WorkItem* items = ar.take<WorkItem>(max_items);
  int64_t* n_items = ar.take<int64_t>(1);
  unsigned long long* work = ar.take<unsigned long long>(1);  // dynamic item counter of the distance kernel
  TileSeg* tsegs = ar.take<TileSeg>(seg_cap);  // compact TileSeg view (seg.a) for the gather kernel
  // quantised mode: bf16 rows (the build's copy, or one made here for fp32 input), per-leaf stats, k2 picks
  const bool need_bf16 = qmode && X->dtype != kDtypeBf16;
  const int ldb = (int)round_up(X->d, 8);
  uint16_t* Xb = need_bf16 ? ar.take<uint16_t>((size_t)X->n * ldb) : nullptr;
  float* qstats = qmode ? ar.take<float>((size_t)seg_cap * (X->d + 1)) : nullptr;
  uint16_t* qcols = qmode ? ar.take<uint16_t>((size_t)max_rows * kq) : nullptr;
  PIPNN_TRY(csr_dist_segs(leaf_off, seg_cap, kq, 1, segs, items, n_items, ar, c, qmode ? 1 : 0));
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (leaf_pick)");
  if (n_leaves == 0 || n_inst == 0) return PIPNN_OK;
  tileseg_view_kernel<<<(unsigned)ceil_div(n_leaves, 256), 256, 0, c.st>>>(segs, n_leaves, tsegs);
  PIPNN_LAUNCHED("tileseg_view_kernel", c.st);
  pipnn_points Xq = *X;  // the rows the quantised gather and the re-rank read
  if (qmode) {
    if (need_bf16) PIPNN_TRY(to_bf16(X, Xb, ldb, c));
    Xq.data = need_bf16 ? (const void*)Xb : X->data;
    Xq.ld = need_bf16 ? ldb : X->ld;
    Xq.dtype = kDtypeBf16;
    leaf_qstats_kernel<<<(unsigned)n_leaves, 256, 0, c.st>>>((const uint16_t*)Xq.data, Xq.ld, X->d, segs, n_leaves,
                                                             leaf_ids, qstats);
    PIPNN_LAUNCHED("leaf_qstats_kernel", c.st);
  }
  PIPNN_TRY(gather_tiled(qmode ? &Xq : X, leaf_ids, tsegs, items, n_items, max_items, T, nrm, c, Kb, 0, augp, par,
                         qstats));
  DistTopkArgs a{};
  a.Ta = T;
  a.Tb = T;
  a.na = nrm;
  a.nb = fold ? (const void*)par : nrm;
  a.uf_aug = augp;
  a.work = work;
  PIPNN_CUDA(kmemset(work, 0, sizeof(unsigned long long), c.st));
  a.Kb = Kb;
  a.segs = segs;
  a.items = items;
  a.n_items = n_items;
  a.col_ids = leaf_ids;
  a.out_idx = qmode ? nullptr : nbr;
  a.out_col = qmode ? qcols : cols;
  a.out_dist = qmode ? nullptr : dist;
  a.err = c.err;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c.tile_events) {
    e0 = pool_event(7 + 2 * c.tile_events->size());
    e1 = pool_event(8 + 2 * c.tile_events->size());
    if (!e0 || !e1) return fail(PIPNN_ECUDA, "timing event");
    PIPNN_CUDA(cudaEventRecord(e0, c.st));
  }
  PIPNN_TRY(launch_dist_topk(a, X->dtype == PIPNN_U8 || qmode, X->metric == PIPNN_MIPS, kq, c.st));
  if (c.tile_events) {
    PIPNN_CUDA(cudaEventRecord(e1, c.st));
    c.tile_events->push_back({e0, e1});
  }
  if (qmode) {
    leaf_rerank_kernel<<<(unsigned)max_items, 256, 0, c.st>>>((const uint16_t*)Xq.data, Xq.ld, X->d, segs, items,
                                                              n_items, leaf_off, leaf_ids, kq, qcols, k, nbr, cols,
                                                              dist);
    PIPNN_LAUNCHED("leaf_rerank_kernel", c.st);
  }
  return PIPNN_OK;
}

}  // namespace pipnn
