// sketch.cu — hyperplanes H (docs/DETERMINISM.md) and per-point sketches S(x)_i = H_i . x
// (§3 "Implementation": "pre-compute m-dimensional sketches for each point"; Eq. 1).
#include <algorithm>

#include "internal.h"

namespace pipnn {

// H[i][j] = sum_{t<4} (2 u_t - 31), u_t = top 5 bits of mix(mix(seed, DOM_H), 4(i d + j) + t).
__global__ void hyperplane_kernel(int m, int d, uint64_t seed, int8_t* __restrict__ H) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * d) return;
  const uint64_t sH = mix64(seed, kDomHyper);
  int v = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) v += 2 * (int)(mix64(sH, 4ull * (uint64_t)e + t) >> 59) - 31;
  H[e] = (int8_t)v;
}

// One thread per point; H in shared memory (uint8: packed as 32-bit words of 4 int8, read by broadcast).
// uint8: exact int32 — 4 coordinates per dp4a (s8 x u8), the row read with 16-B loads when aligned.
// float: the bf16-rounded coordinates accumulated in fp64 in ascending j order, then rounded to fp32 (so the
// value is deterministic and reproducible by any in-order fp64 implementation; reading R8).
__device__ __forceinline__ int32_t dp4a_su(uint32_t h_s8x4, uint32_t x_u8x4, int32_t acc) {
  int32_t r;
  asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(h_s8x4), "r"(x_u8x4), "r"(acc));
  return r;
}

// Float paths: H as fp64 in SMEM, [dp][MP] (MP = m rounded up to even): the m weights of coordinate j are
// read as broadcast 16-B pairs (no int8 -> fp64 conversion per multiply-add).
__host__ __device__ __forceinline__ int sketch_mp(int m) { return (m + 1) & ~1; }

template <int SRC>  // 0: uint8, 1: float32, 2: bf16 (kDtypeBf16)
__global__ void __launch_bounds__(128) sketch_kernel(const void* __restrict__ Xv, int64_t n, int d, int64_t ld, int m,
                                                     const int8_t* __restrict__ Hg, void* __restrict__ S) {
  extern __shared__ __align__(16) int8_t Hs[];  // uint8: [m][dp] int8 with dp = round_up(d, 16), zero padded
  double* Hd = reinterpret_cast<double*>(Hs);   // float: [dp][MP] fp64, zero padded
  const int dp = (d + 15) & ~15;
  const int MP = sketch_mp(m);
  if (SRC == 0) {
    for (int e = threadIdx.x; e < m * dp; e += blockDim.x) {
      const int i = e / dp, j = e - i * dp;
      Hs[e] = j < d ? Hg[i * d + j] : (int8_t)0;
    }
  } else {
    for (int e = threadIdx.x; e < dp * MP; e += blockDim.x) {
      const int j = e / MP, i = e - j * MP;
      Hd[e] = (i < m && j < d) ? (double)Hg[i * d + j] : 0.0;
    }
  }
  __syncthreads();
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n) return;
  constexpr bool U8 = SRC == 0;
  if (U8) {
    int32_t acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0;
    const uint8_t* row = (const uint8_t*)Xv + x * ld;
    const bool vec = ((d & 15) == 0) && ((ld & 15) == 0);
    for (int j0 = 0; j0 < dp; j0 += 16) {
      uint32_t w[4];
      if (vec) {
        const uint4 q = __ldg((const uint4*)(row + j0));
        w[0] = q.x; w[1] = q.y; w[2] = q.z; w[3] = q.w;
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          uint32_t v = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int j = j0 + 4 * t + b;
            if (j < d) v |= (uint32_t)row[j] << (8 * b);
          }
          w[t] = v;
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < m) {
          const uint4 h = *(const uint4*)(Hs + i * dp + j0);
          acc[i] = dp4a_su(h.x, w[0], acc[i]);
          acc[i] = dp4a_su(h.y, w[1], acc[i]);
          acc[i] = dp4a_su(h.z, w[2], acc[i]);
          acc[i] = dp4a_su(h.w, w[3], acc[i]);
        }
      }
    }
    int32_t* out = (int32_t*)S + x * m;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < m) out[i] = acc[i];
  } else {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    if (SRC == 2) {
      const uint16_t* row = (const uint16_t*)Xv + x * ld;  // already bf16, zero padded to ld (multiple of 8)
      for (int j0 = 0; j0 < d; j0 += 8) {
        const uint4 q = __ldg((const uint4*)(row + j0));
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (j0 + t < d) {
            const double v = (double)__uint_as_float(((w[t >> 1] >> (16 * (t & 1))) & 0xFFFFu) << 16);
            const double2* h2 = reinterpret_cast<const double2*>(Hd + (j0 + t) * MP);
#pragma unroll
            for (int i = 0; i < 16; i += 2)
              if (i < m) {
                const double2 h = h2[i >> 1];
                acc[i] += h.x * v;
                acc[i + 1] += h.y * v;  // (i + 1 == MP - 1 > m - 1: a zero weight into an unused accumulator)
              }
          }
        }
      }
    } else {
    const float* row = (const float*)Xv + x * ld;
    const bool vec = ((d & 3) == 0) && ((ld & 3) == 0);
    for (int j0 = 0; j0 < d; j0 += 4) {
      float f[4];
      if (vec) {
        const float4 q = __ldg((const float4*)(row + j0));
        f[0] = q.x; f[1] = q.y; f[2] = q.z; f[3] = q.w;
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) f[t] = j0 + t < d ? row[j0 + t] : 0.0f;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double v = (double)__uint_as_float((uint32_t)f32_to_bf16_rne(f[t]) << 16);
        const double2* h2 = reinterpret_cast<const double2*>(Hd + (j0 + t) * MP);
#pragma unroll
        for (int i = 0; i < 16; i += 2)
          if (i < m) {
            const double2 h = h2[i >> 1];
            acc[i] += h.x * v;
            acc[i + 1] += h.y * v;
          }
      }
    }
    }
    float* out = (float*)S + x * m;
#pragma unroll
    for (int i = 0; i < 16; ++i)  // static indices: acc stays in registers
      if (i < m) out[i] = (float)acc[i];
  }
}

// fp32 -> bf16 (RNE) copy of float data, rows of ldb = round_up(d, 8) elements zero padded; non-finite input
// raises DERR_NONFINITE. Thread per 8 output elements (two 16-B loads when aligned, one 16-B store).
__global__ void to_bf16_kernel(const float* __restrict__ X, int64_t n, int d, int64_t ld, int ldb,
                               uint16_t* __restrict__ Xb, int* err) {
  const int cpr = ldb >> 3;
  const bool vec = (d & 7) == 0 && (ld & 3) == 0;
  const int64_t total = n * cpr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r;
    int ch;
    if (total < (1ll << 32)) {  // 32-bit division when it fits (it does up to 2^32 chunks)
      const uint32_t e32 = (uint32_t)e, r32 = e32 / (uint32_t)cpr;
      r = r32;
      ch = (int)(e32 - r32 * (uint32_t)cpr);
    } else {
      r = e / cpr;
      ch = (int)(e - r * cpr);
    }
    const float* src = X + r * ld + ch * 8;
    float f[8];
    if (vec) {
      const float4 a = __ldg((const float4*)src), b = __ldg((const float4*)src + 1);
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) f[t] = ch * 8 + t < d ? __ldg(src + t) : 0.0f;
    }
    bool bad = false;
    uint32_t w[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      bad |= !isfinite(f[2 * t]) || !isfinite(f[2 * t + 1]);
      w[t] = (uint32_t)f32_to_bf16_rne(f[2 * t]) | ((uint32_t)f32_to_bf16_rne(f[2 * t + 1]) << 16);
    }
    if (bad) atomicExch(err, DERR_NONFINITE);
    *(uint4*)(Xb + r * ldb + ch * 8) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

pipnn_status to_bf16(const pipnn_points* X, uint16_t* Xb, int ldb, const Ctx& c) {
  const int64_t work = X->n * (ldb / 8);
  to_bf16_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), num_sms() * 32)), 256, 0,
                   c.st>>>((const float*)X->data, X->n, X->d, X->ld, ldb, Xb, c.err);
  PIPNN_LAUNCHED("to_bf16_kernel", c.st);
  return PIPNN_OK;
}

pipnn_status sketch_impl(const pipnn_points* X, int m, uint64_t seed, void* sketch, Arena& ar, const Ctx& c) {
  int8_t* H = ar.take<int8_t>((size_t)m * X->d);
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (sketch)");
  return sketch_launch(X, m, seed, sketch, H, c);
}

pipnn_status sketch_launch(const pipnn_points* X, int m, uint64_t seed, void* sketch, int8_t* H, const Ctx& c) {
  const int64_t md = (int64_t)m * X->d;
  hyperplane_kernel<<<(unsigned)ceil_div(md, 256), 256, 0, c.st>>>(m, X->d, seed, H);
  PIPNN_LAUNCHED("hyperplane_kernel", c.st);
  const int64_t dp = (X->d + 15) & ~15;
  const int smem = (int)(X->dtype == PIPNN_U8 ? (int64_t)m * dp : dp * sketch_mp(m) * (int64_t)sizeof(double));
  if (smem > 227 * 1024) return fail(PIPNN_EUNSUPPORTED, "sketch: d too large for the SMEM hyperplane table");
#define SK_LAUNCH(SRC)                                                                                             \
  do {                                                                                                             \
    if (smem > 48 * 1024)                                                                                          \
      PIPNN_CUDA(cudaFuncSetAttribute(sketch_kernel<SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));     \
    sketch_kernel<SRC><<<(unsigned)ceil_div(X->n, 128), 128, smem, c.st>>>(X->data, X->n, X->d, X->ld, m, H, sketch); \
  } while (0)
  if (X->dtype == PIPNN_U8) SK_LAUNCH(0);
  else if (X->dtype == kDtypeBf16) SK_LAUNCH(2);
  else SK_LAUNCH(1);
#undef SK_LAUNCH
  PIPNN_LAUNCHED("sketch_kernel", c.st);
  return PIPNN_OK;
}

}  // namespace pipnn
