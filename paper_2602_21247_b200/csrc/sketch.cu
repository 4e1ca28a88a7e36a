// sketch.cu — hyperplanes H (docs/DETERMINISM.md) and per-point sketches S(x)_i = H_i . x
// (§3 "Implementation": "pre-compute m-dimensional sketches for each point"; Eq. 1).
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

// One thread per point; H in shared memory. uint8: exact int32. float: the bf16-rounded coordinates
// accumulated in fp64 in ascending j order, then rounded to fp32 (so the value is deterministic and
// reproducible by any in-order fp64 implementation; reading R8).
template <bool U8>
__global__ void __launch_bounds__(128) sketch_kernel(const void* __restrict__ Xv, int64_t n, int d, int64_t ld, int m,
                                                     const int8_t* __restrict__ Hg, void* __restrict__ S) {
  extern __shared__ int8_t Hs[];
  for (int e = threadIdx.x; e < m * d; e += blockDim.x) Hs[e] = Hg[e];
  __syncthreads();
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n) return;
  if (U8) {
    int32_t acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0;
    const uint8_t* row = (const uint8_t*)Xv + x * ld;
    for (int j = 0; j < d; ++j) {
      const int v = row[j];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < m) acc[i] += (int)Hs[i * d + j] * v;
    }
    int32_t* out = (int32_t*)S + x * m;
    for (int i = 0; i < m; ++i) out[i] = acc[i];
  } else {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    const float* row = (const float*)Xv + x * ld;
    for (int j = 0; j < d; ++j) {
      const double v = (double)__uint_as_float((uint32_t)f32_to_bf16_rne(row[j]) << 16);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < m) acc[i] += (double)Hs[i * d + j] * v;
    }
    float* out = (float*)S + x * m;
    for (int i = 0; i < m; ++i) out[i] = (float)acc[i];
  }
}

pipnn_status sketch_impl(const pipnn_points* X, int m, uint64_t seed, void* sketch, Arena& ar, const Ctx& c) {
  int8_t* H = ar.take<int8_t>((size_t)m * X->d);
  if (ar.measuring()) return PIPNN_OK;
  if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small (sketch)");
  const int64_t md = (int64_t)m * X->d;
  hyperplane_kernel<<<(unsigned)ceil_div(md, 256), 256, 0, c.st>>>(m, X->d, seed, H);
  PIPNN_LAUNCHED("hyperplane_kernel", c.st);
  const int smem = (int)md;
  if (X->dtype == PIPNN_U8) {
    if (smem > 48 * 1024)
      PIPNN_CUDA(cudaFuncSetAttribute(sketch_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    sketch_kernel<true><<<(unsigned)ceil_div(X->n, 128), 128, smem, c.st>>>(X->data, X->n, X->d, X->ld, m, H, sketch);
  } else {
    if (smem > 48 * 1024)
      PIPNN_CUDA(cudaFuncSetAttribute(sketch_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    sketch_kernel<false><<<(unsigned)ceil_div(X->n, 128), 128, smem, c.st>>>(X->data, X->n, X->d, X->ld, m, H, sketch);
  }
  PIPNN_LAUNCHED("sketch_kernel", c.st);
  return PIPNN_OK;
}

}  // namespace pipnn
