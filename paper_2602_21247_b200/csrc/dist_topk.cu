// dist_topk.cu — instantiations + launcher of the distance-tile / top-k kernel (dist_topk.cuh).
#include <cstdio>
#include <cstdlib>

#include "dist_topk.cuh"

namespace pipnn {

template <bool U8, bool MIPS, int KMAX>
static pipnn_status launch_one(const DistTopkArgs& a0, cudaStream_t st) {
  DistTopkArgs a = a0;
  const char* dbg_env = std::getenv("PIPNN_DEBUG_EPI");  // experiment hook (read per launch)
  a.dbg = dbg_env ? std::atoi(dbg_env) : 0;
  // threshold-pass tiles: any column subset gives a valid bound; fewer tiles trade pass-1 work for a few more
  // pass-2 candidates (measured: 3 tiles for leaves — C2 u8, and C3/C4 float, whose leaf kernel is bound by
  // the producer/MMA pipeline, so every pass-1 tile costs a B-tile load: C4 leaf tiles 2.70 -> 2.40 ms with 3
  // instead of all; 2 for the partition's K <= 4)
  const char* p1_env = std::getenv(KMAX <= 4 ? "PIPNN_P1_PART" : "PIPNN_P1");
  a.p1cap = p1_env ? std::max(1, std::atoi(p1_env)) : (KMAX <= 4 ? 2 : 3);
  if (a.packed && !(KMAX == 2 && U8)) return fail(PIPNN_EUNSUPPORTED, "dist_topk: packed pass needs uint8, K <= 2");
  if (a.packed) a.p1cap = 0;  // no threshold pass
  const char* geo_env = std::getenv("PIPNN_GEOM");  // experiment hook: "NA,planes per chunk"
  a.geo = 0;
  if (geo_env) {
    int na = 0, pc = 0;
    if (std::sscanf(geo_env, "%d,%d", &na, &pc) == 2 && na >= 1 && na <= 2 && pc >= 2 && pc <= 14) a.geo = 16 * na + pc;
  }
  const DtGeom g = dt_geom(a.Kb, !U8, a.geo);
  if (g.stages < 2) return fail(PIPNN_EUNSUPPORTED, "dist_topk: row too long for the SMEM pipeline");
  auto* fn = dist_topk_kernel<U8, MIPS, KMAX>;
  PIPNN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem));
  fn<<<num_sms(), kDtThreads, g.smem, st>>>(a);
  PIPNN_LAUNCHED("dist_topk_kernel", st);
  return PIPNN_OK;
}

template <bool U8, bool MIPS>
static pipnn_status launch_k(const DistTopkArgs& a, int kmax, cudaStream_t st) {
  if (kmax <= 2) return launch_one<U8, MIPS, 2>(a, st);
  if (kmax <= 4) return launch_one<U8, MIPS, 4>(a, st);
  if (kmax <= 8) return launch_one<U8, MIPS, 8>(a, st);
  if (kmax <= 12) return launch_one<U8, MIPS, 12>(a, st);
  return launch_one<U8, MIPS, 16>(a, st);
}

// kmax: the largest k any segment asks for (self exclusion does not need an extra slot).
pipnn_status launch_dist_topk(const DistTopkArgs& a, bool u8, bool mips, int kmax, cudaStream_t st) {
  if (a.Kb <= 0 || a.Kb % 32 != 0 || a.Kb > 512)
    return fail(PIPNN_EUNSUPPORTED, "dist_topk: row bytes must be a multiple of 32 and <= 512");
  if (kmax > kTopkMax) return fail(PIPNN_EUNSUPPORTED, "dist_topk: k too large (<= 16)");
  if (u8 && mips) return fail(PIPNN_EINVAL, "uint8 + MIPS unsupported");
  if (u8) return launch_k<true, false>(a, kmax, st);
  if (mips) return launch_k<false, true>(a, kmax, st);
  return launch_k<false, false>(a, kmax, st);
}

}  // namespace pipnn

// Experiment hook: copy out and clear the pipeline wait profile (PIPNN_DEBUG_EPI bit 64).
extern "C" __attribute__((visibility("default"))) int pipnn_debug_dt_prof(unsigned long long* out16) {
  if (cudaMemcpyFromSymbol(out16, pipnn::g_dt_prof, 16 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  static const unsigned long long zero[16] = {};
  return cudaMemcpyToSymbol(pipnn::g_dt_prof, zero, sizeof(zero)) == cudaSuccess ? 0 : 1;
}
