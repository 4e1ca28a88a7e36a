// dist_topk.cu — instantiations + launcher of the distance-tile / top-k kernel (dist_topk.cuh).
#include <cstdio>
#include <cstdlib>

#include "dist_topk.cuh"
#include "dist_topk_uf2.cuh"

namespace pipnn {

// Experiment hooks, read once per process (environment): PIPNN_DEBUG_EPI (epilogue skips / wait profile),
// PIPNN_P1 / PIPNN_P1_PART (threshold-pass tiles), PIPNN_GEOM ("NA,planes per chunk"), PIPNN_UF2 (bit 0: folded
// uint8 leaves, bit 1: the partition's packed pass on the four-warpgroup dist_topk_uf2_kernel; default 3).
struct DtKnobs {
  int dbg = 0, p1 = 0, p1_part = 0, geo = 0, uf2 = 3;
  DtKnobs() {
    if (const char* e = std::getenv("PIPNN_UF2")) uf2 = std::atoi(e);
    if (const char* e = std::getenv("PIPNN_DEBUG_EPI")) dbg = std::atoi(e);
    if (const char* e = std::getenv("PIPNN_P1")) p1 = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("PIPNN_P1_PART")) p1_part = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("PIPNN_GEOM")) {
      int na = 0, pc = 0;
      if (std::sscanf(e, "%d,%d", &na, &pc) == 2 && na >= 1 && na <= 2 && pc >= 2 && pc <= 14) geo = 16 * na + pc;
    }
  }
};
static const DtKnobs& knobs() {
  static const DtKnobs k;
  return k;
}

template <bool U8, bool MIPS, int KMAX, bool UF = false>
static pipnn_status launch_one(const DistTopkArgs& a0, cudaStream_t st) {
  DistTopkArgs a = a0;
  const DtKnobs& kn = knobs();
  a.dbg = kn.dbg;
  // threshold-pass tiles: any column subset gives a valid bound; fewer tiles trade pass-1 work for more pass-2
  // candidates (measured: 3 tiles for the plain uint8 and float leaves — C3/C4 are bound by the producer/MMA
  // pipeline, so every pass-1 tile costs a B-tile load; 6 for the folded uint8 leaves, C5 leaf pick 88.8 ->
  // 86.1 ms vs 3, whose epilogue pays more for pass-2 candidates than for threshold tiles; 2 for the
  // partition's K <= 4)
  const int p1_req = KMAX <= 4 ? kn.p1_part : kn.p1;
  a.p1cap = p1_req ? p1_req : (KMAX <= 4 ? 2 : (UF ? 6 : 3));
  // folded uint8 leaves: one A slot and a whole tile per ring stage (one copy and one ring commit per tile:
  // C5 leaf pick 91.8 -> 88.8 ms)
  a.geo = kn.geo ? kn.geo : (UF && a.Kb / 16 <= 14 ? 16 + a.Kb / 16 : 0);
  if (a.packed && !(KMAX == 2 && U8)) return fail(PIPNN_EUNSUPPORTED, "dist_topk: packed pass needs uint8, K <= 2");
  if (a.packed) a.p1cap = 0;  // no threshold pass
  if (UF != (a.uf_aug > 0)) return fail(PIPNN_EUNSUPPORTED, "dist_topk: folded layout mismatch");
  if (UF && KMAX == 8 && (kn.uf2 & 1) && !kn.dbg && !a.packed && a.work && uf2_fits(a.Kb, a.uf_aug)) {
    // folded uint8 leaves, k <= 8: two row blocks per item on four epilogue warpgroups (dist_topk_uf2.cuh)
    // threshold pass over 3 tiles (C5 leaf tiles 60.5 ms vs 61.9 at 6, 60.7 at 4: with direct insertion the pass-2
    // threshold tightens as the list fills, so a looser first bound costs less than in dist_topk_kernel)
    if (!kn.p1) a.p1cap = 3;
    const Uf2Geom g2 = uf2_geom(a.Kb, a.uf_aug);
    auto* fn2 = dist_topk_uf2_kernel<8>;
    PIPNN_CUDA(cudaFuncSetAttribute(fn2, cudaFuncAttributeMaxDynamicSharedMemorySize, g2.smem));
    fn2<<<num_sms(), kUf2Threads, g2.smem, st>>>(a);
    PIPNN_LAUNCHED("dist_topk_uf2_kernel", st);
    return PIPNN_OK;
  }
  if (a.pairs != (U8 && !UF && !MIPS && KMAX == 2 && a.packed && dt_packed_pairs(a.Kb) ? 1 : 0))
    return fail(PIPNN_EINVAL, "dist_topk: pair items without the packed uf2 pass (or the reverse)");
  if (a.pairs) {
    // the partition's packed top-2 pass on the same four-warpgroup kernel
    const Uf2Geom g2 = uf2_geom(a.Kb, 0);
    auto* fn2 = dist_topk_uf2_kernel<2, true>;
    PIPNN_CUDA(cudaFuncSetAttribute(fn2, cudaFuncAttributeMaxDynamicSharedMemorySize, g2.smem));
    fn2<<<num_sms(), kUf2Threads, g2.smem, st>>>(a);
    PIPNN_LAUNCHED("dist_topk_uf2_kernel", st);
    return PIPNN_OK;
  }
  const DtGeom g = dt_geom(a.Kb, !U8 ? 2 : a.uf_aug, a.geo);
  if (g.stages < 2) return fail(PIPNN_EUNSUPPORTED, "dist_topk: row too long for the SMEM pipeline");
  auto* fn = dist_topk_kernel<U8, MIPS, KMAX, UF>;
  PIPNN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem));
  fn<<<num_sms(), kDtThreads, g.smem, st>>>(a);
  PIPNN_LAUNCHED("dist_topk_kernel", st);
  return PIPNN_OK;
}

// folded uint8 leaves (DistTopkArgs::uf_aug > 0)
static pipnn_status launch_uf(const DistTopkArgs& a, int kmax, cudaStream_t st) {
  if (kmax <= 2) return launch_one<true, false, 2, true>(a, st);
  if (kmax <= 4) return launch_one<true, false, 4, true>(a, st);
  if (kmax <= 8) return launch_one<true, false, 8, true>(a, st);
  if (kmax <= 12) return launch_one<true, false, 12, true>(a, st);
  return launch_one<true, false, 16, true>(a, st);
}

template <bool U8, bool MIPS>
static pipnn_status launch_k(const DistTopkArgs& a, int kmax, cudaStream_t st) {
  if (kmax <= 2) return launch_one<U8, MIPS, 2>(a, st);
  if (kmax <= 4) return launch_one<U8, MIPS, 4>(a, st);
  if (kmax <= 8) return launch_one<U8, MIPS, 8>(a, st);
  if (kmax <= 12) return launch_one<U8, MIPS, 12>(a, st);
  return launch_one<U8, MIPS, 16>(a, st);
}

bool dt_packed_pairs(int Kb) { return (knobs().uf2 & 2) && !knobs().dbg && uf2_fits(Kb, 0, true); }

// kmax: the largest k any segment asks for (self exclusion does not need an extra slot).
pipnn_status launch_dist_topk(const DistTopkArgs& a, bool u8, bool mips, int kmax, cudaStream_t st) {
  if (a.Kb <= 0 || a.Kb % 32 != 0 || a.Kb > 512)
    return fail(PIPNN_EUNSUPPORTED, "dist_topk: row bytes must be a multiple of 32 and <= 512");
  if (kmax > kTopkMax) return fail(PIPNN_EUNSUPPORTED, "dist_topk: k too large (<= 16)");
  if (u8 && mips) return fail(PIPNN_EINVAL, "uint8 + MIPS unsupported");
  if (u8 && a.uf_aug > 0) return launch_uf(a, kmax, st);
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
