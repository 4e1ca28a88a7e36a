// dist_topk.cu — instantiations + launcher of the distance-tile / top-k kernel (dist_topk.cuh).
#include <cstdlib>

#include "dist_topk.cuh"

namespace pipnn {

template <bool U8, bool MIPS, int KMAX>
static pipnn_status launch_one(const DistTopkArgs& a0, cudaStream_t st) {
  DistTopkArgs a = a0;
  const char* dbg_env = std::getenv("PIPNN_DEBUG_EPI");  // experiment hook (read per launch)
  a.dbg = dbg_env ? std::atoi(dbg_env) : 0;
  const int smem = dt_smem_bytes(a.Kb, U8);
  if (dt_stages(a.Kb, U8) < 2) return fail(PIPNN_EUNSUPPORTED, "dist_topk: row too long for the SMEM pipeline");
  auto* fn = dist_topk_kernel<U8, MIPS, KMAX>;
  PIPNN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  fn<<<num_sms(), kDtThreads, smem, st>>>(a);
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
