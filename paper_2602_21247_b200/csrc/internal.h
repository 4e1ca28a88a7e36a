// internal.h — host-side declarations shared by the libpipnn translation units (not the ABI).
#pragma once
#include <cstdint>
#include <functional>
#include <utility>
#include <vector>
#include <cuda_runtime.h>
#include "common.cuh"
#include "dist_topk.cuh"

namespace pipnn {

struct Ctx {
  cudaStream_t st;
  int* err;  // device error flag (DevErr)
  // optional: event pairs recorded around every distance-tile kernel of the leaf stage (stats)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* tile_events = nullptr;
  // optional: independent work that the partition enqueues behind its first level's read-back, so it fills
  // the GPU while the host plans that level (pipnn_build: the sketches); run by the caller if not taken
  std::function<pipnn_status()>* side_work = nullptr;
  // partition_impl: leave the instance count unread (*n_inst_h = -1); the caller reads leaf_off itself
  bool defer_inst_count = false;
};

// Bytes per row of the tiled (K-major, SWIZZLE_NONE) layout: uint8 -> round_up(d, 32);
// float -> bf16 with round_up(d, 16) elements (so the row is a multiple of 32 B = one MMA K-step).
int tiled_row_bytes(const pipnn_points* X);
pipnn_status validate_points(const pipnn_points* X);

// Gather rows ids[seg.id_off + i] (ids == nullptr: identity) of X into the tiled layout of `T` and their
// squared norms into `nrm` (int32 for uint8, float for bf16-rounded float), one CTA per (segment,
// 128-row block) work item; padding rows are zero. max_items bounds the grid.
pipnn_status gather_tiled(const pipnn_points* X, const uint32_t* ids, const TileSeg* segs, const WorkItem* items,
                          const int64_t* n_items, int64_t max_items, uint8_t* T, void* nrm, const Ctx& c,
                          int Kb = 0 /* 0: tiled_row_bytes(X) */,
                          int packed = 0 /* u8: norms as 32 ||y||^2 + (position mod 32), see DistTopkArgs::packed */,
                          int augp = 0 /* > 0: folded uint8 rows (leaf.cu) with this many augment planes */,
                          uint32_t* par = nullptr /* folded rows: parity bit array */,
                          const float* qstats = nullptr /* NEXT-2: per-segment (centre[d], 1/scale) of bf16 rows X */);
// Folded uint8 rows (leaf.cu): augment planes for dimension d, and the row bytes (0 = not available for d).
int fold_aug_planes(int d);
int fold_row_bytes(int d);

// Build TileSegs/items for CSR segments (off[0..ns]) with pad = round_up(rows, 128): writes segs
// (DistSeg with a == b, self = 1, out_row = off[s], k) and the (segment, row-block) items.
pipnn_status csr_dist_segs(const int64_t* off, int64_t ns, int k, int self, DistSeg* segs, WorkItem* items,
                           int64_t* n_items, Arena& ar, const Ctx& c, int rebase = 0 /* out_off relative to off[0] */);

// max_items: capacity in 128-row work items (0 = exact bound for these leaves); with an explicit capacity
// the caller guarantees sum_b ceil(|b|/128) <= max_items (pipnn_build forms waves of leaves that fit).
int64_t leaf_items_bound(int64_t n_leaves, int64_t n_inst);
// quant (NEXT-2, float L2): pick by per-leaf scalar-quantised int8 distances, then re-rank exactly (leaf.cu)
pipnn_status leaf_pick_impl(const pipnn_points* X, const int64_t* leaf_off, const uint32_t* leaf_ids, int64_t n_leaves,
                            int64_t n_inst, int k, uint32_t* nbr, float* dist, Arena& ar, const Ctx& c,
                            int64_t max_items = 0, uint16_t* cols = nullptr, int quant = 0);

// fp32 -> bf16 copy of float points (kDtypeBf16 rows of ldb = round_up(d, 8) elements).
pipnn_status to_bf16(const pipnn_points* X, uint16_t* Xb, int ldb, const Ctx& c);
pipnn_status sketch_impl(const pipnn_points* X, int m, uint64_t seed, void* sketch, Arena& ar, const Ctx& c);
// The same with the hyperplane buffer H (m x d int8) given: hyperplanes + sketches, enqueued on c.st.
pipnn_status sketch_launch(const pipnn_points* X, int m, uint64_t seed, void* sketch, int8_t* H, const Ctx& c);

pipnn_status hashprune_impl(int m, int l_max, int64_t n, const void* sketch, bool sk_int, uint64_t* slots,
                            uint32_t* count, const uint32_t* owner, const uint32_t* cand, const float* dist,
                            int64_t n_edges, Arena& ar, const Ctx& c);

// Edge emission + merge for pipnn_build: the bidirected edges of the candidate lists (local columns cols and
// distances dist, [I, k], of the leaves leaf_off/leaf_ids) grouped by owner instance inside each leaf and
// merged into the reservoirs (which must start empty: count = 0).
pipnn_status hashprune_from_leaves(int m, int l_max, int64_t n, const void* sketch, bool sk_int, uint64_t* slots,
                                   uint32_t* count, const int64_t* leaf_off, int64_t n_leaves, const uint32_t* leaf_ids,
                                   int64_t n_inst, int k, const uint16_t* cols, const float* dist, int max_leaf,
                                   int64_t* n_edges_dev, Arena& ar, const Ctx& c,
                                   int inst_per_point);  // leaf instances per point (capacity / n): path choice

// order/order_n (device, nullable): the points to prune, in this order (pipnn_build: leaf order, see
// leaf_order); without it every point in id order.
pipnn_status final_prune_impl(const pipnn_points* X, int l_max, const uint64_t* slots, const uint32_t* count,
                              const pipnn_prune_params* p, uint64_t* row_ptr, uint32_t* col_idx, Arena& ar,
                              const Ctx& c, const uint32_t* order = nullptr, const uint32_t* order_n = nullptr,
                              const pipnn_points* Xb = nullptr);
// Every point once, at its first instance in leaf_ids order (order[0..*order_n)).
pipnn_status leaf_order(const uint32_t* leaf_ids, int64_t n_inst, int64_t n, uint32_t* order, uint32_t* order_n,
                        Arena& ar, const Ctx& c);

// Device carving of whole subtrees below depth 0 (partition_subtree.cu): which subproblems fit, and the launch.
bool subtree_fits(const pipnn_points* X, const pipnn_partition_params* p, int64_t size, int depth);
// Pinned host scratch for small device <-> host transfers (thread-local, grows as needed). Copy kernels read
// or write it asynchronously; every user synchronises the stream before the call returns (on error paths
// too: partition_impl), so nothing is pending when the next call reuses it.
uint8_t* pinned_scratch(size_t bytes);  // mapped pinned host memory, reused per thread (api.cu)
// Stream-ordered copy by a kernel (device <-> mapped pinned host or device), not by a copy engine (api.cu).
cudaError_t kcopy(void* dst, const void* src, size_t bytes, cudaStream_t st);
cudaError_t kmemset(void* dst, int value, size_t bytes, cudaStream_t st);  // likewise for cudaMemsetAsync
struct KCopyDesc {
  void* dst;
  const void* src;
  unsigned long long bytes;
};
// n copies in one kernel; descs in mapped pinned (or device) memory, valid until the kernel has run (api.cu)
cudaError_t kcopy_batch(const KCopyDesc* descs, int n, cudaStream_t st);
cudaEvent_t pool_event(size_t i);  // per-thread, per-device reusable timing event i (api.cu)
// Batched beam search (search.cu, Alg. 1): one warp per query; L <= 256.
size_t search_smem_per_warp(const pipnn_points* X);
pipnn_status search_impl(const pipnn_points* X, const uint64_t* row_ptr, const uint32_t* col_idx, const void* Q,
                         int64_t ldq, int64_t nq, uint32_t entry, int L, int k, int excl, uint32_t* out_ids,
                         float* out_dist, int64_t* n_cmps_dev, const Ctx& c);
size_t subtree_group_bytes();
pipnn_status subtree_launch(const pipnn_points* X, const pipnn_partition_params* p, const void* groups, int n_groups,
                            const uint32_t* mem, uint32_t* staging, int64_t stage_cap, unsigned long long* stage_cursor,
                            int64_t* leaf_dst, int64_t* leaf_size, int64_t leaf_cap, unsigned long long* leaf_count,
                            int* work, int* err, int* max_depth, cudaStream_t st);

pipnn_status partition_impl(const pipnn_points* X, const pipnn_partition_params* p, int64_t* leaf_off,
                            int64_t leaf_off_cap, uint32_t* leaf_ids, int64_t leaf_ids_cap, int64_t* n_leaves_h,
                            int64_t* n_inst_h, int* depth_h, Arena& ar, const Ctx& c);

}  // namespace pipnn
