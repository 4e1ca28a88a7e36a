/* pipnn.h — C ABI of the B200-native PiPNN build hot path (arxiv 2602.21247, "PAPER.md" below; the CPU
 * specification "SPEC.md" is cited as S:line).
 *
 * Conventions (every entry point):
 *   - Pointers are DEVICE pointers unless the parameter name ends in _h (host). Every call enqueues its
 *     kernels on `stream` (a cudaStream_t passed as void*; NULL = legacy default stream).
 *   - The library allocates NO device memory. The caller owns every buffer, including the workspace
 *     `ws` of `ws_bytes` bytes; it must be 256-B aligned. pipnn_workspace_size bounds what pipnn_build
 *     needs; any call made with ws == NULL (or too small) returns PIPNN_EWORKSPACE without launching and
 *     pipnn_required_workspace() then gives its exact requirement (two-call size query).
 *   - Validation happens on the host before any launch; a rejected call writes no output.
 *   - Status: PIPNN_OK on success. On any other status pipnn_last_error() returns a thread-local
 *     message (for PIPNN_ECAPACITY / PIPNN_EWORKSPACE it names the required size).
 *   - Calls that return host-side counts (pipnn_partition, pipnn_build) synchronise `stream`. The other
 *     calls return once their work is enqueued; an asynchronous kernel fault surfaces as PIPNN_ECUDA
 *     from the next call on the stream. With PIPNN_SYNC_DEBUG=1 in the environment every kernel is
 *     followed by a stream synchronisation so a fault is attributed to its kernel.
 *   - Reentrant given distinct buffers. No torch types: plain pointers and sizes.
 *
 * Dissimilarity: squared L2 sum (x_i - y_i)^2 or MIPS -<x,y>. uint8 data is computed
 * exactly (int8 tensor-core MMA, int32 accumulation); float32 data is computed on bf16-rounded inputs
 * with fp32 accumulation (north_star; reading R19).
 */
#ifndef PIPNN_H
#define PIPNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PIPNN_ABI_VERSION 2

#if defined(__GNUC__)
#define PIPNN_API __attribute__((visibility("default")))
#else
#define PIPNN_API
#endif

typedef enum {
  PIPNN_OK = 0,
  PIPNN_EINVAL = 1,      /* bad argument (null pointer, bad size, unsupported combination) */
  PIPNN_ECAPACITY = 2,   /* an output capacity is too small; required size in pipnn_last_error() */
  PIPNN_EWORKSPACE = 3,  /* ws_bytes < pipnn_workspace_size(); required size in pipnn_last_error() */
  PIPNN_ECUDA = 4,       /* CUDA runtime error or device-side fault (bounded-wait timeout, bad data) */
  PIPNN_EUNSUPPORTED = 5 /* valid request outside what this build supports (e.g. m > 16) */
} pipnn_status;

typedef enum { PIPNN_U8 = 0, PIPNN_F32 = 1 } pipnn_dtype;   /* Table 1 element types in scope */
typedef enum { PIPNN_L2 = 0, PIPNN_MIPS = 1 } pipnn_metric; /* squared L2; MIPS as -<x,y> */

/* The point set X: n rows of d elements, row-major, row stride `ld` ELEMENTS (ld >= d).
 * uint8 supports L2 only. float32 rows must be finite. */
typedef struct {
  const void* data;
  int64_t n;
  int32_t d, ld;
  int32_t dtype;  /* pipnn_dtype */
  int32_t metric; /* pipnn_metric */
} pipnn_points;

/* Alg. 5 constants: C_max, C_min, P_samp (exact rational p_samp_num/p_samp_den, so the leader
 * count l = min(leader_cap, max(2, ceil(num*|P|/den)), |P|) is an integer computation), the fanout per
 * depth (implicitly 1 beyond n_fanout), replicas, seed.
 * Requires 1 <= c_min, 3*c_min < c_max (merge bound, R15), c_max <= 4096, leader_cap >= 2,
 * 1 <= fanout[i] <= 16, 1 <= n_fanout <= 4, replicas >= 1. */
typedef struct {
  int32_t c_max, c_min;
  int32_t p_samp_num, p_samp_den;
  int32_t leader_cap;
  int32_t fanout[4];
  int32_t n_fanout;
  int32_t replicas;
  uint64_t seed;
} pipnn_partition_params;

/* Leaf pick: bidirected k-NN inside every leaf. 1 <= k <= 15.
 * quant ("quantized GEMM operations"): 0 = the exact path (uint8: exact int8 MMA; float:
 * bf16 MMA). 1 = float L2 data only: every leaf is scalar-quantised (per-leaf centre and one scale, int8 codes), the
 * int8 tensor-core kernel keeps the min(16, k + 8) nearest by the quantised distance and they are re-ranked with
 * the exact bf16-input distances (the k nearest by (D, id) among them are returned). uint8 data ignores it;
 * float MIPS with quant = 1 is PIPNN_EUNSUPPORTED. */
typedef struct {
  int32_t k;
  int32_t quant;
} pipnn_pick_params;

/* HashPrune (Alg. 3): m hash bits (1..16, default 12 per P:636), l_max reservoir slots
 * (1..1024), hyperplane seed. */
typedef struct {
  int32_t m, l_max;
  uint64_t seed;
} pipnn_hashprune_params;

/* Final prune: RobustPrune (Alg. 2) with alpha = alpha_num/alpha_den (1 <= terms <= 127, so
 * uint8 alpha tests stay exact in 32-bit integers), max degree R (1..256). final_prune = 0 keeps the R
 * nearest reservoir entries instead. */
typedef struct {
  int32_t R;
  int32_t alpha_num, alpha_den;
  int32_t final_prune;
} pipnn_prune_params;

/* "BP", the hyper-parameter bag of Alg. 4. */
typedef struct {
  pipnn_partition_params part;
  pipnn_pick_params pick;
  pipnn_hashprune_params hp;
  pipnn_prune_params prune;
} pipnn_build_params;

/* Per-stage device times (CUDA events on `stream`) and counters of the last pipnn_build. */
typedef struct {
  int64_t n_leaves, n_instances, n_edges, max_leaf;
  int64_t leaf_pairs; /* sum over leaves of |b|^2: the leaf distance work is 2 * leaf_pairs * d ops */
  int32_t depth;
  float ms_prep, ms_partition, ms_leaf, ms_hashprune, ms_final, ms_total;
  float ms_leaf_tiles; /* the distance-tile kernel(s) of the leaf stage alone (events around the launches) */
} pipnn_stats;

/* Reservoir slot layout (part of the ABI; "4-byte ID, 2-byte hash, bf16 norm"):
 *   u64 slot = hash << 48 | okey(bf16(D)) << 32 | id,   okey(b) = b ^ (b & 0x8000 ? 0xFFFF : 0x8000)
 * so u64 order = (hash, dist, id). A reservoir holds `count` slots sorted ascending by hash, one per
 * hash value; unused slots are UINT64_MAX. Arena: slots[n * l_max], count[n]. */

PIPNN_API const char* pipnn_last_error(void);
PIPNN_API int32_t pipnn_abi_version(void);
/* Number of kernels this library has launched in this process (diagnostic; CUB scans/sorts it runs
 * internally are not counted). */
PIPNN_API uint64_t pipnn_launch_count(void);
/* After a call returned PIPNN_EWORKSPACE (e.g. a size query with ws == NULL): the bytes it needs. */
PIPNN_API size_t pipnn_required_workspace(void);

/* Upper bound of the workspace every call below needs for X and p (host-only computation). */
PIPNN_API pipnn_status pipnn_workspace_size(const pipnn_points* X, const pipnn_build_params* p, size_t* bytes_h);

/* Alg. 5 Randomized Ball Carving with fanout and merging of small groups (R10-R16).
 * Output: the overlapping LeafSet as CSR, each leaf's ids ascending (canonical form): leaf b holds
 * leaf_ids[leaf_off[b] .. leaf_off[b+1]). Leaf order is unspecified (breadth-first by depth here).
 * Capacities: leaf_ids_cap >= n * prod(fanout) * replicas, leaf_off_cap >= leaf_ids_cap + 1 suffice.
 * Synchronises `stream` (one small device->host copy per recursion depth). */
PIPNN_API pipnn_status pipnn_partition(const pipnn_points* X, const pipnn_partition_params* p, void* ws, size_t ws_bytes,
                             int64_t* leaf_off, int64_t leaf_off_cap, uint32_t* leaf_ids, int64_t leaf_ids_cap,
                             int64_t* n_leaves_h, int64_t* n_instances_h, void* stream);

/* Leaf building: for every instance i (a position in leaf_ids) of point p = leaf_ids[i] in
 * leaf b, the min(k, |b|-1) nearest co-members q != p by (D(p,q), q), ascending, padded with
 * UINT32_MAX / +inf: nbr[i*k + t] (global id), dist[i*k + t] (D as float). The leaf distance matrix is
 * never written to memory. Requires every leaf size <= 4096 and ids ascending within a leaf. */
PIPNN_API pipnn_status pipnn_leaf_pick(const pipnn_points* X, const int64_t* leaf_off, const uint32_t* leaf_ids,
                             int64_t n_leaves, int64_t n_instances, const pipnn_pick_params* p, uint32_t* nbr,
                             float* dist, void* ws, size_t ws_bytes, void* stream);

/* Sketches S(x)_i = H_i . x for the m hyperplanes of docs/DETERMINISM.md: int32 [n*m] for uint8
 * data (exact), float32 [n*m] for float data (fp64 accumulation of the bf16-rounded inputs). */
PIPNN_API pipnn_status pipnn_sketch(const pipnn_points* X, const pipnn_hashprune_params* p, void* sketch, void* ws,
                          size_t ws_bytes, void* stream);

/* Diagnostic: synchronise `stream` and report the device error flag raised by the last call that used
 * workspace `ws` (bounded-wait timeout, non-finite input). PIPNN_OK if none. */
PIPNN_API pipnn_status pipnn_device_error(void* ws, void* stream);

/* HashPrune insert (Alg. 3): stream the directed candidate edges (owner[e] -> cand[e], dissimilarity
 * dist[e]) into the owners' reservoirs. Edges are grouped by owner and each reservoir becomes
 *   top_{l_max by (bf16 dist, id)} { per-hash-bucket minimum of (reservoir U new edges) }
 * — the result Alg. 3 produces for any insertion order (history independence),
 * so repeated calls compose exactly. Before the first call initialise slots to all-ones bytes and count
 * to 0. Bucket = residual hash h_owner(cand) from `sketch`.
 * sketch: as written by pipnn_sketch (sk_dtype PIPNN_U8 => int32 sketches, PIPNN_F32 => float32). */
PIPNN_API pipnn_status hashprune_insert(const pipnn_hashprune_params* p, int64_t n, const void* sketch, int32_t sk_dtype,
                              uint64_t* slots, uint32_t* count, const uint32_t* owner, const uint32_t* cand,
                              const float* dist, int64_t n_edges, void* ws, size_t ws_bytes, void* stream);

/* Final prune (lazy form P:938-942): per point u, candidates = its reservoir, D(u,v)
 * recomputed at path precision, ascending by (D, v); admit c unless an admitted y has
 * alpha_num*D'(y,c) < alpha_den*D'(u,c); stop at R. D' = D for L2; for MIPS the angular dissimilarity
 * 1 - <a,b>/(||a|| ||b||) (R22: alpha >= 1 relaxes the test only on non-negative values). Output
 * CSR: row_ptr[n+1], col_idx (capacity n*R) in admission order. */
PIPNN_API pipnn_status pipnn_final_prune(const pipnn_points* X, const pipnn_hashprune_params* hp, const uint64_t* slots,
                               const uint32_t* count, const pipnn_prune_params* p, uint64_t* row_ptr,
                               uint32_t* col_idx, void* ws, size_t ws_bytes, void* stream);

/* Alg. 4 end to end: partition -> leaf pick -> HashPrune -> final prune -> CSR graph with
 * out-degree <= R. col_idx capacity n*R. *n_edges_h = row_ptr[n]. stats_h may be NULL.
 * Synchronises `stream`. */
PIPNN_API pipnn_status pipnn_build(const pipnn_points* X, const pipnn_build_params* p, void* ws, size_t ws_bytes,
                         uint64_t* row_ptr, uint32_t* col_idx, int64_t* n_edges_h, pipnn_stats* stats_h, void* stream);

/* Diagnostic (the stage-parity tests of the build path): device pointers to the intermediate artefacts the
 * last pipnn_build with the same X and p left in its workspace `ws` — valid until `ws` is used again:
 *   leaf_off [n_leaves+1] i64, leaf_ids [n_instances] u32 (the LeafSet, as pipnn_partition writes it);
 *   cols [n_instances*k] u16: the picks of instance i as local columns of its leaf (0xFFFF = none), in
 *     (D, id) order; dist [n_instances*k] f32: their D (n_leaves, n_instances from pipnn_stats);
 *   sketch [n*m] (int32 for uint8, float32 otherwise); slots [n*l_max] u64 / count [n] u32: the HashPrune
 *     reservoirs before the final prune, slot layout above; inside pipnn_build a reservoir is a set (the
 *     final prune re-sorts it): its first count[u] slots are in hash order, except for owners whose merge
 *     evicted (more buckets than l_max: (dist, id) order) or went through the hash-table kernel (more than 512
 *     streamed keys), and slots at or beyond count[u] are unspecified.
 * Host-only: nothing is launched. */
typedef struct {
  int64_t* leaf_off;
  uint32_t* leaf_ids;
  uint16_t* cols;
  float* dist;
  void* sketch;
  uint64_t* slots;
  uint32_t* count;
} pipnn_build_buffers;
PIPNN_API pipnn_status pipnn_debug_build_buffers(const pipnn_points* X, const pipnn_build_params* p, void* ws,
                                                 size_t ws_bytes, pipnn_build_buffers* out_h);

/* Experiment hook (tools/leaf_exp.py): copies out and clears the distance kernel's wait profile —
 * 16 u64 counters of clock64 cycles summed over the grid, filled only when the process runs with
 * PIPNN_DEBUG_EPI bit 64 set — into out16 (HOST, 16 elements). Returns 0 on success, 1 on a CUDA error. */
PIPNN_API int pipnn_debug_dt_prof(unsigned long long* out16);

/* Batched greedy beam search over a built graph (Alg. 1 BeamSearch), the
 * query side of the k-NN-graph / ANN tasks. Per query: beam of the L best (D, id) seen, start
 * at `entry`; repeatedly expand the first unvisited beam element, adding each out-neighbour that is neither
 * visited nor in the beam; stop when the whole beam is visited; answer = the beam's first k.
 *   queries: DEVICE, [nq, ld_q] of X's dtype (uint8 / float32), row-major; X, row_ptr, col_idx: as built by
 *   pipnn_build (row_ptr[n+1] u64, col_idx u32, any out-degree). 1 <= k <= L <= 256, entry < n.
 *   out_ids [nq, k] u32 (UINT32_MAX past the beam's end), out_dist [nq, k] f32 (nullable): uint8 exact
 *   squared L2; float fp32 squared L2 or -dot (MIPS). n_cmps_dev: nullable DEVICE int64 accumulating the
 *   number of distance evaluations. Workspace: the two-call protocol (ws == NULL -> PIPNN_EWORKSPACE with the
 *   size in pipnn_required_workspace()); holds the device error flag. Asynchronous on `stream`; a visited set
 *   overflow (more than 2048 expansions for one query) is reported as PIPNN_ECAPACITY by the next
 *   synchronising call or pipnn_device_error. */
typedef struct {
  int32_t L, k;
  int32_t exclude_self;  /* 1: query i is base point i (the k-NN-graph task): id i is left out of
                          * its own answer (it still steers the search) */
} pipnn_search_params;
PIPNN_API pipnn_status pipnn_search(const pipnn_points* X, const uint64_t* row_ptr, const uint32_t* col_idx,
                                    const void* queries, int64_t ld_q, int64_t nq, uint32_t entry,
                                    const pipnn_search_params* p, uint32_t* out_ids, float* out_dist,
                                    int64_t* n_cmps_dev, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PIPNN_H */
