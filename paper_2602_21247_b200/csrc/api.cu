// api.cu — the C ABI (include/pipnn.h): validation, workspace sizing, stream plumbing, stage timing.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "internal.h"

namespace pipnn {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static thread_local size_t g_required_ws = 0;

void set_error(const std::string& msg) { g_last_error = msg; }
pipnn_status fail(pipnn_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
bool sync_debug() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("PIPNN_SYNC_DEBUG");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

pipnn_status validate_points(const pipnn_points* X) {
  if (!X) return fail(PIPNN_EINVAL, "X is NULL");
  if (X->n < 1) return fail(PIPNN_EINVAL, "n must be >= 1");
  if (X->n > 0xFFFFFFFEll) return fail(PIPNN_EUNSUPPORTED, "n must fit in 32-bit ids");
  if (X->d < 1 || X->ld < X->d) return fail(PIPNN_EINVAL, "need d >= 1 and ld >= d");
  if (!X->data) return fail(PIPNN_EINVAL, "X->data is NULL");
  // the row loads are 16-B vectors (uint8 rows with 16-B-multiple strides, float4 for float rows)
  if ((reinterpret_cast<uintptr_t>(X->data) & 15) != 0) return fail(PIPNN_EINVAL, "X->data must be 16-B aligned");
  if (X->dtype != PIPNN_U8 && X->dtype != PIPNN_F32) return fail(PIPNN_EINVAL, "dtype must be PIPNN_U8 or PIPNN_F32");
  if (X->metric != PIPNN_L2 && X->metric != PIPNN_MIPS) return fail(PIPNN_EINVAL, "metric must be L2 or MIPS");
  if (X->dtype == PIPNN_U8 && X->metric == PIPNN_MIPS) return fail(PIPNN_EINVAL, "uint8 + MIPS is not supported (S:27)");
  if (tiled_row_bytes(X) > 512)
    return fail(PIPNN_EUNSUPPORTED, "d too large for this build (uint8 d <= 512, float32 d <= 240)");
  return PIPNN_OK;
}

static pipnn_status validate_part(const pipnn_partition_params* p) {
  if (!p) return fail(PIPNN_EINVAL, "partition params NULL");
  if (p->c_max < 2 || p->c_max > 4096) return fail(PIPNN_EINVAL, "c_max must be in [2, 4096]");
  if (p->c_min < 1 || 3ll * p->c_min >= p->c_max) return fail(PIPNN_EINVAL, "need 1 <= c_min and 3*c_min < c_max");
  if (p->p_samp_num < 1 || p->p_samp_den < 1) return fail(PIPNN_EINVAL, "p_samp must be a positive rational");
  if (p->leader_cap < 2 || p->leader_cap > 4096) return fail(PIPNN_EINVAL, "leader_cap must be in [2, 4096]");
  if (p->n_fanout < 1 || p->n_fanout > 4) return fail(PIPNN_EINVAL, "n_fanout must be in [1, 4]");
  for (int i = 0; i < p->n_fanout; ++i)
    if (p->fanout[i] < 1 || p->fanout[i] > 16) return fail(PIPNN_EINVAL, "fanout[i] must be in [1, 16]");
  if (p->replicas < 1 || p->replicas > 64) return fail(PIPNN_EINVAL, "replicas must be in [1, 64]");
  return PIPNN_OK;
}
static pipnn_status validate_hp(const pipnn_hashprune_params* p) {
  if (!p) return fail(PIPNN_EINVAL, "hashprune params NULL");
  if (p->m < 1 || p->m > 16) return fail(PIPNN_EINVAL, "m must be in [1, 16] (2-byte hash, P:446)");
  if (p->l_max < 1 || p->l_max > 1024) return fail(PIPNN_EINVAL, "l_max must be in [1, 1024]");
  return PIPNN_OK;
}
static pipnn_status validate_prune(const pipnn_prune_params* p) {
  if (!p) return fail(PIPNN_EINVAL, "prune params NULL");
  if (p->R < 1 || p->R > 256) return fail(PIPNN_EINVAL, "R must be in [1, 256]");
  if (p->alpha_num < 1 || p->alpha_den < 1 || p->alpha_num > 127 || p->alpha_den > 127)
    return fail(PIPNN_EINVAL, "alpha must be a positive rational alpha_num/alpha_den with terms <= 127");
  return PIPNN_OK;
}

static int64_t prod_fanout(const pipnn_partition_params* p) {
  int64_t f = 1;
  for (int i = 0; i < p->n_fanout; ++i) f *= p->fanout[i];
  return f * p->replicas;
}

// ws == NULL or too small -> PIPNN_EWORKSPACE with the requirement in pipnn_required_workspace()
// (two-call size query).
static pipnn_status check_ws(void* ws, size_t ws_bytes, size_t need) {
  need += 4096;
  g_required_ws = need;
  if (!ws || ws_bytes < need)
    return fail(PIPNN_EWORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(PIPNN_EINVAL, "workspace must be 256-B aligned");
  return PIPNN_OK;
}

// The first 256 B of every workspace hold the device error flag.
static int* err_slot(Arena& ar) { return ar.take<int>(64); }

static pipnn_status pending_cuda() {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(PIPNN_ECUDA, std::string("pending CUDA error: ") + cudaGetErrorString(e));
  }
  return PIPNN_OK;
}

static pipnn_status read_dev_error(int* err, cudaStream_t st) {
  int* hp = reinterpret_cast<int*>(pinned_scratch(sizeof(int)));
  if (!hp) return fail(PIPNN_ECUDA, "pinned host scratch");
  PIPNN_CUDA(kcopy(hp, err, sizeof(int), st));
  PIPNN_CUDA(cudaStreamSynchronize(st));
  const int h = *hp;
  if (h == DERR_NONFINITE) return fail(PIPNN_EINVAL, "non-finite float input");
  if (h != 0) return fail(PIPNN_ECUDA, "device error flag " + std::to_string(h) + " (bounded wait timeout / capacity)");
  return PIPNN_OK;
}

// ------------------------------------------------------------------ build-level workspace plan
struct BuildPlan {
  int64_t leaf_ids_cap, leaf_off_cap;
};
static BuildPlan plan_of(const pipnn_points* X, const pipnn_build_params* p) {
  BuildPlan b;
  b.leaf_ids_cap = X->n * prod_fanout(&p->part);
  b.leaf_off_cap = b.leaf_ids_cap + 1;
  return b;
}

// Timing event i of the calling thread on the current device, created on first use and reused by every later
// build (creating and destroying the stage events per build cost tens of microseconds of host time at the
// start of each build, with the GPU idle).
cudaEvent_t pool_event(size_t i) {
  static thread_local std::map<int, std::vector<cudaEvent_t>> pools;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::vector<cudaEvent_t>& pool = pools[dev];
  while (pool.size() <= i) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    pool.push_back(e);
  }
  return pool[i];
}

// Stream-ordered copy by a kernel between device memory and mapped pinned host memory (UVA pointers). The
// build's small plan uploads and level read-backs then do not queue on the copy engines behind large transfers
// of other streams (a service copying the next input while this build runs: bench.py's pipelined e2e).
__global__ void kcopy_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t bytes) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  size_t done = 0;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const size_t n16 = bytes >> 4;
    for (size_t i = tid; i < n16; i += nt) reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    done = n16 << 4;
  }
  for (size_t i = done + tid; i < bytes; i += nt) dst[i] = src[i];
}
cudaError_t kcopy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  static const bool engine = std::getenv("PIPNN_COPY_ENGINE") != nullptr;  // experiment hook: cudaMemcpyAsync
  if (engine) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
  const unsigned grid = (unsigned)std::min<size_t>(64, (bytes + 4095) / 4096);
  kcopy_kernel<<<grid, 256, 0, st>>>(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes);
  count_launch();
  return cudaGetLastError();
}

// Several copies in one launch: blockIdx.y selects the descriptor, the x blocks split it.
__global__ void kcopy_batch_kernel(const KCopyDesc* __restrict__ descs) {
  const KCopyDesc d = descs[blockIdx.y];
  uint8_t* dst = static_cast<uint8_t*>(d.dst);
  const uint8_t* src = static_cast<const uint8_t*>(d.src);
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  size_t done = 0;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const size_t n16 = d.bytes >> 4;
    for (size_t i = tid; i < n16; i += nt) reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    done = n16 << 4;
  }
  for (size_t i = done + tid; i < d.bytes; i += nt) dst[i] = src[i];
}
cudaError_t kcopy_batch(const KCopyDesc* descs, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  static const bool engine = std::getenv("PIPNN_COPY_ENGINE") != nullptr;  // experiment hook
  if (engine) {
    for (int i = 0; i < n; ++i) {
      cudaError_t e = cudaMemcpyAsync(descs[i].dst, descs[i].src, descs[i].bytes, cudaMemcpyDefault, st);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  unsigned long long mx = 0;
  for (int i = 0; i < n; ++i) mx = std::max(mx, descs[i].bytes);
  const unsigned gx = (unsigned)std::max<unsigned long long>(1, std::min<unsigned long long>(32, (mx + 4095) / 4096));
  kcopy_batch_kernel<<<dim3(gx, (unsigned)n), 256, 0, st>>>(descs);
  count_launch();
  return cudaGetLastError();
}

// Stream-ordered byte fill by a kernel (cudaMemsetAsync's signature), for the same reason as kcopy.
__global__ void kmemset_kernel(uint8_t* __restrict__ dst, uint8_t v, size_t bytes) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  size_t done = 0;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const uint32_t w = 0x01010101u * v;
    const uint4 q = make_uint4(w, w, w, w);
    const size_t n16 = bytes >> 4;
    for (size_t i = tid; i < n16; i += nt) reinterpret_cast<uint4*>(dst)[i] = q;
    done = n16 << 4;
  }
  for (size_t i = done + tid; i < bytes; i += nt) dst[i] = v;
}
cudaError_t kmemset(void* dst, int value, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  static const bool engine = std::getenv("PIPNN_COPY_ENGINE") != nullptr;  // experiment hook: cudaMemsetAsync
  if (engine) return cudaMemsetAsync(dst, value, bytes, st);
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((size_t)num_sms() * 8, (bytes + 4095) / 4096));
  kmemset_kernel<<<grid, 256, 0, st>>>(static_cast<uint8_t*>(dst), (uint8_t)value, bytes);
  count_launch();
  return cudaGetLastError();
}

// Runs the whole build through an Arena; with a measuring Arena it only sizes the workspace.
uint8_t* pinned_scratch(size_t bytes) {
  struct Scratch {
    uint8_t* p = nullptr;
    size_t cap = 0;
    ~Scratch() {
      if (p) cudaFreeHost(p);
    }
  };
  static thread_local Scratch s;
  if (bytes > s.cap) {
    if (s.p) cudaFreeHost(s.p);
    s.p = nullptr;
    s.cap = 0;
    const size_t cap = std::max<size_t>(bytes, (size_t)1 << 16);
    if (cudaHostAlloc((void**)&s.p, cap, cudaHostAllocMapped) != cudaSuccess) return nullptr;  // kcopy'd
    s.cap = cap;
  }
  return s.p;
}

// The build's long-lived buffers, taken first from its workspace in this order (pipnn_debug_build_buffers
// replays the same takes to find them after a build).
struct BuildBufs {
  int* err;
  int64_t* leaf_off;
  uint32_t* leaf_ids;
  uint16_t* cols;  // picks as local leaf columns [I * k]
  float* dist;     // their D [I * k]
  void* sketch;
  uint64_t* slots;
  uint32_t* count;
};
static BuildBufs take_build_bufs(const pipnn_points* X, const pipnn_build_params* p, Arena& ar) {
  const BuildPlan bp = plan_of(X, p);
  BuildBufs b;
  b.err = err_slot(ar);
  b.leaf_off = ar.take<int64_t>(bp.leaf_off_cap);
  b.leaf_ids = ar.take<uint32_t>(bp.leaf_ids_cap);
  b.cols = ar.take<uint16_t>((size_t)bp.leaf_ids_cap * p->pick.k);
  b.dist = ar.take<float>((size_t)bp.leaf_ids_cap * p->pick.k);
  b.sketch = ar.take<int32_t>((size_t)X->n * p->hp.m);
  b.slots = ar.take<uint64_t>((size_t)X->n * p->hp.l_max);
  b.count = ar.take<uint32_t>(X->n);
  return b;
}

static pipnn_status build_impl(const pipnn_points* X, const pipnn_build_params* p, Arena& ar, cudaStream_t st,
                               uint64_t* row_ptr, uint32_t* col_idx, int64_t* n_edges_h, pipnn_stats* stats_h) {
  const BuildPlan bp = plan_of(X, p);
  const BuildBufs B = take_build_bufs(X, p, ar);
  int* err = B.err;
  Ctx c{st, err};
  int64_t* leaf_off = B.leaf_off;
  uint32_t* leaf_ids = B.leaf_ids;
  const int k = p->pick.k;
  uint16_t* cols = B.cols;
  float* dist = B.dist;
  const bool sk_int = X->dtype == PIPNN_U8;
  void* sketch = B.sketch;
  uint64_t* slots = B.slots;
  uint32_t* count = B.count;
  int64_t* n_edges_dev = ar.take<int64_t>(1);
  // float data: one bf16 (RNE) copy of X, made in prep; every later stage gathers its rows (R19)
  const bool is_float = X->dtype != PIPNN_U8;
  const int ldb = (int)round_up(X->d, 8);
  uint16_t* Xb = is_float ? ar.take<uint16_t>((size_t)X->n * ldb) : nullptr;
  pipnn_points Xbv = *X;
  if (is_float) {
    Xbv.data = Xb;
    Xbv.ld = ldb;
    Xbv.dtype = kDtypeBf16;
  }
  const pipnn_points* XS = is_float ? &Xbv : X;  // the rows the stages read
  int8_t* H = ar.take<int8_t>((size_t)p->hp.m * X->d);  // sketch hyperplanes (kept: the sketch runs late)
  const size_t mark = ar.mark();
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tile_ev;
  int64_t leaf_pairs = 0;

  cudaEvent_t ev[7];
  if (!ar.measuring()) {
    if (ar.overflow()) return fail(PIPNN_EWORKSPACE, "workspace too small");
    for (int i = 0; i < 7; ++i)
      if (!(ev[i] = pool_event(i))) return fail(PIPNN_ECUDA, "timing event");
    PIPNN_CUDA(kmemset(err, 0, 256, st));
    PIPNN_CUDA(cudaEventRecord(ev[0], st));
  }
  auto cleanup = [&]() { tile_ev.clear(); };  // (pooled events: nothing to destroy)
  // (a0) bf16 copy (float data); sketches below
  if (is_float && !ar.measuring()) {
    pipnn_status s0 = to_bf16(X, Xb, ldb, c);
    if (s0 != PIPNN_OK) { cleanup(); return s0; }
  }
  // the sketches are needed only by HashPrune: they are enqueued behind the partition's first read-back and
  // run while the host plans that level (or right after the partition if it has no level); H stays reserved
  pipnn_status s = PIPNN_OK;
  if (!ar.measuring()) cudaEventRecord(ev[1], st);
  std::function<pipnn_status()> sketch_work = [&, H]() { return sketch_launch(XS, p->hp.m, p->hp.seed, sketch, H, c); };
  Ctx cp_ctx = c;
  if (!ar.measuring()) cp_ctx.side_work = &sketch_work;
  static const bool dbg_check = std::getenv("PIPNN_DEBUG_CHECK") != nullptr;
  cp_ctx.defer_inst_count = !ar.measuring() && !dbg_check;  // read below with the leaf offsets
  // (a1, a2) partition (Alg. 5)
  int64_t n_leaves = 0, n_inst = 0;
  int depth = 0;
  s = partition_impl(XS, &p->part, leaf_off, bp.leaf_off_cap, leaf_ids, bp.leaf_ids_cap, &n_leaves, &n_inst, &depth,
                     ar, cp_ctx);
  if (s == PIPNN_OK && !ar.measuring() && sketch_work) s = sketch_work();
  if (s != PIPNN_OK) { cleanup(); return s; }
  ar.release(mark);
  if (ar.measuring()) n_inst = bp.leaf_ids_cap;  // size the later stages at their upper bounds
  else if (n_leaves == 0) n_inst = 0;
  if (!ar.measuring() && dbg_check) {
    // debug: host-side check of the partition output (sorted unique ids < n, sizes <= C_max, coverage)
    std::vector<int64_t> ho(n_leaves + 1);
    std::vector<uint32_t> hi(n_inst);
    cudaMemcpy(ho.data(), leaf_off, (n_leaves + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost);
    cudaMemcpy(hi.data(), leaf_ids, n_inst * sizeof(uint32_t), cudaMemcpyDeviceToHost);
    std::vector<uint8_t> cov(X->n, 0);
    int64_t bad = 0;
    for (int64_t b = 0; b < n_leaves; ++b) {
      const int64_t s0 = ho[b], s1 = ho[b + 1];
      if (s1 < s0 || s1 - s0 > p->part.c_max) ++bad;
      for (int64_t i = s0; i < s1; ++i) {
        if (hi[i] >= (uint64_t)X->n || (i > s0 && hi[i] <= hi[i - 1])) {
          ++bad;
          break;
        }
        cov[hi[i]] = 1;
      }
    }
    int64_t uncovered = 0;
    for (int64_t i = 0; i < X->n; ++i) uncovered += !cov[i];
    std::fprintf(stderr, "[pipnn] partition check: leaves %lld instances %lld bad %lld uncovered %lld\n",
                 (long long)n_leaves, (long long)n_inst, (long long)bad, (long long)uncovered);
  }
  if (!ar.measuring()) cudaEventRecord(ev[2], st);
  // (a3, a4) leaf distance tiles + fused pick, in waves of at most `budget` 128-row blocks so
  // the tiled leaf buffer stays bounded (one wave at 1M points).
  const int64_t budget = std::min<int64_t>(bp.leaf_ids_cap / 64 + 1024, (int64_t)1 << 16);
  int max_leaf_h = p->part.c_max;
  if (ar.measuring()) {
    s = leaf_pick_impl(XS, nullptr, nullptr, budget, budget * 128, k, nullptr, dist, ar, c, budget, cols,
                       p->pick.quant);
    if (s != PIPNN_OK) { cleanup(); return s; }
  } else if (n_leaves > 0) {
    std::vector<int64_t> off(n_leaves + 1);
    int64_t* hoff = reinterpret_cast<int64_t*>(pinned_scratch((n_leaves + 1) * sizeof(int64_t)));
    if (!hoff) { cleanup(); return fail(PIPNN_ECUDA, "pinned host scratch"); }
    PIPNN_CUDA(kcopy(hoff, leaf_off, (n_leaves + 1) * sizeof(int64_t), st));
    PIPNN_CUDA(cudaStreamSynchronize(st));
    std::copy(hoff, hoff + n_leaves + 1, off.begin());
    n_inst = off[n_leaves];  // (the partition left it unread: cp_ctx.defer_inst_count)
    max_leaf_h = 1;
    for (int64_t b = 0; b < n_leaves; ++b) {
      leaf_pairs += (off[b + 1] - off[b]) * (off[b + 1] - off[b]);
      max_leaf_h = std::max<int>(max_leaf_h, (int)(off[b + 1] - off[b]));
    }
    if (stats_h) c.tile_events = &tile_ev;
    int64_t b0 = 0;
    while (b0 < n_leaves) {
      int64_t items = 0, b1 = b0;
      while (b1 < n_leaves && items + ceil_div(off[b1 + 1] - off[b1], 128) <= budget) {
        items += ceil_div(off[b1 + 1] - off[b1], 128);
        ++b1;
      }
      if (b1 == b0) { cleanup(); return fail(PIPNN_EUNSUPPORTED, "leaf larger than the wave budget"); }
      s = leaf_pick_impl(XS, leaf_off + b0, leaf_ids, b1 - b0, off[b1] - off[b0], k, nullptr, dist, ar, c, budget, cols,
                         p->pick.quant);
      if (s != PIPNN_OK) { cleanup(); return s; }
      ar.release(mark);
      b0 = b1;
    }
    c.tile_events = nullptr;
  }
  ar.release(mark);
  if (!ar.measuring()) cudaEventRecord(ev[3], st);
  // (a5, a6) bidirected edges -> HashPrune reservoirs (Alg. 3)
  // Reservoirs start empty (count = 0). The build never reads a slot at or beyond count[u] (merge and final
  // prune), so the n*l_max arena is not initialised here (it is internal to pipnn_build).
  if (!ar.measuring()) PIPNN_CUDA(kmemset(count, 0, (size_t)X->n * sizeof(uint32_t), st));
  s = hashprune_from_leaves(p->hp.m, p->hp.l_max, X->n, sketch, sk_int, slots, count, leaf_off, n_leaves, leaf_ids,
                            n_inst, k, cols, dist, max_leaf_h, n_edges_dev, ar, c,
                            (int)std::min<int64_t>(1 << 20, bp.leaf_ids_cap / std::max<int64_t>(1, X->n)));
  if (s != PIPNN_OK) { cleanup(); return s; }
  ar.release(mark);
  if (!ar.measuring()) cudaEventRecord(ev[4], st);
  // (a7, a8) final prune + CSR. Float data (rows larger than L2 at 1M points): points in leaf
  // order, so the candidate rows of consecutive points overlap (L2 reuse); uint8 rows fit L2 at C2 and
  // id order measured slightly faster there.
  // uint8 rows: id order (measured: leaf order made C5's final prune slower, 126 -> 135 ms, and C2's too)
  static const bool u8_leaf_order = std::getenv("PIPNN_U8_LEAF_ORDER") != nullptr;  // experiment hook
  const bool by_leaf = is_float || u8_leaf_order;
  uint32_t* order = by_leaf ? ar.take<uint32_t>(X->n) : nullptr;
  uint32_t* order_n = by_leaf ? ar.take<uint32_t>(1) : nullptr;
  if (by_leaf) {
    s = leaf_order(leaf_ids, n_inst, X->n, order, order_n, ar, c);
    if (s != PIPNN_OK) { cleanup(); return s; }
  }
  s = final_prune_impl(X, p->hp.l_max, slots, count, &p->prune, row_ptr, col_idx, ar, c, order, order_n,
                       is_float ? &Xbv : nullptr);
  if (s != PIPNN_OK) { cleanup(); return s; }
  if (ar.measuring()) return PIPNN_OK;
  PIPNN_CUDA(cudaEventRecord(ev[5], st));
  // one pinned read-back: edge count, streamed-edge count, device error flag
  int64_t* hb = reinterpret_cast<int64_t*>(pinned_scratch(3 * sizeof(int64_t)));
  if (!hb) { cleanup(); return fail(PIPNN_ECUDA, "pinned host scratch"); }
  hb[2] = 0;
  PIPNN_CUDA(kcopy(&hb[0], row_ptr + X->n, sizeof(uint64_t), st));
  PIPNN_CUDA(kcopy(&hb[1], n_edges_dev, sizeof(int64_t), st));
  PIPNN_CUDA(kcopy(&hb[2], err, sizeof(int), st));
  PIPNN_CUDA(cudaStreamSynchronize(st));
  const uint64_t ne = (uint64_t)hb[0];
  const int64_t nstream = hb[1];
  {
    const int h = (int)(hb[2] & 0xFFFFFFFF);
    if (h == DERR_NONFINITE) { cleanup(); return fail(PIPNN_EINVAL, "non-finite float input"); }
    if (h != 0) { cleanup(); return fail(PIPNN_ECUDA, "device error flag " + std::to_string(h) + " (bounded wait timeout / capacity)"); }
  }
  if (n_edges_h) *n_edges_h = (int64_t)ne;
  if (stats_h) {
    float t[6];
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    cudaEventElapsedTime(&t[5], ev[0], ev[5]);
    stats_h->ms_prep = t[0];
    stats_h->ms_partition = t[1];
    stats_h->ms_leaf = t[2];
    stats_h->ms_hashprune = t[3];
    stats_h->ms_final = t[4];
    stats_h->ms_total = t[5];
    stats_h->n_leaves = n_leaves;
    stats_h->n_instances = n_inst;
    stats_h->n_edges = nstream;
    stats_h->depth = depth;
    stats_h->max_leaf = n_leaves > 0 ? max_leaf_h : 0;  // measured from the leaf offsets read after the partition
    stats_h->leaf_pairs = leaf_pairs;
    float tt = 0.0f;
    for (auto& pr : tile_ev) {
      float x = 0.0f;
      cudaEventElapsedTime(&x, pr.first, pr.second);
      tt += x;
    }
    stats_h->ms_leaf_tiles = tt;
  }
  cleanup();
  return PIPNN_OK;
}

}  // namespace pipnn

using namespace pipnn;

extern "C" {

const char* pipnn_last_error(void) { return g_last_error.c_str(); }
size_t pipnn_required_workspace(void) { return g_required_ws; }
uint64_t pipnn_launch_count(void) { return g_launches.load(); }
int32_t pipnn_abi_version(void) { return PIPNN_ABI_VERSION; }

pipnn_status pipnn_workspace_size(const pipnn_points* X, const pipnn_build_params* p, size_t* bytes_h) {
  PIPNN_TRY(validate_points(X));
  if (!p || !bytes_h) return fail(PIPNN_EINVAL, "NULL argument");
  PIPNN_TRY(validate_part(&p->part));
  PIPNN_TRY(validate_hp(&p->hp));
  PIPNN_TRY(validate_prune(&p->prune));
  if (p->pick.k < 1 || p->pick.k > 15) return fail(PIPNN_EINVAL, "k must be in [1, 15]");
  if (p->pick.quant < 0 || p->pick.quant > 1) return fail(PIPNN_EINVAL, "pick.quant must be 0 or 1");
  if (p->pick.quant && X->dtype == PIPNN_F32 && X->metric == PIPNN_MIPS)
    return fail(PIPNN_EUNSUPPORTED, "quantised leaf pick: float L2 only");
  Arena ar;  // measuring
  PIPNN_TRY(build_impl(X, p, ar, nullptr, nullptr, nullptr, nullptr, nullptr));
  *bytes_h = ar.peak + 4096;
  g_required_ws = *bytes_h;
  return PIPNN_OK;
}

// Device error flag of the last call that used `ws` (synchronises `stream`). Test/diagnostic hook.
pipnn_status pipnn_device_error(void* ws, void* stream) {
  if (!ws) return fail(PIPNN_EINVAL, "ws NULL");
  PIPNN_TRY(pending_cuda());
  return read_dev_error((int*)ws, (cudaStream_t)stream);
}

pipnn_status pipnn_partition(const pipnn_points* X, const pipnn_partition_params* p, void* ws, size_t ws_bytes,
                             int64_t* leaf_off, int64_t leaf_off_cap, uint32_t* leaf_ids, int64_t leaf_ids_cap,
                             int64_t* n_leaves_h, int64_t* n_instances_h, void* stream) {
  PIPNN_TRY(validate_points(X));
  PIPNN_TRY(validate_part(p));
  if (!leaf_off || !leaf_ids || !n_leaves_h || !n_instances_h) return fail(PIPNN_EINVAL, "NULL output");
  const int64_t need_ids = X->n * prod_fanout(p);
  if (leaf_ids_cap < need_ids)
    return fail(PIPNN_ECAPACITY, "leaf_ids_cap must be >= n*prod(fanout)*replicas = " + std::to_string(need_ids));
  if (leaf_off_cap < need_ids + 1)
    return fail(PIPNN_ECAPACITY, "leaf_off_cap must be >= " + std::to_string(need_ids + 1));
  cudaStream_t st = (cudaStream_t)stream;
  Arena m;
  m.take<int>(64);
  int dummy_depth = 0;
  int64_t a = 0, b = 0;
  PIPNN_TRY(partition_impl(X, p, nullptr, leaf_off_cap, nullptr, leaf_ids_cap, &a, &b, &dummy_depth, m, Ctx{st, nullptr}));
  PIPNN_TRY(check_ws(ws, ws_bytes, m.peak));
  PIPNN_TRY(pending_cuda());
  Arena ar(ws, ws_bytes);
  int* err = err_slot(ar);
  PIPNN_CUDA(kmemset(err, 0, 256, st));
  int depth = 0;
  PIPNN_TRY(partition_impl(X, p, leaf_off, leaf_off_cap, leaf_ids, leaf_ids_cap, n_leaves_h, n_instances_h, &depth, ar,
                           Ctx{st, err}));
  return read_dev_error(err, st);
}

pipnn_status pipnn_leaf_pick(const pipnn_points* X, const int64_t* leaf_off, const uint32_t* leaf_ids,
                             int64_t n_leaves, int64_t n_instances, const pipnn_pick_params* p, uint32_t* nbr,
                             float* dist, void* ws, size_t ws_bytes, void* stream) {
  PIPNN_TRY(validate_points(X));
  if (!p || p->k < 1 || p->k > 15) return fail(PIPNN_EINVAL, "k must be in [1, 15]");
  if (p->quant < 0 || p->quant > 1) return fail(PIPNN_EINVAL, "quant must be 0 or 1");
  if (n_leaves < 0 || n_instances < 0) return fail(PIPNN_EINVAL, "negative sizes");
  if (n_leaves > 0 && (!leaf_off || !leaf_ids || !nbr)) return fail(PIPNN_EINVAL, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  Arena m;
  m.take<int>(64);
  PIPNN_TRY(leaf_pick_impl(X, leaf_off, leaf_ids, n_leaves, n_instances, p->k, nbr, dist, m, Ctx{st, nullptr}, 0,
                           nullptr, p->quant));
  PIPNN_TRY(check_ws(ws, ws_bytes, m.peak));
  PIPNN_TRY(pending_cuda());
  Arena ar(ws, ws_bytes);
  int* err = err_slot(ar);
  PIPNN_CUDA(kmemset(err, 0, 256, st));
  return leaf_pick_impl(X, leaf_off, leaf_ids, n_leaves, n_instances, p->k, nbr, dist, ar, Ctx{st, err}, 0, nullptr,
                        p->quant);
}

pipnn_status pipnn_sketch(const pipnn_points* X, const pipnn_hashprune_params* p, void* sketch, void* ws,
                          size_t ws_bytes, void* stream) {
  PIPNN_TRY(validate_points(X));
  PIPNN_TRY(validate_hp(p));
  if (!sketch) return fail(PIPNN_EINVAL, "sketch NULL");
  cudaStream_t st = (cudaStream_t)stream;
  Arena m;
  m.take<int>(64);
  PIPNN_TRY(sketch_impl(X, p->m, p->seed, sketch, m, Ctx{st, nullptr}));
  PIPNN_TRY(check_ws(ws, ws_bytes, m.peak));
  PIPNN_TRY(pending_cuda());
  Arena ar(ws, ws_bytes);
  int* err = err_slot(ar);
  PIPNN_CUDA(kmemset(err, 0, 256, st));
  return sketch_impl(X, p->m, p->seed, sketch, ar, Ctx{st, err});
}

pipnn_status hashprune_insert(const pipnn_hashprune_params* p, int64_t n, const void* sketch, int32_t sk_dtype,
                              uint64_t* slots, uint32_t* count, const uint32_t* owner, const uint32_t* cand,
                              const float* dist, int64_t n_edges, void* ws, size_t ws_bytes, void* stream) {
  PIPNN_TRY(validate_hp(p));
  if (n < 1 || n > 0xFFFFFFFEll) return fail(PIPNN_EINVAL, "n out of range");
  if (n_edges < 0) return fail(PIPNN_EINVAL, "n_edges < 0");
  if (!sketch || !slots || !count) return fail(PIPNN_EINVAL, "NULL argument");
  if (n_edges > 0 && (!owner || !cand || !dist)) return fail(PIPNN_EINVAL, "NULL edge arrays");
  if (sk_dtype != PIPNN_U8 && sk_dtype != PIPNN_F32) return fail(PIPNN_EINVAL, "sk_dtype");
  cudaStream_t st = (cudaStream_t)stream;
  Arena m;
  m.take<int>(64);
  PIPNN_TRY(hashprune_impl(p->m, p->l_max, n, sketch, sk_dtype == PIPNN_U8, slots, count, owner, cand, dist, n_edges, m,
                           Ctx{st, nullptr}));
  PIPNN_TRY(check_ws(ws, ws_bytes, m.peak));
  PIPNN_TRY(pending_cuda());
  Arena ar(ws, ws_bytes);
  int* err = err_slot(ar);
  PIPNN_CUDA(kmemset(err, 0, 256, st));
  return hashprune_impl(p->m, p->l_max, n, sketch, sk_dtype == PIPNN_U8, slots, count, owner, cand, dist, n_edges, ar,
                        Ctx{st, err});
}

pipnn_status pipnn_final_prune(const pipnn_points* X, const pipnn_hashprune_params* hp, const uint64_t* slots,
                               const uint32_t* count, const pipnn_prune_params* p, uint64_t* row_ptr,
                               uint32_t* col_idx, void* ws, size_t ws_bytes, void* stream) {
  PIPNN_TRY(validate_points(X));
  PIPNN_TRY(validate_hp(hp));
  PIPNN_TRY(validate_prune(p));
  if (!slots || !count || !row_ptr || !col_idx) return fail(PIPNN_EINVAL, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  Arena m;
  m.take<int>(64);
  PIPNN_TRY(final_prune_impl(X, hp->l_max, slots, count, p, row_ptr, col_idx, m, Ctx{st, nullptr}));
  PIPNN_TRY(check_ws(ws, ws_bytes, m.peak));
  PIPNN_TRY(pending_cuda());
  Arena ar(ws, ws_bytes);
  int* err = err_slot(ar);
  PIPNN_CUDA(kmemset(err, 0, 256, st));
  return final_prune_impl(X, hp->l_max, slots, count, p, row_ptr, col_idx, ar, Ctx{st, err});
}

pipnn_status pipnn_build(const pipnn_points* X, const pipnn_build_params* p, void* ws, size_t ws_bytes,
                         uint64_t* row_ptr, uint32_t* col_idx, int64_t* n_edges_h, pipnn_stats* stats_h, void* stream) {
  size_t need = 0;
  PIPNN_TRY(pipnn_workspace_size(X, p, &need));
  if (!row_ptr || !col_idx) return fail(PIPNN_EINVAL, "NULL output");
  PIPNN_TRY(check_ws(ws, ws_bytes, need - 4096));
  PIPNN_TRY(pending_cuda());
  Arena ar(ws, ws_bytes);
  return build_impl(X, p, ar, (cudaStream_t)stream, row_ptr, col_idx, n_edges_h, stats_h);
}

pipnn_status pipnn_debug_build_buffers(const pipnn_points* X, const pipnn_build_params* p, void* ws, size_t ws_bytes,
                                       pipnn_build_buffers* out_h) {
  size_t need = 0;
  PIPNN_TRY(pipnn_workspace_size(X, p, &need));
  if (!out_h) return fail(PIPNN_EINVAL, "NULL output");
  PIPNN_TRY(check_ws(ws, ws_bytes, need - 4096));
  Arena ar(ws, ws_bytes);
  const BuildBufs b = take_build_bufs(X, p, ar);
  out_h->leaf_off = b.leaf_off;
  out_h->leaf_ids = b.leaf_ids;
  out_h->cols = b.cols;
  out_h->dist = b.dist;
  out_h->sketch = b.sketch;
  out_h->slots = b.slots;
  out_h->count = b.count;
  return PIPNN_OK;
}

pipnn_status pipnn_search(const pipnn_points* X, const uint64_t* row_ptr, const uint32_t* col_idx,
                          const void* queries, int64_t ld_q, int64_t nq, uint32_t entry, const pipnn_search_params* p,
                          uint32_t* out_ids, float* out_dist, int64_t* n_cmps_dev, void* ws, size_t ws_bytes,
                          void* stream) {
  PIPNN_TRY(validate_points(X));
  if (!p) return fail(PIPNN_EINVAL, "search params NULL");
  if (p->k < 1 || p->L < p->k || p->L > 256) return fail(PIPNN_EINVAL, "need 1 <= k <= L <= 256");
  if (p->exclude_self && (p->L < p->k + 1 || nq > X->n)) return fail(PIPNN_EINVAL, "exclude_self needs L > k, nq <= n");
  if (nq < 0 || (nq > 0 && (!queries || !out_ids || !row_ptr || !col_idx))) return fail(PIPNN_EINVAL, "NULL argument");
  if (ld_q < X->d) return fail(PIPNN_EINVAL, "ld_q < d");
  if ((int64_t)entry >= X->n) return fail(PIPNN_EINVAL, "entry out of range");
  if (search_smem_per_warp(X) * 4 > 227 * 1024) return fail(PIPNN_EUNSUPPORTED, "d too large for the search kernel");
  cudaStream_t st = (cudaStream_t)stream;
  PIPNN_TRY(check_ws(ws, ws_bytes, 256));
  PIPNN_TRY(pending_cuda());
  Arena ar(ws, ws_bytes);
  int* err = err_slot(ar);
  PIPNN_CUDA(kmemset(err, 0, 256, st));
  return search_impl(X, row_ptr, col_idx, queries, ld_q, nq, entry, p->L, p->k, p->exclude_self ? 1 : 0, out_ids,
                     out_dist, n_cmps_dev, Ctx{st, err});
}

}  // extern "C"
