// common.cuh — internal helpers of libpipnn (CUDA path). Not part of the ABI.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <cuda_runtime.h>

#include "../../include/pipnn.h"

namespace pipnn {

// ------------------------------------------------------------------ status / last error
void set_error(const std::string& msg);
void count_launch();  // kernels launched by this library (diagnostic counter, pipnn_launch_count)
pipnn_status fail(pipnn_status s, const std::string& msg);
bool sync_debug();  // PIPNN_SYNC_DEBUG=1

struct CudaError {
  cudaError_t e;
  const char* what;
};

#define PIPNN_CUDA(expr)                                                                             \
  do {                                                                                               \
    cudaError_t _e = (expr);                                                                         \
    if (_e != cudaSuccess)                                                                           \
      return ::pipnn::fail(PIPNN_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));         \
  } while (0)

// After a kernel launch: launch error, and in debug mode a synchronisation.
#define PIPNN_LAUNCHED(name, stream)                                                                 \
  do {                                                                                               \
    ::pipnn::count_launch();                                                                         \
    cudaError_t _e = cudaGetLastError();                                                             \
    if (_e == cudaSuccess && ::pipnn::sync_debug()) _e = cudaStreamSynchronize(stream);              \
    if (_e != cudaSuccess)                                                                           \
      return ::pipnn::fail(PIPNN_ECUDA, std::string(name) + ": " + cudaGetErrorString(_e));          \
  } while (0)

#define PIPNN_TRY(expr)                    \
  do {                                     \
    pipnn_status _s = (expr);              \
    if (_s != PIPNN_OK) return _s;         \
  } while (0)

// ------------------------------------------------------------------ workspace bump allocator
// The caller passes one device block; sub-buffers are carved with 256-B alignment. `measure` mode
// (base == nullptr) only accumulates the size, so the same code path computes pipnn_workspace_size.
struct Arena {
  uint8_t* base = nullptr;
  size_t cap = 0, used = 0, peak = 0;
  Arena() = default;
  Arena(void* b, size_t c) : base((uint8_t*)b), cap(c) {}
  template <class T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
    size_t off = used;
    used += bytes;
    if (used > peak) peak = used;
    if (!base || used > cap) return nullptr;
    return (T*)(base + off);
  }
  bool measuring() const { return base == nullptr; }
  bool overflow() const { return base && used > cap; }
  size_t mark() const { return used; }
  void release(size_t m) { used = m; }
};

// Device-side error codes written to the flag word at the start of the workspace.
enum DevErr : int {
  DERR_NONE = 0,
  DERR_WAIT_TIMEOUT = 1,  // bounded mbarrier wait expired (pipeline bug)
  DERR_NONFINITE = 2,     // non-finite float input
  DERR_CAPACITY = 3,      // device-side capacity overflow
};

// ------------------------------------------------------------------ randomness (docs/DETERMINISM.md)
// Independent re-implementation of the counter-based generator fixed in docs/DETERMINISM.md.
__host__ __device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) { return sm64(a ^ sm64(b)); }
constexpr uint64_t kDomHyper = 0x48595045524C4E45ull;
constexpr uint64_t kDomPart = 0x5041525449544E31ull;
constexpr uint64_t kDomMerge = 0x4D45524745535444ull;

// bf16 helpers (RNE), order key of a stored distance (R5).
__host__ __device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
__host__ __device__ __forceinline__ uint16_t dist_order_key(float D) {
  D = D + 0.0f;  // -0 -> +0
  uint16_t b = f32_to_bf16_rne(D);
  return (uint16_t)(b ^ ((b & 0x8000u) ? 0xFFFFu : 0x8000u));
}

// Internal element type: float data already rounded to bf16 (RNE), rows of ld elements, zero padded to ld
// (ld = round_up(d, 8)). Never an ABI value: pipnn_build makes this copy of float X once (prep) and every
// later gather reads it (half the bytes of the fp32 rows).
constexpr int32_t kDtypeBf16 = 2;

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace pipnn
