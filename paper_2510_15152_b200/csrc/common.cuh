// common.cuh -- error plumbing, workspace carving and small device helpers for libtlru.
// Product code: independent of oracle/ (shares no code, headers or constants with it).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "tlru.h"

namespace tlru {

// ----------------------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
void clear_error();

#define TLRU_FAIL(code, ...)          \
  do {                                \
    ::tlru::set_error(__VA_ARGS__);   \
    return (code);                    \
  } while (0)

#define TLRU_CUDA(call)                                                                       \
  do {                                                                                        \
    cudaError_t err__ = (call);                                                               \
    if (err__ != cudaSuccess)                                                                 \
      TLRU_FAIL(TLRU_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(err__)); \
  } while (0)

void count_launch(unsigned n = 1);

#define TLRU_CHECK_LAUNCH()             \
  do {                                  \
    ::tlru::count_launch();             \
    TLRU_CUDA(cudaGetLastError());      \
  } while (0)

#define TLRU_TRY(expr)                 \
  do {                                 \
    tlru_status st__ = (expr);         \
    if (st__ != TLRU_OK) return st__;  \
  } while (0)

// ----------------------------------------------------------------------------- workspace
// Bump allocator over the caller's workspace.  With base == nullptr it only
// measures (the *_workspace_size calls run the same carving code).
struct Carver {
  char* base;
  size_t used = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t count) {
    used = (used + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + used) : nullptr;
    used += count * sizeof(T);
    return p;
  }
};

inline tlru_status check_ws(const Carver& c, void* ws, size_t ws_bytes) {
  if (c.used > 0 && ws == nullptr) TLRU_FAIL(TLRU_ERANGE, "workspace is NULL but %zu bytes are required", c.used);
  if (c.used > ws_bytes) TLRU_FAIL(TLRU_ERANGE, "workspace too small: %zu < %zu bytes", ws_bytes, c.used);
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) TLRU_FAIL(TLRU_EINVAL, "workspace must be 256-byte aligned");
  return TLRU_OK;
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 64u) {
  uint64_t g = (n + block - 1) / block;
  if (g == 0) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// ----------------------------------------------------------------------------- sim view packing
__host__ __device__ __forceinline__ uint64_t pack_sim(uint32_t prev, uint32_t J, uint32_t L_after) {
  return uint64_t(prev) | (uint64_t(J & 0xFFFFu) << 32) | (uint64_t(L_after & 0xFFFFu) << 48);
}
__host__ __device__ __forceinline__ uint32_t sim_prev(uint64_t s) { return uint32_t(s); }
__host__ __device__ __forceinline__ uint32_t sim_J(uint64_t s) { return uint32_t(s >> 32) & 0xFFFFu; }
__host__ __device__ __forceinline__ uint32_t sim_La(uint64_t s) { return uint32_t(s >> 48); }

// ----------------------------------------------------------------------------- warp-aggregated atomics
// One atomic per warp instead of one per lane on the hot single-address counters.
__device__ __forceinline__ void warp_atomic_max_u64(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = w > v ? w : v;
  }
  if ((threadIdx.x & 31) == 0 && v) atomicMax(dst, v);
}

__device__ __forceinline__ void warp_atomic_max_u32(uint32_t* dst, uint32_t v) {
  v = __reduce_max_sync(0xFFFFFFFFu, v);
  if ((threadIdx.x & 31) == 0 && v) atomicMax(dst, v);
}

__device__ __forceinline__ void warp_atomic_add_u64(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

__device__ __forceinline__ void warp_atomic_add_u32(uint32_t* dst, uint32_t v) {
  v = __reduce_add_sync(0xFFFFFFFFu, v);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// Warp-aggregated queue push: returns the slot for lanes with `want`, leader does one atomicAdd.
__device__ __forceinline__ uint32_t warp_push(uint32_t* counter, bool want) {
  const unsigned m = __ballot_sync(0xFFFFFFFFu, want);
  uint32_t base = 0;
  const int lane = threadIdx.x & 31;
  if (lane == 0 && m) base = atomicAdd(counter, static_cast<uint32_t>(__popc(m)));
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  return base + __popc(m & ((1u << lane) - 1u));
}

}  // namespace tlru
