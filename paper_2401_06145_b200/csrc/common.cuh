// Shared device helpers: coordinate keys, error plumbing, PTX wrappers (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>

namespace sconvb {

// ---- coordinate keys (reference geometry.hpp:18-73) ----
constexpr int32_t kCoordBias = 1 << 20;
constexpr int32_t kCoordMax = kCoordBias - 1;
constexpr int32_t kCoordMin = -kCoordMax;
constexpr uint64_t kFieldMask = (uint64_t{1} << 21) - 1;

__host__ __device__ __forceinline__ bool in_range(int64_t v) { return v >= kCoordMin && v <= kCoordMax; }

__host__ __device__ __forceinline__ uint64_t pack_key_unchecked(int32_t x, int32_t y, int32_t z) {
  return (static_cast<uint64_t>(x + kCoordBias) << 42) | (static_cast<uint64_t>(y + kCoordBias) << 21) |
         static_cast<uint64_t>(z + kCoordBias);
}

__host__ __device__ __forceinline__ void unpack_key(uint64_t k, int32_t& x, int32_t& y, int32_t& z) {
  x = static_cast<int32_t>((k >> 42) & kFieldMask) - kCoordBias;
  y = static_cast<int32_t>((k >> 21) & kFieldMask) - kCoordBias;
  z = static_cast<int32_t>(k & kFieldMask) - kCoordBias;
}

// Monotone key of an unbounded triple (see oracle saturating_pack): equals the packed
// key in range, never equals a valid key otherwise, non-decreasing lexicographically.
__host__ __device__ __forceinline__ uint64_t saturating_pack(int64_t x, int64_t y, int64_t z) {
  if (x > kCoordMax) return uint64_t{1} << 63;
  if (x < kCoordMin) return 0;
  const uint64_t X = static_cast<uint64_t>(x + kCoordBias);
  if (y > kCoordMax) return (X + 1) << 42;
  if (y < kCoordMin) return X << 42;
  const uint64_t Y = static_cast<uint64_t>(y + kCoordBias);
  if (z > kCoordMax) return (X << 42) + ((Y + 1) << 21);
  if (z < kCoordMin) return (X << 42) + (Y << 21);
  return (X << 42) | (Y << 21) | static_cast<uint64_t>(z + kCoordBias);
}

// Segment key of q + delta from the packed q key.
__device__ __forceinline__ uint64_t segment_key(uint64_t qkey, int3 d) {
  int32_t x, y, z;
  unpack_key(qkey, x, y, z);
  return saturating_pack(int64_t{x} + d.x, int64_t{y} + d.y, int64_t{z} + d.z);
}

__host__ __device__ __forceinline__ int64_t floor_div(int64_t a, int64_t b) {
  const int64_t q = a / b, r = a % b;
  return (r != 0 && ((r < 0) != (b < 0))) ? q - 1 : q;
}

// ---- small PTX wrappers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}
__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <class T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) {
  return (a + b - 1) / b;
}

}  // namespace sconvb
