// toc_common.cuh -- device helpers shared by the TOC kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "toc_b200.h"

#define TOC_HD __host__ __device__ __forceinline__
#define TOC_D __device__ __forceinline__

namespace toc {

constexpr int kWarp = 32;

// Little-endian read of one `w`-byte packed integer (reference physical.py:54-85 layout:
// fixed width 1..4 bytes, least significant byte first).  Blocks are immutable during a
// kernel, so loads go through the read-only path.
TOC_D uint32_t ld_packed(const uint8_t* __restrict__ p, uint32_t i, uint32_t w) {
  const uint8_t* q = p + (size_t)i * w;
  switch (w) {
    case 1:
      return __ldg(q);
    case 2:
      return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8);
    case 3:
      return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8) | ((uint32_t)__ldg(q + 2) << 16);
    default:
      return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8) | ((uint32_t)__ldg(q + 2) << 16) |
             ((uint32_t)__ldg(q + 3) << 24);
  }
}

TOC_D uint32_t ld_u32_unaligned(const uint8_t* __restrict__ q) {
  return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8) | ((uint32_t)__ldg(q + 2) << 16) |
         ((uint32_t)__ldg(q + 3) << 24);
}

TOC_D double ld_f64_unaligned(const uint8_t* __restrict__ q) {
  uint64_t lo = ld_u32_unaligned(q), hi = ld_u32_unaligned(q + 4);
  return __longlong_as_double((long long)(lo | (hi << 32)));
}

template <typename T>
TOC_D T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exclusive prefix sum over a warp (inclusive - self).
TOC_D uint32_t warp_excl_scan(uint32_t v, uint32_t lane) {
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x - v;
}

TOC_HD uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

}  // namespace toc
