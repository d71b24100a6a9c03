// toc_common.cuh -- device helpers shared by the TOC kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "toc_b200.h"

#define TOC_HD __host__ __device__ __forceinline__
#define TOC_D __device__ __forceinline__

// Bounds checks of the checked build (make checked -> libtoc_b200_checked.so, -DTOC_CHECKED): the
// compute-sanitizer tools are closed on this GPU pool, so index and size invariants of the hot
// kernels are asserted in the kernels themselves (file:line printed, then a trap).  Compiled out
// of the product library.
#ifdef TOC_CHECKED
#include <cstdio>
#define TOC_CHECK(c)                                                                              \
  do {                                                                                            \
    if (!(c)) {                                                                                   \
      printf("TOC_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x, #c);                                                               \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define TOC_CHECK(c) ((void)0)
#endif

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

namespace toc {

// ---- warp-cooperative unpack of packed ints ------------------------------------------------
// A TOC1 section packs fixed-width (W = 1..4 bytes) little-endian ints at an arbitrary byte
// offset (physical.py:54-68).  A warp unpacks a range [lo, hi) in tiles of kTile values: the
// covering aligned 32-bit words are loaded once, coalesced, into a per-warp shared staging
// buffer, and each lane extracts its values with a funnel shift.  f(i, value) is called for
// every i, lane-parallel.  Reading to the next 4-byte boundary past the section is safe because
// every block in an arena starts on, and is padded to, a 16-byte boundary.
constexpr uint32_t kTile = 64;
constexpr uint32_t kStageWords = kTile + 4;  // (3 + 64*4 + 3) / 4 = 65.5 -> 66 words + guard

template <int W, typename F>
TOC_D void warp_unpack(const uint8_t* __restrict__ sec, uint32_t lo, uint32_t hi, uint32_t* stage,
                       uint32_t lane, F&& f) {
  for (uint32_t t = lo; t < hi; t += kTile) {
    const uint32_t n = min(kTile, hi - t);
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(sec) + (uintptr_t)t * W;
    const uintptr_t a0 = b0 & ~(uintptr_t)3;
    const uint32_t nw = (uint32_t)((((b0 + (uintptr_t)n * W) + 3) & ~(uintptr_t)3) - a0) >> 2;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a0);
    for (uint32_t k = lane; k < nw; k += 32) stage[k] = __ldg(src + k);
    if (lane == 0) stage[nw] = 0u;
    __syncwarp();
    const uint32_t d0 = (uint32_t)(b0 - a0);
#pragma unroll 2
    for (uint32_t j = lane; j < n; j += 32) {
      const uint32_t off = d0 + j * W, q = off >> 2, s = (off & 3u) * 8u;
      uint32_t v = __funnelshift_r(stage[q], stage[q + 1], s);
      if constexpr (W < 4) v &= (1u << (8 * W)) - 1u;
      f(t + j, v);
    }
    __syncwarp();
  }
}

// Dispatch a runtime width to the templated unpack.
template <typename F>
TOC_D void warp_unpack_w(uint32_t w, const uint8_t* sec, uint32_t lo, uint32_t hi, uint32_t* stage,
                         uint32_t lane, F&& f) {
  switch (w) {
    case 1: warp_unpack<1>(sec, lo, hi, stage, lane, f); break;
    case 2: warp_unpack<2>(sec, lo, hi, stage, lane, f); break;
    case 3: warp_unpack<3>(sec, lo, hi, stage, lane, f); break;
    default: warp_unpack<4>(sec, lo, hi, stage, lane, f); break;
  }
}

}  // namespace toc

namespace toc {

// Sequential reader of a packed-int section for one thread: walks values i0, i0+1, ... with one
// aligned 32-bit load per 32/(8W) values and a funnel shift per value.  May read up to 4 bytes
// past the last value; arenas carry 16 bytes of tail padding for that.
template <int W>
struct SeqReader {
  const uint32_t* wp;
  uint32_t cur, nxt, sh;
  TOC_D void init(const uint8_t* __restrict__ sec, uint32_t i0) {
    const uintptr_t b = reinterpret_cast<uintptr_t>(sec) + (uintptr_t)i0 * W;
    wp = reinterpret_cast<const uint32_t*>(b & ~(uintptr_t)3);
    sh = (uint32_t)(b & 3u) * 8u;
    cur = __ldg(wp);
    nxt = __ldg(wp + 1);
  }
  TOC_D uint32_t next() {
    uint32_t v = __funnelshift_r(cur, nxt, sh);
    if constexpr (W < 4) v &= (1u << (8 * W)) - 1u;
    sh += 8u * W;
    if (sh >= 32u) {
      sh -= 32u;
      cur = nxt;
      ++wp;
      nxt = __ldg(wp + 1);
    }
    return v;
  }
};

// Call f.template operator()<W>() with the runtime width as a template argument.
template <typename F>
TOC_D void with_width(uint32_t w, F&& f) {
  switch (w) {
    case 1: f.template operator()<1>(); break;
    case 2: f.template operator()<2>(); break;
    case 3: f.template operator()<3>(); break;
    default: f.template operator()<4>(); break;
  }
}

}  // namespace toc

namespace toc {

// Block-wide sum / max of a double over <= 32 warps; s_red holds 33 doubles.
TOC_D double block_sum(double v, double* s_red) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nwarps ? s_red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) s_red[32] = t;
  }
  __syncthreads();
  return s_red[32];
}

TOC_D double block_max_d(double v, double* s_red) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nwarps ? s_red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) s_red[32] = t;
  }
  __syncthreads();
  return s_red[32];
}

}  // namespace toc
