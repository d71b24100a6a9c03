// toc_images.cuh -- pieces shared by the cached-image MGD epochs (toc_images.cu,
// toc_images_large.cu): node tables over every id of a (sub)tree, the flat chain walk, fixed-point
// scales, and the TMA / mbarrier / cluster-barrier / DSMEM wrappers.
#pragma once
#include "toc_glm.cuh"

namespace toc {

constexpr uint32_t kMaxCluster = 16;  // 16: non-portable (cudaFuncAttributeNonPortableClusterSizeAllowed)

// Node table of a step image.
template <bool kWide>
struct Nodes;

template <>
struct Nodes<false> {
  const uint32_t* p;
  const uint16_t* codes;
  TOC_D void get(uint32_t x, uint32_t& par, uint32_t& key) const {
    const uint32_t w = p[x];
    par = w & 0xffffu;
    key = w >> 16;
  }
  TOC_D uint32_t code(uint32_t j) const { return codes[j]; }
  TOC_HD static uint32_t pack(uint32_t par, uint32_t key) { return par | (key << 16); }
};

template <>
struct Nodes<true> {
  const uint2* p;
  const uint32_t* codes;
  TOC_D void get(uint32_t x, uint32_t& par, uint32_t& key) const {
    const uint2 w = p[x];
    par = w.x;
    key = w.y;
  }
  TOC_D uint32_t code(uint32_t j) const { return codes[j]; }
};

// All pairs of codes [j0, j1): one iteration per pair, whatever the chain lengths, so the lanes
// of a warp stay converged except at the loop exit.
template <bool kWide, typename V>
TOC_D void walk_flat(const Nodes<kWide>& N, uint32_t j0, uint32_t j1, V&& visit) {
  if (j0 >= j1) return;
  uint32_t j = j0, x = N.code(j0);
  for (;;) {
    uint32_t par, key;
    N.get(x, par, key);
    visit(key);
    if (par) {
      x = par;
      continue;
    }
    if (++j >= j1) break;
    x = N.code(j);
  }
}

// Fixed-point add (see fix_add, toc_batch.cuh) with the two words in separate arrays, so random
// adds spread over all 32 banks, and no branch.
TOC_D void fix_add_pair(uint32_t* lo, uint32_t* hi, uint32_t i, uint32_t xl, uint32_t xh) {
  const uint32_t old = atomicAdd(lo + i, xl);
  atomicAdd(hi + i, xh + (old + xl < old ? 1u : 0u));
}

// 2^F and 2^-F of fix_scale(bound) from the exponent bits (no division on the step's path).
TOC_D void fix_scales(double bound, double& scale, double& inv) {
  const long long bits = __double_as_longlong(bound);
  const int be = (int)((bits >> 52) & 0x7ff);
  if (!(bound > 0.0) || be == 0 || be == 0x7ff) {  // zero, subnormal, inf / nan: the general path
    scale = fix_scale(bound);
    inv = 1.0 / scale;
    return;
  }
  const int e = be - 1022;  // bound = f * 2^e, f in [0.5, 1)  (frexp)
  scale = __longlong_as_double((long long)(61 - e + 1023) << 52);
  inv = __longlong_as_double((long long)(e - 61 + 1023) << 52);
}

// mbarrier wait that cannot hang the GPU: a copy that never lands traps after 2 s.
TOC_D void mbar_wait_bounded(uint64_t* mbar, uint32_t phase) {
  unsigned long long t0 = 0;
  for (uint32_t it = 0;; ++it) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(mbar)), "r"(phase)
        : "memory");
    if (done) return;
    if ((it & 255u) == 255u) {
      if (!t0) t0 = globaltimer_ns();
      else if (globaltimer_ns() - t0 > 2000000000ull) __trap();
    }
  }
}

TOC_D void mbar_expect(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}

// Bulk copy global -> shared without arming the barrier (the receiving CTA arms it).
TOC_D void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}

// The same bytes to the same offsets in every CTA of `mask`, completing on each one's mbarrier.
TOC_D void bulk_multicast(void* dst, const void* src, uint32_t bytes, uint64_t* mbar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mbar)), "h"(mask)
      : "memory");
}

// Cluster-wide barrier with release/acquire at cluster scope (setup and exit).
TOC_D void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// The per-step barrier: what crosses it is only shared-memory data (the column partials) read
// remotely after it.  A CTA-scope fence commits this thread's shared stores to the CTA's own
// shared memory -- where DSMEM reads are served -- before the relaxed arrive.  ptxas lowers a
// cluster-scope release to a GPU-scope MEMBAR, which this avoids.
TOC_D void cluster_barrier_smem() {
  asm volatile("membar.cta;\n\tbarrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" :::
                   "memory");
}

TOC_D uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Load a double from CTA `rank`'s shared memory at the offset of `p` in this CTA.
TOC_D double ld_dsmem(const double* p, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(p)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
  return v;
}

}  // namespace toc
