// toc_glm.cuh -- GLM pieces shared by the MGD kernels (toc_mgd.cu, toc_images.cu).
#pragma once
#include "toc_batch.cuh"

namespace toc {

constexpr int kTracePoints = 8;

// Per-example scalar of glm_gradient (training.py:272-280).
TOC_D double loss_scalar(int loss, double y, double z) {
  if (loss == TOC_LOSS_SQUARED) return z - y;
  if (loss == TOC_LOSS_LOGISTIC) return -y / (1.0 + exp(y * z));
  return (y * z < 1.0) ? -y : 0.0;  // hinge subgradient: flat side contributes zero
}

TOC_D uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

TOC_D unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

TOC_D void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace toc
