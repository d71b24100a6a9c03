// toc_abi.cu -- self-description entry points of the C ABI (include/toc_b200.h).
#include "toc_common.cuh"

extern "C" const char* toc_version(void) { return "toc_b200 0.1.0 sm_100a"; }

extern "C" int toc_device_info(int32_t* sm_count, int32_t* smem_optin, int64_t* l2_bytes) {
  int dev = 0, sm = 0, smem = 0, l2 = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TOC_E_CUDA;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  if (sm_count) *sm_count = sm;
  if (smem_optin) *smem_optin = smem;
  if (l2_bytes) *l2_bytes = l2;
  return TOC_OK;
}

static_assert(sizeof(TocBlockMeta) == 68, "TocBlockMeta layout is part of the ABI");
static_assert(sizeof(TocPlan) == 40, "TocPlan layout is part of the ABI");

extern "C" int toc_sizeof_meta(void) { return (int)sizeof(TocBlockMeta); }
extern "C" int toc_sizeof_plan(void) { return (int)sizeof(TocPlan); }

static_assert(sizeof(TocBatchInfo) == 48, "TocBatchInfo layout is part of the ABI");
extern "C" int toc_sizeof_batch_info(void) { return (int)sizeof(TocBatchInfo); }
extern "C" int toc_sizeof_sweep_chunk(void) { return (int)sizeof(TocSweepChunk); }
