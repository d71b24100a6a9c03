// toc_sweep.cu -- the host-side pipeline of the batched public sweep (kernels.BatchSweep), native.
//
// Reference: cli.py:299-383 (bench-kernels: a Python loop of matvec / vecmat over batches).  One
// call of the public API uploads host TOC1 blocks and operands, validates the blocks on the device
// (physical.py:138-186 semantics), runs A.v and v^T.A on every batch and downloads the results.  It
// is split into chunks so copies, validation / compute and result downloads of different chunks
// overlap: copies on one stream (host -> device copies are served in submission order across
// streams, so their order is the schedule), validation / compute on a second, result downloads on
// a third; the schedule is enqueued natively:
//   toc_sweep_upload(0, 1)   the first chunk's block bytes
//   (the caller fills the pinned operand buffers meanwhile)
//   toc_sweep_operands       v and u
//   toc_sweep_upload(1, n)   the other chunks' bytes
//   toc_sweep_compute        per chunk: wait for its bytes, validate / index, wait for its operands,
//                            fused A.v + v^T.A; results and the chunk's index -> host.
#include <vector>

#include "toc_common.cuh"

extern "C" int toc_index_blocks(const uint8_t* d_arena, const int64_t* d_block_off, const int64_t* d_block_len,
                                int64_t n_blocks, TocBlockMeta* d_meta, void* stream);
extern "C" int toc_linalg(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                          const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int32_t kind,
                          const double* d_v, double* d_R, const double* d_u, double* d_O, void* d_scratch,
                          void* stream);

namespace {

cudaEvent_t ev(void* e) { return static_cast<cudaEvent_t>(e); }

// diagnostic timeline (toc_sweep_set_timing): timed events per chunk
bool g_timing = false;
std::vector<cudaEvent_t> g_t;  // [0] first upload start, then per chunk: upload end, index start / end, compute end, d2h end
cudaEvent_t tev(size_t i) {
  while (g_t.size() <= i) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    g_t.push_back(e);
  }
  return g_t[i];
}

}  // namespace

extern "C" int toc_sweep_events(TocSweepChunk* chunks, int64_t n_chunks) {
  if (!chunks || n_chunks < 0) return TOC_E_ARG;
  for (int64_t k = 0; k < n_chunks; ++k)
    for (void** slot : {&chunks[k].ev_upload, &chunks[k].ev_operands, &chunks[k].ev_done}) {
      if (*slot) continue;
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return TOC_E_CUDA;
      *slot = e;
    }
  return TOC_OK;
}

extern "C" int toc_sweep_events_free(TocSweepChunk* chunks, int64_t n_chunks) {
  if (!chunks || n_chunks < 0) return TOC_E_ARG;
  for (int64_t k = 0; k < n_chunks; ++k)
    for (void** slot : {&chunks[k].ev_upload, &chunks[k].ev_operands, &chunks[k].ev_done}) {
      if (*slot) cudaEventDestroy(ev(*slot));
      *slot = nullptr;
    }
  return TOC_OK;
}

extern "C" int toc_sweep_set_timing(int32_t on) {
  g_timing = on != 0;
  return TOC_OK;
}

// After a synchronized timed run: out[5 * k + 0..4] = chunk k's upload end, validation start,
// validation end, compute end, download end, in ms from the first upload's start.
extern "C" int toc_sweep_timeline(int64_t n_chunks, float* out) {
  if (!out || n_chunks < 0 || g_t.size() < (size_t)(1 + 5 * n_chunks)) return TOC_E_ARG;
  for (int64_t i = 0; i < 5 * n_chunks; ++i)
    if (cudaEventElapsedTime(out + i, g_t[0], g_t[1 + i]) != cudaSuccess) return TOC_E_CUDA;
  return TOC_OK;
}

// Chunks [k0, k1): their block bytes on copy_stream, an event per chunk.
extern "C" int toc_sweep_upload(const uint8_t* h_blocks, uint8_t* d_blocks, const TocSweepChunk* chunks, int64_t k0,
                                int64_t k1, void* copy_stream) {
  if (!h_blocks || !d_blocks || !chunks || k0 < 0 || k1 < k0) return TOC_E_ARG;
  cudaStream_t cs = (cudaStream_t)copy_stream;
  if (g_timing && k0 == 0) cudaEventRecord(tev(0), cs);
  for (int64_t k = k0; k < k1; ++k) {
    const TocSweepChunk& c = chunks[k];
    if (c.byte_hi < c.byte_lo) return TOC_E_ARG;
    if (cudaMemcpyAsync(d_blocks + c.byte_lo, h_blocks + c.byte_lo, (size_t)(c.byte_hi - c.byte_lo),
                        cudaMemcpyHostToDevice, cs) != cudaSuccess)
      return TOC_E_CUDA;
    if (!c.ev_upload || cudaEventRecord(ev(c.ev_upload), cs) != cudaSuccess) return TOC_E_CUDA;
    if (g_timing) cudaEventRecord(tev(1 + 5 * k), cs);
  }
  return TOC_OK;
}

// v and every chunk's u slice on copy_stream.  Host -> device copies are served in submission
// order whatever the stream, so the operands go on the same stream as the blocks, right after the
// first chunk's: enqueued behind every chunk they would hold the first computation until the end.
extern "C" int toc_sweep_operands(const TocSweepChunk* chunks, int64_t n_chunks, int32_t n_cols, const double* h_v,
                                  double* d_v, const double* h_u, double* d_u, void* copy_stream) {
  if (!chunks || n_chunks < 0 || n_cols < 0 || !h_v || !d_v || !h_u || !d_u) return TOC_E_ARG;
  cudaStream_t cs = (cudaStream_t)copy_stream;
  if (cudaMemcpyAsync(d_v, h_v, sizeof(double) * (size_t)n_cols, cudaMemcpyHostToDevice, cs) != cudaSuccess)
    return TOC_E_CUDA;
  for (int64_t k = 0; k < n_chunks; ++k) {
    const TocSweepChunk& c = chunks[k];
    if (cudaMemcpyAsync(d_u + c.row0, h_u + c.row0, sizeof(double) * (size_t)c.n_rows, cudaMemcpyHostToDevice, cs) !=
        cudaSuccess)
      return TOC_E_CUDA;
    if (!c.ev_operands || cudaEventRecord(ev(c.ev_operands), cs) != cudaSuccess) return TOC_E_CUDA;
  }
  return TOC_OK;
}

// Per chunk, after its bytes and operands: validate / index, fused A.v + v^T.A (compute_stream);
// then R, O and the chunk's index to the pinned host buffers (d2h_stream).
extern "C" int toc_sweep_compute(const TocSweepChunk* chunks, int64_t n_chunks, int32_t n_cols, const double* d_v,
                                 const double* d_u, double* d_R, double* h_R, double* d_O, double* h_O,
                                 TocBlockMeta* h_meta, void* compute_stream, void* d2h_stream) {
  if (!chunks || n_chunks < 0 || n_cols < 0 || !d_v || !d_u || !d_R || !h_R || !d_O || !h_O || !h_meta)
    return TOC_E_ARG;
  cudaStream_t comp = (cudaStream_t)compute_stream, ds = (cudaStream_t)d2h_stream;
  int64_t meta_pos = 0;
  for (int64_t k = 0; k < n_chunks; ++k) {
    const TocSweepChunk& c = chunks[k];
    if (!c.ev_upload || !c.ev_operands || !c.ev_done) return TOC_E_ARG;
    if (cudaStreamWaitEvent(comp, ev(c.ev_upload), 0) != cudaSuccess) return TOC_E_CUDA;
    if (g_timing) cudaEventRecord(tev(2 + 5 * k), comp);
    int rc = toc_index_blocks(c.d_arena, c.d_block_off, c.d_block_len, c.n_blocks, c.d_meta, comp);
    if (rc) return rc;
    if (g_timing) cudaEventRecord(tev(3 + 5 * k), comp);
    if (cudaStreamWaitEvent(comp, ev(c.ev_operands), 0) != cudaSuccess) return TOC_E_CUDA;
    rc = toc_linalg(c.d_arena, c.d_block_off, c.d_meta, c.d_row_base, c.n_blocks, &c.plan, TOC_MATVEC | TOC_VECMAT,
                    d_v, d_R + c.row0, d_u + c.row0, d_O + c.b0 * (int64_t)n_cols, c.d_scratch, comp);
    if (rc) return rc;
    if (g_timing) cudaEventRecord(tev(4 + 5 * k), comp);
    if (cudaEventRecord(ev(c.ev_done), comp) != cudaSuccess || cudaStreamWaitEvent(ds, ev(c.ev_done), 0) != cudaSuccess)
      return TOC_E_CUDA;
    if (cudaMemcpyAsync(h_R + c.row0, d_R + c.row0, sizeof(double) * (size_t)c.n_rows, cudaMemcpyDeviceToHost, ds) !=
            cudaSuccess ||
        cudaMemcpyAsync(h_O + c.b0 * (int64_t)n_cols, d_O + c.b0 * (int64_t)n_cols,
                        sizeof(double) * (size_t)(c.n_blocks * n_cols), cudaMemcpyDeviceToHost, ds) != cudaSuccess ||
        cudaMemcpyAsync(h_meta + meta_pos, c.d_meta, sizeof(TocBlockMeta) * (size_t)c.n_blocks, cudaMemcpyDeviceToHost,
                        ds) != cudaSuccess)
      return TOC_E_CUDA;
    meta_pos += c.n_blocks;
    if (g_timing) cudaEventRecord(tev(5 + 5 * k), ds);
  }
  return TOC_OK;
}
