// toc_decode.cu -- decode TOC1 blocks back to CSR rows on the device.
//
// Reference: codec.py:262-292 (node_sequence / decode: each code expands to its pair sequence,
// rows are the concatenation), used by cli.py:194-221 (verify: decode must reproduce the input
// rows bit for bit).  Two passes over the arena, one CTA per block at a time with the decode tree
// rebuilt in shared memory exactly as for the products (toc_batch.cuh):
//   count  per-row pair counts (sum of the rows' code lengths)  -> the caller scans to row_ptr
//   emit   the S lanes of a row prefix-sum their segments' lengths with shuffles, then each code is
//          walked from its last pair to its first (par links), writing (column, value) into its
//          slots from the end.
// Values are the block's value-index entries, so they come back bit for bit.
#include "toc_batch.cuh"

namespace toc {

struct DecodeArgs {
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  const int64_t* row_base;
  int64_t n_blocks;
  int32_t batch_smem_budget;
  int64_t slab_bytes;
  uint8_t* scratch;
  int64_t* row_nnz;        // count pass
  const int64_t* row_ptr;  // emit pass
  int32_t* cols;
  double* vals;
};

template <bool kWide>
TOC_D uint32_t code_len(const Batch<kWide>& B, uint32_t x) {
  uint32_t l = 1;
  while (x > B.nI) {
    x = B.pk.par(x - 1 - B.nI);
    ++l;
  }
  return l;
}

template <bool kWide, bool kEmit>
__global__ void __launch_bounds__(1024, 1) decode_kernel(DecodeArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  uint8_t* p = smem + kFixedBytes;
  uint8_t* slab = a.scratch ? a.scratch + (int64_t)blockIdx.x * a.slab_bytes : nullptr;
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const TocBlockMeta m = a.meta[b];
    if (m.status != TOC_OK || m.corrupt) continue;  // the host refuses such arenas up front
    uint8_t* tables = batch_layout<kWide>(m).total <= (uint32_t)a.batch_smem_budget ? p : slab;
    __syncthreads();
    Batch<kWide> B;
    const uint8_t* blk = a.arena + a.block_off[b];
    B.init(blk, m, tables);
    B.load_index(s_warp);
    B.build_nodes();
    __syncthreads();
    uint2* rec = reinterpret_cast<uint2*>(B.tab);  // (column, value ref) per pair id
    if (kEmit) {
      B.resolve_keys();
      for (uint32_t i = tid; i < B.nI; i += nth)
        rec[i + 1] = make_uint2(ld_packed(blk + m.off_cols, i, m.w_cols), ld_packed(blk + m.off_refs, i, m.w_refs));
      __syncthreads();
    }
    const int64_t rb = a.row_base[b];
    for (uint32_t k = 0; k < B.passes; ++k) {
      uint32_t r = 0, lo = 0, hi = 0, db = 0, j0 = 0, j1 = 0;
      const bool ok = B.segment(k, r, lo, hi, db, j0, j1);
      auto code_at = [&](uint32_t j) { return (j + 1 < hi) ? B.pk.par(db + (j - lo)) : B.last[r]; };
      uint32_t cnt = 0;
      if (ok)
        for (uint32_t j = j0; j < j1; ++j) cnt += code_len(B, code_at(j));
      if (!kEmit) {
        for (uint32_t o = B.S >> 1; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (ok && B.sub == 0) a.row_nnz[rb + r] = cnt;
        continue;
      }
      uint32_t incl = cnt;  // inclusive scan over the row's S lanes (consecutive lanes of a warp)
      for (uint32_t o = 1; o < B.S; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o, B.S);
        if (B.sub >= o) incl += y;
      }
      if (!ok) continue;
      int64_t pos = a.row_ptr[rb + r] + (incl - cnt);
      for (uint32_t j = j0; j < j1; ++j) {
        uint32_t x = code_at(j);
        int64_t e = pos + code_len(B, x);
        pos = e;
        auto emit = [&](uint32_t i) {
          --e;
          const uint2 cr = rec[i];
          a.cols[e] = (int32_t)cr.x;
          a.vals[e] = B.uniq[cr.y];
        };
        while (x > B.nI) {
          uint32_t par, key;
          B.pk.get(x - 1 - B.nI, par, key);
          emit(key);
          x = par;
        }
        emit(x);
      }
    }
  }
}

// The reference's DecodeTree arrays (codec.py:194-259) for every block: node 0 is the root
// (parent, column, first_col = -1; value, first_val = 0.0), nodes 1..|I| mirror I, derived node
// d has parent = par(d) and the (column, value) of its key pair; first_* is the node's first
// pair, found by following par links to the first layer.  Block b's nodes start at tree_base[b].
struct TreeArrays {
  const int64_t* tree_base;
  int32_t* parent;
  int32_t* column;
  double* value;
  int32_t* first_col;
  double* first_val;
};

template <bool kWide>
__global__ void __launch_bounds__(1024, 1) tree_arrays_kernel(DecodeArgs a, TreeArrays o) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  uint8_t* p = smem + kFixedBytes;
  uint8_t* slab = a.scratch ? a.scratch + (int64_t)blockIdx.x * a.slab_bytes : nullptr;
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const TocBlockMeta m = a.meta[b];
    if (m.status != TOC_OK || m.corrupt) continue;
    uint8_t* tables = batch_layout<kWide>(m).total <= (uint32_t)a.batch_smem_budget ? p : slab;
    __syncthreads();
    Batch<kWide> B;
    const uint8_t* blk = a.arena + a.block_off[b];
    B.init(blk, m, tables);
    B.load_index(s_warp);
    B.build_nodes();
    __syncthreads();
    B.resolve_keys();
    uint2* rec = reinterpret_cast<uint2*>(B.tab);
    for (uint32_t i = tid; i < B.nI; i += nth)
      rec[i + 1] = make_uint2(ld_packed(blk + m.off_cols, i, m.w_cols), ld_packed(blk + m.off_refs, i, m.w_refs));
    __syncthreads();
    const int64_t base = o.tree_base[b];
    const uint32_t T = 1u + B.nI + m.n_derived;
    for (uint32_t x = tid; x < T; x += nth) {
      int32_t par = -1, col = -1, fcol = -1;
      double val = 0.0, fval = 0.0;
      if (x >= 1) {
        uint32_t key = x, f = x;
        par = 0;
        if (x > B.nI) {
          uint32_t pr;
          B.pk.get(x - 1 - B.nI, pr, key);
          par = (int32_t)pr;
          f = pr;
          while (f > B.nI) f = B.pk.par(f - 1 - B.nI);
        }
        col = (int32_t)rec[key].x;
        val = B.uniq[rec[key].y];
        fcol = (int32_t)rec[f].x;
        fval = B.uniq[rec[f].y];
      }
      o.parent[base + x] = par;
      o.column[base + x] = col;
      o.value[base + x] = val;
      o.first_col[base + x] = fcol;
      o.first_val[base + x] = fval;
    }
  }
}

}  // namespace toc

// ------------------------------------------------------------------------------------------
namespace {

int decode_launch(const toc::DecodeArgs& a0, const TocPlan* plan, bool emit, cudaStream_t s) {
  toc::DecodeArgs a = a0;
  a.batch_smem_budget = plan->smem_bytes - (int32_t)toc::kFixedBytes;
  a.slab_bytes = plan->global_tables ? plan->scratch_bytes / plan->ctas : 0;
  void* fn = plan->wide ? (emit ? (void*)toc::decode_kernel<true, true> : (void*)toc::decode_kernel<true, false>)
                        : (emit ? (void*)toc::decode_kernel<false, true> : (void*)toc::decode_kernel<false, false>);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan->smem_bytes) != cudaSuccess)
    return TOC_E_CUDA;
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3(plan->ctas), dim3(plan->threads), args, plan->smem_bytes, s) == cudaSuccess
             ? TOC_OK
             : TOC_E_CUDA;
}

}  // namespace

extern "C" int toc_decode_counts(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                 const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int64_t* d_row_nnz,
                                 void* d_scratch, void* stream) {
  if (!plan || n_blocks < 0 || !d_row_nnz) return TOC_E_ARG;
  if (plan->global_tables && !d_scratch) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  toc::DecodeArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.n_blocks = n_blocks;
  a.scratch = (uint8_t*)d_scratch;
  a.row_nnz = d_row_nnz;
  return decode_launch(a, plan, false, (cudaStream_t)stream);
}

extern "C" int toc_decode_rows(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                               const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, const int64_t* d_row_ptr,
                               int32_t* d_cols, double* d_vals, void* d_scratch, void* stream) {
  if (!plan || n_blocks < 0 || !d_row_ptr) return TOC_E_ARG;
  if (plan->global_tables && !d_scratch) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  toc::DecodeArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.n_blocks = n_blocks;
  a.scratch = (uint8_t*)d_scratch;
  a.row_ptr = d_row_ptr;
  a.cols = d_cols;
  a.vals = d_vals;
  return decode_launch(a, plan, true, (cudaStream_t)stream);
}

extern "C" int toc_tree_arrays(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                               int64_t n_blocks, const TocPlan* plan, const int64_t* d_tree_base, int32_t* d_parent,
                               int32_t* d_column, double* d_value, int32_t* d_first_col, double* d_first_val,
                               void* d_scratch, void* stream) {
  if (!plan || n_blocks < 0 || !d_tree_base || !d_parent || !d_column || !d_value || !d_first_col || !d_first_val)
    return TOC_E_ARG;
  if (plan->global_tables && !d_scratch) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  toc::DecodeArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.n_blocks = n_blocks;
  a.scratch = (uint8_t*)d_scratch;
  a.batch_smem_budget = plan->smem_bytes - (int32_t)toc::kFixedBytes;
  a.slab_bytes = plan->global_tables ? plan->scratch_bytes / plan->ctas : 0;
  toc::TreeArrays o{d_tree_base, d_parent, d_column, d_value, d_first_col, d_first_val};
  void* fn = plan->wide ? (void*)toc::tree_arrays_kernel<true> : (void*)toc::tree_arrays_kernel<false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan->smem_bytes) != cudaSuccess)
    return TOC_E_CUDA;
  void* args[] = {&a, &o};
  return cudaLaunchKernel(fn, dim3(plan->ctas), dim3(plan->threads), args, plan->smem_bytes, (cudaStream_t)stream) ==
                 cudaSuccess
             ? TOC_OK
             : TOC_E_CUDA;
}
