// toc_matmat.cu -- A.M and M.A directly on TOC1 blocks (sm_100a).
//
// Reference: kernels.py:177-203 (matmat_right, Algorithm 8) and kernels.py:206-234
// (matmat_left, Algorithm 9); used by the network trainer (training.py:224-228, 284-293).
//
// Both kernels rebuild the batch's node tables in shared memory (toc_batch.cuh) and unpack the
// first layer to (column, value ref) words in place of P1.
//   A.M  [n x p] = A [n x m] . M [m x p]: a warp per row, lanes across the p columns of M; the
//        chain walk of each code is warp-uniform (every lane follows the same chain), each pair
//        adds value * M[col, :] -- one coalesced row read of M per pair.  No atomics.
//   M.A  [p x m] = M [p x n] . A [n x m]: the grid splits the m output columns into ranges, one
//        CTA per (batch, range); each warp privately owns a sub-range of columns, walks every row
//        and keeps out^T[c, :] for its columns in shared memory, lanes across p.  M is given
//        transposed ([n x p], lanes read contiguous rows).  No atomics.
// Arithmetic is fp64 FMA-free multiply + add in the per-pair order (within 1e-9 of the reference,
// which sums node prefixes first).
#include "toc_batch.cuh"

namespace toc {

struct MatmatArgs {
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  const int64_t* row_base;
  int64_t n_blocks;
  int32_t n_cols;   // m
  int32_t p;        // lanes of M
  int32_t splits;   // row splits (right) / column ranges (left) per batch
  int32_t batch_smem_budget;
  int64_t slab_bytes;
  const double* M;  // right: [m x p];  left: M^T [n_total x p]
  double* out;      // right: [n_total x p];  left: [n_blocks x p x m]
  uint8_t* scratch;
};

constexpr int kMaxLaneTiles = 8;  // p <= 256 per pass (lanes x tiles); larger p loops

template <bool kWide>
TOC_D void unpack_pairs(Batch<kWide>& B) {
  if (B.p0 >= B.p1) return;
  with_width(B.m.w_cols, [&]<int W>() {
    SeqReader<W> rd;
    rd.init(B.blk + B.m.off_cols, B.p0);
    for (uint32_t i = B.p0; i < B.p1; ++i) B.tabw[2 * (i + 1)] = rd.next();
  });
  with_width(B.m.w_refs, [&]<int W>() {
    SeqReader<W> rd;
    rd.init(B.blk + B.m.off_refs, B.p0);
    for (uint32_t i = B.p0; i < B.p1; ++i) B.tabw[2 * (i + 1) + 1] = rd.next();
  });
}

template <bool kWide>
TOC_D void build_tables(Batch<kWide>& B, uint32_t* s_warp) {
  B.load_index(s_warp);
  B.build_nodes();
  unpack_pairs(B);
  __syncthreads();
  B.resolve_keys();
  __syncthreads();
}

// Each code of row r (positions [lo, hi)) visited in order; visit(i) per pair, warp-uniform.
template <bool kWide, typename V>
TOC_D void walk_row(const Batch<kWide>& B, uint32_t r, V&& visit) {
  const uint32_t lo = B.rowoff[r], hi = B.rowoff[r + 1], db = B.dbase[r];
  B.walk(r, lo, hi, db, lo, hi, visit);
}

template <bool kWide>
__global__ void __launch_bounds__(512, 1) matmat_right_kernel(MatmatArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  uint8_t* p = smem + kFixedBytes;
  const int64_t b = blockIdx.x;
  const TocBlockMeta m = a.meta[b];
  if (m.status != TOC_OK || m.corrupt) return;
  const uint32_t need = batch_layout<kWide>(m).total;
  uint8_t* tables = need <= (uint32_t)a.batch_smem_budget ? p : a.scratch + (int64_t)blockIdx.x * a.slab_bytes;
  Batch<kWide> B;
  B.init(a.arena + a.block_off[b], m, tables);
  build_tables(B, s_warp);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t P = (uint32_t)a.p;
  const int64_t rb = a.row_base[b];
  for (uint32_t r = blockIdx.y * nwarps + warp; r < B.n; r += gridDim.y * nwarps) {
    for (uint32_t j0 = 0; j0 < P; j0 += 32 * kMaxLaneTiles) {
      double acc[kMaxLaneTiles];
#pragma unroll
      for (int k = 0; k < kMaxLaneTiles; ++k) acc[k] = 0.0;
      walk_row(B, r, [&](uint32_t i) {
        const uint32_t col = B.tabw[2 * i];
        const double val = B.uniq[B.tabw[2 * i + 1]];
        const double* mrow = a.M + (int64_t)col * P;
#pragma unroll
        for (int k = 0; k < kMaxLaneTiles; ++k) {
          const uint32_t j = j0 + lane + 32 * k;
          if (j < P) acc[k] = __dadd_rn(acc[k], __dmul_rn(val, __ldg(mrow + j)));
        }
      });
      double* o = a.out + (rb + r) * (int64_t)P;
#pragma unroll
      for (int k = 0; k < kMaxLaneTiles; ++k) {
        const uint32_t j = j0 + lane + 32 * k;
        if (j < P) o[j] = acc[k];
      }
    }
  }
}

// M.A: CTA (b, range); warp w owns columns [c0 + w*cw, c0 + (w+1)*cw) of the range; for each of
// its columns an out^T row of p doubles lives in shared memory.
template <bool kWide>
__global__ void __launch_bounds__(512, 1) matmat_left_kernel(MatmatArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  uint8_t* p = smem + kFixedBytes;
  const int64_t b = blockIdx.x;
  const TocBlockMeta m = a.meta[b];
  if (m.status != TOC_OK || m.corrupt) return;
  const uint32_t P = (uint32_t)a.p, ncol = (uint32_t)a.n_cols;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t range = (ncol + gridDim.y - 1) / gridDim.y;
  const uint32_t c0 = min(ncol, blockIdx.y * range), c1 = min(ncol, c0 + range);
  const uint32_t cw = (c1 - c0 + nwarps - 1) / nwarps;
  const uint32_t wc0 = min(c1, c0 + warp * cw), wc1 = min(c1, wc0 + cw);
  double* acc = reinterpret_cast<double*>(p);  // [(c1 - c0) x P]
  p += align16(8u * range * P);
  const uint32_t need = batch_layout<kWide>(m).total;
  uint8_t* tables = need <= (uint32_t)a.batch_smem_budget ? p : a.scratch + (int64_t)(blockIdx.x * gridDim.y + blockIdx.y) * a.slab_bytes;
  for (uint32_t k = threadIdx.x; k < (c1 - c0) * P; k += blockDim.x) acc[k] = 0.0;
  Batch<kWide> B;
  B.init(a.arena + a.block_off[b], m, tables);
  build_tables(B, s_warp);
  const int64_t rb = a.row_base[b];
  if (wc0 < wc1) {
    for (uint32_t r = 0; r < B.n; ++r) {
      const double* mt = a.M + (rb + r) * (int64_t)P;  // M[:, row r]
      walk_row(B, r, [&](uint32_t i) {
        const uint32_t col = B.tabw[2 * i];
        if (col < wc0 || col >= wc1) return;
        const double val = B.uniq[B.tabw[2 * i + 1]];
        double* row = acc + (col - c0) * P;
        for (uint32_t j = lane; j < P; j += 32) row[j] = __dadd_rn(row[j], __dmul_rn(val, __ldg(mt + j)));
      });
    }
  }
  __syncthreads();
  double* o = a.out + b * (int64_t)P * ncol;  // [p x m] for batch b
  for (uint32_t k = threadIdx.x; k < (c1 - c0) * P; k += blockDim.x) {
    const uint32_t c = k / P, j = k % P;
    o[(int64_t)j * ncol + c0 + c] = acc[k];
  }
}

}  // namespace toc

namespace {

int dev_attr(cudaDeviceAttr attr, int fallback) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, attr, dev) != cudaSuccess || v <= 0)
    return fallback;
  return v;
}

}  // namespace

extern "C" int toc_matmat(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                          const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks, int32_t n_cols,
                          int32_t side, int32_t p, const double* d_M, double* d_out, void* d_scratch,
                          int64_t scratch_bytes, void* stream) {
  if (n_blocks < 0 || p < 1 || !h_meta || !d_M || !d_out || (side != 0 && side != 1)) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  bool wide = false;
  uint32_t max_need = 0;
  for (int64_t b = 0; b < n_blocks; ++b) {
    if (h_meta[b].status != TOC_OK || h_meta[b].corrupt) return TOC_E_ARG;
    if (1ull + h_meta[b].n_pairs + h_meta[b].n_derived > 65536ull) wide = true;
  }
  for (int64_t b = 0; b < n_blocks; ++b) {
    const uint32_t need = wide ? toc::batch_layout<true>(h_meta[b]).total : toc::batch_layout<false>(h_meta[b]).total;
    if (need > max_need) max_need = need;
  }
  const int optin = dev_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448);
  const int sms = dev_attr(cudaDevAttrMultiProcessorCount, 148);
  toc::MatmatArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.n_blocks = n_blocks;
  a.n_cols = n_cols;
  a.p = p;
  a.M = d_M;
  a.out = d_out;
  a.scratch = (uint8_t*)d_scratch;
  const int threads = 512;
  // enough CTAs to fill the GPU: splits per batch so that n_blocks * splits >= 2 * SMs
  int splits = (int)((2 * sms + n_blocks - 1) / n_blocks);
  if (splits < 1) splits = 1;
  uint32_t fixed = toc::kFixedBytes;
  if (side == 1) {
    // column ranges: the out^T slice must fit next to the tables
    if (splits < 8) splits = 8;
    while (toc::align16(8u * ((n_cols + splits - 1) / splits) * (uint32_t)p) > 64u * 1024u) splits *= 2;
    if (splits > n_cols) splits = n_cols > 0 ? n_cols : 1;
    fixed += toc::align16(8u * ((n_cols + splits - 1) / splits) * (uint32_t)p);
  } else if (splits > 16) {
    splits = 16;
  }
  if (fixed > (uint32_t)optin) return TOC_E_ARG;
  const uint32_t budget = (uint32_t)optin - fixed;
  a.batch_smem_budget = (int32_t)(max_need <= budget ? max_need : budget);
  a.splits = splits;
  if (max_need > budget) {
    a.slab_bytes = toc::align16(max_need);
    if (!d_scratch || scratch_bytes < a.slab_bytes * n_blocks * splits) return TOC_E_ARG;
  }
  const int smem = (int)(fixed + (uint32_t)a.batch_smem_budget);
  void* fn = side == 0 ? (wide ? (void*)toc::matmat_right_kernel<true> : (void*)toc::matmat_right_kernel<false>)
                       : (wide ? (void*)toc::matmat_left_kernel<true> : (void*)toc::matmat_left_kernel<false>);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return TOC_E_CUDA;
  void* args[] = {&a};
  cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)n_blocks, (unsigned)splits), dim3(threads), args, smem,
                                   (cudaStream_t)stream);
  return e == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_matmat_scratch(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t side,
                                  int32_t p, int64_t* bytes) {
  // Oversized batches use a global slab per CTA; report the worst case (no device needed).
  if (!h_meta || n_blocks < 0 || !bytes) return TOC_E_ARG;
  uint32_t max_need = 0;
  bool wide = false;
  for (int64_t b = 0; b < n_blocks; ++b)
    if (1ull + h_meta[b].n_pairs + h_meta[b].n_derived > 65536ull) wide = true;
  for (int64_t b = 0; b < n_blocks; ++b) {
    const uint32_t need = wide ? toc::batch_layout<true>(h_meta[b]).total : toc::batch_layout<false>(h_meta[b]).total;
    if (need > max_need) max_need = need;
  }
  const int sms = dev_attr(cudaDevAttrMultiProcessorCount, 148);
  int splits = (int)((2 * sms + (n_blocks ? n_blocks : 1) - 1) / (n_blocks ? n_blocks : 1));
  if (side == 1) {
    if (splits < 8) splits = 8;
    while (toc::align16(8u * ((n_cols + splits - 1) / splits) * (uint32_t)p) > 64u * 1024u) splits *= 2;
    if (splits > n_cols) splits = n_cols > 0 ? n_cols : 1;
  } else if (splits > 16) {
    splits = 16;
  }
  *bytes = (int64_t)toc::align16(max_need) * n_blocks * (splits < 1 ? 1 : splits);
  return TOC_OK;
}
