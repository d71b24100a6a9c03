// toc_exact.cu -- A.v and v^T.A in the reference's own operation order, bit for bit.
//
// Reference: kernels.py:115-142 (matvec: H[i] = value[i] * v[col[i]] + H[parent[i]] for ascending
// i, then each row sums H over its codes left to right) and kernels.py:145-174 (vecmat: h[code] +=
// u[row] row by row, then for descending i: out[col[i]] += value[i] * h[i]; h[parent[i]] += h[i]).
//
// Every floating-point result above depends on a fixed sequence of operands, and the same
// sequence can be evaluated in parallel:
//   H[i]      needs only H[parent[i]]: nodes level by level (a launch per tree depth);
//   R[r]      left-to-right sum of row r's H: a thread per row;
//   h[i]      the u of its occurrences in row order, then the final h of its children in
//             descending id order: a thread per node, level by level from the deepest;
//   out[c]    value * h over the column's nodes in descending id order: a thread per column.
// Products and sums are rounded separately (no contraction), as Python's floats are, so the
// results equal the reference's exactly.  The schedule (levels, child / column / occurrence lists)
// is built on the host from the DecodeTree (kernels.CompressedMatrix, the single-matrix API).
#include "toc_common.cuh"

namespace toc {

__global__ void exact_h_level(const int32_t* __restrict__ nodes, int32_t n, const int32_t* __restrict__ parent,
                              const int32_t* __restrict__ column, const double* __restrict__ value,
                              const double* __restrict__ v, double* H) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t i = nodes[k];
  H[i] = __dadd_rn(__dmul_rn(value[i], v[column[i]]), H[parent[i]]);
}

__global__ void exact_row_sums(const int64_t* __restrict__ rowoff, const int32_t* __restrict__ codes, int32_t n_rows,
                               const double* __restrict__ H, double* R) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  double acc = 0.0;
  for (int64_t j = rowoff[r]; j < rowoff[r + 1]; ++j) acc = __dadd_rn(acc, H[codes[j]]);
  R[r] = acc;
}

// h[i] = the u of node i's occurrences, in row order (the forward pass).
__global__ void exact_occurrences(const int64_t* __restrict__ occ_off, const int32_t* __restrict__ occ_row,
                                  int32_t T, const double* __restrict__ u, double* h) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T) return;
  double acc = 0.0;
  for (int64_t k = occ_off[i]; k < occ_off[i + 1]; ++k) acc = __dadd_rn(acc, u[occ_row[k]]);
  h[i] = acc;
}

// One level of the backward pass: h[p] += h[c] for p's children in descending id order.
__global__ void exact_up_level(const int32_t* __restrict__ nodes, int32_t n, const int64_t* __restrict__ child_off,
                               const int32_t* __restrict__ child, double* h) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t p = nodes[k];
  double acc = h[p];
  for (int64_t q = child_off[p]; q < child_off[p + 1]; ++q) acc = __dadd_rn(acc, h[child[q]]);
  h[p] = acc;
}

// out[c] = sum over the column's nodes in descending id order of value * h.
__global__ void exact_column_sums(const int64_t* __restrict__ col_off, const int32_t* __restrict__ col_node,
                                  int32_t n_cols, const double* __restrict__ value, const double* __restrict__ h,
                                  double* out) {
  const int32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  double acc = 0.0;
  for (int64_t q = col_off[c]; q < col_off[c + 1]; ++q) {
    const int32_t i = col_node[q];
    acc = __dadd_rn(acc, __dmul_rn(value[i], h[i]));
  }
  out[c] = acc;
}

}  // namespace toc

namespace {
unsigned blocks(int64_t n) { return (unsigned)((n + 255) / 256); }
}  // namespace

extern "C" int toc_exact_matvec(const int32_t* d_parent, const int32_t* d_column, const double* d_value,
                                const int32_t* d_level_nodes, const int64_t* h_level_off, int32_t n_levels,
                                const int64_t* d_rowoff, const int32_t* d_codes, int32_t n_rows, const double* d_v,
                                double* d_R, double* d_H, void* stream) {
  if (n_levels < 0 || n_rows < 0 || !h_level_off || (n_rows && (!d_rowoff || !d_R))) return TOC_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(d_H, 0, sizeof(double), s) != cudaSuccess) return TOC_E_CUDA;  // H[root] = 0
  for (int32_t l = 0; l < n_levels; ++l) {
    const int64_t a = h_level_off[l], n = h_level_off[l + 1] - a;
    if (n > 0)
      toc::exact_h_level<<<blocks(n), 256, 0, s>>>(d_level_nodes + a, (int32_t)n, d_parent, d_column, d_value, d_v,
                                                   d_H);
  }
  if (n_rows) toc::exact_row_sums<<<blocks(n_rows), 256, 0, s>>>(d_rowoff, d_codes, n_rows, d_H, d_R);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_exact_vecmat(const int32_t* d_column, const double* d_value, int32_t T,
                                const int32_t* d_level_nodes, const int64_t* h_level_off, int32_t n_levels,
                                const int64_t* d_occ_off, const int32_t* d_occ_row, const int64_t* d_child_off,
                                const int32_t* d_child, const int64_t* d_col_off, const int32_t* d_col_node,
                                int32_t n_cols, const double* d_u, double* d_out, double* d_h, void* stream) {
  if (T < 1 || n_levels < 0 || n_cols < 0 || !h_level_off) return TOC_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  toc::exact_occurrences<<<blocks(T), 256, 0, s>>>(d_occ_off, d_occ_row, T, d_u, d_h);
  for (int32_t l = n_levels - 1; l >= 0; --l) {  // deepest first: children are final
    const int64_t a = h_level_off[l], n = h_level_off[l + 1] - a;
    if (n > 0) toc::exact_up_level<<<blocks(n), 256, 0, s>>>(d_level_nodes + a, (int32_t)n, d_child_off, d_child, d_h);
  }
  if (n_cols) toc::exact_column_sums<<<blocks(n_cols), 256, 0, s>>>(d_col_off, d_col_node, n_cols, d_value, d_h, d_out);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}
