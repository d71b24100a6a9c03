// toc_dense.cu -- the reference's uncompressed baselines, on the device, bit for bit.
//
// Reference: matrix.py:164-279 (dense_matvec, dense_vecmat, dense_matmat, csr_matvec,
// csr_vecmat, csr_matmat_right, csr_matmat_left).  The reference accumulates every output in a
// fixed ascending order with separate IEEE multiplies and adds (Python floats / numpy elementwise
// ops).  One thread owns one output element and runs exactly that chain with __dmul_rn /
// __dadd_rn (no FMA contraction), so every result equals the reference's bit for bit.  These are
// the dense / CSR execution layouts of train() (training.py:159-203) and the parity oracles the
// reference's own tests compare the compressed kernels against -- not the hot path.
#include <cstdint>

#include "toc_b200.h"

namespace {

__global__ void dense_matvec_kernel(const double* __restrict__ A, int64_t n, int64_t m, const double* __restrict__ v,
                                    double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double* row = A + i * m;
    double acc = 0.0;
    for (int64_t j = 0; j < m; ++j) acc = __dadd_rn(acc, __dmul_rn(row[j], v[j]));  // matrix.py:169-171
    out[i] = acc;
  }
}

__global__ void dense_vecmat_kernel(const double* __restrict__ v, const double* __restrict__ A, int64_t n, int64_t m,
                                    double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, __dmul_rn(v[i], A[i * m + j]));  // matrix.py:181-184
    out[j] = acc;
  }
}

__global__ void dense_matmat_kernel(const double* __restrict__ A, const double* __restrict__ M, int64_t n, int64_t k,
                                    int64_t p, double* __restrict__ out) {
  const int64_t total = n * p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / p, j = e % p;
    double acc = 0.0;
    for (int64_t q = 0; q < k; ++q) acc = __dadd_rn(acc, __dmul_rn(A[i * k + q], M[q * p + j]));  // matrix.py:199-204
    out[e] = acc;
  }
}

__global__ void csr_matvec_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                  const double* __restrict__ vals, int64_t n, const double* __restrict__ v,
                                  double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) acc = __dadd_rn(acc, __dmul_rn(vals[e], v[cols[e]]));  // :235-238
    out[i] = acc;
  }
}

// Column-major (CSC) view of the same entries, rows ascending within a column: the reference's
// row-order scatter out[col] += v_i * val (matrix.py:242-249) as a per-column ordered sum.
__global__ void csc_vecmat_kernel(const int64_t* __restrict__ cp, const int32_t* __restrict__ rows,
                                  const double* __restrict__ vals, int64_t m, const double* __restrict__ v,
                                  double* __restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t e = cp[c]; e < cp[c + 1]; ++e) acc = __dadd_rn(acc, __dmul_rn(v[rows[e]], vals[e]));
    out[c] = acc;
  }
}

__global__ void csr_matmat_right_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                        const double* __restrict__ vals, int64_t n, const double* __restrict__ M,
                                        int64_t p, double* __restrict__ out) {
  const int64_t total = n * p;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / p, j = x % p;
    double acc = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) acc = __dadd_rn(acc, __dmul_rn(vals[e], M[cols[e] * p + j]));  // :262-264
    out[x] = acc;
  }
}

__global__ void csc_matmat_left_kernel(const int64_t* __restrict__ cp, const int32_t* __restrict__ rows,
                                       const double* __restrict__ vals, int64_t m, const double* __restrict__ M,
                                       int64_t p, int64_t n, double* __restrict__ out) {
  const int64_t total = p * m;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = x / m, c = x % m;
    double acc = 0.0;
    for (int64_t e = cp[c]; e < cp[c + 1]; ++e) acc = __dadd_rn(acc, __dmul_rn(M[r * n + rows[e]], vals[e]));  // :276-278
    out[x] = acc;
  }
}

int grid_for(int64_t work) {
  int64_t g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

int done() { return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA; }

}  // namespace

extern "C" int toc_dense_matvec(const double* d_A, int64_t n, int64_t m, const double* d_v, double* d_out,
                                void* stream) {
  if (n < 0 || m < 0 || (n && !d_out) || (n && m && !d_A) || (m && !d_v)) return TOC_E_ARG;
  if (n == 0) return TOC_OK;
  dense_matvec_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_A, n, m, d_v, d_out);
  return done();
}

extern "C" int toc_dense_vecmat(const double* d_v, const double* d_A, int64_t n, int64_t m, double* d_out,
                                void* stream) {
  if (n < 0 || m < 0 || (m && !d_out) || (n && m && (!d_A || !d_v))) return TOC_E_ARG;
  if (m == 0) return TOC_OK;
  dense_vecmat_kernel<<<grid_for(m), 256, 0, (cudaStream_t)stream>>>(d_v, d_A, n, m, d_out);
  return done();
}

extern "C" int toc_dense_matmat(const double* d_A, const double* d_M, int64_t n, int64_t k, int64_t p, double* d_out,
                                void* stream) {
  if (n < 0 || k < 0 || p < 0 || (n * p && !d_out) || (n * k && !d_A) || (k * p && !d_M)) return TOC_E_ARG;
  if (n * p == 0) return TOC_OK;
  dense_matmat_kernel<<<grid_for(n * p), 256, 0, (cudaStream_t)stream>>>(d_A, d_M, n, k, p, d_out);
  return done();
}

extern "C" int toc_csr_matvec(const int64_t* d_row_ptr, const int32_t* d_cols, const double* d_vals, int64_t n_rows,
                              const double* d_v, double* d_out, void* stream) {
  if (n_rows < 0 || (n_rows && (!d_row_ptr || !d_out))) return TOC_E_ARG;
  if (n_rows == 0) return TOC_OK;
  csr_matvec_kernel<<<grid_for(n_rows), 256, 0, (cudaStream_t)stream>>>(d_row_ptr, d_cols, d_vals, n_rows, d_v, d_out);
  return done();
}

extern "C" int toc_csc_vecmat(const int64_t* d_col_ptr, const int32_t* d_rows, const double* d_vals, int64_t n_cols,
                              const double* d_v, double* d_out, void* stream) {
  if (n_cols < 0 || (n_cols && (!d_col_ptr || !d_out))) return TOC_E_ARG;
  if (n_cols == 0) return TOC_OK;
  csc_vecmat_kernel<<<grid_for(n_cols), 256, 0, (cudaStream_t)stream>>>(d_col_ptr, d_rows, d_vals, n_cols, d_v, d_out);
  return done();
}

extern "C" int toc_csr_matmat_right(const int64_t* d_row_ptr, const int32_t* d_cols, const double* d_vals,
                                    int64_t n_rows, const double* d_M, int64_t p, double* d_out, void* stream) {
  if (n_rows < 0 || p < 0 || (n_rows * p && (!d_row_ptr || !d_out))) return TOC_E_ARG;
  if (n_rows * p == 0) return TOC_OK;
  csr_matmat_right_kernel<<<grid_for(n_rows * p), 256, 0, (cudaStream_t)stream>>>(d_row_ptr, d_cols, d_vals, n_rows,
                                                                                   d_M, p, d_out);
  return done();
}

extern "C" int toc_csc_matmat_left(const int64_t* d_col_ptr, const int32_t* d_rows, const double* d_vals,
                                   int64_t n_cols, const double* d_M, int64_t p, int64_t n_rows, double* d_out,
                                   void* stream) {
  if (n_cols < 0 || p < 0 || n_rows < 0 || (n_cols * p && (!d_col_ptr || !d_out))) return TOC_E_ARG;
  if (n_cols * p == 0) return TOC_OK;
  csc_matmat_left_kernel<<<grid_for(n_cols * p), 256, 0, (cudaStream_t)stream>>>(d_col_ptr, d_rows, d_vals, n_cols,
                                                                                  d_M, p, n_rows, d_out);
  return done();
}
