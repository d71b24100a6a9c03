// toc_matcache.cu -- A.M and M.A over large batches from a per-batch node-record cache.
//
// Reference: kernels.py:177-203 (matmat_right, Algorithm 8), kernels.py:206-234 (matmat_left,
// Algorithm 9); the network trainer calls them once per step on one batch (training.py:224-228,
// 284-293).  toc_matmat.cu rebuilds each batch's node tables in shared memory; a batch whose tree
// is larger than shared memory (config 5: 250 dense 784-column rows, ~10^5 nodes) then rebuilds
// them in a global slab inside every CTA, and its M.A kernel walks the whole batch once per column
// range.  Here the tables are built once per arena into a cache entry per batch:
//   header   n_rows, n_codes, T, |I|, n_cols (u32), max |value| (f64)           32 B
//   rowoff   u32[n + 1]         codes   u32[C] (the code stream D)
//   nodes    {par u32, col u32, value f64}[T]: node x's own pair and parent (node 0 unused), so
//            one 16-byte load advances a chain by one pair
// and both products walk chains with K codes in flight per warp (a slot takes the row's next code
// as soon as its chain ends), lanes across 32 columns of M (warp-uniform control flow).
//   A.M   CTA (row, 32-column chunk of M): 8 warps take consecutive eighths of the row's codes;
//         partial sums reduced in shared memory in warp order.  No atomics.
//   M.A   CTA (row group, chunk, column range): 32 warps walk the group's codes and add
//         value * M^T[row, chunk] into a shared (columns x 32) tile in exact fixed point (split
//         words, consecutive lanes -> consecutive banks); tiles of the row groups are summed
//         exactly in a second pass.  Per-column scales from sum_r |M^T[r, j]| * max |value|.
#include <algorithm>

#include "toc_batch.cuh"

namespace toc {

struct NodeRec {
  uint32_t par, col;
  double val;
};

struct McLayout {
  uint32_t off_rowoff, off_codes, off_nodes, total;
};

constexpr uint32_t kMcHeader = 32;

TOC_HD McLayout mc_layout(const TocBlockMeta& m) {
  McLayout L;
  uint32_t o = kMcHeader;
  L.off_rowoff = o;
  o += align16(4u * (m.n_rows + 1));
  L.off_codes = o;
  o += align16(4u * m.n_codes);
  L.off_nodes = o;
  o += 16u * (1u + m.n_pairs + m.n_derived);
  L.total = o;
  return L;
}

struct McArgs {
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  int64_t n_blocks;
  int32_t batch_smem_budget;
  int64_t slab_bytes;
  uint8_t* scratch;
  uint8_t* cache;
  const int64_t* cache_off;
};

// One CTA per block: tables rebuilt (shared memory or slab), then the entry written.
template <bool kWide>
__global__ void __launch_bounds__(1024, 1) mc_build_kernel(McArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  double* s_red = reinterpret_cast<double*>(smem + 160);
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
    const McLayout L = mc_layout(m);
    uint8_t* e = a.cache + a.cache_off[b];
    uint32_t* rowoff = reinterpret_cast<uint32_t*>(e + L.off_rowoff);
    uint32_t* codes = reinterpret_cast<uint32_t*>(e + L.off_codes);
    NodeRec* nodes = reinterpret_cast<NodeRec*>(e + L.off_nodes);
    for (uint32_t r = tid; r <= B.n; r += nth) rowoff[r] = B.rowoff[r];
    for (uint32_t k = 0; k < B.passes; ++k) {
      uint32_t r, lo, hi, db, j0, j1;
      if (!B.segment(k, r, lo, hi, db, j0, j1)) break;
      for (uint32_t j = j0; j < j1; ++j) codes[j] = (j + 1 < hi) ? B.pk.par(db + (j - lo)) : B.last[r];
    }
    const uint32_t T = 1u + B.nI + m.n_derived;
    for (uint32_t x = tid; x < T; x += nth) {
      NodeRec n{0u, 0u, 0.0};
      if (x >= 1) {
        uint32_t key = x;
        if (x > B.nI) B.pk.get(x - 1 - B.nI, n.par, key);
        n.col = rec[key].x;
        n.val = B.uniq[rec[key].y];
      }
      nodes[x] = n;
    }
    const double vmax = block_max_d(B.vmax, s_red);
    if (tid == 0) {
      uint32_t* h = reinterpret_cast<uint32_t*>(e);
      h[0] = B.n;
      h[1] = m.n_codes;
      h[2] = T;
      h[3] = B.nI;
      h[4] = m.n_cols;
      reinterpret_cast<double*>(e)[3] = vmax;
    }
  }
}

TOC_D NodeRec ld_node(const NodeRec* nodes, uint32_t x) {
  const uint4 w = __ldg(reinterpret_cast<const uint4*>(nodes) + x);
  NodeRec n;
  n.par = w.x;
  n.col = w.y;
  n.val = __hiloint2double((int)w.w, (int)w.z);
  return n;
}

// Codes [j0, j1) with K chains in flight: visit(pair column, pair value, code position).
template <int K, typename V>
TOC_D void walk_slots(const NodeRec* nodes, const uint32_t* codes, uint32_t j0, uint32_t j1, V&& visit) {
  uint32_t x[K], pos[K];
  uint32_t nj = j0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    pos[k] = nj;
    x[k] = nj < j1 ? __ldg(codes + nj) : 0u;
    nj += nj < j1 ? 1u : 0u;
  }
  for (;;) {
    bool any = false;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (x[k]) {
        const NodeRec n = ld_node(nodes, x[k]);
        visit(n.col, n.val, pos[k]);
        x[k] = n.par;
        if (!x[k] && nj < j1) {
          pos[k] = nj;
          x[k] = __ldg(codes + nj);
          ++nj;
        }
        any = true;
      }
    }
    if (!any) break;
  }
}

constexpr int kSlots = 8;

struct McRightArgs {
  const uint8_t* cache;
  const int64_t* cache_off;
  const int64_t* row_base;  // first output row of each batch
  int64_t n_blocks;
  int32_t p;
  const double* M;  // [m x p]
  double* out;      // [rows x p]
};

// CTA (output row, 32-column chunk); 8 warps split the row's codes.
__global__ void __launch_bounds__(256) mc_right_kernel(McRightArgs a) {
  __shared__ double s_part[8][32];
  const int64_t row = blockIdx.x;
  int64_t lo = 0, hi = a.n_blocks - 1;  // batch of this row: last b with row_base[b] <= row
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (a.row_base[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  const int64_t b = lo;
  const uint8_t* e = a.cache + a.cache_off[b];
  const uint32_t* h = reinterpret_cast<const uint32_t*>(e);
  TocBlockMeta m{};
  m.n_rows = h[0];
  m.n_codes = h[1];
  m.n_pairs = h[3];
  m.n_derived = h[2] - 1 - h[3];
  const McLayout L = mc_layout(m);
  const uint32_t r = (uint32_t)(row - a.row_base[b]);
  const uint32_t* rowoff = reinterpret_cast<const uint32_t*>(e + L.off_rowoff);
  const uint32_t* codes = reinterpret_cast<const uint32_t*>(e + L.off_codes);
  const NodeRec* nodes = reinterpret_cast<const NodeRec*>(e + L.off_nodes);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t P = (uint32_t)a.p, j = blockIdx.y * 32 + lane;
  const uint32_t c0 = __ldg(rowoff + r), len = __ldg(rowoff + r + 1) - c0;
  const uint32_t j0 = c0 + (len * warp) / 8, j1 = c0 + (len * (warp + 1)) / 8;
  double acc = 0.0;
  const bool on = j < P;
  walk_slots<kSlots>(nodes, codes, j0, j1, [&](uint32_t col, double val, uint32_t) {
    if (on) acc = __dadd_rn(acc, __dmul_rn(val, __ldg(a.M + (int64_t)col * P + j)));
  });
  s_part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && on) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += s_part[w][lane];
    a.out[row * (int64_t)P + j] = s;
  }
}

struct McLeftArgs {
  const uint8_t* entry;  // one batch's cache entry
  int32_t p, n_cols;
  int32_t groups, cw;    // row groups; columns per range
  const double* MT;      // M^T rows of this batch: [n x p]
  const double* scale;   // [p] fixed-point scale per output column of M
  long long* tiles;      // [groups][chunks][ranges][cw][32]
};

// Sum_r |M^T[r, j]| * max|value| -> fix_scale per j (one thread per j).
__global__ void mc_scale_kernel(const double* MT, int32_t n, int32_t p, const uint8_t* entry, double* scale) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p) return;
  double s = 0.0;
  for (int32_t r = 0; r < n; ++r) s += fabs(MT[(int64_t)r * p + j]);
  scale[j] = fix_scale(s * reinterpret_cast<const double*>(entry)[3]);
}

__global__ void __launch_bounds__(1024, 1) mc_left_kernel(McLeftArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint8_t* e = a.entry;
  const uint32_t* h = reinterpret_cast<const uint32_t*>(e);
  TocBlockMeta m{};
  m.n_rows = h[0];
  m.n_codes = h[1];
  m.n_pairs = h[3];
  m.n_derived = h[2] - 1 - h[3];
  const McLayout L = mc_layout(m);
  const uint32_t* rowoff = reinterpret_cast<const uint32_t*>(e + L.off_rowoff);
  const uint32_t* codes = reinterpret_cast<const uint32_t*>(e + L.off_codes);
  const NodeRec* nodes = reinterpret_cast<const NodeRec*>(e + L.off_nodes);
  const uint32_t g = blockIdx.x, chunk = blockIdx.y, range = blockIdx.z;
  const uint32_t n = m.n_rows, G = (uint32_t)a.groups, CW = (uint32_t)a.cw;
  const uint32_t r0 = (uint32_t)(((uint64_t)n * g) / G), r1 = (uint32_t)(((uint64_t)n * (g + 1)) / G);
  const uint32_t cbase = range * CW, cend = min((uint32_t)a.n_cols, cbase + CW);
  uint32_t* tlo = reinterpret_cast<uint32_t*>(smem);
  uint32_t* thi = tlo + CW * 32;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (uint32_t k = tid; k < 2 * CW * 32; k += blockDim.x) tlo[k] = 0u;
  __syncthreads();
  const uint32_t P = (uint32_t)a.p, j = chunk * 32 + lane;
  const bool on = j < P;
  const double sc = on ? a.scale[j] : 0.0;
  const uint32_t q0 = __ldg(rowoff + r0), q1 = __ldg(rowoff + r1), span = q1 - q0;
  const uint32_t w0 = q0 + (uint32_t)(((uint64_t)span * warp) / nwarps);
  const uint32_t w1 = q0 + (uint32_t)(((uint64_t)span * (warp + 1)) / nwarps);
  uint32_t rr = r0;  // row of code position `pos` (positions visited in increasing order per slot refill)
  double mt = 0.0;
  uint32_t mt_row = 0xffffffffu;
  walk_slots<kSlots>(nodes, codes, w0, w1, [&](uint32_t col, double val, uint32_t pos) {
    if (col < cbase || col >= cend) return;
    uint32_t r = rr;
    while (__ldg(rowoff + r + 1) <= pos) ++r;  // rows advance monotonically with new codes
    while (__ldg(rowoff + r) > pos) --r;       // an older slot may still hold an earlier row
    rr = r;
    if (r != mt_row) {
      mt = on ? __ldg(a.MT + (int64_t)r * P + j) : 0.0;
      mt_row = r;
    }
    const long long f = __double2ll_rn(__dmul_rn(val, mt) * sc);
    if (f) fix_add_split(tlo, thi, (col - cbase) * 32 + lane, (uint32_t)f, (uint32_t)((unsigned long long)f >> 32));
  });
  __syncthreads();
  long long* t = a.tiles + ((((int64_t)g * gridDim.y + chunk) * gridDim.z + range) * CW) * 32;
  for (uint32_t k = tid; k < CW * 32; k += blockDim.x)
    t[k] = (long long)(((unsigned long long)thi[k] << 32) | tlo[k]);
}

// out[j][c] (one batch: [p x m]) = sum over row groups of the tiles, fixed point -> f64.
__global__ void mc_left_reduce_kernel(const long long* tiles, int32_t groups, int32_t chunks, int32_t ranges,
                                      int32_t cw, int32_t p, int32_t n_cols, const double* scale, double* out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // over p * n_cols, j-major
  if (k >= (int64_t)p * n_cols) return;
  const int32_t jj = (int32_t)(k / n_cols), c = (int32_t)(k % n_cols);
  const int32_t chunk = jj >> 5, lane = jj & 31, range = c / cw, cc = c % cw;
  unsigned long long s = 0;
  for (int32_t g = 0; g < groups; ++g)
    s += (unsigned long long)tiles[((((int64_t)g * chunks + chunk) * ranges + range) * cw + cc) * 32 + lane];
  out[k] = (double)(long long)s / scale[jj];
}

}  // namespace toc

// ------------------------------------------------------------------------------------------
namespace {

int mc_attr(cudaDeviceAttr attr, int fallback) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, attr, dev) != cudaSuccess || v <= 0)
    return fallback;
  return v;
}

}  // namespace

extern "C" int toc_matcache_offsets(const TocBlockMeta* h_meta, int64_t n_blocks, int64_t* h_cache_off) {
  if (!h_meta || n_blocks < 0 || !h_cache_off) return TOC_E_ARG;
  int64_t o = 0;
  for (int64_t b = 0; b < n_blocks; ++b) {
    h_cache_off[b] = o;
    o += toc::mc_layout(h_meta[b]).total;
  }
  h_cache_off[n_blocks] = o;
  return TOC_OK;
}

extern "C" int toc_matcache_build(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                  int64_t n_blocks, const TocPlan* plan, const int64_t* d_cache_off, uint8_t* d_cache,
                                  void* d_scratch, void* stream) {
  if (!plan || n_blocks < 0 || !d_cache || !d_cache_off) return TOC_E_ARG;
  if (plan->global_tables && !d_scratch) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  toc::McArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.n_blocks = n_blocks;
  a.scratch = (uint8_t*)d_scratch;
  a.cache = d_cache;
  a.cache_off = d_cache_off;
  a.batch_smem_budget = plan->smem_bytes - (int32_t)toc::kFixedBytes;
  a.slab_bytes = plan->global_tables ? plan->scratch_bytes / plan->ctas : 0;
  void* fn = plan->wide ? (void*)toc::mc_build_kernel<true> : (void*)toc::mc_build_kernel<false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan->smem_bytes) != cudaSuccess)
    return TOC_E_CUDA;
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3(plan->ctas), dim3(plan->threads), args, plan->smem_bytes, (cudaStream_t)stream) ==
                 cudaSuccess
             ? TOC_OK
             : TOC_E_CUDA;
}

extern "C" int toc_matcache_right(const uint8_t* d_cache, const int64_t* d_cache_off, const int64_t* d_row_base,
                                  int64_t n_blocks, int64_t n_rows, int32_t p, const double* d_M, double* d_out,
                                  void* stream) {
  if (n_blocks < 0 || n_rows < 0 || p < 1 || !d_cache || !d_cache_off || !d_row_base || !d_M || !d_out)
    return TOC_E_ARG;
  if (n_blocks == 0 || n_rows == 0) return TOC_OK;
  toc::McRightArgs a{d_cache, d_cache_off, d_row_base, n_blocks, p, d_M, d_out};
  toc::mc_right_kernel<<<dim3((unsigned)n_rows, (unsigned)((p + 31) / 32)), 256, 0, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_matcache_left_scratch(const TocBlockMeta* h_meta, int32_t p, int32_t n_cols, int64_t* bytes) {
  if (!h_meta || p < 1 || n_cols < 1 || !bytes) return TOC_E_ARG;
  const int optin = mc_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448);
  const int32_t cw = std::min<int32_t>(n_cols, (optin - 1024) / 256);
  const int32_t ranges = (n_cols + cw - 1) / cw, chunks = (p + 31) / 32;
  const int sms = mc_attr(cudaDevAttrMultiProcessorCount, 148);
  const int32_t groups = std::max<int32_t>(1, std::min<int32_t>((int32_t)h_meta->n_rows,
                                                                (sms + chunks * ranges - 1) / (chunks * ranges)));
  *bytes = 8ll * groups * chunks * ranges * cw * 32 + 8ll * p;
  return TOC_OK;
}

// One batch: out [p x m] = M_b . A_b with M given transposed (M^T rows of the batch, [n x p]).
extern "C" int toc_matcache_left(const uint8_t* d_entry, const TocBlockMeta* h_meta, int32_t p, int32_t n_cols,
                                 const double* d_MT, double* d_out, void* d_scratch, int64_t scratch_bytes,
                                 void* stream) {
  if (!d_entry || !h_meta || p < 1 || n_cols < 1 || !d_MT || !d_out || !d_scratch) return TOC_E_ARG;
  int64_t need = 0;
  toc_matcache_left_scratch(h_meta, p, n_cols, &need);
  if (scratch_bytes < need) return TOC_E_ARG;
  const int optin = mc_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448);
  const int32_t cw = std::min<int32_t>(n_cols, (optin - 1024) / 256);
  const int32_t ranges = (n_cols + cw - 1) / cw, chunks = (p + 31) / 32;
  const int sms = mc_attr(cudaDevAttrMultiProcessorCount, 148);
  const int32_t groups = std::max<int32_t>(1, std::min<int32_t>((int32_t)h_meta->n_rows,
                                                                (sms + chunks * ranges - 1) / (chunks * ranges)));
  double* scale = reinterpret_cast<double*>(d_scratch);
  long long* tiles = reinterpret_cast<long long*>(reinterpret_cast<uint8_t*>(d_scratch) + 8ll * p);
  cudaStream_t s = (cudaStream_t)stream;
  toc::mc_scale_kernel<<<(p + 127) / 128, 128, 0, s>>>(d_MT, (int32_t)h_meta->n_rows, p, d_entry, scale);
  toc::McLeftArgs a{d_entry, p, n_cols, groups, cw, d_MT, scale, tiles};
  const int smem = cw * 32 * 8;
  if (cudaFuncSetAttribute(toc::mc_left_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return TOC_E_CUDA;
  toc::mc_left_kernel<<<dim3(groups, chunks, ranges), 1024, smem, s>>>(a);
  const int64_t total = (int64_t)p * n_cols;
  toc::mc_left_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(tiles, groups, chunks, ranges, cw, p,
                                                                               n_cols, scale, d_out);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}
