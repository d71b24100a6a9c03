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
//   pstart   u32[C + 1]: each code's first pair, counted from the batch's first pair
// A row is expanded in shared memory by threads walking different codes' chains (each chain once,
// not once per output lane), each into its slot range, then the dense part runs with lanes across
// 32 columns of M:
//   A.M   CTA per output row: expand, then warps take 32-column chunks of M and sum value *
//         M[col, j] over the row's pairs in row order.  No atomics.
//   M.A   CTA (row group, chunk): rows one at a time -- expand, then warps split the row's pairs
//         and add value * M^T[r, j] into a shared (m x 32) fp64 tile.  A row's pairs have distinct
//         columns, so within a row no two threads touch one entry: plain adds in row order, no
//         atomics; the row groups' tiles are summed in group order by a second kernel.
#include <algorithm>

#include "toc_batch.cuh"

namespace toc {

struct NodeRec {
  uint32_t par, col;
  double val;
};

struct McLayout {
  uint32_t off_rowoff, off_codes, off_pstart, off_nodes, total;
};

constexpr uint32_t kMcHeader = 32;

TOC_HD McLayout mc_layout(const TocBlockMeta& m) {
  McLayout L;
  uint32_t o = kMcHeader;
  L.off_rowoff = o;
  o += align16(4u * (m.n_rows + 1));
  L.off_codes = o;
  o += align16(4u * m.n_codes);
  L.off_pstart = o;  // first pair of each code, counted from the batch's first pair (C + 1)
  o += align16(4u * (m.n_codes + 1));
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
    __syncthreads();
    {  // pstart: exclusive prefix of code lengths over the batch, in chunks of the block width
      uint32_t* pstart = reinterpret_cast<uint32_t*>(e + L.off_pstart);
      uint32_t carry = 0;
      const uint32_t lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
      for (uint32_t base = 0; base < m.n_codes; base += nth) {
        const uint32_t j = base + tid;
        uint32_t len = 0;
        if (j < m.n_codes) {
          uint32_t x = codes[j];
          len = 1;
          while (x > B.nI) {
            x = B.pk.par(x - 1 - B.nI);
            ++len;
          }
        }
        const uint32_t xs = warp_excl_scan(len, lane);
        if (lane == 31) s_warp[warp] = xs + len;
        __syncthreads();
        if (warp == 0) {
          const uint32_t t = lane < nwarps ? s_warp[lane] : 0u;
          const uint32_t ex = warp_excl_scan(t, lane);
          if (lane < nwarps) s_warp[lane] = ex;
          if (lane == 31) s_warp[32] = ex + t;
        }
        __syncthreads();
        if (j < m.n_codes) pstart[j] = carry + s_warp[warp] + xs;
        carry += s_warp[32];
        __syncthreads();
      }
      if (tid == 0) pstart[m.n_codes] = carry;
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

// ---- the MLP step cache (toc_mlp.cu decodes each step's batch from it) -----------------------
// The decode tree of a batch in 4 bytes per node, read together with the TOC1 block's own packed
// code stream (the cache does not repeat the codes, a quarter of the node records above):
//   header   u32[16]: n_rows, n_codes, T, |I|, n_cols, n_uniques, off_codes (in the block),
//            w_codes, off_rowoff, off_pairs, off_nodes, off_uniq                             64 B
//   rowoff   u32[n + 1]
//   pairs    u32[|I| + 1]: column | value ref << 16 of pair id i (i >= 1)
//   nodes    u32[T]: derived node x: parent | key << 17 (codec.py:243-251: its parent is the code
//            at the position that created it, its key the first pair of the next code); 0 for pairs
//   uniq     f64[n_uniques]: the value index
// Batches whose ids do not fit (T > 2^17 nodes, 2^15 pairs, more than 2^16 columns or values) are
// refused (toc_mlpcache_offsets returns TOC_E_ARG; the caller keeps the node-record cache).
struct DcLayout {
  uint32_t off_rowoff, off_pairs, off_nodes, off_uniq, total;
};

constexpr uint32_t kDcHeader = 64;

TOC_HD bool dc_fits(const TocBlockMeta& m) {
  return 1ull + m.n_pairs + m.n_derived <= (1ull << 17) && m.n_pairs < (1u << 15) && m.n_cols <= 65536u &&
         m.n_uniques <= 65536u;
}

TOC_HD DcLayout dc_layout(const TocBlockMeta& m) {
  DcLayout L;
  uint32_t o = kDcHeader;
  L.off_rowoff = o;
  o += align16(4u * (m.n_rows + 1));
  L.off_pairs = o;
  o += align16(4u * (m.n_pairs + 1));
  L.off_nodes = o;
  o += align16(4u * (1u + m.n_pairs + m.n_derived));
  L.off_uniq = o;
  o += align16(8u * m.n_uniques);
  L.total = o;
  return L;
}

template <bool kWide>
__global__ void __launch_bounds__(1024, 1) dc_build_kernel(McArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  uint8_t* p = smem + kFixedBytes;
  uint8_t* slab = a.scratch ? a.scratch + (int64_t)blockIdx.x * a.slab_bytes : nullptr;
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const TocBlockMeta m = a.meta[b];
    if (m.status != TOC_OK || m.corrupt || !dc_fits(m)) continue;
    uint8_t* tables = batch_layout<kWide>(m).total <= (uint32_t)a.batch_smem_budget ? p : slab;
    __syncthreads();
    Batch<kWide> B;
    const uint8_t* blk = a.arena + a.block_off[b];
    B.init(blk, m, tables);
    B.load_index(s_warp);
    B.build_nodes();
    __syncthreads();
    B.resolve_keys();
    __syncthreads();
    const DcLayout L = dc_layout(m);
    uint8_t* e = a.cache + a.cache_off[b];
    uint32_t* rowoff = reinterpret_cast<uint32_t*>(e + L.off_rowoff);
    uint32_t* pairs = reinterpret_cast<uint32_t*>(e + L.off_pairs);
    uint32_t* nodes = reinterpret_cast<uint32_t*>(e + L.off_nodes);
    double* uniq = reinterpret_cast<double*>(e + L.off_uniq);
    for (uint32_t r = tid; r <= B.n; r += nth) rowoff[r] = B.rowoff[r];
    for (uint32_t i = tid; i < B.nI; i += nth)
      pairs[i + 1] = ld_packed(blk + m.off_cols, i, m.w_cols) | (ld_packed(blk + m.off_refs, i, m.w_refs) << 16);
    if (tid == 0) pairs[0] = 0u;
    for (uint32_t i = tid; i < m.n_uniques; i += nth) uniq[i] = B.uniq[i];
    const uint32_t T = 1u + B.nI + m.n_derived;
    for (uint32_t x = tid; x < T; x += nth) {
      uint32_t w = 0u;
      if (x > B.nI) {
        uint32_t par, key;
        B.pk.get(x - 1 - B.nI, par, key);
        w = par | (key << 17);
      }
      nodes[x] = w;
    }
    if (tid == 0) {
      uint32_t* h = reinterpret_cast<uint32_t*>(e);
      h[0] = B.n;
      h[1] = m.n_codes;
      h[2] = T;
      h[3] = B.nI;
      h[4] = m.n_cols;
      h[5] = m.n_uniques;
      h[6] = m.off_codes;
      h[7] = m.w_codes;
      h[8] = L.off_rowoff;
      h[9] = L.off_pairs;
      h[10] = L.off_nodes;
      h[11] = L.off_uniq;
      for (int k = 12; k < 16; ++k) h[k] = 0u;
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

// Expand codes [j0, j1) (one row) into shared (column, value) arrays in row order: threads take
// different codes and walk their chains (last pair first) into the code's slot range, given by
// the cached pair offsets.  Returns the row's pair count.
TOC_D uint32_t expand_row(const uint32_t* codes, const uint32_t* pstart, const NodeRec* nodes, uint32_t j0,
                          uint32_t j1, uint32_t* s_col, double* s_val) {
  const uint32_t base = __ldg(pstart + j0);
  for (uint32_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    uint32_t x = __ldg(codes + j);
    uint32_t e = __ldg(pstart + j + 1) - base;
    while (x) {
      const NodeRec n = ld_node(nodes, x);
      --e;
      s_col[e] = n.col;
      s_val[e] = n.val;
      x = n.par;
    }
  }
  return __ldg(pstart + j1) - base;
}

struct McEntry {
  const uint32_t* rowoff;
  const uint32_t* codes;
  const uint32_t* pstart;
  const NodeRec* nodes;
  uint32_t n_rows;
};

TOC_D McEntry mc_entry(const uint8_t* e) {
  const uint32_t* h = reinterpret_cast<const uint32_t*>(e);
  TocBlockMeta m{};
  m.n_rows = h[0];
  m.n_codes = h[1];
  m.n_pairs = h[3];
  m.n_derived = h[2] - 1 - h[3];
  const McLayout L = mc_layout(m);
  McEntry E;
  E.rowoff = reinterpret_cast<const uint32_t*>(e + L.off_rowoff);
  E.codes = reinterpret_cast<const uint32_t*>(e + L.off_codes);
  E.pstart = reinterpret_cast<const uint32_t*>(e + L.off_pstart);
  E.nodes = reinterpret_cast<const NodeRec*>(e + L.off_nodes);
  E.n_rows = m.n_rows;
  return E;
}

struct McRightArgs {
  const uint8_t* cache;
  const int64_t* cache_off;
  const int64_t* row_base;  // first output row of each batch
  int64_t n_blocks;
  int32_t p, n_cols;
  const double* M;  // [m x p]
  double* out;      // [rows x p]
};

// CTA per output row: expand the row in shared memory, then each warp takes 32-column chunks of
// M and sums value * M[col, j] over the row's pairs in row order.  No atomics.  (Measured: four
// split accumulators or pair slices over more warps are slower, 80 vs 52 us at config 5.)
constexpr uint32_t kRightThreads = 256;

__global__ void __launch_bounds__(kRightThreads) mc_right_kernel(McRightArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* s_val = reinterpret_cast<double*>(smem);
  uint32_t* s_col = reinterpret_cast<uint32_t*>(smem + 8u * (uint32_t)a.n_cols);
  const int64_t row = blockIdx.x;
  int64_t lo = 0, hi = a.n_blocks - 1;  // batch of this row: last b with row_base[b] <= row
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (a.row_base[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  const McEntry E = mc_entry(a.cache + a.cache_off[lo]);
  const uint32_t r = (uint32_t)(row - a.row_base[lo]);
  const uint32_t nnz = expand_row(E.codes, E.pstart, E.nodes, __ldg(E.rowoff + r), __ldg(E.rowoff + r + 1), s_col, s_val);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t P = (uint32_t)a.p;
  for (uint32_t chunk = warp; chunk * 32 < P; chunk += nwarps) {
    const uint32_t j = chunk * 32 + lane;
    if (j >= P) continue;
    double acc = 0.0;
#pragma unroll 4
    for (uint32_t q = 0; q < nnz; ++q) acc = __dadd_rn(acc, __dmul_rn(s_val[q], __ldg(a.M + (int64_t)s_col[q] * P + j)));
    a.out[row * (int64_t)P + j] = acc;
  }
}

struct McLeftArgs {
  const uint8_t* entry;  // one batch's cache entry
  int32_t p, n_cols;
  int32_t groups;        // row groups
  const double* MT;      // M^T rows of this batch: [n x p]
  double* tiles;         // [groups][chunks][n_cols][32]
};

// CTA (row group, 32-column chunk of M^T): rows one at a time -- expand, then warps split the
// row's pairs and add value * M^T[r, j] into a shared (n_cols x 32) fp64 tile.  A row's pairs
// have distinct columns, so no two threads touch one tile entry within a row and rows are
// separated by barriers: plain adds in row order, deterministic, no atomics.
__global__ void __launch_bounds__(512, 1) mc_left_kernel(McLeftArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t ncol = (uint32_t)a.n_cols;
  double* tile = reinterpret_cast<double*>(smem);       // [ncol][32]
  double* s_val = tile + (size_t)ncol * 32;             // [ncol]
  uint32_t* s_col = reinterpret_cast<uint32_t*>(s_val + ncol);
  const McEntry E = mc_entry(a.entry);
  const uint32_t g = blockIdx.x, chunk = blockIdx.y, G = (uint32_t)a.groups, n = E.n_rows;
  const uint32_t r0 = (uint32_t)(((uint64_t)n * g) / G), r1 = (uint32_t)(((uint64_t)n * (g + 1)) / G);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (uint32_t k = tid; k < ncol * 32; k += blockDim.x) tile[k] = 0.0;
  const uint32_t P = (uint32_t)a.p, j = chunk * 32 + lane;
  const bool on = j < P;
  for (uint32_t r = r0; r < r1; ++r) {
    __syncthreads();  // the previous row's adds are done before its buffer is overwritten
    const uint32_t nnz = expand_row(E.codes, E.pstart, E.nodes, __ldg(E.rowoff + r), __ldg(E.rowoff + r + 1), s_col, s_val);
    const double mt = on ? __ldg(a.MT + (int64_t)r * P + j) : 0.0;
    __syncthreads();
#pragma unroll 4
    for (uint32_t q = warp; q < nnz; q += nwarps) {
      double* t = tile + (size_t)s_col[q] * 32 + lane;
      *t = __dadd_rn(*t, __dmul_rn(s_val[q], mt));
    }
  }
  __syncthreads();
  double* out = a.tiles + ((int64_t)g * gridDim.y + chunk) * (int64_t)ncol * 32;
  for (uint32_t k = tid; k < ncol * 32; k += blockDim.x) out[k] = tile[k];
}

// out[j][c] (one batch: [p x m]) = sum over row groups of the tiles, in group order.
__global__ void mc_left_reduce_kernel(const double* tiles, int32_t groups, int32_t chunks, int32_t p, int32_t n_cols,
                                      double* out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // over p * n_cols, j-major
  if (k >= (int64_t)p * n_cols) return;
  const int32_t jj = (int32_t)(k / n_cols), c = (int32_t)(k % n_cols);
  const int32_t chunk = jj >> 5, lane = jj & 31;
  double s = 0.0;
  for (int32_t g = 0; g < groups; ++g) s += tiles[(((int64_t)g * chunks + chunk) * n_cols + c) * 32 + lane];
  out[k] = s;
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

extern "C" int toc_mlpcache_offsets(const TocBlockMeta* h_meta, int64_t n_blocks, int64_t* h_cache_off) {
  if (!h_meta || n_blocks < 0 || !h_cache_off) return TOC_E_ARG;
  int64_t o = 0;
  for (int64_t b = 0; b < n_blocks; ++b) {
    if (!toc::dc_fits(h_meta[b])) return TOC_E_ARG;
    h_cache_off[b] = o;
    o += toc::dc_layout(h_meta[b]).total;
  }
  h_cache_off[n_blocks] = o;
  return TOC_OK;
}

extern "C" int toc_mlpcache_build(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
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
  void* fn = plan->wide ? (void*)toc::dc_build_kernel<true> : (void*)toc::dc_build_kernel<false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan->smem_bytes) != cudaSuccess)
    return TOC_E_CUDA;
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3(plan->ctas), dim3(plan->threads), args, plan->smem_bytes, (cudaStream_t)stream) ==
                 cudaSuccess
             ? TOC_OK
             : TOC_E_CUDA;
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
                                  int64_t n_blocks, int64_t n_rows, int32_t n_cols, int32_t p, const double* d_M,
                                  double* d_out, void* stream) {
  if (n_blocks < 0 || n_rows < 0 || p < 1 || n_cols < 1 || !d_cache || !d_cache_off || !d_row_base || !d_M || !d_out)
    return TOC_E_ARG;
  if (n_blocks == 0 || n_rows == 0) return TOC_OK;
  const int smem = 12 * n_cols;  // one row's (value, column) pairs: at most n_cols
  if (smem > mc_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448)) return TOC_E_ARG;
  if (cudaFuncSetAttribute(toc::mc_right_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return TOC_E_CUDA;
  toc::McRightArgs a{d_cache, d_cache_off, d_row_base, n_blocks, p, n_cols, d_M, d_out};
  toc::mc_right_kernel<<<(unsigned)n_rows, toc::kRightThreads, smem, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

namespace {
int32_t left_groups(const TocBlockMeta* h_meta, int32_t p) {
  const int sms = mc_attr(cudaDevAttrMultiProcessorCount, 148);
  const int32_t chunks = (p + 31) / 32;
  return std::max<int32_t>(1, std::min<int32_t>((int32_t)h_meta->n_rows, (sms + chunks - 1) / chunks));
}
}  // namespace

extern "C" int toc_matcache_left_scratch(const TocBlockMeta* h_meta, int32_t p, int32_t n_cols, int64_t* bytes) {
  if (!h_meta || p < 1 || n_cols < 1 || !bytes) return TOC_E_ARG;
  *bytes = 8ll * left_groups(h_meta, p) * ((p + 31) / 32) * n_cols * 32;
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
  const int smem = 8 * 32 * n_cols + 12 * n_cols;  // tile + one row's pairs
  if (smem > mc_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448)) return TOC_E_ARG;
  const int32_t groups = left_groups(h_meta, p), chunks = (p + 31) / 32;
  cudaStream_t s = (cudaStream_t)stream;
  toc::McLeftArgs a{d_entry, p, n_cols, groups, d_MT, reinterpret_cast<double*>(d_scratch)};
  if (cudaFuncSetAttribute(toc::mc_left_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return TOC_E_CUDA;
  toc::mc_left_kernel<<<dim3(groups, chunks), 512, smem, s>>>(a);
  const int64_t total = (int64_t)p * n_cols;
  toc::mc_left_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(reinterpret_cast<double*>(d_scratch),
                                                                               groups, chunks, p, n_cols, d_out);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}
