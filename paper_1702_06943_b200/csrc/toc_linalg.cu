// toc_linalg.cu -- A.v and v^T.A directly on TOC1 blocks resident in HBM (sm_100a).
//
// Reference: kernels.py:115-142 (matvec, Algorithm 5) and kernels.py:145-174 (vecmat,
// Algorithm 6).  A persistent grid walks the arena, one CTA per mini-batch at a time, the next
// block prefetched into L2; the per-batch machinery (node tables rebuilt from the block in
// shared memory, chain walks, fixed-point v^T.A) is in toc_batch.cuh.  DESIGN.md section 4.1.
#include <atomic>
#include <functional>
#include <mutex>

#include "toc_batch.cuh"

namespace toc {

struct LinalgArgs {
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  const int64_t* row_base;
  int64_t n_blocks;
  int32_t kind;
  int32_t n_cols;
  int32_t batch_smem_budget;  // bytes of dynamic smem available for one batch's tables
  int64_t slab_bytes;         // global fallback slab per CTA
  const double* v;
  double* R;
  const double* u;
  double* O;
  uint8_t* scratch;
  const uint8_t* trees;     // optional device tree cache (toc_build_trees); NULL: rebuild per call
  const int64_t* tree_off;  // byte offset of batch b's tree prefix in `trees`
  int32_t use_splits;       // cached pair-balanced lane splits (tuning knob)
  int32_t depth_order;      // tree cache build: order each lane range's codes by depth (tuning knob)
};

// One batch of the sweep.  `tables` points either into shared memory or into this CTA's slab.
template <bool kWide, bool kVecSmem, bool kCached>
__device__ __forceinline__ void process_batch(const LinalgArgs& a, int64_t b, const TocBlockMeta& m,
                                              uint8_t* tables, bool in_smem, const double* vec_s, uint32_t* acc_s,
                                              uint32_t* s_warp, double* s_red, uint64_t* mbar, uint32_t& phase) {
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  const bool do_mv = a.kind & TOC_MATVEC, do_vm = a.kind & TOC_VECMAT;
  const int64_t row_base = a.row_base[b];
  const int32_t ncol = a.n_cols;
  const uint8_t* blk = a.arena + a.block_off[b];
  Batch<kWide> B;
  constexpr bool cached = kCached;
  using Rec = typename PairRec<kWide>::T;
  const Rec* irec = nullptr;
  const Rec* prec = nullptr;
  const uint2* segs = nullptr;
  uint32_t n_segs = kNoSegs;
  double vmax_c = 0.0;
  if (cached) {
    // Tree prefix from the device cache: one bulk copy into shared memory (or read in place
    // from global memory when the batch's tables do not fit), overlapped with the value work.
    uint8_t* tree = const_cast<uint8_t*>(a.trees + a.tree_off[b]);
    const CacheLayout CL = cache_layout<kWide>(m);
    irec = reinterpret_cast<const Rec*>(tree + CL.off_irec);
    prec = reinterpret_cast<const Rec*>(tree + CL.off_prec);
    segs = reinterpret_cast<const uint2*>(tree + CL.off_segs);
    n_segs = __ldg(reinterpret_cast<const uint32_t*>(tree + CL.off_info));
    vmax_c = __ldg(reinterpret_cast<const double*>(tree + CL.off_info + 8));
    B.init(blk, m, tables, in_smem ? nullptr : tree);
    if (a.use_splits && __ldg(reinterpret_cast<const uint32_t*>(tree + CL.off_info) + 1) == B.S)
      B.splits = reinterpret_cast<const uint16_t*>(tree + CL.off_splits);
    if (in_smem && tid == 0) bulk_load(tables, tree, CL.tree, mbar);
    B.load_values();
  } else {
    B.init(blk, m, tables);
  }
  if (do_vm && kVecSmem)
    for (int32_t c = tid; c < 2 * ncol; c += nth) acc_s[c] = 0u;
  if (!cached) B.load_index(s_warp);
  double g_scale = 1.0, o_scale = 1.0;
  bool g_f64 = false;  // fixed point too coarse for this batch: accumulate in fp64
  if (do_vm && !cached) {  // a-priori bounds of every partial sum (see fix_add): sum |u| and max |value|
    double su = 0.0;
    for (uint32_t r = tid; r < B.n; r += nth) su += fabs(a.u[row_base + r]);
    su = block_sum(su, s_red);
    const double vmax = block_max_d(B.vmax, s_red);
    g_scale = fix_scale(su);
    o_scale = fix_scale(su * vmax);
    g_f64 = fixed_point_too_coarse(B.n, vmax, 1.0 / g_scale + 1.0 / (o_scale * vmax));
  }
  if (cached) {
    if (do_vm) {  // sum |u| as warp partials, read after the barrier below (no extra barrier)
      double su = 0.0;
      for (uint32_t r = tid; r < B.n; r += nth) su += fabs(a.u[row_base + r]);
      su = warp_sum(su);
      if ((tid & 31) == 0) s_red[tid >> 5] = su;
    }
    __syncthreads();  // uniq and the partials complete
    if (do_vm) {
      double su = 0.0;
      for (uint32_t w = 0; w < (nth >> 5); ++w) su += s_red[w];
      g_scale = n_segs != kNoSegs ? limb_scale(su, limb_bits(B.n)) : fix_scale(su);
      const double vmax = vmax_c;
      if (n_segs == kNoSegs) o_scale = fix_scale(su * vmax);  // fixed-point scatter only
      g_f64 = fixed_point_too_coarse(B.n, vmax, 1.0 / g_scale + (n_segs == kNoSegs ? 1.0 / (o_scale * vmax) : 0.0));
    }
    if (do_mv) B.compute_p1_records(irec, kVecSmem ? vec_s : a.v);
    else B.zero_tab();
    if (in_smem) {
      mbar_wait(mbar, phase);
      phase ^= 1u;
    }
    __syncthreads();
  } else {
    B.build_nodes();
    if (do_mv) B.template compute_p1<false>(kVecSmem ? vec_s : a.v);
    else B.zero_tab();
    __syncthreads();
    B.resolve_keys();
    __syncthreads();
  }
  if (do_mv) B.matvec_rows([&](uint32_t r, double s) { a.R[row_base + r] = s; });
  if (do_vm) {
    if (do_mv) {
      __syncthreads();
      B.zero_tab();
      __syncthreads();
    }
    if (n_segs != kNoSegs) {
      // split-word G, then out[col] as a fixed-order segmented sum over the column-sorted pairs
      const uint32_t L = g_f64 ? kGF64 : limb_bits(B.n);
      if (g_f64)
        B.vecmat_rows_f64([&](uint32_t r) { return a.u[row_base + r]; });
      else
        B.vecmat_rows_limbs([&](uint32_t r) { return a.u[row_base + r]; }, g_scale, L);
      __syncthreads();
      double* o = a.O + b * (int64_t)ncol;
      if (kVecSmem) {
        double* os = reinterpret_cast<double*>(acc_s);  // zeroed above: absent columns stay 0
        B.column_sums(prec, segs, n_segs, 1.0 / g_scale, [&](uint32_t c, double x) { os[c] = x; }, L);
        __syncthreads();
        for (int32_t c = tid; c < ncol; c += nth) o[c] = os[c];
      } else {  // O zeroed by the host
        B.column_sums(prec, segs, n_segs, 1.0 / g_scale, [&](uint32_t c, double x) { o[c] = x; }, L);
      }
      return;
    }
    double* o = a.O + b * (int64_t)ncol;
    if (g_f64) {  // fp64 G and out (O zeroed by the host when it is not staged in shared memory)
      B.vecmat_rows_f64([&](uint32_t r) { return a.u[row_base + r]; });
      __syncthreads();
      double* os = kVecSmem ? reinterpret_cast<double*>(acc_s) : o;
      B.scatter_columns_f64(os);
      __syncthreads();
      if (kVecSmem)
        for (int32_t c = tid; c < ncol; c += nth) o[c] = os[c];
      return;
    }
    B.vecmat_rows([&](uint32_t r) { return a.u[row_base + r]; }, g_scale);
    __syncthreads();
    uint32_t* out = kVecSmem ? acc_s : reinterpret_cast<uint32_t*>(a.O + b * (int64_t)ncol);
    B.scatter_columns(out, 1.0 / g_scale, o_scale);
    __syncthreads();
    const double o_inv = 1.0 / o_scale;
    if (kVecSmem) {
      for (int32_t c = tid; c < ncol; c += nth) o[c] = fix_value(acc_s[2 * c], acc_s[2 * c + 1], o_inv);
    } else {
      uint32_t* ow = reinterpret_cast<uint32_t*>(o);
      for (int32_t c = tid; c < ncol; c += nth) o[c] = fix_value(__ldcg(ow + 2 * c), __ldcg(ow + 2 * c + 1), o_inv);
    }
  }
}

template <bool kWide, bool kVecSmem, bool kCached>
__global__ void __launch_bounds__(1024, 1) linalg_kernel(LinalgArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);  // 33 words
  uint8_t* p = smem + kFixedBytes;
  double* s_red = reinterpret_cast<double*>(smem + 160);  // 33 doubles
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 448);  // tree-cache bulk copies
  uint32_t phase = 0;
  if (threadIdx.x == 0) mbar_init(mbar, 1);
  __syncthreads();
  double* vec_s = nullptr;
  uint32_t* acc_s = nullptr;
  if (kVecSmem) {
    if (a.kind & TOC_MATVEC) {
      vec_s = reinterpret_cast<double*>(p);
      p += align16(8u * a.n_cols);
    }
    if (a.kind & TOC_VECMAT) {
      acc_s = reinterpret_cast<uint32_t*>(p);
      p += align16(8u * a.n_cols);
    }
    if (vec_s)
      for (int32_t c = threadIdx.x; c < a.n_cols; c += blockDim.x) vec_s[c] = a.v[c];
  }
  uint8_t* slab = a.scratch ? a.scratch + (int64_t)blockIdx.x * a.slab_bytes : nullptr;
  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const TocBlockMeta m = a.meta[b];
    if (m.status != TOC_OK || m.corrupt) continue;  // host refuses such arenas up front
    const uint32_t need = batch_layout<kWide>(m).total;
    if (threadIdx.x == 0 && b + gridDim.x < a.n_blocks) {  // pull what the next batch reads into L2
      const int64_t bn = b + gridDim.x;
      const TocBlockMeta& mn = a.meta[bn];
      const uint8_t* nb = a.arena + a.block_off[bn];
      // block-only: the whole block; tree cache: the block's value index (columns, refs and
      // codes are in the cache entry) plus the cache entry itself
      const uint32_t bytes = kCached ? align16(mn.off_uniques + 8u * mn.n_uniques)
                                     : align16(mn.off_offsets + (mn.n_rows + 1u) * mn.w_offsets);
      if (mn.status == TOC_OK && bytes > 0) {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nb), "r"(bytes) : "memory");
        if (kCached)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.trees + a.tree_off[bn]),
                       "r"(cache_layout<kWide>(mn).total)
                       : "memory");
      }
    }
    __syncthreads();
    if (need <= (uint32_t)a.batch_smem_budget)
      process_batch<kWide, kVecSmem, kCached>(a, b, m, p, true, vec_s, acc_s, s_warp, s_red, mbar, phase);
    else
      process_batch<kWide, kVecSmem, kCached>(a, b, m, slab, false, vec_s, acc_s, s_warp, s_red, mbar, phase);
  }
}

// Device tree cache: rebuild each batch's tree prefix (row offsets, derived-node bases, final
// codes, node table with resolved keys) once and store it, byte for byte as it sits in shared
// memory, at trees + tree_off[b].
template <bool kWide>
__global__ void __launch_bounds__(1024, 1) build_trees_kernel(LinalgArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  uint8_t* p = smem + kFixedBytes;
  uint8_t* slab = a.scratch ? a.scratch + (int64_t)blockIdx.x * a.slab_bytes : nullptr;
  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const TocBlockMeta m = a.meta[b];
    if (m.status != TOC_OK || m.corrupt) continue;
    const BatchLayout L = batch_layout<kWide>(m);
    uint8_t* tables = L.total <= (uint32_t)a.batch_smem_budget ? p : slab;
    __syncthreads();
    Batch<kWide> B;
    B.init(a.arena + a.block_off[b], m, tables);
    B.load_index(s_warp);
    B.build_nodes();
    __syncthreads();
    B.resolve_keys();
    __syncthreads();
    uint8_t* entry = const_cast<uint8_t*>(a.trees) + a.tree_off[b];
    const CacheLayout CL = cache_layout<kWide>(m);
    {  // max |value| of the value index (info[2..3]): the sweep's fixed-point accuracy check
      const double vmax = block_max_d(B.vmax, reinterpret_cast<double*>(smem + 160));
      if (threadIdx.x == 0) *reinterpret_cast<double*>(entry + CL.off_info + 8) = vmax;
    }
    {  // pair-balanced lane splits for kSplitThreads-thread CTAs (row offsets fit u16: rows <= n_cols)
      const uint32_t S = seg_lanes(m.n_rows, kSplitThreads);
      const bool ok = m.n_cols <= 65535u;
      if (ok) B.write_splits(reinterpret_cast<uint16_t*>(entry + CL.off_splits), S);
      if (threadIdx.x == 0) reinterpret_cast<uint32_t*>(entry + CL.off_info)[1] = ok ? S : 0u;
    }
    const uint4* src = reinterpret_cast<const uint4*>(tables);
    uint4* dst = reinterpret_cast<uint4*>(entry);
    // (scratch: the old positions in the entry's node-table region, the id map in its pair-record
    // regions -- both rewritten below)
    const bool relabel = !kWide && a.depth_order && m.n_cols <= 65535u && m.n_derived < 65536u &&
                         2u * m.n_derived <= CL.off_splits - CL.off_irec;
    if (!relabel) {
      for (uint32_t k = threadIdx.x; k < L.tree / 16u; k += blockDim.x) dst[k] = src[k];
    } else {
      // Depth order: within each lane range of every row, the positions are renumbered so that the
      // codes come deepest first (stable) -- the lanes of a warp then walk chains of similar length
      // in lockstep.  A renumbering of the row's derived ids: every reference (par fields, final
      // codes) is remapped, keys (pairs) are unchanged, so every walk computes the same products.
      const BatchLayout BL = batch_layout<false>(m);
      uint16_t* sig = reinterpret_cast<uint16_t*>(entry + BL.off_pk);  // new index -> old position
      const uint32_t S = seg_lanes(m.n_rows, kSplitThreads), nI = B.nI;
      const uint16_t* sp = reinterpret_cast<const uint16_t*>(entry + CL.off_splits);
      for (uint32_t r = threadIdx.x; r < B.n; r += blockDim.x) {
        const uint32_t lo = B.rowoff[r], hi = B.rowoff[r + 1], db = B.dbase[r];
        if (hi - lo < 2) continue;
        for (uint32_t s2 = 0; s2 < S; ++s2) {
          const uint32_t a0 = lo + __ldcg(sp + r * S + s2);
          uint32_t a1 = s2 + 1 < S ? lo + __ldcg(sp + r * S + s2 + 1) : hi;
          a1 = min(a1, hi - 1);  // the final code has no derived node: it stays last
          // insertion sort of the range's positions by code depth (descending), kept in sig
          for (uint32_t j = a0; j < a1; ++j) {
            uint32_t x = B.pk.par(db + (j - lo)), dj = 1;
            while (x > nI) {
              x = B.pk.par(x - 1 - nI);
              ++dj;
            }
            uint32_t k = j;
            while (k > a0) {  // sig[db + (k - 1 - lo)] holds the old position now at k - 1
              const uint32_t op = sig[db + (k - 1 - lo)];
              uint32_t y = B.pk.par(db + (op - lo)), dk = 1;
              while (y > nI) {
                y = B.pk.par(y - 1 - nI);
                ++dk;
              }
              if (dk >= dj) break;
              sig[db + (k - lo)] = (uint16_t)op;
              --k;
            }
            sig[db + (k - lo)] = (uint16_t)j;
          }
        }
      }
      __syncthreads();
      // sig[new index] = old position; invert into the id map, then write the relabelled prefix
      uint16_t* inv = reinterpret_cast<uint16_t*>(entry + CL.off_irec);  // old derived index -> new
      for (uint32_t r = threadIdx.x; r < B.n; r += blockDim.x) {
        const uint32_t lo = B.rowoff[r], hi = B.rowoff[r + 1], db = B.dbase[r];
        for (uint32_t j = lo; j + 1 < hi; ++j) inv[db + (__ldcg(sig + db + (j - lo)) - lo)] = (uint16_t)(db + (j - lo));
      }
      __syncthreads();
      auto map = [&](uint32_t x) -> uint32_t { return x <= nI ? x : nI + 1u + __ldcg(inv + (x - 1 - nI)); };
      uint32_t* e32 = reinterpret_cast<uint32_t*>(entry);
      for (uint32_t k = threadIdx.x; k < BL.off_last / 4u; k += blockDim.x)  // row offsets, derived bases
        e32[k] = reinterpret_cast<const uint32_t*>(tables)[k];
      uint32_t* elast = reinterpret_cast<uint32_t*>(entry + BL.off_last);
      for (uint32_t r = threadIdx.x; r < B.n; r += blockDim.x)  // (empty rows have no final code)
        elast[r] = B.rowoff[r + 1] > B.rowoff[r] ? map(B.last[r]) : 0u;
      uint32_t* epk = reinterpret_cast<uint32_t*>(entry + BL.off_pk);
      for (uint32_t d = threadIdx.x; d < m.n_derived; d += blockDim.x) {
        uint32_t par, key;
        B.pk.get(d, par, key);
        epk[__ldcg(inv + d)] = (map(par) & 0xffffu) | (key << 16);
      }
    }
    // unpacked first-layer records, and the (column, pair)-sorted order with column segments
    const uint8_t* blk = a.arena + a.block_off[b];
    const uint32_t nI = m.n_pairs, tid = threadIdx.x, nth = blockDim.x;
    using R = PairRec<kWide>;
    typename R::T* irec = reinterpret_cast<typename R::T*>(entry + CL.off_irec);
    uint32_t npad = 1;
    while (npad < nI) npad <<= 1;
    const bool sort_here = tables == p && 8ull * npad <= (uint64_t)a.batch_smem_budget;
    __syncthreads();  // the tables have been copied out: their shared memory is free
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(p);
    for (uint32_t i = tid; i < npad; i += nth) {
      if (i < nI) {
        const uint32_t c = ld_packed(blk + m.off_cols, i, m.w_cols), r = ld_packed(blk + m.off_refs, i, m.w_refs);
        irec[i] = R::make(c, r);
        if (sort_here) keys[i] = ((unsigned long long)c << 32) | i;
      } else if (sort_here) {
        keys[i] = ~0ull;
      }
    }
    uint32_t* info = reinterpret_cast<uint32_t*>(entry + CL.off_info);
    if (!sort_here) {
      if (tid == 0) info[0] = kNoSegs;
      continue;
    }
    for (uint32_t k = 2; k <= npad; k <<= 1) {  // bitonic sort of (column, pair id): stable order
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        __syncthreads();
        for (uint32_t i = tid; i < npad; i += nth) {
          const uint32_t ij = i ^ j;
          if (ij > i) {
            const unsigned long long x = keys[i], z = keys[ij];
            if ((x > z) == ((i & k) == 0)) {
              keys[i] = z;
              keys[ij] = x;
            }
          }
        }
      }
    }
    __syncthreads();
    typename R::T* prec = reinterpret_cast<typename R::T*>(entry + CL.off_prec);
    for (uint32_t q = tid; q < nI; q += nth) {
      const uint32_t i = (uint32_t)keys[q];
      prec[q] = R::make(i, ld_packed(blk + m.off_refs, i, m.w_refs));
    }
    if (tid < 32) {  // column segments of the sorted order
      const uint32_t lane = tid;
      uint2* segs = reinterpret_cast<uint2*>(entry + CL.off_segs);
      uint32_t carry = 0;
      for (uint32_t base = 0; base < nI; base += 32) {
        const uint32_t q = base + lane;
        const uint32_t c = q < nI ? (uint32_t)(keys[q] >> 32) : 0u;
        const bool f = q < nI && (q == 0 || (uint32_t)(keys[q - 1] >> 32) != c);
        const uint32_t bal = __ballot_sync(0xffffffffu, f);
        if (f) segs[carry + __popc(bal & ((1u << lane) - 1u))] = make_uint2(q, c);
        carry += __popc(bal);
      }
      if (lane == 0) {
        segs[carry] = make_uint2(nI, 0u);
        info[0] = carry;
      }
    }
  }
}

}  // namespace toc

// ------------------------------------------------------------------------------------------
// Host side: planning and launch.
namespace {

// Process-wide tuning knobs (tools only; set before launching, read at planning / launch time).
std::atomic<int> g_use_splits{1};
std::atomic<int> g_depth_order{1};

struct DevProps {
  int sm_count = 0, smem_optin = 0, smem_per_sm = 0;
  int64_t l2 = 0;
};

constexpr int kMaxDevices = 64;

// The current device's properties, queried once per device (thread-safe).
DevProps dev_props() {
  static DevProps props[kMaxDevices];
  static std::once_flag once[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = -1;
  auto query = [](int d, DevProps& p) {
    if (d >= 0) {
      cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, d);
      cudaDeviceGetAttribute(&p.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
      cudaDeviceGetAttribute(&p.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, d);
      int l2 = 0;
      cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, d);
      p.l2 = l2;
    }
    if (p.sm_count <= 0) {  // no device visible (planning on a CPU host): B200 figures
      p.sm_count = 148;
      p.smem_optin = 232448;
      p.smem_per_sm = 233472;
      p.l2 = 126 << 20;
    }
  };
  if (dev < 0) {
    DevProps p;
    query(-1, p);
    return p;
  }
  std::call_once(once[dev], query, dev, std::ref(props[dev]));
  return props[dev];
}

// Raise the kernel's dynamic shared-memory limit to `bytes` on the current device (once per device
// and size; concurrent callers may both set it, which is harmless).
template <typename K>
cudaError_t ensure_smem(K* fn, int bytes, std::atomic<int>* configured) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (configured[dev].load() >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) {
    int cur = configured[dev].load();
    while (cur < bytes && !configured[dev].compare_exchange_weak(cur, bytes)) {
    }
  }
  return e;
}

template <bool W, bool V, bool C>
cudaError_t launch_mode(const toc::LinalgArgs& a, const TocPlan& plan, cudaStream_t s) {
  static std::atomic<int> configured[kMaxDevices];  // zero-initialised (static storage)
  if (const cudaError_t e = ensure_smem(toc::linalg_kernel<W, V, C>, plan.smem_bytes, configured); e != cudaSuccess)
    return e;
  toc::linalg_kernel<W, V, C><<<plan.ctas, plan.threads, plan.smem_bytes, s>>>(a);
  return cudaGetLastError();
}

template <bool W, bool V>
cudaError_t launch(const toc::LinalgArgs& a, const TocPlan& plan, cudaStream_t s) {
  return a.trees ? launch_mode<W, V, true>(a, plan, s) : launch_mode<W, V, false>(a, plan, s);
}

}  // namespace

extern "C" int toc_plan(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t kind, TocPlan* plan) {
  if (!plan || (n_blocks > 0 && !h_meta) || !(kind & (TOC_MATVEC | TOC_VECMAT))) return TOC_E_ARG;
  memset(plan, 0, sizeof(*plan));
  const DevProps d = dev_props();
  uint64_t max_T = 0;
  int32_t n_cols = n_blocks ? (int32_t)h_meta[0].n_cols : 0;
  for (int64_t b = 0; b < n_blocks; b++) {
    const TocBlockMeta& m = h_meta[b];
    if ((int32_t)m.n_cols != n_cols) return TOC_E_ARG;
    uint64_t T = 1ull + m.n_pairs + m.n_derived;
    if (T > max_T) max_T = T;
    if ((int32_t)m.n_rows > plan->max_rows) plan->max_rows = (int32_t)m.n_rows;
  }
  plan->wide = max_T > 65536ull || n_cols > 65536;  // narrow: every id fits u16 (PairRec)
  plan->n_cols = n_cols;
  uint32_t max_need = 0;
  for (int64_t b = 0; b < n_blocks; b++) {
    uint32_t need = plan->wide ? toc::batch_layout<true>(h_meta[b]).total
                               : toc::batch_layout<false>(h_meta[b]).total;
    if (need > max_need) max_need = need;
  }
  const int nvec = ((kind & TOC_MATVEC) ? 1 : 0) + ((kind & TOC_VECMAT) ? 1 : 0);
  const uint32_t vec_bytes = nvec * toc::align16(8u * (uint32_t)n_cols);
  plan->vec_in_smem = vec_bytes <= 64u * 1024u;
  const uint32_t fixed = toc::kFixedBytes + (plan->vec_in_smem ? vec_bytes : 0u);
  const uint32_t optin = (uint32_t)d.smem_optin;
  if (fixed + max_need <= optin) {
    plan->smem_bytes = (int32_t)(fixed + max_need);
    plan->global_tables = 0;
  } else {
    plan->smem_bytes = (int32_t)optin;
    plan->global_tables = 1;
  }
  int per_sm = (int)(((uint32_t)d.smem_per_sm) / ((uint32_t)plan->smem_bytes + 1024u));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  plan->threads = per_sm == 1 ? 1024 : 512;
  if (per_sm * plan->threads > 2048) per_sm = 2048 / plan->threads;
  int64_t ctas = (int64_t)d.sm_count * per_sm;
  if (ctas > n_blocks) ctas = n_blocks > 0 ? n_blocks : 1;
  plan->ctas = (int32_t)ctas;
  plan->scratch_bytes = plan->global_tables ? (int64_t)plan->ctas * toc::align16(max_need) : 0;
  return TOC_OK;
}

extern "C" int toc_linalg_trees(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int32_t kind,
                                const double* d_v, double* d_R, const double* d_u, double* d_O, void* d_scratch,
                                const uint8_t* d_trees, const int64_t* d_tree_off, void* stream);

extern "C" int toc_linalg(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                          const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int32_t kind,
                          const double* d_v, double* d_R, const double* d_u, double* d_O, void* d_scratch,
                          void* stream) {
  return toc_linalg_trees(d_arena, d_block_off, d_meta, d_row_base, n_blocks, plan, kind, d_v, d_R, d_u, d_O,
                          d_scratch, nullptr, nullptr, stream);
}

extern "C" int toc_linalg_set_splits(int on) {
  g_use_splits = on ? 1 : 0;
  return TOC_OK;
}

extern "C" int toc_tree_set_depth_order(int on) {
  g_depth_order = on ? 1 : 0;
  return TOC_OK;
}

extern "C" int toc_tree_offsets(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t wide, int64_t* h_tree_off) {
  if (!h_meta || !h_tree_off || n_blocks < 0) return TOC_E_ARG;
  int64_t o = 0;
  for (int64_t b = 0; b < n_blocks; ++b) {
    h_tree_off[b] = o;
    o += wide ? toc::cache_layout<true>(h_meta[b]).total : toc::cache_layout<false>(h_meta[b]).total;
  }
  h_tree_off[n_blocks] = o;
  return TOC_OK;
}

extern "C" int toc_build_trees(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                               int64_t n_blocks, const TocPlan* plan, const int64_t* d_tree_off, uint8_t* d_trees,
                               void* d_scratch, void* stream) {
  if (!plan || n_blocks < 0 || !d_trees || !d_tree_off) return TOC_E_ARG;
  if (plan->global_tables && !d_scratch) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  toc::LinalgArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.n_blocks = n_blocks;
  a.batch_smem_budget = plan->smem_bytes - (int32_t)toc::kFixedBytes;
  a.slab_bytes = plan->global_tables ? plan->scratch_bytes / plan->ctas : 0;
  a.scratch = (uint8_t*)d_scratch;
  a.trees = d_trees;
  a.tree_off = d_tree_off;
  a.depth_order = g_depth_order;
  void* fn = plan->wide ? (void*)toc::build_trees_kernel<true> : (void*)toc::build_trees_kernel<false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan->smem_bytes) != cudaSuccess)
    return TOC_E_CUDA;
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3(plan->ctas), dim3(plan->threads), args, plan->smem_bytes, (cudaStream_t)stream) ==
                 cudaSuccess
             ? TOC_OK
             : TOC_E_CUDA;
}

extern "C" int toc_linalg_trees(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int32_t kind,
                                const double* d_v, double* d_R, const double* d_u, double* d_O, void* d_scratch,
                                const uint8_t* d_trees, const int64_t* d_tree_off, void* stream) {
  if (!plan || n_blocks < 0 || !(kind & (TOC_MATVEC | TOC_VECMAT))) return TOC_E_ARG;
  if ((kind & TOC_MATVEC) && (!d_v || !d_R)) return TOC_E_ARG;
  if ((kind & TOC_VECMAT) && (!d_u || !d_O)) return TOC_E_ARG;
  if (plan->global_tables && !d_scratch) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  toc::LinalgArgs a;
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.n_blocks = n_blocks;
  a.kind = kind;
  a.n_cols = plan->n_cols;
  const int nvec = ((kind & TOC_MATVEC) ? 1 : 0) + ((kind & TOC_VECMAT) ? 1 : 0);
  const uint32_t fixed = toc::kFixedBytes + (plan->vec_in_smem ? nvec * toc::align16(8u * (uint32_t)plan->n_cols) : 0u);
  a.batch_smem_budget = plan->smem_bytes - (int32_t)fixed;
  a.slab_bytes = plan->global_tables ? plan->scratch_bytes / plan->ctas : 0;
  a.v = d_v;
  a.R = d_R;
  a.u = d_u;
  a.O = d_O;
  a.scratch = (uint8_t*)d_scratch;
  a.trees = d_trees;
  a.tree_off = d_tree_off;
  a.use_splits = g_use_splits;
  if ((kind & TOC_VECMAT) && !plan->vec_in_smem) {
    if (cudaMemsetAsync(d_O, 0, sizeof(double) * (size_t)n_blocks * plan->n_cols, s) != cudaSuccess)
      return TOC_E_CUDA;
  }
  cudaError_t e;
  if (plan->wide)
    e = plan->vec_in_smem ? launch<true, true>(a, *plan, s) : launch<true, false>(a, *plan, s);
  else
    e = plan->vec_in_smem ? launch<false, true>(a, *plan, s) : launch<false, false>(a, *plan, s);
  return e == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}
