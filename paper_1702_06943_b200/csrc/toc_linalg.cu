// toc_linalg.cu -- A.v and v^T.A directly on TOC1 blocks resident in HBM (sm_100a).
//
// Reference: kernels.py:115-142 (matvec, Algorithm 5) and kernels.py:145-174 (vecmat,
// Algorithm 6); the tree they walk is codec.py:215-259 (build_prefix_tree).
//
// Design: a persistent grid, one CTA per mini-batch at a time.  The CTA
// reads only the batch's TOC1 bytes and rebuilds, in shared memory, the part of the decode tree
// C' the products need:
//   par[d] = D-code at the position that derived node d           (codec.py:247)
//   key[d] = first-layer pair that node d appends = F(next code)   (codec.py:248-249)
// (d = derived node id - 1 - |I|).  Node values are never materialised: a code's partial sum
// is produced by walking par[] to the first layer, summing P1[key] (P1[i] = value_i * v[col_i])
// on the way.  Work per batch is O(|I| + C + nnz) shared-memory accesses, no HBM traffic
// beyond the block itself, v / u and the outputs.
//
//   matvec: P1 in tab[1..|I|]; each warp owns rows; lanes expand 32 codes at a time, a warp
//           reduction folds them into the row sum.
//   vecmat: G in tab[1..|I|]: each code adds u[row] to every pair key on its chain (the
//           transpose of the matvec walk, an fp64 shared-memory atomic per pair), then
//           out[col_i] += value_i * G[i].
#include "toc_common.cuh"

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
};

// Byte layout of one batch's tables (all regions 16-B aligned).
struct BatchLayout {
  uint32_t off_rowoff, off_dbase, off_last, off_uniq, off_tab, off_pk, total;
};

template <bool kWide>
TOC_HD BatchLayout batch_layout(const TocBlockMeta& m) {
  BatchLayout L;
  uint32_t o = 0;
  L.off_rowoff = o;
  o += align16(4u * (m.n_rows + 1));
  L.off_dbase = o;
  o += align16(4u * (m.n_rows + 1));
  L.off_last = o;
  o += align16(4u * (m.n_rows + 1));
  L.off_uniq = o;
  o += align16(8u * m.n_uniques);
  L.off_tab = o;
  o += align16(8u * (m.n_pairs + 1));
  L.off_pk = o;
  o += align16((kWide ? 8u : 4u) * m.n_derived);
  L.total = o;
  return L;
}

// Fixed shared-memory prefix of every CTA: block-scan scratch.
constexpr uint32_t kFixedBytes = 512;  // s_warp (33 words) at 0, s_red (33 doubles) at 160

// Node-table accessors.  Derived node d (id 1 + |I| + d) stores par = the D-code at the
// position that created it (its parent, codec.py:247) and, in the second field, first the
// following D-code and then -- after the key pass -- the first-layer pair node d appends, the
// first pair of that following code (codec.py:248-249).  Narrow trees pack the two fields as u16
// halves of one u32; wide ones use uint2.
template <bool kWide>
struct PK;

template <>
struct PK<false> {
  uint32_t* p;
  TOC_D void set_par(uint32_t d, uint32_t x) { reinterpret_cast<uint16_t*>(p)[2 * d] = (uint16_t)x; }
  TOC_D void set_nxt(uint32_t d, uint32_t x) { reinterpret_cast<uint16_t*>(p)[2 * d + 1] = (uint16_t)x; }
  TOC_D void set(uint32_t d, uint32_t par, uint32_t nxt) { p[d] = (par & 0xffffu) | (nxt << 16); }
  TOC_D uint32_t par(uint32_t d) const { return reinterpret_cast<const uint16_t*>(p)[2 * d]; }
  TOC_D uint32_t nxt(uint32_t d) const { return reinterpret_cast<const uint16_t*>(p)[2 * d + 1]; }
  TOC_D void get(uint32_t d, uint32_t& par, uint32_t& nxt) const {
    uint32_t w = p[d];
    par = w & 0xffffu;
    nxt = w >> 16;
  }
};

template <>
struct PK<true> {
  uint2* p;
  TOC_D void set_par(uint32_t d, uint32_t x) { p[d].x = x; }
  TOC_D void set_nxt(uint32_t d, uint32_t x) { p[d].y = x; }
  TOC_D void set(uint32_t d, uint32_t par, uint32_t nxt) { p[d] = make_uint2(par, nxt); }
  TOC_D uint32_t par(uint32_t d) const { return p[d].x; }
  TOC_D uint32_t nxt(uint32_t d) const { return p[d].y; }
  TOC_D void get(uint32_t d, uint32_t& par, uint32_t& nxt) const {
    uint2 w = p[d];
    par = w.x;
    nxt = w.y;
  }
};

// Exclusive scan over rows of max(len-1, 0): the id base of the nodes each row derives.
TOC_D void scan_derived_base(const uint32_t* rowoff, uint32_t* dbase, uint32_t n, uint32_t* s_warp) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < n; base += blockDim.x) {
    uint32_t r = base + tid;
    uint32_t len = (r < n) ? rowoff[r + 1] - rowoff[r] : 0u;
    uint32_t v = len ? len - 1 : 0u;
    uint32_t x = warp_excl_scan(v, lane);
    if (lane == 31) s_warp[warp] = x + v;
    __syncthreads();
    if (warp == 0) {
      uint32_t t = lane < nwarps ? s_warp[lane] : 0u;
      uint32_t e = warp_excl_scan(t, lane);
      if (lane < nwarps) s_warp[lane] = e;
      if (lane == 31) s_warp[32] = e + t;
    }
    __syncthreads();
    if (r < n) dbase[r] = carry + s_warp[warp] + x;
    carry += s_warp[32];
    __syncthreads();
  }
}

// Lanes per row: the largest power of two <= min(32, threads / rows).  Each thread then owns
// one contiguous segment of one row, so the code stream is walked sequentially per thread.
TOC_D uint32_t seg_lanes(uint32_t n, uint32_t nthreads) {
  uint32_t s = 1;
  while (s < 32 && 2 * s * (n ? n : 1) <= nthreads) s <<= 1;
  return s;
}

// ---- exact fixed-point accumulation with native 32-bit shared/global atomics ---------------
// fp64 atomics are CAS loops on sm_100a (shared) and the reduction order would make v^T.A
// non-deterministic.  Instead each accumulator is a 64-bit two's-complement integer (lo, hi
// words) holding value * 2^F; an add is atomicAdd on lo plus, when needed, atomicAdd of
// (x_hi + carry) on hi, the carry taken from lo's returned old value.  Modular 64-bit addition
// commutes, so concurrent adds are exact.  F is chosen per batch from an a-priori bound of the
// largest partial sum (below), so nothing overflows; the conversion error per term is 2^-(F+1).
TOC_D void fix_add(uint32_t* acc, long long x) {
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)((unsigned long long)x >> 32);
  const uint32_t old = atomicAdd(acc, xl);
  const uint32_t hi = xh + (old + xl < old ? 1u : 0u);
  if (hi) atomicAdd(acc + 1, hi);
}

TOC_D double fix_value(const uint32_t* acc, double inv_scale) {
  const long long v = (long long)(((unsigned long long)acc[1] << 32) | acc[0]);
  return (double)v * inv_scale;
}

// 2^F such that |sum| <= bound stays below 2^62.
TOC_D double fix_scale(double bound) {
  if (!(bound > 0.0)) return 1.0;
  int e;
  frexp(bound, &e);  // bound < 2^e
  return ldexp(1.0, 61 - e);
}

// One batch.  `tables` points either into shared memory or into this CTA's global slab.
template <bool kWide, bool kVecSmem>
__device__ __forceinline__ void process_batch(const LinalgArgs& a, int64_t b, const TocBlockMeta& m,
                                              uint8_t* tables, const double* vec_s, uint32_t* acc_s,
                                              uint32_t* s_warp, double* s_red) {
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  const uint8_t* blk = a.arena + a.block_off[b];
  const BatchLayout L = batch_layout<kWide>(m);
  uint32_t* rowoff = reinterpret_cast<uint32_t*>(tables + L.off_rowoff);
  uint32_t* dbase = reinterpret_cast<uint32_t*>(tables + L.off_dbase);
  uint32_t* last = reinterpret_cast<uint32_t*>(tables + L.off_last);
  double* uniq = reinterpret_cast<double*>(tables + L.off_uniq);
  double* tab = reinterpret_cast<double*>(tables + L.off_tab);
  uint32_t* tabw = reinterpret_cast<uint32_t*>(tab);  // tab as words: ref staging / fixed point
  PK<kWide> pk;
  pk.p = reinterpret_cast<decltype(pk.p)>(tables + L.off_pk);

  const uint32_t n = m.n_rows, nI = m.n_pairs, nU = m.n_uniques;
  const uint8_t* cols = blk + m.off_cols;
  const uint8_t* refs = blk + m.off_refs;
  const uint8_t* codes = blk + m.off_codes;
  const int64_t row_base = a.row_base[b];
  const int32_t ncol = a.n_cols;
  const double* vec = kVecSmem ? vec_s : a.v;
  const bool do_mv = a.kind & TOC_MATVEC, do_vm = a.kind & TOC_VECMAT;

  // ---- phase 0: row offsets, value index, bounds for the fixed-point scales -----------------
  const uint32_t wo = m.w_offsets;
  for (uint32_t r = tid; r <= n; r += nth) rowoff[r] = ld_packed(blk + m.off_offsets, r, wo);
  double umax = 0.0, vmax = 0.0;
  for (uint32_t i = tid; i < nU; i += nth) {
    const double x = ld_f64_unaligned(blk + m.off_uniques + 8u * i);
    uniq[i] = x;
    vmax = fmax(vmax, fabs(x));
  }
  if (do_vm) {
    for (uint32_t r = tid; r < n; r += nth) umax += fabs(a.u[row_base + r]);
    if (kVecSmem)
      for (int32_t c = tid; c < 2 * ncol; c += nth) acc_s[c] = 0u;
  }
  __syncthreads();
  scan_derived_base(rowoff, dbase, n, s_warp);
  double g_scale = 1.0, o_scale = 1.0;
  if (do_vm) {  // sum |u| over the batch and max |value|: the a-priori bounds (see fix_add)
    const double su = block_sum(umax, s_red), mv = block_max_d(vmax, s_red);
    g_scale = fix_scale(su);
    o_scale = fix_scale(su * mv);
  }

  const uint32_t S = seg_lanes(n, nth), RP = nth / S, passes = (n + RP - 1) / RP, sub = tid % S;
  const uint32_t per_pair = (nI + nth - 1) / nth, p0 = min(nI, tid * per_pair), p1 = min(nI, p0 + per_pair);

  // ---- phase 1: one sequential pass over each thread's code segment -------------------------
  with_width(m.w_codes, [&]<int W>() {
    for (uint32_t k = 0; k < passes; ++k) {
      const uint32_t r = tid / S + k * RP;
      if (r >= n) break;
      const uint32_t lo = rowoff[r], hi = rowoff[r + 1], db = dbase[r], len = hi - lo;
      const uint32_t j0 = lo + (len * sub) / S, j1 = lo + (len * (sub + 1)) / S;
      if (j0 >= j1) continue;
      SeqReader<W> rd;
      rd.init(codes, j0);
      uint32_t c = rd.next();
      for (uint32_t j = j0; j < j1; ++j) {
        if (j + 1 < hi) {  // non-final: node (par = this code, nxt = next code), one store
          const uint32_t cn = rd.next();
          pk.set(db + (j - lo), c, cn);
          c = cn;
        } else {
          last[r] = c;
        }
      }
    }
  });
  // first-layer products P1[i] = value_i * v[col_i] (matvec), or G = 0 (vecmat only)
  if (do_mv) {
    if (p0 < p1) {
      with_width(m.w_refs, [&]<int W>() {
        SeqReader<W> rd;
        rd.init(refs, p0);
        for (uint32_t i = p0; i < p1; ++i) tabw[2 * (i + 1)] = rd.next();
      });
      with_width(m.w_cols, [&]<int W>() {
        SeqReader<W> rd;
        rd.init(cols, p0);
        for (uint32_t i = p0; i < p1; ++i) tab[i + 1] = uniq[tabw[2 * (i + 1)]] * vec[rd.next()];
      });
    }
  } else {
    for (uint32_t i = tid; i <= nI; i += nth) tab[i] = 0.0;
  }
  __syncthreads();

  // ---- key pass: the pair each derived node appends is the first pair of its next code:
  //      follow par[] from that code down to the first layer (codec.py:248-251) ---------------
  for (uint32_t k = 0; k < passes; ++k) {
    const uint32_t r = tid / S + k * RP;
    if (r >= n) break;
    const uint32_t lo = rowoff[r], hi = rowoff[r + 1], db = dbase[r], len = hi - lo;
    const uint32_t j0 = lo + (len * sub) / S, j1 = min(lo + (len * (sub + 1)) / S, hi - 1);
    for (uint32_t j = j0; j < j1; ++j) {
      const uint32_t d = db + (j - lo);
      uint32_t x = pk.nxt(d);
      while (x > nI) x = pk.par(x - 1 - nI);
      pk.set_nxt(d, x);
    }
  }
  __syncthreads();

  // The walk of one code x: each derived node on the chain contributes its key, the first-layer
  // node at the end contributes itself.  visit(i) is called once per pair, i = first-layer id.
  auto walk_segment = [&](uint32_t r, uint32_t j0, uint32_t j1, uint32_t lo, uint32_t hi, uint32_t db,
                          auto&& visit) {
    for (uint32_t j = j0; j < j1; ++j) {
      uint32_t x = (j + 1 < hi) ? pk.par(db + (j - lo)) : last[r];
      while (x > nI) {
        uint32_t p, key;
        pk.get(x - 1 - nI, p, key);
        visit(key);
        x = p;
      }
      visit(x);
    }
  };

  // ---- phase 2: A.v -------------------------------------------------------------------------
  if (do_mv) {
    for (uint32_t k = 0; k < passes; ++k) {
      const uint32_t r = tid / S + k * RP;
      double part = 0.0;
      if (r < n) {
        const uint32_t lo = rowoff[r], hi = rowoff[r + 1], db = dbase[r], len = hi - lo;
        const uint32_t j0 = lo + (len * sub) / S, j1 = lo + (len * (sub + 1)) / S;
        walk_segment(r, j0, j1, lo, hi, db, [&](uint32_t i) { part += tab[i]; });
      }
      __syncwarp();
      for (uint32_t o = S >> 1; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (r < n && sub == 0) a.R[row_base + r] = part;
    }
  }

  // ---- phase 3: u^T.A -----------------------------------------------------------------------
  if (do_vm) {
    if (do_mv) {
      __syncthreads();
      for (uint32_t i = tid; i <= nI; i += nth) tab[i] = 0.0;
      __syncthreads();
    }
    for (uint32_t k = 0; k < passes; ++k) {
      const uint32_t r = tid / S + k * RP;
      if (r >= n) break;
      const uint32_t lo = rowoff[r], hi = rowoff[r + 1], db = dbase[r], len = hi - lo;
      const uint32_t j0 = lo + (len * sub) / S, j1 = lo + (len * (sub + 1)) / S;
      const long long w = __double2ll_rn(a.u[row_base + r] * g_scale);
      if (w == 0) continue;
      walk_segment(r, j0, j1, lo, hi, db, [&](uint32_t i) { fix_add(tabw + 2 * i, w); });
    }
    __syncthreads();
    uint32_t* out = kVecSmem ? acc_s : reinterpret_cast<uint32_t*>(a.O + b * (int64_t)ncol);
    const double g_inv = 1.0 / g_scale;
    if (p0 < p1) {
      // contribution value_i * G[i] replaces G[i] in place, then scatter by column
      with_width(m.w_refs, [&]<int W>() {
        SeqReader<W> rd;
        rd.init(refs, p0);
        for (uint32_t i = p0; i < p1; ++i) tab[i + 1] = uniq[rd.next()] * fix_value(tabw + 2 * (i + 1), g_inv);
      });
      with_width(m.w_cols, [&]<int W>() {
        SeqReader<W> rd;
        rd.init(cols, p0);
        for (uint32_t i = p0; i < p1; ++i) {
          const uint32_t c = rd.next();
          const long long g = __double2ll_rn(tab[i + 1] * o_scale);
          if (g) fix_add(out + 2 * c, g);
        }
      });
    }
    __syncthreads();
    const double o_inv = 1.0 / o_scale;
    double* o = a.O + b * (int64_t)ncol;
    if (kVecSmem) {
      for (int32_t c = tid; c < ncol; c += nth) o[c] = fix_value(acc_s + 2 * c, o_inv);
    } else {
      uint32_t* ow = reinterpret_cast<uint32_t*>(o);
      for (int32_t c = tid; c < ncol; c += nth) {
        const uint32_t w2[2] = {__ldcg(ow + 2 * c), __ldcg(ow + 2 * c + 1)};
        o[c] = fix_value(w2, o_inv);
      }
    }
  }
}

template <bool kWide, bool kVecSmem>
__global__ void __launch_bounds__(1024, 1) linalg_kernel(LinalgArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);  // 33 words
  uint8_t* p = smem + kFixedBytes;
  double* s_red = reinterpret_cast<double*>(smem + 160);  // 33 doubles
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
    if (threadIdx.x == 0 && b + gridDim.x < a.n_blocks) {  // pull the CTA's next block into L2
      const TocBlockMeta& mn = a.meta[b + gridDim.x];
      const uint32_t bytes = align16(mn.off_offsets + (mn.n_rows + 1u) * mn.w_offsets);
      const uint8_t* nb = a.arena + a.block_off[b + gridDim.x];
      if (mn.status == TOC_OK && bytes > 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nb), "r"(bytes) : "memory");
    }
    __syncthreads();
    if (need <= (uint32_t)a.batch_smem_budget)
      process_batch<kWide, kVecSmem>(a, b, m, p, vec_s, acc_s, s_warp, s_red);
    else
      process_batch<kWide, kVecSmem>(a, b, m, slab, vec_s, acc_s, s_warp, s_red);
  }
}

}  // namespace toc

// ------------------------------------------------------------------------------------------
// Host side: planning and launch.
namespace {

struct DevProps {
  int sm_count = 0, smem_optin = 0, smem_per_sm = 0;
  int64_t l2 = 0;
};

const DevProps& dev_props() {
  static DevProps p;
  static bool init = false;
  if (!init) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&p.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&p.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    p.l2 = l2;
    if (p.sm_count <= 0) {  // no device visible (planning on a CPU host): B200 figures
      p.sm_count = 148;
      p.smem_optin = 232448;
      p.smem_per_sm = 233472;
      p.l2 = 126 << 20;
    }
    init = true;
  }
  return p;
}

template <bool W, bool V>
cudaError_t launch(const toc::LinalgArgs& a, const TocPlan& plan, cudaStream_t s) {
  static int configured = -1;
  if (configured < plan.smem_bytes) {
    cudaError_t e = cudaFuncSetAttribute(toc::linalg_kernel<W, V>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, plan.smem_bytes);
    if (e != cudaSuccess) return e;
    configured = plan.smem_bytes;
  }
  toc::linalg_kernel<W, V><<<plan.ctas, plan.threads, plan.smem_bytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

extern "C" int toc_plan(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t kind, TocPlan* plan) {
  if (!plan || (n_blocks > 0 && !h_meta) || !(kind & (TOC_MATVEC | TOC_VECMAT))) return TOC_E_ARG;
  memset(plan, 0, sizeof(*plan));
  const DevProps& d = dev_props();
  uint64_t max_T = 0;
  int32_t n_cols = n_blocks ? (int32_t)h_meta[0].n_cols : 0;
  for (int64_t b = 0; b < n_blocks; b++) {
    const TocBlockMeta& m = h_meta[b];
    if ((int32_t)m.n_cols != n_cols) return TOC_E_ARG;
    uint64_t T = 1ull + m.n_pairs + m.n_derived;
    if (T > max_T) max_T = T;
    if ((int32_t)m.n_rows > plan->max_rows) plan->max_rows = (int32_t)m.n_rows;
  }
  plan->wide = max_T > 65536ull;
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

extern "C" int toc_linalg(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                          const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int32_t kind,
                          const double* d_v, double* d_R, const double* d_u, double* d_O, void* d_scratch,
                          void* stream) {
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
