// toc_batch.cuh -- per-mini-batch device machinery shared by the compressed linear-algebra
// sweep (toc_linalg.cu) and the MGD kernels (toc_mgd.cu).
//
// Reference: codec.py:215-259 (build_prefix_tree: the decode tree C'), kernels.py:115-142
// (matvec, Algorithm 5), kernels.py:145-174 (vecmat, Algorithm 6).
//
// One CTA works on one TOC1 block at a time.  It reads only the block's bytes and rebuilds in
// shared memory (or in a global slab for oversized batches) the part of C' the products need:
//   node[d] = (par, key) for derived node d = id - 1 - |I|:
//     par = the D-code at the position that derived node d           (codec.py:247)
//     key = the first-layer pair node d appends = first pair of the next D-code (codec.py:248)
//   last[r] = the final code of row r (the only codes that derive no node)
// so the code stream D itself is recoverable from node[] + last[] and is read from HBM once.
// Node partial sums are never materialised: a code's contribution is produced by walking par
// links down to the first layer, visiting key on the way (Algorithm 5's H recurrence unrolled).
#pragma once
#include "toc_common.cuh"

namespace toc {

// Byte layout of one batch's tables (all regions 16-B aligned).  The first four regions --
// row offsets, derived-node bases, final codes and the node table -- depend only on the block and
// form the "tree" prefix [0, tree): the device tree cache stores exactly these bytes per batch so a
// kernel can pull them into shared memory with one bulk copy instead of rebuilding them.
struct BatchLayout {
  uint32_t off_rowoff, off_dbase, off_last, off_pk, tree, off_uniq, off_tab, total;
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
  L.off_pk = o;
  o += align16((kWide ? 8u : 4u) * m.n_derived);
  L.tree = o;
  L.off_uniq = o;
  o += align16(8u * m.n_uniques);
  L.off_tab = o;
  o += align16(8u * (m.n_pairs + 1));
  L.total = o;
  return L;
}

// Device tree cache entry of one batch (toc_build_trees): the tree prefix above, then
//   irec  (column, value ref) per first-layer pair, unpacked   -- P1 with coalesced loads
//   prec  (pair id, value ref) sorted by (column, pair id)    } v^T.A's output as a fixed-order
//   segs  (start in prec, column) per distinct column, + end  } segmented sum, no atomics
//   info  n_segs (0xffffffff: not sorted, the atomic scatter is used)
//   splits (first code of each lane's range, relative to the row start) per (row, lane) for the
//         S = seg_lanes(n_rows, kSplitThreads) lanes of a row, balanced by PAIR count (the
//         lanes' flat walks then take equal numbers of iterations); info[1] = S
struct CacheLayout {
  uint32_t tree, off_irec, off_prec, off_segs, off_info, off_splits, total;
};

// Lanes per row: the largest power of two <= min(32, threads / rows).  Each thread then owns
// one contiguous segment of one row, so the code stream is walked sequentially per thread.
TOC_HD uint32_t seg_lanes(uint32_t n, uint32_t nthreads) {
  uint32_t s = 1;
  while (s < 32 && 2 * s * (n ? n : 1) <= nthreads) s <<= 1;
  return s;
}

// The CTA size the cached lane splits are computed for (the sweep's plan for tables that need
// most of shared memory); other CTA sizes fall back to code-count splits.
constexpr uint32_t kSplitThreads = 1024;

// A pair record (two small ids).  Narrow trees (< 65,536 nodes, n_cols <= 65,536: toc_plan) pack
// both as u16 halves of one u32; wide ones use uint2.
template <bool kWide>
struct PairRec;

template <>
struct PairRec<false> {
  using T = uint32_t;
  TOC_HD static T make(uint32_t a, uint32_t b) { return a | (b << 16); }
  TOC_D static uint32_t a(T r) { return r & 0xffffu; }
  TOC_D static uint32_t b(T r) { return r >> 16; }
  TOC_D static T none() { return 0u; }
};

template <>
struct PairRec<true> {
  using T = uint2;
  TOC_HD static T make(uint32_t a, uint32_t b) { return T{a, b}; }
  TOC_D static uint32_t a(T r) { return r.x; }
  TOC_D static uint32_t b(T r) { return r.y; }
  TOC_D static T none() { return make_uint2(0u, 0u); }
};

template <bool kWide>
TOC_HD CacheLayout cache_layout(const TocBlockMeta& m) {
  CacheLayout C;
  const uint32_t nI = m.n_pairs, segs = (nI < m.n_cols ? nI : m.n_cols) + 1u;
  C.tree = batch_layout<kWide>(m).tree;
  uint32_t o = C.tree;
  C.off_irec = o;
  o += align16((uint32_t)sizeof(typename PairRec<kWide>::T) * nI);
  C.off_prec = o;
  o += align16((uint32_t)sizeof(typename PairRec<kWide>::T) * nI);
  C.off_segs = o;
  o += align16(8u * segs);
  C.off_info = o;
  o += 16u;
  C.off_splits = o;
  o += align16(2u * m.n_rows * seg_lanes(m.n_rows, kSplitThreads));
  C.total = o;
  return C;
}

constexpr uint32_t kNoSegs = 0xffffffffu;

// ---- TMA bulk copy global -> shared with an mbarrier (sm_90+ async proxy) ------------------
TOC_D uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

TOC_D void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// One thread: order earlier generic shared accesses before the async copy, announce the bytes,
// start the copy (dst, src 16-B aligned, bytes a multiple of 16).
TOC_D void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}

TOC_D void mbar_wait(uint64_t* mbar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(mbar)), "r"(phase)
        : "memory");
  }
}

// Fixed shared-memory prefix of every CTA: block-scan words and block-reduction doubles.
constexpr uint32_t kFixedBytes = 512;  // s_warp (33 words) at 0, s_red (33 doubles) at 160

// Node table.  Narrow trees (< 65536 nodes) pack the two fields as u16 halves of one u32;
// wide ones use uint2.  The second field first holds the next D-code and, after the key pass,
// the key.
template <bool kWide>
struct PK;

template <>
struct PK<false> {
  uint32_t* p;
  TOC_D void set(uint32_t d, uint32_t par, uint32_t nxt) { p[d] = (par & 0xffffu) | (nxt << 16); }
  TOC_D void set_key(uint32_t d, uint32_t x) { reinterpret_cast<uint16_t*>(p)[2 * d + 1] = (uint16_t)x; }
  TOC_D uint32_t par(uint32_t d) const { return reinterpret_cast<const uint16_t*>(p)[2 * d]; }
  TOC_D uint32_t nxt(uint32_t d) const { return reinterpret_cast<const uint16_t*>(p)[2 * d + 1]; }
  TOC_D void get(uint32_t d, uint32_t& par, uint32_t& key) const {
    uint32_t w = p[d];
    par = w & 0xffffu;
    key = w >> 16;
  }
};

template <>
struct PK<true> {
  uint2* p;
  TOC_D void set(uint32_t d, uint32_t par, uint32_t nxt) { p[d] = make_uint2(par, nxt); }
  TOC_D void set_key(uint32_t d, uint32_t x) { p[d].y = x; }
  TOC_D uint32_t par(uint32_t d) const { return p[d].x; }
  TOC_D uint32_t nxt(uint32_t d) const { return p[d].y; }
  TOC_D void get(uint32_t d, uint32_t& par, uint32_t& key) const {
    uint2 w = p[d];
    par = w.x;
    key = w.y;
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

// ---- exact fixed-point accumulation with native 32-bit atomics -----------------------------
// fp64 atomics are CAS loops on sm_100a (shared) and their order would make v^T.A
// non-deterministic.  Each accumulator is a 64-bit two's-complement integer (lo, hi words)
// holding value * 2^F; an add is atomicAdd on lo plus, when needed, atomicAdd of (x_hi + carry)
// on hi, the carry taken from lo's returned old value.  Modular 64-bit addition commutes, so
// concurrent adds are exact.  F is chosen from an a-priori bound of the largest partial sum so
// nothing overflows; the conversion error per term is at most 2^-(F+1).
TOC_D void fix_add(uint32_t* acc, long long x) {
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)((unsigned long long)x >> 32);
  const uint32_t old = atomicAdd(acc, xl);
  const uint32_t hi = xh + (old + xl < old ? 1u : 0u);
  if (hi) atomicAdd(acc + 1, hi);
}

// The same with the two words in separate arrays (lo[i], hi[i]): random adds then spread over
// all 32 banks instead of the 16 even ones.  No branch: at the scales used the high word of an
// addend is almost never zero, so skipping its add only costs divergence handling.
TOC_D void fix_add_split(uint32_t* lo, uint32_t* hi, uint32_t i, uint32_t xl, uint32_t xh) {
  const uint32_t old = atomicAdd(lo + i, xl);
  atomicAdd(hi + i, xh + (old + xl < old ? 1u : 0u));
}

// Carry-free variant (two "limbs", both added with fire-and-forget RED.ADD): an addend x (exact
// integer, value * 2^F) is split as x = xh * 2^L + xl with 0 <= xl < 2^L; lo[i] sums the xl
// unsigned and hi[i] the xh signed.  A pair gets at most one add per row, so with
// L = 32 - bits(n_rows) the lo word cannot wrap; F is chosen so |sum of x| < 2^(L+30) and the hi
// word cannot either.  Exact and order-independent like fix_add, without the dependent
// return-value carry.
TOC_D uint32_t limb_bits(uint32_t n_rows) { return 32u - (32u - __clz(n_rows ? n_rows : 1u)); }

TOC_D double limb_scale(double bound, uint32_t L) {  // 2^F with |sum| <= bound -> < 2^(L+30)
  if (!(bound > 0.0)) return 1.0;
  int e;
  frexp(bound, &e);
  return ldexp(1.0, (int)L + 30 - e);
}

TOC_D void limb_add(uint32_t* lo, int32_t* hi, uint32_t i, uint32_t xl, int32_t xh) {
  atomicAdd(lo + i, xl);
  atomicAdd(hi + i, xh);
}

TOC_D double limb_value(uint32_t lo, int32_t hi, uint32_t L, double inv_scale) {
  return (double)(((long long)hi << L) + (long long)lo) * inv_scale;
}

TOC_D double fix_value(uint32_t lo, uint32_t hi, double inv_scale) {
  const long long v = (long long)(((unsigned long long)hi << 32) | lo);
  return (double)v * inv_scale;
}

// Fixed point is exact in the accumulation but rounds every addend to the quantum 1/scale, which
// is set by the batch's whole sum |u|.  When n_rows * max|value| quanta could exceed 2^-31 (a
// row weight far above the others, or a heavy-tailed u), the batch accumulates in fp64 instead
// (shared-memory atomics; order-dependent only at the last bit): the reference's own
// accuracy, since the 1e-9 bar applies to every output column.
constexpr uint32_t kGF64 = 64;  // column_sums mode: G held as doubles in tab
TOC_D bool fixed_point_too_coarse(uint32_t n_rows, double vmax, double err_per_unit_value) {
  return (double)n_rows * vmax * err_per_unit_value > 0x1p-31;
}

// 2^F such that |sum| <= bound stays below 2^62.
TOC_D double fix_scale(double bound) {
  if (!(bound > 0.0)) return 1.0;
  int e;
  frexp(bound, &e);  // bound < 2^e
  return ldexp(1.0, 61 - e);
}

// ---- one batch in one CTA -------------------------------------------------------------------
template <bool kWide>
struct Batch {
  const uint8_t* blk;
  TocBlockMeta m;
  uint32_t* rowoff;
  uint32_t* dbase;
  uint32_t* last;
  double* uniq;
  double* tab;     // P1 (matvec) or G (vecmat, fixed point), index = first-layer id
  uint32_t* tabw;  // tab as words
  PK<kWide> pk;
  const uint16_t* splits = nullptr;  // cached pair-balanced lane splits (tree cache), or NULL
  uint32_t n, nI, S, lgS, RP, passes, sub, p0, p1;
  double vmax;     // max |value| over the value index (this thread's part until reduced)

  // tables: shared (or slab) base of the whole layout; tree: where the tree prefix lives (the same
  // base, or a cached tree blob in global memory read in place).
  TOC_D void init(const uint8_t* block, const TocBlockMeta& meta, uint8_t* tables, uint8_t* tree = nullptr) {
    blk = block;
    m = meta;
    const BatchLayout L = batch_layout<kWide>(m);
    uint8_t* t = tree ? tree : tables;
    rowoff = reinterpret_cast<uint32_t*>(t + L.off_rowoff);
    dbase = reinterpret_cast<uint32_t*>(t + L.off_dbase);
    last = reinterpret_cast<uint32_t*>(t + L.off_last);
    pk.p = reinterpret_cast<decltype(pk.p)>(t + L.off_pk);
    uniq = reinterpret_cast<double*>(tables + L.off_uniq);
    tab = reinterpret_cast<double*>(tables + L.off_tab);
    tabw = reinterpret_cast<uint32_t*>(tab);
    shape();
  }

  // A batch whose tree prefix, value index and tables all live elsewhere (a cached step image,
  // toc_mgd.cu): P1 in p1tab, G (fixed point) in gtab -- separate, so G needs no zeroing barrier
  // after A.v has read P1.
  TOC_D void bind(const TocBlockMeta& meta, uint8_t* tree, double* uniq_, double* p1tab, uint32_t* gtab) {
    blk = nullptr;
    m = meta;
    const BatchLayout L = batch_layout<kWide>(m);
    rowoff = reinterpret_cast<uint32_t*>(tree + L.off_rowoff);
    dbase = reinterpret_cast<uint32_t*>(tree + L.off_dbase);
    last = reinterpret_cast<uint32_t*>(tree + L.off_last);
    pk.p = reinterpret_cast<decltype(pk.p)>(tree + L.off_pk);
    uniq = uniq_;
    tab = p1tab;
    tabw = gtab;
    shape();
  }

  TOC_D void shape() {
    n = m.n_rows;
    nI = m.n_pairs;
    const uint32_t nth = blockDim.x, tid = threadIdx.x;
    S = seg_lanes(n, nth);
    lgS = __ffs(S) - 1;
    RP = nth / S;
    passes = (n + RP - 1) / RP;
    sub = tid % S;
    const uint32_t per = (nI + nth - 1) / nth;
    p0 = min(nI, tid * per);
    p1 = min(nI, p0 + per);
  }

  // Row r's code range and this thread's segment of it.
  TOC_D bool segment(uint32_t k, uint32_t& r, uint32_t& lo, uint32_t& hi, uint32_t& db, uint32_t& j0,
                     uint32_t& j1) const {
    r = (threadIdx.x >> lgS) + k * RP;
    if (r >= n) return false;
    lo = rowoff[r];
    hi = rowoff[r + 1];
    db = dbase[r];
    if (splits) {
      j0 = lo + __ldg(splits + r * S + sub);
      j1 = sub + 1 < S ? lo + __ldg(splits + r * S + sub + 1) : hi;
      return true;
    }
    const uint32_t len = hi - lo;
    j0 = lo + ((len * sub) >> lgS);
    j1 = lo + ((len * (sub + 1)) >> lgS);
    return true;
  }

  // Pair-balanced splits of every row for S lanes (after the key pass; node tables complete):
  // lane s starts at the first code whose preceding pairs reach s/S of the row's pairs.
  TOC_D void write_splits(uint16_t* out, uint32_t S_) const {
    for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) {
      const uint32_t lo = rowoff[r], hi = rowoff[r + 1], db = dbase[r];
      auto depth = [&](uint32_t j) {
        uint32_t x = (j + 1 < hi) ? pk.par(db + (j - lo)) : last[r], dpt = 1;
        while (x > nI) {
          x = pk.par(x - 1 - nI);
          ++dpt;
        }
        return dpt;
      };
      uint32_t total = 0;
      for (uint32_t j = lo; j < hi; ++j) total += depth(j);
      uint32_t acc = 0, s = 1;
      out[r * S_] = 0;
      for (uint32_t j = lo; j < hi && s < S_; ++j) {
        while (s < S_ && (uint64_t)acc * S_ >= (uint64_t)total * s) out[r * S_ + s++] = (uint16_t)(j - lo);
        acc += depth(j);
      }
      while (s < S_) out[r * S_ + s++] = (uint16_t)(hi - lo);
    }
  }

  // The value index (and this thread's part of max |value|).  No barrier.
  TOC_D void load_values() {
    vmax = 0.0;
    for (uint32_t i = threadIdx.x; i < m.n_uniques; i += blockDim.x) {
      const double x = ld_f64_unaligned(blk + m.off_uniques + 8u * i);
      uniq[i] = x;
      vmax = fmax(vmax, fabs(x));
    }
  }

  // Phase 0: row offsets, value index, derived-node bases.  Ends with a barrier.
  TOC_D void load_index(uint32_t* s_warp) {
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    for (uint32_t r = tid; r <= n; r += nth) rowoff[r] = ld_packed(blk + m.off_offsets, r, m.w_offsets);
    load_values();
    __syncthreads();
    scan_derived_base(rowoff, dbase, n, s_warp);
  }

  // Phase 1: one sequential pass over each thread's code segment: node[] + last[].
  TOC_D void build_nodes() {
    const uint8_t* codes = blk + m.off_codes;
    with_width(m.w_codes, [&]<int W>() {
      for (uint32_t k = 0; k < passes; ++k) {
        uint32_t r, lo, hi, db, j0, j1;
        if (!segment(k, r, lo, hi, db, j0, j1)) break;
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
  }

  // Key pass (after a barrier following build_nodes): key = first pair of the next code, found
  // by following par links down to the first layer (codec.py:248-251).
  TOC_D void resolve_keys() {
    for (uint32_t k = 0; k < passes; ++k) {
      uint32_t r, lo, hi, db, j0, j1;
      if (!segment(k, r, lo, hi, db, j0, j1)) break;
      j1 = min(j1, hi - 1);
      for (uint32_t j = j0; j < j1; ++j) {
        const uint32_t d = db + (j - lo);
        uint32_t x = pk.nxt(d);
        while (x > nI) x = pk.par(x - 1 - nI);
        pk.set_key(d, x);
      }
    }
  }

  // First-layer products P1[i] = value_i * vec[col_i] (Algorithm 5's H for depth-1 nodes).
  // kCG: vec lives in global memory written by other CTAs of the same launch (read via L2).
  template <bool kCG>
  TOC_D void compute_p1(const double* vec) {
    if (p0 >= p1) return;
    with_width(m.w_refs, [&]<int W>() {
      SeqReader<W> rd;
      rd.init(blk + m.off_refs, p0);
      for (uint32_t i = p0; i < p1; ++i) tabw[2 * (i + 1)] = rd.next();
    });
    with_width(m.w_cols, [&]<int W>() {
      SeqReader<W> rd;
      rd.init(blk + m.off_cols, p0);
      for (uint32_t i = p0; i < p1; i += 8) {  // 8 independent vec loads in flight
        uint32_t c[8];
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = (i + k < p1) ? rd.next() : 0u;
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = (i + k < p1) ? (kCG ? __ldcg(vec + c[k]) : vec[c[k]]) : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (i + k < p1) tab[i + k + 1] = uniq[tabw[2 * (i + k + 1)]] * x[k];
      }
    });
  }

  TOC_D void zero_tab() {
    for (uint32_t i = threadIdx.x; i <= nI; i += blockDim.x) tab[i] = 0.0;
  }

  // Walk the codes of [j0, j1) of row r; visit(i) once per pair (i = first-layer id).
  // Two codes per iteration, their chains stepped in lockstep: the dependent shared loads of one
  // chain overlap those of the other (the walk is latency-bound on these loads).  The visit is
  // inlined at four sites, so this suits a cheap visit (A.v: one gather and an add).
  template <typename V>
  TOC_D void walk(uint32_t r, uint32_t lo, uint32_t hi, uint32_t db, uint32_t j0, uint32_t j1, V&& visit) const {
    uint32_t j = j0;
    for (; j + 1 < j1; j += 2) {
      uint32_t x = pk.par(db + (j - lo));  // j + 1 < j1 <= hi: j is never the final code
      uint32_t y = (j + 2 < hi) ? pk.par(db + (j + 1 - lo)) : last[r];
      while (x > nI || y > nI) {
        TOC_CHECK((x <= nI || x - 1 - nI < m.n_derived) && (y <= nI || y - 1 - nI < m.n_derived));
        uint32_t px = x, kx = 0, py = y, ky = 0;
        if (x > nI) pk.get(x - 1 - nI, px, kx);
        if (y > nI) pk.get(y - 1 - nI, py, ky);
        if (kx) visit(kx);
        if (ky) visit(ky);
        x = px;
        y = py;
      }
      visit(x);
      visit(y);
    }
    if (j < j1) {
      uint32_t x = (j + 1 < hi) ? pk.par(db + (j - lo)) : last[r];
      while (x > nI) {
        uint32_t p, key;
        pk.get(x - 1 - nI, p, key);
        visit(key);
        x = p;
      }
      visit(x);
    }
  }

  // The same walk one node per iteration, the visit inlined once: for a costly visit (v^T.A: two
  // dependent atomics), where walk's predicated duplicate sites cost more than its overlap gains.
  // A code <= nI is a pair and ends its chain.
  template <typename V>
  TOC_D void walk_flat(uint32_t r, uint32_t lo, uint32_t hi, uint32_t db, uint32_t j0, uint32_t j1,
                       V&& visit) const {
    if (j0 >= j1) return;
    uint32_t j = j0;
    uint32_t x = (j + 1 < hi) ? pk.par(db + (j - lo)) : last[r];
    for (;;) {
      uint32_t par = 0, key = x;
      TOC_CHECK(x >= 1 && (x <= nI || x - 1 - nI < m.n_derived));
      if (x > nI) pk.get(x - 1 - nI, par, key);
      visit(key);
      if (par) {
        x = par;
        continue;
      }
      if (++j >= j1) break;
      x = (j + 1 < hi) ? pk.par(db + (j - lo)) : last[r];
    }
  }

  // A.v with P1 in tab: emit(r, (A.v)[r]) once per row (by the row's first segment lane).
  // Lane ranges: the cached pair-balanced splits when present (the cache build orders each range's
  // codes deepest first, so the lockstep walks of a warp's lanes stay in step), else code counts.
  template <typename E>
  TOC_D void matvec_rows(E&& emit) {
    for (uint32_t k = 0; k < passes; ++k) {
      uint32_t r, lo, hi, db, j0, j1;
      double part = 0.0;
      const bool ok = segment(k, r, lo, hi, db, j0, j1);
      if (ok) walk(r, lo, hi, db, j0, j1, [&](uint32_t i) { part += tab[i]; });
      __syncwarp();
      for (uint32_t o = S >> 1; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (ok && sub == 0) emit(r, part);
    }
  }

  // G[i] += sum over the pair occurrences of weight(r) (fixed point, scale g_scale); tab must be
  // zeroed.  weight(r) returns u[r].
  template <typename Wt>
  TOC_D void vecmat_rows(Wt&& weight, double g_scale) {
    for (uint32_t k = 0; k < passes; ++k) {
      uint32_t r, lo, hi, db, j0, j1;
      if (!segment(k, r, lo, hi, db, j0, j1)) break;
      const long long w = __double2ll_rn(weight(r) * g_scale);
      if (w == 0) continue;
      walk_flat(r, lo, hi, db, j0, j1, [&](uint32_t i) { fix_add(tabw + 2 * i, w); });
    }
  }

  // G in fp64 (the fallback for coarse fixed point, see fixed_point_too_coarse); tab zeroed.
  template <typename Wt>
  TOC_D void vecmat_rows_f64(Wt&& weight) {
    for (uint32_t k = 0; k < passes; ++k) {
      uint32_t r, lo_, hi_, db, j0, j1;
      if (!segment(k, r, lo_, hi_, db, j0, j1)) break;
      const double w = weight(r);
      if (w == 0.0) continue;
      walk_flat(r, lo_, hi_, db, j0, j1, [&](uint32_t i) { atomicAdd(tab + i, w); });
    }
  }

  // G with split words (fix_add_split): lo = tabw[0..nI], hi = tabw[nI+1..2nI+1]; tab zeroed.
  template <typename Wt>
  TOC_D void vecmat_rows_split(Wt&& weight, double g_scale) {
    uint32_t* lo = tabw;
    uint32_t* hi = tabw + (nI + 1);
    for (uint32_t k = 0; k < passes; ++k) {
      uint32_t r, lo_, hi_, db, j0, j1;
      if (!segment(k, r, lo_, hi_, db, j0, j1)) break;
      const long long w = __double2ll_rn(weight(r) * g_scale);
      if (w == 0) continue;
      const uint32_t xl = (uint32_t)w, xh = (uint32_t)((unsigned long long)w >> 32);
      walk_flat(r, lo_, hi_, db, j0, j1, [&](uint32_t i) { fix_add_split(lo, hi, i, xl, xh); });
    }
  }

  // G with carry-free limbs (limb_add): lo = tabw[0..nI], hi = tabw[nI+1..2nI+1]; tab zeroed.
  template <typename Wt>
  TOC_D void vecmat_rows_limbs(Wt&& weight, double g_scale, uint32_t L) {
    uint32_t* lo = tabw;
    int32_t* hi = reinterpret_cast<int32_t*>(tabw + (nI + 1));
    for (uint32_t k = 0; k < passes; ++k) {
      uint32_t r, lo_, hi_, db, j0, j1;
      if (!segment(k, r, lo_, hi_, db, j0, j1)) break;
      const long long w = __double2ll_rn(weight(r) * g_scale);
      if (w == 0) continue;
      const int32_t xh = (int32_t)(w >> L);
      const uint32_t xl = (uint32_t)(w - ((long long)xh << L));
      walk_flat(r, lo_, hi_, db, j0, j1, [&](uint32_t i) { limb_add(lo, hi, i, xl, xh); });
    }
  }

  // out[col] = sum over the column's pairs of value * G, in (column, pair) order (G: split words,
  // limbs when L > 0, doubles when L == kGF64):
  // 4 lanes per column, a fixed shuffle tree.  prec / segs from the tree cache (global, in L2):
  // each lane issues its record loads as one batch, so a column costs one L2 round trip.
  template <typename Out>
  TOC_D void column_sums(const typename PairRec<kWide>::T* prec, const uint2* segs, uint32_t n_segs, double g_inv,
                         Out&& out, uint32_t L = 0) const {
    using R = PairRec<kWide>;
    // G lanes per column, up to U record loads in flight per lane; the next round's segment bounds
    // are loaded while this round's records are summed (the rounds are L2-latency bound)
    constexpr uint32_t G = 2, U = 8;
    const uint32_t* lo = tabw;
    const uint32_t* hi = tabw + (nI + 1);
    const uint32_t tid = threadIdx.x, groups = blockDim.x / G, sub = tid % G;
    const uint32_t span = ((n_segs + groups - 1) / groups) * groups;
    uint32_t s = tid / G;
    uint2 sg = s < n_segs ? __ldg(segs + s) : make_uint2(0u, 0u);
    uint32_t end = s < n_segs ? __ldg(&segs[s + 1].x) : 0u;
    for (; s < span; s += groups) {
      const uint32_t sn = s + groups;
      const uint2 sgn = sn < n_segs ? __ldg(segs + sn) : make_uint2(0u, 0u);
      const uint32_t endn = sn < n_segs ? __ldg(&segs[sn + 1].x) : 0u;
      double c = 0.0;
      if (s < n_segs) {
        for (uint32_t q0 = sg.x + sub; q0 < end; q0 += G * U) {
          typename R::T pr[U];
#pragma unroll
          for (uint32_t k = 0; k < U; ++k) pr[k] = q0 + G * k < end ? __ldg(prec + q0 + G * k) : R::none();
#pragma unroll
          for (uint32_t k = 0; k < U; ++k)
            if (q0 + G * k < end) {
              const uint32_t i = R::a(pr[k]) + 1;
              c += uniq[R::b(pr[k])] * (L == kGF64 ? tab[i]
                                        : L ? limb_value(lo[i], (int32_t)hi[i], L, g_inv)
                                            : fix_value(lo[i], hi[i], g_inv));
            }
        }
      }
#pragma unroll
      for (uint32_t o = 1; o < G; o <<= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (s < n_segs && sub == 0) out(sg.y, c);
      sg = sgn;
      end = endn;
    }
  }

  // P1 from the cache's unpacked pair records, interleaved over the threads (coalesced loads,
  // conflict-free stores); up to 8 record loads in flight per thread.
  TOC_D void compute_p1_records(const typename PairRec<kWide>::T* irec, const double* vec) {
    using R = PairRec<kWide>;
    constexpr uint32_t U = 8;
    const uint32_t nth = blockDim.x;
    for (uint32_t i0 = threadIdx.x; i0 < nI; i0 += U * nth) {
      typename R::T r[U];
#pragma unroll
      for (uint32_t k = 0; k < U; ++k) r[k] = i0 + k * nth < nI ? __ldg(irec + i0 + k * nth) : R::none();
#pragma unroll
      for (uint32_t k = 0; k < U; ++k)
        if (i0 + k * nth < nI) tab[i0 + k * nth + 1] = uniq[R::b(r[k])] * vec[R::a(r[k])];
    }
  }

  // out[col_i] += value_i * G[i] for this thread's pairs (fixed point at o_scale).
  TOC_D void scatter_columns(uint32_t* out, double g_inv, double o_scale) {
    if (p0 >= p1) return;
    with_width(m.w_refs, [&]<int W>() {
      SeqReader<W> rd;
      rd.init(blk + m.off_refs, p0);
      for (uint32_t i = p0; i < p1; ++i)
        tab[i + 1] = uniq[rd.next()] * fix_value(tabw[2 * (i + 1)], tabw[2 * (i + 1) + 1], g_inv);
    });
    with_width(m.w_cols, [&]<int W>() {
      SeqReader<W> rd;
      rd.init(blk + m.off_cols, p0);
      for (uint32_t i = p0; i < p1; ++i) {
        const uint32_t c = rd.next();
        const long long g = __double2ll_rn(tab[i + 1] * o_scale);
        if (g) fix_add(out + 2 * c, g);
      }
    });
  }

  // out[col_i] += value_i * G[i] with G and out in fp64 (fallback of scatter_columns).
  TOC_D void scatter_columns_f64(double* out) {
    if (p0 >= p1) return;
    with_width(m.w_refs, [&]<int W>() {
      SeqReader<W> rd;
      rd.init(blk + m.off_refs, p0);
      for (uint32_t i = p0; i < p1; ++i) tab[i + 1] *= uniq[rd.next()];
    });
    with_width(m.w_cols, [&]<int W>() {
      SeqReader<W> rd;
      rd.init(blk + m.off_cols, p0);
      for (uint32_t i = p0; i < p1; ++i) {
        const uint32_t c = rd.next();
        if (tab[i + 1] != 0.0) atomicAdd(out + c, tab[i + 1]);
      }
    });
  }

  // Column c of this batch's first layer, for the thread's pairs (used to visit touched columns).
  template <typename F>
  TOC_D void for_each_pair_column(F&& f) const {
    if (p0 >= p1) return;
    with_width(m.w_cols, [&]<int W>() {
      SeqReader<W> rd;
      rd.init(blk + m.off_cols, p0);
      for (uint32_t i = p0; i < p1; ++i) f(i, rd.next());
    });
  }
};

}  // namespace toc
