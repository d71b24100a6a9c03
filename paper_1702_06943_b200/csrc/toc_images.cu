// toc_images.cu -- MGD over cached step images: a thread-block cluster runs a whole epoch.
//
// Reference: kernels.py:68-77 (the once-only per-batch decode-tree cache), training.py:261-281
// (glm_gradient), :296-316 (apply_update / mgd_step), :336-361 (train: batches fixed, epochs
// iterate them in order).
//
// The reference builds each batch's decode tree C' once and reuses it every epoch.  The device
// equivalent is a per-batch step image, built once per training run, holding everything a step
// reads except w, laid out for the step rather than for storage.  Shared region (every CTA):
//   header    counts, cluster shape, region offsets, sum |y|
//   codes     the code stream D (u16, u32 for wide trees)
//   nodes     (par, key) for EVERY id of C': first-layer id i is (0, i), derived ids as in
//             toc_batch.cuh.  A code's pairs are one uniform loop: visit key, follow par until 0.
//   irec      (column, value ref) per first-layer pair
//   prec      (pair id, value ref) sorted by (column, pair id)  } the column gradient is a
//   segs      (start in prec, column) per distinct column       } fixed-order sum, no atomics
//   uniq      the value index (f64)
// and one part per CTA c of the cluster (rows [c n / C, (c + 1) n / C)):
//   split     per (row, lane) the first code of the lane's range: the S lanes of a row get
//             consecutive code ranges with about equal pair counts (balanced walks)
//   labels    y of the part's rows
//
// With the weight-independent work out of the epoch, a step is the dependency chain
// P1 -> A.w -> s -> s^T.A -> g -> update.  It is bound by shared-memory wavefronts (random
// gathers of P1 and fixed-point atomics into G), so the step is spread over a cluster of C SMs:
// each CTA walks its rows against its own copy of the tables (one TMA multicast per batch), keeps
// a partial G, reduces it to per-column partial sums, and after ONE cluster barrier every CTA
// reads the C partials over DSMEM in rank order and applies the same update to its copy of w.
// The next batch's image lands in a second buffer during the current step.
#include <algorithm>

#include "toc_images.cuh"

#ifndef TOC_IMG_LPC
#define TOC_IMG_LPC 4
#endif

namespace toc {

constexpr uint32_t kImageHeader = 336;

// Header (u32 words unless noted):
//   [0] n_rows [1] n_pairs [2] n_derived [3] n_uniques [4] n_codes [5] n_segs [6] cluster [7] threads
//   f64 at byte 32: sum |y|
//   [10..15] codes, nodes, irec, prec, segs, uniq offsets
//   [16] shared-region bytes [17] image bytes (the next image starts right after) [18] next
//        image's shared-region bytes
//   [20 + 2c], [21 + 2c]: rows and log2 lanes per row of CTA c's part (c < kMaxCluster = 16)
//   [52 + 2c], [53 + 2c]: offset and bytes of CTA c's part in the NEXT image
// so each step finds its own part and the next batch's copy parameters in the image it already
// holds, with no dependent global load on the step's path.
enum { kCodes, kNodes, kIrec, kPrec, kSegs, kUniq };
enum { kHShared = 16, kHTotal = 17, kHNextShared = 18, kHPart = 20, kHNextPart = 52 };

struct ImageLayout {
  uint32_t off[6], shared;        // shared region [0, shared)
  uint32_t part_off, part_bytes;  // the queried CTA's part
  uint32_t r0, nr, lg;            // its rows and log2 lanes per row
  uint32_t off_labels;            // labels within the part
  uint32_t total;
};

// Lanes per row: the largest power of two S <= 32 with 2 S rows <= threads.
TOC_HD uint32_t lanes_lg(uint32_t rows, uint32_t threads) {
  uint32_t lg = 0;
  while (lg < 5 && (2u << lg) * (rows ? rows : 1u) <= threads) ++lg;
  return lg;
}

TOC_HD uint32_t part_row(uint32_t n, uint32_t c, uint32_t C) { return (uint32_t)(((uint64_t)n * c) / C); }

TOC_HD uint32_t part_size(uint32_t nr, uint32_t lg) { return align16(4u * ((nr << lg) + 1u)) + align16(8u * nr); }

// Layout of one batch's image for a cluster of C CTAs of T threads; part fields for CTA `cta`.
// n_segs <= min(|I|, n_cols) distinct columns: that many (+1 sentinel) are reserved.
template <bool kWide>
TOC_HD ImageLayout image_layout(const TocBlockMeta& m, uint32_t n_cols, uint32_t C, uint32_t T, uint32_t cta) {
  ImageLayout L;
  const uint32_t nI = m.n_pairs, segs = (nI < n_cols ? nI : n_cols) + 1u;
  uint32_t o = kImageHeader;
  L.off[kCodes] = o;
  o += align16((kWide ? 4u : 2u) * m.n_codes);
  L.off[kNodes] = o;
  o += align16((kWide ? 8u : 4u) * (1u + nI + m.n_derived));
  L.off[kIrec] = o;
  o += align16(8u * nI);
  L.off[kPrec] = o;
  o += align16(8u * nI);
  L.off[kSegs] = o;
  o += align16(8u * segs);
  L.off[kUniq] = o;
  o += align16(8u * m.n_uniques);
  L.shared = o;
  L.part_off = L.part_bytes = L.r0 = L.nr = L.lg = L.off_labels = 0;
  for (uint32_t c = 0; c < C; ++c) {
    const uint32_t r0 = part_row(m.n_rows, c, C), nr = part_row(m.n_rows, c + 1, C) - r0;
    const uint32_t lg = lanes_lg(nr, T), bytes = part_size(nr, lg);
    if (c == cta) {
      L.part_off = o;
      L.part_bytes = bytes;
      L.r0 = r0;
      L.nr = nr;
      L.lg = lg;
      L.off_labels = align16(4u * ((nr << lg) + 1u));
    }
    o += bytes;
  }
  L.total = o;
  return L;
}

struct ImageArgs {
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  const int64_t* row_base;
  int64_t n_blocks;
  const double* labels;
  uint8_t* images;
  const int64_t* image_off;
  int32_t n_cols, loss;
  double lr;
  double* w;
  uint32_t cluster, threads;  // the epoch kernel's shape, fixed into the images
  uint32_t max_shared, max_part, max_pairs, max_part_rows, max_segs, sort_slots, max_codes;
  long long* trace;  // optional: kTracePoints clock64 stamps per step (CTA 0)
  // Data-parallel epoch with the gradient exchange fused into the kernel (world > 0): each step
  // CTA 0 stores this rank's dense gradient into every rank's receive buffer over NVLink
  // (peer_buf[q] + ((seq0 + t) & 1) * world * m + rank * m), fences, and raises its flag in every rank's
  // flag array (peer_flag[q][rank] = seq0 + t + 1); every CTA then waits for all ranks' flags and
  // applies w -= (lr / gsize[t]) * (sum of the ranks' gradients in rank order).
  double* const* peer_buf;
  uint32_t* const* peer_flag;
  const int32_t* gsize;
  int32_t world, rank;
  uint32_t seq0;
  // Emulated data parallelism (toc_glm_epoch_images_dp_emulated): one launch of `world` clusters
  // on one GPU, cluster r acting as rank r with its own images, metadata and weights.
  const TocDpRank* ranks;
};

// System-scope release store / acquire load of a flag (NVLink peers).
TOC_D void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
TOC_D uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Rebuild each batch's decode tree in shared memory (toc_batch.cuh, the code the relay runs per
// step) and write its image.  Grid-stride over batches; tables, sort keys and per-code lengths fit
// shared memory (host-checked).
template <bool kWide>
__global__ void __launch_bounds__(1024, 1) image_build_kernel(ImageArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  double* s_red = reinterpret_cast<double*>(smem + 160);
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem + kFixedBytes);
  uint16_t* clen = reinterpret_cast<uint16_t*>(smem + kFixedBytes + 8u * a.sort_slots);
  uint8_t* tables = smem + kFixedBytes + 8u * a.sort_slots + align16(2u * a.max_codes);
  const uint32_t tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t m = (uint32_t)a.n_cols, C = a.cluster;
  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const TocBlockMeta mb = a.meta[b];
    const ImageLayout IL = image_layout<kWide>(mb, m, C, a.threads, 0);
    uint8_t* img = a.images + a.image_off[b];
    const uint8_t* blk = a.arena + a.block_off[b];
    __syncthreads();
    Batch<kWide> B;
    B.init(blk, mb, tables);
    B.load_index(s_warp);
    B.build_nodes();
    const uint32_t nI = mb.n_pairs;
    uint32_t npad = 1;
    while (npad < nI) npad <<= 1;
    uint2* irec = reinterpret_cast<uint2*>(img + IL.off[kIrec]);
    for (uint32_t i = tid; i < npad; i += nth) {
      if (i < nI) {
        const uint32_t c = ld_packed(blk + mb.off_cols, i, mb.w_cols);
        irec[i] = make_uint2(c, ld_packed(blk + mb.off_refs, i, mb.w_refs));
        keys[i] = ((unsigned long long)c << 32) | i;
      } else {
        keys[i] = ~0ull;
      }
    }
    const int64_t rb = a.row_base[b];
    double ys = 0.0;
    for (uint32_t r = tid; r < B.n; r += nth) ys += fabs(a.labels[rb + r]);
    double* u = reinterpret_cast<double*>(img + IL.off[kUniq]);
    for (uint32_t i = tid; i < mb.n_uniques; i += nth) u[i] = B.uniq[i];
    __syncthreads();
    B.resolve_keys();
    // bitonic sort of (column, pair id): stable column order for the segmented gradient
    for (uint32_t k = 2; k <= npad; k <<= 1) {
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
    __syncthreads();  // keys sorted, node keys resolved
    // code stream (position j of row r: the par of its derived node, or the row's final code)
    // and each code's length in pairs
    for (uint32_t k = 0; k < B.passes; ++k) {
      uint32_t r, lo, hi, db, j0, j1;
      if (!B.segment(k, r, lo, hi, db, j0, j1)) break;
      for (uint32_t j = j0; j < j1; ++j) {
        const uint32_t c = (j + 1 < hi) ? B.pk.par(db + (j - lo)) : B.last[r];
        if constexpr (kWide) reinterpret_cast<uint32_t*>(img + IL.off[kCodes])[j] = c;
        else reinterpret_cast<uint16_t*>(img + IL.off[kCodes])[j] = (uint16_t)c;
        uint32_t len = 1, x = c;
        while (x > nI) {
          x = B.pk.par(x - 1 - nI);
          ++len;
        }
        clen[j] = (uint16_t)min(len, 65535u);
      }
    }
    const uint32_t T = 1u + nI + mb.n_derived;
    for (uint32_t x = tid; x < T; x += nth) {
      uint32_t par = 0, key = x;
      if (x == 0) key = 0;
      else if (x > nI) B.pk.get(x - 1 - nI, par, key);
      if constexpr (kWide) reinterpret_cast<uint2*>(img + IL.off[kNodes])[x] = make_uint2(par, key);
      else reinterpret_cast<uint32_t*>(img + IL.off[kNodes])[x] = Nodes<false>::pack(par, key);
    }
    uint2* prec = reinterpret_cast<uint2*>(img + IL.off[kPrec]);
    for (uint32_t q = tid; q < nI; q += nth) {
      const uint32_t i = (uint32_t)keys[q];
      prec[q] = make_uint2(i, irec[i].y);
    }
    __syncthreads();  // clen complete
    // parts: the S lanes of each row take consecutive code ranges with ~equal pair counts
    for (uint32_t c = 0; c < C; ++c) {
      const ImageLayout P = image_layout<kWide>(mb, m, C, a.threads, c);
      const uint32_t S = 1u << P.lg;
      uint32_t* split = reinterpret_cast<uint32_t*>(img + P.part_off);
      double* y = reinterpret_cast<double*>(img + P.part_off + P.off_labels);
      for (uint32_t q = tid; q < P.nr; q += nth) {
        const uint32_t r = P.r0 + q, lo = B.rowoff[r], hi = B.rowoff[r + 1];
        y[q] = a.labels[rb + r];
        uint32_t V = 0;
        for (uint32_t j = lo; j < hi; ++j) V += clen[j];
        split[q * S] = lo;
        uint32_t sub = 0, cum = 0;
        for (uint32_t j = lo; j < hi; ++j) {
          const uint32_t want = (uint32_t)(((unsigned long long)S * cum) / (V ? V : 1u));
          while (sub < want) split[q * S + ++sub] = j;
          cum += clen[j];
        }
        while (sub + 1 < S) split[q * S + ++sub] = hi;
      }
      if (tid == 0) split[P.nr * S] = B.rowoff[P.r0 + P.nr];
    }
    if (warp == 0) {  // column segments of the sorted order
      uint2* segs = reinterpret_cast<uint2*>(img + IL.off[kSegs]);
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
        uint32_t* h = reinterpret_cast<uint32_t*>(img);
        h[0] = mb.n_rows;
        h[1] = nI;
        h[2] = mb.n_derived;
        h[3] = mb.n_uniques;
        h[4] = mb.n_codes;
        h[5] = carry;
        h[6] = C;
        h[7] = a.threads;
        for (int k = 0; k < 6; ++k) h[10 + k] = IL.off[k];
        h[kHShared] = IL.shared;
        h[kHTotal] = IL.total;
        for (uint32_t c = 0; c < kMaxCluster; ++c) {
          const ImageLayout P = image_layout<kWide>(mb, m, C, a.threads, c);
          h[kHPart + 2 * c] = c < C ? P.nr : 0u;
          h[kHPart + 2 * c + 1] = c < C ? P.lg : 0u;
        }
        h[kHNextShared] = 0;
        for (uint32_t c = 0; c < 2 * kMaxCluster; ++c) h[kHNextPart + c] = 0;
        if (b + 1 < a.n_blocks) {
          const TocBlockMeta mn = a.meta[b + 1];
          for (uint32_t c = 0; c < C; ++c) {
            const ImageLayout P = image_layout<kWide>(mn, m, C, a.threads, c);
            h[kHNextShared] = P.shared;
            h[kHNextPart + 2 * c] = P.part_off;
            h[kHNextPart + 2 * c + 1] = P.part_bytes;
          }
        }
      }
    }
    const double ysum = block_sum(ys, s_red);
    if (tid == 0) reinterpret_cast<double*>(img)[4] = ysum;
  }
}

// The C CTAs' partials at the offset of p, summed in rank order; loads issued 8 at a time.
TOC_D double sum_partials(const double* p, uint32_t C) {
  double g = 0.0;
  for (uint32_t c0 = 0; c0 < C; c0 += 8) {
    double r[8];
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) r[j] = c0 + j < C ? ld_dsmem(p, c0 + j) : 0.0;
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) g += r[j];
  }
  return g;
}

TOC_D void trace_stamp(const ImageArgs& a, uint32_t cta, int64_t t, int k) {
  if (a.trace && cta == 0 && threadIdx.x == 0) a.trace[t * kTracePoints + k] = clock64();
}

struct NextImage {  // thread 0's view of the batch to fetch next
  const uint8_t* src;
  uint32_t shared, part_off, part_bytes;
};

// Copy parameters of batch 0 (the prologue's only dependent global loads).
template <bool kWide>
TOC_D NextImage first_image(const ImageArgs& a, uint32_t cta) {
  NextImage x;
  const ImageLayout L = image_layout<kWide>(a.meta[0], (uint32_t)a.n_cols, a.cluster, a.threads, cta);
  x.src = a.images + a.image_off[0];
  x.shared = L.shared;
  x.part_off = L.part_off;
  x.part_bytes = L.part_bytes;
  return x;
}

// Arm this CTA's barrier for the image and start the copies into `buf`: the CTA's own part, and
// (rank 0) the shared region multicast to every CTA.
TOC_D void fetch_image(const NextImage& x, uint8_t* buf, uint64_t* mbar, uint32_t cta, uint32_t C) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect(mbar, x.shared + x.part_bytes);
  bulk_copy(buf + x.shared, x.src + x.part_off, x.part_bytes, mbar);
  if (cta == 0) {
    if (C > 1) bulk_multicast(buf, x.src, x.shared, mbar, (uint16_t)((1u << C) - 1u));
    else bulk_copy(buf, x.src, x.shared, mbar);
  }
}

// One epoch (mgd_step, training.py:303-316, for each batch in order) on a cluster of C CTAs.
// Shared memory: fixed | w | P1 | G lo | G hi | z/s | column partials x2 | segment columns |
// image buffer 0 | image buffer 1  (a buffer: shared region, then this CTA's part).
template <bool kWide>
__global__ void __launch_bounds__(1024, 1) epoch_cluster_kernel(ImageArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t cta = cluster_rank(), C = a.cluster;
  if (a.ranks) {  // emulated ranks: this cluster is rank blockIdx.x / C
    const uint32_t r = blockIdx.x / C;
    const TocDpRank rk = a.ranks[r];
    a.images = const_cast<uint8_t*>(rk.images);
    a.image_off = rk.image_off;
    a.meta = rk.meta;
    a.w = rk.w;
    a.rank = (int32_t)r;
  }
  double* s_red = reinterpret_cast<double*>(smem + 160);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 448);
  const uint32_t tid = threadIdx.x, nth = blockDim.x, m = (uint32_t)a.n_cols;
  const uint32_t lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
  uint8_t* p = smem + kFixedBytes;
  double* ws = reinterpret_cast<double*>(p);
  p += align16(8u * m);
  double* p1 = reinterpret_cast<double*>(p);
  p += align16(8u * (a.max_pairs + 1));
  uint32_t* glo = reinterpret_cast<uint32_t*>(p);
  p += align16(4u * (a.max_pairs + 1));
  uint32_t* ghi = reinterpret_cast<uint32_t*>(p);
  p += align16(4u * (a.max_pairs + 1));
  double* srow = reinterpret_cast<double*>(p);
  p += align16(8u * a.max_part_rows);
  double* cpart = reinterpret_cast<double*>(p);  // [2][max_segs] per-column partial sums
  p += align16(16u * a.max_segs);
  uint32_t* segcol = reinterpret_cast<uint32_t*>(p);
  p += align16(4u * a.max_segs);
  const uint32_t buf_bytes = align16(a.max_shared) + align16(a.max_part);
  uint8_t* buf0 = p;
  uint8_t* buf1 = p + buf_bytes;
  for (uint32_t c = tid; c < m; c += nth) ws[c] = a.w[c];
  const uint8_t* src = nullptr;  // thread 0: global address of the current image
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
  }
  cluster_barrier();  // every CTA's barriers exist before any multicast targets them
  if (tid == 0) {
    const NextImage x = first_image<kWide>(a, cta);
    src = x.src;
    TOC_CHECK(x.shared <= a.max_shared && x.part_bytes <= a.max_part);
    fetch_image(x, buf0, &mbar[0], cta, C);
  }
  const bool squared = a.loss == TOC_LOSS_SQUARED;
  uint32_t step_n = 0;
  double step = 0.0;
  for (int64_t t = 0; t < a.n_blocks; ++t) {
    const uint32_t k = (uint32_t)t & 1u;
    const uint8_t* img = k ? buf1 : buf0;
    trace_stamp(a, cta, t, 0);
    mbar_wait_bounded(&mbar[k], (uint32_t)(t >> 1) & 1u);
    trace_stamp(a, cta, t, 1);
    const uint32_t* h = reinterpret_cast<const uint32_t*>(img);
    if (tid == 0 && t + 1 < a.n_blocks) {
      // the other buffer held batch t-1, which every CTA finished before the cluster barrier of
      // step t-1 (the update after it reads only registers, w and partials)
      NextImage x;
      x.src = src + h[kHTotal];
      x.shared = h[kHNextShared];
      x.part_off = h[kHNextPart + 2 * cta];
      x.part_bytes = h[kHNextPart + 2 * cta + 1];
      src = x.src;
      TOC_CHECK(x.shared <= a.max_shared && x.part_bytes <= a.max_part);
      fetch_image(x, k ? buf0 : buf1, &mbar[k ^ 1u], cta, C);
    }
    const uint32_t n = h[0], nI = h[1], n_segs = h[5];
    const double ysum = reinterpret_cast<const double*>(img)[4];
    const uint32_t* ho = h + 10;
    const uint32_t nr = h[kHPart + 2 * cta], lg = h[kHPart + 2 * cta + 1], shared = h[kHShared];
    Nodes<kWide> N;
    N.codes = reinterpret_cast<decltype(N.codes)>(img + ho[kCodes]);
    N.p = reinterpret_cast<decltype(N.p)>(img + ho[kNodes]);
    const uint2* irec = reinterpret_cast<const uint2*>(img + ho[kIrec]);
    const uint2* prec = reinterpret_cast<const uint2*>(img + ho[kPrec]);
    const uint2* segs = reinterpret_cast<const uint2*>(img + ho[kSegs]);
    const double* uniq = reinterpret_cast<const double*>(img + ho[kUniq]);
    const uint32_t* split = reinterpret_cast<const uint32_t*>(img + shared);
    const double* y = reinterpret_cast<const double*>(img + shared + align16(4u * ((nr << lg) + 1u)));
    if (n != step_n) {  // lr / |B| (apply_update, training.py:296-300): all batches but the last share it
      step = a.lr / (double)n;
      step_n = n;
    }
    // P1[i] = value_i * w[col_i] (Algorithm 5, first layer) for every pair; G cleared
#pragma unroll 4
    for (uint32_t i = tid; i < nI; i += nth) {
      const uint2 r = irec[i];
      p1[i + 1] = uniq[r.y] * ws[r.x];
      glo[i + 1] = 0u;
      ghi[i + 1] = 0u;
    }
    const uint32_t S = 1u << lg, RP = nth >> lg, sub = tid & (S - 1u);
    __syncthreads();
    trace_stamp(a, cta, t, 2);
    // z = A.w for this CTA's rows: the S lanes of a row walk their code ranges, then reduce
    const uint32_t nr_up = ((nr + RP - 1) / RP) * RP;
    double bp = 0.0;
    for (uint32_t q = tid >> lg; q < nr_up; q += RP) {
      double part = 0.0;
      if (q < nr) walk_flat(N, split[(q << lg) + sub], split[(q << lg) + sub + 1], [&](uint32_t i) { part += p1[i]; });
      for (uint32_t o = S >> 1; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (q < nr && sub == 0) {  // s = loss'(y, z) (training.py:272-280)
        const double sc = loss_scalar(a.loss, y[q], part);
        srow[q] = sc;
        bp += fabs(sc);
      }
    }
    trace_stamp(a, cta, t, 3);
    if (squared) {  // sum |s| over this CTA's rows bounds its G
      for (uint32_t o = 16; o > 0; o >>= 1) bp += __shfl_xor_sync(0xffffffffu, bp, o);
      if (lane == 0) s_red[warp] = bp;
    }
    __syncthreads();
    trace_stamp(a, cta, t, 4);
    double bound = ysum;  // logistic / hinge: |s| <= |y| (the whole batch bounds any part)
    if (squared) {
      bound = 0.0;
      for (uint32_t w = 0; w < nwarps; ++w) bound += s_red[w];
    }
    // G[i] = sum of s_r over this CTA's occurrences of pair i (vecmat, Algorithm 6), exact fixed
    // point in two carry-free limbs (limb_add; a pair occurs at most once per row, so at most nr adds)
    const uint32_t L = limb_bits(nr);
    const double g_scale = limb_scale(bound, L), g_inv = 1.0 / g_scale;
    for (uint32_t q = tid >> lg; q < nr; q += RP) {
      const long long wr = __double2ll_rn(srow[q] * g_scale);
      if (wr == 0) continue;
      const int32_t xh = (int32_t)(wr >> L);
      const uint32_t xl = (uint32_t)(wr - ((long long)xh << L));
      walk_flat(N, split[(q << lg) + sub], split[(q << lg) + sub + 1],
                [&](uint32_t i) { limb_add(glo, reinterpret_cast<int32_t*>(ghi), i, xl, xh); });
    }
    __syncthreads();
    trace_stamp(a, cta, t, 5);
    // per-column partial sums of value * G: LPC lanes per column, pairs strided over the lanes
    // (up to U record loads in flight per lane), then a fixed shuffle tree (deterministic)
    double* cp = cpart + (size_t)k * a.max_segs;
    constexpr uint32_t LPC = TOC_IMG_LPC, U = 4;
    const uint32_t seg_span = ((n_segs + (nth / LPC) - 1) / (nth / LPC)) * (nth / LPC);
    for (uint32_t sgi = tid / LPC; sgi < seg_span; sgi += nth / LPC) {
      double c = 0.0;
      uint2 sg = make_uint2(0u, 0u);
      if (sgi < n_segs) {
        sg = segs[sgi];
        const uint32_t end = segs[sgi + 1].x;
        for (uint32_t q0 = sg.x + (tid % LPC); q0 < end; q0 += LPC * U) {
          uint2 pr[U];
#pragma unroll
          for (uint32_t u = 0; u < U; ++u) pr[u] = q0 + LPC * u < end ? prec[q0 + LPC * u] : make_uint2(0u, 0u);
#pragma unroll
          for (uint32_t u = 0; u < U; ++u)
            if (q0 + LPC * u < end)
              c += uniq[pr[u].y] * limb_value(glo[pr[u].x + 1], (int32_t)ghi[pr[u].x + 1], L, g_inv);
        }
      }
#pragma unroll
      for (uint32_t o = 1; o < LPC; o <<= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (sgi < n_segs && (tid % LPC) == 0) {
        cp[sgi] = c;
        segcol[sgi] = sg.y;
      }
    }
    cluster_barrier_smem();  // every CTA's partials of step t are complete and visible
    trace_stamp(a, cta, t, 6);
    if (a.world > 0) {  // data parallel: exchange the gradient over NVLink inside the step
      const uint32_t W = (uint32_t)a.world, seq = a.seq0 + (uint32_t)t + 1u;
      double* gl = p1;  // this batch's P1 is dead: dense local gradient scratch [m]
      if (cta == 0) {
        for (uint32_t c = tid; c < m; c += nth) gl[c] = 0.0;
        __syncthreads();
        for (uint32_t sgi = tid; sgi < n_segs; sgi += nth) {
          gl[segcol[sgi]] = sum_partials(cp + sgi, C);  // rank order (as the 1-GPU epoch)
        }
        __syncthreads();
        // receive slot from the global step sequence, so back-to-back epochs alternate slots too
        const size_t slot = ((size_t)((seq - 1u) & 1u) * W + (uint32_t)a.rank) * m;
        for (uint32_t q = 0; q < W; ++q)
          for (uint32_t c = tid; c < m; c += nth) a.peer_buf[q][slot + c] = gl[c];
        __syncthreads();  // the CTA's stores happen before the flag releases (release is cumulative)
        if (tid < W) st_release_sys(a.peer_flag[tid] + a.rank, seq);
      }
      if (tid < W) {  // every CTA: wait for every rank's gradient of step t (bounded: trap, not hang)
        const uint32_t* f = a.peer_flag[a.rank] + tid;
        const long long t0c = clock64();
        while ((int32_t)(ld_acquire_sys(f) - seq) < 0)
          if (clock64() - t0c > (1ll << 34)) __trap();
      }
      __syncthreads();
      const double* recv = a.peer_buf[a.rank] + (size_t)((seq - 1u) & 1u) * W * m;
      const double stp = a.lr / (double)a.gsize[t];
      for (uint32_t c = tid; c < m; c += nth) {
        double g = __ldcv(recv + c);
        for (uint32_t q = 1; q < W; ++q) g += __ldcv(recv + (size_t)q * m + c);  // rank order
        ws[c] = __dsub_rn(ws[c], __dmul_rn(stp, g));
      }
      __syncthreads();
      trace_stamp(a, cta, t, 7);
      continue;
    }
    // g[c] = partials summed in rank order (identical in every CTA), w[c] -= (lr/|B|) g[c]
    // (apply_update, training.py:296-300)
    for (uint32_t sgi = tid; sgi < n_segs; sgi += nth) {
      const double g = sum_partials(cp + sgi, C);  // rank order
      const uint32_t col = segcol[sgi];
      ws[col] = __dsub_rn(ws[col], __dmul_rn(step, g));
    }
    __syncthreads();
    trace_stamp(a, cta, t, 7);
  }
  if (cta == 0)
    for (uint32_t c = tid; c < m; c += nth) a.w[c] = ws[c];
  cluster_barrier();  // no CTA exits while another may still read its partials
}

}  // namespace toc

// ------------------------------------------------------------------------------------------
namespace {

int g_image_threads = 0;  // diagnostic: CTA width of a cluster epoch (0: 512)

int dev_attr(cudaDeviceAttr attr, int fallback) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, attr, dev) != cudaSuccess || v <= 0)
    return fallback;
  return v;
}

struct ImagePlan {
  bool wide, build_ok, epoch_ok;
  uint32_t cluster, threads;
  int build_smem, epoch_smem;
  uint32_t max_shared, max_part, max_pairs, max_part_rows, max_segs, sort_slots, max_codes;
};

// Images for a cluster of C CTAs (1024 threads alone, 512 in a cluster: measured best on config 3,
// profiles/r01/mgd_cluster_sweep.txt).  cluster_req = 0: the
// largest of 8, 4, 2, 1 that leaves every CTA at least 24 rows and fits shared memory.
ImagePlan image_plan(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t cluster_req) {
  ImagePlan P{};
  const int optin = dev_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448);
  for (int64_t b = 0; b < n_blocks; ++b)
    if (1ull + h_meta[b].n_pairs + h_meta[b].n_derived > 65536ull) P.wide = true;
  const uint32_t m = (uint32_t)std::max(n_cols, 0);
  uint32_t max_tables = 0, max_rows = 0;
  for (int64_t b = 0; b < n_blocks; ++b) {
    const TocBlockMeta& mb = h_meta[b];
    max_tables = std::max(max_tables, P.wide ? toc::batch_layout<true>(mb).total : toc::batch_layout<false>(mb).total);
    P.max_pairs = std::max(P.max_pairs, mb.n_pairs);
    P.max_codes = std::max(P.max_codes, mb.n_codes);
    max_rows = std::max(max_rows, mb.n_rows);
    P.max_segs = std::max(P.max_segs, std::min(mb.n_pairs, m) + 1u);
  }
  P.sort_slots = 1;
  while (P.sort_slots < P.max_pairs) P.sort_slots <<= 1;
  const uint64_t build = (uint64_t)toc::kFixedBytes + 8ull * P.sort_slots + toc::align16(2u * P.max_codes) + max_tables;
  P.build_ok = build <= (uint64_t)optin;
  P.build_smem = (int)std::min<uint64_t>(build, INT32_MAX);
  for (uint32_t C : {16u, 8u, 4u, 2u, 1u}) {
    if (cluster_req > 0 && C != (uint32_t)cluster_req) continue;
    if (cluster_req <= 0 && C > 1 && max_rows < 24u * C) continue;
    const uint32_t T = C == 1 ? 1024u : (g_image_threads > 0 ? (uint32_t)g_image_threads : 512u);
    uint32_t max_shared = 0, max_part = 0, max_part_rows = 0;
    for (int64_t b = 0; b < n_blocks; ++b)
      for (uint32_t c = 0; c < C; ++c) {
        const toc::ImageLayout L = P.wide ? toc::image_layout<true>(h_meta[b], m, C, T, c)
                                          : toc::image_layout<false>(h_meta[b], m, C, T, c);
        max_shared = std::max(max_shared, L.shared);
        max_part = std::max(max_part, L.part_bytes);
        max_part_rows = std::max(max_part_rows, L.nr);
      }
    const uint64_t epoch = (uint64_t)toc::kFixedBytes + toc::align16(8u * std::min(m, 1u << 24)) +
                           toc::align16(8u * (P.max_pairs + 1)) + 2ull * toc::align16(4u * (P.max_pairs + 1)) +
                           toc::align16(8u * max_part_rows) + toc::align16(16u * P.max_segs) +
                           toc::align16(4u * P.max_segs) + 2ull * (toc::align16(max_shared) + toc::align16(max_part));
    if (epoch > (uint64_t)optin || m > (1u << 20)) continue;
    P.epoch_ok = P.build_ok;
    P.cluster = C;
    P.threads = T;
    P.epoch_smem = (int)epoch;
    P.max_shared = max_shared;
    P.max_part = max_part;
    P.max_part_rows = max_part_rows;
    break;
  }
  return P;
}

int check_blocks(const TocBlockMeta* h_meta, int64_t n_blocks) {
  for (int64_t b = 0; b < n_blocks; ++b) {
    if (h_meta[b].status != TOC_OK) return h_meta[b].status;
    if (h_meta[b].corrupt) return TOC_E_CORRUPT;
  }
  return TOC_OK;
}

toc::ImageArgs plan_args(const ImagePlan& P, int64_t n_blocks, int32_t n_cols) {
  toc::ImageArgs a{};
  a.n_blocks = n_blocks;
  a.n_cols = n_cols;
  a.cluster = P.cluster;
  a.threads = P.threads;
  a.max_shared = P.max_shared;
  a.max_part = P.max_part;
  a.max_pairs = P.max_pairs;
  a.max_part_rows = P.max_part_rows;
  a.max_segs = P.max_segs;
  a.sort_slots = P.sort_slots;
  a.max_codes = P.max_codes;
  return a;
}

}  // namespace

extern "C" int toc_mgd_set_image_threads(int32_t threads) {
  if (threads != 0 && (threads < 64 || threads > 1024 || (threads & (threads - 1)))) return TOC_E_ARG;
  g_image_threads = threads;
  return TOC_OK;
}

extern "C" int toc_mgd_image_plan(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t cluster_req,
                                  int32_t* cluster, int64_t* h_image_off) {
  if (!h_meta || n_blocks < 0 || !h_image_off || !cluster || n_cols < 0 || cluster_req < 0 ||
      cluster_req > (int32_t)toc::kMaxCluster)
    return TOC_E_ARG;
  if (int rc = check_blocks(h_meta, n_blocks)) return rc;
  const ImagePlan P = image_plan(h_meta, n_blocks, n_cols, cluster_req);
  *cluster = P.epoch_ok ? (int32_t)P.cluster : 0;
  h_image_off[0] = 0;
  for (int64_t b = 0; b < n_blocks; ++b)
    h_image_off[b + 1] =
        h_image_off[b] +
        (!P.epoch_ok ? 0
         : P.wide    ? toc::image_layout<true>(h_meta[b], (uint32_t)n_cols, P.cluster, P.threads, 0).total
                     : toc::image_layout<false>(h_meta[b], (uint32_t)n_cols, P.cluster, P.threads, 0).total);
  return TOC_OK;
}

extern "C" int toc_mgd_build_images(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                    const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                                    int32_t n_cols, int32_t cluster, const double* d_labels, uint8_t* d_images,
                                    const int64_t* d_image_off, void* stream) {
  if (n_blocks <= 0) return n_blocks == 0 ? TOC_OK : TOC_E_ARG;
  if (!h_meta || !d_images || !d_image_off || !d_labels || n_cols < 0 || cluster < 1 ||
      cluster > (int32_t)toc::kMaxCluster)
    return TOC_E_ARG;
  if (int rc = check_blocks(h_meta, n_blocks)) return rc;
  const ImagePlan P = image_plan(h_meta, n_blocks, n_cols, cluster);
  if (!P.epoch_ok) return TOC_E_ARG;
  toc::ImageArgs a = plan_args(P, n_blocks, n_cols);
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.labels = d_labels;
  a.images = d_images;
  a.image_off = d_image_off;
  void* fn = P.wide ? (void*)toc::image_build_kernel<true> : (void*)toc::image_build_kernel<false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, P.build_smem) != cudaSuccess)
    return TOC_E_CUDA;
  void* args[] = {&a};
  const int ctas = (int)std::min<int64_t>(n_blocks, dev_attr(cudaDevAttrMultiProcessorCount, 148));
  return cudaLaunchKernel(fn, dim3(ctas), dim3(1024), args, P.build_smem, (cudaStream_t)stream) == cudaSuccess
             ? TOC_OK
             : TOC_E_CUDA;
}

static int epoch_images_launch(const uint8_t* d_images, const int64_t* d_image_off, const TocBlockMeta* d_meta,
                               const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t cluster,
                               int32_t loss, double lr, double* d_w, long long* d_trace, int32_t world, int32_t rank,
                               double* const* d_peer_buf, uint32_t* const* d_peer_flag, const int32_t* d_gsize,
                               uint32_t seq0, void* stream) {
  if (n_blocks <= 0) return n_blocks == 0 ? TOC_OK : TOC_E_ARG;
  if (!h_meta || !d_meta || !d_images || !d_image_off || !d_w || n_cols < 0 || loss < 0 || loss > 2 ||
      cluster < 1 || cluster > (int32_t)toc::kMaxCluster)
    return TOC_E_ARG;
  const ImagePlan P = image_plan(h_meta, n_blocks, n_cols, cluster);
  if (!P.epoch_ok) return TOC_E_ARG;
  toc::ImageArgs a = plan_args(P, n_blocks, n_cols);
  a.meta = d_meta;
  a.images = const_cast<uint8_t*>(d_images);
  a.image_off = d_image_off;
  a.loss = loss;
  a.lr = lr;
  a.w = d_w;
  a.trace = d_trace;
  if (world > 0) {  // the dense gradient scratch reuses the P1 table
    if (rank < 0 || rank >= world || !d_peer_buf || !d_peer_flag || !d_gsize || n_cols > (int32_t)a.max_pairs + 1)
      return TOC_E_ARG;
    a.world = world;
    a.rank = rank;
    a.peer_buf = d_peer_buf;
    a.peer_flag = d_peer_flag;
    a.gsize = d_gsize;
    a.seq0 = seq0;
  }
  void* fn = P.wide ? (void*)toc::epoch_cluster_kernel<true> : (void*)toc::epoch_cluster_kernel<false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, P.epoch_smem) != cudaSuccess)
    return TOC_E_CUDA;
  if (P.cluster > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return TOC_E_CUDA;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(P.cluster);
  cfg.blockDim = dim3(P.threads);
  cfg.dynamicSmemBytes = (size_t)P.epoch_smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&a};
  return cudaLaunchKernelExC(&cfg, fn, args) == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_glm_epoch_images_traced(const uint8_t* d_images, const int64_t* d_image_off,
                                           const TocBlockMeta* d_meta, const TocBlockMeta* h_meta, int64_t n_blocks,
                                           int32_t n_cols, int32_t cluster, int32_t loss, double lr, double* d_w,
                                           long long* d_trace, void* stream) {
  return epoch_images_launch(d_images, d_image_off, d_meta, h_meta, n_blocks, n_cols, cluster, loss, lr, d_w, d_trace,
                             0, 0, nullptr, nullptr, nullptr, 0, stream);
}

extern "C" int toc_glm_epoch_images(const uint8_t* d_images, const int64_t* d_image_off, const TocBlockMeta* d_meta,
                                    const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t cluster,
                                    int32_t loss, double lr, double* d_w, void* stream) {
  return epoch_images_launch(d_images, d_image_off, d_meta, h_meta, n_blocks, n_cols, cluster, loss, lr, d_w, nullptr,
                             0, 0, nullptr, nullptr, nullptr, 0, stream);
}

extern "C" int toc_glm_epoch_images_dp_emulated(const TocDpRank* d_ranks, const TocBlockMeta* h_meta_all,
                                                int64_t n_blocks, int32_t n_cols, int32_t cluster, int32_t loss,
                                                double lr, int32_t world, double* const* d_peer_buf,
                                                uint32_t* const* d_peer_flag, const int32_t* d_gsize, uint32_t seq0,
                                                void* stream) {
  if (n_blocks <= 0 || world < 1 || !d_ranks || !h_meta_all || !d_peer_buf || !d_peer_flag || !d_gsize ||
      n_cols < 0 || loss < 0 || loss > 2 || cluster < 1 || cluster > (int32_t)toc::kMaxCluster)
    return TOC_E_ARG;
  // the shared-memory plan covers every rank's batches; each rank's images were built for the same
  // shape (cluster, threads, node-id width)
  const ImagePlan P = image_plan(h_meta_all, world * n_blocks, n_cols, cluster);
  if (!P.epoch_ok || n_cols > (int32_t)P.max_pairs + 1) return TOC_E_ARG;
  for (int32_t r = 0; r < world; ++r) {
    const ImagePlan Pr = image_plan(h_meta_all + (int64_t)r * n_blocks, n_blocks, n_cols, cluster);
    if (!Pr.epoch_ok || Pr.wide != P.wide || Pr.threads != P.threads || Pr.cluster != P.cluster) return TOC_E_ARG;
  }
  toc::ImageArgs a = plan_args(P, n_blocks, n_cols);
  a.loss = loss;
  a.lr = lr;
  a.world = world;
  a.peer_buf = d_peer_buf;
  a.peer_flag = d_peer_flag;
  a.gsize = d_gsize;
  a.seq0 = seq0;
  a.ranks = d_ranks;
  void* fn = P.wide ? (void*)toc::epoch_cluster_kernel<true> : (void*)toc::epoch_cluster_kernel<false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, P.epoch_smem) != cudaSuccess)
    return TOC_E_CUDA;
  if (P.cluster > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return TOC_E_CUDA;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(P.cluster * (uint32_t)world);
  cfg.blockDim = dim3(P.threads);
  cfg.dynamicSmemBytes = (size_t)P.epoch_smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeCooperative;  // the ranks spin on each other: all co-resident
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  void* args[] = {&a};
  return cudaLaunchKernelExC(&cfg, fn, args) == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_glm_epoch_images_dp(const uint8_t* d_images, const int64_t* d_image_off, const TocBlockMeta* d_meta,
                                       const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t cluster,
                                       int32_t loss, double lr, double* d_w, int32_t world, int32_t rank,
                                       double* const* d_peer_buf, uint32_t* const* d_peer_flag,
                                       const int32_t* d_gsize, uint32_t seq0, void* stream) {
  if (world < 1) return TOC_E_ARG;
  return epoch_images_launch(d_images, d_image_off, d_meta, h_meta, n_blocks, n_cols, cluster, loss, lr, d_w, nullptr,
                             world, rank, d_peer_buf, d_peer_flag, d_gsize, seq0, stream);
}
