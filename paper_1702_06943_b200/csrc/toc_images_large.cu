// toc_images_large.cu -- MGD epochs for models too wide for shared memory (config 4: 47,236
// weights), on a thread-block cluster over per-CTA part images.
//
// Reference: training.py:261-316 (glm_gradient, apply_update, mgd_step), kernels.py:68-77 (trees
// built once, reused every epoch).  The relay (toc_mgd.cu) runs each step on ONE SM, whose
// critical path at config 4 is gathering ~14 k weights and updating ~10 k of them through L2 (about
// 120 k of its 135 k cycles per step).  Here a step is spread over the C CTAs of a cluster, each
// owning 1/C of the batch's rows, so the gathers run on C SMs:
//   part image (built once per run, per batch and CTA): the CTA's rows' code stream and the part
//   of C' those codes reach, renumbered locally (pairs 1..nP, then derived nodes, node 0 the
//   root), each local pair's column and value, the columns this CTA owns (c mod C) among those the
//   batch touches, and the rows' labels;
//   per step, each CTA: P1 for its pairs from w (global), A.w and the loss scalar on its rows, s^T.A
//   into a fixed-point G, then each pair's contribution value * G added into a global 64-bit
//   fixed-point gradient with a native RED.ADD.U64 (exact, order-independent: deterministic);
//   cluster barrier; each CTA applies w[c] -= (lr/|B|) g[c] for its owned columns and clears them;
//   cluster barrier.
// Logistic and hinge (|s| <= |y| gives the fixed-point scales a priori); squared loss uses the relay.
#include <algorithm>

#include "toc_images.cuh"

namespace toc {

// Part images and their epochs take clusters up to 16 CTAs (sizes above 8 are non-portable:
// the launch opts in with cudaFuncAttributeNonPortableClusterSizeAllowed).
constexpr uint32_t kMaxPartsCluster = 16;

// Part header (64 B): u32 [0] rows [1] pairs nP [2] derived nD [3] codes [4] owned columns
// [5] batch rows; f64 at 24: sum |y| of the batch, at 32: max |value| of the batch; i64 at 40:
// byte offset of the same CTA's part of the NEXT batch relative to this part, u32 at 48: its bytes;
// u32 [13]: the batch's value-index size nU.
constexpr uint32_t kPartHeader = 64;

// Local ids (1 + nP + nD per part), columns and value refs fit 16 bits (toc_mgd_parts_fit checks):
// codes, columns and value refs are u16, node records u32 (parent | key << 16, Nodes<false>), and
// each part carries the batch's value index (nU doubles, header u32 [13]).
struct PartLayout {
  uint32_t off_rowoff, off_codes, off_nodes, off_pcol, off_pref, off_uniq, off_own, off_labels, total;
};

TOC_HD PartLayout part_layout(uint32_t nr, uint32_t nP, uint32_t nD, uint32_t nC, uint32_t n_own, uint32_t C,
                              uint32_t nU) {
  PartLayout L;
  uint32_t o = kPartHeader;
  L.off_rowoff = o;
  o += align16(4u * (nr + 1));
  L.off_codes = o;
  o += align16(2u * nC);
  L.off_nodes = o;
  o += align16(4u * (1u + nP + nD));
  L.off_pcol = o;
  o += align16(2u * nP);
  L.off_pref = o;
  o += align16(2u * nP);
  L.off_uniq = o;
  o += align16(8u * nU);
  L.off_own = o;
  o += align16(2u * n_own);
  L.off_labels = o;
  o += align16(8u * nr);
  L.total = o;
  return L;
}

// Bits of a 32-column word whose column is congruent to o mod C (C divides 32).
TOC_HD uint32_t residue_mask(uint32_t o, uint32_t C) {
  const uint32_t base = C == 1    ? 0xffffffffu
                        : C == 2  ? 0x55555555u
                        : C == 4  ? 0x11111111u
                        : C == 8  ? 0x01010101u
                                  : 0x00010001u;  // C == 16 (cluster sizes are powers of two)
  return base << o;
}

struct LargeArgs {
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  const int64_t* row_base;
  int64_t n_blocks;
  const double* labels;
  int32_t n_cols, cluster;
  int32_t* counts;          // count pass: [n_blocks][C][4] = nP, nD, nC, n_own
  uint8_t* images;          // write pass
  const int64_t* part_off;  // [n_blocks * C + 1]
  uint32_t* scratch;        // per CTA: mark[words] | base[words] | colmark[col words] | rpre[C][col words]
  uint32_t id_words, col_words;
  int32_t batch_smem_budget;
  int64_t slab_bytes;
  uint8_t* slab;
};

template <bool kWide, bool kWrite>
__global__ void __launch_bounds__(1024, 1) large_image_kernel(LargeArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  double* s_red = reinterpret_cast<double*>(smem + 160);
  __shared__ uint32_t s_cnt[4 + kMaxPartsCluster];
  uint8_t* p = smem + kFixedBytes;
  const uint32_t tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
  const uint32_t C = (uint32_t)a.cluster, m = (uint32_t)a.n_cols;
  uint32_t* mark = a.scratch + (int64_t)blockIdx.x * (2 * a.id_words + (1 + kMaxPartsCluster) * a.col_words);
  uint32_t* base = mark + a.id_words;
  uint32_t* colmark = base + a.id_words;
  uint32_t* rpre = colmark + a.col_words;  // per owner: touched owned columns in earlier words
  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const TocBlockMeta mb = a.meta[b];
    if (mb.status != TOC_OK || mb.corrupt) continue;
    uint8_t* tables = batch_layout<kWide>(mb).total <= (uint32_t)a.batch_smem_budget
                          ? p
                          : a.slab + (int64_t)blockIdx.x * a.slab_bytes;
    __syncthreads();
    Batch<kWide> B;
    const uint8_t* blk = a.arena + a.block_off[b];
    B.init(blk, mb, tables);
    B.load_index(s_warp);
    B.build_nodes();
    const uint32_t nI = B.nI, T = 1u + nI + mb.n_derived, n = B.n;
    for (uint32_t w = tid; w < (m + 31) / 32; w += nth) colmark[w] = 0u;
    if (tid < kMaxPartsCluster) s_cnt[4 + tid] = 0u;
    const int64_t rb = a.row_base[b];
    double ys = 0.0;
    for (uint32_t r = tid; r < n; r += nth) ys += fabs(a.labels[rb + r]);
    __syncthreads();
    B.resolve_keys();
    // the batch's touched columns, each owned by CTA (column mod C)
    for (uint32_t i = tid; i < nI; i += nth) {
      const uint32_t c = ld_packed(blk + mb.off_cols, i, mb.w_cols), bit = 1u << (c & 31);
      if (atomicOr(colmark + (c >> 5), bit) & bit) continue;
      atomicAdd(&s_cnt[4 + c % C], 1u);
    }
    const double vmax = block_max_d(B.vmax, s_red);
    const double ysum = block_sum(ys, s_red);  // barriers: the key pass and column marks are done
    const uint32_t cw = (m + 31) / 32;
    // the rank of a touched column in its owner's ascending own list
    auto own_rank = [&](uint32_t col) {
      const uint32_t o = col % C, w = col >> 5, bit = col & 31;
      return __ldcg(rpre + o * cw + w) + __popc(__ldcg(colmark + w) & residue_mask(o, C) & ((1u << bit) - 1u));
    };
    if (kWrite) {  // own lists in ascending column order (deterministic ranks)
      if (tid < C) {
        uint32_t acc = 0;
        const uint32_t mk = residue_mask(tid, C);
        for (uint32_t w = 0; w < cw; ++w) {
          rpre[tid * cw + w] = acc;
          acc += __popc(__ldcg(colmark + w) & mk);
        }
      }
      __syncthreads();
      for (uint32_t w = tid; w < cw; w += nth) {
        uint32_t bits = __ldcg(colmark + w);
        while (bits) {
          const uint32_t col = w * 32 + (__ffs(bits) - 1), o = col % C;
          bits &= bits - 1u;
          const uint32_t* h = reinterpret_cast<const uint32_t*>(a.counts + (b * C + o) * 4);
          const uint32_t pr0 = (uint32_t)(((uint64_t)n * o) / C), pr1 = (uint32_t)(((uint64_t)n * (o + 1)) / C);
          const PartLayout PL = part_layout(pr1 - pr0, h[0], h[1], h[2], h[3], C, mb.n_uniques);
          reinterpret_cast<uint16_t*>(a.images + a.part_off[b * C + o] + PL.off_own)[own_rank(col)] = (uint16_t)col;
        }
      }
    }
    for (uint32_t part = 0; part < C; ++part) {
      const uint32_t r0 = (uint32_t)(((uint64_t)n * part) / C), r1 = (uint32_t)(((uint64_t)n * (part + 1)) / C);
      const uint32_t q0 = B.rowoff[r0], q1 = B.rowoff[r1];
      for (uint32_t w = tid; w < a.id_words; w += nth) mark[w] = 0u;
      __syncthreads();
      // the nodes the part's codes reach: every chain node, its key pair, and the final pair
      auto mark_id = [&](uint32_t x) { atomicOr(mark + (x >> 5), 1u << (x & 31)); };
      for (uint32_t k = 0; k < B.passes; ++k) {
        uint32_t r, lo, hi, db, j0, j1;
        if (!B.segment(k, r, lo, hi, db, j0, j1)) break;
        if (r < r0 || r >= r1) continue;
        for (uint32_t j = j0; j < j1; ++j) {
          uint32_t x = (j + 1 < hi) ? B.pk.par(db + (j - lo)) : B.last[r];
          while (x > nI) {
            mark_id(x);
            uint32_t par, key;
            B.pk.get(x - 1 - nI, par, key);
            mark_id(key);
            x = par;
          }
          mark_id(x);
        }
      }
      __syncthreads();
      // local id of a marked id x = 1 + (marked ids below x): word prefix counts
      uint32_t carry = 0;
      for (uint32_t w0 = 0; w0 < a.id_words; w0 += nth) {
        const uint32_t w = w0 + tid;
        const uint32_t v = w < a.id_words ? __popc(__ldcg(mark + w)) : 0u;  // set by L2 atomics
        const uint32_t xs = warp_excl_scan(v, lane);
        if (lane == 31) s_warp[warp] = xs + v;
        __syncthreads();
        if (warp == 0) {
          const uint32_t t = lane < nwarps ? s_warp[lane] : 0u;
          const uint32_t ex = warp_excl_scan(t, lane);
          if (lane < nwarps) s_warp[lane] = ex;
          if (lane == 31) s_warp[32] = ex + t;
        }
        __syncthreads();
        if (w < a.id_words) base[w] = carry + s_warp[warp] + xs;
        carry += s_warp[32];
        __syncthreads();
      }
      const uint32_t total = carry;
      // marked first-layer ids (<= nI): all ranks below those of derived ids
      uint32_t nP = 0;
      {
        const uint32_t wI = (nI + 1) >> 5, rem = (nI + 1) & 31;  // ids 0..nI
        uint32_t cnt = (wI < a.id_words ? base[wI] : total);
        if (rem && wI < a.id_words) cnt += __popc(__ldcg(mark + wI) & ((1u << rem) - 1u));
        nP = cnt;
      }
      const uint32_t nD = total - nP, nC = q1 - q0;
      if (!kWrite) {
        if (tid == 0) {
          int32_t* cn = a.counts + (b * C + part) * 4;
          cn[0] = (int32_t)nP;
          cn[1] = (int32_t)nD;
          cn[2] = (int32_t)nC;
          cn[3] = (int32_t)s_cnt[4 + part];
        }
        __syncthreads();
        continue;
      }
      auto lid = [&](uint32_t x) -> uint32_t {
        return 1u + base[x >> 5] + __popc(__ldcg(mark + (x >> 5)) & ((1u << (x & 31)) - 1u));
      };
      const int32_t* cn = a.counts + (b * C + part) * 4;
      const uint32_t n_own = (uint32_t)cn[3];
      const PartLayout L = part_layout(r1 - r0, nP, nD, nC, n_own, C, mb.n_uniques);
      uint8_t* img = a.images + a.part_off[b * C + part];
      uint32_t* rowoff = reinterpret_cast<uint32_t*>(img + L.off_rowoff);
      uint16_t* codes = reinterpret_cast<uint16_t*>(img + L.off_codes);
      uint32_t* nodes = reinterpret_cast<uint32_t*>(img + L.off_nodes);
      uint16_t* pcol = reinterpret_cast<uint16_t*>(img + L.off_pcol);
      uint16_t* pref = reinterpret_cast<uint16_t*>(img + L.off_pref);
      double* puq = reinterpret_cast<double*>(img + L.off_uniq);
      for (uint32_t i = tid; i < mb.n_uniques; i += nth) puq[i] = B.uniq[i];
      double* y = reinterpret_cast<double*>(img + L.off_labels);
      for (uint32_t r = r0 + tid; r <= r1; r += nth) rowoff[r - r0] = B.rowoff[r] - q0;
      for (uint32_t r = r0 + tid; r < r1; r += nth) y[r - r0] = a.labels[rb + r];
      for (uint32_t k = 0; k < B.passes; ++k) {
        uint32_t r, lo, hi, db, j0, j1;
        if (!B.segment(k, r, lo, hi, db, j0, j1)) break;
        if (r < r0 || r >= r1) continue;
        for (uint32_t j = j0; j < j1; ++j)
          codes[j - q0] = (uint16_t)lid((j + 1 < hi) ? B.pk.par(db + (j - lo)) : B.last[r]);
      }
      if (tid == 0) nodes[0] = 0u;
      for (uint32_t x = 1 + tid; x < T; x += nth) {
        if (!(__ldcg(mark + (x >> 5)) & (1u << (x & 31)))) continue;
        const uint32_t l = lid(x);
        if (x <= nI) {
          nodes[l] = Nodes<false>::pack(0u, l);
          pcol[l - 1] = (uint16_t)ld_packed(blk + mb.off_cols, x - 1, mb.w_cols);
          pref[l - 1] = (uint16_t)ld_packed(blk + mb.off_refs, x - 1, mb.w_refs);
        } else {
          uint32_t par, key;
          B.pk.get(x - 1 - nI, par, key);
          nodes[l] = Nodes<false>::pack(lid(par), lid(key));
        }
      }
      if (tid == 0) {
        uint32_t* h = reinterpret_cast<uint32_t*>(img);
        h[0] = r1 - r0;
        h[1] = nP;
        h[2] = nD;
        h[3] = nC;
        h[4] = n_own;
        h[5] = n;
        h[13] = mb.n_uniques;
        reinterpret_cast<double*>(img)[3] = ysum;
        reinterpret_cast<double*>(img)[4] = vmax;
        const int64_t here = a.part_off[b * C + part];
        int64_t* nx = reinterpret_cast<int64_t*>(img + 40);
        if (b + 1 < a.n_blocks) {
          nx[0] = a.part_off[(b + 1) * C + part] - here;
          h[12] = (uint32_t)(a.part_off[(b + 1) * C + part + 1] - a.part_off[(b + 1) * C + part]);
        } else {
          nx[0] = 0;
          h[12] = 0u;
        }
      }
      __syncthreads();
    }
  }
}

struct LargeEpochArgs {
  const uint8_t* images;
  const int64_t* part_off;  // [n_blocks * C + 1]
  int64_t n_blocks;
  int32_t n_cols, loss, cluster;
  double lr;
  double* w;                 // n_cols, global
  unsigned long long* gacc;  // n_cols, zero between steps
  uint32_t max_part, max_pairs, max_rows;
  int64_t t0, t1;            // steps [t0, t1) of the epoch
  double* grad_out;          // gradient-only mode (data-parallel step): the summed gradient of the
                             // batch into grad_out[touched columns] instead of the update
};

// Phase trace (tools/mgd_bench.py, toc_mgd_parts_set_trace): when set, CTA 0 of the cluster stamps
// clock64 at 7 points of each step: start, part landed, P1, A.w + loss, s^T.A, gradient added +
// cluster barrier, update + cluster barrier.
__constant__ long long* g_parts_trace = nullptr;
#define parts_stamp(t, k) \
  if (g_parts_trace && cluster_rank() == 0 && tid == 0) g_parts_trace[((t) - a.t0) * 8 + (k)] = clock64()

// One epoch on a cluster of C CTAs; w and the fixed-point gradient live in global memory.
// Shared memory: fixed | P1 | G lo | G hi | s | part buffer 0 | part buffer 1.
__global__ void __launch_bounds__(1024, 1) epoch_large_kernel(LargeEpochArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 448);
  const uint32_t cta = cluster_rank();
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  uint8_t* p = smem + kFixedBytes;
  double* p1 = reinterpret_cast<double*>(p);
  p += align16(8u * (a.max_pairs + 1));
  uint32_t* glo = reinterpret_cast<uint32_t*>(p);
  p += align16(4u * (a.max_pairs + 1));
  uint32_t* ghi = reinterpret_cast<uint32_t*>(p);
  p += align16(4u * (a.max_pairs + 1));
  double* srow = reinterpret_cast<double*>(p);
  p += align16(8u * a.max_rows);
  uint8_t* buf0 = p;
  uint8_t* buf1 = p + a.max_part;
  const uint8_t* src = a.images + a.part_off[a.t0 * a.cluster + cta];  // thread 0: the current part
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    const uint32_t bytes = (uint32_t)(a.part_off[a.t0 * a.cluster + cta + 1] - a.part_off[a.t0 * a.cluster + cta]);
    TOC_CHECK(bytes <= a.max_part);
    mbar_expect(&mbar[0], bytes);
    bulk_copy(buf0, src, bytes, &mbar[0]);
  }
  __syncthreads();
  uint32_t step_n = 0;
  double step = 0.0;
  for (int64_t t = a.t0; t < a.t1; ++t) {
    parts_stamp(t, 0);
    const uint32_t k = (uint32_t)(t - a.t0) & 1u;
    const uint8_t* img = k ? buf1 : buf0;
    mbar_wait_bounded(&mbar[k], (uint32_t)((t - a.t0) >> 1) & 1u);
    parts_stamp(t, 1);
    const uint32_t* h = reinterpret_cast<const uint32_t*>(img);
    if (tid == 0 && t + 1 < a.t1) {  // every thread is past step t-1: the other buffer is free
      const int64_t d = *reinterpret_cast<const int64_t*>(img + 40);
      const uint32_t bytes = h[12];
      src += d;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&mbar[k ^ 1u], bytes);
      bulk_copy(k ? buf0 : buf1, src, bytes, &mbar[k ^ 1u]);
    }
    const uint32_t nr = h[0], nP = h[1], nD = h[2], nC = h[3], n_own = h[4], n = h[5];
    const double ysum = reinterpret_cast<const double*>(img)[3], vmax = reinterpret_cast<const double*>(img)[4];
    const PartLayout L = part_layout(nr, nP, nD, nC, n_own, (uint32_t)a.cluster, h[13]);
    const uint32_t* rowoff = reinterpret_cast<const uint32_t*>(img + L.off_rowoff);
    Nodes<false> N;
    N.codes = reinterpret_cast<const uint16_t*>(img + L.off_codes);
    N.p = reinterpret_cast<const uint32_t*>(img + L.off_nodes);
    const uint16_t* pcol = reinterpret_cast<const uint16_t*>(img + L.off_pcol);
    const uint16_t* pref = reinterpret_cast<const uint16_t*>(img + L.off_pref);
    const double* puq = reinterpret_cast<const double*>(img + L.off_uniq);
    const uint16_t* own = reinterpret_cast<const uint16_t*>(img + L.off_own);
    const double* y = reinterpret_cast<const double*>(img + L.off_labels);
    if (n != step_n) {
      step = a.lr / (double)n;
      step_n = n;
    }
    // P1 for this CTA's pairs from the current weights (global; updated by every CTA of the cluster):
    // a thread's weight gathers (L2 round trips) are all in flight at once
    for (uint32_t i0 = tid; i0 < nP; i0 += 4 * nth) {
      uint32_t col[4];
      double wv[4];
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) col[u] = i0 + u * nth < nP ? pcol[i0 + u * nth] : 0u;
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) wv[u] = i0 + u * nth < nP ? __ldcg(a.w + col[u]) : 0.0;
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u)
        if (i0 + u * nth < nP) {
          const uint32_t i = i0 + u * nth;
          p1[i + 1] = puq[pref[i]] * wv[u];
          glo[i + 1] = 0u;
          ghi[i + 1] = 0u;
        }
    }
    uint32_t lg = 0;
    while (lg < 5 && (2u << lg) * (nr ? nr : 1u) <= nth) ++lg;
    const uint32_t S = 1u << lg, RP = nth >> lg, sub = tid & (S - 1u);
    __syncthreads();
    parts_stamp(t, 2);
    // z = A.w and s = loss'(y, z) (training.py:272-280) for this CTA's rows
    const uint32_t nr_up = ((nr + RP - 1) / RP) * RP;
    for (uint32_t q = tid >> lg; q < nr_up; q += RP) {
      double part = 0.0;
      if (q < nr) {
        const uint32_t lo = rowoff[q], len = rowoff[q + 1] - lo;
        walk_flat(N, lo + ((len * sub) >> lg), lo + ((len * (sub + 1)) >> lg), [&](uint32_t i) { part += p1[i]; });
      }
      for (uint32_t o = S >> 1; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (q < nr && sub == 0) srow[q] = loss_scalar(a.loss, y[q], part);
    }
    __syncthreads();
    parts_stamp(t, 3);
    double g_scale, g_inv, o_scale, o_inv;
    fix_scales(ysum, g_scale, g_inv);  // |s| <= |y| (logistic, hinge)
    fix_scales(ysum * vmax, o_scale, o_inv);
    // G[i] = sum of s_r over this CTA's occurrences of local pair i, fixed point
    for (uint32_t q = tid >> lg; q < nr; q += RP) {
      const long long wr = __double2ll_rn(srow[q] * g_scale);
      if (wr == 0) continue;
      const uint32_t lo = rowoff[q], len = rowoff[q + 1] - lo;
      const uint32_t xl = (uint32_t)wr, xh = (uint32_t)((unsigned long long)wr >> 32);
      walk_flat(N, lo + ((len * sub) >> lg), lo + ((len * (sub + 1)) >> lg),
                [&](uint32_t i) { fix_add_pair(glo, ghi, i, xl, xh); });
    }
    __syncthreads();
    parts_stamp(t, 4);
    // value * G per pair into the global fixed-point gradient: integer adds, order-independent
    for (uint32_t i = tid; i < nP; i += nth) {
      const double c = puq[pref[i]] * fix_value(glo[i + 1], ghi[i + 1], g_inv);
      const long long f = __double2ll_rn(c * o_scale);
      if (f) atomicAdd(a.gacc + pcol[i], (unsigned long long)f);
    }
    cluster_barrier();  // every CTA's contributions are in the gradient
    parts_stamp(t, 5);
    if (a.grad_out) {  // data-parallel step: hand the summed gradient to the all-reduce
      for (uint32_t o = tid; o < n_own; o += nth) {
        const uint32_t c = own[o];
        const unsigned long long f = __ldcg(a.gacc + c);
        a.gacc[c] = 0ull;
        a.grad_out[c] = (double)(long long)f * o_inv;
      }
      continue;  // (one step per launch: nothing reads the weights after this)
    }
    // apply_update (training.py:296-300) for the columns this CTA owns, then clear them
    for (uint32_t o = tid; o < n_own; o += nth) {
      const uint32_t c = own[o];
      const unsigned long long f = __ldcg(a.gacc + c);
      if (f) {
        a.gacc[c] = 0ull;
        a.w[c] = __dsub_rn(__ldcg(a.w + c), __dmul_rn(step, (double)(long long)f * o_inv));
      }
    }
    cluster_barrier();  // the weights of step t are final before step t+1 reads them
    parts_stamp(t, 6);
  }
}


}  // namespace toc

// ------------------------------------------------------------------------------------------
namespace {

int la_attr(cudaDeviceAttr attr, int fallback) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, attr, dev) != cudaSuccess || v <= 0)
    return fallback;
  return v;
}

struct LargePlan {
  bool wide;
  int build_smem;
  int32_t budget;
  uint32_t id_words, col_words, max_tables;
  int64_t slab;
};

LargePlan large_plan(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols) {
  LargePlan P{};
  uint64_t maxT = 1;
  for (int64_t b = 0; b < n_blocks; ++b) {
    const uint64_t T = 1ull + h_meta[b].n_pairs + h_meta[b].n_derived;
    if (T > 65536ull) P.wide = true;
    maxT = std::max(maxT, T);
  }
  for (int64_t b = 0; b < n_blocks; ++b)
    P.max_tables = std::max(P.max_tables, P.wide ? toc::batch_layout<true>(h_meta[b]).total
                                                 : toc::batch_layout<false>(h_meta[b]).total);
  const int optin = la_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448);
  P.id_words = (uint32_t)((maxT + 31) / 32);
  P.col_words = (uint32_t)((std::max(n_cols, 1) + 31) / 32);
  const uint32_t avail = (uint32_t)optin - toc::kFixedBytes;
  P.budget = (int32_t)std::min(P.max_tables, avail);
  P.build_smem = (int)(toc::kFixedBytes + (uint32_t)P.budget);
  P.slab = P.max_tables > avail ? (int64_t)toc::align16(P.max_tables) : 0;
  return P;
}

int large_launch(const toc::LargeArgs& a0, const LargePlan& P, bool write, void* d_scratch, cudaStream_t s) {
  toc::LargeArgs a = a0;
  const int sms = la_attr(cudaDevAttrMultiProcessorCount, 148);
  const int ctas = (int)std::min<int64_t>(a.n_blocks, sms);
  a.scratch = reinterpret_cast<uint32_t*>(d_scratch);
  a.id_words = P.id_words;
  a.col_words = P.col_words;
  a.batch_smem_budget = P.budget;
  a.slab_bytes = P.slab;
  a.slab = reinterpret_cast<uint8_t*>(d_scratch) + (int64_t)ctas * 4 * (2 * P.id_words + (1 + toc::kMaxPartsCluster) * P.col_words);
  void* fn = P.wide ? (write ? (void*)toc::large_image_kernel<true, true> : (void*)toc::large_image_kernel<true, false>)
                    : (write ? (void*)toc::large_image_kernel<false, true> : (void*)toc::large_image_kernel<false, false>);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, P.build_smem) != cudaSuccess)
    return TOC_E_CUDA;
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3(ctas), dim3(1024), args, P.build_smem, s) == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

}  // namespace

extern "C" int toc_mgd_parts_scratch(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int64_t* bytes) {
  if (!h_meta || n_blocks < 0 || !bytes) return TOC_E_ARG;
  const LargePlan P = large_plan(h_meta, n_blocks, n_cols);
  const int sms = la_attr(cudaDevAttrMultiProcessorCount, 148);
  const int64_t ctas = std::min<int64_t>(std::max<int64_t>(n_blocks, 1), sms);
  *bytes = ctas * 4 * (2ll * P.id_words + (1 + toc::kMaxPartsCluster) * P.col_words) + ctas * P.slab + 16;
  return TOC_OK;
}

extern "C" int toc_mgd_parts_count(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                   const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                                   int32_t n_cols, int32_t cluster, const double* d_labels, int32_t* d_counts,
                                   void* d_scratch, void* stream) {
  if (n_blocks <= 0) return n_blocks == 0 ? TOC_OK : TOC_E_ARG;
  if (!h_meta || !d_counts || !d_scratch || !d_labels || cluster < 1 || cluster > (int32_t)toc::kMaxPartsCluster || (cluster & (cluster - 1)))
    return TOC_E_ARG;
  for (int64_t b = 0; b < n_blocks; ++b)
    if (h_meta[b].status != TOC_OK || h_meta[b].corrupt) return h_meta[b].status ? h_meta[b].status : TOC_E_CORRUPT;
  toc::LargeArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.n_blocks = n_blocks;
  a.labels = d_labels;
  a.n_cols = n_cols;
  a.cluster = cluster;
  a.counts = d_counts;
  return large_launch(a, large_plan(h_meta, n_blocks, n_cols), false, d_scratch, (cudaStream_t)stream);
}

extern "C" int toc_mgd_parts_offsets(const TocBlockMeta* h_meta, const int32_t* h_counts, int64_t n_blocks,
                                     int32_t cluster, int64_t* h_part_off, int64_t* max_part) {
  if (!h_meta || !h_counts || !h_part_off || !max_part || n_blocks < 0 || cluster < 1) return TOC_E_ARG;
  int64_t o = 0, mx = 0;
  for (int64_t b = 0; b < n_blocks; ++b)
    for (int32_t c = 0; c < cluster; ++c) {
      const uint32_t n = h_meta[b].n_rows;
      const uint32_t r0 = (uint32_t)(((uint64_t)n * c) / cluster), r1 = (uint32_t)(((uint64_t)n * (c + 1)) / cluster);
      const int32_t* cn = h_counts + (b * cluster + c) * 4;
      const uint32_t sz =
          toc::part_layout(r1 - r0, (uint32_t)cn[0], (uint32_t)cn[1], (uint32_t)cn[2], (uint32_t)cn[3], (uint32_t)cluster,
                           h_meta[b].n_uniques)
              .total;
      h_part_off[b * cluster + c] = o;
      o += sz;
      mx = std::max<int64_t>(mx, sz);
    }
  h_part_off[n_blocks * cluster] = o;
  *max_part = mx;
  return TOC_OK;
}

extern "C" int toc_mgd_parts_build(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                   const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                                   int32_t n_cols, int32_t cluster, const double* d_labels, const int32_t* d_counts,
                                   const int64_t* d_part_off, uint8_t* d_images, void* d_scratch, void* stream) {
  if (n_blocks <= 0) return n_blocks == 0 ? TOC_OK : TOC_E_ARG;
  if (!h_meta || !d_counts || !d_part_off || !d_images || !d_scratch || !d_labels || cluster < 1 ||
      cluster > (int32_t)toc::kMaxPartsCluster || (cluster & (cluster - 1)))
    return TOC_E_ARG;
  toc::LargeArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.n_blocks = n_blocks;
  a.labels = d_labels;
  a.n_cols = n_cols;
  a.cluster = cluster;
  a.counts = const_cast<int32_t*>(d_counts);
  a.images = d_images;
  a.part_off = d_part_off;
  return large_launch(a, large_plan(h_meta, n_blocks, n_cols), true, d_scratch, (cudaStream_t)stream);
}

namespace {
uint64_t parts_smem(const TocBlockMeta* h_meta, const int32_t* h_counts, int64_t n_blocks, int32_t cluster,
                    int64_t max_part, uint32_t& max_pairs, uint32_t& max_rows) {
  max_pairs = max_rows = 0;
  for (int64_t b = 0; b < n_blocks; ++b)
    for (int32_t c = 0; c < cluster; ++c) {
      const uint32_t n = h_meta[b].n_rows;
      max_rows = std::max(max_rows, (uint32_t)(((uint64_t)n * (c + 1)) / cluster - ((uint64_t)n * c) / cluster));
      max_pairs = std::max(max_pairs, (uint32_t)h_counts[(b * cluster + c) * 4]);
    }
  return (uint64_t)toc::kFixedBytes + toc::align16(8u * (max_pairs + 1)) + 2ull * toc::align16(4u * (max_pairs + 1)) +
         toc::align16(8u * max_rows) + 2ull * toc::align16((uint32_t)max_part);
}
}  // namespace

extern "C" int toc_mgd_parts_fit(const TocBlockMeta* h_meta, const int32_t* h_counts, int64_t n_blocks,
                                 int32_t cluster, int64_t max_part, int32_t* fits) {
  if (!h_meta || !h_counts || !fits || n_blocks < 0 || cluster < 1) return TOC_E_ARG;
  uint32_t mp, mr;
  *fits = parts_smem(h_meta, h_counts, n_blocks, cluster, max_part, mp, mr) <=
                  (uint64_t)la_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448)
              ? 1
              : 0;
  for (int64_t b = 0; b < n_blocks && *fits; ++b) {  // 16-bit local ids and columns (PartLayout)
    if (h_meta[b].n_cols > 65536u || h_meta[b].n_uniques > 65536u) *fits = 0;
    for (int32_t c = 0; c < cluster; ++c) {
      const int32_t* cn = h_counts + (b * cluster + c) * 4;
      if (1ll + cn[0] + cn[1] > 65535ll) *fits = 0;
    }
  }
  return TOC_OK;
}

static int parts_launch(const uint8_t* d_images, const int64_t* d_part_off, const TocBlockMeta* h_meta,
                        const int32_t* h_counts, int64_t n_blocks, int32_t n_cols, int32_t cluster, int32_t loss,
                        double lr, double* d_w, unsigned long long* d_gacc, int64_t max_part, int64_t t0, int64_t t1,
                        double* d_grad, void* stream) {
  if (n_blocks <= 0) return n_blocks == 0 ? TOC_OK : TOC_E_ARG;
  if (!d_images || !d_part_off || !h_meta || !h_counts || !d_w || !d_gacc || cluster < 1 ||
      cluster > (int32_t)toc::kMaxPartsCluster || (cluster & (cluster - 1)) || (loss != TOC_LOSS_LOGISTIC && loss != TOC_LOSS_HINGE))
    return TOC_E_ARG;
  uint32_t max_pairs = 0, max_rows = 0;
  const uint32_t mp = toc::align16((uint32_t)max_part);
  const uint64_t smem = parts_smem(h_meta, h_counts, n_blocks, cluster, max_part, max_pairs, max_rows);
  if (smem > (uint64_t)la_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448)) return TOC_E_ARG;
  toc::LargeEpochArgs a{};
  a.images = d_images;
  a.part_off = d_part_off;
  a.n_blocks = n_blocks;
  a.n_cols = n_cols;
  a.loss = loss;
  a.cluster = cluster;
  a.lr = lr;
  a.w = d_w;
  a.gacc = d_gacc;
  a.max_part = mp;
  a.max_pairs = max_pairs;
  a.max_rows = max_rows;
  a.t0 = t0;
  a.t1 = t1;
  a.grad_out = d_grad;
  if (cluster > 8 && cudaFuncSetAttribute(toc::epoch_large_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                          cudaSuccess)
    return TOC_E_CUDA;
  if (cudaFuncSetAttribute(toc::epoch_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return TOC_E_CUDA;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&a};
  return cudaLaunchKernelExC(&cfg, (void*)toc::epoch_large_kernel, args) == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_glm_epoch_parts(const uint8_t* d_images, const int64_t* d_part_off, const TocBlockMeta* h_meta,
                                   const int32_t* h_counts, int64_t n_blocks, int32_t n_cols, int32_t cluster,
                                   int32_t loss, double lr, double* d_w, unsigned long long* d_gacc, int64_t max_part,
                                   void* stream) {
  return parts_launch(d_images, d_part_off, h_meta, h_counts, n_blocks, n_cols, cluster, loss, lr, d_w, d_gacc,
                      max_part, 0, n_blocks, nullptr, stream);
}

extern "C" int toc_glm_grad_parts(const uint8_t* d_images, const int64_t* d_part_off, const TocBlockMeta* h_meta,
                                  const int32_t* h_counts, int64_t n_blocks, int32_t n_cols, int32_t cluster,
                                  int32_t loss, int64_t step, const double* d_w, unsigned long long* d_gacc,
                                  double* d_grad, int64_t max_part, void* stream) {
  if (step < 0 || step >= n_blocks || !d_grad) return TOC_E_ARG;
  return parts_launch(d_images, d_part_off, h_meta, h_counts, n_blocks, n_cols, cluster, loss, 0.0,
                      const_cast<double*>(d_w), d_gacc, max_part, step, step + 1, d_grad, stream);
}

extern "C" int toc_mgd_parts_set_trace(long long* d_trace) {
  return cudaMemcpyToSymbol(toc::g_parts_trace, &d_trace, sizeof d_trace) == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_mgd_parts_cluster_max(int32_t* cluster) {
  if (!cluster) return TOC_E_ARG;
  const int optin = la_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448);
  if (cudaFuncSetAttribute(toc::epoch_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin) !=
          cudaSuccess ||
      cudaFuncSetAttribute(toc::epoch_large_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return TOC_E_CUDA;
  for (int32_t c = (int32_t)toc::kMaxPartsCluster; c >= 1; c >>= 1) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = (size_t)optin;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void*)toc::epoch_large_kernel, &cfg) == cudaSuccess && n >= 1) {
      *cluster = c;
      return TOC_OK;
    }
    (void)cudaGetLastError();
  }
  return TOC_E_CUDA;
}
