// toc_levels.cu -- A.v and v^T.A over the "slot cache": each batch's decode tree reduced to the
// nodes the products actually need, plus a code stream cut into equal per-thread ranges.
//
// Reference: codec.py:215-259 (build_prefix_tree, C'), kernels.py:115-142 (matvec, Algorithm 5:
// H[i] = value[i]*v[col[i]] + H[parent[i]], R[r] = sum_j H[D[r][j]]) and kernels.py:145-174 (vecmat,
// Algorithm 6: H[code] += u[row]; descending i: out[col[i]] += value[i]*H[i], H[parent[i]] += H[i]).
//
// Which nodes need a table slot.  Every code x of row r contributes H[x] to R[r] (A.v) and u[r] to
// every pair of x's expansion (v^T.A).  A derived node x is (par, key) with H[x] = H[par] + P1[key],
// so a code whose node is a *leaf* of the used tree is evaluated from two slots, H[par] + H[key],
// and needs no slot itself.  Slots exist only for
//   the pairs (depth 1: H = P1 = value * v[col]), numbered by column (within a column in the
//   order that spreads the value-index gather over the banks), and
//   the inner nodes: derived nodes some used derived node hangs off (closed under parents) --
//   ~3.2 k of a config-2 batch's ~24 k derived nodes -- numbered for the banks of their chains.
// Cache entry (built once per arena on the host, the counterpart of the reference's cached
// CompressedMatrix.tree, kernels.py:68-77), self-contained so a launch reads nothing else:
//   header  LvlHdr (80 B)
//   staged region, one TMA bulk copy into shared memory per batch:
//     uniq   f64[nU]    the block's value index (physical.py:49-130), aligned
//     rowoff u32[n+1]   row offsets into the record stream
//     prs    u32[nP]    column | value ref << 16 of pair slot 1 + i
//     inner  u32[nQ]    ref(par) | ref(key) << 16 of inner slot nP + 1 + q   (key is a pair; a
//                       reference is the slot's low-limb word index, see slot_ref)
//     colst  u16[n_cols + 1]  first pair slot of every column (pairs are column-sorted)
//     trow   u16[T]     row of thread t's first record | (the record starts its row) << 15
//   stream u16[T*K]  one record per slot reference, in row order: reference | row-end flag << 15.
//                    A code whose node has a slot is one record, a leaf two (slot(par), slot(key)),
//                    an empty row one record of slot 0 (a zero) -- every row ends with a flagged
//                    record, every access instruction runs with full warps.  Thread t owns records
//                    [t*K, t*K + K), stored interleaved in groups of eight so a warp's 16-byte
//                    loads are contiguous; which of a row's records sits at which of the row's
//                    positions is chosen for the banks (schedule_banks, refine_banks)
// Per batch (one 1024-thread CTA, tables in shared memory):
//   A.v   P1 for the pair slots; H of the inner slots, each the sum of P1 over its own chain (no
//         level barriers); every thread sums its K records row by row; rows crossing a range
//         boundary are finished from per-thread head / tail partials in thread order
//   v^T.A T[slot] += u[r] for every record: exact fixed point (two 32-bit limbs added with
//         native shared-memory atomics, carry-free, see limb_add) -- order-independent
//         push: every inner slot adds its T to each pair slot of its chain
//         O[c] = sum over column c's pair slots of value * T, in slot order
// Every thread does the same number of records (no divergence on chain lengths), the stream is
// read with coalesced loads, a record costs one table access, every sum has a fixed order.
// DESIGN.md 4.1.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <thread>
#include <vector>

#include "toc_batch.cuh"  // TMA bulk copy + mbarrier helpers, fixed-point limbs

namespace toc {

// Probe builds (tools/probe_two_ctas.sh) override these: CTA size the streams are cut for, and CTAs
// per SM the kernels are compiled and launched for.
#ifndef TOC_LVL_THREADS
#define TOC_LVL_THREADS 1024
#endif
#ifndef TOC_LVL_CTAS_PER_SM
#define TOC_LVL_CTAS_PER_SM 1
#endif
constexpr uint32_t kLvlThreads = TOC_LVL_THREADS;  // the CTA size the streams are cut for

// Entry header; section offsets relative to the entry start, 16-B aligned.  The staged region is
// [off_uniq, off_stream).
struct LvlHdr {
  uint32_t nP, nQ, S;  // pair slots, inner slots, S = 1 + nP + nQ (slot 0 is a zero)
  uint32_t C, K, T;    // codes, codes per thread (a multiple of 4), threads
  uint32_t n_rows, n_cols, nU;
  uint32_t off_uniq, off_rowoff, off_prs, off_inner, off_colst, off_stream;
  uint32_t off_trow;
  double vmax;  // max |value| of the value index (fixed-point precision check)
  uint32_t invK, invM;  // 2^32 / K and 2^32 / M rounded up (M = pair slots per thread in the column pass):
                        // x / K == umulhi(x, invK) for x < 2^16
};
static_assert(sizeof(LvlHdr) == 80, "slot cache header");
constexpr uint32_t kHdrBytes = 80;

TOC_HD uint32_t align4(uint32_t x) { return (x + 3u) & ~3u; }

// Shared-memory layout (bytes from the dynamic base).
struct LvlSmem {
  uint32_t red, v, u, wt, part, rowcur, stage, tab, total;
};

// The fixed-size regions come first, at compile-time offsets (no address arithmetic from kernel
// parameters in the loops that use them): mbarrier | sum |u| partials | head / tail partials | u.
constexpr uint32_t kRedOff = 16, kPartOff = kRedOff + 48 * 8, kUOff = kPartOff + 16u * kLvlThreads;

TOC_HD LvlSmem lvl_smem(int kind, uint32_t n_cols, uint32_t max_slots, uint32_t max_stage, uint32_t max_rows) {
  LvlSmem L;
  L.red = kRedOff;  // sum |u| partials and total
  L.part = kPartOff;  // head / tail partials (rows, columns)
  L.u = kUOff;
  uint32_t o = kUOff + ((kind & TOC_VECMAT) ? align16(8u * max_rows) : 0u);
  L.wt = o;  // each row's fixed-point weight (v^T.A)
  o += (kind & TOC_VECMAT) ? align16(8u * max_rows) : 0u;
  L.v = o;
  // A.v: v; v^T.A alone: a private copy of the column starts (the stage is refilled while the
  // column totals still read them)
  o += (kind & TOC_MATVEC) ? align16(8u * n_cols) : align16(2u * (n_cols + 1));
  L.rowcur = o;
  o += (kind & TOC_MATVEC) ? align16(4u * (max_rows + 1)) : 0u;
  L.stage = o;
  o += align16(max_stage);
  L.tab = o;
  o += 8u * align4(max_slots);
  L.total = o;
  return L;
}

struct LvlArgs {
  LvlSmem sl;  // shared-memory layout (host-computed: the offsets stay kernel parameters, not registers)
  const int64_t* row_base;
  int64_t n_blocks;
  int32_t kind, n_cols, max_slots, max_stage, max_rows;
  const uint8_t* lvl;
  const int64_t* lvl_off;
  const double* v;
  double* R;
  const double* u;
  double* O;
};

// L2 prefetch knob: 1 (default) = the CTA's next entry at the start of the current batch; 0 = none.
__constant__ int g_prefetch_mode = 1;
// Phase trace (tools/slots_trace.py): when set, CTA 0 records clock64 after each phase of its
// first 64 batches, 10 stamps per batch.
__constant__ long long* g_trace = nullptr;


// Slot references.  Slot p owns the 8 table bytes at 8p: H[p] as a double (A.v), or the two 32-bit
// limbs of T[p] (v^T.A) with the low limb in the first or the second word by bit 4 of p, so that the
// low limbs of any 32 consecutive slots (and the high limbs) cover all 32 banks -- a warp-wide
// atomic on one limb of random slots spreads like one on a plain 32-bit array, while a slot's T
// and H share their bytes (the fused kernel turns T[p] into H[p] in place, pair by pair).  A
// reference is q = 2p + ((p >> 4) & 1), the word index of the low limb: low limb at byte 4q, high
// limb at 4(q ^ 1), the double at 4(q & ~1).
// Stream records (16 bits): reference (bits 0-14) | row-end flag (bit 15); two per 32-bit word.
constexpr uint32_t kRowEnd = 0x8000u;
constexpr uint32_t kMaxSlots = 16384;  // 15-bit references

TOC_HD uint32_t slot_ref(uint32_t p) { return 2u * p + ((p >> 4) & 1u); }

// Byte offset of the low limb from a record (the double: & ~7).
TOC_D uint32_t ref_lo(uint32_t w) { return (w << 2) & 0x1fffcu; }   // the record in the low half of w
TOC_D uint32_t ref_hi(uint32_t w) { return (w >> 14) & 0x1fffcu; }  // and in the high half

// T[slot] += x (carry-free limbs, see limb_add in toc_batch.cuh) for the slot whose low limb is at
// byte `lo` of the table.
TOC_D void limb_add_at(uint8_t* tab, uint32_t lo, uint32_t xl, int32_t xh) {
  atomicAdd(reinterpret_cast<uint32_t*>(tab + lo), xl);
  atomicAdd(reinterpret_cast<int32_t*>(tab + (lo ^ 4u)), xh);
}

// Slot p's limbs (lo, hi) from its 8 bytes.
TOC_D uint2 limbs_of(const uint8_t* tab, uint32_t p) {
  const uint2 w = *reinterpret_cast<const uint2*>(tab + 8u * p);
  return (p & 16u) ? make_uint2(w.y, w.x) : w;
}

// The row containing code s (the largest r with rowoff[r] <= s; rowoff[r + 1] > s then).
TOC_D uint32_t row_of(const uint32_t* rowoff_s, uint32_t n, uint32_t s) {
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (rowoff_s[mid] <= s) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Walk this thread's K records (zero-padded past the last one: slot 0, no row end), eight per
// 16-byte load, two loads in flight.  chunk(w) handles eight records; w0 / w1 are the first two
// chunks, loaded by the caller ahead of time.
template <typename Chunk>
TOC_D void walk_stream(const uint4* __restrict__ st, uint32_t nth, uint32_t K, uint4 w0, uint4 w1, Chunk&& chunk) {
  const uint32_t nq = K >> 3;
  for (uint32_t q = 0; q < nq; ++q) {
    const uint4 w = w0;
    w0 = w1;
    if (q + 2 < nq) w1 = __ldg(st + (size_t)(q + 2) * nth);
    chunk(w);
  }
}

#define TOC_LVL_STAMP(k)                                                                      \
  if constexpr (kTrace)                                                                       \
    if (g_trace && blockIdx.x == 0 && tid == 0 && b < 64 * (int64_t)gridDim.x) \
  g_trace[(b / gridDim.x) * 10 + (k)] = clock64()

// Stage entry bn (header + value index + row offsets + pair / inner records + column starts) into
// shared memory with one TMA bulk copy, and pull the entry after it into L2.  One thread.
TOC_D void issue_stage(const LvlArgs& a, int64_t bn, uint8_t* stage, uint64_t* mbar) {
  const uint8_t* ent = a.lvl + a.lvl_off[bn];
  const uint32_t bytes = __ldg(reinterpret_cast<const uint32_t*>(ent) + offsetof(LvlHdr, off_stream) / 4);
  bulk_load(stage, ent, bytes, mbar);
  const int64_t bp = bn + gridDim.x;
  if (g_prefetch_mode == 1 && bp < a.n_blocks) {
    const uint32_t ebytes = (uint32_t)(a.lvl_off[bp + 1] - a.lvl_off[bp]) & ~15u;
    if (ebytes)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.lvl + a.lvl_off[bp]), "r"(ebytes) : "memory");
  }
}

// The next batch's u in three steps so no load latency sits on a phase: its row base and row
// count (at the batch start), the first u per thread (a phase later), then all of them into
// shared memory (u_s, the scatter's row weights) and this thread's part of sum |u| (v^T.A's
// fixed-point bound).
struct UPrefetch {
  int64_t rb = 0;
  uint32_t n = 0;
  double u0 = 0.0;
  TOC_D void bounds(const LvlArgs& a, int64_t bn) {
    rb = a.row_base[bn];
    n = __ldg(reinterpret_cast<const uint32_t*>(a.lvl + a.lvl_off[bn]) + offsetof(LvlHdr, n_rows) / 4);
  }
  TOC_D void load(const LvlArgs& a) { u0 = threadIdx.x < n ? __ldg(a.u + rb + threadIdx.x) : 0.0; }
  TOC_D double stash(const LvlArgs& a, double* u_s) const {
    double su = fabs(u0);
    if (threadIdx.x < n) u_s[threadIdx.x] = u0;
    for (uint32_t r = threadIdx.x + blockDim.x; r < n; r += blockDim.x) {
      const double x = __ldg(a.u + rb + r);
      u_s[r] = x;
      su += fabs(x);
    }
    return su;
  }
};

TOC_D void su_store(double su, double* s_red) {
  su = warp_sum(su);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = su;
}

// The fixed-point weight of every row of the batch whose u is in u_s (limb_add's two words, see
// limb_scale): each warp sums the sum |u| partials itself, then thread r converts u[r].  Thread 0
// keeps the batch's sum |u| in s_red[32].
TOC_D void row_weights(double* s_red, const double* u_s, uint2* wt_s, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const double su = warp_sum(lane < nwarps ? s_red[lane] : 0.0);
  const uint32_t L = limb_bits(n);
  const double g = limb_scale(su, L);
  for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) {
    const long long w = __double2ll_rn(u_s[r] * g);
    const int32_t xh = (int32_t)(w >> L);
    wt_s[r] = make_uint2((uint32_t)(w - ((long long)xh << L)), (uint32_t)xh);
  }
  if (threadIdx.x == 0) s_red[32] = su;
}

// Per batch, phases separated by block barriers (MV: A.v, VM: v^T.A):
//   VM  scatter T  |  push  |  column partials  |  column totals, next batch's sum |u|
//   MV  P1  |  inner H  |  row partials  |  row totals
//   VM  zero T for the next batch (beside the row totals)
// Fused kernel: P1 is formed in the column-partials pass (each pair slot's T becomes its H in
// place) and the inner H sits beside the column totals: 6 barriers per batch.
// The next batch's staged region is copied in while the A.v rows run (the rows read only the
// stream, H and a private copy of the row offsets).
template <int kKind, bool kTrace>
__global__ void __launch_bounds__(TOC_LVL_THREADS, TOC_LVL_CTAS_PER_SM) levels_kernel(LvlArgs a) {
  constexpr bool MV = kKind & TOC_MATVEC, VM = kKind & TOC_VECMAT;
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  const uint32_t ncol = (uint32_t)a.n_cols;
  const LvlSmem& SL = a.sl;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  double* s_red = reinterpret_cast<double*>(smem + kRedOff);  // [0, 32) partials; [32] this batch's sum |u|
  double* v_s = reinterpret_cast<double*>(smem + SL.v);
  double* u_s = reinterpret_cast<double*>(smem + kUOff);  // this batch's u (v^T.A row weights)
  uint2* wt_s = reinterpret_cast<uint2*>(smem + SL.wt);    // and its rows' fixed-point weights
  double* head_s = reinterpret_cast<double*>(smem + kPartOff);
  double* tail_s = head_s + kLvlThreads;
  uint32_t* rowcur_s = reinterpret_cast<uint32_t*>(smem + SL.rowcur);
  uint8_t* stage = smem + SL.stage;
  uint8_t* tabp = smem + SL.tab;
  double* H = reinterpret_cast<double*>(tabp);  // A.v; v^T.A: limbs (lo, hi arrays) or fp64 T
  const uint32_t S4max = align4(a.max_slots);
  const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
  uint32_t phase = 0;
  int64_t b = blockIdx.x;
  TOC_LVL_STAMP(9);  // kernel entry (the first batch's row of the trace)
  if (tid == 0) mbar_init(mbar, 1);
  if (MV)
    for (uint32_t c = tid; c < ncol; c += nth) v_s[c] = a.v[c];
  if (VM)
    for (uint32_t i = tid; i < S4max / 2; i += nth) reinterpret_cast<uint4*>(tabp)[i] = z4;
  __syncthreads();
  if (b < a.n_blocks) {
    if (tid == 0) issue_stage(a, b, stage, mbar);
  }
  UPrefetch p0;
  if (VM && b < a.n_blocks) {
    p0.bounds(a, b);
    p0.load(a);
    su_store(p0.stash(a, u_s), s_red);
  }
  __syncthreads();
  if (VM && b < a.n_blocks) row_weights(s_red, u_s, wt_s, p0.n);
  __syncthreads();

  for (; b < a.n_blocks; b += gridDim.x) {
    const int64_t bn = b + gridDim.x;
    const bool has_next = bn < a.n_blocks;
    mbar_wait(mbar, phase);
    phase ^= 1u;
    TOC_LVL_STAMP(0);
    const LvlHdr h = *reinterpret_cast<const LvlHdr*>(stage);  // the stage is refilled mid-batch
    const uint32_t n = h.n_rows, nP = h.nP, nQ = h.nQ, K = h.K;
    TOC_CHECK(h.S <= (uint32_t)a.max_slots && h.off_stream <= (uint32_t)a.max_stage && n <= (uint32_t)a.max_rows &&
              h.T == nth && h.n_cols == ncol && h.S == 1 + nP + nQ && K % 8 == 0 && h.C <= h.T * K);
    const double* uniq_s = reinterpret_cast<const double*>(stage + h.off_uniq);
    const uint32_t* rowoff_s = reinterpret_cast<const uint32_t*>(stage + h.off_rowoff);
    const uint32_t* prs_s = reinterpret_cast<const uint32_t*>(stage + h.off_prs);
    const uint32_t* inner_s = reinterpret_cast<const uint32_t*>(stage + h.off_inner);
    const uint16_t* colst_s = reinterpret_cast<const uint16_t*>(stage + h.off_colst);
    const int64_t rb = a.row_base[b];
    const uint4* stream = reinterpret_cast<const uint4*>(a.lvl + a.lvl_off[b] + h.off_stream) + tid;
    const bool active = tid * K < h.C;
    uint4 w0 = active ? __ldg(stream) : z4, w1 = active && K > 8 ? __ldg(stream + nth) : z4;
    const uint32_t tr0 = active ? reinterpret_cast<const uint16_t*>(stage + h.off_trow)[tid] : 0u;
    const uint32_t r0 = tr0 & 0x7fffu;  // this thread's first row, and whether its range starts it
    const bool here0 = (tr0 >> 15) != 0;
    TOC_CHECK(!active || (r0 == row_of(rowoff_s, n, tid * K) && here0 == (rowoff_s[r0] == tid * K)));
    UPrefetch pre;  // the next batch's u (v^T.A)
    if (VM && has_next) pre.bounds(a, bn);

    if (VM) {
      double* Tf = reinterpret_cast<double*>(tabp);
      const uint32_t L = limb_bits(n);
      const double g_scale = limb_scale(s_red[32], L), g_inv = 1.0 / g_scale;
      const bool f64 = fixed_point_too_coarse(n, h.vmax, g_inv);  // fp64 accumulation instead
      // T[slot] += u[r] for the slot(s) of every code of this thread's range
      if (active) {
        uint32_t r = r0;
        if (!f64) {
          auto weight = [&](uint32_t row, uint32_t& xl, int32_t& xh) {
            const uint2 q = wt_s[row];
            xl = q.x;
            xh = (int32_t)q.y;
          };
          uint32_t xl;
          int32_t xh;
          weight(r, xl, xh);
          walk_stream(stream, nth, K, w0, w1, [&](const uint4& w) {
            const uint32_t rec[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
              TOC_CHECK(ref_lo(rec[i]) < 8 * h.S && ref_hi(rec[i]) < 8 * h.S && (rec[i] == 0 || r < n));
              limb_add_at(tabp, ref_lo(rec[i]), xl, xh);
              if (rec[i] & kRowEnd)
                if (++r < n) weight(r, xl, xh);
              limb_add_at(tabp, ref_hi(rec[i]), xl, xh);
              if (rec[i] & (kRowEnd << 16))
                if (++r < n) weight(r, xl, xh);
            }
          });
        } else {
          double wu = u_s[r];
          walk_stream(stream, nth, K, w0, w1, [&](const uint4& w) {
            const uint32_t rec[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
              if (wu != 0.0) atomicAdd(reinterpret_cast<double*>(tabp + (ref_lo(rec[i]) & ~7u)), wu);
              if (rec[i] & kRowEnd)
                if (++r < n) wu = u_s[r];
              if (wu != 0.0) atomicAdd(reinterpret_cast<double*>(tabp + (ref_hi(rec[i]) & ~7u)), wu);
              if (rec[i] & (kRowEnd << 16))
                if (++r < n) wu = u_s[r];
            }
          });
        }
        if (MV) {  // the stream again for A.v
          w0 = __ldg(stream);
          w1 = K > 8 ? __ldg(stream + nth) : z4;
        }
      }
      if (!MV)  // the column starts into a private copy: the stage is refilled before the column totals
        for (uint32_t c = tid; c <= ncol; c += nth) reinterpret_cast<uint16_t*>(v_s)[c] = colst_s[c];
      __syncthreads();
      TOC_LVL_STAMP(1);
      // push: each inner slot's own T goes to every pair slot of its chain (inner records hold
      // references: parent | key << 16)
      const uint32_t q_inner = 2u * nP + 2u;  // references from here on are inner slots
      if (!f64) {
        for (uint32_t y = tid; y < nQ; y += nth) {
          const uint32_t x = nP + 1 + y;
          uint32_t rec = inner_s[y];
          TOC_CHECK((rec >> 17) >= 1 && (rec >> 17) <= nP && ((rec & 0xffffu) >> 1) >= 1 && ((rec & 0xffffu) >> 1) < h.S);
          const uint2 t = limbs_of(tabp, x);
          const uint32_t l = t.x;
          const int32_t hh = (int32_t)t.y;
          if (l | (uint32_t)hh) {
            uint32_t q = rec & 0xffffu;
            limb_add_at(tabp, (rec >> 14) & 0x3fffcu, l, hh);
            while (q >= q_inner) {
              TOC_CHECK((q >> 1) - nP - 1 < nQ);
              rec = inner_s[(q >> 1) - nP - 1];
              limb_add_at(tabp, (rec >> 14) & 0x3fffcu, l, hh);
              q = rec & 0xffffu;
            }
            limb_add_at(tabp, q << 2, l, hh);
          }
        }
      } else {
        for (uint32_t y = tid; y < nQ; y += nth) {
          uint32_t rec = inner_s[y];
          const double t = Tf[nP + 1 + y];
          if (t != 0.0) {
            uint32_t q = rec & 0xffffu;
            atomicAdd(Tf + (rec >> 17), t);
            while (q >= q_inner) {
              rec = inner_s[(q >> 1) - nP - 1];
              atomicAdd(Tf + (rec >> 17), t);
              q = rec & 0xffffu;
            }
            atomicAdd(Tf + (q >> 1), t);
          }
        }
      }
      __syncthreads();
      TOC_LVL_STAMP(2);
      pre.load(a);
      // column partials: thread t sums value * T over pair slots [1 + tM, 1 + tM + M) (M odd, so
      // the lanes' slot reads are conflict-free), column by column; a column ending inside the
      // range is complete (started here) or the range's head partial.  Fused kernel: the same pass
      // turns each pair slot into A.v's P1 = value * v[column] (Algorithm 5's H at depth 1) once
      // its T has been read -- one pair record and one value-index gather for both products.
      double* o = a.O + b * (int64_t)ncol;
      const uint32_t M = ((nP + nth - 1) / nth) | 1u;
      {
        const uint32_t p0 = 1 + tid * M, p1 = min(p0 + M, nP + 1);
        if (p0 < p1) {
          bool here = colst_s[prs_s[p0 - 1] & 0xffffu] == p0;
          double acc = 0.0;
          auto pass = [&](auto tval) {  // one loop per accumulation mode (no per-pair select)
            for (uint32_t p = p0; p < p1; ++p) {
              const uint32_t x = prs_s[p - 1];
              TOC_CHECK(((x >> 16) & 0x7fffu) < h.nU && (x & 0xffffu) < ncol);
              const double val = uniq_s[(x >> 16) & 0x7fffu];
              acc += val * tval(p);
              if (MV) H[p] = val * v_s[x & 0xffffu];
              if (x >> 31) {  // last pair slot of its column
                if (here) o[x & 0xffffu] = acc;
                else head_s[tid] = acc;
                acc = 0.0;
                here = true;
              }
            }
          };
          if (f64) pass([&](uint32_t p) { return Tf[p]; });
          else pass([&](uint32_t p) {
            const uint2 t = limbs_of(tabp, p);
            return limb_value(t.x, (int32_t)t.y, L, g_inv);
          });
          tail_s[tid] = acc;
        }
      }
      __syncthreads();
      TOC_LVL_STAMP(3);
      // column totals: columns spanning several ranges (tail, whole middle ranges, head), and 0
      // for the columns no pair touches
      const uint16_t* colst_t = MV ? colst_s : reinterpret_cast<const uint16_t*>(v_s);
      for (uint32_t c = tid; c < ncol; c += nth) {
        const uint32_t lo = colst_t[c], hi = colst_t[c + 1];
        TOC_CHECK(lo >= 1 && lo <= hi && hi <= nP + 1);
        if (lo == hi) {
          o[c] = 0.0;
        } else {
          const uint32_t t0 = M == 1 ? lo - 1 : __umulhi(lo - 1, h.invM), t1 = M == 1 ? hi - 2 : __umulhi(hi - 2, h.invM);
          TOC_CHECK(t0 == (lo - 1) / M && t1 == (hi - 2) / M);
          if (t0 != t1) {
            double x = tail_s[t0];
            for (uint32_t t = t0 + 1; t < t1; ++t) x += tail_s[t];
            o[c] = x + head_s[t1];
          }
        }
      }
      su_store(pre.stash(a, u_s), s_red);
    }
    if (MV) {
      if (!VM) {
        // P1 for the pair slots (Algorithm 5's H at depth 1)
        for (uint32_t i = tid; i < nP; i += nth) {
          const uint32_t x = prs_s[i];
          TOC_CHECK(((x >> 16) & 0x7fffu) < h.nU && (x & 0xffffu) < ncol);
          H[1 + i] = uniq_s[(x >> 16) & 0x7fffu] * v_s[x & 0xffffu];
        }
      }
      if (tid == 0) H[0] = 0.0;  // padding records scatter to slot 0
      // the row offsets into a private copy (the stage is refilled while the rows run)
      for (uint32_t r = tid; r <= n; r += nth) rowcur_s[r] = rowoff_s[r];
      if (!VM) __syncthreads();
      TOC_LVL_STAMP(4);
      // H of the inner slots: the sum of P1 over the node's chain (reads pair slots only); fused
      // kernel: beside the column totals (slot 0 keeps its zero: no record scatters to it)
      const uint32_t q_inner = 2u * nP + 2u;
      for (uint32_t y = tid; y < nQ; y += nth) {
        uint32_t rec = inner_s[y];
        double hv = H[rec >> 17];
        uint32_t q = rec & 0xffffu;
        while (q >= q_inner) {
          TOC_CHECK((q >> 1) - nP - 1 < nQ);
          rec = inner_s[(q >> 1) - nP - 1];
          hv += H[rec >> 17];
          q = rec & 0xffffu;
        }
        H[nP + 1 + y] = hv + H[q >> 1];
      }
      __syncthreads();
      TOC_LVL_STAMP(5);
    }
    // issued by the last thread: its warp has few or no records, while thread 0's warp would start its
    // row walk only after the issue's dependent global loads
    if (tid == nth - 1 && has_next) issue_stage(a, bn, stage, mbar);  // the stage is no longer read
    if (MV) {
      // row partials over this thread's codes; a row ending inside the range is complete (started
      // here) or the range's head partial
      if (active) {
        double acc = 0.0;
        uint32_t r = r0;
        bool here = here0;
        walk_stream(stream, nth, K, w0, w1, [&](const uint4& w) {
          const uint32_t rec[4] = {w.x, w.y, w.z, w.w};
          double ha[4], hb[4];
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) {
            TOC_CHECK(ref_lo(rec[i]) < 8 * h.S && ref_hi(rec[i]) < 8 * h.S);
            ha[i] = *reinterpret_cast<const double*>(tabp + (ref_lo(rec[i]) & ~7u));
            hb[i] = *reinterpret_cast<const double*>(tabp + (ref_hi(rec[i]) & ~7u));
          }
          auto row_end = [&]() {
            TOC_CHECK(r < n);
            if (here) a.R[rb + r] = acc;
            else head_s[tid] = acc;
            acc = 0.0;
            here = true;
            ++r;
          };
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) {
            acc += ha[i];
            if (rec[i] & kRowEnd) row_end();
            acc += hb[i];
            if (rec[i] & (kRowEnd << 16)) row_end();
          }
        });
        tail_s[tid] = acc;
      }
      __syncthreads();
      TOC_LVL_STAMP(6);
      // row totals: rows spanning several ranges, and 0 for empty rows
      for (uint32_t r = tid; r < n; r += nth) {
        const uint32_t lo = rowcur_s[r], hi = rowcur_s[r + 1];
        if (lo == hi) {
          a.R[rb + r] = 0.0;
        } else {
          const uint32_t t0 = __umulhi(lo, h.invK), t1 = __umulhi(hi - 1, h.invK);
          TOC_CHECK(t0 == lo / K && t1 == (hi - 1) / K);
          if (t0 != t1) {
            double x = tail_s[t0];
            for (uint32_t t = t0 + 1; t < t1; ++t) x += tail_s[t];
            a.R[rb + r] = x + head_s[t1];
          }
        }
      }
    }
    if (VM) {  // a zero T table and the next batch's row weights (its u and partials are in)
      for (uint32_t i = tid; i < S4max / 2; i += nth) reinterpret_cast<uint4*>(tabp)[i] = z4;
      if (has_next) row_weights(s_red, u_s, wt_s, pre.n);
    }
    __syncthreads();  // tables and partials are reused by the next batch
    TOC_LVL_STAMP(7);
  }
}

#undef TOC_LVL_STAMP

// ---- the fp32 variant over the same cache entries ------------------------------------------------
// BASELINE.json north_star: "1e-4 for the fp32 variant" (the reference itself is fp64 only).  Same
// entries, same shared-memory layout and phases as levels_kernel; a slot's 8 bytes hold one 32-bit
// payload at its reference word q (so the banks the placement was made for stay the same): H[p] as
// a float (A.v), T[p] in 32-bit fixed point (v^T.A: ONE native atomic per record; scale 2^(30 - e)
// with sum |u| < 2^e, so no partial sum leaves int32), or as a float added with float atomics when
// that quantum would be too coarse for the 1e-4 bar (heavy-tailed u; order-dependent in the last
// bits only).  Operands and results are float; the value index stays double and is rounded once per
// product.
struct Lvl32Args {
  LvlSmem sl;
  const int64_t* row_base;
  int64_t n_blocks;
  int32_t kind, n_cols, max_slots, max_stage, max_rows;
  const uint8_t* lvl;
  const int64_t* lvl_off;
  const float* v;
  float* R;
  const float* u;
  float* O;
};

TOC_D void issue_stage32(const Lvl32Args& a, int64_t bn, uint8_t* stage, uint64_t* mbar) {
  const uint8_t* ent = a.lvl + a.lvl_off[bn];
  const uint32_t bytes = __ldg(reinterpret_cast<const uint32_t*>(ent) + offsetof(LvlHdr, off_stream) / 4);
  bulk_load(stage, ent, bytes, mbar);
  const int64_t bp = bn + gridDim.x;
  if (g_prefetch_mode == 1 && bp < a.n_blocks) {
    const uint32_t ebytes = (uint32_t)(a.lvl_off[bp + 1] - a.lvl_off[bp]) & ~15u;
    if (ebytes)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.lvl + a.lvl_off[bp]), "r"(ebytes) : "memory");
  }
}

// The next batch's u a batch ahead, as UPrefetch does for the fp64 kernel.
struct UPrefetch32 {
  int64_t rb = 0;
  uint32_t n = 0;
  float u0 = 0.0f;
  TOC_D void bounds(const Lvl32Args& a, int64_t bn) {
    rb = a.row_base[bn];
    n = __ldg(reinterpret_cast<const uint32_t*>(a.lvl + a.lvl_off[bn]) + offsetof(LvlHdr, n_rows) / 4);
  }
  TOC_D void load(const Lvl32Args& a) { u0 = threadIdx.x < n ? __ldg(a.u + rb + threadIdx.x) : 0.0f; }
  TOC_D double stash(const Lvl32Args& a, float* u_s) const {
    double su = fabs((double)u0);
    if (threadIdx.x < n) u_s[threadIdx.x] = u0;
    for (uint32_t r = threadIdx.x + blockDim.x; r < n; r += blockDim.x) {
      const float x = __ldg(a.u + rb + r);
      u_s[r] = x;
      su += fabs((double)x);
    }
    return su;
  }
};

// 2^(30 - e) for sum |u| < 2^e: no partial sum of the fixed-point weights leaves int32.
TOC_D double fix32_scale_of(double su) {
  if (!(su > 0.0)) return 1.0;
  int e;
  frexp(su, &e);
  return ldexp(1.0, 30 - e);
}

// Rounding errors of +-q/2 per addend (q = 1/scale) are independent: a column's error has standard
// deviation q * max|value| * sqrt(n/12); fixed point is used while 6 of them stay under 2^-15 (the
// bar is 1e-4), float atomics otherwise.
TOC_D bool fix32_too_coarse(uint32_t n, double vmax, double scale) {
  return 6.0 * vmax * sqrt((double)n / 12.0) / scale > 0x1p-15;
}

// The fixed-point weight of every row of the batch whose u is in u_s; thread 0 keeps the batch's
// sum |u| in s_red[32].
TOC_D void row_weights32(double* s_red, const float* u_s, int32_t* wt_s, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const double su = warp_sum(lane < nwarps ? s_red[lane] : 0.0);
  const double g = fix32_scale_of(su);
  for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) wt_s[r] = __double2int_rn((double)u_s[r] * g);
  if (threadIdx.x == 0) s_red[32] = su;
}

template <int kKind>
__global__ void __launch_bounds__(TOC_LVL_THREADS, TOC_LVL_CTAS_PER_SM) levels32_kernel(Lvl32Args a) {
  constexpr bool MV = kKind & TOC_MATVEC, VM = kKind & TOC_VECMAT;
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  const uint32_t ncol = (uint32_t)a.n_cols;
  const LvlSmem& SL = a.sl;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  double* s_red = reinterpret_cast<double*>(smem + kRedOff);  // [0, 32) partials of sum |u|
  float* v_s = reinterpret_cast<float*>(smem + SL.v);
  float* u_s = reinterpret_cast<float*>(smem + kUOff);     // this batch's u
  int32_t* wt_s = reinterpret_cast<int32_t*>(smem + SL.wt);  // and its rows' fixed-point weights
  float* head_s = reinterpret_cast<float*>(smem + kPartOff);
  float* tail_s = head_s + kLvlThreads;
  uint32_t* rowcur_s = reinterpret_cast<uint32_t*>(smem + SL.rowcur);
  uint8_t* stage = smem + SL.stage;
  uint8_t* tabp = smem + SL.tab;
  const uint32_t S4max = align4(a.max_slots);
  const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
  auto Hf = [&](uint32_t ref) -> float& { return *reinterpret_cast<float*>(tabp + 4u * ref); };  // by reference word
  uint32_t phase = 0;
  if (tid == 0) mbar_init(mbar, 1);
  if (MV)
    for (uint32_t c = tid; c < ncol; c += nth) v_s[c] = a.v[c];
  if (VM)
    for (uint32_t i = tid; i < S4max / 2; i += nth) reinterpret_cast<uint4*>(tabp)[i] = z4;
  __syncthreads();
  int64_t b = blockIdx.x;
  if (tid == 0 && b < a.n_blocks) issue_stage32(a, b, stage, mbar);
  UPrefetch32 p0;
  if (VM && b < a.n_blocks) {
    p0.bounds(a, b);
    p0.load(a);
    su_store(p0.stash(a, u_s), s_red);
  }
  __syncthreads();
  if (VM && b < a.n_blocks) row_weights32(s_red, u_s, wt_s, p0.n);
  __syncthreads();

  for (; b < a.n_blocks; b += gridDim.x) {
    const int64_t bn = b + gridDim.x;
    const bool has_next = bn < a.n_blocks;
    mbar_wait(mbar, phase);
    phase ^= 1u;
    const LvlHdr h = *reinterpret_cast<const LvlHdr*>(stage);  // the stage is refilled mid-batch
    const uint32_t n = h.n_rows, nP = h.nP, nQ = h.nQ, K = h.K;
    UPrefetch32 pre;  // the next batch's u
    if (VM && has_next) pre.bounds(a, bn);
    TOC_CHECK(h.S <= (uint32_t)a.max_slots && h.off_stream <= (uint32_t)a.max_stage && n <= (uint32_t)a.max_rows &&
              h.T == nth && h.n_cols == ncol && h.S == 1 + nP + nQ && K % 8 == 0 && h.C <= h.T * K);
    const double* uniq_s = reinterpret_cast<const double*>(stage + h.off_uniq);
    const uint32_t* rowoff_s = reinterpret_cast<const uint32_t*>(stage + h.off_rowoff);
    const uint32_t* prs_s = reinterpret_cast<const uint32_t*>(stage + h.off_prs);
    const uint32_t* inner_s = reinterpret_cast<const uint32_t*>(stage + h.off_inner);
    const uint16_t* colst_s = reinterpret_cast<const uint16_t*>(stage + h.off_colst);
    const int64_t rb = a.row_base[b];
    const uint4* stream = reinterpret_cast<const uint4*>(a.lvl + a.lvl_off[b] + h.off_stream) + tid;
    const bool active = tid * K < h.C;
    uint4 w0 = active ? __ldg(stream) : z4, w1 = active && K > 8 ? __ldg(stream + nth) : z4;
    const uint32_t tr0 = active ? reinterpret_cast<const uint16_t*>(stage + h.off_trow)[tid] : 0u;
    const uint32_t r0 = tr0 & 0x7fffu;
    const bool here0 = (tr0 >> 15) != 0;
    const uint32_t q_inner = 2u * nP + 2u;  // references from here on are inner slots
    const uint32_t M = ((nP + nth - 1) / nth) | 1u;

    if (VM) {
      // u_s, wt_s and s_red[32] (sum |u|) were prepared during the previous batch (or the prologue)
      const double g_scale = fix32_scale_of(s_red[32]);
      const bool flt = fix32_too_coarse(n, h.vmax, g_scale);  // float accumulation instead
      const float g_inv = (float)(1.0 / g_scale);
      // T[slot] += u[r] for every record of this thread's range
      if (active) {
        uint32_t r = r0;
        if (!flt) {
          int32_t w = wt_s[r];
          walk_stream(stream, nth, K, w0, w1, [&](const uint4& ww) {
            const uint32_t rec[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
              TOC_CHECK(ref_lo(rec[i]) < 8 * h.S && ref_hi(rec[i]) < 8 * h.S && (rec[i] == 0 || r < n));
              atomicAdd(reinterpret_cast<int32_t*>(tabp + ref_lo(rec[i])), w);
              if (rec[i] & kRowEnd)
                if (++r < n) w = wt_s[r];
              atomicAdd(reinterpret_cast<int32_t*>(tabp + ref_hi(rec[i])), w);
              if (rec[i] & (kRowEnd << 16))
                if (++r < n) w = wt_s[r];
            }
          });
        } else {
          float wu = u_s[r];
          walk_stream(stream, nth, K, w0, w1, [&](const uint4& ww) {
            const uint32_t rec[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
              if (wu != 0.0f) atomicAdd(reinterpret_cast<float*>(tabp + ref_lo(rec[i])), wu);
              if (rec[i] & kRowEnd)
                if (++r < n) wu = u_s[r];
              if (wu != 0.0f) atomicAdd(reinterpret_cast<float*>(tabp + ref_hi(rec[i])), wu);
              if (rec[i] & (kRowEnd << 16))
                if (++r < n) wu = u_s[r];
            }
          });
        }
        if (MV) {  // the stream again for A.v
          w0 = __ldg(stream);
          w1 = K > 8 ? __ldg(stream + nth) : z4;
        }
      }
      if (!MV)  // the column starts into a private copy: the stage is refilled before the column totals
        for (uint32_t c = tid; c <= ncol; c += nth) reinterpret_cast<uint16_t*>(v_s)[c] = colst_s[c];
      __syncthreads();
      // push: each inner slot's own T goes to every pair slot of its chain
      for (uint32_t y = tid; y < nQ; y += nth) {
        uint32_t rec = inner_s[y];
        const uint32_t own = 4u * slot_ref(nP + 1 + y);
        if (!flt) {
          const int32_t t = *reinterpret_cast<const int32_t*>(tabp + own);
          if (t) {
            uint32_t q = rec & 0xffffu;
            atomicAdd(reinterpret_cast<int32_t*>(tabp + ((rec >> 14) & 0x3fffcu)), t);
            while (q >= q_inner) {
              rec = inner_s[(q >> 1) - nP - 1];
              atomicAdd(reinterpret_cast<int32_t*>(tabp + ((rec >> 14) & 0x3fffcu)), t);
              q = rec & 0xffffu;
            }
            atomicAdd(reinterpret_cast<int32_t*>(tabp + (q << 2)), t);
          }
        } else {
          const float t = *reinterpret_cast<const float*>(tabp + own);
          if (t != 0.0f) {
            uint32_t q = rec & 0xffffu;
            atomicAdd(reinterpret_cast<float*>(tabp + ((rec >> 14) & 0x3fffcu)), t);
            while (q >= q_inner) {
              rec = inner_s[(q >> 1) - nP - 1];
              atomicAdd(reinterpret_cast<float*>(tabp + ((rec >> 14) & 0x3fffcu)), t);
              q = rec & 0xffffu;
            }
            atomicAdd(reinterpret_cast<float*>(tabp + (q << 2)), t);
          }
        }
      }
      __syncthreads();
      pre.load(a);
      // column partials (and, fused, each pair slot's T turned into its P1 in place)
      float* o = a.O + b * (int64_t)ncol;
      {
        const uint32_t p0 = 1 + tid * M, p1 = min(p0 + M, nP + 1);
        if (p0 < p1) {
          bool here = colst_s[prs_s[p0 - 1] & 0xffffu] == p0;
          float acc = 0.0f;
          for (uint32_t p = p0; p < p1; ++p) {
            const uint32_t x = prs_s[p - 1];
            TOC_CHECK(((x >> 16) & 0x7fffu) < h.nU && (x & 0xffffu) < ncol);
            const float val = (float)uniq_s[(x >> 16) & 0x7fffu];
            float& cell = Hf(slot_ref(p));
            const float t = flt ? cell : (float)__float_as_int(cell) * g_inv;
            acc += val * t;
            if (MV) cell = val * v_s[x & 0xffffu];
            if (x >> 31) {  // last pair slot of its column
              if (here) o[x & 0xffffu] = acc;
              else head_s[tid] = acc;
              acc = 0.0f;
              here = true;
            }
          }
          tail_s[tid] = acc;
        }
      }
      __syncthreads();
      // column totals: columns spanning several ranges, and 0 for the columns no pair touches
      const uint16_t* colst_t = MV ? colst_s : reinterpret_cast<const uint16_t*>(v_s);
      for (uint32_t c = tid; c < ncol; c += nth) {
        const uint32_t lo = colst_t[c], hi = colst_t[c + 1];
        if (lo == hi) {
          o[c] = 0.0f;
        } else {
          const uint32_t t0 = M == 1 ? lo - 1 : __umulhi(lo - 1, h.invM), t1 = M == 1 ? hi - 2 : __umulhi(hi - 2, h.invM);
          if (t0 != t1) {
            float x = tail_s[t0];
            for (uint32_t t = t0 + 1; t < t1; ++t) x += tail_s[t];
            o[c] = x + head_s[t1];
          }
        }
      }
      su_store(pre.stash(a, u_s), s_red);  // the next batch's u (this batch's was last read by the scatter)
    }
    if (MV) {
      if (!VM) {
        for (uint32_t i = tid; i < nP; i += nth) {
          const uint32_t x = prs_s[i];
          Hf(slot_ref(1 + i)) = (float)uniq_s[(x >> 16) & 0x7fffu] * v_s[x & 0xffffu];
        }
      }
      if (tid == 0) Hf(0) = 0.0f;  // padding and empty-row records read slot 0
      for (uint32_t r = tid; r <= n; r += nth) rowcur_s[r] = rowoff_s[r];
      if (!VM) __syncthreads();
      // H of the inner slots: the sum of P1 over the node's chain (reads pair slots only)
      for (uint32_t y = tid; y < nQ; y += nth) {
        uint32_t rec = inner_s[y];
        float hv = Hf(rec >> 16);
        uint32_t q = rec & 0xffffu;
        while (q >= q_inner) {
          rec = inner_s[(q >> 1) - nP - 1];
          hv += Hf(rec >> 16);
          q = rec & 0xffffu;
        }
        Hf(slot_ref(nP + 1 + y)) = hv + Hf(q);
      }
      __syncthreads();
    } else {
      __syncthreads();  // v^T.A alone: nothing reads the stage after the column totals' private copy
    }
    if (tid == 0 && has_next) issue_stage32(a, bn, stage, mbar);  // the stage is no longer read
    if (MV) {
      if (active) {
        float acc = 0.0f;
        uint32_t r = r0;
        bool here = here0;
        walk_stream(stream, nth, K, w0, w1, [&](const uint4& ww) {
          const uint32_t rec[4] = {ww.x, ww.y, ww.z, ww.w};
          float ha[4], hb[4];
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) {
            ha[i] = *reinterpret_cast<const float*>(tabp + ref_lo(rec[i]));
            hb[i] = *reinterpret_cast<const float*>(tabp + ref_hi(rec[i]));
          }
          auto row_end = [&]() {
            TOC_CHECK(r < n);
            if (here) a.R[rb + r] = acc;
            else head_s[tid] = acc;
            acc = 0.0f;
            here = true;
            ++r;
          };
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) {
            acc += ha[i];
            if (rec[i] & kRowEnd) row_end();
            acc += hb[i];
            if (rec[i] & (kRowEnd << 16)) row_end();
          }
        });
        tail_s[tid] = acc;
      }
      __syncthreads();
      for (uint32_t r = tid; r < n; r += nth) {
        const uint32_t lo = rowcur_s[r], hi = rowcur_s[r + 1];
        if (lo == hi) {
          a.R[rb + r] = 0.0f;
        } else {
          const uint32_t t0 = __umulhi(lo, h.invK), t1 = __umulhi(hi - 1, h.invK);
          if (t0 != t1) {
            float x = tail_s[t0];
            for (uint32_t t = t0 + 1; t < t1; ++t) x += tail_s[t];
            a.R[rb + r] = x + head_s[t1];
          }
        }
      }
    }
    if (VM) {  // a zero T table and the next batch's row weights (its u and partials are in)
      for (uint32_t i = tid; i < S4max / 2; i += nth) reinterpret_cast<uint4*>(tabp)[i] = z4;
      if (has_next) row_weights32(s_red, u_s, wt_s, pre.n);
    }
    __syncthreads();  // tables and partials are reused by the next batch
  }
}

}  // namespace toc

// ------------------------------------------------------------------------------------------
// Host side: building the cache (once per arena) and launching.
namespace {

using toc::LvlHdr;

inline uint32_t rd_packed(const uint8_t* p, uint64_t i, uint32_t w) {
  uint32_t v = 0;
  memcpy(&v, p + i * w, w);  // little endian (physical.py:54-68)
  return v;
}

struct LvlEntry {
  std::vector<uint8_t> bytes;
  uint32_t S = 0, stage = 0, n_rows = 0;
  int status = TOC_OK;
};

struct LvlCache {
  std::vector<LvlEntry> entries;
  int64_t total = 0;
  int32_t max_slots = 0, max_stage = 0, max_rows = 0;
  int32_t status = TOC_OK;
};

// Bank-aware placement of the records.  The kernel's T scatter and row sums are bound by shared-
// memory wavefronts: a warp's 32-bit atomics cost one wavefront per lane in the most loaded bank
// (the low-limb word q mod 32; the high limb q ^ 1 mirrors it), a 64-bit gather one per distinct
// word in the most loaded bank pair ((q >> 1) mod 16) of each half-warp.  Position j = t*K + k is
// thread t's k-th record; a row's positions keep their row (so the per-thread row logic and the
// row-end flags are unchanged) but which of the row's records sits at which of its positions is
// free (the row's sums do not depend on it).  Warp by warp, step by step, each lane (fewest choices
// first) takes from its row's remaining records the one whose word hits the least used bank and
// bank pair among the lanes placed so far in this step.
void schedule_banks(std::vector<uint32_t>& rec, const std::vector<uint32_t>& rowid, const std::vector<uint32_t>& off,
                    uint32_t n, uint32_t C, uint32_t K, uint32_t T) {
  std::vector<std::vector<uint32_t>> pool(n);
  for (uint32_t r = 0; r < n; ++r) pool[r].assign(rec.begin() + off[r], rec.begin() + off[r + 1]);
  // seen[h][word] == stamp: the 8-byte word is already gathered by a placed lane of half-warp h in
  // this step (a 64-bit gather of the same word is a broadcast, not a conflict)
  std::vector<uint32_t> seen[2] = {std::vector<uint32_t>(toc::kMaxSlots, 0), std::vector<uint32_t>(toc::kMaxSlots, 0)};
  uint32_t stamp = 0;
  uint32_t lanes[32];
  for (uint32_t w = 0; w < T / 32; ++w) {
    if ((uint64_t)w * 32 * K >= C) break;
    for (uint32_t k = 0; k < K; ++k) {
      uint32_t na = 0;
      for (uint32_t l = 0; l < 32; ++l) {
        const uint64_t j = (uint64_t)(w * 32 + l) * K + k;
        if (j < C) lanes[na++] = l;
      }
      if (!na) continue;
      std::stable_sort(lanes, lanes + na, [&](uint32_t x, uint32_t y) {
        return pool[rowid[(w * 32 + x) * K + k]].size() < pool[rowid[(w * 32 + y) * K + k]].size();
      });
      // ca: lanes per 32-bit bank of the low-limb words (the scatter's atomics); ga: distinct 8-byte
      // words per bank pair and half-warp (the row gathers)
      uint8_t ca[32] = {0}, ga[2][16] = {{0}};
      ++stamp;
      for (uint32_t q = 0; q < na; ++q) {
        const uint32_t j = (w * 32 + lanes[q]) * K + k, hf = lanes[q] >> 4;
        std::vector<uint32_t>& P = pool[rowid[j]];
        size_t best = 0;
        uint32_t bc = ~0u;
        for (size_t i = 0; i < P.size() && bc; ++i) {
          const uint32_t a = P[i];
          const uint32_t c = 4u * ca[a & 31] + (seen[hf][a >> 1] == stamp ? 0u : 3u * ga[hf][(a >> 1) & 15]);
          if (c < bc) bc = c, best = i;
        }
        const uint32_t a = P[best];
        P[best] = P.back();
        P.pop_back();
        ++ca[a & 31];
        if (seen[hf][a >> 1] != stamp) ++ga[hf][(a >> 1) & 15];
        seen[hf][a >> 1] = stamp;
        rec[j] = a;
      }
    }
  }
}

// Local search after the greedy placement: for every (warp, step) above its conflict-free cost, a
// lane sitting in a most loaded bank trades records with another position of its row when that
// lowers the modelled wavefronts of the two steps involved.  Model (what tools/bank_model.py
// reports, with lanes counted instead of distinct words): per step 2 x the most loaded 32-bit bank
// of the atomics + per half-warp the most loaded bank pair of the gathers.
struct StepBanks {
  uint8_t ca[32], ga[2][16];
  void add(uint32_t lane, uint32_t x, int d) { ca[x & 31u] += d, ga[lane >> 4][(x >> 1) & 15u] += d; }
  struct Max {
    uint32_t a, g[2];  // most loaded bank of the atomics, bank pair of the gathers per half-warp
    uint32_t cost() const { return 2u * a + g[0] + g[1]; }
  };
  Max maxes() const {
    Max m{0, {0, 0}};
    for (uint32_t i = 0; i < 32; ++i) m.a = std::max<uint32_t>(m.a, ca[i]);
    for (uint32_t i = 0; i < 16; ++i)
      m.g[0] = std::max<uint32_t>(m.g[0], ga[0][i]), m.g[1] = std::max<uint32_t>(m.g[1], ga[1][i]);
    return m;
  }
  uint32_t cost() const { return maxes().cost(); }
  // the step's cost with record x added at `lane`, given the maxes without it
  uint32_t cost_with(const Max& m, uint32_t lane, uint32_t x) const {
    const uint32_t h = lane >> 4;
    return m.cost() + 2u * (std::max<uint32_t>(m.a, ca[x & 31u] + 1u) - m.a) +
           (std::max<uint32_t>(m.g[h], ga[h][(x >> 1) & 15u] + 1u) - m.g[h]);
  }
  // is lane's record x in a most loaded (> 1) bank?
  bool hot(uint32_t lane, uint32_t x) const {
    auto top = [](const uint8_t* c, uint32_t n, uint32_t i) {
      if (c[i] < 2) return false;
      for (uint32_t k = 0; k < n; ++k)
        if (c[k] > c[i]) return false;
      return true;
    };
    return top(ca, 32, x & 31u) || top(ga[lane >> 4], 16, (x >> 1) & 15u);
  }
};

void refine_banks(std::vector<uint32_t>& rec, const std::vector<uint32_t>& rowid, const std::vector<uint32_t>& off,
                  uint32_t C, uint32_t K, uint32_t T, int passes) {
  const uint32_t W = (uint32_t)std::min<uint64_t>(T / 32, ((uint64_t)C + 32ull * K - 1) / (32ull * K));
  std::vector<StepBanks> sb((size_t)W * K);
  memset(sb.data(), 0, sb.size() * sizeof(StepBanks));
  std::vector<uint32_t> cost((size_t)W * K);
  for (uint32_t j = 0; j < C; ++j) sb[(size_t)(j / K / 32) * K + j % K].add((j / K) & 31, rec[j], 1);
  for (size_t i = 0; i < sb.size(); ++i) cost[i] = sb[i].cost();
  for (int pass = 0; pass < passes; ++pass) {
    bool any = false;
    for (uint32_t w = 0; w < W; ++w)
      for (uint32_t k = 0; k < K; ++k) {
        const size_t si = (size_t)w * K + k;
        StepBanks& s = sb[si];
        for (uint32_t l = 0; l < 32; ++l) {
          const uint64_t j64 = (uint64_t)(w * 32 + l) * K + k;
          if (j64 >= C) break;
          const uint32_t j = (uint32_t)j64;
          if (!s.hot(l, rec[j])) continue;
          const uint32_t r = rowid[j], x = rec[j];
          s.add(l, x, -1);
          const StepBanks::Max m = s.maxes();
          if (m.cost() >= cost[si]) {  // removing x alone does not lower the step: no trade of x can
            s.add(l, x, 1);
            continue;
          }
          uint32_t best_gain = 0, best_j2 = j, best_c = 0, best_c2 = 0;
          for (uint32_t j2 = off[r]; j2 < off[r + 1]; ++j2) {
            if (j2 == j || rec[j2] == x) continue;
            const uint32_t t2 = j2 / K, l2 = t2 & 31;
            const size_t si2 = (size_t)(t2 / 32) * K + j2 % K;
            if (si2 == si) continue;  // same step: only the half-warp would change
            const uint32_t y = rec[j2];
            const uint32_t c1 = s.cost_with(m, l, y);
            if (c1 >= cost[si]) continue;  // the gain has to come from this step
            StepBanks& s2 = sb[si2];
            s2.add(l2, y, -1);
            const uint32_t c2 = s2.cost_with(s2.maxes(), l2, x);
            s2.add(l2, y, 1);
            const uint32_t before = cost[si] + cost[si2], after = c1 + c2;
            if (after < before && before - after > best_gain)
              best_gain = before - after, best_j2 = j2, best_c = c1, best_c2 = c2;
          }
          if (best_gain == 0) {
            s.add(l, x, 1);
            continue;
          }
          any = true;
          const uint32_t t2 = best_j2 / K, l2 = t2 & 31;
          const size_t si2 = (size_t)(t2 / 32) * K + best_j2 % K;
          const uint32_t y = rec[best_j2];
          sb[si2].add(l2, y, -1);
          sb[si2].add(l2, x, 1);
          s.add(l, y, 1);
          rec[j] = y, rec[best_j2] = x;
          cost[si] = best_c, cost[si2] = best_c2;
        }
      }
    if (!any) break;
  }
}

// One batch's entry.  Fails with TOC_E_CORRUPT for blocks the reference's tree build rejects, and
// TOC_E_ARG when slots or columns do not fit the 15/16-bit fields (the caller then keeps the
// chain-walk path).
int build_entry(const uint8_t* blk, const TocBlockMeta& m, LvlEntry& out) {
  constexpr uint32_t T = toc::kLvlThreads;
  if (m.status != TOC_OK) return m.status;
  if (m.corrupt) return TOC_E_CORRUPT;
  const uint32_t n = m.n_rows, nI = m.n_pairs, C = m.n_codes, nU = m.n_uniques;
  const uint64_t NT = 1ull + nI + m.n_derived;
  if (NT > (1ull << 26) || m.n_cols > 65536u || nU > 32768u || nI >= 32767u || n >= 32768u) return TOC_E_ARG;
  std::vector<uint32_t> off(n + 1), code(C);
  for (uint32_t r = 0; r <= n; ++r) off[r] = rd_packed(blk + m.off_offsets, r, m.w_offsets);
  for (uint32_t j = 0; j < C; ++j) code[j] = rd_packed(blk + m.off_codes, j, m.w_codes);
  std::vector<uint32_t> pcol(nI + 1), pref(nI + 1);
  for (uint32_t i = 0; i < nI; ++i) {
    pcol[i + 1] = rd_packed(blk + m.off_cols, i, m.w_cols);
    pref[i + 1] = rd_packed(blk + m.off_refs, i, m.w_refs);
  }
  // C' (codec.py:227-251): parent, first pair, key, depth of every node; ids 1..NT-1
  std::vector<uint32_t> par(NT, 0), first(NT, 0), key(NT, 0), depth(NT, 0);
  for (uint32_t i = 1; i <= nI; ++i) first[i] = key[i] = i, depth[i] = 1;
  uint32_t d = nI + 1;
  for (uint32_t r = 0; r < n; ++r) {
    for (uint32_t j = off[r]; j < off[r + 1]; ++j) {
      const uint32_t x = code[j];
      if (x < 1 || x >= d) return TOC_E_CORRUPT;
      if (j + 1 < off[r + 1]) {
        const uint32_t y = code[j + 1];
        if (y < 1 || y >= d) return TOC_E_CORRUPT;
        par[d] = x;
        first[d] = first[x];
        key[d] = first[y];
        depth[d] = depth[x] + 1;
        ++d;
      }
    }
  }
  // inner nodes: parents of the derived codes, closed under parents (children have larger ids)
  std::vector<uint8_t> inner(NT, 0);
  for (uint32_t j = 0; j < C; ++j)
    if (code[j] > nI && par[code[j]] > nI) inner[par[code[j]]] = 1;
  for (uint64_t x = NT - 1; x > nI; --x)
    if (inner[x] && par[x] > nI) inner[par[x]] = 1;
  // slots: 0 = zero; pairs by (column, id) -> 1..nI; inner nodes by (depth, id) -> nI+1..
  std::vector<uint32_t> slot(NT, 0), order;
  order.reserve(nI);
  for (uint32_t i = 1; i <= nI; ++i) order.push_back(i);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return pcol[x] < pcol[y]; });
  // Which of a column's pairs takes which of the column's slots is free too.  The column pass
  // walks slots [1 + tM, 1 + tM + M) in thread t, gathering each pair's value from the value index:
  // per iteration and half-warp, the 16 lanes' value refs should fall into distinct bank pairs (ref
  // mod 16; equal refs are a broadcast).  Column by column, each slot takes the remaining pair of
  // its column whose ref is least loaded in its (warp, iteration, half-warp) group so far.
  if (!getenv("TOC_LVL_PAIRS_PLAIN")) {
    const uint32_t M = ((nI + T - 1) / T) | 1u;
    std::vector<uint8_t> cnt((size_t)(T / 16) * M * 16, 0);       // [half-warp][iteration][bank pair]
    std::vector<uint16_t> grp((size_t)(T / 16) * M * 16, 0xffffu);  // refs already gathered by the group
    for (uint32_t k0 = 0; k0 < nI;) {
      uint32_t k1 = k0 + 1;
      while (k1 < nI && pcol[order[k1]] == pcol[order[k0]]) ++k1;
      for (uint32_t k = k0; k < k1; ++k) {
        const size_t g = ((size_t)(k / M / 16) * M + k % M) * 16;
        uint32_t best = k, bc = ~0u;
        for (uint32_t i = k; i < k1 && bc; ++i) {
          const uint32_t ref = pref[order[i]];
          uint32_t c = 1u + cnt[g + (ref & 15)];
          for (uint32_t e = 0; e < 16 && grp[g + e] != 0xffffu; ++e)
            if (grp[g + e] == ref) c = 0;
          if (c < bc) bc = c, best = i;
        }
        std::swap(order[k], order[best]);
        const uint32_t ref = pref[order[k]];
        if (bc) {  // a new word for the group
          ++cnt[g + (ref & 15)];
          for (uint32_t e = 0; e < 16; ++e)
            if (grp[g + e] == 0xffffu) {
              grp[g + e] = (uint16_t)ref;
              break;
            }
        }
      }
      k0 = k1;
    }
  }
  for (uint32_t k = 0; k < nI; ++k) slot[order[k]] = k + 1;
  std::vector<uint32_t> inn;
  for (uint64_t x = nI + 1; x < NT; ++x)
    if (inner[x]) inn.push_back((uint32_t)x);
  std::stable_sort(inn.begin(), inn.end(), [&](uint32_t x, uint32_t y) { return depth[x] < depth[y]; });
  const uint32_t nQ = (uint32_t)inn.size();
  if (1ull + nI + nQ > toc::kMaxSlots) return TOC_E_ARG;  // 15-bit slot references
  // Which inner node gets which inner slot is free (push and inner H touch pair slots only), and
  // the kernel's warps take 32 consecutive inner slots, level by level up their chains.  Within a
  // depth class (equal chain lengths: no divergence) each lane takes, from the next nodes of the
  // class, the one whose chain slots (own key, ancestors' keys, root pair) hit the least used banks
  // of its warp at every level: 32-bit banks of the low limb for the push atomics, bank pairs per
  // half-warp for the inner-H gathers.
  if (!getenv("TOC_LVL_INNER_PLAIN")) {
    constexpr uint32_t kLv = 8, kScan = 1024;  // levels tracked (deeper ones share the last), candidates scanned
    std::vector<uint32_t> placed;
    placed.reserve(nQ);
    std::vector<uint8_t> used(nQ, 0);
    uint8_t ca[kLv][32], ga[kLv][2][16];
    uint32_t lo = 0;  // first unplaced node of the sorted list
    auto refs_of = [&](uint32_t x, uint32_t* r) {  // chain references of node x, the root last
      uint32_t nl = 0;
      for (uint32_t y = x; y > nI; y = par[y]) {
        if (nl < kLv - 1) r[nl++] = toc::slot_ref(slot[key[y]]);
        if (par[y] <= nI) r[nl++] = toc::slot_ref(slot[par[y]]);
      }
      return nl;
    };
    for (uint32_t q = 0; q < nQ; ++q) {
      const uint32_t lane = q & 31, hf = lane >> 4;
      if (lane == 0) memset(ca, 0, sizeof ca), memset(ga, 0, sizeof ga);
      while (lo < nQ && used[lo]) ++lo;
      const uint32_t d0 = depth[inn[lo]];
      uint32_t best = lo, bc = ~0u, seen = 0;
      for (uint32_t i = lo; i < nQ && seen < kScan && depth[inn[i]] == d0 && bc; ++i) {
        if (used[i]) continue;
        ++seen;
        uint32_t r[kLv], c = 0;
        const uint32_t nl = refs_of(inn[i], r);
        for (uint32_t l = 0; l < nl; ++l) {
          const uint32_t lv = l + 1 == nl ? kLv - 1 : l;  // the root adds run converged, after the loop
          c += 4u * ca[lv][r[l] & 31] + 3u * ga[lv][hf][(r[l] >> 1) & 15];
        }
        if (c < bc) bc = c, best = i;
      }
      used[best] = 1;
      uint32_t r[kLv];
      const uint32_t nl = refs_of(inn[best], r);
      for (uint32_t l = 0; l < nl; ++l) {
        const uint32_t lv = l + 1 == nl ? kLv - 1 : l;
        ++ca[lv][r[l] & 31], ++ga[lv][hf][(r[l] >> 1) & 15];
      }
      placed.push_back(inn[best]);
    }
    inn.swap(placed);
  }
  for (uint32_t q = 0; q < nQ; ++q) slot[inn[q]] = nI + 1 + q;
  const uint32_t S = 1 + nI + nQ;
  // records in row order, one slot reference each: a code whose node has a slot is one record, a
  // leaf two (its parent's slot and its key's); an empty row is one record of slot 0 (a zero), so
  // every row ends with a flagged record and the kernel never searches for the next row
  std::vector<uint32_t> rec, rowid, roff(n + 1, 0);
  rec.reserve((size_t)C + C / 2 + n);
  rowid.reserve(rec.capacity());
  for (uint32_t r = 0; r < n; ++r) {
    roff[r] = (uint32_t)rec.size();
    for (uint32_t j = off[r]; j < off[r + 1]; ++j) {
      const uint32_t x = code[j];
      if (x <= nI || inner[x]) {
        rec.push_back(toc::slot_ref(slot[x]));
      } else {
        rec.push_back(toc::slot_ref(slot[par[x]]));
        rec.push_back(toc::slot_ref(slot[key[x]]));
      }
    }
    if (rec.size() == roff[r]) rec.push_back(0u);
    rowid.resize(rec.size(), r);
  }
  roff[n] = (uint32_t)rec.size();
  const uint32_t NR = (uint32_t)rec.size();
  // stream: thread t owns records [t*K, t*K + K); record k of thread t is the u16 at
  // (k/8)*8T + 8t + k%8
  uint32_t K = (NR + T - 1) / T;
  K = std::max(8u, (K + 7u) & ~7u);
  // serialize
  LvlHdr hd{};
  hd.nP = nI, hd.nQ = nQ, hd.S = S, hd.C = NR, hd.K = K, hd.T = T, hd.n_rows = n, hd.n_cols = m.n_cols, hd.nU = nU;
  uint32_t o = toc::kHdrBytes;
  auto sec = [&](uint64_t bytes) {
    const uint32_t s = o;
    o += toc::align16((uint32_t)bytes);
    return s;
  };
  hd.off_uniq = sec(8ull * nU);
  hd.off_rowoff = sec(4ull * (n + 1));
  hd.off_prs = sec(4ull * nI);
  hd.off_inner = sec(4ull * nQ);
  hd.off_colst = sec(2ull * (m.n_cols + 1));
  hd.off_trow = sec(2ull * T);
  hd.off_stream = sec(2ull * T * K);
  out.bytes.assign(o, 0);
  uint8_t* e = out.bytes.data();
  double vmax = 0.0;
  for (uint32_t i = 0; i < nU; ++i) {
    double x;
    memcpy(&x, blk + m.off_uniques + 8ull * i, 8);
    memcpy(e + hd.off_uniq + 8ull * i, &x, 8);
    vmax = std::max(vmax, std::fabs(x));
  }
  hd.vmax = vmax;
  hd.invK = (uint32_t)(0xffffffffu / K + 1u);
  hd.invM = (uint32_t)(0xffffffffu / (((nI + T - 1) / T) | 1u) + 1u);
  memcpy(e, &hd, sizeof hd);
  memcpy(e + hd.off_rowoff, roff.data(), 4ull * (n + 1));
  uint32_t* pr = reinterpret_cast<uint32_t*>(e + hd.off_prs);
  for (uint32_t k = 0; k < nI; ++k) {  // column | value ref << 16 | last-of-its-column << 31
    const bool last = k + 1 == nI || pcol[order[k + 1]] != pcol[order[k]];
    pr[k] = pcol[order[k]] | (pref[order[k]] << 16) | (last ? 0x80000000u : 0u);
  }
  uint32_t* ir = reinterpret_cast<uint32_t*>(e + hd.off_inner);
  for (uint32_t q = 0; q < nQ; ++q)  // references: parent | key << 16
    ir[q] = toc::slot_ref(slot[par[inn[q]]]) | (toc::slot_ref(slot[key[inn[q]]]) << 16);
  uint16_t* cs = reinterpret_cast<uint16_t*>(e + hd.off_colst);
  for (uint32_t c = 0, k = 0; c <= m.n_cols; ++c) {
    while (k < nI && pcol[order[k]] < c) ++k;
    cs[c] = (uint16_t)(k + 1);
  }
  schedule_banks(rec, rowid, roff, n, NR, K, T);
  {
    const char* e_ref = getenv("TOC_LVL_REFINE");  // experiment knob: local-search passes (default 2)
    const int passes = e_ref ? atoi(e_ref) : 2;
    if (passes > 0) refine_banks(rec, rowid, roff, NR, K, T, passes);
  }
  uint16_t* tr = reinterpret_cast<uint16_t*>(e + hd.off_trow);
  for (uint32_t t = 0; t < T && (uint64_t)t * K < NR; ++t) {
    const uint32_t r = rowid[t * K];
    tr[t] = (uint16_t)(r | (roff[r] == t * K ? 0x8000u : 0u));
  }
  uint16_t* st = reinterpret_cast<uint16_t*>(e + hd.off_stream);
  for (uint32_t j = 0; j < NR; ++j) {
    const uint32_t flag = j + 1 == roff[rowid[j] + 1] ? toc::kRowEnd : 0u;  // last record of its row
    const uint32_t t = j / K, k = j % K;
    st[(uint64_t)(k >> 3) * 8 * T + 8 * t + (k & 7u)] = (uint16_t)(rec[j] | flag);
  }
  out.S = S;
  out.stage = hd.off_stream;  // header included
  out.n_rows = n;
  return TOC_OK;
}

std::atomic<bool> g_lvl_traced{false};  // toc_levels_set_trace: launch the stamped kernel instances

}  // namespace

extern "C" void* toc_levels_build(const uint8_t* h_arena, const int64_t* h_block_off, const TocBlockMeta* h_meta,
                                  int64_t n_blocks, int32_t n_threads) {
  if (n_blocks < 0 || (n_blocks > 0 && (!h_arena || !h_block_off || !h_meta))) return nullptr;
  auto* c = new LvlCache;
  c->entries.resize((size_t)n_blocks);
  int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(n_blocks, 1));
  std::atomic<int64_t> next{0};
  auto work = [&]() {
    for (int64_t b; (b = next.fetch_add(1)) < n_blocks;) {
      LvlEntry& e = c->entries[(size_t)b];
      e.status = build_entry(h_arena + h_block_off[b], h_meta[b], e);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  for (const LvlEntry& e : c->entries) {
    if (e.status != TOC_OK && c->status == TOC_OK) c->status = e.status;
    c->total += (int64_t)e.bytes.size();
    c->max_slots = std::max<int32_t>(c->max_slots, (int32_t)e.S);
    c->max_stage = std::max<int32_t>(c->max_stage, (int32_t)e.stage);
    c->max_rows = std::max<int32_t>(c->max_rows, (int32_t)e.n_rows);
  }
  return c;
}

extern "C" int toc_levels_info(const void* handle, int64_t* total_bytes, int32_t* max_slots, int32_t* max_stage,
                               int32_t* max_rows) {
  const auto* c = static_cast<const LvlCache*>(handle);
  if (!c) return TOC_E_ARG;
  if (total_bytes) *total_bytes = c->total;
  if (max_slots) *max_slots = c->max_slots;
  if (max_stage) *max_stage = c->max_stage;
  if (max_rows) *max_rows = c->max_rows;
  return c->status;
}

extern "C" int toc_levels_copy(const void* handle, uint8_t* h_out, int64_t* h_off) {
  const auto* c = static_cast<const LvlCache*>(handle);
  if (!c || !h_off || (c->total > 0 && !h_out)) return TOC_E_ARG;
  if (c->status != TOC_OK) return c->status;
  int64_t o = 0;
  for (size_t b = 0; b < c->entries.size(); ++b) {
    h_off[b] = o;
    memcpy(h_out + o, c->entries[b].bytes.data(), c->entries[b].bytes.size());
    o += (int64_t)c->entries[b].bytes.size();
  }
  h_off[c->entries.size()] = o;
  return TOC_OK;
}

extern "C" int toc_levels_set_prefetch(int mode) {
  return cudaMemcpyToSymbol(toc::g_prefetch_mode, &mode, sizeof mode) == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_levels_set_trace(long long* d_trace) {
  if (cudaMemcpyToSymbol(toc::g_trace, &d_trace, sizeof d_trace) != cudaSuccess) return TOC_E_CUDA;
  g_lvl_traced.store(d_trace != nullptr);  // the stamped kernel instance is launched only then
  return TOC_OK;
}

extern "C" void toc_levels_free(void* handle) { delete static_cast<LvlCache*>(handle); }

extern "C" int64_t toc_levels_smem(int32_t kind, int32_t n_cols, int32_t max_slots, int32_t max_stage,
                                   int32_t max_rows) {
  if (n_cols < 0 || max_slots < 0 || max_stage < 0 || max_rows < 0) return -1;
  return toc::lvl_smem(kind, (uint32_t)n_cols, (uint32_t)max_slots, (uint32_t)max_stage, (uint32_t)max_rows).total;
}

extern "C" int toc_linalg_levels32(const int64_t* d_row_base, int64_t n_blocks, int32_t kind, int32_t n_cols,
                                   int32_t max_slots, int32_t max_stage, int32_t max_rows, const float* d_v,
                                   float* d_R, const float* d_u, float* d_O, const uint8_t* d_lvl,
                                   const int64_t* d_lvl_off, void* stream) {
  if (n_blocks < 0 || !(kind & (TOC_MATVEC | TOC_VECMAT)) || (kind & ~(TOC_MATVEC | TOC_VECMAT))) return TOC_E_ARG;
  if ((kind & TOC_MATVEC) && (!d_v || !d_R)) return TOC_E_ARG;
  if ((kind & TOC_VECMAT) && (!d_u || !d_O)) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  if (!d_row_base || !d_lvl || !d_lvl_off || n_cols < 0 || n_cols > 65536) return TOC_E_ARG;
  int dev = 0, sms = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TOC_E_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // the fp64 kernel's layout (the float arrays use the front of its double arrays)
  const int64_t smem = toc_levels_smem(kind, n_cols, max_slots, max_stage, max_rows);
  if (smem < 0 || smem > optin) return TOC_E_ARG;
  toc::Lvl32Args a{toc::lvl_smem(kind, (uint32_t)n_cols, (uint32_t)max_slots, (uint32_t)max_stage, (uint32_t)max_rows),
                   d_row_base, n_blocks, kind, n_cols, max_slots, max_stage, max_rows, d_lvl, d_lvl_off, d_v, d_R, d_u, d_O};
  void* fn = kind == TOC_MATVEC   ? (void*)toc::levels32_kernel<TOC_MATVEC>
             : kind == TOC_VECMAT ? (void*)toc::levels32_kernel<TOC_VECMAT>
                                  : (void*)toc::levels32_kernel<TOC_MATVEC | TOC_VECMAT>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return TOC_E_CUDA;
  const int64_t grid = std::min<int64_t>(n_blocks, (int64_t)TOC_LVL_CTAS_PER_SM * (sms > 0 ? sms : 148));
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(toc::kLvlThreads), args, (size_t)smem,
                          (cudaStream_t)stream) == cudaSuccess
             ? TOC_OK
             : TOC_E_CUDA;
}

extern "C" int toc_linalg_levels(const int64_t* d_row_base, int64_t n_blocks, int32_t kind, int32_t n_cols,
                                 int32_t max_slots, int32_t max_stage, int32_t max_rows, const double* d_v,
                                 double* d_R,
                                 const double* d_u, double* d_O, const uint8_t* d_lvl, const int64_t* d_lvl_off,
                                 void* stream) {
  if (n_blocks < 0 || !(kind & (TOC_MATVEC | TOC_VECMAT)) || (kind & ~(TOC_MATVEC | TOC_VECMAT))) return TOC_E_ARG;
  if ((kind & TOC_MATVEC) && (!d_v || !d_R)) return TOC_E_ARG;
  if ((kind & TOC_VECMAT) && (!d_u || !d_O)) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  if (!d_row_base || !d_lvl || !d_lvl_off || n_cols < 0 || n_cols > 65536) return TOC_E_ARG;
  int dev = 0, sms = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TOC_E_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int64_t smem = toc_levels_smem(kind, n_cols, max_slots, max_stage, max_rows);
  if (smem < 0 || smem > optin) return TOC_E_ARG;
  toc::LvlArgs a{toc::lvl_smem(kind, (uint32_t)n_cols, (uint32_t)max_slots, (uint32_t)max_stage, (uint32_t)max_rows),
                 d_row_base, n_blocks, kind, n_cols, max_slots, max_stage, max_rows, d_lvl, d_lvl_off, d_v, d_R, d_u, d_O};
  const bool tr = g_lvl_traced.load();
  void* fn = kind == TOC_MATVEC   ? (tr ? (void*)toc::levels_kernel<TOC_MATVEC, true> : (void*)toc::levels_kernel<TOC_MATVEC, false>)
             : kind == TOC_VECMAT ? (tr ? (void*)toc::levels_kernel<TOC_VECMAT, true> : (void*)toc::levels_kernel<TOC_VECMAT, false>)
             : (tr ? (void*)toc::levels_kernel<TOC_MATVEC | TOC_VECMAT, true>
                   : (void*)toc::levels_kernel<TOC_MATVEC | TOC_VECMAT, false>);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return TOC_E_CUDA;
  const int64_t grid = std::min<int64_t>(n_blocks, (int64_t)TOC_LVL_CTAS_PER_SM * (sms > 0 ? sms : 148));
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(toc::kLvlThreads), args, (size_t)smem,
                          (cudaStream_t)stream) == cudaSuccess
             ? TOC_OK
             : TOC_E_CUDA;
}
