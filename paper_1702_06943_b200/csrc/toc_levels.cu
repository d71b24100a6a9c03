// toc_levels.cu -- A.v and v^T.A over a breadth-first "level cache" of each batch's decode tree.
//
// Reference: codec.py:215-259 (build_prefix_tree, C'), kernels.py:115-142 (matvec, Algorithm 5:
// H[i] = value[i]*v[col[i]] + H[parent[i]], R[r] = sum_j H[D[r][j]]) and kernels.py:145-174 (vecmat,
// Algorithm 6: H[code] += u[row]; descending i: out[col[i]] += value[i]*H[i], H[parent[i]] += H[i]).
//
// The chain-walk kernel (toc_linalg.cu) visits every non-zero through a lane's private pointer
// chase: lanes of a warp walk chains of different lengths, so many issue slots idle, and v^T.A's
// scatter needs shared-memory atomics.  Here the tree is evaluated the way the reference's own
// recurrences run -- node by node -- but one LEVEL (tree depth) at a time, every lane busy:
//
//   cache entry (built once per arena on the host, the counterpart of the reference's cached
//   CompressedMatrix.tree, kernels.py:68-77): only the nodes some code uses (every parent of a
//   derived node is itself a code, so that set is closed under parents), renumbered breadth
//   first: the |I| pairs sorted by column, then depth-2 nodes, depth-3 nodes, ..., each level
//   sorted by its parents' new ids so siblings are contiguous.
//
//   A.v   P1[p] = value_p * v[col_p]                 pairs
//         H[x]  = P1[key_x] + H[par_x]                level 2, 3, ... (the reference's H, same operands)
//         R[r]  = sum of H over row r's codes         one warp per row
//   v^T.A S[x]  = sum of u[r] over x's occurrences   node-indexed occurrence rows
//         S[p] += sum of S over p's children          levels max..2, one thread per sibling run
//         O[c]  = sum over the pairs p of column c of value_p * (S[p] + sum of S[x] over the derived
//                 x whose key is p)                   pairs are column-sorted: a column is a range
// No atomics, every sum has a fixed order (deterministic fp64), and the only shared table is one
// fp64 slot per used node (H, then S).  DESIGN.md section 4.1.
#include <algorithm>
#include <atomic>
#include <thread>
#include <type_traits>
#include <vector>

#include "toc_batch.cuh"  // TMA bulk copy + mbarrier helpers

namespace toc {

// Entry header (80 B); section offsets relative to the entry start, 16-B aligned.
struct LvlHdr {
  uint32_t nP, nD, N, C;       // pairs, used derived nodes, N = nP + nD, codes
  uint32_t n_rows, maxd;       // rows; levels (depth of the deepest used node)
  uint32_t n_multi, n_runs;    // multi-occurrence records; sibling runs
  uint32_t n_csegs;            // distinct pair columns
  uint32_t off_lvl;            // u32[maxd + 1]: first new id of depth 1, 2, ..., then N
  uint32_t off_runlvl;         // u32[maxd + 1]: first run of the children at each level
  uint32_t off_prs;            // u32[nP]: column | value ref << 16 (pairs in new, column order)
  uint32_t off_nrec;           // u32[nD]: par | key << 16 (new ids; key is a pair)
  uint32_t off_codes;          // u16[C]: the code stream in new ids (row offsets: the TOC1 block)
  uint32_t off_occ;            // u8/u16[N]: the one row a node occurs in, or none / multi
  uint32_t off_multi;          // u32[n_multi]: node | row << 16, sorted by (node, row)
  uint32_t off_runs;           // u32[n_runs]: first child | parent << 16, per level by parent
  uint32_t off_kstart;         // u16[nP + 1]: start in kl of the derived nodes keyed by each pair
  uint32_t off_kl;             // u16[nD]: derived nodes sorted by (key, node)
  uint32_t off_csegs;          // u32[n_csegs + 1]: first pair | column << 16; sentinel nP
};
static_assert(sizeof(LvlHdr) == 80, "level cache header");

TOC_HD uint32_t occ_none(uint32_t w) { return w == 1 ? 0xffu : 0xffffu; }
TOC_HD uint32_t occ_multi(uint32_t w) { return w == 1 ? 0xfeu : 0xfffeu; }

struct LvlArgs {
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  const int64_t* row_base;
  int64_t n_blocks;
  int32_t kind, n_cols, max_uniques, max_rows;
  int32_t max_nodes, stage_bytes;  // shared staging area after the table (TMA copies of sections)
  const uint8_t* lvl;  // entries; occurrence width is 1 byte when every batch has <= 253 rows
  const int64_t* lvl_off;
  const double* v;
  double* R;
  const double* u;
  double* O;
};

TOC_D uint32_t ld16(const uint16_t* p) { return __ldg(p); }

// TMA bulk copy global -> shared completing on mbar (the caller announced the bytes).
TOC_D void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}
TOC_D uint32_t ld32(const uint32_t* p) { return __ldg(p); }

// U loads in flight per thread: every phase streams its records with U independent loads issued
// before any is used (one CTA per SM holds the whole table, so latency is hidden by ILP, not by
// other CTAs).
constexpr uint32_t kU = 4;
__constant__ int g_prefetch_mode = 0;  // tuning knob: L2 prefetch of the next entry (measured: costs DRAM re-reads)

template <int kKind, int OW>
__global__ void __launch_bounds__(1024, 1) levels_kernel(LvlArgs a) {
  constexpr bool MV = kKind & TOC_MATVEC, VM = kKind & TOC_VECMAT;
  constexpr uint32_t U = kU;
  using OccT = std::conditional_t<OW == 1, uint8_t, uint16_t>;
  constexpr uint32_t kNone = OW == 1 ? 0xffu : 0xffffu, kMulti = OW == 1 ? 0xfeu : 0xfffeu;
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
  const int32_t ncol = a.n_cols;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  double* v_s = reinterpret_cast<double*>(smem + 16);
  double* uniq_s = v_s + (MV ? ncol : 0);
  double* u_s = uniq_s + a.max_uniques;
  double* tab = u_s + (VM ? a.max_rows : 0);
  uint8_t* stage = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tab + a.max_nodes) + 15) & ~(uintptr_t)15);
  const uint32_t stage_bytes = (uint32_t)a.stage_bytes;
  uint32_t phase = 0;
  if (tid == 0) mbar_init(mbar, 1);
  if (MV)
    for (int32_t c = tid; c < ncol; c += nth) v_s[c] = a.v[c];

  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const uint8_t* ent = a.lvl + a.lvl_off[b];
    LvlHdr h;
    {
      const uint4* hp = reinterpret_cast<const uint4*>(ent);
      uint4 w[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) w[k] = __ldg(hp + k);
      memcpy(&h, w, sizeof h);
    }
    const uint8_t* blk = a.arena + a.block_off[b];
    const TocBlockMeta& mg = a.meta[b];
    const uint32_t nU = mg.n_uniques, off_uniq = mg.off_uniques;
    const int64_t rb = a.row_base[b];
    if (g_prefetch_mode && tid == 0 && b + gridDim.x < a.n_blocks) {
      const int64_t bn = b + gridDim.x;
      const uint32_t ebytes = (uint32_t)(a.lvl_off[bn + 1] - a.lvl_off[bn]) & ~15u;
      if (ebytes)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.lvl + a.lvl_off[bn]), "r"(ebytes) : "memory");
    }
    // sections the level loops read (parent/key records; sibling runs and key lists) go to shared
    // memory by TMA when they fit the staging area, overlapped with the streaming phases before them
    const uint32_t nrec_bytes = align16(4u * h.nD), runs_bytes = align16(4u * h.n_runs), kl_bytes = align16(2u * h.nD);
    const bool st_nrec = MV && h.nD && nrec_bytes <= stage_bytes;
    const bool st_runs = VM && h.n_runs && runs_bytes <= stage_bytes;
    const bool st_kl = VM && h.nD && runs_bytes + kl_bytes <= stage_bytes;
    auto stage_vm = [&]() {  // one thread; one mbarrier phase for both copies
      if (!st_runs && !st_kl) return;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)),
                   "r"((st_runs ? runs_bytes : 0u) + (st_kl ? kl_bytes : 0u))
                   : "memory");
      if (st_runs) bulk_copy(stage, ent + h.off_runs, runs_bytes, mbar);
      if (st_kl) bulk_copy(stage + runs_bytes, ent + h.off_kl, kl_bytes, mbar);
    };
    if (tid == 0) {
      if (st_nrec) bulk_load(stage, ent + h.off_nrec, nrec_bytes, mbar);
      else if (!MV) stage_vm();
    }
    for (uint32_t i = tid; i < nU; i += nth) uniq_s[i] = ld_f64_unaligned(blk + off_uniq + 8u * i);
    if (VM)
      for (uint32_t r = tid; r < h.n_rows; r += nth) u_s[r] = a.u[rb + r];
    const uint32_t* lvl = reinterpret_cast<const uint32_t*>(ent + h.off_lvl);
    const uint32_t* nrec = st_nrec ? reinterpret_cast<const uint32_t*>(stage)
                                   : reinterpret_cast<const uint32_t*>(ent + h.off_nrec);
    const uint32_t* prs = reinterpret_cast<const uint32_t*>(ent + h.off_prs);
    const uint32_t nP = h.nP, N = h.N;
    __syncthreads();

    if (MV) {
      // first layer: P1[p] = value_p * v[col_p] (the reference's H for depth-1 nodes)
      for (uint32_t p0 = tid; p0 < nP; p0 += U * nth) {
        uint32_t r[U];
#pragma unroll
        for (uint32_t k = 0; k < U; ++k) r[k] = p0 + k * nth < nP ? ld32(prs + p0 + k * nth) : 0u;
#pragma unroll
        for (uint32_t k = 0; k < U; ++k)
          if (p0 + k * nth < nP) tab[p0 + k * nth] = uniq_s[r[k] >> 16] * v_s[r[k] & 0xffffu];
      }
      __syncthreads();
      // H[x] = P1[key] + H[par], level by level (Algorithm 5's recurrence, same operands)
      if (st_nrec) {
        mbar_wait(mbar, phase);
        phase ^= 1u;
      }
      for (uint32_t d = 1; d < h.maxd; ++d) {
        const uint32_t lo = ld32(lvl + d), hi = ld32(lvl + d + 1);
        for (uint32_t x0 = lo + tid; x0 < hi; x0 += U * nth) {
          uint32_t r[U];
#pragma unroll
          for (uint32_t k = 0; k < U; ++k) r[k] = x0 + k * nth < hi ? nrec[x0 + k * nth - nP] : 0u;
#pragma unroll
          for (uint32_t k = 0; k < U; ++k)
            if (x0 + k * nth < hi) tab[x0 + k * nth] = tab[r[k] >> 16] + tab[r[k] & 0xffffu];
        }
        __syncthreads();
      }
      if (VM && tid == 0) {
        stage_vm();  // the staged records are no longer read (barrier above)
      }
      // R[r] = sum of H over the row's codes: one warp per row, U codes in flight per lane
      const uint8_t* offs = blk + mg.off_offsets;
      const uint32_t wo = mg.w_offsets;
      const uint16_t* codes = reinterpret_cast<const uint16_t*>(ent + h.off_codes);
      for (uint32_t r = warp; r < h.n_rows; r += nwarps) {
        const uint32_t j0 = ld_packed(offs, r, wo), j1 = ld_packed(offs, r + 1, wo);
        double s = 0.0;
        for (uint32_t j = j0 + lane; j < j1; j += 32 * U) {
          uint32_t c[U];
#pragma unroll
          for (uint32_t k = 0; k < U; ++k) c[k] = j + 32 * k < j1 ? ld16(codes + j + 32 * k) : 0xffffffffu;
#pragma unroll
          for (uint32_t k = 0; k < U; ++k)
            if (c[k] != 0xffffffffu) s += tab[c[k]];
        }
        s = warp_sum(s);
        if (lane == 0) a.R[rb + r] = s;
      }
      if (VM) __syncthreads();
    }

    if (VM) {
      double* o = a.O + b * (int64_t)ncol;
      for (int32_t c = tid; c < ncol; c += nth) o[c] = 0.0;  // columns no pair touches
      // S[x] = sum of u over x's occurrences as a code
      const OccT* occ = reinterpret_cast<const OccT*>(ent + h.off_occ);
      for (uint32_t x0 = tid; x0 < N; x0 += U * nth) {
        uint32_t r[U];
#pragma unroll
        for (uint32_t k = 0; k < U; ++k) r[k] = x0 + k * nth < N ? (uint32_t)__ldg(occ + x0 + k * nth) : kMulti;
#pragma unroll
        for (uint32_t k = 0; k < U; ++k) {
          if (r[k] < kMulti) tab[x0 + k * nth] = u_s[r[k]];
          else if (r[k] == kNone) tab[x0 + k * nth] = 0.0;
        }
      }
      const uint32_t* mrec = reinterpret_cast<const uint32_t*>(ent + h.off_multi);
      for (uint32_t k = tid; k < h.n_multi; k += nth) {  // nodes with several occurrences: the first
        const uint32_t e = ld32(mrec + k), x = e & 0xffffu;  // record of a run sums it in row order
        if (k > 0 && (ld32(mrec + k - 1) & 0xffffu) == x) continue;
        double s = u_s[e >> 16];
        for (uint32_t q = k + 1; q < h.n_multi; ++q) {
          const uint32_t f = ld32(mrec + q);
          if ((f & 0xffffu) != x) break;
          s += u_s[f >> 16];
        }
        tab[x] = s;
      }
      __syncthreads();
      // bottom-up: each parent adds its children's subtree sums (one sibling run per parent, in order)
      const uint32_t* runlvl = reinterpret_cast<const uint32_t*>(ent + h.off_runlvl);
      const uint32_t* runs = st_runs ? reinterpret_cast<const uint32_t*>(stage)
                                     : reinterpret_cast<const uint32_t*>(ent + h.off_runs);
      if (st_runs || st_kl) {
        mbar_wait(mbar, phase);
        phase ^= 1u;
      }
      for (uint32_t d = h.maxd - 1; d >= 1 && d < h.maxd; --d) {
        const uint32_t k0 = ld32(runlvl + d), k1 = ld32(runlvl + d + 1), hi = ld32(lvl + d + 1);
        for (uint32_t q0 = k0 + tid; q0 < k1; q0 += U * nth) {
          uint32_t e[U], f[U];
#pragma unroll
          for (uint32_t k = 0; k < U; ++k) {
            const uint32_t q = q0 + k * nth;
            e[k] = q < k1 ? runs[q] : 0u;
            f[k] = q + 1 < k1 ? runs[q + 1] & 0xffffu : hi;
          }
#pragma unroll
          for (uint32_t k = 0; k < U; ++k) {
            if (q0 + k * nth >= k1) continue;
            double s = 0.0;
            for (uint32_t y = e[k] & 0xffffu; y < f[k]; ++y) s += tab[y];
            tab[e[k] >> 16] += s;
          }
        }
        __syncthreads();
      }
      // O[c] = sum over column c's pairs p of value_p * (S[p] + sum of S[x] over the derived x keyed
      // by p), in (pair, node) order: 4 lanes per column, a fixed shuffle tree
      const uint16_t* kstart = reinterpret_cast<const uint16_t*>(ent + h.off_kstart);
      const uint16_t* kl = st_kl ? reinterpret_cast<const uint16_t*>(stage + runs_bytes)
                                 : reinterpret_cast<const uint16_t*>(ent + h.off_kl);
      const uint32_t* csegs = reinterpret_cast<const uint32_t*>(ent + h.off_csegs);
      const uint32_t quads = nth >> 2, span = ((h.n_csegs + quads - 1) / quads) * quads;
      for (uint32_t s = tid >> 2; s < span; s += quads) {
        double c = 0.0;
        uint32_t col = 0;
        if (s < h.n_csegs) {
          const uint32_t sg = ld32(csegs + s), end = ld32(csegs + s + 1) & 0xffffu;
          col = sg >> 16;
          for (uint32_t p0 = (sg & 0xffffu) + (tid & 3u); p0 < end; p0 += 4 * U) {
            uint32_t pr[U], ks[U], ke[U];
#pragma unroll
            for (uint32_t k = 0; k < U; ++k) {
              const uint32_t p = p0 + 4 * k;
              pr[k] = p < end ? ld32(prs + p) : 0u;
              ks[k] = p < end ? ld16(kstart + p) : 0u;
              ke[k] = p < end ? ld16(kstart + p + 1) : 0u;
            }
#pragma unroll
            for (uint32_t k = 0; k < U; ++k) {
              if (p0 + 4 * k >= end) continue;
              double g = tab[p0 + 4 * k];
              for (uint32_t q = ks[k]; q < ke[k]; ++q) g += tab[kl[q]];
              c += uniq_s[pr[k] >> 16] * g;
            }
          }
        }
        c += __shfl_xor_sync(0xffffffffu, c, 1);
        c += __shfl_xor_sync(0xffffffffu, c, 2);
        if (s < h.n_csegs && (tid & 3u) == 0) o[col] = c;
      }
    }
    __syncthreads();  // tables and staged vectors are reused by the next batch
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
  uint32_t N = 0;
  int status = TOC_OK;
};

struct LvlCache {
  std::vector<LvlEntry> entries;
  int64_t total = 0;
  int32_t max_nodes = 0;
  int32_t status = TOC_OK;
};

// One batch's entry.  Fails with TOC_E_CORRUPT for blocks the reference's tree build rejects, and
// TOC_E_ARG when ids do not fit the 16-bit fields (the caller then keeps the chain-walk path).
int build_entry(const uint8_t* blk, const TocBlockMeta& m, uint32_t ow, LvlEntry& out) {
  if (m.status != TOC_OK) return m.status;
  if (m.corrupt) return TOC_E_CORRUPT;
  const uint32_t n = m.n_rows, nI = m.n_pairs, C = m.n_codes;
  const uint64_t T = 1ull + nI + m.n_derived;
  if (T > (1ull << 26) || m.n_cols > 65536u || m.n_uniques > 65536u || n > 65533u || C > 0xffffffu) return TOC_E_ARG;
  std::vector<uint32_t> off(n + 1), code(C);
  for (uint32_t r = 0; r <= n; ++r) off[r] = rd_packed(blk + m.off_offsets, r, m.w_offsets);
  for (uint32_t j = 0; j < C; ++j) code[j] = rd_packed(blk + m.off_codes, j, m.w_codes);
  std::vector<uint32_t> pcol(nI + 1), pref(nI + 1);
  for (uint32_t i = 0; i < nI; ++i) {
    pcol[i + 1] = rd_packed(blk + m.off_cols, i, m.w_cols);
    pref[i + 1] = rd_packed(blk + m.off_refs, i, m.w_refs);
  }
  // C' (codec.py:227-251): parent, first pair, key, depth of every node; old ids 1..T-1
  std::vector<uint32_t> par(T, 0), first(T, 0), key(T, 0), depth(T, 0), cnt(T, 0);
  for (uint32_t i = 1; i <= nI; ++i) first[i] = key[i] = i, depth[i] = 1;
  uint32_t d = nI + 1;
  for (uint32_t r = 0; r < n; ++r) {
    for (uint32_t j = off[r]; j < off[r + 1]; ++j) {
      const uint32_t x = code[j];
      if (x < 1 || x >= d) return TOC_E_CORRUPT;
      ++cnt[x];
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
  // new ids: pairs by (column, old id); used derived nodes by depth, each level ordered by (new id
  // of the parent, old id)
  std::vector<uint32_t> nid(T, 0xffffffffu), order;  // order: old id of every new id
  for (uint32_t i = 1; i <= nI; ++i) order.push_back(i);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return pcol[x] < pcol[y]; });
  for (uint32_t k = 0; k < nI; ++k) nid[order[k]] = k;
  uint32_t maxd = nI ? 1u : 0u;
  for (uint64_t x = nI + 1; x < T; ++x)
    if (cnt[x]) maxd = std::max(maxd, depth[x]);
  std::vector<std::vector<uint32_t>> lv(maxd + 1);
  for (uint64_t x = nI + 1; x < T; ++x)
    if (cnt[x]) lv[depth[x]].push_back((uint32_t)x);
  std::vector<uint32_t> lvl_start{0u}, run_start{0u}, runs;
  if (maxd >= 1) {
    lvl_start.push_back(nI);
    run_start.push_back(0u);
  }
  for (uint32_t dd = 2; dd <= maxd; ++dd) {
    auto& L = lv[dd];
    std::stable_sort(L.begin(), L.end(), [&](uint32_t x, uint32_t y) { return nid[par[x]] < nid[par[y]]; });
    for (uint32_t x : L) {
      const uint32_t y = (uint32_t)order.size();
      if (y >= 65535u) return TOC_E_ARG;
      nid[x] = y;
      order.push_back(x);
      if (runs.empty() || y == lvl_start.back() || (runs.back() >> 16) != nid[par[x]]) runs.push_back(y | (nid[par[x]] << 16));
    }
    lvl_start.push_back((uint32_t)order.size());
    run_start.push_back((uint32_t)runs.size());
  }
  const uint32_t N = (uint32_t)order.size(), nD = N - nI;
  // occurrence rows
  const uint32_t none = toc::occ_none(ow), multi = toc::occ_multi(ow);
  std::vector<uint32_t> occ(N, none), mrec;
  for (uint32_t r = 0; r < n; ++r)
    for (uint32_t j = off[r]; j < off[r + 1]; ++j) {
      const uint32_t x = code[j], y = nid[x];
      if (cnt[x] == 1) occ[y] = r;
      else {
        occ[y] = multi;
        mrec.push_back(y | (r << 16));
      }
    }
  std::stable_sort(mrec.begin(), mrec.end(), [](uint32_t a, uint32_t b) { return (a & 0xffffu) < (b & 0xffffu); });
  // derived nodes grouped by key pair; column segments over the column-sorted pairs
  std::vector<uint32_t> kcount(nI + 1, 0), kl(nD);
  for (uint32_t k = 0; k < nD; ++k) ++kcount[nid[key[order[nI + k]]] + 1];
  std::vector<uint32_t> kstart(nI + 1, 0);
  for (uint32_t p = 0; p < nI; ++p) kstart[p + 1] = kstart[p] + kcount[p + 1];
  {
    std::vector<uint32_t> fill(kstart.begin(), kstart.end() - 1);
    for (uint32_t k = 0; k < nD; ++k) kl[fill[nid[key[order[nI + k]]]]++] = nI + k;  // ascending node
  }
  std::vector<uint32_t> csegs;
  for (uint32_t p = 0; p < nI; ++p)
    if (p == 0 || pcol[order[p]] != pcol[order[p - 1]]) csegs.push_back(p | (pcol[order[p]] << 16));
  const uint32_t n_csegs = (uint32_t)csegs.size();
  csegs.push_back(nI);
  // serialize
  LvlHdr hd{};
  hd.nP = nI, hd.nD = nD, hd.N = N, hd.C = C, hd.n_rows = n, hd.maxd = maxd;
  hd.n_multi = (uint32_t)mrec.size(), hd.n_runs = (uint32_t)runs.size(), hd.n_csegs = n_csegs;
  uint32_t o = sizeof(LvlHdr);
  auto sec = [&](uint32_t bytes) {
    const uint32_t s = o;
    o += toc::align16(bytes);
    return s;
  };
  hd.off_lvl = sec(4u * (uint32_t)lvl_start.size());
  hd.off_runlvl = sec(4u * (uint32_t)run_start.size());
  hd.off_prs = sec(4u * nI);
  hd.off_nrec = sec(4u * nD);
  hd.off_codes = sec(2u * C);
  hd.off_occ = sec(ow * N);
  hd.off_multi = sec(4u * hd.n_multi);
  hd.off_runs = sec(4u * hd.n_runs);
  hd.off_kstart = sec(2u * (nI + 1));
  hd.off_kl = sec(2u * nD);
  hd.off_csegs = sec(4u * (n_csegs + 1));
  out.bytes.assign(o, 0);
  uint8_t* e = out.bytes.data();
  memcpy(e, &hd, sizeof hd);
  memcpy(e + hd.off_lvl, lvl_start.data(), 4 * lvl_start.size());
  memcpy(e + hd.off_runlvl, run_start.data(), 4 * run_start.size());
  uint32_t* pr = reinterpret_cast<uint32_t*>(e + hd.off_prs);
  for (uint32_t p = 0; p < nI; ++p) pr[p] = pcol[order[p]] | (pref[order[p]] << 16);
  uint32_t* nr = reinterpret_cast<uint32_t*>(e + hd.off_nrec);
  for (uint32_t k = 0; k < nD; ++k) nr[k] = nid[par[order[nI + k]]] | (nid[key[order[nI + k]]] << 16);
  uint16_t* cd = reinterpret_cast<uint16_t*>(e + hd.off_codes);
  for (uint32_t j = 0; j < C; ++j) cd[j] = (uint16_t)nid[code[j]];
  for (uint32_t y = 0; y < N; ++y) {
    if (ow == 1) e[hd.off_occ + y] = (uint8_t)occ[y];
    else reinterpret_cast<uint16_t*>(e + hd.off_occ)[y] = (uint16_t)occ[y];
  }
  if (!mrec.empty()) memcpy(e + hd.off_multi, mrec.data(), 4 * mrec.size());
  if (!runs.empty()) memcpy(e + hd.off_runs, runs.data(), 4 * runs.size());
  uint16_t* ks = reinterpret_cast<uint16_t*>(e + hd.off_kstart);
  for (uint32_t p = 0; p <= nI; ++p) ks[p] = (uint16_t)kstart[p];
  uint16_t* klp = reinterpret_cast<uint16_t*>(e + hd.off_kl);
  for (uint32_t k = 0; k < nD; ++k) klp[k] = (uint16_t)kl[k];
  memcpy(e + hd.off_csegs, csegs.data(), 4 * csegs.size());
  out.N = N;
  return TOC_OK;
}

}  // namespace

extern "C" void* toc_levels_build(const uint8_t* h_arena, const int64_t* h_block_off, const TocBlockMeta* h_meta,
                                  int64_t n_blocks, int32_t n_threads) {
  if (n_blocks < 0 || (n_blocks > 0 && (!h_arena || !h_block_off || !h_meta))) return nullptr;
  auto* c = new LvlCache;
  c->entries.resize((size_t)n_blocks);
  int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(n_blocks, 1));
  uint32_t max_rows = 0;  // occurrence entries are one byte when every batch has <= 253 rows
  for (int64_t b = 0; b < n_blocks; ++b) max_rows = std::max(max_rows, h_meta[b].n_rows);
  const uint32_t ow = max_rows <= 253u ? 1u : 2u;
  std::atomic<int64_t> next{0};
  auto work = [&]() {
    for (int64_t b; (b = next.fetch_add(1)) < n_blocks;) {
      LvlEntry& e = c->entries[(size_t)b];
      e.status = build_entry(h_arena + h_block_off[b], h_meta[b], ow, e);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  for (const LvlEntry& e : c->entries) {
    if (e.status != TOC_OK && c->status == TOC_OK) c->status = e.status;
    c->total += (int64_t)e.bytes.size();
    c->max_nodes = std::max<int32_t>(c->max_nodes, (int32_t)e.N);
  }
  return c;
}

extern "C" int toc_levels_info(const void* handle, int64_t* total_bytes, int32_t* max_nodes) {
  const auto* c = static_cast<const LvlCache*>(handle);
  if (!c) return TOC_E_ARG;
  if (total_bytes) *total_bytes = c->total;
  if (max_nodes) *max_nodes = c->max_nodes;
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

extern "C" void toc_levels_free(void* handle) { delete static_cast<LvlCache*>(handle); }

extern "C" int64_t toc_levels_smem(int32_t kind, int32_t n_cols, int32_t max_nodes, int32_t max_rows,
                                   int32_t max_uniques) {
  return 16 + 8ll * (((kind & TOC_MATVEC) ? n_cols : 0) + max_uniques + ((kind & TOC_VECMAT) ? max_rows : 0) + max_nodes);
}

extern "C" int toc_linalg_levels(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                 const int64_t* d_row_base, int64_t n_blocks, int32_t kind, int32_t n_cols,
                                 int32_t max_nodes, int32_t max_rows, int32_t max_uniques, const double* d_v,
                                 double* d_R, const double* d_u, double* d_O, const uint8_t* d_lvl,
                                 const int64_t* d_lvl_off, void* stream) {
  if (n_blocks < 0 || !(kind & (TOC_MATVEC | TOC_VECMAT)) || (kind & ~(TOC_MATVEC | TOC_VECMAT))) return TOC_E_ARG;
  if ((kind & TOC_MATVEC) && (!d_v || !d_R)) return TOC_E_ARG;
  if ((kind & TOC_VECMAT) && (!d_u || !d_O)) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  if (!d_lvl || !d_lvl_off) return TOC_E_ARG;
  int dev = 0, sms = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int64_t need = toc_levels_smem(kind, n_cols, max_nodes, max_rows, max_uniques);
  if (need + 16 > optin) return TOC_E_ARG;
  const int64_t smem = optin;  // the rest is the TMA staging area
  const int32_t stage = (int32_t)((optin - need - 16) & ~15ll);
  toc::LvlArgs a{d_arena, d_block_off, d_meta, d_row_base, n_blocks, kind,  n_cols, max_uniques, max_rows,
                 max_nodes, stage,    d_lvl,  d_lvl_off,  d_v,      d_R,    d_u,   d_O};
  const bool narrow = max_rows <= 253;  // the builder's occurrence width rule
  void* fn;
  if (narrow)
    fn = kind == TOC_MATVEC   ? (void*)toc::levels_kernel<TOC_MATVEC, 1>
         : kind == TOC_VECMAT ? (void*)toc::levels_kernel<TOC_VECMAT, 1>
                              : (void*)toc::levels_kernel<TOC_MATVEC | TOC_VECMAT, 1>;
  else
    fn = kind == TOC_MATVEC   ? (void*)toc::levels_kernel<TOC_MATVEC, 2>
         : kind == TOC_VECMAT ? (void*)toc::levels_kernel<TOC_VECMAT, 2>
                              : (void*)toc::levels_kernel<TOC_MATVEC | TOC_VECMAT, 2>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return TOC_E_CUDA;
  const int64_t grid = std::min<int64_t>(n_blocks, sms > 0 ? sms : 148);
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(1024), args, (size_t)smem, (cudaStream_t)stream) == cudaSuccess
             ? TOC_OK
             : TOC_E_CUDA;
}
