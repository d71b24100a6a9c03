// toc_levels.cu -- A.v and v^T.A over a breadth-first "level cache" of each batch's decode tree.
//
// Reference: codec.py:215-259 (build_prefix_tree, C'), kernels.py:115-142 (matvec, Algorithm 5:
// H[i] = value[i]*v[col[i]] + H[parent[i]], R[r] = sum_j H[D[r][j]]) and kernels.py:145-174 (vecmat,
// Algorithm 6: H[code] += u[row]; descending i: out[col[i]] += value[i]*H[i], H[parent[i]] += H[i]).
//
// The chain-walk kernel (toc_linalg.cu) visits every non-zero through a lane's private pointer
// chase (two random shared-memory reads per non-zero, lanes diverging on chain lengths).  Here the
// tree is evaluated the way the reference's own recurrences run -- node by node, one tree depth at
// a time -- so each used node is touched once:
//
//   cache entry (built once per arena on the host, the counterpart of the reference's cached
//   CompressedMatrix.tree, kernels.py:68-77): only the nodes some code uses (every parent of a
//   derived node is itself a code, so that set is closed under parents), renumbered breadth
//   first: the |I| pairs sorted by column, then depth-2 nodes, depth-3 nodes, ..., each level
//   sorted by its parents' new ids, so siblings are contiguous and every subtree occupies one
//   contiguous range per level.  The pairs (roots) are cut into 32 slices of similar subtree
//   weight, one per warp: the tree phases run warp by warp with no block-wide barrier per level.
//
//   A.v   P1[p] = value_p * v[col_p]                 pairs
//         H[x]  = P1[key_x] + H[par_x]                warp-local, depth 2, 3, ... (the reference's H)
//         R[r]  = sum of H over row r's codes         one warp per row
//   v^T.A S[x]  = sum of u[r] over x's occurrences   node-indexed occurrence rows
//         S[p] += sum of S over p's children          warp-local, depth max..2
//         G[p]  = S[p] + sum of S[x] over the derived x keyed by p
//         O[c]  = sum over column c's pairs of value_p * G[p]   (pairs are column-sorted: a range)
//   The three scatters (children -> parent, derived node -> key pair, occurrence -> node) walk
//   lists sorted by their target, 32 entries per warp step, and reduce equal targets with a warp
//   segmented scan before one plain read-modify-write per target (a target split across steps is
//   finished by the same warp in its next step).
// No atomics, every sum has a fixed order (deterministic fp64), and the only shared table is one
// fp64 slot per used node (H, then S).  DESIGN.md section 4.1.
#include <algorithm>
#include <atomic>
#include <thread>
#include <type_traits>
#include <vector>

#include "toc_batch.cuh"  // TMA bulk copy + mbarrier helpers

namespace toc {

constexpr uint32_t kSlices = 32;  // one per warp of the 1024-thread CTA

// Entry header (80 B); section offsets relative to the entry start, 16-B aligned.
struct LvlHdr {
  uint32_t nP, nD, N, C;       // pairs, used derived nodes, N = nP + nD, codes
  uint32_t n_rows, maxd;       // rows; levels (depth of the deepest used node)
  uint32_t n_multi, n_segs;    // multi-occurrence records; distinct pair columns
  uint32_t off_lvl;            // u32[maxd + 1]: first new id of depth 1, 2, ..., then N
  uint32_t off_prs;            // u32[nP]: column | value ref << 16 (pairs in new, column order)
  uint32_t off_nrec;           // u32[nD]: par | key << 16 (new ids; key is a pair)
  uint32_t off_codes;          // u16[C]: the code stream in new ids (row offsets: the TOC1 block)
  uint32_t off_occ;            // u8/u16[N]: the one row a node occurs in, or none / multi
  uint32_t off_multi;          // u32[n_multi]: node | row << 16, sorted by (node, row)
  uint32_t off_slnode;         // u16[maxd][33]: per depth-(d+1) level, first node of each slice
  uint32_t off_kl;             // u16[nD]: derived nodes sorted by (key pair, node)
  uint32_t off_wsplit;         // u16[2][33]: per warp, first kl entry / first multi record (cut at
                               // key / node boundaries)
  uint32_t off_segs;           // u32[n_segs + 1]: first pair | column << 16; sentinel nP
  uint32_t pad[2];
};
static_assert(sizeof(LvlHdr) == 80, "level cache header");

// Warp step of a scatter whose targets arrive sorted: lanes with equal `key` (contiguous) are
// summed by a segmented inclusive scan; returns true on the lane that holds its segment's sum
// (the segment's last lane in this step).  Invalid lanes must carry distinct keys.
TOC_D bool seg_reduce(double& v, uint32_t key, uint32_t lane) {
  // Hillis-Steele steps, stopping at the first distance no segment spans (segments are short)
#pragma unroll 1
  for (uint32_t o = 1; o < 32; o <<= 1) {
    const uint32_t k = __shfl_up_sync(0xffffffffu, key, o);
    const bool same = lane >= o && k == key;
    if (__ballot_sync(0xffffffffu, same) == 0u) break;
    const double t = __shfl_up_sync(0xffffffffu, v, o);
    if (same) v += t;
  }
  const uint32_t knext = __shfl_down_sync(0xffffffffu, key, 1);
  return lane == 31 || knext != key;
}

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
TOC_D uint32_t ld32(const uint32_t* p) { return __ldg(p); }

// TMA bulk copy global -> shared completing on mbar (the caller announced the bytes).
TOC_D void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}

constexpr uint32_t kU = 4;  // independent loads in flight per thread in the streaming phases
// L2 prefetch knob: 3 (default) = this batch's later sections at its start (measured 338 -> 310 us);
// 1 = the next batch's whole entry (measured: +90 MB DRAM re-reads, no gain); 0 = none.
__constant__ int g_prefetch_mode = 3;

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
    if (g_prefetch_mode == 3 && tid == 0) {  // this batch's later sections, ahead of their phases
      const uint32_t from = h.off_codes, ebytes = (uint32_t)(a.lvl_off[b + 1] - a.lvl_off[b]);
      if (ebytes > from)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ent + from), "r"((ebytes - from) & ~15u)
                     : "memory");
    }
    if (g_prefetch_mode == 1 && tid == 0 && b + gridDim.x < a.n_blocks) {
      const int64_t bn = b + gridDim.x;
      const uint32_t ebytes = (uint32_t)(a.lvl_off[bn + 1] - a.lvl_off[bn]) & ~15u;
      if (ebytes)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.lvl + a.lvl_off[bn]), "r"(ebytes) : "memory");
    }
    // the parent/key records (read by every tree phase) go to shared memory by TMA when they fit the
    // staging area, overlapped with the streaming phases before their first use
    const uint32_t nrec_bytes = align16(4u * h.nD);
    const bool st_nrec = h.nD && nrec_bytes <= stage_bytes;
    if (tid == 0 && st_nrec) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(nrec_bytes) : "memory");
      bulk_copy(stage, ent + h.off_nrec, nrec_bytes, mbar);
    }
    bool nrec_pending = st_nrec;
    const uint32_t* nrec = st_nrec ? reinterpret_cast<const uint32_t*>(stage)
                                   : reinterpret_cast<const uint32_t*>(ent + h.off_nrec);
    auto nrec_wait = [&]() {  // before the barrier that precedes nrec's first use
      if (nrec_pending) {
        mbar_wait(mbar, phase);
        phase ^= 1u;
        nrec_pending = false;
      }
    };
    for (uint32_t i = tid; i < nU; i += nth) uniq_s[i] = ld_f64_unaligned(blk + off_uniq + 8u * i);
    if (VM)
      for (uint32_t r = tid; r < h.n_rows; r += nth) u_s[r] = a.u[rb + r];
    const uint16_t* slnode = reinterpret_cast<const uint16_t*>(ent + h.off_slnode);
    const uint16_t* wsplit = reinterpret_cast<const uint16_t*>(ent + h.off_wsplit);
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
      nrec_wait();
      __syncthreads();
      // H[x] = P1[key] + H[par] (Algorithm 5's recurrence, same operands), this warp's slice of
      // every level in turn; parents are in the same slice one level up
      for (uint32_t d = 1; d < h.maxd; ++d) {
        const uint32_t lo = ld16(slnode + d * (kSlices + 1) + warp), hi = ld16(slnode + d * (kSlices + 1) + warp + 1);
        for (uint32_t x = lo + lane; x < hi; x += 32) {
          const uint32_t rec = nrec[x - nP];
          tab[x] = tab[rec >> 16] + tab[rec & 0xffffu];
        }
        __syncwarp();
      }
      __syncthreads();
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
      // S[x] = u of the one row x occurs in (nodes with several occurrences below; none: 0)
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
      // nodes with several occurrences: this warp's range of (node, row) records, summed in row order
      const uint32_t* mrec = reinterpret_cast<const uint32_t*>(ent + h.off_multi);
      {
        const uint32_t q0 = ld16(wsplit + (kSlices + 1) + warp), q1 = ld16(wsplit + (kSlices + 1) + warp + 1);
        uint32_t carry = 0xffffffffu;  // node of the previous step's last record
        for (uint32_t q = q0; q < q1; q += 32) {
          const bool ok = q + lane < q1;
          const uint32_t e = ok ? ld32(mrec + q + lane) : 0u;
          const uint32_t x = ok ? e & 0xffffu : 0xffff0000u + lane;
          double s = ok ? u_s[e >> 16] : 0.0;
          const uint32_t x0 = __shfl_sync(0xffffffffu, x, 0);
          if (seg_reduce(s, x, lane) && ok) {
            if (x == carry && x == x0) tab[x] += s;  // continues the previous step's run
            else tab[x] = s;
          }
          carry = __shfl_sync(0xffffffffu, x, 31);
          __syncwarp();
        }
      }
      nrec_wait();
      __syncthreads();
      // bottom-up, this warp's slice: S[par] += S[x] for depth max .. 2 (children sorted by parent)
      for (uint32_t d = h.maxd - 1; d >= 1 && d < h.maxd; --d) {
        const uint32_t lo = ld16(slnode + d * (kSlices + 1) + warp), hi = ld16(slnode + d * (kSlices + 1) + warp + 1);
        for (uint32_t x0 = lo; x0 < hi; x0 += 32) {
          const uint32_t x = x0 + lane;
          const bool ok = x < hi;
          const uint32_t p = ok ? nrec[x - nP] & 0xffffu : 0xffff0000u + lane;
          double s = ok ? tab[x] : 0.0;
          if (seg_reduce(s, p, lane) && ok) tab[p] += s;
          __syncwarp();
        }
      }
      __syncthreads();
      // G[p] = S[p] + sum of S[x] over the derived x keyed by p: this warp's range of the key-sorted
      // derived nodes
      const uint16_t* kl = reinterpret_cast<const uint16_t*>(ent + h.off_kl);
      {
        const uint32_t k0 = ld16(wsplit + warp), k1 = ld16(wsplit + warp + 1);
        for (uint32_t k = k0; k < k1; k += 32) {
          const bool ok = k + lane < k1;
          const uint32_t x = ok ? ld16(kl + k + lane) : 0u;
          const uint32_t p = ok ? nrec[x - nP] >> 16 : 0xffff0000u + lane;
          double s = ok ? tab[x] : 0.0;
          if (seg_reduce(s, p, lane) && ok) tab[p] += s;
          __syncwarp();
        }
      }
      __syncthreads();
      // O[c] = sum over column c's pairs p (a contiguous range) of value_p * G[p], in pair order:
      // 4 lanes per column, a fixed shuffle tree
      const uint32_t* segs = reinterpret_cast<const uint32_t*>(ent + h.off_segs);
      const uint32_t quads = nth >> 2, span = ((h.n_segs + quads - 1) / quads) * quads;
      for (uint32_t s = tid >> 2; s < span; s += quads) {
        double c = 0.0;
        uint32_t col = 0;
        if (s < h.n_segs) {
          const uint32_t sg = ld32(segs + s), end = ld32(segs + s + 1) & 0xffffu;
          col = sg >> 16;
          uint32_t p = (sg & 0xffffu) + (tid & 3u);
          for (; p + 4 < end; p += 8) {
            const uint32_t r0 = ld32(prs + p), r1 = ld32(prs + p + 4);
            c += uniq_s[r0 >> 16] * tab[p];
            c += uniq_s[r1 >> 16] * tab[p + 4];
          }
          if (p < end) c += uniq_s[ld32(prs + p) >> 16] * tab[p];
        }
        c += __shfl_xor_sync(0xffffffffu, c, 1);
        c += __shfl_xor_sync(0xffffffffu, c, 2);
        if (s < h.n_segs && (tid & 3u) == 0) o[col] = c;
      }
    } else {
      nrec_wait();  // (MV only: already waited)
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
  constexpr uint32_t W = toc::kSlices;
  if (m.status != TOC_OK) return m.status;
  if (m.corrupt) return TOC_E_CORRUPT;
  const uint32_t n = m.n_rows, nI = m.n_pairs, C = m.n_codes;
  const uint64_t T = 1ull + nI + m.n_derived;
  if (T > (1ull << 26) || m.n_cols > 65536u || m.n_uniques > 65536u || n > 65533u) return TOC_E_ARG;
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
  // of the parent, old id) -- so each pair's subtree is one contiguous range per level
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
  std::vector<uint32_t> lvl_start{0u};
  if (maxd >= 1) lvl_start.push_back(nI);
  for (uint32_t dd = 2; dd <= maxd; ++dd) {
    auto& L = lv[dd];
    std::stable_sort(L.begin(), L.end(), [&](uint32_t x, uint32_t y) { return nid[par[x]] < nid[par[y]]; });
    for (uint32_t x : L) {
      if (order.size() >= 65535u) return TOC_E_ARG;
      nid[x] = (uint32_t)order.size();
      order.push_back(x);
    }
    lvl_start.push_back((uint32_t)order.size());
  }
  const uint32_t N = (uint32_t)order.size(), nD = N - nI;
  // root pair of every new id; slices of the roots with similar subtree weight (one per warp)
  std::vector<uint32_t> root(N), npar(N, 0xffffffffu);
  for (uint32_t y = 0; y < nI; ++y) root[y] = y;
  for (uint32_t y = nI; y < N; ++y) {
    npar[y] = nid[par[order[y]]];
    root[y] = root[npar[y]];
  }
  std::vector<uint64_t> wsum(nI + 1, 0);  // prefix of per-root weight: 1 + derived nodes below
  {
    std::vector<uint32_t> wt(nI, 1);
    for (uint32_t y = nI; y < N; ++y) ++wt[root[y]];
    for (uint32_t p = 0; p < nI; ++p) wsum[p + 1] = wsum[p] + wt[p];
  }
  std::vector<uint32_t> rcut(W + 1, nI);  // slice w owns roots [rcut[w], rcut[w+1])
  rcut[0] = 0;
  for (uint32_t w = 1; w < W; ++w)
    rcut[w] = (uint32_t)(std::lower_bound(wsum.begin(), wsum.end(), wsum[nI] * w / W) - wsum.begin());
  for (uint32_t w = 1; w <= W; ++w) rcut[w] = std::max(std::min(rcut[w], nI), rcut[w - 1]);
  // per level, first node of each slice (nodes are ordered by root)
  std::vector<uint16_t> slnode((maxd + 1) * (W + 1), 0);
  for (uint32_t L = 1; L < maxd; ++L) {  // level index L = depth L + 1
    const uint32_t lo = lvl_start[L], hi = lvl_start[L + 1];
    uint32_t y = lo;
    for (uint32_t w = 0; w <= W; ++w) {
      if (w == W) y = hi;
      else
        while (y < hi && root[y] < rcut[w]) ++y;
      slnode[L * (W + 1) + w] = (uint16_t)y;
    }
  }
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
  if (mrec.size() > 65535u) return TOC_E_ARG;
  // derived nodes sorted by key pair; per-warp ranges of it and of the multi records, cut at
  // key / node boundaries; column segments over the pairs
  std::vector<uint32_t> kl(nD);
  for (uint32_t k = 0; k < nD; ++k) kl[k] = nI + k;
  auto kof = [&](uint32_t y) { return nid[key[order[y]]]; };
  std::stable_sort(kl.begin(), kl.end(), [&](uint32_t a, uint32_t b) { return kof(a) < kof(b); });
  std::vector<uint16_t> wsplit(2 * (W + 1), 0);
  auto cut = [&](uint32_t count, auto&& tgt, uint16_t* out) {
    uint32_t q = 0;
    for (uint32_t w = 0; w <= W; ++w) {
      q = std::max(q, (uint32_t)((uint64_t)count * w / W));
      while (q > 0 && q < count && tgt(q) == tgt(q - 1)) ++q;  // move to a target boundary
      out[w] = (uint16_t)(w == W ? count : q);
    }
  };
  cut(nD, [&](uint32_t k) { return kof(kl[k]); }, wsplit.data());
  cut((uint32_t)mrec.size(), [&](uint32_t k) { return mrec[k] & 0xffffu; }, wsplit.data() + (W + 1));
  std::vector<uint32_t> segs;
  for (uint32_t p = 0; p < nI; ++p)
    if (p == 0 || pcol[order[p]] != pcol[order[p - 1]]) segs.push_back(p | (pcol[order[p]] << 16));
  const uint32_t n_segs = (uint32_t)segs.size();
  segs.push_back(nI);
  // serialize
  LvlHdr hd{};
  hd.nP = nI, hd.nD = nD, hd.N = N, hd.C = C, hd.n_rows = n, hd.maxd = maxd;
  hd.n_multi = (uint32_t)mrec.size(), hd.n_segs = n_segs;
  uint32_t o = sizeof(LvlHdr);
  auto sec = [&](uint32_t bytes) {
    const uint32_t s = o;
    o += toc::align16(bytes);
    return s;
  };
  hd.off_lvl = sec(4u * (uint32_t)lvl_start.size());
  hd.off_prs = sec(4u * nI);
  hd.off_nrec = sec(4u * nD);
  hd.off_codes = sec(2u * C);
  hd.off_occ = sec(ow * N);
  hd.off_multi = sec(4u * hd.n_multi);
  hd.off_slnode = sec(2u * (uint32_t)slnode.size());
  hd.off_kl = sec(2u * nD);
  hd.off_wsplit = sec(2u * (uint32_t)wsplit.size());
  hd.off_segs = sec(4u * (n_segs + 1));
  out.bytes.assign(o, 0);
  uint8_t* e = out.bytes.data();
  memcpy(e, &hd, sizeof hd);
  memcpy(e + hd.off_lvl, lvl_start.data(), 4 * lvl_start.size());
  uint32_t* pr = reinterpret_cast<uint32_t*>(e + hd.off_prs);
  for (uint32_t p = 0; p < nI; ++p) pr[p] = pcol[order[p]] | (pref[order[p]] << 16);
  uint32_t* nr = reinterpret_cast<uint32_t*>(e + hd.off_nrec);
  for (uint32_t k = 0; k < nD; ++k) nr[k] = npar[nI + k] | (nid[key[order[nI + k]]] << 16);
  uint16_t* cd = reinterpret_cast<uint16_t*>(e + hd.off_codes);
  for (uint32_t j = 0; j < C; ++j) cd[j] = (uint16_t)nid[code[j]];
  for (uint32_t y = 0; y < N; ++y) {
    if (ow == 1) e[hd.off_occ + y] = (uint8_t)occ[y];
    else reinterpret_cast<uint16_t*>(e + hd.off_occ)[y] = (uint16_t)occ[y];
  }
  if (!mrec.empty()) memcpy(e + hd.off_multi, mrec.data(), 4 * mrec.size());
  memcpy(e + hd.off_slnode, slnode.data(), 2 * slnode.size());
  uint16_t* klp = reinterpret_cast<uint16_t*>(e + hd.off_kl);
  for (uint32_t k = 0; k < nD; ++k) klp[k] = (uint16_t)kl[k];
  memcpy(e + hd.off_wsplit, wsplit.data(), 2 * wsplit.size());
  memcpy(e + hd.off_segs, segs.data(), 4 * segs.size());
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
