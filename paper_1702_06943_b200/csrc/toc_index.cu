// toc_index.cu -- parse and validate TOC1 blocks resident in HBM; one warp per block.
//
// Restates, on the device, the checks of the reference's deserialize_block
// (reference physical.py:138-186), LogicalEncoding.__post_init__ (codec.py:151-162) and the
// undefined-node checks of build_prefix_tree (codec.py:233-244), in the reference's order, so
// the first failing check is the one the reference would raise.  Format errors are eager (the
// reference raises them at deserialize time); the tree check is recorded in `corrupt` and raised
// lazily by the host API when a kernel first needs the tree (kernels.py:68-77).
#include "toc_common.cuh"

namespace toc {

namespace {

struct Cursor {
  const uint8_t* p;
  int64_t len;
};

__device__ void fail(TocBlockMeta& m, int status, uint32_t detail, uint32_t a, uint32_t b) {
  m.status = status;
  m.detail = detail;
  m.detail_a = a;
  m.detail_b = b;
}

// Header of a packed array (count u32 | width u8), physical.py:71-85.
__device__ bool packed_hdr(const Cursor& c, int64_t off, uint32_t& count, uint32_t& width,
                           int64_t& payload, int64_t& end, TocBlockMeta& m) {
  if (off + 5 > c.len) {
    fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0);
    return false;
  }
  count = ld_u32_unaligned(c.p + off);
  width = __ldg(c.p + off + 4);
  off += 5;
  if (width < 1 || width > 4) {
    fail(m, TOC_E_FORMAT, TOC_D_WIDTH, (uint32_t)(off - 1), width);
    return false;
  }
  payload = off;
  end = off + (int64_t)count * width;
  if (end > c.len) {
    fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0);
    return false;
  }
  return true;
}

// First index in [0, n) (in order) for which pred(i) holds, evaluated by the whole warp;
// returns n if none.
template <typename Pred>
__device__ uint32_t warp_first(uint32_t n, uint32_t lane, Pred pred) {
  for (uint32_t base = 0; base < n; base += 32) {
    uint32_t i = base + lane;
    bool bad = (i < n) && pred(i);
    uint32_t mask = __ballot_sync(0xffffffffu, bad);
    if (mask) return base + (uint32_t)(__ffs(mask) - 1);
  }
  return n;
}

}  // namespace

__global__ void __launch_bounds__(256) index_blocks_kernel(const uint8_t* __restrict__ arena,
                                                           const int64_t* __restrict__ block_off,
                                                           const int64_t* __restrict__ block_len,
                                                           int64_t n_blocks,
                                                           TocBlockMeta* __restrict__ meta_out) {
  const uint32_t lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (b >= n_blocks) return;
  Cursor c{arena + block_off[b], block_len[b]};
  TocBlockMeta m;
  memset(&m, 0, sizeof(m));
  m.status = TOC_OK;

  // ---- sequential header walk (lane-uniform: every lane computes it) -------------------
  uint32_t n_refs_arr = 0, i_count = 0, total_codes = 0, n_offs = 0;
  bool ok = true;
  do {
    if (c.len < 4) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, 0, 0); ok = false; break; }
    if (ld_u32_unaligned(c.p) != 0x31434F54u) {  // "TOC1" little-endian
      fail(m, TOC_E_BAD_MAGIC, TOC_D_MAGIC, 0, 0); ok = false; break;
    }
    if (c.len < 13) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, 4, 0); ok = false; break; }
    uint32_t version = __ldg(c.p + 4);
    m.n_rows = ld_u32_unaligned(c.p + 5);
    m.n_cols = ld_u32_unaligned(c.p + 9);
    if (version != 1) { fail(m, TOC_E_BAD_VERSION, TOC_D_VERSION, version, 0); ok = false; break; }
    int64_t off = 13;
    if (off + 4 > c.len) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0); ok = false; break; }
    m.n_uniques = ld_u32_unaligned(c.p + off);
    off += 4;
    if (off + 8 * (int64_t)m.n_uniques > c.len) {
      fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0); ok = false; break;
    }
    m.off_uniques = (uint32_t)off;
    off += 8 * (int64_t)m.n_uniques;
    if (off + 4 > c.len) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0); ok = false; break; }
    i_count = ld_u32_unaligned(c.p + off);
    off += 4;
    uint32_t cnt, w;
    int64_t payload, end;
    if (!packed_hdr(c, off, cnt, w, payload, end, m)) { ok = false; break; }
    uint32_t n_cols_arr = cnt;
    m.w_cols = (uint8_t)w;
    m.off_cols = (uint32_t)payload;
    off = end;
    if (!packed_hdr(c, off, cnt, w, payload, end, m)) { ok = false; break; }
    n_refs_arr = cnt;
    m.w_refs = (uint8_t)w;
    m.off_refs = (uint32_t)payload;
    off = end;
    if (n_cols_arr != i_count || n_refs_arr != i_count) {
      fail(m, TOC_E_FORMAT, TOC_D_PAIR_COUNT, i_count, n_cols_arr); ok = false; break;
    }
    m.n_pairs = i_count;
    // value_index_lookup range check, in pair order (physical.py:155 -> :104-107)
    const uint8_t* refs = c.p + m.off_refs;
    const uint32_t wr = m.w_refs, nu = m.n_uniques;
    uint32_t bad = warp_first(i_count, lane, [&](uint32_t i) { return ld_packed(refs, i, wr) >= nu; });
    if (bad < i_count) {
      fail(m, TOC_E_FORMAT, TOC_D_REF_RANGE, bad, ld_packed(refs, bad, wr)); ok = false; break;
    }
    if (off + 4 > c.len) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0); ok = false; break; }
    total_codes = ld_u32_unaligned(c.p + off);
    off += 4;
    if (!packed_hdr(c, off, cnt, w, payload, end, m)) { ok = false; break; }
    if (cnt != total_codes) { fail(m, TOC_E_FORMAT, TOC_D_CODE_COUNT, total_codes, cnt); ok = false; break; }
    m.n_codes = total_codes;
    m.w_codes = (uint8_t)w;
    m.off_codes = (uint32_t)payload;
    off = end;
    if (!packed_hdr(c, off, cnt, w, payload, end, m)) { ok = false; break; }
    n_offs = cnt;
    m.w_offsets = (uint8_t)w;
    m.off_offsets = (uint32_t)payload;
    off = end;
    if (off != c.len) {
      fail(m, TOC_E_FORMAT, TOC_D_TRAILING, (uint32_t)(c.len - off), 0); ok = false; break;
    }
    if ((int64_t)n_offs != (int64_t)m.n_rows + 1) {
      fail(m, TOC_E_FORMAT, TOC_D_OFFS_COUNT, m.n_rows + 1, n_offs); ok = false; break;
    }
  } while (0);

  if (ok) {
    const uint8_t* offs = c.p + m.off_offsets;
    const uint32_t wo = m.w_offsets;
    uint32_t first = ld_packed(offs, 0, wo), last = ld_packed(offs, m.n_rows, wo);
    if (first != 0 || last != total_codes) {
      fail(m, TOC_E_FORMAT, TOC_D_OFFS_SPAN, first, last);
      ok = false;
    }
  }
  if (ok) {  // monotone offsets (physical.py:170-174), first failing row
    const uint8_t* offs = c.p + m.off_offsets;
    const uint32_t wo = m.w_offsets;
    uint32_t bad = warp_first(m.n_rows, lane, [&](uint32_t r) {
      return ld_packed(offs, r, wo) > ld_packed(offs, r + 1, wo);
    });
    if (bad < m.n_rows) {
      fail(m, TOC_E_FORMAT, TOC_D_OFFS_MONO, bad, 0);
      ok = false;
    }
  }
  if (ok) {  // LogicalEncoding pair checks (codec.py:154-158), first failing pair
    const uint8_t* cols = c.p + m.off_cols;
    const uint8_t* refs = c.p + m.off_refs;
    const uint8_t* uniq = c.p + m.off_uniques;
    const uint32_t wc = m.w_cols, wr = m.w_refs, nc = m.n_cols;
    uint32_t bad = warp_first(m.n_pairs, lane, [&](uint32_t i) {
      if (ld_packed(cols, i, wc) >= nc) return true;
      double v = ld_f64_unaligned(uniq + 8u * ld_packed(refs, i, wr));
      return !isfinite(v);
    });
    if (bad < m.n_pairs) {
      uint32_t col = ld_packed(cols, bad, wc);
      if (col >= nc) fail(m, TOC_E_FORMAT, TOC_D_PAIR_COL, bad, col);
      else fail(m, TOC_E_FORMAT, TOC_D_PAIR_VAL, bad, col);
      ok = false;
    }
  }
  if (ok) {
    // Row walk: code >= 1 (codec.py:159-162, eager), count derived nodes, and the lazy
    // undefined-node check of build_prefix_tree (codec.py:233-244): at position j of row r
    // (rows' codes at flat positions lo..hi-1), code[j] must be < 1 + nI + D(r) + max(j-lo-1,0)
    // where D(r) counts the nodes derived by earlier rows.
    const uint8_t* offs = c.p + m.off_offsets;
    const uint8_t* codes = c.p + m.off_codes;
    const uint32_t wo = m.w_offsets, wk = m.w_codes, nI = m.n_pairs;
    uint32_t derived = 0;
    uint32_t lt1_row = 0xffffffffu, undef_row = 0xffffffffu, undef_code = 0;
    for (uint32_t r = 0; r < m.n_rows; ++r) {
      uint32_t lo = ld_packed(offs, r, wo), hi = ld_packed(offs, r + 1, wo);
      for (uint32_t base = lo; base < hi; base += 32) {
        uint32_t j = base + lane;
        uint32_t code = (j < hi) ? ld_packed(codes, j, wk) : 1u;
        bool lt1 = (j < hi) && code < 1;
        uint64_t bound = 1ull + nI + derived + (j > lo ? (uint64_t)(j - lo - 1) : 0ull);
        bool undef = (j < hi) && (uint64_t)code >= bound;
        uint32_t m1 = __ballot_sync(0xffffffffu, lt1);
        if (m1 && lt1_row == 0xffffffffu) lt1_row = r;
        uint32_t m2 = __ballot_sync(0xffffffffu, undef);
        if (m2 && undef_row == 0xffffffffu) {
          undef_row = r;
          undef_code = __shfl_sync(0xffffffffu, code, __ffs(m2) - 1);
        }
      }
      if (hi > lo) derived += hi - lo - 1;
    }
    m.n_derived = derived;
    if (lt1_row != 0xffffffffu) {
      fail(m, TOC_E_FORMAT, TOC_D_CODE_LT1, lt1_row, 0);
    } else if (undef_row != 0xffffffffu) {
      m.corrupt = 1;
      m.detail = TOC_D_UNDEF;
      m.detail_a = undef_row;
      m.detail_b = undef_code;
    }
  }
  if (lane == 0) meta_out[b] = m;
}

}  // namespace toc

extern "C" int toc_index_blocks(const uint8_t* d_arena, const int64_t* d_block_off,
                                const int64_t* d_block_len, int64_t n_blocks, TocBlockMeta* d_meta,
                                void* stream) {
  if (n_blocks < 0) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  const int warps = 8;
  int64_t grid = (n_blocks + warps - 1) / warps;
  toc::index_blocks_kernel<<<(unsigned)grid, warps * 32, 0, (cudaStream_t)stream>>>(
      d_arena, d_block_off, d_block_len, n_blocks, d_meta);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}
