// toc_index.cu -- parse and validate TOC1 blocks resident in HBM; one CTA per block.
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

// The checks run out of shared memory when the block fits kStageBytes (copied in once with 16-byte
// loads: the stages' scattered reads would otherwise each pay a global-memory latency, ~0.1 ms per
// block), else straight from global memory; the readers below use generic loads for both.
constexpr uint32_t kStageBytes = 110u * 1024u;

struct Cursor {
  const uint8_t* p;
  int64_t len;
};

__device__ __forceinline__ uint32_t gu32(const uint8_t* q) {
  return (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16) | ((uint32_t)q[3] << 24);
}

__device__ __forceinline__ uint32_t gpacked(const uint8_t* p, uint32_t i, uint32_t w) {
  const uint8_t* q = p + (size_t)i * w;
  switch (w) {
    case 1: return q[0];
    case 2: return (uint32_t)q[0] | ((uint32_t)q[1] << 8);
    case 3: return (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16);
    default: return gu32(q);
  }
}

__device__ __forceinline__ double gf64(const uint8_t* q) {
  const uint64_t lo = gu32(q), hi = gu32(q + 4);
  return __longlong_as_double((long long)(lo | (hi << 32)));
}

// Sequential reader of a packed section (one value per call), byte loads from either space.
template <int W>
struct GSeqReader {
  const uint8_t* q;
  __device__ __forceinline__ void init(const uint8_t* sec, uint32_t i0) { q = sec + (size_t)i0 * W; }
  __device__ __forceinline__ uint32_t next() {
    uint32_t v = q[0];
    if constexpr (W > 1) v |= (uint32_t)q[1] << 8;
    if constexpr (W > 2) v |= (uint32_t)q[2] << 16;
    if constexpr (W > 3) v |= (uint32_t)q[3] << 24;
    q += W;
    return v;
  }
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
  count = gu32(c.p + off);
  width = c.p[off + 4];
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

}  // namespace

// Parse + validate one block per CTA.  Thread 0 walks the header (a handful of fields); the
// per-element checks run block-wide, each stage recording its first failure (in the reference's
// scan order) with atomicMin, and stages run in the reference's order so the reported error is the
// one it would raise first.
__global__ void __launch_bounds__(256) index_blocks_kernel(const uint8_t* __restrict__ arena,
                                                           const int64_t* __restrict__ block_off,
                                                           const int64_t* __restrict__ block_len,
                                                           int64_t n_blocks,
                                                           TocBlockMeta* __restrict__ meta_out) {
  extern __shared__ __align__(16) uint8_t s_bytes[];
  __shared__ TocBlockMeta sm;
  __shared__ uint32_t s_warp[33];
  __shared__ uint32_t s_first, s_carry, s_ok;
  __shared__ unsigned long long s_first64;
  const int64_t b = blockIdx.x;
  if (b >= n_blocks) return;
  const uint32_t tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
  const Cursor g{arena + block_off[b], block_len[b]};
  bool staged = false;
  uint32_t head = 0;
  {
    // stage the 16-byte granules covering the block (each holds a block byte, so none can fault),
    // plus a zero guard for the readers' look-ahead
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(g.p) & ~(uintptr_t)15;
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(g.p) + (uintptr_t)max(g.len, (int64_t)0) + 15) & ~(uintptr_t)15;
    head = (uint32_t)(reinterpret_cast<uintptr_t>(g.p) - a0);
    if (g.len >= 0 && a1 - a0 + 16 <= kStageBytes) {
      const uint4* src = reinterpret_cast<const uint4*>(a0);
      uint4* dst = reinterpret_cast<uint4*>(s_bytes);
      const uint32_t n16 = (uint32_t)((a1 - a0) >> 4);
#pragma unroll 8
      for (uint32_t k = tid; k < n16; k += nth) dst[k] = __ldg(src + k);
      if (tid == 0) dst[n16] = make_uint4(0u, 0u, 0u, 0u);
      staged = true;
      __syncthreads();
    }
  }
  // the stages, instantiated separately for the staged copy (shared loads) and global memory
  auto validate = [&](const Cursor c) {

  // ---- stage A (thread 0): header up to the refs array ------------------------------------
  if (tid == 0) {
    TocBlockMeta m;
    memset(&m, 0, sizeof(m));
    uint32_t ok = 1;
    do {
      if (c.len < 4) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, 0, 0); ok = 0; break; }
      if (gu32(c.p) != 0x31434F54u) { fail(m, TOC_E_BAD_MAGIC, TOC_D_MAGIC, 0, 0); ok = 0; break; }
      if (c.len < 13) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, 4, 0); ok = 0; break; }
      const uint32_t version = c.p[4];
      m.n_rows = gu32(c.p + 5);
      m.n_cols = gu32(c.p + 9);
      if (version != 1) { fail(m, TOC_E_BAD_VERSION, TOC_D_VERSION, version, 0); ok = 0; break; }
      int64_t off = 13;
      if (off + 4 > c.len) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0); ok = 0; break; }
      m.n_uniques = gu32(c.p + off);
      off += 4;
      if (off + 8 * (int64_t)m.n_uniques > c.len) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0); ok = 0; break; }
      m.off_uniques = (uint32_t)off;
      off += 8 * (int64_t)m.n_uniques;
      if (off + 4 > c.len) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0); ok = 0; break; }
      const uint32_t i_count = gu32(c.p + off);
      off += 4;
      uint32_t cnt, w;
      int64_t payload, end;
      if (!packed_hdr(c, off, cnt, w, payload, end, m)) { ok = 0; break; }
      const uint32_t n_cols_arr = cnt;
      m.w_cols = (uint8_t)w;
      m.off_cols = (uint32_t)payload;
      off = end;
      if (!packed_hdr(c, off, cnt, w, payload, end, m)) { ok = 0; break; }
      m.w_refs = (uint8_t)w;
      m.off_refs = (uint32_t)payload;
      if (n_cols_arr != i_count || cnt != i_count) {
        fail(m, TOC_E_FORMAT, TOC_D_PAIR_COUNT, i_count, n_cols_arr); ok = 0; break;
      }
      m.n_pairs = i_count;
      m.off_codes = (uint32_t)end;  // temporarily: where the code count starts
    } while (0);
    sm = m;
    s_ok = ok;
    s_first = 0xffffffffu;
  }
  __syncthreads();
  if (s_ok) {  // ---- stage B: value refs in range (physical.py:155 -> :104-107) ------------
    const uint8_t* refs = c.p + sm.off_refs;
    const uint32_t wr = sm.w_refs, nu = sm.n_uniques, nI = sm.n_pairs;
    for (uint32_t i = tid; i < nI; i += nth)
      if (gpacked(refs, i, wr) >= nu) atomicMin(&s_first, i);
    __syncthreads();
    if (tid == 0 && s_first != 0xffffffffu) {
      fail(sm, TOC_E_FORMAT, TOC_D_REF_RANGE, s_first, gpacked(refs, s_first, wr));
      s_ok = 0;
    }
  }
  __syncthreads();
  if (s_ok && tid == 0) {  // ---- stage C (thread 0): rest of the header --------------------
    TocBlockMeta& m = sm;
    uint32_t ok = 1;
    do {
      int64_t off = m.off_codes;
      if (off + 4 > c.len) { fail(m, TOC_E_TRUNCATED, TOC_D_TRUNC, (uint32_t)off, 0); ok = 0; break; }
      const uint32_t total_codes = gu32(c.p + off);
      off += 4;
      uint32_t cnt, w;
      int64_t payload, end;
      if (!packed_hdr(c, off, cnt, w, payload, end, m)) { ok = 0; break; }
      if (cnt != total_codes) { fail(m, TOC_E_FORMAT, TOC_D_CODE_COUNT, total_codes, cnt); ok = 0; break; }
      m.n_codes = total_codes;
      m.w_codes = (uint8_t)w;
      m.off_codes = (uint32_t)payload;
      off = end;
      if (!packed_hdr(c, off, cnt, w, payload, end, m)) { ok = 0; break; }
      m.w_offsets = (uint8_t)w;
      m.off_offsets = (uint32_t)payload;
      off = end;
      if (off != c.len) { fail(m, TOC_E_FORMAT, TOC_D_TRAILING, (uint32_t)(c.len - off), 0); ok = 0; break; }
      if ((int64_t)cnt != (int64_t)m.n_rows + 1) { fail(m, TOC_E_FORMAT, TOC_D_OFFS_COUNT, m.n_rows + 1, cnt); ok = 0; break; }
      const uint32_t first = gpacked(c.p + m.off_offsets, 0, m.w_offsets);
      const uint32_t last = gpacked(c.p + m.off_offsets, m.n_rows, m.w_offsets);
      if (first != 0 || last != total_codes) { fail(m, TOC_E_FORMAT, TOC_D_OFFS_SPAN, first, last); ok = 0; break; }
    } while (0);
    s_ok = ok;
    s_first = 0xffffffffu;
  }
  __syncthreads();
  const uint8_t* offs = c.p + sm.off_offsets;
  const uint32_t wo = sm.w_offsets, n = sm.n_rows;
  if (s_ok) {  // ---- stage D: monotone offsets (physical.py:170-174) -------------------------
    for (uint32_t r = tid; r < n; r += nth)
      if (gpacked(offs, r, wo) > gpacked(offs, r + 1, wo)) atomicMin(&s_first, r);
    __syncthreads();
    if (tid == 0 && s_first != 0xffffffffu) {
      fail(sm, TOC_E_FORMAT, TOC_D_OFFS_MONO, s_first, 0);
      s_ok = 0;
    }
    if (tid == 0) s_first = 0xffffffffu;
  }
  __syncthreads();
  if (s_ok) {  // ---- stage E: LogicalEncoding pair checks (codec.py:154-158) -----------------
    const uint8_t* cols = c.p + sm.off_cols;
    const uint8_t* refs = c.p + sm.off_refs;
    const uint8_t* uniq = c.p + sm.off_uniques;
    const uint32_t wc = sm.w_cols, wr = sm.w_refs, nc = sm.n_cols;
    for (uint32_t i = tid; i < sm.n_pairs; i += nth) {
      bool bad = gpacked(cols, i, wc) >= nc;
      if (!bad) bad = !isfinite(gf64(uniq + 8u * gpacked(refs, i, wr)));
      if (bad) atomicMin(&s_first, i);
    }
    __syncthreads();
    if (tid == 0 && s_first != 0xffffffffu) {
      const uint32_t col = gpacked(cols, s_first, wc);
      if (col >= nc) fail(sm, TOC_E_FORMAT, TOC_D_PAIR_COL, s_first, col);
      else fail(sm, TOC_E_FORMAT, TOC_D_PAIR_VAL, s_first, col);
      s_ok = 0;
    }
  }
  __syncthreads();
  if (s_ok) {
    // ---- stage F: per-row code walk.  code >= 1 (codec.py:159-162, eager), derived-node
    // count, and the lazy undefined-node check of build_prefix_tree (codec.py:233-244): at
    // position j of row r, code[j] < 1 + |I| + D(r) + max(j - lo - 1, 0) with D(r) the nodes
    // derived by earlier rows.  Rows in chunks of blockDim: a block scan gives D(r), then each
    // thread walks its own row.
    if (tid == 0) {
      s_carry = 0;
      s_first64 = ~0ull;  // (row << 32 | code) of the first code < 1
      s_first = 0xffffffffu;  // flat position of the first undefined reference
    }
    __syncthreads();
    const uint8_t* codes = c.p + sm.off_codes;
    const uint32_t wk = sm.w_codes, nI = sm.n_pairs;
    for (uint32_t base = 0; base < n; base += nth) {
      const uint32_t r = base + tid;
      uint32_t lo = 0, hi = 0;
      if (r < n) {
        lo = gpacked(offs, r, wo);
        hi = gpacked(offs, r + 1, wo);
      }
      const uint32_t v = hi > lo ? hi - lo - 1 : 0u;
      const uint32_t x = warp_excl_scan(v, lane);
      if (lane == 31) s_warp[warp] = x + v;
      __syncthreads();
      if (warp == 0) {
        const uint32_t t = lane < nwarps ? s_warp[lane] : 0u;
        const uint32_t e = warp_excl_scan(t, lane);
        if (lane < nwarps) s_warp[lane] = e;
        if (lane == 31) s_warp[32] = e + t;
      }
      __syncthreads();
      const uint32_t D = s_carry + s_warp[warp] + x;
      if (r < n && hi > lo) {
        with_width(wk, [&]<int W>() {
          GSeqReader<W> rd;
          rd.init(codes, lo);
          bool undef = false;
          for (uint32_t j = lo; j < hi; ++j) {
            const uint32_t code = rd.next();
            if (code < 1) {
              atomicMin(&s_first64, ((unsigned long long)r << 32));
              break;
            }
            const uint64_t bound = 1ull + nI + D + (j > lo ? (uint64_t)(j - lo - 1) : 0ull);
            if ((uint64_t)code >= bound && !undef) {  // keep scanning: code < 1 outranks it
              atomicMin(&s_first, j);
              undef = true;
            }
          }
        });
      }
      __syncthreads();
      if (tid == 0) s_carry += s_warp[32];
      __syncthreads();
    }
    if (tid == 0) {
      sm.n_derived = s_carry;
      if (s_first64 != ~0ull) {
        fail(sm, TOC_E_FORMAT, TOC_D_CODE_LT1, (uint32_t)(s_first64 >> 32), 0);
      } else if (s_first != 0xffffffffu) {
        uint32_t lo = 0, hi = n;  // row containing flat position s_first
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) / 2;
          if (gpacked(offs, mid, wo) <= s_first) lo = mid;
          else hi = mid;
        }
        sm.corrupt = 1;
        sm.detail = TOC_D_UNDEF;
        sm.detail_a = lo;
        sm.detail_b = gpacked(codes, s_first, wk);
      }
    }
  }
  };
  if (staged) validate(Cursor{s_bytes + head, g.len});
  else validate(g);
  __syncthreads();
  if (tid == 0) meta_out[b] = sm;
}

}  // namespace toc

extern "C" int toc_index_blocks(const uint8_t* d_arena, const int64_t* d_block_off,
                                const int64_t* d_block_len, int64_t n_blocks, TocBlockMeta* d_meta,
                                void* stream) {
  if (n_blocks < 0) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(toc::index_blocks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)toc::kStageBytes) != cudaSuccess)
      return TOC_E_CUDA;
    attr = true;
  }
  toc::index_blocks_kernel<<<(unsigned)n_blocks, 256, toc::kStageBytes, (cudaStream_t)stream>>>(
      d_arena, d_block_off, d_block_len, n_blocks, d_meta);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}
