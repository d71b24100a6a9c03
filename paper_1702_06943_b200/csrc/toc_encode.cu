// toc_encode.cu -- TOC compression on the device: row-bounded LZW encoding of many mini-batches
// at once, the value index, and packing into bit-exact TOC1 blocks.
//
// Reference: codec.py:112-139 (encode_rows), :177-191 (encode), physical.py:49-68 (widths,
// pack_ints), :88-101 (build_value_index), :110-130 (serialize_block), and the unpack side
// physical.py:71-85 / :138-186.
//
// One CTA encodes one mini-batch.  Per-batch open-addressing hash tables live in a global
// workspace (they are too large for shared memory at the configs' sizes):
//   value table  key = f64 bit pattern           -> slot index = internal value id
//   pair table   key = column << 32 | value id   -> min scan position, first-layer id
//   child table  key = parent code << 32 | pair  -> code of the child entry
// Seeding (codec.py:122-125) keeps the scan order of first occurrences: atomicMin of the
// element position per distinct pair, then a block scan over "is first occurrence" flags.
// Rows are encoded in order.  Within a row every start position's longest match is computed in
// parallel against the dictionary as it stood when the row began -- valid because an entry
// created while encoding row r starts at a column strictly left of any later match start in the
// same row (columns strictly increase, matrix.py:100-103), so it can never be matched in row r.
// One thread then walks the greedy chain (match, jump to its end) and the row's new entries
// (one per non-final code, codec.py:132-135) are inserted in parallel with consecutive codes.
// Codes are produced directly in the stored (decoder) numbering: first-layer pairs 1..|I|,
// derived entries |I|+1.. in creation order (codec.py:187-190).
#include "toc_common.cuh"

namespace toc {

namespace {

constexpr uint64_t kEmpty = ~0ull;
constexpr uint32_t kNone = 0xffffffffu;
constexpr int kEncThreads = 256;
constexpr uint32_t kRowCap = 1024;  // rows up to this length use shared-memory scratch

TOC_HD uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

TOC_HD int64_t hash_cap(int64_t nnz) {
  int64_t want = nnz + nnz / 2 + 16, cap = 32;
  while (cap < want) cap <<= 1;
  return cap;
}

TOC_D uint32_t hash_insert(uint64_t* keys, uint32_t cap, uint64_t k) {
  uint32_t s = (uint32_t)mix64(k) & (cap - 1);
  for (;;) {
    unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(keys + s), kEmpty, k);
    if (prev == kEmpty || prev == k) return s;
    s = (s + 1) & (cap - 1);
  }
}

TOC_D uint32_t hash_find(const uint64_t* keys, uint32_t cap, uint64_t k) {
  uint32_t s = (uint32_t)mix64(k) & (cap - 1);
  for (;;) {
    uint64_t cur = keys[s];
    if (cur == k) return s;
    if (cur == kEmpty) return kNone;
    s = (s + 1) & (cap - 1);
  }
}

TOC_D uint64_t f64_bits(double x) { return (uint64_t)__double_as_longlong(x); }

TOC_HD uint32_t int_width(uint64_t largest) {  // physical.py:49-51
  uint32_t w = 1;
  while (w < 4 && (largest >> (8 * w)) != 0) ++w;
  return w;
}

// Block-wide exclusive scan of data[0..n) in place; returns the total.  s_warp: 33 words.
TOC_D uint32_t block_scan(uint32_t* data, uint32_t n, uint32_t* s_warp) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < n; base += blockDim.x) {
    uint32_t i = base + tid;
    uint32_t v = i < n ? data[i] : 0u;
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
    if (i < n) data[i] = carry + s_warp[warp] + x;
    carry += s_warp[32];
    __syncthreads();
  }
  return carry;
}

TOC_D uint32_t block_max(uint32_t v, uint32_t* s_warp) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) s_warp[warp] = v;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < nwarps ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = max(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) s_warp[32] = t;
  }
  __syncthreads();
  uint32_t r = s_warp[32];
  __syncthreads();
  return r;
}

struct Work {  // carved from the caller's workspace (layout: toc_encode_sizes)
  int64_t* hash_base;  // n_batches + 1
  uint64_t* vkey;
  uint32_t* vmin;
  uint32_t* vidx;
  uint64_t* pkey;
  uint32_t* pmin;
  uint32_t* piid;
  uint64_t* ckey;
  uint32_t* cval;
  uint32_t* e_a;  // per element scratch
  uint32_t* e_b;
  uint32_t* e_c;
  uint32_t* e_d;
};

TOC_HD int64_t al256(int64_t x) { return (x + 255) & ~(int64_t)255; }

TOC_HD Work carve(uint8_t* base, int64_t n_batches, int64_t slots, int64_t n_elems) {
  Work w;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    uint8_t* p = base + o;
    o += al256(bytes);
    return p;
  };
  w.hash_base = (int64_t*)take(8 * (n_batches + 1));
  w.vkey = (uint64_t*)take(8 * slots);
  w.pkey = (uint64_t*)take(8 * slots);
  w.ckey = (uint64_t*)take(8 * slots);
  w.vmin = (uint32_t*)take(4 * slots);
  w.vidx = (uint32_t*)take(4 * slots);
  w.pmin = (uint32_t*)take(4 * slots);
  w.piid = (uint32_t*)take(4 * slots);
  w.cval = (uint32_t*)take(4 * slots);
  w.e_a = (uint32_t*)take(4 * (n_elems + 1));
  w.e_b = (uint32_t*)take(4 * (n_elems + 1));
  w.e_c = (uint32_t*)take(4 * (n_elems + 1));
  w.e_d = (uint32_t*)take(4 * (n_elems + 1));
  return w;
}

TOC_HD int64_t carve_bytes(int64_t n_batches, int64_t slots, int64_t n_elems) {
  return al256(8 * (n_batches + 1)) + 3 * al256(8 * slots) + 5 * al256(4 * slots) + 4 * al256(4 * (n_elems + 1));
}

}  // namespace

// Per-batch hash capacities and their exclusive prefix (single CTA; n_batches is modest).
__global__ void encode_prepare_kernel(int64_t n_batches, const int64_t* __restrict__ elem_base, Work w) {
  __shared__ int64_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n_batches; base += blockDim.x) {
    // simple serial prefix per chunk by thread 0 (n_batches is at most tens of thousands)
    if (threadIdx.x == 0) {
      int64_t c = s_carry;
      for (int64_t b = base; b < n_batches && b < base + blockDim.x; ++b) {
        w.hash_base[b] = c;
        c += hash_cap(elem_base[b + 1] - elem_base[b]);
      }
      s_carry = c;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) w.hash_base[n_batches] = s_carry;
}

struct EncodeArgs {
  int64_t n_batches;
  int32_t n_cols;
  const int64_t* row_ptr;    // CSR over all rows, int64 [n_rows_total + 1]
  const int32_t* cols;
  const double* vals;
  const int64_t* batch_row;  // [n_batches + 1]
  Work w;
  uint32_t* I_cols;          // element-indexed logical outputs (base row_ptr[batch_row[b]])
  double* I_vals;
  uint32_t* codes;
  uint32_t* offsets;         // indexed batch_row[b] + b
  TocBatchInfo* info;
};

__global__ void __launch_bounds__(kEncThreads) encode_kernel(EncodeArgs a) {
  __shared__ uint32_t s_warp[33];
  __shared__ uint32_t s_mcode[kRowCap], s_mend[kRowCap], s_npar[kRowCap], s_nkey[kRowCap], s_pid[kRowCap];
  __shared__ uint32_t s_cnt[2];
  __shared__ unsigned long long s_bad;
  const int64_t b = blockIdx.x;
  if (b >= a.n_batches) return;
  const uint32_t tid = threadIdx.x;
  const int64_t r0 = a.batch_row[b], r1 = a.batch_row[b + 1];
  const uint32_t n = (uint32_t)(r1 - r0);
  const int64_t e0 = a.row_ptr[r0];
  const uint32_t nnz = (uint32_t)(a.row_ptr[r1] - e0);
  const int64_t hb = a.w.hash_base[b];
  const uint32_t cap = (uint32_t)(a.w.hash_base[b + 1] - hb);
  uint64_t* vkey = a.w.vkey + hb;
  uint64_t* pkey = a.w.pkey + hb;
  uint64_t* ckey = a.w.ckey + hb;
  uint32_t* pmin = a.w.pmin + hb;
  uint32_t* piid = a.w.piid + hb;
  uint32_t* cval = a.w.cval + hb;
  uint32_t* e_ps = a.w.e_a + e0;   // pair slot per element
  uint32_t* e_pid = a.w.e_b + e0;  // value slot, then first-layer id per element
  uint32_t* e_flag = a.w.e_c + e0;
  const int32_t* cols = a.cols + e0;
  const double* vals = a.vals + e0;
  const int64_t* rp = a.row_ptr + r0;
  TocBatchInfo info;
  memset(&info, 0, sizeof(info));
  info.n_rows = n;
  info.n_cols = (uint32_t)a.n_cols;

  // ---- input contract of SparseRowMatrix (matrix.py:90-114): first offending element -----
  if (tid == 0) s_bad = ~0ull;
  __syncthreads();
  for (uint32_t r = tid >> 5; r < n; r += blockDim.x >> 5) {
    const uint32_t lo = (uint32_t)(rp[r] - e0), hi = (uint32_t)(rp[r + 1] - e0);
    for (uint32_t e = lo + (tid & 31); e < hi; e += 32) {
      int32_t c = cols[e];
      double v = vals[e];
      bool bad = c < 0 || c >= a.n_cols || (e > lo && c <= cols[e - 1]) || v == 0.0 || !isfinite(v);
      if (bad) atomicMin(&s_bad, ((unsigned long long)r << 32) | (e - lo));
    }
  }
  __syncthreads();
  if (s_bad != ~0ull) {
    if (tid == 0) {
      info.status = TOC_E_INPUT;
      info.detail_a = (uint32_t)(s_bad >> 32);
      info.detail_b = (uint32_t)(s_bad & 0xffffffffu);
      a.info[b] = info;
    }
    return;
  }

  // ---- hash tables ----------------------------------------------------------------------
  for (uint32_t s = tid; s < cap; s += blockDim.x) {
    vkey[s] = kEmpty;
    pkey[s] = kEmpty;
    ckey[s] = kEmpty;
    pmin[s] = kNone;
  }
  __syncthreads();
  for (uint32_t e = tid; e < nnz; e += blockDim.x) e_pid[e] = hash_insert(vkey, cap, f64_bits(vals[e]));
  __syncthreads();
  for (uint32_t e = tid; e < nnz; e += blockDim.x) {
    uint32_t ps = hash_insert(pkey, cap, ((uint64_t)(uint32_t)cols[e] << 32) | e_pid[e]);
    e_ps[e] = ps;
    atomicMin(&pmin[ps], e);
  }
  __syncthreads();
  // ---- seeding: distinct pairs in first-occurrence scan order (codec.py:122-125) ---------
  for (uint32_t e = tid; e < nnz; e += blockDim.x) e_flag[e] = pmin[e_ps[e]] == e ? 1u : 0u;
  __syncthreads();
  const uint32_t nI = block_scan(e_flag, nnz, s_warp);
  for (uint32_t e = tid; e < nnz; e += blockDim.x) {
    uint32_t ps = e_ps[e];
    if (pmin[ps] == e) {
      uint32_t iid = e_flag[e] + 1;
      piid[ps] = iid;
      a.I_cols[e0 + iid - 1] = (uint32_t)cols[e];
      a.I_vals[e0 + iid - 1] = vals[e];
    }
  }
  __syncthreads();
  for (uint32_t e = tid; e < nnz; e += blockDim.x) e_pid[e] = piid[e_ps[e]];
  __syncthreads();

  // ---- rows (codec.py:126-138) ------------------------------------------------------------
  uint32_t* out_codes = a.codes + e0;
  uint32_t* out_offs = a.offsets + r0 + b;
  uint32_t C = 0, next_id = nI + 1;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t lo = (uint32_t)(rp[r] - e0), L = (uint32_t)(rp[r + 1] - rp[r]);
    if (tid == 0) out_offs[r] = C;
    if (L == 0) continue;
    const uint32_t* P = e_pid + lo;
    if (L <= kRowCap) {  // the row's pair ids in shared memory: the match walks and the greedy
      for (uint32_t j = tid; j < L; j += blockDim.x) s_pid[j] = P[j];  // chain read them repeatedly
      P = s_pid;
      __syncthreads();
    }
    uint32_t* mcode = L <= kRowCap ? s_mcode : a.w.e_c + e0 + lo;  // e_c reused: seeding is done
    uint32_t* mend = L <= kRowCap ? s_mend : a.w.e_d + e0 + lo;
    uint32_t* npar = L <= kRowCap ? s_npar : a.w.e_a + e0 + lo;    // e_a reused likewise
    uint32_t* nkey = L <= kRowCap ? s_nkey : e_flag + lo;
    // longest match from every start position (get_longest_match, codec.py:90-109)
    for (uint32_t j = tid; j < L; j += blockDim.x) {
      uint32_t code = P[j], k = j + 1;
      while (k < L) {
        uint32_t s = hash_find(ckey, cap, ((uint64_t)code << 32) | P[k]);
        if (s == kNone) break;
        code = cval[s];
        ++k;
      }
      mcode[j] = code;
      mend[j] = k;
    }
    __syncthreads();
    if (tid == 0) {  // the greedy chain; new entries for non-final matches (codec.py:132-135)
      uint32_t j = 0, cnt = 0, nnew = 0;
      while (j < L) {
        uint32_t c = mcode[j], e = mend[j];
        out_codes[C + cnt++] = c;
        if (e < L) {
          npar[nnew] = c;
          nkey[nnew] = P[e];
          ++nnew;
        }
        j = e;
      }
      s_cnt[0] = cnt;
      s_cnt[1] = nnew;
    }
    __syncthreads();
    const uint32_t cnt = s_cnt[0], nnew = s_cnt[1];
    for (uint32_t t = tid; t < nnew; t += blockDim.x) {
      uint32_t s = hash_insert(ckey, cap, ((uint64_t)npar[t] << 32) | nkey[t]);
      cval[s] = next_id + t;
    }
    __syncthreads();
    C += cnt;
    next_id += nnew;
  }
  if (tid == 0) {
    out_offs[n] = C;
    info.n_pairs = nI;
    info.n_codes = C;
    info.status = TOC_OK;
    a.info[b] = info;
  }
}

// ---- serialization: value index, widths and sizes (physical.py:88-130) --------------------
struct SerialArgs {
  int64_t n_batches;
  const int64_t* batch_row;  // [n_batches + 1]: rows (offsets are at batch_row[b] + b)
  const int64_t* elem_base;  // [n_batches + 1]: base of each batch's pair / code arrays
  const uint32_t* I_cols;
  const double* I_vals;
  const uint32_t* codes;
  const uint32_t* offsets;
  Work w;
  uint32_t* refs;            // element-indexed
  double* uniques;           // element-indexed
  TocBatchInfo* info;        // in: n_rows, n_cols, n_pairs, n_codes; out: the rest
};

__global__ void __launch_bounds__(kEncThreads) serialize_sizes_kernel(SerialArgs a) {
  __shared__ uint32_t s_warp[33];
  const int64_t b = blockIdx.x;
  if (b >= a.n_batches) return;
  TocBatchInfo info = a.info[b];
  if (info.status != TOC_OK) return;
  const uint32_t tid = threadIdx.x;
  const int64_t e0 = a.elem_base[b];
  const int64_t hb = a.w.hash_base[b];
  const uint32_t cap = (uint32_t)(a.w.hash_base[b + 1] - hb);
  const uint32_t nI = info.n_pairs, C = info.n_codes, n = info.n_rows;
  uint64_t* vkey = a.w.vkey + hb;
  uint32_t* vmin = a.w.vmin + hb;
  uint32_t* vidx = a.w.vidx + hb;
  uint32_t* slot = a.w.e_a + e0;
  uint32_t* flag = a.w.e_b + e0;
  for (uint32_t s = tid; s < cap; s += blockDim.x) {
    vkey[s] = kEmpty;
    vmin[s] = kNone;
  }
  __syncthreads();
  for (uint32_t i = tid; i < nI; i += blockDim.x) {
    uint32_t s = hash_insert(vkey, cap, f64_bits(a.I_vals[e0 + i]));
    slot[i] = s;
    atomicMin(&vmin[s], i);
  }
  __syncthreads();
  for (uint32_t i = tid; i < nI; i += blockDim.x) flag[i] = vmin[slot[i]] == i ? 1u : 0u;
  __syncthreads();
  const uint32_t nU = block_scan(flag, nI, s_warp);
  for (uint32_t i = tid; i < nI; i += blockDim.x)
    if (vmin[slot[i]] == i) {
      vidx[slot[i]] = flag[i];
      a.uniques[e0 + flag[i]] = a.I_vals[e0 + i];
    }
  __syncthreads();
  uint32_t mc = 0, mk = 0;
  for (uint32_t i = tid; i < nI; i += blockDim.x) {
    a.refs[e0 + i] = vidx[slot[i]];
    mc = max(mc, a.I_cols[e0 + i]);
  }
  for (uint32_t p = tid; p < C; p += blockDim.x) mk = max(mk, a.codes[e0 + p]);
  mc = block_max(mc, s_warp);
  mk = block_max(mk, s_warp);
  if (tid == 0) {
    info.n_uniques = nU;
    info.w_cols = (uint8_t)int_width(mc);
    info.w_refs = (uint8_t)int_width(nU ? nU - 1 : 0);
    info.w_codes = (uint8_t)int_width(mk);
    info.w_offsets = (uint8_t)int_width(C);
    info.block_bytes = 4 + 9 + 4 + 8ll * nU + 4 + (5 + (int64_t)nI * info.w_cols) + (5 + (int64_t)nI * info.w_refs) +
                       4 + (5 + (int64_t)C * info.w_codes) + (5 + ((int64_t)n + 1) * info.w_offsets);
    a.info[b] = info;
  }
}

struct PackArgs {
  int64_t n_batches;
  const int64_t* batch_row;
  const int64_t* elem_base;
  const uint32_t* I_cols;
  const uint32_t* refs;
  const double* uniques;
  const uint32_t* codes;
  const uint32_t* offsets;
  const TocBatchInfo* info;
  const int64_t* block_off;
  uint8_t* arena;
};

TOC_D void put_u32(uint8_t* p, uint32_t x) {
  p[0] = (uint8_t)x;
  p[1] = (uint8_t)(x >> 8);
  p[2] = (uint8_t)(x >> 16);
  p[3] = (uint8_t)(x >> 24);
}

TOC_D void put_packed(uint8_t* p, uint32_t i, uint32_t w, uint32_t x) {
  uint8_t* q = p + (size_t)i * w;
  for (uint32_t k = 0; k < w; ++k) q[k] = (uint8_t)(x >> (8 * k));
}

__global__ void __launch_bounds__(kEncThreads) pack_kernel(PackArgs a) {
  const int64_t b = blockIdx.x;
  if (b >= a.n_batches) return;
  const TocBatchInfo info = a.info[b];
  if (info.status != TOC_OK) return;
  const uint32_t tid = threadIdx.x;
  const int64_t e0 = a.elem_base[b];
  const uint32_t nI = info.n_pairs, C = info.n_codes, n = info.n_rows, nU = info.n_uniques;
  const uint32_t wc = info.w_cols, wr = info.w_refs, wk = info.w_codes, wo = info.w_offsets;
  uint8_t* p = a.arena + a.block_off[b];
  const uint32_t o_uniq = 17, o_icount = o_uniq + 8 * nU, o_cols = o_icount + 4;
  const uint32_t o_refs = o_cols + 5 + nI * wc, o_ccount = o_refs + 5 + nI * wr;
  const uint32_t o_codes = o_ccount + 4, o_offs = o_codes + 5 + C * wk;
  if (tid == 0) {
    put_u32(p, 0x31434F54u);  // "TOC1"
    p[4] = 1;                 // VERSION
    put_u32(p + 5, n);
    put_u32(p + 9, info.n_cols);
    put_u32(p + 13, nU);
    put_u32(p + o_icount, nI);
    put_u32(p + o_cols, nI);
    p[o_cols + 4] = (uint8_t)wc;
    put_u32(p + o_refs, nI);
    p[o_refs + 4] = (uint8_t)wr;
    put_u32(p + o_ccount, C);
    put_u32(p + o_codes, C);
    p[o_codes + 4] = (uint8_t)wk;
    put_u32(p + o_offs, n + 1);
    p[o_offs + 4] = (uint8_t)wo;
  }
  for (uint32_t i = tid; i < nU; i += blockDim.x) {
    uint64_t bits = (uint64_t)__double_as_longlong(a.uniques[e0 + i]);
    put_u32(p + o_uniq + 8 * i, (uint32_t)bits);
    put_u32(p + o_uniq + 8 * i + 4, (uint32_t)(bits >> 32));
  }
  for (uint32_t i = tid; i < nI; i += blockDim.x) {
    put_packed(p + o_cols + 5, i, wc, a.I_cols[e0 + i]);
    put_packed(p + o_refs + 5, i, wr, a.refs[e0 + i]);
  }
  for (uint32_t q = tid; q < C; q += blockDim.x) put_packed(p + o_codes + 5, q, wk, a.codes[e0 + q]);
  const uint32_t* offs = a.offsets + a.batch_row[b] + b;
  for (uint32_t r = tid; r <= n; r += blockDim.x) put_packed(p + o_offs + 5, r, wo, offs[r]);
}

// ---- unpack (deserialize) indexed blocks into logical arrays (physical.py:138-186) ---------
struct UnpackArgs {
  int64_t n_blocks;
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  const int64_t* pair_base;
  const int64_t* code_base;
  const int64_t* offs_base;
  uint32_t* I_cols;
  double* I_vals;
  uint32_t* codes;
  uint32_t* offsets;
};

__global__ void __launch_bounds__(kEncThreads) unpack_kernel(UnpackArgs a) {
  const int64_t b = blockIdx.x;
  if (b >= a.n_blocks) return;
  const TocBlockMeta m = a.meta[b];
  if (m.status != TOC_OK) return;
  const uint8_t* blk = a.arena + a.block_off[b];
  for (uint32_t i = threadIdx.x; i < m.n_pairs; i += blockDim.x) {
    a.I_cols[a.pair_base[b] + i] = ld_packed(blk + m.off_cols, i, m.w_cols);
    a.I_vals[a.pair_base[b] + i] =
        ld_f64_unaligned(blk + m.off_uniques + 8u * ld_packed(blk + m.off_refs, i, m.w_refs));
  }
  for (uint32_t q = threadIdx.x; q < m.n_codes; q += blockDim.x)
    a.codes[a.code_base[b] + q] = ld_packed(blk + m.off_codes, q, m.w_codes);
  for (uint32_t r = threadIdx.x; r <= m.n_rows; r += blockDim.x)
    a.offsets[a.offs_base[b] + r] = ld_packed(blk + m.off_offsets, r, m.w_offsets);
}

}  // namespace toc

// ------------------------------------------------------------------------------------------
extern "C" int toc_encode_sizes(int64_t n_batches, const int64_t* h_elem_base, TocEncodeSizes* out) {
  if (!out || n_batches < 0 || (n_batches > 0 && !h_elem_base)) return TOC_E_ARG;
  int64_t slots = 0;
  for (int64_t b = 0; b < n_batches; ++b) {
    int64_t nnz = h_elem_base[b + 1] - h_elem_base[b];
    if (nnz < 0 || nnz > 0x7fffffffll) return TOC_E_ARG;
    slots += toc::hash_cap(nnz);
  }
  const int64_t n_elems = n_batches ? h_elem_base[n_batches] - h_elem_base[0] : 0;
  out->hash_slots = slots;
  out->n_elems = n_elems + (n_batches ? h_elem_base[0] : 0);
  out->work_bytes = toc::carve_bytes(n_batches, slots, out->n_elems);
  return TOC_OK;
}

extern "C" int toc_encode(int64_t n_batches, int32_t n_cols, const int64_t* d_row_ptr, const int32_t* d_cols,
                          const double* d_vals, const int64_t* d_batch_row, const int64_t* d_elem_base,
                          const TocEncodeSizes* sizes, void* d_work, uint32_t* d_I_cols, double* d_I_vals,
                          uint32_t* d_codes, uint32_t* d_offsets, TocBatchInfo* d_info, void* stream) {
  if (n_batches < 0 || !sizes || n_cols < 0) return TOC_E_ARG;
  if (n_batches == 0) return TOC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  toc::Work w = toc::carve((uint8_t*)d_work, n_batches, sizes->hash_slots, sizes->n_elems);
  toc::encode_prepare_kernel<<<1, 256, 0, s>>>(n_batches, d_elem_base, w);
  toc::EncodeArgs a{n_batches, n_cols, d_row_ptr, d_cols, d_vals, d_batch_row, w,
                    d_I_cols, d_I_vals, d_codes, d_offsets, d_info};
  toc::encode_kernel<<<(unsigned)n_batches, toc::kEncThreads, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_serialize_sizes(int64_t n_batches, const int64_t* d_batch_row, const int64_t* d_elem_base,
                                   const uint32_t* d_I_cols, const double* d_I_vals, const uint32_t* d_codes,
                                   const uint32_t* d_offsets, const TocEncodeSizes* sizes, void* d_work,
                                   uint32_t* d_refs, double* d_uniques, TocBatchInfo* d_info, void* stream) {
  if (n_batches < 0 || !sizes) return TOC_E_ARG;
  if (n_batches == 0) return TOC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  toc::Work w = toc::carve((uint8_t*)d_work, n_batches, sizes->hash_slots, sizes->n_elems);
  toc::encode_prepare_kernel<<<1, 256, 0, s>>>(n_batches, d_elem_base, w);
  toc::SerialArgs a{n_batches, d_batch_row, d_elem_base, d_I_cols, d_I_vals, d_codes, d_offsets,
                    w, d_refs, d_uniques, d_info};
  toc::serialize_sizes_kernel<<<(unsigned)n_batches, toc::kEncThreads, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_pack_blocks(int64_t n_batches, const int64_t* d_batch_row, const int64_t* d_elem_base,
                               const uint32_t* d_I_cols, const uint32_t* d_refs, const double* d_uniques,
                               const uint32_t* d_codes, const uint32_t* d_offsets, const TocBatchInfo* d_info,
                               const int64_t* d_block_off, uint8_t* d_arena, void* stream) {
  if (n_batches < 0) return TOC_E_ARG;
  if (n_batches == 0) return TOC_OK;
  toc::PackArgs a{n_batches, d_batch_row, d_elem_base, d_I_cols, d_refs, d_uniques, d_codes, d_offsets,
                  d_info, d_block_off, d_arena};
  toc::pack_kernel<<<(unsigned)n_batches, toc::kEncThreads, 0, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_unpack_blocks(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                 int64_t n_blocks, const int64_t* d_pair_base, const int64_t* d_code_base,
                                 const int64_t* d_offs_base, uint32_t* d_I_cols, double* d_I_vals,
                                 uint32_t* d_codes, uint32_t* d_offsets, void* stream) {
  if (n_blocks < 0) return TOC_E_ARG;
  if (n_blocks == 0) return TOC_OK;
  toc::UnpackArgs a{n_blocks, d_arena, d_block_off, d_meta, d_pair_base, d_code_base, d_offs_base,
                    d_I_cols, d_I_vals, d_codes, d_offsets};
  toc::unpack_kernel<<<(unsigned)n_blocks, toc::kEncThreads, 0, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}
