/*
 * oracle/toc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference TOC algorithm (arXiv 1702.06943, reference package `toc`
 * under /root/reference/pkg/src/toc).  It is the parity checker for the B200 product path and the
 * CPU baseline timed by bench.py (`cpu_baseline`, `--impl reference`).  Nothing in the product
 * package (paper_1702_06943_b200/) may import, link or call it.
 *
 * Every function cites the reference file:line it restates.  Floating-point work follows the
 * reference's exact operation order (separate multiply and add, no FMA contraction: built with
 * -ffp-contract=off), so matvec / vecmat / matmat results are bit-identical to the Python
 * reference; the pins live in tests/golden (generated from the reference by
 * tests/golden/make_golden.py) and tests/test_oracle.py checks them.
 *
 * Codes are uint32 (a TOC1 block packs every integer in <= 4 bytes, physical.py:54-68).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_BAD_MAGIC 1   /* physical.py:33-34 BadMagicError            */
#define OR_BAD_VERSION 2 /* physical.py:37-38 UnsupportedVersionError  */
#define OR_TRUNCATED 3   /* physical.py:41-42 TruncatedBlockError      */
#define OR_FORMAT 4      /* physical.py:33 BlockFormatError            */
#define OR_CORRUPT 5     /* codec.py:33 CorruptEncodingError           */
#define OR_VALUE 6       /* ValueError (bad input)                     */
#define OR_NOMEM 7

/* Detail codes (second output) so the Python wrapper can rebuild the reference's messages. */
#define ORD_NONE 0
#define ORD_WIDTH 1      /* bytes_per_int must be 1..4              physical.py:77-78   */
#define ORD_PAIR_COUNT 2 /* pair count does not match               physical.py:159-162 */
#define ORD_CODE_COUNT 3 /* code count does not match               physical.py:168-169 */
#define ORD_TRAILING 4   /* trailing bytes after block              physical.py:171-172 */
#define ORD_OFFS_COUNT 5 /* expected n_rows+1 row offsets           physical.py:173-174 */
#define ORD_OFFS_SPAN 6  /* row offsets do not span the code array  physical.py:175-176 */
#define ORD_OFFS_MONO 7  /* row offsets not monotone                physical.py:180-181 */
#define ORD_REF_RANGE 8  /* value ref out of range                  physical.py:104-107 */
#define ORD_PAIR_COL 9   /* pair column out of range                codec.py:155-156    */
#define ORD_PAIR_VAL 10  /* pair value is not finite                codec.py:157-158    */
#define ORD_CODE_LT1 11  /* code is not a valid node                codec.py:159-162    */
#define ORD_UNDEF 12     /* code references an undefined node       codec.py:235-244    */
#define ORD_MAGIC 13
#define ORD_VERSION 14
#define ORD_TRUNC 15

/* ------------------------------------------------------------------------------------------ */
/* Open-addressing hash map with a two-word key.  Restates the Python dicts of
 * EncoderDictionary._children (codec.py:56,68,73) and build_value_index (physical.py:84).     */
typedef struct {
  uint64_t a, b;
  uint32_t v, used;
} or_slot;

typedef struct {
  or_slot* s;
  uint64_t cap; /* power of two */
  uint64_t n;
} or_map;

static uint64_t or_mix(uint64_t a, uint64_t b) {
  uint64_t h = a * 0x9E3779B97F4A7C15ull;
  h ^= b + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2);
  h ^= h >> 31;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 29;
  return h;
}

static int or_map_init(or_map* m, uint64_t expect) {
  uint64_t cap = 16;
  while (cap < 2 * expect + 2) cap <<= 1;
  m->s = (or_slot*)calloc(cap, sizeof(or_slot));
  m->cap = cap;
  m->n = 0;
  return m->s ? 0 : -1;
}

static void or_map_free(or_map* m) {
  free(m->s);
  m->s = NULL;
}

static int or_map_get(const or_map* m, uint64_t a, uint64_t b, uint32_t* v) {
  uint64_t i = or_mix(a, b) & (m->cap - 1);
  for (;;) {
    const or_slot* s = &m->s[i];
    if (!s->used) return 0;
    if (s->a == a && s->b == b) {
      *v = s->v;
      return 1;
    }
    i = (i + 1) & (m->cap - 1);
  }
}

static int or_map_grow(or_map* m) {
  or_map n2;
  if (or_map_init(&n2, m->cap) != 0) return -1;
  for (uint64_t i = 0; i < m->cap; i++)
    if (m->s[i].used) {
      uint64_t j = or_mix(m->s[i].a, m->s[i].b) & (n2.cap - 1);
      while (n2.s[j].used) j = (j + 1) & (n2.cap - 1);
      n2.s[j] = m->s[i];
      n2.n++;
    }
  free(m->s);
  *m = n2;
  return 0;
}

static int or_map_put(or_map* m, uint64_t a, uint64_t b, uint32_t v) {
  if (2 * (m->n + 1) > m->cap && or_map_grow(m) != 0) return -1;
  uint64_t i = or_mix(a, b) & (m->cap - 1);
  for (;;) {
    or_slot* s = &m->s[i];
    if (!s->used) {
      s->a = a;
      s->b = b;
      s->v = v;
      s->used = 1;
      m->n++;
      return 0;
    }
    if (s->a == a && s->b == b) {
      s->v = v;
      return 0;
    }
    i = (i + 1) & (m->cap - 1);
  }
}

static uint64_t or_bits(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
}

/* Dictionary key (parent working code, column, value): parent and column share word a.  Python
 * float equality equals bit equality here because stored values are finite and never zero
 * (matrix.py:100-107). */
#define OR_KEY_A(parent, col) (((uint64_t)(uint32_t)(parent) << 32) | (uint64_t)(uint32_t)(col))

/* ------------------------------------------------------------------------------------------ */
/* encode: codec.py:112-139 (encode_rows) + codec.py:177-191 (encode).
 * Input rows in CSR form.  Outputs (caller-allocated: capacity nnz for I and codes, n_rows+1 for
 * offsets) are the first-layer pairs I in first-emission order and the stored (decoder-numbered)
 * codes of every row, concatenated, plus row offsets.                                          */
int or_encode(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int32_t* cols,
              const double* vals, int64_t* out_nI, int32_t* I_cols, double* I_vals,
              int64_t* out_C, uint32_t* codes, int64_t* offsets) {
  const int64_t nnz = row_ptr[n_rows];
  or_map d;
  if (or_map_init(&d, (uint64_t)nnz + 16) != 0) return OR_NOMEM;
  /* Working codes 0..n_cols-1 are the per-column start markers (codec.py:52-55). */
  uint32_t next = (uint32_t)n_cols;
  /* Seed one entry per distinct pair, in scan order (codec.py:122-125): key (col, col, val). */
  int64_t nI = 0;
  for (int64_t e = 0; e < nnz; e++) {
    uint32_t got;
    uint64_t a = OR_KEY_A(cols[e], cols[e]), b = or_bits(vals[e]);
    if (!or_map_get(&d, a, b, &got)) {
      if (or_map_put(&d, a, b, next++) != 0) goto oom;
      I_cols[nI] = cols[e];
      I_vals[nI] = vals[e];
      nI++;
    }
  }
  /* Stored code = working code - (n_cols - 1) (codec.py:187-190). */
  const uint32_t shift = (uint32_t)(n_cols - 1);
  int64_t C = 0;
  for (int64_t r = 0; r < n_rows; r++) {
    offsets[r] = C;
    int64_t pos = row_ptr[r], end_row = row_ptr[r + 1];
    while (pos < end_row) {
      /* get_longest_match (codec.py:90-109) */
      uint32_t code;
      if (!or_map_get(&d, OR_KEY_A(cols[pos], cols[pos]), or_bits(vals[pos]), &code)) {
        or_map_free(&d);
        return OR_VALUE; /* codec.py:100-101: pair not present (cannot happen after seeding) */
      }
      int64_t p = pos + 1;
      while (p < end_row) {
        uint32_t nxt;
        if (!or_map_get(&d, OR_KEY_A(code, cols[p]), or_bits(vals[p]), &nxt)) break;
        code = nxt;
        p++;
      }
      if (p < end_row) {
        /* grow by the match plus one pair, never across the row boundary (codec.py:132-135) */
        if (or_map_put(&d, OR_KEY_A(code, cols[p]), or_bits(vals[p]), next++) != 0) goto oom;
      }
      codes[C++] = code - shift;
      pos = p;
    }
  }
  offsets[n_rows] = C;
  *out_nI = nI;
  *out_C = C;
  or_map_free(&d);
  return OR_OK;
oom:
  or_map_free(&d);
  return OR_NOMEM;
}

/* ------------------------------------------------------------------------------------------ */
/* TOC1 physical layout: physical.py:1-21 (layout), 49-68 (widths / pack_ints), 88-101 (value
 * index), 110-130 (serialize_block).                                                          */
static int or_int_width(uint64_t largest) { /* physical.py:49-51 */
  int bl = 0;
  while (largest) {
    bl++;
    largest >>= 1;
  }
  int w = (bl + 7) / 8;
  return w < 1 ? 1 : w;
}

static uint8_t* or_put_u32(uint8_t* p, uint32_t x) {
  p[0] = (uint8_t)x;
  p[1] = (uint8_t)(x >> 8);
  p[2] = (uint8_t)(x >> 16);
  p[3] = (uint8_t)(x >> 24);
  return p + 4;
}

static uint32_t or_get_u32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

/* pack_ints over a generic accessor (physical.py:54-68) */
typedef uint64_t (*or_getter)(const void* arr, int64_t i);
static uint64_t or_get_i32(const void* a, int64_t i) { return (uint64_t)((const int32_t*)a)[i]; }
static uint64_t or_get_u32a(const void* a, int64_t i) { return (uint64_t)((const uint32_t*)a)[i]; }
static uint64_t or_get_i64(const void* a, int64_t i) { return (uint64_t)((const int64_t*)a)[i]; }

static int64_t or_packed_size(const void* arr, int64_t n, or_getter g, int* width) {
  uint64_t largest = 0;
  for (int64_t i = 0; i < n; i++) {
    uint64_t v = g(arr, i);
    if (v > largest) largest = v;
  }
  *width = or_int_width(largest);
  return 5 + n * (int64_t)(*width);
}

static uint8_t* or_pack(uint8_t* p, const void* arr, int64_t n, or_getter g, int width) {
  p = or_put_u32(p, (uint32_t)n);
  *p++ = (uint8_t)width;
  for (int64_t i = 0; i < n; i++) {
    uint64_t v = g(arr, i);
    for (int k = 0; k < width; k++) *p++ = (uint8_t)(v >> (8 * k));
  }
  return p;
}

/* Value index: deduplicate by bit pattern in first-occurrence order (physical.py:88-101).
 * uniques/refs are caller-allocated with capacity nI.                                          */
int or_value_index(int64_t nI, const double* I_vals, int64_t* out_nU, double* uniques,
                   int32_t* refs) {
  or_map m;
  if (or_map_init(&m, (uint64_t)nI + 16) != 0) return OR_NOMEM;
  int64_t nU = 0;
  for (int64_t i = 0; i < nI; i++) {
    uint32_t r;
    uint64_t b = or_bits(I_vals[i]);
    if (!or_map_get(&m, 0, b, &r)) {
      r = (uint32_t)nU;
      if (or_map_put(&m, 0, b, r) != 0) {
        or_map_free(&m);
        return OR_NOMEM;
      }
      uniques[nU++] = I_vals[i];
    }
    refs[i] = (int32_t)r;
  }
  or_map_free(&m);
  *out_nU = nU;
  return OR_OK;
}

/* serialize_block (physical.py:110-130).  Call with out == NULL to get the size. */
int or_serialize(int64_t n_rows, int64_t n_cols, int64_t nI, const int32_t* I_cols,
                 const double* I_vals, int64_t C, const uint32_t* codes, const int64_t* offsets,
                 uint8_t* out, int64_t* out_len) {
  double* uniques = (double*)malloc(sizeof(double) * (size_t)(nI + 1));
  int32_t* refs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nI + 1));
  if (!uniques || !refs) {
    free(uniques);
    free(refs);
    return OR_NOMEM;
  }
  int64_t nU;
  int rc = or_value_index(nI, I_vals, &nU, uniques, refs);
  if (rc) {
    free(uniques);
    free(refs);
    return rc;
  }
  int wc, wr, wk, wo;
  int64_t size = 4 + 9 + 4 + 8 * nU + 4;
  size += or_packed_size(I_cols, nI, or_get_i32, &wc);
  size += or_packed_size(refs, nI, or_get_i32, &wr);
  size += 4 + or_packed_size(codes, C, or_get_u32a, &wk);
  size += or_packed_size(offsets, n_rows + 1, or_get_i64, &wo);
  *out_len = size;
  if (out) {
    uint8_t* p = out;
    memcpy(p, "TOC1", 4);
    p += 4;
    *p++ = 1; /* VERSION, physical.py:30 */
    p = or_put_u32(p, (uint32_t)n_rows);
    p = or_put_u32(p, (uint32_t)n_cols);
    p = or_put_u32(p, (uint32_t)nU);
    memcpy(p, uniques, (size_t)(8 * nU)); /* little-endian host */
    p += 8 * nU;
    p = or_put_u32(p, (uint32_t)nI);
    p = or_pack(p, I_cols, nI, or_get_i32, wc);
    p = or_pack(p, refs, nI, or_get_i32, wr);
    p = or_put_u32(p, (uint32_t)C);
    p = or_pack(p, codes, C, or_get_u32a, wk);
    p = or_pack(p, offsets, n_rows + 1, or_get_i64, wo);
  }
  free(uniques);
  free(refs);
  return OR_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* deserialize_block (physical.py:138-186) + LogicalEncoding validation (codec.py:151-162).
 * Pass 1 (arrays NULL) returns counts; pass 2 fills caller-allocated arrays.  On error *detail
 * names the failed check and *detail_off the byte offset / index involved.                    */
typedef struct {
  int64_t n_rows, n_cols, nU, nI, C;
  int64_t off_uniques, off_cols, off_refs, off_codes, off_offsets;
  int w_cols, w_refs, w_codes, w_offs;
} or_layout;

static int or_unpack_hdr(const uint8_t* data, int64_t len, int64_t off, int64_t* count,
                         int* width, int64_t* payload, int64_t* end, int64_t* detail,
                         int64_t* doff) {
  if (off + 5 > len) { /* physical.py:73-74 */
    *detail = ORD_TRUNC;
    *doff = off;
    return OR_TRUNCATED;
  }
  *count = or_get_u32(data + off);
  *width = data[off + 4];
  off += 5;
  if (*width < 1 || *width > 4) { /* physical.py:77-78 */
    *detail = ORD_WIDTH;
    *doff = off - 1;
    return OR_FORMAT;
  }
  *payload = off;
  *end = off + *count * (int64_t)*width;
  if (*end > len) { /* physical.py:79-83 */
    *detail = ORD_TRUNC;
    *doff = off;
    return OR_TRUNCATED;
  }
  return OR_OK;
}

static uint64_t or_read_w(const uint8_t* p, int w) {
  uint64_t v = 0;
  for (int k = 0; k < w; k++) v |= (uint64_t)p[k] << (8 * k);
  return v;
}

int or_parse_layout(const uint8_t* data, int64_t len, or_layout* L, int64_t* detail,
                    int64_t* doff) {
  *detail = ORD_NONE;
  *doff = 0;
  if (len < 4) { /* _need magic */
    *detail = ORD_TRUNC;
    return OR_TRUNCATED;
  }
  if (memcmp(data, "TOC1", 4) != 0) {
    *detail = ORD_MAGIC;
    return OR_BAD_MAGIC;
  }
  if (len < 13) {
    *detail = ORD_TRUNC;
    *doff = 4;
    return OR_TRUNCATED;
  }
  int version = data[4];
  L->n_rows = or_get_u32(data + 5);
  L->n_cols = or_get_u32(data + 9);
  if (version != 1) {
    *detail = ORD_VERSION;
    *doff = version;
    return OR_BAD_VERSION;
  }
  int64_t off = 13;
  if (off + 4 > len) {
    *detail = ORD_TRUNC;
    *doff = off;
    return OR_TRUNCATED;
  }
  L->nU = or_get_u32(data + off);
  off += 4;
  if (off + 8 * L->nU > len) {
    *detail = ORD_TRUNC;
    *doff = off;
    return OR_TRUNCATED;
  }
  L->off_uniques = off;
  off += 8 * L->nU;
  if (off + 4 > len) {
    *detail = ORD_TRUNC;
    *doff = off;
    return OR_TRUNCATED;
  }
  int64_t i_count = or_get_u32(data + off);
  off += 4;
  int64_t cnt, end;
  int rc;
  rc = or_unpack_hdr(data, len, off, &cnt, &L->w_cols, &L->off_cols, &end, detail, doff);
  if (rc) return rc;
  int64_t ncols_arr = cnt;
  off = end;
  rc = or_unpack_hdr(data, len, off, &cnt, &L->w_refs, &L->off_refs, &end, detail, doff);
  if (rc) return rc;
  int64_t nrefs_arr = cnt;
  off = end;
  if (ncols_arr != i_count || nrefs_arr != i_count) { /* physical.py:151-154 */
    *detail = ORD_PAIR_COUNT;
    *doff = i_count;
    return OR_FORMAT;
  }
  L->nI = i_count;
  /* value_index_lookup range check happens while building pairs (physical.py:155) */
  for (int64_t i = 0; i < L->nI; i++) {
    uint64_t r = or_read_w(data + L->off_refs + i * L->w_refs, L->w_refs);
    if ((int64_t)r >= L->nU) {
      *detail = ORD_REF_RANGE;
      *doff = (int64_t)r;
      return OR_FORMAT;
    }
  }
  if (off + 4 > len) {
    *detail = ORD_TRUNC;
    *doff = off;
    return OR_TRUNCATED;
  }
  int64_t total_codes = or_get_u32(data + off);
  off += 4;
  rc = or_unpack_hdr(data, len, off, &cnt, &L->w_codes, &L->off_codes, &end, detail, doff);
  if (rc) return rc;
  if (cnt != total_codes) { /* physical.py:160-161 */
    *detail = ORD_CODE_COUNT;
    *doff = total_codes;
    return OR_FORMAT;
  }
  L->C = total_codes;
  off = end;
  rc = or_unpack_hdr(data, len, off, &cnt, &L->w_offs, &L->off_offsets, &end, detail, doff);
  if (rc) return rc;
  off = end;
  if (off != len) { /* physical.py:163-164 */
    *detail = ORD_TRAILING;
    *doff = len - off;
    return OR_FORMAT;
  }
  if (cnt != L->n_rows + 1) { /* physical.py:165-166 */
    *detail = ORD_OFFS_COUNT;
    *doff = cnt;
    return OR_FORMAT;
  }
  if (cnt > 0) { /* physical.py:167-168 */
    uint64_t first = or_read_w(data + L->off_offsets, L->w_offs);
    uint64_t last = or_read_w(data + L->off_offsets + (cnt - 1) * L->w_offs, L->w_offs);
    if (first != 0 || (int64_t)last != total_codes) {
      *detail = ORD_OFFS_SPAN;
      return OR_FORMAT;
    }
  }
  for (int64_t r = 0; r < L->n_rows; r++) { /* physical.py:170-174 */
    uint64_t lo = or_read_w(data + L->off_offsets + r * L->w_offs, L->w_offs);
    uint64_t hi = or_read_w(data + L->off_offsets + (r + 1) * L->w_offs, L->w_offs);
    if (lo > hi) {
      *detail = ORD_OFFS_MONO;
      *doff = r;
      return OR_FORMAT;
    }
  }
  /* LogicalEncoding.__post_init__ (codec.py:151-162), surfaced as BlockFormatError
   * (physical.py:175-178). */
  for (int64_t i = 0; i < L->nI; i++) {
    uint64_t c = or_read_w(data + L->off_cols + i * L->w_cols, L->w_cols);
    if ((int64_t)c >= L->n_cols) {
      *detail = ORD_PAIR_COL;
      *doff = (int64_t)c;
      return OR_FORMAT;
    }
    uint64_t r = or_read_w(data + L->off_refs + i * L->w_refs, L->w_refs);
    double v;
    memcpy(&v, data + L->off_uniques + 8 * r, 8);
    if (!isfinite(v)) {
      *detail = ORD_PAIR_VAL;
      *doff = (int64_t)c;
      return OR_FORMAT;
    }
  }
  for (int64_t r = 0; r < L->n_rows; r++) {
    uint64_t lo = or_read_w(data + L->off_offsets + r * L->w_offs, L->w_offs);
    uint64_t hi = or_read_w(data + L->off_offsets + (r + 1) * L->w_offs, L->w_offs);
    for (uint64_t p = lo; p < hi; p++) {
      uint64_t code = or_read_w(data + L->off_codes + (int64_t)p * L->w_codes, L->w_codes);
      if (code < 1) {
        *detail = ORD_CODE_LT1;
        *doff = r;
        return OR_FORMAT;
      }
    }
  }
  return OR_OK;
}

/* Unpack a parsed block into arrays (caller-allocated by the sizes in the layout). */
int or_deserialize(const uint8_t* data, int64_t len, int64_t* dims /* n_rows,n_cols,nI,C */,
                   int32_t* I_cols, double* I_vals, uint32_t* codes, int64_t* offsets,
                   int64_t* detail, int64_t* doff) {
  or_layout L;
  int rc = or_parse_layout(data, len, &L, detail, doff);
  if (rc) return rc;
  dims[0] = L.n_rows;
  dims[1] = L.n_cols;
  dims[2] = L.nI;
  dims[3] = L.C;
  if (!I_cols) return OR_OK;
  for (int64_t i = 0; i < L.nI; i++) {
    I_cols[i] = (int32_t)or_read_w(data + L.off_cols + i * L.w_cols, L.w_cols);
    uint64_t r = or_read_w(data + L.off_refs + i * L.w_refs, L.w_refs);
    memcpy(&I_vals[i], data + L.off_uniques + 8 * r, 8);
  }
  for (int64_t p = 0; p < L.C; p++)
    codes[p] = (uint32_t)or_read_w(data + L.off_codes + p * L.w_codes, L.w_codes);
  for (int64_t r = 0; r <= L.n_rows; r++)
    offsets[r] = (int64_t)or_read_w(data + L.off_offsets + r * L.w_offs, L.w_offs);
  return OR_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Decode tree C' (codec.py:194-259).  parent/column/value arrays of length T = tree length;
 * node 0 is the root.  first_col/first_val are kept only while building (codec.py:225-251).   */
typedef struct {
  int64_t n_rows, n_cols, nI, C, T;
  int32_t* parent;
  int32_t* column;
  double* value;
  uint32_t* codes;  /* copy of D */
  int64_t* offsets; /* n_rows + 1 */
} or_tree;

void or_tree_free(or_tree* t) {
  if (!t) return;
  free(t->parent);
  free(t->column);
  free(t->value);
  free(t->codes);
  free(t->offsets);
  free(t);
}

/* build_prefix_tree (codec.py:215-259).  Returns NULL with *rc set on error. */
or_tree* or_tree_build(int64_t n_rows, int64_t n_cols, int64_t nI, const int32_t* I_cols,
                       const double* I_vals, int64_t C, const uint32_t* codes,
                       const int64_t* offsets, int* rc, int64_t* bad_row, int64_t* bad_code) {
  *rc = OR_OK;
  int64_t derived = 0;
  for (int64_t r = 0; r < n_rows; r++)
    if (offsets[r + 1] > offsets[r]) derived += offsets[r + 1] - offsets[r] - 1;
  int64_t T = 1 + nI + derived; /* LogicalEncoding.tree_length, codec.py:172-174 */
  or_tree* t = (or_tree*)calloc(1, sizeof(or_tree));
  if (!t) {
    *rc = OR_NOMEM;
    return NULL;
  }
  t->n_rows = n_rows;
  t->n_cols = n_cols;
  t->nI = nI;
  t->C = C;
  t->T = T;
  t->parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)T);
  t->column = (int32_t*)malloc(sizeof(int32_t) * (size_t)T);
  t->value = (double*)malloc(sizeof(double) * (size_t)T);
  int32_t* fcol = (int32_t*)malloc(sizeof(int32_t) * (size_t)T);
  double* fval = (double*)malloc(sizeof(double) * (size_t)T);
  t->codes = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(C + 1));
  t->offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
  if (!t->parent || !t->column || !t->value || !fcol || !fval || !t->codes || !t->offsets) {
    free(fcol);
    free(fval);
    or_tree_free(t);
    *rc = OR_NOMEM;
    return NULL;
  }
  memcpy(t->codes, codes, sizeof(uint32_t) * (size_t)C);
  memcpy(t->offsets, offsets, sizeof(int64_t) * (size_t)(n_rows + 1));
  t->parent[0] = -1; /* NOT_FOUND, codec.py:222-226 */
  t->column[0] = -1;
  t->value[0] = 0.0;
  fcol[0] = -1;
  fval[0] = 0.0;
  int64_t len = 1;
  for (int64_t i = 0; i < nI; i++, len++) { /* codec.py:227-232 */
    t->parent[len] = 0;
    t->column[len] = I_cols[i];
    t->value[len] = I_vals[i];
    fcol[len] = I_cols[i];
    fval[len] = I_vals[i];
  }
  for (int64_t r = 0; r < n_rows; r++) { /* codec.py:233-251 */
    for (int64_t p = offsets[r]; p < offsets[r + 1]; p++) {
      int64_t code = codes[p];
      if (!(code >= 1 && code < len)) {
        *rc = OR_CORRUPT;
        *bad_row = r;
        *bad_code = code;
        goto fail;
      }
      if (p + 1 < offsets[r + 1]) {
        int64_t nxt = codes[p + 1];
        if (!(nxt >= 1 && nxt < len)) {
          *rc = OR_CORRUPT;
          *bad_row = r;
          *bad_code = nxt;
          goto fail;
        }
        t->parent[len] = (int32_t)code;
        t->column[len] = fcol[nxt];
        t->value[len] = fval[nxt];
        fcol[len] = fcol[code];
        fval[len] = fval[code];
        len++;
      }
    }
  }
  free(fcol);
  free(fval);
  return t;
fail:
  free(fcol);
  free(fval);
  or_tree_free(t);
  return NULL;
}

int64_t or_tree_len(const or_tree* t) { return t->T; }

void or_tree_arrays(const or_tree* t, int32_t* parent, int32_t* column, double* value) {
  memcpy(parent, t->parent, sizeof(int32_t) * (size_t)t->T);
  memcpy(column, t->column, sizeof(int32_t) * (size_t)t->T);
  memcpy(value, t->value, sizeof(double) * (size_t)t->T);
}

/* matvec, Algorithm 5 (kernels.py:115-142): H ascending, separate multiply and add (no FMA),
 * then left-to-right row sums from 0.0.  h is caller scratch of length T.                     */
void or_matvec(const or_tree* t, const double* v, double* out, double* h) {
  h[0] = 0.0;
  for (int64_t i = 1; i < t->T; i++) {
    double prod = t->value[i] * v[t->column[i]];
    h[i] = prod + h[t->parent[i]];
  }
  for (int64_t r = 0; r < t->n_rows; r++) {
    double acc = 0.0;
    for (int64_t p = t->offsets[r]; p < t->offsets[r + 1]; p++) acc += h[t->codes[p]];
    out[r] = acc;
  }
}

/* vecmat, Algorithm 6 (kernels.py:145-174): bank the row coefficient per code in row-major
 * order, then sweep nodes in descending index order. */
void or_vecmat(const or_tree* t, const double* u, double* out, double* h) {
  for (int64_t i = 0; i < t->T; i++) h[i] = 0.0;
  for (int64_t r = 0; r < t->n_rows; r++) {
    double ui = u[r];
    for (int64_t p = t->offsets[r]; p < t->offsets[r + 1]; p++) h[t->codes[p]] += ui;
  }
  for (int64_t c = 0; c < t->n_cols; c++) out[c] = 0.0;
  for (int64_t i = t->T - 1; i > 0; i--) {
    double hi = h[i];
    double prod = t->value[i] * hi;
    out[t->column[i]] += prod;
    h[t->parent[i]] += hi;
  }
}

/* matmat_right, Algorithm 8 (kernels.py:177-203): M row-major [n_cols x p] -> out [n_rows x p].
 * h is caller scratch of T*p doubles. */
void or_matmat_right(const or_tree* t, const double* M, int64_t p, double* out, double* h) {
  for (int64_t j = 0; j < p; j++) h[j] = 0.0;
  for (int64_t i = 1; i < t->T; i++) {
    const double* mrow = M + (int64_t)t->column[i] * p;
    const double* hp = h + (int64_t)t->parent[i] * p;
    double* hi = h + i * p;
    double val = t->value[i];
    for (int64_t j = 0; j < p; j++) {
      double prod = val * mrow[j];
      hi[j] = prod + hp[j];
    }
  }
  for (int64_t r = 0; r < t->n_rows; r++) {
    double* acc = out + r * p;
    for (int64_t j = 0; j < p; j++) acc[j] = 0.0;
    for (int64_t q = t->offsets[r]; q < t->offsets[r + 1]; q++) {
      const double* hc = h + (int64_t)t->codes[q] * p;
      for (int64_t j = 0; j < p; j++) acc[j] += hc[j];
    }
  }
}

/* matmat_left, Algorithm 9 (kernels.py:206-234): M row-major [p x n_rows] -> out [p x n_cols].
 * h is caller scratch of T*p doubles (stored node-major: h[i*p + j]). */
void or_matmat_left(const or_tree* t, const double* M, int64_t p, double* out, double* h) {
  for (int64_t i = 0; i < t->T * p; i++) h[i] = 0.0;
  for (int64_t r = 0; r < t->n_rows; r++) {
    for (int64_t q = t->offsets[r]; q < t->offsets[r + 1]; q++) {
      double* hc = h + (int64_t)t->codes[q] * p;
      for (int64_t j = 0; j < p; j++) hc[j] += M[j * t->n_rows + r];
    }
  }
  for (int64_t i = 0; i < p * t->n_cols; i++) out[i] = 0.0;
  for (int64_t i = t->T - 1; i > 0; i--) {
    double* hi = h + i * p;
    double* hp = h + (int64_t)t->parent[i] * p;
    double val = t->value[i];
    int64_t col = t->column[i];
    for (int64_t j = 0; j < p; j++) {
      double prod = val * hi[j];
      out[j * t->n_cols + col] += prod;
    }
    for (int64_t j = 0; j < p; j++) hp[j] += hi[j];
  }
}

/* ------------------------------------------------------------------------------------------ */
/* Block-level helpers used by the CPU baseline: parse + build the tree from TOC1 bytes.       */
or_tree* or_tree_from_block(const uint8_t* data, int64_t len, int* rc, int64_t* detail,
                            int64_t* doff) {
  int64_t dims[4];
  *rc = or_deserialize(data, len, dims, NULL, NULL, NULL, NULL, detail, doff);
  if (*rc) return NULL;
  int32_t* I_cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)(dims[2] + 1));
  double* I_vals = (double*)malloc(sizeof(double) * (size_t)(dims[2] + 1));
  uint32_t* codes = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(dims[3] + 1));
  int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(dims[0] + 1));
  or_tree* t = NULL;
  if (I_cols && I_vals && codes && offsets) {
    *rc = or_deserialize(data, len, dims, I_cols, I_vals, codes, offsets, detail, doff);
    if (!*rc) t = or_tree_build(dims[0], dims[1], dims[2], I_cols, I_vals, dims[3], codes, offsets,
                                rc, detail, doff);
  } else {
    *rc = OR_NOMEM;
  }
  free(I_cols);
  free(I_vals);
  free(codes);
  free(offsets);
  return t;
}

/* Many independent batches with prebuilt trees, as the reference's own bench-kernels harness
 * times them (cli.py:299-383: trees built outside the timed region, one shared v, a per-batch
 * slice of u).  kind: 0 = matvec, 1 = vecmat, 2 = both.  R: concatenated row outputs; O:
 * n_batches x n_cols.  Parallel over batches with OpenMP (the reference itself is single
 * threaded; the thread count is reported).                                                    */
int or_sweep(int64_t n_batches, or_tree** trees, const int64_t* row_base, const double* v,
             const double* u, double* R, double* O, int kind, int nthreads) {
  int64_t max_t = 0;
  for (int64_t b = 0; b < n_batches; b++)
    if (trees[b]->T > max_t) max_t = trees[b]->T;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int fail = 0;
#pragma omp parallel
  {
    double* h = (double*)malloc(sizeof(double) * (size_t)(max_t + 1));
    if (!h) {
#pragma omp atomic write
      fail = 1;
    } else {
#pragma omp for schedule(dynamic, 4)
      for (int64_t b = 0; b < n_batches; b++) {
        const or_tree* t = trees[b];
        if (kind == 0 || kind == 2) or_matvec(t, v, R + row_base[b], h);
        if (kind == 1 || kind == 2) or_vecmat(t, u + row_base[b], O + b * t->n_cols, h);
      }
      free(h);
    }
  }
  return fail ? OR_NOMEM : OR_OK;
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------------------------ */
/* csr_matvec (matrix.py:225-239): per row, left to right from 0.0. */
void or_csr_matvec(int64_t n_rows, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                   const double* v, double* out) {
  for (int64_t r = 0; r < n_rows; r++) {
    double acc = 0.0;
    for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; e++) {
      double prod = vals[e] * v[cols[e]];
      acc += prod;
    }
    out[r] = acc;
  }
}

/* One MGD epoch over compressed batches for a GLM: mgd_step -> glm_gradient -> apply_update
 * (training.py:261-281, 296-316).  loss: 0 squared, 1 logistic, 2 hinge.  labels are the
 * batch labels concatenated in batch order (row_base[b] is batch b's first row).  w (n_cols) is
 * updated in place.  The per-example scalar uses libm exp; numpy's exp may differ in the last
 * ulp, so the GLM curves agree with the reference to ~1e-15, not bit for bit (tests state it). */
int or_glm_epoch(int64_t n_batches, or_tree** trees, const int64_t* row_base, const double* labels,
                 double* w, int loss, double lr) {
  int64_t max_t = 0, max_n = 0, m = n_batches ? trees[0]->n_cols : 0;
  for (int64_t b = 0; b < n_batches; b++) {
    if (trees[b]->T > max_t) max_t = trees[b]->T;
    if (trees[b]->n_rows > max_n) max_n = trees[b]->n_rows;
  }
  double* h = (double*)malloc(sizeof(double) * (size_t)(max_t + 1));
  double* z = (double*)malloc(sizeof(double) * (size_t)(max_n + 1));
  double* g = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  if (!h || !z || !g) {
    free(h);
    free(z);
    free(g);
    return OR_NOMEM;
  }
  for (int64_t b = 0; b < n_batches; b++) {
    const or_tree* t = trees[b];
    const double* y = labels + row_base[b];
    or_matvec(t, w, z, h);
    for (int64_t r = 0; r < t->n_rows; r++) {
      double s;
      if (loss == 0) {
        s = z[r] - y[r];
      } else if (loss == 1) {
        double yz = y[r] * z[r];
        double den = 1.0 + exp(yz);
        s = -y[r] / den;
      } else {
        double yz = y[r] * z[r];
        s = (yz < 1.0) ? -y[r] : 0.0;
      }
      z[r] = s;
    }
    or_vecmat(t, z, g, h);
    double step = lr / (double)t->n_rows; /* training.py:300 */
    for (int64_t j = 0; j < m; j++) {
      double d = step * g[j];
      w[j] = w[j] - d;
    }
  }
  free(h);
  free(z);
  free(g);
  return OR_OK;
}
