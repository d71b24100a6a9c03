/*
 * toc_b200.h -- C ABI of the B200-native TOC (tuple-oriented compression, arXiv 1702.06943)
 * hot path: compress -> TOC1 blocks in HBM -> A.v / v^T.A / A.M / M.A over compressed
 * mini-batches -> the MGD step that drives them.
 *
 * Plain C: device pointers, sizes and a cudaStream_t passed as void*.  No torch types.  Every
 * call is asynchronous on `stream` unless it says otherwise; no call allocates device memory or
 * synchronises except toc_encode_plan (one device->host copy of the per-batch sizes).
 *
 * The reference is a pure-Python package (`toc`, reference pkg/src/toc); its public functions are
 * the interface each entry point replaces.  INTEGRATION.md shows the ctypes binding.
 *
 * Return value of every function: TOC_OK or a TOC_E* code.  Per-batch format / encoding errors
 * are reported in TocBlockMeta.status and map to the reference's exception classes:
 *   TOC_E_BAD_MAGIC   -> BadMagicError            (reference physical.py:33-34)
 *   TOC_E_BAD_VERSION -> UnsupportedVersionError  (physical.py:37-38)
 *   TOC_E_TRUNCATED   -> TruncatedBlockError      (physical.py:41-42)
 *   TOC_E_FORMAT      -> BlockFormatError         (physical.py:33)
 *   TOC_E_CORRUPT     -> CorruptEncodingError     (codec.py:33, raised lazily like codec.py:235-244)
 *   TOC_E_INPUT       -> ValueError               (matrix.py:90-114 row validation)
 */
#ifndef TOC_B200_H
#define TOC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TOC_OK = 0,
  TOC_E_BAD_MAGIC = 1,
  TOC_E_BAD_VERSION = 2,
  TOC_E_TRUNCATED = 3,
  TOC_E_FORMAT = 4,
  TOC_E_CORRUPT = 5,
  TOC_E_INPUT = 6,
  TOC_E_CUDA = 7,
  TOC_E_ARG = 8,
};

/* detail codes for TocBlockMeta.detail (which check failed; messages are rebuilt on the host) */
enum {
  TOC_D_NONE = 0,
  TOC_D_WIDTH = 1,       /* bytes_per_int must be 1..4           physical.py:77-78   */
  TOC_D_PAIR_COUNT = 2,  /* pair count does not match            physical.py:151-154 */
  TOC_D_CODE_COUNT = 3,  /* code count does not match            physical.py:160-161 */
  TOC_D_TRAILING = 4,    /* trailing bytes after block           physical.py:163-164 */
  TOC_D_OFFS_COUNT = 5,  /* expected n_rows+1 row offsets        physical.py:165-166 */
  TOC_D_OFFS_SPAN = 6,   /* row offsets do not span the codes    physical.py:167-168 */
  TOC_D_OFFS_MONO = 7,   /* row offsets not monotone             physical.py:172-173 */
  TOC_D_REF_RANGE = 8,   /* value ref out of range               physical.py:104-107 */
  TOC_D_PAIR_COL = 9,    /* pair column out of range             codec.py:155-156    */
  TOC_D_PAIR_VAL = 10,   /* pair value is not finite             codec.py:157-158    */
  TOC_D_CODE_LT1 = 11,   /* code is not a valid node             codec.py:159-162    */
  TOC_D_UNDEF = 12,      /* code references an undefined node    codec.py:235-244    */
  TOC_D_MAGIC = 13,
  TOC_D_VERSION = 14,
  TOC_D_TRUNC = 15,
};

/*
 * Per-batch index of one TOC1 block (layout: reference physical.py:1-21), written on the device
 * by toc_index_blocks.  68 bytes.  Offsets are relative to the block's first byte.
 */
typedef struct TocBlockMeta {
  uint32_t n_rows, n_cols;   /* header                                                  */
  uint32_t n_uniques;        /* distinct value bit patterns                             */
  uint32_t n_pairs;          /* |I|: first-layer pairs                                  */
  uint32_t n_codes;          /* C = sum len(D[r])                                       */
  uint32_t n_derived;        /* sum max(len(D[r]) - 1, 0)  (codec.py:168-170)           */
  uint32_t off_uniques;      /* raw f64 x n_uniques                                     */
  uint32_t off_cols;         /* packed pair columns payload                             */
  uint32_t off_refs;         /* packed value refs payload                               */
  uint32_t off_codes;        /* packed concatenated codes payload                       */
  uint32_t off_offsets;      /* packed row offsets payload (n_rows + 1 entries)         */
  uint8_t w_cols, w_refs, w_codes, w_offsets; /* bytes per packed int, 1..4              */
  int32_t status;            /* TOC_OK or TOC_E_* (format errors, eager like deserialize)*/
  int32_t corrupt;           /* 1 if the tree build would raise CorruptEncodingError     */
  uint32_t detail;           /* TOC_D_* for status / corrupt                            */
  uint32_t detail_a;         /* offset / row of the failed check                         */
  uint32_t detail_b;         /* offending value (code, column, ref, count)               */
} TocBlockMeta;

/* Launch plan for the compressed linear-algebra kernels over an arena of indexed blocks. */
typedef struct TocPlan {
  int32_t threads;           /* CTA size                                                */
  int32_t ctas;              /* persistent grid size                                     */
  int32_t smem_bytes;        /* dynamic shared memory per CTA                            */
  int32_t wide;              /* 1 if some tree has >= 65536 nodes (32-bit node ids)      */
  int32_t vec_in_smem;       /* 1 if the n_cols-long vectors are staged in shared memory */
  int32_t n_cols;            /* common n_cols of the arena                                */
  int32_t max_rows;
  int32_t global_tables;     /* 1 if some batch's tables exceed shared memory            */
  int64_t scratch_bytes;     /* device workspace needed when global_tables (0 otherwise) */
} TocPlan;

/* kind bits for toc_plan / toc_linalg */
enum { TOC_MATVEC = 1, TOC_VECMAT = 2 };

/* ---- indexing (replaces physical.deserialize_block's parse + LogicalEncoding validation,
 *      reference physical.py:138-186, codec.py:151-162, and the tree-validity checks of
 *      codec.build_prefix_tree, codec.py:233-244) ---------------------------------------- */
int toc_index_blocks(const uint8_t* d_arena, const int64_t* d_block_off, const int64_t* d_block_len,
                     int64_t n_blocks, TocBlockMeta* d_meta, void* stream);

/* Host-side planning from a host copy of the metadata (pure host code, no CUDA calls except
 * reading device properties).  kind = TOC_MATVEC | TOC_VECMAT. */
int toc_plan(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t kind, TocPlan* plan);

/* ---- compressed linear algebra (reference kernels.py:115-174) ----------------------------
 * Batch b's rows are rows [d_row_base[b], d_row_base[b] + n_rows_b) of the concatenated row
 * space.  matvec:  d_R[row_base[b] + r] = (A_b . v)[r]                 (kernels.py:115 matvec)
 * vecmat:  d_O[b * n_cols + c] = (u_b^T . A_b)[c], u_b = d_u[row_base[b] ...] (kernels.py:145)
 * kind selects one or both; with both, each block is read once for the pair.
 * d_scratch: plan.scratch_bytes of device memory (may be NULL when scratch_bytes == 0). */
int toc_linalg(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
               const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int32_t kind,
               const double* d_v, double* d_R, const double* d_u, double* d_O, void* d_scratch,
               void* stream);

/* ---- device tree cache (the reference's lazily built, reused CompressedMatrix.tree,
 * kernels.py:68-77) -----------------------------------------------------------------------
 * toc_tree_offsets (host): byte offsets (n_blocks + 1 entries) of each batch's cache entry given
 * plan.wide: the tree prefix (row offsets, derived-node bases, final codes, node table), the
 * unpacked first-layer pairs, and the pairs sorted by column with column segments (16-B aligned;
 * layout: csrc/toc_batch.cuh CacheLayout).  toc_build_trees: build every entry once into d_trees.
 * toc_linalg_trees: toc_linalg reading the entries (one bulk copy of the prefix per batch) instead
 * of rebuilding the tree; v^T.A's output is then a fixed-order per-column sum. */
int toc_tree_offsets(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t wide, int64_t* h_tree_off);
/* tuning knob: 1 (default) = cached pair-balanced lane splits + flat chain walk for A.v, 0 = code-count splits */
int toc_linalg_set_splits(int on);
/* tuning knob: 1 (default) = toc_build_trees orders each lane range's codes by chain depth (a renumbering of
 * each row's derived ids; the products are unchanged), 0 = reference order */
int toc_tree_set_depth_order(int on);
int toc_build_trees(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                    int64_t n_blocks, const TocPlan* plan, const int64_t* d_tree_off, uint8_t* d_trees,
                    void* d_scratch, void* stream);
int toc_linalg_trees(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                     const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int32_t kind,
                     const double* d_v, double* d_R, const double* d_u, double* d_O, void* d_scratch,
                     const uint8_t* d_trees, const int64_t* d_tree_off, void* stream);

/* ---- slot cache (csrc/toc_levels.cu; replaces the per-call tree walk of kernels.py:115-174 with
 * the reference's node recurrence H[x] = H[par] + P1[key] evaluated only where a node is shared) --
 * toc_levels_build (host): from a HOST copy of the arena, per batch a self-contained entry: the
 * value index and row offsets, the pairs numbered by column (slots 1..|I|), the "inner" derived
 * nodes -- those some used derived node hangs off, closed under parents -- with their (parent,
 * key) slot records, and the code stream as 16-bit slot records (the node's own slot, or two
 * records -- parent slot, key slot -- for a leaf; one record of slot 0 for an empty row) cut into
 * equal per-thread ranges and placed within each row to spread the shared-memory banks -- built
 * once, like the reference's cached CompressedMatrix.tree (kernels.py:68-77).  Returns an opaque handle (NULL on
 * bad arguments).  toc_levels_info: total bytes, the largest slot count and staged-region size,
 * and the build status (TOC_E_CORRUPT for a block the reference's tree build rejects,
 * codec.py:235-244; TOC_E_ARG when some batch needs slots wider than 15 bits or columns wider
 * than 16 -- keep the tree-cache path then).  toc_levels_copy: the entries back to back into
 * h_out, offsets (n_blocks + 1) into h_off.  toc_levels_smem: dynamic shared memory
 * toc_linalg_levels needs (it returns TOC_E_ARG if that exceeds the device's per-CTA limit).
 * toc_linalg_levels: A.v / v^T.A as toc_linalg, same operand layout (d_row_base: first row of
 * each batch); reads only the cache entries and the operands; every sum has a fixed order (v^T.A
 * in exact fixed point, fp64 when that would be too coarse), deterministic.
 * toc_levels_set_trace: tools only (per-phase clock64 stamps of CTA 0; NULL turns it off). */
void* toc_levels_build(const uint8_t* h_arena, const int64_t* h_block_off, const TocBlockMeta* h_meta,
                       int64_t n_blocks, int32_t n_threads);
int toc_levels_info(const void* handle, int64_t* total_bytes, int32_t* max_slots, int32_t* max_stage,
                    int32_t* max_rows);
int toc_levels_copy(const void* handle, uint8_t* h_out, int64_t* h_off);
void toc_levels_free(void* handle);
int toc_levels_set_prefetch(int mode); /* tuning knob: L2 prefetch of the CTA's next entry (1, default) or none (0) */
int toc_levels_set_trace(long long* d_trace);
int64_t toc_levels_smem(int32_t kind, int32_t n_cols, int32_t max_slots, int32_t max_stage, int32_t max_rows);
int toc_linalg_levels(const int64_t* d_row_base, int64_t n_blocks, int32_t kind, int32_t n_cols, int32_t max_slots,
                      int32_t max_stage, int32_t max_rows, const double* d_v, double* d_R, const double* d_u,
                      double* d_O, const uint8_t* d_lvl, const int64_t* d_lvl_off, void* stream);
/* The fp32 variant (BASELINE.json north_star: within 1e-4 of the fp64 results; the reference is fp64
 * only) over the same cache entries: float operands and results, H in fp32, v^T.A in 32-bit fixed
 * point -- one native shared-memory atomic per record -- or float atomics when that would be too
 * coarse for the bar (heavy-tailed u). */
int toc_linalg_levels32(const int64_t* d_row_base, int64_t n_blocks, int32_t kind, int32_t n_cols, int32_t max_slots,
                        int32_t max_stage, int32_t max_rows, const float* d_v, float* d_R, const float* d_u,
                        float* d_O, const uint8_t* d_lvl, const int64_t* d_lvl_off, void* stream);

/* ---- the reference's own operation order, bit for bit (csrc/toc_exact.cu; kernels.py:115-174) ---
 * Over one batch's DecodeTree (device arrays parent / column / value, node 0 the root) and a
 * schedule built on the host: nodes grouped by tree depth (d_level_nodes, level l's nodes at
 * [h_level_off[l], h_level_off[l + 1])), each row's codes (d_rowoff / d_codes), each node's
 * occurrence rows in row order, its children in descending id order, each column's nodes in
 * descending id order.  toc_exact_matvec: H level by level (H[i] = value[i] * v[col[i]] +
 * H[parent[i]]), then every row's left-to-right sum -- equal to the reference's matvec bit for bit;
 * d_H: T doubles of scratch.  toc_exact_vecmat: the occurrence sums, the children's h bottom-up,
 * the column sums in descending node order -- equal to the reference's vecmat bit for bit; d_h: T
 * doubles.  Products and sums rounded separately (no FMA contraction). */
int toc_exact_matvec(const int32_t* d_parent, const int32_t* d_column, const double* d_value,
                     const int32_t* d_level_nodes, const int64_t* h_level_off, int32_t n_levels, const int64_t* d_rowoff,
                     const int32_t* d_codes, int32_t n_rows, const double* d_v, double* d_R, double* d_H, void* stream);
int toc_exact_vecmat(const int32_t* d_column, const double* d_value, int32_t T, const int32_t* d_level_nodes,
                     const int64_t* h_level_off, int32_t n_levels, const int64_t* d_occ_off, const int32_t* d_occ_row,
                     const int64_t* d_child_off, const int32_t* d_child, const int64_t* d_col_off,
                     const int32_t* d_col_node, int32_t n_cols, const double* d_u, double* d_out, double* d_h,
                     void* stream);

/* ---- compressed matrix-matrix products (reference kernels.py:177-234) ----------------------
 * side 0 (matmat_right, kernels.py:177-203): d_out[row_base[b] + r, :] = (A_b . M)[r, :],
 *         d_M = M [n_cols x p] row-major, d_out [n_rows_total x p].
 * side 1 (matmat_left, kernels.py:206-234): d_out[b] = M_b . A_b  [p x n_cols] per batch,
 *         d_M = M^T [n_rows_total x p] row-major (rows of M^T are batch rows), d_out
 *         [n_blocks x p x n_cols].
 * h_meta: host copy of the metadata.  d_scratch: toc_matmat_scratch bytes (0 unless some batch's
 * tables exceed shared memory). */
int toc_matmat(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
               const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks, int32_t n_cols,
               int32_t side, int32_t p, const double* d_M, double* d_out, void* d_scratch,
               int64_t scratch_bytes, void* stream);
int toc_matmat_scratch(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t side,
                       int32_t p, int64_t* bytes);

/* ---- compression (replaces codec.encode, codec.py:112-191, and physical.serialize_block,
 *      physical.py:88-130; physical.deserialize_block's unpack, physical.py:138-186) --------
 * Mini-batch b is rows [batch_row[b], batch_row[b+1]) of a CSR matrix (row_ptr int64, cols
 * int32, vals f64; SparseRowMatrix contract, matrix.py:90-114, checked on the device).
 * elem_base[b] = row_ptr[batch_row[b]] (n_batches + 1 entries).  The logical encoding of batch b
 * is written at element base elem_base[b] (I_cols, I_vals, codes) and at batch_row[b] + b
 * (offsets, n_rows_b + 1 entries); TocBatchInfo[b] receives the counts. */
typedef struct TocBatchInfo {
  uint32_t n_rows, n_cols, n_pairs, n_codes, n_uniques;
  uint8_t w_cols, w_refs, w_codes, w_offsets;
  int32_t status;      /* TOC_OK, or TOC_E_INPUT for a row violating the input contract */
  uint32_t detail_a;   /* offending row                                                  */
  uint32_t detail_b;   /* offending position within the row                              */
  uint32_t pad_;
  int64_t block_bytes; /* serialized TOC1 size (after toc_serialize_sizes)               */
} TocBatchInfo;        /* 48 bytes */

typedef struct TocEncodeSizes {
  int64_t hash_slots;  /* total hash-table slots over the batches                        */
  int64_t n_elems;     /* element-index extent of the logical arrays                      */
  int64_t work_bytes;  /* device workspace for toc_encode / toc_serialize_sizes           */
} TocEncodeSizes;

/* Host-only sizing from a host copy of elem_base. */
int toc_encode_sizes(int64_t n_batches, const int64_t* h_elem_base, TocEncodeSizes* out);

/* Row-bounded LZW encoding of every batch (codec.encode), bit-exact with the reference. */
int toc_encode(int64_t n_batches, int32_t n_cols, const int64_t* d_row_ptr, const int32_t* d_cols,
               const double* d_vals, const int64_t* d_batch_row, const int64_t* d_elem_base,
               const TocEncodeSizes* sizes, void* d_work, uint32_t* d_I_cols, double* d_I_vals,
               uint32_t* d_codes, uint32_t* d_offsets, TocBatchInfo* d_info, void* stream);

/* Value index (physical.py:88-101), packed widths (physical.py:49-51) and the TOC1 size of each
 * batch's logical encoding; fills the remaining TocBatchInfo fields, refs and uniques. */
int toc_serialize_sizes(int64_t n_batches, const int64_t* d_batch_row, const int64_t* d_elem_base,
                        const uint32_t* d_I_cols, const double* d_I_vals, const uint32_t* d_codes,
                        const uint32_t* d_offsets, const TocEncodeSizes* sizes, void* d_work,
                        uint32_t* d_refs, double* d_uniques, TocBatchInfo* d_info, void* stream);

/* Write each batch's TOC1 bytes at d_arena + d_block_off[b] (serialize_block, physical.py:110-130). */
int toc_pack_blocks(int64_t n_batches, const int64_t* d_batch_row, const int64_t* d_elem_base,
                    const uint32_t* d_I_cols, const uint32_t* d_refs, const double* d_uniques,
                    const uint32_t* d_codes, const uint32_t* d_offsets, const TocBatchInfo* d_info,
                    const int64_t* d_block_off, uint8_t* d_arena, void* stream);

/* Unpack indexed blocks into logical arrays (deserialize_block): pairs at pair_base[b], codes at
 * code_base[b], offsets at offs_base[b]. */
int toc_unpack_blocks(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                      int64_t n_blocks, const int64_t* d_pair_base, const int64_t* d_code_base,
                      const int64_t* d_offs_base, uint32_t* d_I_cols, double* d_I_vals,
                      uint32_t* d_codes, uint32_t* d_offsets, void* stream);

/* ---- mini-batch gradient descent for GLMs (training.py:261-361) ---------------------------
 * The arena's blocks are the epoch's mini-batches in order (shuffle_once + make_batches,
 * training.py:131-167); labels are per row in the same order.  Losses: */
enum { TOC_LOSS_SQUARED = 0, TOC_LOSS_LOGISTIC = 1, TOC_LOSS_HINGE = 2 };

/* Launch plan of the MGD kernels (diagnostic): info[8] = smem, table budget, small_m,
 * 0, max |I|, ctas, slab bytes, wide. */
int toc_mgd_plan_info(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t kind,
                      int64_t* info);

/* Diagnostic: cap the MGD grid at n CTAs (0 restores one CTA per SM). */
int toc_mgd_set_max_ctas(int32_t n);

/* Device workspace (bytes) for toc_glm_epoch (kind 0) or toc_glm_grad (kind 1); host-only. */
int toc_mgd_workspace(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t kind,
                      int64_t* scratch_bytes);

/* One epoch: for each batch b in order, g = s^T A_b with s = loss'(A_b w, y_b) and
 * w -= (lr / n_rows_b) * g (mgd_step, training.py:303-316).  One cooperative launch; d_sync:
 * 2 device words of scratch (step counter, abort flag).  h_meta: host copy of the metadata. */
int toc_glm_epoch(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                  const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                  int32_t n_cols, int32_t loss, double lr, const double* d_labels, double* d_w,
                  uint32_t* d_sync, void* d_scratch, void* stream);

/* toc_glm_epoch plus a phase trace: d_trace receives 8 clock64 stamps per step (tables built,
 * weights acquired, P1, A.w + loss scalar, bound, s^T.A, column update, published).  Diagnostic. */
int toc_glm_epoch_traced(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                         const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                         int32_t n_cols, int32_t loss, double lr, const double* d_labels, double* d_w,
                         uint32_t* d_sync, void* d_scratch, long long* d_trace, void* stream);

/* Summed gradient of every batch at fixed w (glm_gradient, training.py:261-281):
 * d_grad[b * n_cols + c].  The data-parallel trainer all-reduces these. */
int toc_glm_grad(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                 const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                 int32_t n_cols, int32_t loss, const double* d_labels, const double* d_w,
                 double* d_grad, void* d_scratch, void* stream);

/* Per-row loss of empirical_risk (training.py:231-258) summed into n_partial partial sums. */
int toc_glm_risk(const double* d_z, const double* d_y, int64_t n, int32_t loss, double* d_partial,
                 int32_t n_partial, void* stream);

/* Cached step images (the device form of the reference's once-only per-batch tree cache,
 * kernels.py:68-77): each batch's code stream, decode-tree node table, unpacked first-layer pairs
 * (also sorted by column), value index, and per-CTA row parts (lane splits, labels), 16-byte
 * aligned, built once per training run (layout: toc_images.cu).  The epoch runs on a cluster of
 * `cluster` CTAs (1, 2, 4 or 8) that split each batch's rows.
 * toc_mgd_image_plan: host-only.  cluster_req 0 = choose; *cluster = the chosen size, or 0 when
 * images do not fit shared memory (use toc_glm_epoch); h_image_off: n_blocks + 1 byte offsets.
 * TOC_E_* of the first malformed / corrupt block. */
int toc_mgd_image_plan(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t cluster_req,
                       int32_t* cluster, int64_t* h_image_off);
int toc_mgd_build_images(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                         const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                         int32_t n_cols, int32_t cluster, const double* d_labels, uint8_t* d_images,
                         const int64_t* d_image_off, void* stream);
/* One epoch (training.py:303-316) on one cluster: weights in shared memory, the next image
 * prefetched by TMA (multicast) during each step, one cluster barrier per step.  Same results as
 * toc_glm_epoch up to fp64 summation order of the per-column sums (fixed, deterministic). */
int toc_glm_epoch_images(const uint8_t* d_images, const int64_t* d_image_off, const TocBlockMeta* d_meta,
                         const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t cluster,
                         int32_t loss, double lr, double* d_w, void* stream);
/* MGD for models too wide for shared memory (csrc/toc_images_large.cu): per-CTA part images of
 * every batch (the CTA's rows, the part of C' their codes reach renumbered locally, its pairs'
 * columns and values, the columns it owns, labels), built once per run in two passes:
 * toc_mgd_parts_count -> d_counts[n_blocks][cluster][4] (pairs, derived nodes, codes, owned
 * columns); toc_mgd_parts_offsets (host) -> h_part_off[n_blocks * cluster + 1] and the largest part;
 * toc_mgd_parts_build writes them.  d_scratch: toc_mgd_parts_scratch bytes.
 * toc_glm_epoch_parts: one epoch on a cluster (logistic / hinge); w and d_gacc (n_cols u64, zero,
 * left zero) in global memory; each step's gradient accumulated in exact 64-bit fixed point.
 * toc_mgd_parts_fit: whether the epoch's part buffers fit shared memory. */
int toc_mgd_parts_scratch(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int64_t* bytes);
int toc_mgd_parts_count(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                        const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                        int32_t n_cols, int32_t cluster, const double* d_labels, int32_t* d_counts,
                        void* d_scratch, void* stream);
int toc_mgd_parts_offsets(const TocBlockMeta* h_meta, const int32_t* h_counts, int64_t n_blocks,
                          int32_t cluster, int64_t* h_part_off, int64_t* max_part);
int toc_mgd_parts_build(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                        const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                        int32_t n_cols, int32_t cluster, const double* d_labels, const int32_t* d_counts,
                        const int64_t* d_part_off, uint8_t* d_images, void* d_scratch, void* stream);
int toc_mgd_parts_fit(const TocBlockMeta* h_meta, const int32_t* h_counts, int64_t n_blocks,
                      int32_t cluster, int64_t max_part, int32_t* fits);
int toc_glm_epoch_parts(const uint8_t* d_images, const int64_t* d_part_off, const TocBlockMeta* h_meta,
                        const int32_t* h_counts, int64_t n_blocks, int32_t n_cols, int32_t cluster,
                        int32_t loss, double lr, double* d_w, unsigned long long* d_gacc, int64_t max_part,
                        void* stream);

/* The largest power-of-two cluster (<= 16; sizes above 8 are non-portable) this device co-schedules
 * for the part-image epoch with a full shared-memory carve-out per CTA, into *cluster.  The part
 * images are built for one cluster size (toc_mgd_parts_count / _build take it). */
/* Diagnostic: per-step clock64 stamps of toc_glm_epoch_parts (8 per step from step t0; NULL: off). */
int toc_mgd_parts_set_trace(long long* d_trace);
int toc_mgd_parts_cluster_max(int32_t* cluster);

/* One data-parallel MGD step on the same part images (training.py:261-281 per rank; the caller
 * all-reduces and applies training.py:296-300): the summed gradient of batch `step` at weights d_w
 * into d_grad[touched columns] (d_grad zero elsewhere; d_gacc left zero). */
int toc_glm_grad_parts(const uint8_t* d_images, const int64_t* d_part_off, const TocBlockMeta* h_meta,
                       const int32_t* h_counts, int64_t n_blocks, int32_t n_cols, int32_t cluster, int32_t loss,
                       int64_t step, const double* d_w, unsigned long long* d_gacc, double* d_grad,
                       int64_t max_part, void* stream);

/* Diagnostic: CTA width (power of two, 64..1024; 0 = 512) of cluster epochs planned afterwards. */
int toc_mgd_set_image_threads(int32_t threads);
/* Data-parallel toc_glm_epoch_images with the gradient all-reduce fused into the kernel (NVLink
 * peer memory, no NCCL on the step path): this rank's images are its local batch of every global
 * step; each step CTA 0 writes the rank's dense gradient into every rank's receive buffer
 * (d_peer_buf[q], 2 * world * n_cols doubles, double-buffered by step parity), fences, and sets
 * d_peer_flag[q][rank] = seq0 + t + 1; every rank waits for all flags of step t and applies
 * w -= (lr / d_gsize[t]) * (sum over ranks in rank order) -- training.py:296-300 at the global
 * batch.  Pointers: device arrays of world device pointers (e.g. torch symmetric memory's buffer /
 * signal-pad pointers).  seq0 must grow across epochs (e.g. epoch * n_blocks).  n_cols must not
 * exceed the largest batch's pair count + 1 (the gradient scratch reuses the P1 table). */
int toc_glm_epoch_images_dp(const uint8_t* d_images, const int64_t* d_image_off, const TocBlockMeta* d_meta,
                            const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t cluster,
                            int32_t loss, double lr, double* d_w, int32_t world, int32_t rank,
                            double* const* d_peer_buf, uint32_t* const* d_peer_flag, const int32_t* d_gsize,
                            uint32_t seq0, void* stream);

/* One rank's data for toc_glm_epoch_images_dp_emulated (device pointers, as for
 * toc_glm_epoch_images_dp). */
typedef struct {
  const uint8_t* images;
  const int64_t* image_off;
  const TocBlockMeta* meta;
  double* w;
} TocDpRank;

/* toc_glm_epoch_images_dp for `world` ranks in ONE cooperative launch on one GPU: thread-block
 * cluster r runs rank r (d_ranks[r]: its step images, metadata and weights) and exchanges its
 * gradient with the other clusters through the same receive-slot / flag protocol (the buffers can
 * be plain device memory).  Separate launches that spin on each other's flags are never
 * guaranteed to be co-resident on one GPU, so this is how the multi-rank protocol is exercised
 * with fewer GPUs than ranks.  h_meta_all: the ranks' host metadata, rank-major (world x n_blocks);
 * every rank's images must have been built for the same cluster shape. */
int toc_glm_epoch_images_dp_emulated(const TocDpRank* d_ranks, const TocBlockMeta* h_meta_all, int64_t n_blocks,
                                     int32_t n_cols, int32_t cluster, int32_t loss, double lr, int32_t world,
                                     double* const* d_peer_buf, uint32_t* const* d_peer_flag, const int32_t* d_gsize,
                                     uint32_t seq0, void* stream);

/* toc_glm_epoch_images plus 8 clock64 stamps per step from CTA 0 (step start, image landed, P1,
 * A.w and loss, bound, s^T.A, cluster barrier passed, update).  Diagnostic. */
int toc_glm_epoch_images_traced(const uint8_t* d_images, const int64_t* d_image_off,
                                const TocBlockMeta* d_meta, const TocBlockMeta* h_meta, int64_t n_blocks,
                                int32_t n_cols, int32_t cluster, int32_t loss, double lr, double* d_w,
                                long long* d_trace, void* stream);

/* The fp32 variant of toc_linalg_trees (tree cache required; every batch's tables in shared memory,
 * i.e. !plan->global_tables): v, R, u, O in float32, P1 in fp32, G in 32-bit fixed point, and a
 * fused TOC_MATVEC | TOC_VECMAT walks every code once for both products.  Within 1e-4 of the fp64
 * oracle (BASELINE.json north_star); the reference has no fp32 mode. */
int toc_linalg32(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                 const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int32_t kind,
                 const float* d_v, float* d_R, const float* d_u, float* d_O, const uint8_t* d_trees,
                 const int64_t* d_tree_off, void* stream);

/* ---- matmat over cached node records (kernels.py:177-234 for large batches) ----------------
 * toc_matcache_offsets (host): byte offsets (n_blocks + 1) of each batch's cache entry (row
 * offsets, code stream, each code's first-pair offset, a {parent, column, value} record per tree
 * node; csrc/toc_matcache.cu).  Rows are expanded in shared memory: 12 * n_cols bytes (A.M),
 * 268 * n_cols (M.A); TOC_E_ARG when that exceeds shared memory (use toc_matmat).
 * toc_matcache_build: every entry, once (plan from toc_plan(TOC_MATVEC) + its scratch).
 * toc_matcache_right: out [rows x p] = A . M (M [m x p]) for the rows of n_blocks consecutive
 * entries, d_row_base giving each batch's first output row.
 * toc_matcache_left: one batch, out [p x m] = M_b . A_b with M^T given ([n x p]), deterministic
 * (fixed summation order); d_scratch of toc_matcache_left_scratch bytes. */
int toc_matcache_offsets(const TocBlockMeta* h_meta, int64_t n_blocks, int64_t* h_cache_off);
int toc_matcache_build(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                       int64_t n_blocks, const TocPlan* plan, const int64_t* d_cache_off, uint8_t* d_cache,
                       void* d_scratch, void* stream);
int toc_matcache_right(const uint8_t* d_cache, const int64_t* d_cache_off, const int64_t* d_row_base,
                       int64_t n_blocks, int64_t n_rows, int32_t n_cols, int32_t p, const double* d_M,
                       double* d_out, void* stream);
int toc_matcache_left_scratch(const TocBlockMeta* h_meta, int32_t p, int32_t n_cols, int64_t* bytes);
int toc_matcache_left(const uint8_t* d_entry, const TocBlockMeta* h_meta, int32_t p, int32_t n_cols,
                      const double* d_MT, double* d_out, void* d_scratch, int64_t scratch_bytes,
                      void* stream);

/* ---- MLP step cache (csrc/toc_matcache.cu): the decode tree of each batch in 4 bytes per node
 * (parent | key << 17), its pair records and value index -- read together with the TOC1 block's
 * own code stream, so the cache does not repeat the codes (config 5: 0.45 MB per batch, 1.5x the
 * TOC1 block; the node-record cache above is 2.3 MB).  toc_mlpcache_offsets (host): entry offsets,
 * TOC_E_ARG if some batch's ids do not fit (more than 2^17 nodes, 2^15 pairs, 2^16 columns or
 * values).  toc_mlpcache_build: every entry, once (plan from toc_plan(TOC_MATVEC) + its scratch). */
int toc_mlpcache_offsets(const TocBlockMeta* h_meta, int64_t n_blocks, int64_t* h_cache_off);
int toc_mlpcache_build(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                       int64_t n_blocks, const TocPlan* plan, const int64_t* d_cache_off, uint8_t* d_cache,
                       void* d_scratch, void* stream);

/* ---- config-5 MLP epoch (oracle.train_mlp's step; first layer = kernels.py:177-234) ---------
 * One epoch over the batches in order, four kernels per step on `stream` (toc_mlp.cu): each
 * step's batch decoded from its TOC1 block (d_arena + h_block_off[b]) and step-cache entry
 * (toc_mlpcache_build) into a dense tile buffer, A_b . W1 and A_b^T . delta on the fp64 tensor
 * cores, the softmax cross-entropy tail and the parameter updates.  Weights are updated in place.
 * h_block_off / h_cache_off / h_row_base / h_n_rows: host copies; d_labels: class ids (f64).
 * k must be 10; dense = 1 only if every row has all m columns (the decode then skips zeroing);
 * scratch: toc_mlp_scratch(max rows per batch, m, h, k).  toc_mlp_risk: the per-row cross-entropy
 * of the current parameters over every batch (forward only) into d_loss [rows]. */
/* Diagnostic: launch only the step kernels in mask (bit 0 decode, 1 right, 2 tail, 3 left; 15 =
 * all, the default) -- for timing them in the stream; any other mask trains wrongly. */
int toc_mlp_set_kernels(int32_t mask);
/* 1 (default): toc_mlp_epoch captures the epoch's launches into a CUDA graph on its first call and
 * replays it while the arguments (and the host arrays' contents) are unchanged; 0: plain launches. */
int toc_mlp_set_graph(int32_t on);
int toc_mlp_set_pdl(int32_t on); /* tuning knob: programmatic dependent launch of the step kernels (default 1) */
int toc_mlp_set_decode_ctas(int32_t per_sm); /* tuning knob: decode CTAs per SM (1..32, default 8) */
int toc_mlp_set_fused(int32_t on); /* 1 (default): A.W1 and the softmax tail as one cluster kernel; 0: two kernels */
int toc_mlp_scratch(int32_t max_rows, int32_t m, int32_t h, int32_t k, int64_t* bytes);
int toc_mlp_epoch(const uint8_t* d_arena, const int64_t* h_block_off, const uint8_t* d_cache,
                  const int64_t* h_cache_off, const int64_t* h_row_base, const int32_t* h_n_rows, int64_t n_blocks,
                  int32_t m, int32_t h, int32_t k, const double* d_labels, double* d_W1, double* d_b1, double* d_W2,
                  double* d_b2, double lr, int32_t dense, void* d_scratch, int64_t scratch_bytes, void* stream);
int toc_mlp_risk(const uint8_t* d_arena, const int64_t* h_block_off, const uint8_t* d_cache, const int64_t* h_cache_off,
                 const int64_t* h_row_base, const int32_t* h_n_rows, int64_t n_blocks, int32_t m, int32_t h, int32_t k,
                 const double* d_labels, const double* d_W1, const double* d_b1, const double* d_W2,
                 const double* d_b2, int32_t dense, double* d_loss, void* d_scratch, int64_t scratch_bytes,
                 void* stream);
/* One data-parallel step of the same model (the per-rank half of toc_mlp_epoch's step; the caller
 * all-reduces and applies the update): the summed gradient of batch `step` at the given weights
 * into d_grad = [W1 m*h | W2 h*k | b1 h | b2 k].  Steps of one epoch must be issued in batch order
 * starting at step 0 (the decode buffers alternate by step parity). */
int toc_mlp_step_grad(const uint8_t* d_arena, const int64_t* h_block_off, const uint8_t* d_cache,
                      const int64_t* h_cache_off, const int64_t* h_row_base, const int32_t* h_n_rows, int64_t n_blocks,
                      int64_t step, int32_t m, int32_t h, int32_t k, const double* d_labels, const double* d_W1,
                      const double* d_b1, const double* d_W2, const double* d_b2, int32_t dense, double* d_grad,
                      void* d_scratch, int64_t scratch_bytes, void* stream);

/* ---- decode (codec.py:262-292 node_sequence / decode; cli.py:194-221 verify) -----------------
 * Two passes with a plan from toc_plan(kind = TOC_MATVEC) and its scratch: toc_decode_counts writes
 * each row's pair count at d_row_nnz[row_base[b] + r]; the caller scans them into d_row_ptr
 * (total_rows + 1 entries, row_ptr[0] = 0); toc_decode_rows writes every row's (column, value)
 * pairs in row order, values bit for bit from the block's value index. */
int toc_decode_counts(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                      const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int64_t* d_row_nnz,
                      void* d_scratch, void* stream);
int toc_decode_rows(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                    const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, const int64_t* d_row_ptr,
                    int32_t* d_cols, double* d_vals, void* d_scratch, void* stream);
/* The reference's DecodeTree arrays (build_prefix_tree, codec.py:194-259) for every block, node 0
 * the root (-1 / 0.0 sentinels); block b's T_b = 1 + |I| + derived nodes start at d_tree_base[b]. */
int toc_tree_arrays(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                    int64_t n_blocks, const TocPlan* plan, const int64_t* d_tree_base, int32_t* d_parent,
                    int32_t* d_column, double* d_value, int32_t* d_first_col, double* d_first_val,
                    void* d_scratch, void* stream);

/* ---- the batched public sweep's pipeline (kernels.BatchSweep; reference cli.py:299-383) --------
 * One chunk of the sweep: its byte range in the host and device block buffers, its indexed view
 * (offsets relative to d_arena; rows relative to the chunk), its plan / scratch, and the chunk's
 * own CUDA events (upload done, operands done, compute done; toc_sweep_events creates them,
 * toc_sweep_events_free destroys them) -- per-sweep state, so sweeps on several threads or devices
 * do not share events. */
typedef struct TocSweepChunk {
  int64_t byte_lo, byte_hi;
  const uint8_t* d_arena;
  const int64_t* d_block_off;
  const int64_t* d_block_len;
  TocBlockMeta* d_meta;
  const int64_t* d_row_base;
  void* d_scratch;
  int64_t n_blocks, b0, row0, n_rows;
  TocPlan plan;
  void* ev_upload;
  void* ev_operands;
  void* ev_done;
} TocSweepChunk; /* 160 bytes */
int toc_sweep_events(TocSweepChunk* chunks, int64_t n_chunks);
int toc_sweep_events_free(TocSweepChunk* chunks, int64_t n_chunks);

/* Enqueue the block bytes of chunks [k0, k1) host -> device on copy_stream (pinned h_blocks). */
int toc_sweep_upload(const uint8_t* h_blocks, uint8_t* d_blocks, const TocSweepChunk* chunks, int64_t k0,
                     int64_t k1, void* copy_stream);
/* Enqueue v and every chunk's u slice on copy_stream (host -> device copies are served in
 * submission order: enqueue them after the first chunk's bytes, before the others). */
int toc_sweep_operands(const TocSweepChunk* chunks, int64_t n_chunks, int32_t n_cols, const double* h_v,
                       double* d_v, const double* h_u, double* d_u, void* copy_stream);
/* Enqueue per chunk, after its bytes and operands: toc_index_blocks and the fused A.v + v^T.A
 * (compute_stream), then R, O and the chunk's index to the pinned host buffers (d2h_stream).  The
 * caller synchronizes d2h_stream and checks h_meta for format / corruption errors. */
int toc_sweep_compute(const TocSweepChunk* chunks, int64_t n_chunks, int32_t n_cols, const double* d_v,
                      const double* d_u, double* d_R, double* h_R, double* d_O, double* h_O,
                      TocBlockMeta* h_meta, void* compute_stream, void* d2h_stream);
int toc_sizeof_sweep_chunk(void); /* 160 */
/* Diagnostic: record timed events in later runs; toc_sweep_timeline reads chunk k's upload end,
 * validation start / end, compute end and download end (out[5k..5k+4], ms from the first upload)
 * after a synchronized run. */
int toc_sweep_set_timing(int32_t on);
int toc_sweep_timeline(int64_t n_chunks, float* out);

/* ---- the uncompressed baselines (matrix.py:164-279), bit for bit --------------------------------
 * Each output element is accumulated by one thread in the reference's ascending order with
 * separate IEEE multiplies and adds, so results equal the reference's Python / numpy sums exactly.
 * Dense operands row-major; CSR row_ptr int64 (n_rows + 1), cols int32; the CSC forms take the same
 * entries grouped by column with rows ascending (the reference's row-order scatters as ordered
 * per-column sums).
 *   toc_dense_matvec      replaces matrix.dense_matvec      (matrix.py:164-173)
 *   toc_dense_vecmat      replaces matrix.dense_vecmat      (matrix.py:176-186)
 *   toc_dense_matmat      replaces matrix.dense_matmat      (matrix.py:189-206)
 *   toc_csr_matvec        replaces matrix.csr_matvec        (matrix.py:225-239)
 *   toc_csc_vecmat        replaces matrix.csr_vecmat        (matrix.py:242-249)
 *   toc_csr_matmat_right  replaces matrix.csr_matmat_right  (matrix.py:252-264)
 *   toc_csc_matmat_left   replaces matrix.csr_matmat_left   (matrix.py:267-279) */
int toc_dense_matvec(const double* d_A, int64_t n, int64_t m, const double* d_v, double* d_out, void* stream);
int toc_dense_vecmat(const double* d_v, const double* d_A, int64_t n, int64_t m, double* d_out, void* stream);
int toc_dense_matmat(const double* d_A, const double* d_M, int64_t n, int64_t k, int64_t p, double* d_out,
                     void* stream);
int toc_csr_matvec(const int64_t* d_row_ptr, const int32_t* d_cols, const double* d_vals, int64_t n_rows,
                   const double* d_v, double* d_out, void* stream);
int toc_csc_vecmat(const int64_t* d_col_ptr, const int32_t* d_rows, const double* d_vals, int64_t n_cols,
                   const double* d_v, double* d_out, void* stream);
int toc_csr_matmat_right(const int64_t* d_row_ptr, const int32_t* d_cols, const double* d_vals, int64_t n_rows,
                         const double* d_M, int64_t p, double* d_out, void* stream);
int toc_csc_matmat_left(const int64_t* d_col_ptr, const int32_t* d_rows, const double* d_vals, int64_t n_cols,
                        const double* d_M, int64_t p, int64_t n_rows, double* d_out, void* stream);

/* ---- version / self-description ---------------------------------------------------------- */
const char* toc_version(void);
int toc_device_info(int32_t* sm_count, int32_t* smem_optin, int64_t* l2_bytes);
int toc_sizeof_meta(void); /* 68: ABI check for bindings */
int toc_sizeof_plan(void); /* 40 */
int toc_sizeof_batch_info(void); /* 48 */

#ifdef __cplusplus
}
#endif
#endif /* TOC_B200_H */
