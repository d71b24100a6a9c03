// toc_linalg32.cu -- the fp32 variant of A.v / v^T.A over the device tree cache.
//
// Reference: kernels.py:115-174 (matvec / vecmat, Algorithms 5 and 6); the reference itself is fp64
// end to end, so this variant's bar is 1e-4 relative against the fp64 oracle (BASELINE.json
// north_star).  Same per-batch machinery as toc_linalg.cu's tree-cache path (prefix bulk copy,
// unpacked and column-sorted pair records) with the table of 8-byte entries split in two 4-byte
// halves: P1 in fp32 and G in 32-bit fixed point.  Both fit beside the node table at once, so a
// fused launch walks every code ONCE for both products (each visit: one P1 gather, one native
// 32-bit shared atomic) where the fp64 path walks twice and adds two words per visit.  G's scale is
// 2^(30 - e) with sum |u| < 2^e, so no partial sum leaves int32.
#include "toc_batch.cuh"

namespace toc {

struct Linalg32Args {
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  const int64_t* row_base;
  int64_t n_blocks;
  int32_t kind, n_cols, batch_smem_budget;
  const float* v;
  float* R;
  const float* u;
  float* O;
  const uint8_t* trees;
  const int64_t* tree_off;
};

// 2^(30 - e) for bound < 2^e: |sum| <= bound stays below 2^30.
TOC_D double fix32_scale(double bound) {
  if (!(bound > 0.0)) return 1.0;
  int e;
  frexp(bound, &e);
  return ldexp(1.0, 30 - e);
}

template <bool kWide, bool kVecSmem>
__global__ void __launch_bounds__(1024, 1) linalg32_kernel(Linalg32Args a) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* s_red = reinterpret_cast<double*>(smem + 160);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 448);
  uint8_t* p = smem + kFixedBytes;
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  const bool do_mv = a.kind & TOC_MATVEC, do_vm = a.kind & TOC_VECMAT;
  const int32_t ncol = a.n_cols;
  float* vec_s = nullptr;
  float* out_s = nullptr;
  if (kVecSmem) {
    vec_s = reinterpret_cast<float*>(p);
    p += align16(4u * ncol);
    out_s = reinterpret_cast<float*>(p);
    p += align16(4u * ncol);
    if (do_mv)
      for (int32_t c = tid; c < ncol; c += nth) vec_s[c] = a.v[c];
  }
  uint32_t phase = 0;
  if (tid == 0) mbar_init(mbar, 1);
  __syncthreads();
  using Rec = typename PairRec<kWide>::T;
  using RP = PairRec<kWide>;
  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const TocBlockMeta m = a.meta[b];
    if (m.status != TOC_OK || m.corrupt) continue;
    if (tid == 0 && b + gridDim.x < a.n_blocks) {  // the next batch's value index and cache entry into L2
      const int64_t bn = b + gridDim.x;
      const TocBlockMeta& mn = a.meta[bn];
      if (mn.status == TOC_OK) {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.arena + a.block_off[bn]),
                     "r"(align16(mn.off_uniques + 8u * mn.n_uniques))
                     : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.trees + a.tree_off[bn]),
                     "r"(cache_layout<kWide>(mn).total)
                     : "memory");
      }
    }
    __syncthreads();
    const int64_t rb = a.row_base[b];
    uint8_t* tree = const_cast<uint8_t*>(a.trees + a.tree_off[b]);
    const CacheLayout CL = cache_layout<kWide>(m);
    const Rec* irec = reinterpret_cast<const Rec*>(tree + CL.off_irec);
    const Rec* prec = reinterpret_cast<const Rec*>(tree + CL.off_prec);
    const uint2* segs = reinterpret_cast<const uint2*>(tree + CL.off_segs);
    const uint32_t n_segs = __ldg(reinterpret_cast<const uint32_t*>(tree + CL.off_info));
    Batch<kWide> B;
    B.init(a.arena + a.block_off[b], m, p);
    if (tid == 0) bulk_load(p, tree, CL.tree, mbar);
    B.load_values();
    float* p1 = reinterpret_cast<float*>(B.tab);  // [nI + 1]
    uint32_t* g = B.tabw + (B.nI + 1);            // [nI + 1]
    if (do_vm) {
      double su = 0.0;
      for (uint32_t r = tid; r < B.n; r += nth) su += fabs((double)a.u[rb + r]);
      su = warp_sum(su);
      if ((tid & 31) == 0) s_red[tid >> 5] = su;
      if (kVecSmem)
        for (int32_t c = tid; c < ncol; c += nth) out_s[c] = 0.0f;
    }
    __syncthreads();  // uniq and the partial sums complete
    double g_scale = 1.0;
    bool g_f32 = false;  // 32-bit fixed point too coarse for this batch: accumulate G in fp32
    if (do_vm) {
      double su = 0.0;
      for (uint32_t w = 0; w < (nth >> 5); ++w) su += s_red[w];
      g_scale = fix32_scale(su);
      // rounding errors of +-q/2 per addend (q = 1/g_scale) are independent: a column's error has
      // standard deviation q * max|value| * sqrt(n/12); keep 6 of them under 2^-15 (the bar is 1e-4)
      const double vmax = __ldg(reinterpret_cast<const double*>(tree + CL.off_info + 8));
      g_f32 = 6.0 * vmax * sqrt((double)B.n / 12.0) / g_scale > 0x1p-15;
    }
    float* gf = reinterpret_cast<float*>(g);
    for (uint32_t i = tid; i < B.nI; i += nth) {
      const Rec r = __ldg(irec + i);
      if (do_mv) p1[i + 1] = (float)(B.uniq[RP::b(r)] * (double)(kVecSmem ? vec_s[RP::a(r)] : a.v[RP::a(r)]));
      if (do_vm) g[i + 1] = 0u;
    }
    mbar_wait(mbar, phase);
    phase ^= 1u;
    __syncthreads();
    // one walk for both products: A.v reads P1, v^T.A adds the row's fixed-point weight to G
    for (uint32_t k = 0; k < B.passes; ++k) {
      uint32_t r, lo, hi, db, j0, j1;
      const bool ok = B.segment(k, r, lo, hi, db, j0, j1);
      float part = 0.0f;
      if (ok) {
        const uint32_t wr = do_vm && !g_f32 ? (uint32_t)__double2int_rn((double)a.u[rb + r] * g_scale) : 0u;
        const float wf = do_vm ? a.u[rb + r] : 0.0f;
        if (do_vm && g_f32) {
          if (do_mv)
            B.walk_flat(r, lo, hi, db, j0, j1, [&](uint32_t i) {
              part += p1[i];
              atomicAdd(gf + i, wf);
            });
          else if (wf != 0.0f)
            B.walk_flat(r, lo, hi, db, j0, j1, [&](uint32_t i) { atomicAdd(gf + i, wf); });
        } else if (do_mv && do_vm)
          B.walk_flat(r, lo, hi, db, j0, j1, [&](uint32_t i) {
            part += p1[i];
            atomicAdd(g + i, wr);
          });
        else if (do_mv)
          B.walk(r, lo, hi, db, j0, j1, [&](uint32_t i) { part += p1[i]; });
        else if (wr)
          B.walk_flat(r, lo, hi, db, j0, j1, [&](uint32_t i) { atomicAdd(g + i, wr); });
      }
      if (do_mv) {
        __syncwarp();
        for (uint32_t o = B.S >> 1; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (ok && B.sub == 0) a.R[rb + r] = part;
      }
    }
    if (!do_vm) continue;
    __syncthreads();
    // out[col] = sum over the column's pairs of value * G, in (column, pair) order
    const double g_inv = 1.0 / g_scale;
    float* o = a.O + b * (int64_t)ncol;
    const uint32_t quads = nth >> 2;
    const uint32_t span = ((n_segs + quads - 1) / quads) * quads;
    for (uint32_t s = tid >> 2; s < span; s += quads) {
      double c = 0.0;
      uint2 sg = make_uint2(0u, 0u);
      if (s < n_segs) {
        sg = __ldg(segs + s);
        const uint32_t end = __ldg(&segs[s + 1].x);
        for (uint32_t q = sg.x + (tid & 3u); q < end; q += 4) {
          const Rec pr = __ldg(prec + q);
          const uint32_t i = RP::a(pr) + 1;
          c += B.uniq[RP::b(pr)] * (g_f32 ? (double)gf[i] : (double)(int32_t)g[i] * g_inv);
        }
      }
      c += __shfl_xor_sync(0xffffffffu, c, 1);
      c += __shfl_xor_sync(0xffffffffu, c, 2);
      if (s < n_segs && (tid & 3u) == 0) {
        if (kVecSmem) out_s[sg.y] = (float)c;
        else o[sg.y] = (float)c;
      }
    }
    if (kVecSmem) {
      __syncthreads();
      for (int32_t c = tid; c < ncol; c += nth) o[c] = out_s[c];
    }
  }
}

}  // namespace toc

extern "C" int toc_linalg32(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                            const int64_t* d_row_base, int64_t n_blocks, const TocPlan* plan, int32_t kind,
                            const float* d_v, float* d_R, const float* d_u, float* d_O, const uint8_t* d_trees,
                            const int64_t* d_tree_off, void* stream) {
  if (!plan || n_blocks < 0 || !(kind & (TOC_MATVEC | TOC_VECMAT)) || !d_trees || !d_tree_off) return TOC_E_ARG;
  if ((kind & TOC_MATVEC) && (!d_v || !d_R)) return TOC_E_ARG;
  if ((kind & TOC_VECMAT) && (!d_u || !d_O)) return TOC_E_ARG;
  if (plan->global_tables) return TOC_E_ARG;  // the variant needs every batch's tables in shared memory
  if (n_blocks == 0) return TOC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  toc::Linalg32Args a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.n_blocks = n_blocks;
  a.kind = kind;
  a.n_cols = plan->n_cols;
  a.v = d_v;
  a.R = d_R;
  a.u = d_u;
  a.O = d_O;
  a.trees = d_trees;
  a.tree_off = d_tree_off;
  // the fp64 plan's vector region (two f64 vectors when both products) holds the two f32 vectors
  const int nvec = ((kind & TOC_MATVEC) ? 1 : 0) + ((kind & TOC_VECMAT) ? 1 : 0);
  const uint32_t fixed64 = toc::kFixedBytes + (plan->vec_in_smem ? nvec * toc::align16(8u * (uint32_t)plan->n_cols) : 0u);
  const uint32_t fixed32 = toc::kFixedBytes + (plan->vec_in_smem ? 2u * toc::align16(4u * (uint32_t)plan->n_cols) : 0u);
  const int smem = plan->smem_bytes - (int)fixed64 + (int)fixed32;
  a.batch_smem_budget = smem - (int)fixed32;
  if ((kind & TOC_VECMAT) && !plan->vec_in_smem)
    if (cudaMemsetAsync(d_O, 0, sizeof(float) * (size_t)n_blocks * plan->n_cols, s) != cudaSuccess) return TOC_E_CUDA;
  void* fn;
  if (plan->wide)
    fn = plan->vec_in_smem ? (void*)toc::linalg32_kernel<true, true> : (void*)toc::linalg32_kernel<true, false>;
  else
    fn = plan->vec_in_smem ? (void*)toc::linalg32_kernel<false, true> : (void*)toc::linalg32_kernel<false, false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return TOC_E_CUDA;
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3(plan->ctas), dim3(plan->threads), args, smem, s) == cudaSuccess ? TOC_OK
                                                                                                   : TOC_E_CUDA;
}
