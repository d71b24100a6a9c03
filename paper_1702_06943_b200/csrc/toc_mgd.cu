// toc_mgd.cu -- mini-batch gradient descent for GLMs directly on TOC-compressed batches.
//
// Reference: training.py:261-281 (glm_gradient: z = A.w, per-example scalar s, g = s^T.A, summed),
// :296-316 (apply_update / mgd_step: w - (lr / |B|) * g), :336-361 (train), :231-258
// (empirical_risk).
//
// Epoch kernel ("relay"): one cooperative launch runs a whole epoch.  CTA c owns steps
// t = c, c + G, c + 2G, ...  For step t it first rebuilds batch t's node tables (independent of
// w, so this overlaps the G-1 steps in flight on other SMs), then waits until the global step
// counter reaches t, reads the current weights through L2, runs A.w -> s -> s^T.A -> update,
// and publishes the new weights with a release store of t + 1.  The dependency chain therefore
// costs only the weight-dependent part of each step plus one L2 handoff.
#include <algorithm>

#include "toc_glm.cuh"

namespace toc {

struct MgdArgs {
  const uint8_t* arena;
  const int64_t* block_off;
  const TocBlockMeta* meta;
  const int64_t* row_base;
  int64_t n_blocks;       // steps of the epoch, in batch order
  int32_t n_cols;
  int32_t loss;           // TOC_LOSS_*
  double lr;
  const double* labels;   // per row, batch order
  double* w;              // weights (n_cols), updated in place
  uint32_t* counter;      // completed steps (0 at launch)
  uint32_t* abort_flag;   // set on a spin timeout; every CTA then exits
  int32_t batch_smem_budget;
  int32_t small_m;        // 1: gradient accumulators + touched bitmap in shared memory
  int64_t slab_bytes;     // global slab per CTA (tables of oversized batches)
  uint8_t* scratch;       // [ctas * slab_bytes] tables, then [ctas * 8 * n_cols] accumulators
  double* grad_out;       // gradient kernel only: [n_blocks x n_cols] summed gradients
  long long* trace;       // optional: kTracePoints clock64 stamps per step (phase profiling)
  uint32_t* minidx;       // large n_cols: per-CTA [n_cols] scratch, all 0xffffffff between steps
  uint32_t* leaders;      // large n_cols: per-CTA [max |I|] leader of each first-layer pair
  uint2* irec;            // large n_cols: per-CTA [max |I|] unpacked (column, value ref) per pair
  int32_t max_pairs;
};

TOC_D void stamp(const MgdArgs& a, int64_t t, int k) {
  if (a.trace && threadIdx.x == 0) a.trace[t * kTracePoints + k] = clock64();
}

// Gradient of one batch into fixed-point column accumulators `acc` (2 words per column).
// Returns the inverse output scale.  srow: n doubles of shared memory.  Entered after the node
// tables are complete (keys resolved) and `w` is current.
// Weight-independent part of a step, done while earlier steps run on other SMs: the node
// tables plus the bounds that fix the fixed-point scales (max |value|, sum |y|).
template <bool kWide>
TOC_D void build_step(Batch<kWide>& B, const MgdArgs& a, int64_t b, uint32_t* s_warp, double* s_red,
                      double& vmax, double& ysum, uint32_t* minidx = nullptr, uint32_t* leaders = nullptr) {
  const int64_t rb = a.row_base[b];
  if (threadIdx.x == 0) {  // the whole block into L2: the weight-dependent phases re-read I
    const uint32_t bytes = align16(B.m.off_offsets + (B.m.n_rows + 1u) * B.m.w_offsets);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(B.blk), "r"(bytes) : "memory");
  }
  B.load_index(s_warp);
  B.build_nodes();
  double ys = 0.0;
  for (uint32_t r = threadIdx.x; r < B.n; r += blockDim.x) ys += fabs(a.labels[rb + r]);
  __syncthreads();
  B.resolve_keys();
  if (minidx) {
    // Unpack every first-layer pair to an aligned record and find each column's leader (its
    // smallest pair id in this batch).  All weight-independent, so it runs here, off the critical
    // path: atomicMin into a per-CTA column table, read back, then reset for the CTA's next step.
    const uint8_t* cols = B.blk + B.m.off_cols;
    const uint8_t* refs = B.blk + B.m.off_refs;
    for (uint32_t i = threadIdx.x; i < B.nI; i += blockDim.x) {
      const uint32_t c = ld_packed(cols, i, B.m.w_cols);
      a.irec[i] = make_uint2(c, ld_packed(refs, i, B.m.w_refs));
      atomicMin(minidx + c, i);
    }
    __threadfence();  // the minima are performed in L2; read them back through L2
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < B.nI; i += blockDim.x) leaders[i] = __ldcg(minidx + __ldcg(&a.irec[i].x));
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < B.nI; i += blockDim.x) minidx[__ldcg(&a.irec[i].x)] = 0xffffffffu;
  }
  vmax = block_max_d(B.vmax, s_red);
  ysum = block_sum(ys, s_red);
}

// Large n_cols: g[c] = sum of value_i * G_i over the first-layer pairs i of column c, reduced in
// shared memory into the column's leader slot (fixed point: exact and order-independent), then
// w[c] -= (lr / |B|) * g[c] by the leader with one plain read-modify-write (apply_update,
// training.py:296-300).  No global atomics on the critical path.
template <bool kWide>
TOC_D void update_leaders(Batch<kWide>& B, const MgdArgs& a, const uint32_t* leaders, double g_scale,
                          double o_scale) {
  const double g_inv = 1.0 / g_scale, o_inv = 1.0 / o_scale, step = a.lr / (double)B.n;
  const uint32_t nI = B.nI, nth = blockDim.x, tid = threadIdx.x;
  // contributions value_i * G_i, as fixed point at o_scale, in place
#pragma unroll 4
  for (uint32_t i = tid; i < nI; i += nth) {
    const uint32_t ref = __ldcg(&a.irec[i].y);
    const double c = B.uniq[ref] * fix_value(B.tabw[2 * (i + 1)], B.tabw[2 * (i + 1) + 1], g_inv);
    const long long f = __double2ll_rn(c * o_scale);
    B.tabw[2 * (i + 1)] = (uint32_t)f;
    B.tabw[2 * (i + 1) + 1] = (uint32_t)((unsigned long long)f >> 32);
  }
  __syncthreads();
#pragma unroll 4
  for (uint32_t i = tid; i < nI; i += nth) {  // non-leaders fold into their leader
    const uint32_t l = __ldcg(leaders + i);
    if (l != i) {
      const long long f = (long long)(((unsigned long long)B.tabw[2 * (i + 1) + 1] << 32) | B.tabw[2 * (i + 1)]);
      if (f) fix_add(B.tabw + 2 * (l + 1), f);
    }
  }
  __syncthreads();
#pragma unroll 4
  for (uint32_t i = tid; i < nI; i += nth) {
    if (__ldcg(leaders + i) != i) continue;
    const double g = fix_value(B.tabw[2 * (i + 1)], B.tabw[2 * (i + 1) + 1], o_inv);
    if (g == 0.0) continue;
    const uint32_t c = __ldcg(&a.irec[i].x);
    a.w[c] = __dsub_rn(__ldcg(a.w + c), __dmul_rn(step, g));
  }
}

// P1[i] = value_i * w[col_i] from the unpacked records (large n_cols: thread-strided and unrolled
// so the dependent record -> weight loads of different pairs overlap).
template <bool kWide>
TOC_D void p1_records(Batch<kWide>& B, const MgdArgs& a) {
#pragma unroll 4
  for (uint32_t i = threadIdx.x; i < B.nI; i += blockDim.x) {
    const uint2 rec = __ldcg(a.irec + i);
    B.tab[i + 1] = B.uniq[rec.y] * __ldcg(a.w + rec.x);
  }
}

// Gradient of one batch: P1 from w, A.w, the loss scalar, s^T.A into G (fixed point).  Returns
// g_scale.  srow: n doubles of shared memory.  For logistic and hinge |s| <= |y|, so the scale
// comes from the precomputed sum |y| and no reduction sits on the critical path.
template <bool kWide, bool kCG>
TOC_D double batch_gradient(Batch<kWide>& B, const MgdArgs& a, int64_t b, double* srow, double ysum,
                            double* s_red, double& bound_out) {
  const uint32_t tid = threadIdx.x, nth = blockDim.x;
  const int64_t rb = a.row_base[b];
  if (a.irec) p1_records(B, a);
  else B.template compute_p1<kCG>(a.w);
  __syncthreads();
  stamp(a, b, 2);
  B.matvec_rows([&](uint32_t r, double z) { srow[r] = loss_scalar(a.loss, a.labels[rb + r], z); });
  __syncthreads();
  stamp(a, b, 3);
  double bound = ysum;
  if (a.loss == TOC_LOSS_SQUARED) {
    double su = 0.0;
    for (uint32_t r = tid; r < B.n; r += nth) su += fabs(srow[r]);
    bound = block_sum(su, s_red);
  }
  B.zero_tab();
  __syncthreads();
  stamp(a, b, 4);
  const double g_scale = fix_scale(bound);
  bound_out = bound;
  B.vecmat_rows([&](uint32_t r) { return srow[r]; }, g_scale);
  __syncthreads();
  stamp(a, b, 5);
  return g_scale;
}

// Small n_cols: column gradients in shared fixed-point accumulators (deterministic), then
// w[c] -= (lr / |B|) * g[c] once per touched column (apply_update, training.py:296-300; untouched
// columns have g = 0 and stay bit-identical).  Accumulators are cleared for the next step.
template <bool kWide>
TOC_D void update_small(Batch<kWide>& B, const MgdArgs& a, uint32_t* acc, uint32_t* touched, double g_scale,
                        double vmax, double ysum_or_bound) {
  const double o_scale = fix_scale(ysum_or_bound * vmax), o_inv = 1.0 / o_scale;
  B.scatter_columns(acc, 1.0 / g_scale, o_scale);
  __syncthreads();
  const double step = a.lr / (double)B.n;
  B.for_each_pair_column([&](uint32_t, uint32_t c) {
    const uint32_t bit = 1u << (c & 31);
    if (atomicOr(&touched[c >> 5], bit) & bit) return;  // another pair of this column won
    const double g = fix_value(acc[2 * c], acc[2 * c + 1], o_inv);
    a.w[c] = __dsub_rn(__ldcg(a.w + c), __dmul_rn(step, g));  // L2: other CTAs wrote w
    acc[2 * c] = 0u;
    acc[2 * c + 1] = 0u;
  });
}

template <bool kWide>
__global__ void __launch_bounds__(1024, 1) glm_epoch_kernel(MgdArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  double* s_red = reinterpret_cast<double*>(smem + 160);
  __shared__ uint32_t s_go;
  uint8_t* p = smem + kFixedBytes;
  const uint32_t tid = threadIdx.x, nth = blockDim.x, m = (uint32_t)a.n_cols, words = (m + 31) / 32;
  uint32_t* touched = nullptr;
  uint32_t* acc = nullptr;
  uint32_t* minidx = nullptr;
  uint32_t* leaders = nullptr;
  if (!a.small_m) {
    // scratch after the slabs: [ctas][m4] minidx, [ctas][p4] leaders, [ctas][p4] irec (uint2);
    // m4 / p4 rounded to multiples of 4 so every region stays 16-byte aligned
    const int64_t m4 = ((int64_t)m + 3) & ~3ll, p4 = ((int64_t)a.max_pairs + 3) & ~3ll;
    uint8_t* base = a.scratch + (int64_t)gridDim.x * a.slab_bytes;
    minidx = reinterpret_cast<uint32_t*>(base) + (int64_t)blockIdx.x * m4;
    base += (int64_t)gridDim.x * 4 * m4;
    leaders = reinterpret_cast<uint32_t*>(base) + (int64_t)blockIdx.x * p4;
    base += (int64_t)gridDim.x * 4 * p4;
    a.irec = reinterpret_cast<uint2*>(base) + (int64_t)blockIdx.x * p4;
  } else {
    a.irec = nullptr;
  }
  if (a.small_m) {
    touched = reinterpret_cast<uint32_t*>(p);
    p += align16(4u * words);
    acc = reinterpret_cast<uint32_t*>(p);
    p += align16(8u * m);
    for (uint32_t c = tid; c < 2 * m; c += nth) acc[c] = 0u;
  }
  for (int64_t t = blockIdx.x; t < a.n_blocks; t += gridDim.x) {
    const TocBlockMeta mt = a.meta[t];
    Batch<kWide> B;
    double* srow = reinterpret_cast<double*>(p);
    uint8_t* tables = p + align16(8u * mt.n_rows);
    const uint32_t need = batch_layout<kWide>(mt).total + align16(8u * mt.n_rows);
    if (need > (uint32_t)a.batch_smem_budget) tables = a.scratch + (int64_t)blockIdx.x * a.slab_bytes;
    B.init(a.arena + a.block_off[t], mt, tables);
    if (a.small_m)
      for (uint32_t w = tid; w < words; w += nth) touched[w] = 0u;
    double vmax, ysum;
    build_step(B, a, t, s_warp, s_red, vmax, ysum, minidx, leaders);
    stamp(a, t, 0);
    // Wait for the weights of step t.  Only the owner of the next step polls tightly; owners of
    // later steps back off in proportion to their distance, so the counter's L2 slice is not
    // flooded (a hot slice stalls every access hashed to it, including the critical path's).
    // Bounded by a 4 s timeout: a hang would take the GPU down with it.
    if (tid == 0) {
      uint32_t go = 1;
      const unsigned long long t0 = globaltimer_ns();
      for (uint32_t it = 0;; ++it) {
        const uint32_t c = ld_acquire(a.counter);
        if (c == (uint32_t)t) break;
        const uint32_t dist = (uint32_t)t - c;
        if ((it & 255u) == 255u) {
          if (ld_acquire(a.abort_flag)) { go = 0; break; }
          if (globaltimer_ns() - t0 > 4000000000ull) { atomicExch(a.abort_flag, 1u); go = 0; break; }
        }
        __nanosleep(dist <= 1 ? 20u : (dist < 16 ? 200u * dist : 4000u));
      }
      s_go = go;
    }
    __syncthreads();
    if (!s_go) return;
    stamp(a, t, 1);
    double bound;
    const double g_scale = batch_gradient<kWide, true>(B, a, t, srow, ysum, s_red, bound);
    if (a.small_m) update_small(B, a, acc, touched, g_scale, vmax, bound);
    else update_leaders(B, a, leaders, g_scale, fix_scale(bound * vmax));
    stamp(a, t, 6);
    __threadfence();
    __syncthreads();
    stamp(a, t, 7);
    if (tid == 0) st_release(a.counter, (uint32_t)t + 1);
  }
}

// Summed gradient of each batch (no update): grad_out[b, :] = s_b^T A_b.  Data-parallel MGD
// all-reduces these across ranks before the update.
template <bool kWide>
__global__ void __launch_bounds__(1024, 1) glm_grad_kernel(MgdArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem);
  double* s_red = reinterpret_cast<double*>(smem + 160);
  uint8_t* p = smem + kFixedBytes;
  const uint32_t tid = threadIdx.x, nth = blockDim.x, m = (uint32_t)a.n_cols;
  uint32_t* acc;
  if (a.small_m) {
    acc = reinterpret_cast<uint32_t*>(p);
    p += align16(8u * m);
  }
  for (int64_t b = blockIdx.x; b < a.n_blocks; b += gridDim.x) {
    const TocBlockMeta mb = a.meta[b];
    double* srow = reinterpret_cast<double*>(p);
    uint8_t* tables = p + align16(8u * mb.n_rows);
    const uint32_t need = batch_layout<kWide>(mb).total + align16(8u * mb.n_rows);
    if (need > (uint32_t)a.batch_smem_budget) tables = a.scratch + (int64_t)blockIdx.x * a.slab_bytes;
    double* g = a.grad_out + b * (int64_t)m;
    if (!a.small_m) acc = reinterpret_cast<uint32_t*>(g);  // accumulate in place (zeroed by the host)
    __syncthreads();
    if (a.small_m)
      for (uint32_t c = tid; c < 2 * m; c += nth) acc[c] = 0u;
    Batch<kWide> B;
    B.init(a.arena + a.block_off[b], mb, tables);
    double vmax, ysum, bound;
    build_step(B, a, b, s_warp, s_red, vmax, ysum);
    __syncthreads();
    const double g_scale = batch_gradient<kWide, false>(B, a, b, srow, ysum, s_red, bound);
    const double o_scale = fix_scale(bound * vmax), o_inv = 1.0 / o_scale;
    B.scatter_columns(acc, 1.0 / g_scale, o_scale);
    __syncthreads();
    if (a.small_m) {
      for (uint32_t c = tid; c < m; c += nth) g[c] = fix_value(acc[2 * c], acc[2 * c + 1], o_inv);
    } else {
      uint32_t* gw = reinterpret_cast<uint32_t*>(g);
      for (uint32_t c = tid; c < m; c += nth) g[c] = fix_value(__ldcg(gw + 2 * c), __ldcg(gw + 2 * c + 1), o_inv);
    }
  }
}

// Per-row loss of empirical_risk (training.py:231-258) and its sum (one double per CTA).
__global__ void risk_kernel(const double* z, const double* y, int64_t n, int32_t loss, double* part) {
  __shared__ double s_red[33];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double yz = y[i] * z[i];
    double l;
    if (loss == TOC_LOSS_SQUARED) {
      const double d = y[i] - z[i];
      l = 0.5 * d * d;
    } else if (loss == TOC_LOSS_LOGISTIC) {  // softplus(-y z), overflow-free (training.py:206-212)
      const double t = -yz;
      l = t > 0.0 ? t + log1p(exp(-t)) : log1p(exp(t));
    } else {
      l = fmax(0.0, 1.0 - yz);
    }
    acc += l;
  }
  acc = block_sum(acc, s_red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

}  // namespace toc

// ------------------------------------------------------------------------------------------
namespace {

int g_max_ctas = 0;  // diagnostic cap on the MGD grid (0: one CTA per SM)

struct MgdLaunch {
  int threads, ctas, smem;
  int32_t budget, small_m, max_pairs;
  int64_t slab, scratch;
};

int dev_count(int attr) {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, (cudaDeviceAttr)attr, dev);
  return v;
}

MgdLaunch mgd_plan(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, bool wide, bool epoch) {
  MgdLaunch L{};
  int sm = dev_count(cudaDevAttrMultiProcessorCount), optin = dev_count(cudaDevAttrMaxSharedMemoryPerBlockOptin);
  if (sm <= 0) {
    sm = 148;
    optin = 232448;
  }
  uint32_t max_need = 0;
  for (int64_t b = 0; b < n_blocks; ++b) {
    const uint32_t need = (wide ? toc::batch_layout<true>(h_meta[b]).total : toc::batch_layout<false>(h_meta[b]).total) +
                          toc::align16(8u * h_meta[b].n_rows);
    if (need > max_need) max_need = need;
  }
  const uint32_t m = (uint32_t)n_cols;
  const uint32_t small_bytes = toc::align16(8u * m);
  L.small_m = small_bytes <= 32u * 1024u;
  uint32_t fixed = toc::kFixedBytes + (L.small_m ? small_bytes + (epoch ? toc::align16(4u * ((m + 31) / 32)) : 0u) : 0u);
  uint32_t max_ni = 0;
  for (int64_t b = 0; b < n_blocks; ++b) max_ni = max_ni > h_meta[b].n_pairs ? max_ni : h_meta[b].n_pairs;
  L.max_pairs = (int32_t)max_ni;
  uint32_t avail = (uint32_t)optin > fixed ? (uint32_t)optin - fixed : 0u;
  L.budget = (int32_t)(max_need <= avail ? max_need : avail);
  L.smem = (int)(fixed + (uint32_t)L.budget);
  L.threads = 1024;
  L.ctas = (int)(n_blocks < sm ? (n_blocks > 0 ? n_blocks : 1) : sm);
  if (g_max_ctas > 0 && L.ctas > g_max_ctas) L.ctas = g_max_ctas;
  L.slab = max_need > (uint32_t)L.budget ? (int64_t)toc::align16(max_need) : 0;
  L.scratch = (int64_t)L.ctas * L.slab;
  if (epoch && !L.small_m)  // minidx, leaders, irec (see glm_epoch_kernel)
    L.scratch += (int64_t)L.ctas * 4 * ((((int64_t)m + 3) & ~3ll) + 3 * (((int64_t)max_ni + 3) & ~3ll));
  return L;
}

}  // namespace

extern "C" int toc_mgd_set_max_ctas(int32_t n) {
  g_max_ctas = n;
  return TOC_OK;
}

extern "C" int toc_mgd_plan_info(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t kind,
                                 int64_t* info /* 8: smem, budget, small_m, sorted_cols, key_slots, ctas, slab, wide */) {
  if (!h_meta || n_blocks < 0 || !info) return TOC_E_ARG;
  bool wide = false;
  for (int64_t b = 0; b < n_blocks; ++b)
    if (1ull + h_meta[b].n_pairs + h_meta[b].n_derived > 65536ull) wide = true;
  MgdLaunch L = mgd_plan(h_meta, n_blocks, n_cols, wide, kind == 0);
  info[0] = L.smem;
  info[1] = L.budget;
  info[2] = L.small_m;
  info[3] = 0;
  info[4] = L.max_pairs;
  info[5] = L.ctas;
  info[6] = L.slab;
  info[7] = wide;
  return TOC_OK;
}

extern "C" int toc_mgd_workspace(const TocBlockMeta* h_meta, int64_t n_blocks, int32_t n_cols, int32_t kind,
                                 int64_t* scratch_bytes) {
  if (!h_meta || n_blocks < 0 || !scratch_bytes) return TOC_E_ARG;
  bool wide = false;
  for (int64_t b = 0; b < n_blocks; ++b)
    if (1ull + h_meta[b].n_pairs + h_meta[b].n_derived > 65536ull) wide = true;
  *scratch_bytes = mgd_plan(h_meta, n_blocks, n_cols, wide, kind == 0).scratch;
  return TOC_OK;
}

static int mgd_launch(const TocBlockMeta* h_meta, const toc::MgdArgs& a0, bool epoch, cudaStream_t s) {
  bool wide = false;
  for (int64_t b = 0; b < a0.n_blocks; ++b)
    if (1ull + h_meta[b].n_pairs + h_meta[b].n_derived > 65536ull) wide = true;
  MgdLaunch L = mgd_plan(h_meta, a0.n_blocks, a0.n_cols, wide, epoch);
  toc::MgdArgs a = a0;
  a.batch_smem_budget = L.budget;
  a.small_m = L.small_m;
  a.max_pairs = L.max_pairs;
  if (epoch && !L.small_m)  // column tables start "empty"
    if (cudaMemsetAsync(a.scratch + (int64_t)L.ctas * L.slab, 0xff, (size_t)L.ctas * 4 * ((a.n_cols + 3) & ~3), s) !=
        cudaSuccess)
      return TOC_E_CUDA;
  a.slab_bytes = L.slab;
  if (L.scratch > 0 && !a.scratch) return TOC_E_ARG;
  void* fn;
  if (epoch) fn = wide ? (void*)toc::glm_epoch_kernel<true> : (void*)toc::glm_epoch_kernel<false>;
  else fn = wide ? (void*)toc::glm_grad_kernel<true> : (void*)toc::glm_grad_kernel<false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem) != cudaSuccess) return TOC_E_CUDA;
  void* args[] = {&a};
  cudaError_t e;
  if (epoch) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, L.threads, L.smem);
    if (per_sm < 1) return TOC_E_CUDA;
    e = cudaLaunchCooperativeKernel(fn, dim3(L.ctas), dim3(L.threads), args, L.smem, s);
  } else {
    e = cudaLaunchKernel(fn, dim3(L.ctas), dim3(L.threads), args, L.smem, s);
  }
  return e == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_glm_epoch_traced(const uint8_t*, const int64_t*, const TocBlockMeta*, const TocBlockMeta*,
                                    const int64_t*, int64_t, int32_t, int32_t, double, const double*, double*, uint32_t*,
                                    void*, long long*, void*);

extern "C" int toc_glm_epoch(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                             const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks, int32_t n_cols,
                             int32_t loss, double lr, const double* d_labels, double* d_w, uint32_t* d_sync,
                             void* d_scratch, void* stream) {
  return toc_glm_epoch_traced(d_arena, d_block_off, d_meta, h_meta, d_row_base, n_blocks, n_cols, loss, lr, d_labels,
                              d_w, d_sync, d_scratch, nullptr, stream);
}

extern "C" int toc_glm_epoch_traced(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                                    const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks,
                                    int32_t n_cols, int32_t loss, double lr, const double* d_labels, double* d_w,
                                    uint32_t* d_sync, void* d_scratch, long long* d_trace, void* stream) {
  if (n_blocks <= 0) return n_blocks == 0 ? TOC_OK : TOC_E_ARG;
  if (!h_meta || !d_w || !d_labels || !d_sync || loss < 0 || loss > 2) return TOC_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(d_sync, 0, 256, s) != cudaSuccess) return TOC_E_CUDA;
  toc::MgdArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.n_blocks = n_blocks;
  a.n_cols = n_cols;
  a.loss = loss;
  a.lr = lr;
  a.labels = d_labels;
  a.w = d_w;
  a.counter = d_sync;
  a.abort_flag = d_sync + 32;  // its own 128-byte line
  a.scratch = (uint8_t*)d_scratch;
  a.trace = d_trace;
  return mgd_launch(h_meta, a, true, s);
}

extern "C" int toc_glm_grad(const uint8_t* d_arena, const int64_t* d_block_off, const TocBlockMeta* d_meta,
                            const TocBlockMeta* h_meta, const int64_t* d_row_base, int64_t n_blocks, int32_t n_cols,
                            int32_t loss, const double* d_labels, const double* d_w, double* d_grad,
                            void* d_scratch, void* stream) {
  if (n_blocks <= 0) return n_blocks == 0 ? TOC_OK : TOC_E_ARG;
  if (!h_meta || !d_w || !d_labels || !d_grad || loss < 0 || loss > 2) return TOC_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(d_grad, 0, sizeof(double) * (size_t)n_blocks * n_cols, s) != cudaSuccess) return TOC_E_CUDA;
  toc::MgdArgs a{};
  a.arena = d_arena;
  a.block_off = d_block_off;
  a.meta = d_meta;
  a.row_base = d_row_base;
  a.n_blocks = n_blocks;
  a.n_cols = n_cols;
  a.loss = loss;
  a.labels = d_labels;
  a.w = const_cast<double*>(d_w);
  a.scratch = (uint8_t*)d_scratch;
  a.grad_out = d_grad;
  return mgd_launch(h_meta, a, false, s);
}

extern "C" int toc_glm_risk(const double* d_z, const double* d_y, int64_t n, int32_t loss, double* d_partial,
                            int32_t n_partial, void* stream) {
  if (n < 0 || n_partial < 1 || loss < 0 || loss > 2) return TOC_E_ARG;
  toc::risk_kernel<<<n_partial, 256, 0, (cudaStream_t)stream>>>(d_z, d_y, n, loss, d_partial);
  return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}
