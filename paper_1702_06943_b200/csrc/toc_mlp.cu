// toc_mlp.cu -- one epoch of the config-5 MLP (784-h-k, ReLU, softmax cross-entropy, biases) on
// TOC batches, launched natively: per step four kernels, no host round trip.
//
// Reference: the step restated in oracle.train_mlp (first layer through matmat_right /
// matmat_left, kernels.py:177-234, Algorithms 8 and 9; the dense tail as training.py:284-316 does
// for its own net).  The two first-layer products are GEMM-shaped (n x m times m x h and m x n
// times n x h, h = 200), so here they run on the fp64 tensor cores (mma.sync m8n8k4 f64, DMMA):
// the step's batch is decoded from the node-record cache (toc_matcache.cu) into a dense buffer the
// size of one batch (1.6 MB at config 5: it lives in L2 between the kernels of the step; HBM keeps
// only the compressed form and the cache) and both products read their tiles from it.  Per step:
//   mlp_decode  one thread per code walks its chain into the buffer; the other buffer (read by the
//               previous step) is zeroed for the next.
//   mlp_right   Z1 = A_b . W1 (CTA per 8 rows x 40 hidden units; K split over 16 warps, the
//               partial tiles summed in warp order); epilogue A1 = relu(Z1 + b1).
//   mlp_tail    per row (warp): logits = A1 W2 + b2, P = softmax - onehot(y), delta = (P W2^T) *
//               [A1 > 0]; per CTA the sums over its 8 rows of A1^T P, delta and P.
//   mlp_left    G = A_b^T . delta (CTA per 16 columns x 40 hidden units, K = rows split over the
//               warps); epilogue W1 -= s G.  Extra CTAs sum the tail CTAs' parts in CTA order and
//               update W2, b1, b2 (the tail has finished reading them).
// s = lr / n_b.  Every sum is in a fixed order, so an epoch is deterministic.
#include <vector>

#include "toc_batch.cuh"
#include "toc_images.cuh"  // cluster barrier / rank / DSMEM load helpers

namespace toc {

// MLP step cache entry (layout: toc_matcache.cu, dc_layout): 4-byte node records (parent | key <<
// 17), pair records (column | value ref << 16), the value index and row offsets; the code stream is
// read from the batch's TOC1 block itself.
struct MlpEntry {
  const uint32_t* rowoff;
  const uint32_t* pairs;
  const uint32_t* nodes;
  const double* uniq;
  uint32_t n_rows, n_codes, nI, nU, off_codes, w_codes;
};

TOC_D MlpEntry mlp_entry(const uint8_t* e) {
  const uint32_t* h = reinterpret_cast<const uint32_t*>(e);
  MlpEntry E;
  E.n_rows = __ldg(h);
  E.n_codes = __ldg(h + 1);
  E.nI = __ldg(h + 3);
  E.nU = __ldg(h + 5);
  E.off_codes = __ldg(h + 6);
  E.w_codes = __ldg(h + 7);
  E.rowoff = reinterpret_cast<const uint32_t*>(e + __ldg(h + 8));
  E.pairs = reinterpret_cast<const uint32_t*>(e + __ldg(h + 9));
  E.nodes = reinterpret_cast<const uint32_t*>(e + __ldg(h + 10));
  E.uniq = reinterpret_cast<const double*>(e + __ldg(h + 11));
  return E;
}

// D = A.B + C on the fp64 tensor cores, 8x8x4.  Fragments (lane = 4 * g + q): A[g][q], B[q][g],
// C/D[g][2q], [g][2q + 1].
TOC_D void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

constexpr uint32_t kMlpThreads = 256;  // 8 warps
constexpr uint32_t kNT = 5;            // n-tiles (8 hidden units each) per CTA: 40 units
constexpr uint32_t kKMax = 16;         // classes

struct MlpStep {
  const uint8_t* entry;  // the batch's step cache entry
  const uint8_t* blk;    // the batch's TOC1 block (its packed code stream is decoded in place)
  double* loss;          // risk mode (toc_mlp_risk): per-row cross-entropy out, no backward pass
  int32_t m, h, k;
  double* W1;            // [m x h]
  double* b1;            // [h]
  double* W2;            // [h x k]
  double* b2;            // [k]
  const double* y;       // [n] class ids
  double* A1;            // [n x h]
  double* P;             // [n x k]
  double* D;             // [n x h]
  double* Ad;            // [n x m] this step's decoded batch
  double* Az;            // the other decode buffer, zero-filled here for the next step
  int64_t az_elems;      // its size (doubles, even); 0 when every row is dense (all overwritten)
  double* part;          // per tail CTA: sums over its rows of A1^T P [h x k], delta [h], P [k]
  double step;           // lr / n
  double* grad;          // gradient-only mode (data-parallel step): the batch's summed gradient
                         // [W1 m*h | W2 h*k | b1 h | b2 k] instead of the update; NULL: update
};

// The batch decoded into Ad: one thread per code walks its chain and stores each pair at (row,
// column); the other buffer is zeroed meanwhile (it was read by the previous step).

// Programmatic dependent launch (the step's kernels are launched with programmatic stream
// serialization): a kernel waits for its predecessor's completion and memory only where it first
// needs them, and lets its successor launch right after that wait -- so by induction every kernel
// before the predecessor has completed whenever a kernel runs.  Both are no-ops without PDL.
TOC_D void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
TOC_D void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

constexpr uint32_t kDecodeUniq = 2048;  // value-index entries kept in shared memory

constexpr uint32_t kDecodeRows = 1024;  // row offsets kept in shared memory

__global__ void __launch_bounds__(kMlpThreads) mlp_decode_kernel(MlpStep s, uint32_t n) {
  __shared__ uint32_t s_ro[kDecodeRows + 1];
  __shared__ double s_uq[kDecodeUniq];
  const MlpEntry E = mlp_entry(s.entry);
  const bool ro_s = n <= kDecodeRows, uq_s = E.nU <= kDecodeUniq;
  if (ro_s)
    for (uint32_t i = threadIdx.x; i <= n; i += blockDim.x) s_ro[i] = __ldg(E.rowoff + i);
  if (uq_s)
    for (uint32_t i = threadIdx.x; i < E.nU; i += blockDim.x) s_uq[i] = __ldg(E.uniq + i);
  __syncthreads();
  auto rowoff = [&](uint32_t r) { return ro_s ? s_ro[r] : __ldg(E.rowoff + r); };
  const uint32_t C = E.n_codes, m = (uint32_t)s.m, nI = E.nI;
  const uint8_t* codes = s.blk + E.off_codes;
  // each CTA a contiguous range of codes, its threads consecutive codes: one row search per thread,
  // then the row advances with the code index
  const uint32_t per = (C + gridDim.x - 1) / gridDim.x, c0 = blockIdx.x * per, c1 = min(C, c0 + per);
  uint32_t r = 0;
  if (c0 + threadIdx.x < c1) {
    uint32_t lo = 0, hi = n;  // row of the first code: last r with rowoff[r] <= j
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (rowoff(mid) <= c0 + threadIdx.x) lo = mid;
      else hi = mid;
    }
    r = lo;
  }
  for (uint32_t j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
    while (rowoff(r + 1) <= j) ++r;
    double* row = s.Ad + (int64_t)r * m;
    uint32_t x = ld_packed(codes, j, E.w_codes);  // the TOC1 code stream (physical.py:54-68)
    while (x > nI) {  // the code's chain, last pair first: a derived node's own pair is its key
      const uint32_t w = __ldg(E.nodes + x), pair = w >> 17;
      TOC_CHECK(pair >= 1 && pair <= nI && (w & 0x1ffffu) >= 1 && (w & 0x1ffffu) < x);
      const uint32_t pr = __ldg(E.pairs + pair);
      row[pr & 0xffffu] = uq_s ? s_uq[pr >> 16] : __ldg(E.uniq + (pr >> 16));
      x = w & 0x1ffffu;
    }
    TOC_CHECK(x >= 1);
    const uint32_t pr = __ldg(E.pairs + x);
    TOC_CHECK((pr & 0xffffu) < m && (pr >> 16) < E.nU);
    row[pr & 0xffffu] = uq_s ? s_uq[pr >> 16] : __ldg(E.uniq + (pr >> 16));
  }
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  // (the walks above only read the static cache and write this step's buffer, last read two steps
  // ago; the other buffer is still read by the previous step's kernels)
  pdl_wait();
  pdl_trigger();
  double2* z = reinterpret_cast<double2*>(s.Az);
  for (int64_t i = gt; i < s.az_elems / 2; i += gs) z[i] = make_double2(0.0, 0.0);
}

// The NW warps' partial accumulator tiles (MT m-tiles x kNT n-tiles) summed in warp order; f(row,
// col, value) for each of the CTA's outputs.
template <int MT, int NW, typename F>
TOC_D void reduce_warps(double (&acc)[MT][kNT][2], double* red, F&& f) {
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t per = MT * kNT * 64;  // doubles per warp
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (uint32_t t = 0; t < kNT; ++t)
#pragma unroll
      for (int i = 0; i < 2; ++i) red[warp * per + ((mt * kNT + t) * 2 + i) * 32 + lane] = acc[mt][t][i];
  __syncthreads();
  for (uint32_t e = tid; e < per; e += blockDim.x) {
    double s = 0.0;
    for (uint32_t w = 0; w < NW; ++w) s += red[w * per + e];
    const uint32_t ln = e & 31, rest = e >> 5, i = rest & 1, mtt = rest >> 1, t = mtt % kNT, mt = mtt / kNT;
    f(mt * 8 + (ln >> 2), t * 8 + (ln & 3) * 2 + i, s);
  }
}

// Z1 = A_b . W1 for 8*MT rows x 40 hidden units (K = m split over the warps); A1 = relu(Z1 + b1).
constexpr uint32_t kRightWarps = 16;

template <int MT>
__global__ void __launch_bounds__(32 * kRightWarps) mlp_right_kernel(MlpStep s, uint32_t n) {
  extern __shared__ __align__(16) double red[];
  pdl_wait();  // the decoded batch, and W1 / b1 as the previous step left them
  pdl_trigger();
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const uint32_t m = (uint32_t)s.m, h = (uint32_t)s.h;
  const uint32_t r0 = blockIdx.x * (8 * MT), n0 = blockIdx.y * (8 * kNT);
  double acc[MT][kNT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (uint32_t t = 0; t < kNT; ++t) acc[mt][t][0] = acc[mt][t][1] = 0.0;
  const uint32_t ksteps = (m + 3) >> 2, ks0 = warp * ksteps / kRightWarps, ks1 = (warp + 1) * ksteps / kRightWarps;
  const double* W1 = s.W1;
  const double* Ad = s.Ad;
  constexpr uint32_t G = 4;  // k-steps per group: all their fragments loaded before their DMMAs
  for (uint32_t k0 = ks0; k0 < ks1; k0 += G) {
    double a[G][MT], b[G][kNT];
#pragma unroll
    for (uint32_t u = 0; u < G; ++u) {
      const uint32_t kr = (k0 + u) * 4 + tq;
      const bool kin = k0 + u < ks1 && kr < m;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const uint32_t r = r0 + mt * 8 + g;
        a[u][mt] = (kin && r < n) ? Ad[(int64_t)r * m + kr] : 0.0;
      }
#pragma unroll
      for (uint32_t t = 0; t < kNT; ++t) {
        const uint32_t col = n0 + t * 8 + g;
        b[u][t] = (kin && col < h) ? W1[(int64_t)kr * h + col] : 0.0;
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < G; ++u)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (uint32_t t = 0; t < kNT; ++t) dmma(acc[mt][t], a[u][mt], b[u][t]);
  }
  const double* b1 = s.b1;
  double* A1 = s.A1;
  reduce_warps<MT, kRightWarps>(acc, red, [&](uint32_t row, uint32_t c, double z) {
    const uint32_t r = r0 + row, col = n0 + c;
    if (r < n && col < h) A1[(int64_t)r * h + col] = fmax(z + b1[col], 0.0);
  });
}

// mlp_right with the tail fused in: a thread-block cluster of the ncb CTAs that share a row tile
// (one per 40 hidden units).  Each CTA computes its A1 tile as mlp_right does, then the partial
// logits of its units, A1_tile . W2[units]; after a cluster barrier every CTA sums the ncb partials
// over DSMEM in rank order (identical in every CTA), adds b2 and forms P = softmax - onehot for the
// tile's rows; then delta = (P W2^T) * [A1 > 0] for its own units and its parts of the W2 / b1 / b2
// gradients (sums over the tile's rows in row order; the P sums by rank 0), laid out as the tail's
// parts, one per row tile.  Risk mode: rank 0 writes each row's -log softmax[y] instead.
template <int MT, int K>
__global__ void __launch_bounds__(32 * kRightWarps) mlp_right_tail_kernel(MlpStep s, uint32_t n) {
  extern __shared__ __align__(16) double red[];
  constexpr uint32_t RT = 8 * MT, NU = 8 * kNT;
  double* a1s = red + kRightWarps * MT * kNT * 64;  // [RT][NU] this CTA's A1 tile
  double* lgp = a1s + RT * NU;                      // [RT][K] its partial logits (read by the cluster)
  double* ps = lgp + RT * K;                        // [RT][K] P = softmax - onehot
  double* w2s = ps + RT * K;                        // [NU][K] its rows of W2
  pdl_wait();  // the decoded batch, and the parameters as the previous step left them
  pdl_trigger();
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const uint32_t m = (uint32_t)s.m, h = (uint32_t)s.h;
  const uint32_t r0 = blockIdx.x * RT, n0 = blockIdx.y * NU, rank = cluster_rank(), C = gridDim.y;
  double acc[MT][kNT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (uint32_t t = 0; t < kNT; ++t) acc[mt][t][0] = acc[mt][t][1] = 0.0;
  const uint32_t ksteps = (m + 3) >> 2, ks0 = warp * ksteps / kRightWarps, ks1 = (warp + 1) * ksteps / kRightWarps;
  const double* W1 = s.W1;
  const double* Ad = s.Ad;
  constexpr uint32_t G = 4;  // k-steps per group: all their fragments loaded before their DMMAs
  for (uint32_t k0 = ks0; k0 < ks1; k0 += G) {
    double a[G][MT], b[G][kNT];
#pragma unroll
    for (uint32_t u = 0; u < G; ++u) {
      const uint32_t kr = (k0 + u) * 4 + tq;
      const bool kin = k0 + u < ks1 && kr < m;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const uint32_t r = r0 + mt * 8 + g;
        a[u][mt] = (kin && r < n) ? Ad[(int64_t)r * m + kr] : 0.0;
      }
#pragma unroll
      for (uint32_t t = 0; t < kNT; ++t) {
        const uint32_t col = n0 + t * 8 + g;
        b[u][t] = (kin && col < h) ? W1[(int64_t)kr * h + col] : 0.0;
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < G; ++u)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (uint32_t t = 0; t < kNT; ++t) dmma(acc[mt][t], a[u][mt], b[u][t]);
  }
  const double* b1 = s.b1;
  const double* W2 = s.W2;
  double* A1 = s.A1;
  for (uint32_t e = tid; e < NU * K; e += blockDim.x) {
    const uint32_t col = n0 + e / K;
    w2s[e] = col < h ? W2[(int64_t)col * K + e % K] : 0.0;
  }
  reduce_warps<MT, kRightWarps>(acc, red, [&](uint32_t row, uint32_t c, double z) {
    const uint32_t r = r0 + row, col = n0 + c;
    double a = 0.0;
    if (r < n && col < h) {
      a = fmax(z + b1[col], 0.0);
      A1[(int64_t)r * h + col] = a;
    }
    a1s[row * NU + c] = a;
  });
  __syncthreads();
  for (uint32_t e = tid; e < RT * K; e += blockDim.x) {  // partial logits of this CTA's units
    const uint32_t r = e / K, c = e % K;
    double t = 0.0;
    for (uint32_t u = 0; u < NU; ++u) t = fma(a1s[r * NU + u], w2s[u * K + c], t);
    lgp[e] = t;
  }
  cluster_barrier();  // every CTA's partial logits are visible
  double* lgs = ps;  // [RT][K] the logits (P overwrites them row by row below, after a barrier)
  for (uint32_t e = tid; e < RT * K; e += blockDim.x) {  // logits: the C partials in rank order, + b2
    double v[8];
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) v[q] = q < C ? ld_dsmem(lgp + e, q) : 0.0;  // all in flight
    double t = 0.0;
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) t += v[q];
    lgs[e] = t + __ldg(s.b2 + e % K);
  }
  __syncthreads();
  double pv = 0.0;
  const uint32_t pr = tid / K, pc = tid % K, prow = r0 + pr;
  if (tid < RT * K) {  // P = softmax - onehot for (row, class) = (pr, pc)
    double mx = -INFINITY, se = 0.0;
#pragma unroll
    for (int c = 0; c < K; ++c) mx = fmax(mx, lgs[pr * K + c]);
#pragma unroll
    for (int c = 0; c < K; ++c) se += exp(lgs[pr * K + c] - mx);
    const int y = prow < n ? (int)s.y[prow] : -1;
    pv = prow < n ? exp(lgs[tid] - mx) / se - ((int)pc == y ? 1.0 : 0.0) : 0.0;
    if (s.loss && prow < n && rank == 0 && (int)pc == y) s.loss[prow] = -((lgs[tid] - mx) - log(se));
  }
  __syncthreads();
  if (tid < RT * K) ps[tid] = pv;
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");  // done reading the others' partials
  __syncthreads();
  if (!s.loss) {
    double* dsm = red;  // [RT][NU] delta (the reduction buffer is free)
    for (uint32_t e = tid; e < RT * NU; e += blockDim.x) {  // delta = (P W2^T) * [A1 > 0], own units
      const uint32_t r = e / NU, u = e % NU, row = r0 + r, col = n0 + u;
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < K; ++c) t = fma(ps[r * K + c], w2s[u * K + c], t);
      t = a1s[e] > 0.0 ? t : 0.0;
      dsm[e] = t;
      if (row < n && col < h) s.D[(int64_t)row * h + col] = t;
    }
    __syncthreads();
    const uint32_t pw = h * K + h + K;
    double* part = s.part + (int64_t)blockIdx.x * pw;
    for (uint32_t e = tid; e < NU * K + NU + K; e += blockDim.x) {
      double t = 0.0;
      if (e < NU * K) {  // A1^T P over the tile's rows, own units
        const uint32_t u = e / K, c = e % K;
        if (n0 + u >= h) continue;
        for (uint32_t r = 0; r < RT; ++r) t = fma(a1s[r * NU + u], ps[r * K + c], t);
        part[(n0 + u) * K + c] = t;
      } else if (e < NU * K + NU) {  // delta sums, own units
        const uint32_t u = e - NU * K;
        if (n0 + u >= h) continue;
        for (uint32_t r = 0; r < RT; ++r) t += dsm[r * NU + u];
        part[h * K + n0 + u] = t;
      } else if (rank == 0) {  // P sums
        const uint32_t c = e - NU * K - NU;
        for (uint32_t r = 0; r < RT; ++r) t += ps[r * K + c];
        part[h * K + h + c] = t;
      }
    }
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // my partials may now go
}

// Per row (one warp, 8 rows per CTA): logits = A1 W2 + b2, P = softmax - onehot, delta = (P W2^T) *
// [A1 > 0]; then the CTA's sums over its rows of A1^T P, delta and P (its part of the W2 / b1 / b2
// gradients, summed over the CTAs by mlp_left in CTA order).
#ifndef MLP_TAIL_ROWS
#define MLP_TAIL_ROWS 8
#endif
constexpr uint32_t kTailRows = MLP_TAIL_ROWS;  // rows (one warp each) per tail CTA

template <int K>
__global__ void __launch_bounds__(kMlpThreads) mlp_tail_kernel(MlpStep s, uint32_t n) {
  extern __shared__ __align__(16) double sh[];
  pdl_wait();  // A1
  pdl_trigger();
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, h = (uint32_t)s.h;
  double* ps = sh;               // [8][K]
  double* as = ps + kTailRows * K;  // [rows][h]
  double* ds = as + kTailRows * h;  // [rows][h]
  const double* W2 = s.W2;       // [h x K], read through L1
  const uint32_t r0 = blockIdx.x * kTailRows, r = r0 + warp, nr = min(kTailRows, n - r0);
  if (r < n) {
    const double* a1 = s.A1 + (int64_t)r * h;
    double* arow = as + warp * h;
    double lg[K];
#pragma unroll
    for (int c = 0; c < K; ++c) lg[c] = 0.0;
#pragma unroll 4
    for (uint32_t j = lane; j < h; j += 32) {
      const double a = a1[j];
      arow[j] = a;
#pragma unroll
      for (int c = 0; c < K; ++c) lg[c] = fma(a, __ldg(W2 + j * K + c), lg[c]);
    }
    // lane c < K owns class c: its logit, exp and probability
    double mine = -INFINITY;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const double t = warp_sum(lg[c]);
      if ((int)lane == c) mine = t + __ldg(s.b2 + c);
    }
    double mx = mine;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const double e = (int)lane < K ? exp(mine - mx) : 0.0;
    const double se = warp_sum(e);
    const int y = (int)s.y[r];
    if (s.loss && (int)lane == y) s.loss[r] = -((mine - mx) - log(se));  // risk mode: -log softmax[y]
    const double pr = e / se - ((int)lane == y ? 1.0 : 0.0);
    if ((int)lane < K) {
      s.P[(int64_t)r * K + lane] = pr;
      ps[warp * K + lane] = pr;
    }
#pragma unroll
    for (int c = 0; c < K; ++c) lg[c] = __shfl_sync(0xffffffffu, pr, c);
    double* d = s.D + (int64_t)r * h;
    double* drow = ds + warp * h;
    __syncwarp();
#pragma unroll 4
    for (uint32_t j = lane; j < h; j += 32) {
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < K; ++c) t = fma(lg[c], __ldg(W2 + j * K + c), t);
      t = arow[j] > 0.0 ? t : 0.0;
      d[j] = t;
      drow[j] = t;
    }
  }
  if (s.loss) return;  // risk mode: no backward pass
  __syncthreads();
  const uint32_t pw = h * K + h + K;
  double* part = s.part + (int64_t)blockIdx.x * pw;
  for (uint32_t e = tid; e < pw; e += blockDim.x) {
    double t = 0.0;
    if (e < h * K) {
      const uint32_t j = e / K, c = e - j * K;
      for (uint32_t w = 0; w < nr; ++w) t = fma(as[w * h + j], ps[w * K + c], t);
    } else if (e < h * K + h) {
      const uint32_t j = e - h * K;
      for (uint32_t w = 0; w < nr; ++w) t += ds[w * h + j];
    } else {
      const uint32_t c = e - h * K - h;
      for (uint32_t w = 0; w < nr; ++w) t += ps[w * K + c];
    }
    part[e] = t;
  }
}

// G = A_b^T . delta for 8*MT columns x 40 hidden units (K = the batch's rows); W1 -= s G.  The last
// n_upd CTAs sum the tail CTAs' parts in CTA order and update W2, b1, b2.
template <int MT>
__global__ void __launch_bounds__(kMlpThreads) mlp_left_kernel(MlpStep s, uint32_t n, uint32_t n_gemm,
                                                               uint32_t n_tail) {
  extern __shared__ __align__(16) double red[];
  pdl_wait();  // delta and the tail's parts
  pdl_trigger();
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const uint32_t m = (uint32_t)s.m, h = (uint32_t)s.h;
  if (blockIdx.x >= n_gemm) {
    const uint32_t k = (uint32_t)s.k, pw = h * k + h + k;
    const uint32_t e = (blockIdx.x - n_gemm) * blockDim.x + tid;
    if (e >= pw) return;
    double t = 0.0;
    const double* pe = s.part + e;
    uint32_t c = 0;
    for (; c + 8 <= n_tail; c += 8) {  // 8 loads in flight, summed in CTA order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = pe[(int64_t)(c + u) * pw];
#pragma unroll
      for (int u = 0; u < 8; ++u) t += v[u];
    }
    for (; c < n_tail; ++c) t += pe[(int64_t)c * pw];
    if (s.grad) s.grad[(int64_t)m * h + e] = t;
    else if (e < h * k) s.W2[e] -= s.step * t;
    else if (e < h * k + h) s.b1[e - h * k] -= s.step * t;
    else s.b2[e - h * k - h] -= s.step * t;
    return;
  }
  const uint32_t ncx = (m + 8 * MT - 1) / (8 * MT);
  const uint32_t c0 = (blockIdx.x % ncx) * (8 * MT), n0 = (blockIdx.x / ncx) * (8 * kNT);
  double acc[MT][kNT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (uint32_t t = 0; t < kNT; ++t) acc[mt][t][0] = acc[mt][t][1] = 0.0;
  const uint32_t ksteps = (n + 3) >> 2, ks0 = warp * ksteps / 8, ks1 = (warp + 1) * ksteps / 8;
  const double* Ad = s.Ad;
  const double* D = s.D;
  constexpr uint32_t G = 4;
  for (uint32_t k0 = ks0; k0 < ks1; k0 += G) {
    double a[G][MT], b[G][kNT];
#pragma unroll
    for (uint32_t u = 0; u < G; ++u) {
      const uint32_t r = (k0 + u) * 4 + tq;
      const bool kin = k0 + u < ks1 && r < n;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const uint32_t c = c0 + mt * 8 + g;
        a[u][mt] = (kin && c < m) ? Ad[(int64_t)r * m + c] : 0.0;
      }
#pragma unroll
      for (uint32_t t = 0; t < kNT; ++t) {
        const uint32_t col = n0 + t * 8 + g;
        b[u][t] = (kin && col < h) ? D[(int64_t)r * h + col] : 0.0;
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < G; ++u)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (uint32_t t = 0; t < kNT; ++t) dmma(acc[mt][t], a[u][mt], b[u][t]);
  }
  double* W1 = s.W1;
  double* grad = s.grad;
  const double st = s.step;
  reduce_warps<MT, 8>(acc, red, [&](uint32_t row, uint32_t cc, double gsum) {
    const uint32_t c = c0 + row, col = n0 + cc;
    if (c < m && col < h) {
      if (grad) grad[(int64_t)c * h + col] = gsum;
      else W1[(int64_t)c * h + col] -= st * gsum;
    }
  });
}

#ifndef MLP_RIGHT_MT
#define MLP_RIGHT_MT 2
#endif
constexpr int kRightMT = MLP_RIGHT_MT;
#ifndef MLP_LEFT_MT
#define MLP_LEFT_MT 2
#endif
constexpr int kLeftMT = MLP_LEFT_MT;

}  // namespace toc

namespace {

struct MlpScratch {
  int64_t a1, p, d, ad, part, total;  // offsets in doubles
};

MlpScratch mlp_scratch_layout(int32_t nmax, int32_t m, int32_t h, int32_t k) {
  MlpScratch L;
  int64_t o = 0;
  L.a1 = o;
  o += (int64_t)nmax * h;
  L.p = o;
  o += (int64_t)nmax * k;
  L.d = o;
  o += (int64_t)nmax * h;
  o = (o + 1) & ~1ll;
  L.ad = o;  // two decode buffers
  o += 2 * (((int64_t)nmax * m + 1) & ~1ll);
  L.part = o;
  o += (int64_t)((nmax + toc::kTailRows - 1) / toc::kTailRows) * (h * k + h + k);
  L.total = o;
  return L;
}

}  // namespace

namespace {
int32_t g_mlp_mask = 15;  // diagnostic: which of decode / right / tail / left launch (bits 0..3)
int32_t g_mlp_decode_ctas = 8;  // decode CTAs per SM (tuning knob, toc_mlp_set_decode_ctas)
bool g_mlp_fuse = true;  // right + tail as one cluster kernel (mlp_right_tail_kernel) where it applies
bool g_mlp_graph = true;  // replay the epoch as one CUDA graph (built on the first call)

// What a captured epoch depends on: every argument but the stream, plus a hash of the host arrays.
struct MlpGraphKey {
  const void *cache, *off, *rb, *nr;
  int64_t n_blocks;
  int32_t m, h, k;
  const void *labels, *W1, *b1, *W2, *b2;
  double lr;
  int32_t dense;
  const void* scratch;
  int32_t mask;
  uint64_t hash;
  bool operator==(const MlpGraphKey& o) const {
    return cache == o.cache && off == o.off && rb == o.rb && nr == o.nr && n_blocks == o.n_blocks && m == o.m &&
           h == o.h && k == o.k && labels == o.labels && W1 == o.W1 && b1 == o.b1 && W2 == o.W2 && b2 == o.b2 &&
           lr == o.lr && dense == o.dense && scratch == o.scratch && mask == o.mask && hash == o.hash;
  }
};
MlpGraphKey g_mlp_key{};
cudaGraphExec_t g_mlp_exec = nullptr;
}  // namespace

namespace {
bool g_mlp_pdl = true;  // launch the step kernels with programmatic dependent launch

// One launch, with programmatic stream serialization when enabled (the kernel's pdl_wait then
// overlaps its launch -- and the decode's chain walks -- with the predecessor's tail).
template <typename... KArgs, typename... Args>
void pdl_launch(void (*fn)(KArgs...), dim3 grid, uint32_t block, int smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_mlp_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, fn, static_cast<KArgs>(args)...);
}

// The same with a (1, cy, 1) thread-block cluster.
template <typename... KArgs, typename... Args>
void pdl_launch_cluster(void (*fn)(KArgs...), dim3 grid, uint32_t cy, uint32_t block, int smem, cudaStream_t st,
                        Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = cy;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_mlp_pdl ? 2 : 1;
  cudaLaunchKernelEx(&cfg, fn, static_cast<KArgs>(args)...);
}

constexpr int kFusedSmem = 8 * ((int)toc::kRightWarps * toc::kRightMT * toc::kNT * 64 +
                                (8 * toc::kRightMT) * (8 * toc::kNT) + 2 * (8 * toc::kRightMT) * 10 +
                                (8 * toc::kNT) * 10);

// Dynamic shared memory of the three GEMM-shaped kernels (set once per process).
int mlp_attrs(int32_t h, int32_t k) {
  const int smem_right = 8 * (int)toc::kRightWarps * toc::kRightMT * toc::kNT * 64;
  const int smem_left = 8 * 8 * toc::kLeftMT * toc::kNT * 64;
  const int smem_tail = 8 * (int)toc::kTailRows * (k + 2 * h);
  if (smem_tail > 200 * 1024) return TOC_E_ARG;
  if (cudaFuncSetAttribute(toc::mlp_right_kernel<toc::kRightMT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem_right) != cudaSuccess ||
      cudaFuncSetAttribute(toc::mlp_right_tail_kernel<toc::kRightMT, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kFusedSmem) != cudaSuccess ||
      cudaFuncSetAttribute(toc::mlp_tail_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tail) !=
          cudaSuccess ||
      cudaFuncSetAttribute(toc::mlp_left_kernel<toc::kLeftMT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem_left) != cudaSuccess)
    return TOC_E_CUDA;
  return TOC_OK;
}

// Launches of steps [b0, b1) (decode buffers zeroed first when b0 == 0; a later b0 continues the
// parity of the preceding call).  grad: gradient-only mode for a single step (see MlpStep).
int mlp_enqueue(const uint8_t* d_arena, const int64_t* h_block_off, const uint8_t* d_cache,
                const int64_t* h_cache_off, const int64_t* h_row_base, const int32_t* h_n_rows, int64_t b0, int64_t b1,
                int32_t nmax, int32_t m, int32_t h, int32_t k, const double* d_labels, double* d_W1, double* d_b1,
                double* d_W2, double* d_b2, double lr, int32_t dense, void* d_scratch, double* d_grad, double* d_loss,
                cudaStream_t st) {
    const MlpScratch SL = mlp_scratch_layout(nmax, m, h, k);
    const int smem_right = 8 * (int)toc::kRightWarps * toc::kRightMT * toc::kNT * 64;
    const int smem_left = 8 * 8 * toc::kLeftMT * toc::kNT * 64;
    const int smem_tail = 8 * (int)toc::kTailRows * (k + 2 * h);
    double* base = reinterpret_cast<double*>(d_scratch);
    const int64_t ad_elems = ((int64_t)nmax * m + 1) & ~1ll;
    double* adbuf[2] = {base + SL.ad, base + SL.ad + ad_elems};
    if (b0 == 0 && cudaMemsetAsync(adbuf[0], 0, 8 * 2 * ad_elems, st) != cudaSuccess) return TOC_E_CUDA;
    toc::MlpStep s{};
    s.m = m;
    s.h = h;
    s.k = k;
    s.W1 = d_W1;
    s.b1 = d_b1;
    s.W2 = d_W2;
    s.b2 = d_b2;
    s.A1 = base + SL.a1;
    s.P = base + SL.p;
    s.D = base + SL.d;
    s.part = base + SL.part;
    s.az_elems = dense ? 0 : ad_elems;
    int sms = 148;
    {
      int dev = 0;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const uint32_t ncb = (uint32_t)((h + 8 * toc::kNT - 1) / (8 * toc::kNT));
    const uint32_t n_gemm_left = (uint32_t)((m + 8 * toc::kLeftMT - 1) / (8 * toc::kLeftMT)) * ncb;
    const uint32_t pw = (uint32_t)(h * k + h + k), n_upd = (pw + toc::kMlpThreads - 1) / toc::kMlpThreads;
    s.grad = d_grad;
    for (int64_t b = b0; b < b1; ++b) {
      const uint32_t n = (uint32_t)h_n_rows[b];
      if (n == 0) continue;
      s.entry = d_cache + h_cache_off[b];
      s.blk = d_arena + h_block_off[b];
      s.y = d_labels + h_row_base[b];
      s.loss = d_loss ? d_loss + h_row_base[b] : nullptr;
      s.step = lr / (double)n;
      s.Ad = adbuf[b & 1];
      s.Az = adbuf[(b + 1) & 1];
      const uint32_t row_tiles = (n + 8 * toc::kRightMT - 1) / (8 * toc::kRightMT);
      const bool fused = g_mlp_fuse && k == 10 && ncb <= 8;  // parts: one per row tile
      const uint32_t n_tail = fused ? row_tiles : (n + toc::kTailRows - 1) / toc::kTailRows;
      if (g_mlp_mask & 1)
        pdl_launch(toc::mlp_decode_kernel, dim3((unsigned)(g_mlp_decode_ctas * sms)), toc::kMlpThreads, 0, st, s, n);
      if ((g_mlp_mask & 2) && fused)
        pdl_launch_cluster(toc::mlp_right_tail_kernel<toc::kRightMT, 10>, dim3(row_tiles, ncb), ncb,
                           32 * toc::kRightWarps, kFusedSmem, st, s, n);
      if ((g_mlp_mask & 2) && !fused)
        pdl_launch(toc::mlp_right_kernel<toc::kRightMT>, dim3(row_tiles, ncb), 32 * toc::kRightWarps, smem_right, st,
                   s, n);
      if ((g_mlp_mask & 4) && !fused)
        pdl_launch(toc::mlp_tail_kernel<10>, dim3(n_tail), 32 * toc::kTailRows, smem_tail, st, s, n);
      if ((g_mlp_mask & 8) && !d_loss)
        pdl_launch(toc::mlp_left_kernel<toc::kLeftMT>, dim3(n_gemm_left + n_upd), toc::kMlpThreads, smem_left, st, s, n,
                   n_gemm_left, n_tail);
    }
    return cudaGetLastError() == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}
}  // namespace

extern "C" int toc_mlp_set_fused(int32_t on) {
  g_mlp_fuse = on != 0;
  if (g_mlp_exec) cudaGraphExecDestroy(g_mlp_exec);  // the captured epoch depends on it
  g_mlp_exec = nullptr;
  return TOC_OK;
}

extern "C" int toc_mlp_set_decode_ctas(int32_t per_sm) {
  if (per_sm < 1 || per_sm > 32) return TOC_E_ARG;
  g_mlp_decode_ctas = per_sm;
  if (g_mlp_exec) cudaGraphExecDestroy(g_mlp_exec);  // the captured epoch depends on it
  g_mlp_exec = nullptr;
  return TOC_OK;
}

extern "C" int toc_mlp_set_kernels(int32_t mask) {
  g_mlp_mask = mask & 15;
  return TOC_OK;
}

extern "C" int toc_mlp_set_pdl(int32_t on) {
  g_mlp_pdl = on != 0;
  if (g_mlp_exec) cudaGraphExecDestroy(g_mlp_exec);  // the captured epoch depends on it
  g_mlp_exec = nullptr;
  return TOC_OK;
}

extern "C" int toc_mlp_set_graph(int32_t on) {
  g_mlp_graph = on != 0;
  return TOC_OK;
}

extern "C" int toc_mlp_scratch(int32_t max_rows, int32_t m, int32_t h, int32_t k, int64_t* bytes) {
  if (max_rows < 0 || m < 1 || h < 1 || k < 1 || !bytes) return TOC_E_ARG;
  *bytes = 8 * mlp_scratch_layout(max_rows, m, h, k).total;
  return TOC_OK;
}

// One epoch: for each batch in order, the four kernels of the step.  h_cache_off / h_row_base /
// h_n_rows are host copies (the launch loop reads them); d_labels holds class ids as f64.  dense:
// every row has all m columns, so each decode overwrites the whole buffer and none is zeroed.
extern "C" int toc_mlp_epoch(const uint8_t* d_arena, const int64_t* h_block_off, const uint8_t* d_cache,
                             const int64_t* h_cache_off, const int64_t* h_row_base, const int32_t* h_n_rows,
                             int64_t n_blocks, int32_t m, int32_t h, int32_t k, const double* d_labels, double* d_W1,
                             double* d_b1, double* d_W2, double* d_b2, double lr, int32_t dense, void* d_scratch,
                             int64_t scratch_bytes, void* stream) {
  if (!d_arena || !h_block_off || !d_cache || !h_cache_off || !h_row_base || !h_n_rows || n_blocks < 0 || m < 1 ||
      h < 1 || k < 1 ||
      k > (int32_t)toc::kKMax || !d_labels || !d_W1 || !d_b1 || !d_W2 || !d_b2 || !d_scratch)
    return TOC_E_ARG;
  if (k != 10) return TOC_E_ARG;  // the tail kernel is instantiated for config 5's 10 classes
  int32_t nmax = 0;
  for (int64_t b = 0; b < n_blocks; ++b) nmax = h_n_rows[b] > nmax ? h_n_rows[b] : nmax;
  if (scratch_bytes < 8 * mlp_scratch_layout(nmax, m, h, k).total) return TOC_E_ARG;
  if (const int rc = mlp_attrs(h, k)) return rc;
  // the whole epoch's launches; enqueued directly, or captured once into a CUDA graph and replayed
  auto enqueue = [&](cudaStream_t st) -> int {
    return mlp_enqueue(d_arena, h_block_off, d_cache, h_cache_off, h_row_base, h_n_rows, 0, n_blocks, nmax, m, h, k,
                       d_labels, d_W1, d_b1, d_W2, d_b2, lr, dense, d_scratch, nullptr, nullptr, st);
  };
  if (!g_mlp_graph) return enqueue((cudaStream_t)stream);
  MlpGraphKey key{d_cache, h_cache_off, h_row_base, h_n_rows, n_blocks, m, h, k, d_labels, d_W1, d_b1, d_W2, d_b2,
                  lr, dense, d_scratch, g_mlp_mask, 0};
  key.hash = (uint64_t)(uintptr_t)d_arena;
  for (int64_t b = 0; b < n_blocks; ++b)
    key.hash = key.hash * 1099511628211ull ^ ((uint64_t)h_cache_off[b] * 31 + (uint64_t)h_row_base[b] * 7 +
                                               (uint64_t)h_n_rows[b] + (uint64_t)h_block_off[b] * 131);
  if (!(g_mlp_exec && key == g_mlp_key)) {
    if (g_mlp_exec) cudaGraphExecDestroy(g_mlp_exec);
    g_mlp_exec = nullptr;
    cudaStream_t cs;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return TOC_E_CUDA;
    cudaGraph_t graph = nullptr;
    int rc = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess ? TOC_OK : TOC_E_CUDA;
    if (rc == TOC_OK) rc = enqueue(cs);
    if (cudaStreamEndCapture(cs, &graph) != cudaSuccess && rc == TOC_OK) rc = TOC_E_CUDA;
    cudaStreamDestroy(cs);
    if (rc == TOC_OK && cudaGraphInstantiate(&g_mlp_exec, graph, 0) != cudaSuccess) rc = TOC_E_CUDA;
    if (graph) cudaGraphDestroy(graph);
    if (rc != TOC_OK) {
      g_mlp_exec = nullptr;
      return rc;
    }
    g_mlp_key = key;
  }
  return cudaGraphLaunch(g_mlp_exec, (cudaStream_t)stream) == cudaSuccess ? TOC_OK : TOC_E_CUDA;
}

extern "C" int toc_mlp_step_grad(const uint8_t* d_arena, const int64_t* h_block_off, const uint8_t* d_cache,
                                 const int64_t* h_cache_off, const int64_t* h_row_base, const int32_t* h_n_rows,
                                 int64_t n_blocks, int64_t step, int32_t m, int32_t h, int32_t k,
                                 const double* d_labels, const double* d_W1, const double* d_b1, const double* d_W2,
                                 const double* d_b2, int32_t dense, double* d_grad, void* d_scratch,
                                 int64_t scratch_bytes, void* stream) {
  if (!d_arena || !h_block_off || !d_cache || !h_cache_off || !h_row_base || !h_n_rows || step < 0 ||
      step >= n_blocks || m < 1 || h < 1 ||
      k != 10 || !d_labels || !d_W1 || !d_b1 || !d_W2 || !d_b2 || !d_grad || !d_scratch)
    return TOC_E_ARG;
  int32_t nmax = 0;
  for (int64_t b = 0; b < n_blocks; ++b) nmax = h_n_rows[b] > nmax ? h_n_rows[b] : nmax;
  if (scratch_bytes < 8 * mlp_scratch_layout(nmax, m, h, k).total) return TOC_E_ARG;
  if (const int rc = mlp_attrs(h, k)) return rc;
  if (h_n_rows[step] == 0)
    return cudaMemsetAsync(d_grad, 0, 8 * ((size_t)m * h + (size_t)h * k + h + k), (cudaStream_t)stream) ==
                   cudaSuccess
               ? TOC_OK
               : TOC_E_CUDA;
  return mlp_enqueue(d_arena, h_block_off, d_cache, h_cache_off, h_row_base, h_n_rows, step, step + 1, nmax, m, h, k,
                     d_labels, const_cast<double*>(d_W1), const_cast<double*>(d_b1), const_cast<double*>(d_W2),
                     const_cast<double*>(d_b2), 0.0, dense, d_scratch, d_grad, nullptr, (cudaStream_t)stream);
}

// The per-row cross-entropy of the current parameters over every batch (forward only: decode, A.W1
// on the tensor cores with the ReLU epilogue, logits and -log softmax[y]); d_loss [rows].
extern "C" int toc_mlp_risk(const uint8_t* d_arena, const int64_t* h_block_off, const uint8_t* d_cache,
                            const int64_t* h_cache_off, const int64_t* h_row_base, const int32_t* h_n_rows,
                            int64_t n_blocks, int32_t m, int32_t h, int32_t k, const double* d_labels,
                            const double* d_W1, const double* d_b1, const double* d_W2, const double* d_b2,
                            int32_t dense, double* d_loss, void* d_scratch, int64_t scratch_bytes, void* stream) {
  if (!d_arena || !h_block_off || !d_cache || !h_cache_off || !h_row_base || !h_n_rows || n_blocks < 0 || m < 1 ||
      h < 1 || k != 10 || !d_labels || !d_W1 || !d_b1 || !d_W2 || !d_b2 || !d_loss || !d_scratch)
    return TOC_E_ARG;
  int32_t nmax = 0;
  for (int64_t b = 0; b < n_blocks; ++b) nmax = h_n_rows[b] > nmax ? h_n_rows[b] : nmax;
  if (scratch_bytes < 8 * mlp_scratch_layout(nmax, m, h, k).total) return TOC_E_ARG;
  if (const int rc = mlp_attrs(h, k)) return rc;
  return mlp_enqueue(d_arena, h_block_off, d_cache, h_cache_off, h_row_base, h_n_rows, 0, n_blocks, nmax, m, h, k,
                     d_labels, const_cast<double*>(d_W1), const_cast<double*>(d_b1), const_cast<double*>(d_W2),
                     const_cast<double*>(d_b2), 0.0, dense, d_scratch, nullptr, d_loss, (cudaStream_t)stream);
}
