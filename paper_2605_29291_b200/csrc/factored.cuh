// factored.cuh -- the sparse factored path (BASELINE config 3): Q_i = R_i^T R_i.
//
// The U-cache of the dense path becomes a W-cache: W = R x for the stacked R
// (65 x 1e5 rows at C3, 52 MB), from which
//   g_i(x)      = 1/2 |W_i|^2 + c_i . x + d_i                (x'Q_i x = |R_i x|^2)
//   grad_x Phi  = sum_i w_i (R_i^T W_i + c_i) + A^T mu       (w_0 = 1, w_i = lam_i)
// and the linear block A x <= b enters as orthant constraints with Q = 0
// (g = A x - b, multipliers mu = lam[mq:]).
//
// Kernels (host-launched at a stop of the persistent kernel -- a request in
// the solver state, like an exchange point -- because these latency-bound
// gathers want more resident warps and registers than the persistent CTAs have):
//   gradient     fac_grad_kernel, one launch per row phase of R^T: warps in
//                two roles -- a warp per 32-column slice of R^T (lane = column,
//                gather w_blk(r) W[r] in row order) and of A^T, while every
//                4th warp streams the block-weighted c_i part;
//                fac_grad_fin_kernel combines them into grad_x Phi and, in a
//                fused yx trial, takes the primal step x_new = clip(x_k -
//                tau grad) with the D_p / <grad, dx> partials
//   row pass     fac_row_kernel: warps in two roles -- W = R x (+ |W_i|^2
//                partials per 128-row chunk) and A x - b (lane = row), and the
//                c_i . x chunk partials -- so the pure HBM stream over C runs
//                beside the gather-bound sparse rows
// The sparse operands are sliced ELLPACK (rapdb_dev.cuh Sell): coalesced
// streams with no staging, each row / column summed in stored order without
// FMA.  The passes are bound by the 32-byte L2 sectors their 8-byte gathers
// move (~65 M per pass at C3; tools/gather_probe.cu), not by HBM bytes: the
// dense C streams ride along in the same launches, which saves a pass and a
// stop.  Per yx trial ~2.7 GB from HBM (R and R^T 780 MB each, C 2 x 520 MB,
// A, A^T), ~7.6 GB of L2 -> SM sectors, and one stop of the persistent
// kernel.  Every reduction has a fixed order.
#pragma once
#include "solver_kernel.cuh"

namespace rapdb {

__device__ __forceinline__ long long gwarp() { return (long long)blockIdx.x * kWarps + (threadIdx.x >> 5); }
__device__ __forceinline__ long long nwarps() { return (long long)gridDim.x * kWarps; }

constexpr int kWChunk = 128;    // rows of W per |W_i|^2 partial (inside one block)
constexpr int kCxCols = 1024;   // columns per c_i . x partial
// tunables of the standalone kernels (A/B builds: tools/c3_variants.sh)
#ifndef RAPDB_ROWU
#define RAPDB_ROWU 5
#endif
#ifndef RAPDB_GXU
#define RAPDB_GXU 4
#endif
#ifndef RAPDB_ROWCTAS
#define RAPDB_ROWCTAS 4
#endif
#ifndef RAPDB_GRADCTAS
#define RAPDB_GRADCTAS 4
#endif
constexpr int kRowU = RAPDB_ROWU;       // gathers in flight per lane in the row pass (C3: 10 entries per row of R)

// One slice of a Sell operand against a gathered vector: lane l folds the
// entries of slot 32 * slice + l in stored order without FMA -- the operation
// order of scipy's csr_matvec, so W = R x and the R^T / A^T column sums match
// the factored restatement bit for bit -- starting from s.  The t-th loads of
// val / idx are one coalesced access per warp (no shared-memory staging), U
// entries per lane at a time.  The passes are bound by their gathers: every
// 8-byte gather is one L1 wavefront (a 128-byte line lookup per lane) and
// moves a 32-byte sector from L2 to the SM; tools/gather_probe.cu puts the
// ceiling at ~250-270 G gathers/s on a B200 (~1 wavefront per cycle and SM,
// ~9-10 TB/s of sectors with the index stream), whatever the width,
// instruction or occupancy.  At C3 the row pass issues ~83 M wavefronts, 67.5 M
// of them gathers (the rest: the R, C and x streams), in 355-360 us: 0.92 per
// cycle and SM, 3.65 GB of sectors at 10.3 TB/s; the gradient 2 x 205 us.  Every
// variant tried lands there or worse (U = 2..10 at 2..8 CTAs per SM, double-
// buffered loads with TMA L2 prefetch, TMA-fed shared-memory rings with 7 / 14
// gather warps, dedicated c_i . x CTAs: profiles/r02j_c3_variant_sweep.log),
// so the plain form stays: U = 4..5, 4 CTAs per SM, a contiguous run of slices
// per warp.
constexpr int kRtTagShift = 23;
constexpr int kRtRowMask = (1 << kRtTagShift) - 1;

// TAG: entry (r | blk << 23, v) of R^T adds v * (wq[blk] * W[r]).  A zero
// weight adds +-0 to a sum that starts at +0 -- a no-op -- so its gather is
// skipped: the pass costs the active blocks.
template <int U, bool TAG>
__device__ __forceinline__ double sell_dot(const Sell& M, long long slice, const double* x, const double* wq,
                                           double s, uint64_t ef) {
  const int lane = threadIdx.x & 31;
  const long long base = __ldg(M.sp + slice);
  const int width = (int)((__ldg(M.sp + slice + 1) - base) >> 5);
  const int len = __ldg(M.len + slice * 32 + lane);
  const int* ip = M.idx + base + lane;
  const double* vp = M.val + base + lane;
  for (int t0 = 0; t0 < width; t0 += U) {
    int c[U];
    double v[U], xv[U], wt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      wt[u] = 0.0;
      if (t0 + u < len) {
        c[u] = ld_stream(ip + (long long)(t0 + u) * 32, ef);
        v[u] = ld_stream(vp + (long long)(t0 + u) * 32, ef);
        wt[u] = TAG ? wq[c[u] >> kRtTagShift] : 1.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (wt[u] != 0.0) xv[u] = ldcg(x + (TAG ? (c[u] & kRtRowMask) : c[u]));
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (wt[u] != 0.0) s = __dadd_rn(s, __dmul_rn(v[u], TAG ? __dmul_rn(wt[u], xv[u]) : xv[u]));
  }
  return s;
}

// the contiguous share [lo, hi) of `items` items for member `me` of `n`
__device__ __forceinline__ void my_range(long long items, long long me, long long n, long long& lo, long long& hi) {
  lo = items * me / n;
  hi = items * (me + 1) / n;
}

// rows [r0, r1) of W chunk c (wch[i] = first chunk of local block i)
__device__ __forceinline__ void wchunk_rows(const DevProblem& P, long long c, long long& r0, long long& r1,
                                            long long& rb) {
  int lo = 0, hi = P.fnb;                 // local block of chunk c: wch[lo] <= c < wch[lo+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(P.wch + mid) <= c) lo = mid; else hi = mid;
  }
  rb = __ldg(P.rblk + lo);                // first row of the block
  r0 = rb + (c - __ldg(P.wch + lo)) * kWChunk;
  r1 = min(r0 + kWChunk, __ldg(P.rblk + lo + 1));
}

// c_i . x over columns [ch*1024, +1024): lane-strided fma chain, butterfly
// (the partial pcx[i * nchx + ch]).  x is read through L1 (ld.global.ca): a
// warp walks the blocks i of ONE column chunk back to back (fac_row_kernel), so
// the 8 KB chunk of x is fetched from L2 once instead of once per block --
// 520 MB of L2 -> SM sectors per pass at C3, on the path the gathers saturate.
__device__ __forceinline__ double cx_item(const DevProblem& P, const double* x, long long i, long long ch) {
  const int lane = threadIdx.x & 31;
  const long long n = P.n;
  const long long j0 = ch * kCxCols, j1 = min(j0 + kCxCols, n);
  const double* ci = P.q + i * n;
  double s = 0.0;
  long long j = j0 + lane;
  for (; j + 7 * 32 < j1; j += 8 * 32) {   // 16 loads in flight, the same fma chain
    double c[8], xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { c[k] = __ldcs(ci + j + 32 * k); xv[k] = __ldca(x + j + 32 * k); }
#pragma unroll
    for (int k = 0; k < 8; ++k) s = fma(c[k], xv[k], s);
  }
  for (; j < j1; j += 32) s = fma(__ldcs(ci + j), __ldca(x + j), s);
  return warp_sum(s);
}

// ---------------------------------------------------------------- gradient
__device__ __forceinline__ void fac_wq(const DevProblem& P, const double* lam, double* wq, int nthreads) {
  for (int i = threadIdx.x; i < P.fnb; i += nthreads) {
    const int gi = P.fb0 + i;             // global block id (0 = objective)
    wq[i] = gi == 0 ? 1.0 : ldcg(lam + (gi - 1));
  }
}

// Wl[r] = w_blk(r) W[r] (untagged R^T only: more than 2^23 rows or 256 blocks)
__device__ __forceinline__ void fac_wl(const DevProblem& P, const Work& w, const double* Wpar, const double* wq) {
  const uint64_t ef = evict_first_policy();
  const uint64_t el = sym::evict_last_policy();
  for (long long r = gtid(); r < P.nr; r += gstride())
    st_keep(w.wl + r, wq[ld_stream(P.rmat + r, ef)] * ldcg(Wpar + r), el);
}

// grad_x Phi column j = (acc + s) + t, every path the same bits:
//   acc  sum_i w_i c_ij over the blocks in order, skipping zero weights
//        (one thread per column: a plain HBM stream over C), in phase p the
//        blocks [fnb p / nph, fnb (p + 1) / nph) continuing the chain;
//   s    the R^T gather sum_r v (w_blk(r) W[r]), the column's entries folded
//        one by one in row order across the row phases (sell_dot<., true>);
//   t    A^T mu the same way (sell_dot<., false>).
// The gather of phase p reads only rows [rt_b[p], rt_b[p+1]) of the W-cache:
// phases run one after the other over the whole grid (separate launches), so
// the gathered slice stays L2-resident.
constexpr int kGxU = RAPDB_GXU;       // gathers in flight per lane in the transposed passes
// resident CTAs per SM of the standalone kernels: the latency chain of a slice
// (offsets -> (idx, val) -> gathers) is hidden by warps, not by unrolling --
// 4 CTAs (32 warps, 64 registers) beat both 2-3 CTAs with U = 8..10 and 6-8
// CTAs whose 32-40 registers spill (profiles/r02j_c3_variant_sweep.log)
constexpr int kRowCtas = RAPDB_ROWCTAS, kGradCtas = RAPDB_GRADCTAS;

// U (symmetric stacks only, else null): the W-cache, whose block i is u_i =
// Q_i x -- the term becomes w_i (u_ij + c_ij), the reference's own grouping
// (problem.py:205-214: out + lam_i * (Q_i x + q_i)).
__device__ __forceinline__ double fac_c_acc(const DevProblem& P, const double* wq, const double* U, long long j,
                                            int i0, int i1, double acc, uint64_t ef) {
  const long long n = P.n;
  int i = i0;
  for (; i + 8 <= i1; i += 8) {           // 8 (16) independent loads in flight
    double c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = ld_stream(P.q + (long long)(i + k) * n + j, ef);
    if (U) {
#pragma unroll
      for (int k = 0; k < 8; ++k) c[k] = ldcg(U + (long long)(i + k) * n + j) + c[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double l = wq[i + k];
      acc = (l != 0.0) ? acc + l * c[k] : acc;
    }
  }
  for (; i < i1; ++i) {
    const double l = wq[i];
    double c = ld_stream(P.q + (long long)i * n + j, ef);
    if (U) c = ldcg(U + (long long)i * n + j) + c;
    acc = (l != 0.0) ? acc + l * c : acc;
  }
  return acc;
}

// gather item `it` of phase ph for the warp: the slices of R^T's phase, then
// (phase 0 only) the slices of A^T.  s continues in out[], t goes to aux2[].
template <bool TAG>
__device__ __forceinline__ void fac_gather_item(const DevProblem& P, const Work& w, const double* Wsrc,
                                                const double* wq, const double* lam, double* out, int ph,
                                                long long it, uint64_t ef) {
  const int lane = threadIdx.x & 31;
  const Sell& M = P.sell[kSellRt + ph];
  const long long nrt = M.nslots >> 5;
  if (it < nrt) {
    const int j = __ldg(M.map + it * 32 + lane);
    double s = (ph > 0 && j >= 0) ? ldcg(out + j) : 0.0;
    s = sell_dot<kGxU, TAG>(M, it, Wsrc, wq, s, ef);
    if (j >= 0) out[j] = s;
  } else {
    const long long sl = it - nrt;
    const Sell& T = P.sell[kSellAt];
    const int j = __ldg(T.map + sl * 32 + lane);
    const double t = sell_dot<kGxU, false>(T, sl, lam + P.mq + P.l0, nullptr, 0.0, ef);
    if (j >= 0) w.aux2[j] = t;
  }
}
// ---------------------------------------------------------------- row pass
// |W_i|^2 over chunk c: lane r0 + lane, + 32, ... with fma, then the butterfly
// (formed on the fly by the row pass: 4 slices of 32 rows per chunk); for a
// symmetric stack (P.sym: the blocks are the Q_i) the chunk's part of x . Q_i x
__device__ __forceinline__ void fac_chunk(const DevProblem& P, const Work& w, const double* x, double* W,
                                          long long c, uint64_t ef, uint64_t el) {
  const int lane = threadIdx.x & 31;
  long long r0, r1, rb;
  wchunk_rows(P, c, r0, r1, rb);
  double s2 = 0.0;
  for (int g = 0; g < kWChunk / 32; ++g) {
    const long long row = r0 + 32 * g + lane;
    if (r0 + 32 * g >= r1) break;
    const double v = sell_dot<kRowU, false>(P.sell[kSellR], c * (kWChunk / 32) + g, x, nullptr, 0.0, ef);
    if (row < r1) {
      st_keep(W + row, v, el);
      s2 = P.sym ? fma(ldcg(x + (row - rb)), v, s2) : fma(v, v, s2);   // x . (Q_i x), or |R_i x|^2
    }
  }
  s2 = warp_sum(s2);
  if (lane == 0) w.pw2[c] = s2;
}

// 32 rows of A x - b into the linear part of gval
__device__ __forceinline__ void fac_arows(const DevProblem& P, const double* x, double* gv_lin, long long sl,
                                          uint64_t ef) {
  const long long j = sl * 32 + (threadIdx.x & 31);
  const double v = sell_dot<kRowU, false>(P.sell[kSellA], sl, x, nullptr, 0.0, ef);
  if (j < P.Lloc) gv_lin[j] = v - __ldg(P.b + j);
}

// g_i (i = 0..mq, 0 = f) at parity par from the chunk partials: one CTA per
// local block, warp q sums the q-th eighth of the block's W chunks and of its
// c_i . x chunks (lane-strided, butterfly), the CTA adds the 8 warps in
// order; a sharded rank writes 0 for the entries it does not own (the
// all-reduce of g is then exact: disjoint supports)
__device__ void g_factored(const KArgs& K, int par) {
  const DevProblem& P = K.P;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  double* gv = K.w.gval + (long long)par * (P.m + 1);
  __shared__ double gred[2 * kWarps];
  for (long long i = blockIdx.x; i < P.fnb; i += gridDim.x) {
    const long long c0 = __ldg(P.wch + i), c1 = __ldg(P.wch + i + 1);
    const long long nw = c1 - c0, per = (nw + kWarps - 1) / kWarps;
    const long long w0 = c0 + wp * per, w1 = min(w0 + per, c1);
    const long long px = (P.nchx + kWarps - 1) / kWarps;
    const long long x0 = wp * px, x1 = min(x0 + px, (long long)P.nchx);
    double sw = 0.0, sc = 0.0;
    for (long long c = w0 + lane; c < w1; c += 32) sw += ldcg(K.w.pw2 + c);
    for (long long c = x0 + lane; c < x1; c += 32) sc += ldcg(K.w.pcx + i * P.nchx + c);
    sw = warp_sum(sw);
    sc = warp_sum(sc);
    __syncthreads();
    if (lane == 0) { gred[wp] = sw; gred[kWarps + wp] = sc; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = gred[0], b = gred[kWarps];
      for (int q = 1; q < kWarps; ++q) { a = a + gred[q]; b = b + gred[kWarps + q]; }
      gv[P.fb0 + i] = 0.5 * a + b + __ldg(P.r + i);
    }
  }
  if (P.fnb < P.mq + 1 || P.Lloc < P.L) {
    for (long long idx = gtid(); idx <= P.m; idx += gstride()) {
      const bool mine = idx <= P.mq ? (idx >= P.fb0 && idx < P.fb0 + P.fnb)
                                    : (idx - 1 - P.mq >= P.l0 && idx - 1 - P.mq < P.l0 + P.Lloc);
      if (!mine) gv[idx] = 0.0;
    }
  }
}

// ---- standalone kernels the host launches at a factored stop (fq requests)

// Row pass at x into parity par.  Warps with gwarp % 4 == 3 form the c_i . x
// items (1024-column chunks of each c_i row: a pure HBM stream beside the
// gather-bound rows); the others take the W chunks (4 slices of R each, W
// stored with an evict-last hint for the next gradient's gather, lane-ordered
// |W|^2 fma chain and a butterfly) and then the slices of A.
__global__ void __launch_bounds__(kThreads, kRowCtas) fac_row_kernel(DevProblem P, Work w, const double* x, int par) {
  const uint64_t ef = evict_first_policy();
  const uint64_t el = sym::evict_last_policy();
  const int lane = threadIdx.x & 31;
  const long long gw = gwarp(), nw = nwarps();
  if ((gw & 3) == 3) {                       // c_i . x role
    // items in chunk-major order (ch, i), a contiguous run per warp: the
    // blocks of one column chunk back to back, its x chunk L1-resident
    const long long items = (long long)P.fnb * P.nchx;
    long long lo, hi;
    my_range(items, gw >> 2, nw >> 2, lo, hi);
    for (long long it = lo; it < hi; ++it) {
      const long long ch = it / P.fnb, i = it - ch * P.fnb;
      const double s = cx_item(P, x, i, ch);
      if (lane == 0) w.pcx[i * P.nchx + ch] = s;
    }
    return;
  }
  // row-role warps are numbered densely: 3 of every 4 (the grid is a multiple of 4 warps)
  const long long me = (gw >> 2) * 3 + (gw & 3), nrole = (nw >> 2) * 3;
  double* W = w.W + (long long)par * P.nr;
  double* gv = w.gval + (long long)par * (P.m + 1) + 1 + P.mq + P.l0;
  const long long nch = __ldg(P.wch + P.fnb);
  long long lo, hi;
  my_range(nch, me, nrole, lo, hi);                       // a contiguous run of W chunks ...
  for (long long it = lo; it < hi; ++it) fac_chunk(P, w, x, W, it, ef, el);
  my_range(P.sell[kSellA].nslots >> 5, me, nrole, lo, hi);   // ... then one of A's slices
  for (long long it = lo; it < hi; ++it) fac_arows(P, x, gv, it, ef);
}

// Gradient part 1, row phase ph (lam = the trial multipliers) at the W-cache
// Wsrc, two warp roles in one launch so the HBM stream over C runs beside the
// gather-bound R^T walk: warps with gwarp % 4 == 3 continue acc over this
// phase's share of the blocks (thread per column) in aux; the others continue
// s in out and (phase 0) form t in aux2.  Dynamic shared memory: wq [fnb].
template <bool TAG>
__global__ void __launch_bounds__(kThreads, kGradCtas) fac_grad_kernel(DevProblem P, Work w, const double* Wsrc,
                                                               const double* lam, double* out, int ph) {
  extern __shared__ double wq[];
  fac_wq(P, lam, wq, kThreads);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t ef = evict_first_policy();
  const long long n = P.n;
  const long long gw = gwarp(), nw = nwarps();
  if ((gw & 3) == 3) {
    const int i0 = (int)((long long)P.fnb * ph / P.rt_nph), i1 = (int)((long long)P.fnb * (ph + 1) / P.rt_nph);
    for (long long j = (gw >> 2) * 32 + lane; j < n; j += (nw >> 2) * 32)
      w.aux[j] = fac_c_acc(P, wq, P.sym ? Wsrc : nullptr, j, i0, i1, ph > 0 ? ldcg(w.aux + j) : 0.0, ef);
    return;
  }
  const long long me = (gw >> 2) * 3 + (gw & 3), nrole = (nw >> 2) * 3;
  const long long nrt = P.sell[kSellRt + ph].nslots >> 5;
  long long lo, hi;
  my_range(nrt, me, nrole, lo, hi);                       // a contiguous run of R^T's slices ...
  for (long long it = lo; it < hi; ++it) fac_gather_item<TAG>(P, w, Wsrc, wq, lam, out, ph, it, ef);
  if (ph == 0) {                                          // ... then one of A^T's
    my_range(P.sell[kSellAt].nslots >> 5, me, nrole, lo, hi);
    for (long long it = lo; it < hi; ++it) fac_gather_item<TAG>(P, w, Wsrc, wq, lam, out, ph, nrt + it, ef);
  }
}

// Gradient part 2, thread per column: gx = (acc + s) + t into out.  With
// TRIAL, the fused yx trial's primal step too: x_new = clip(x_k - tau gx)
// (engine.py:190) into x[cur ^ 1], and this warp's partials of D_p and
// <gx, dx> into fpart[gwarp] / fpart[P.nfpart + gwarp] (a TRIAL launch uses
// exactly P.nfpart warps -- fixed per device -- so the partials' order is too).
template <bool TRIAL>
__global__ void __launch_bounds__(kThreads) fac_grad_fin_kernel(DevProblem P, Work w, double* out, double tau,
                                                                int cur) {
  const long long n = P.n;
  const double* xk = w.x + (long long)cur * n;
  double* xn = w.x + (long long)(cur ^ 1) * n;
  double dp = 0.0, gd = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) {
    const double g = (ldcg(w.aux + j) + ldcg(out + j)) + ldcg(w.aux2 + j);
    out[j] = g;
    if (TRIAL) {
      const double xj = ldcg(xk + j);
      const double xnj = clipd(xj - tau * g, __ldg(P.lo + j), __ldg(P.hi + j));
      xn[j] = xnj;
      const double d = xnj - xj;
      dp += d * d;
      gd += g * d;
    }
  }
  if (TRIAL) {
    dp = warp_sum(dp);
    gd = warp_sum(gd);
    if ((threadIdx.x & 31) == 0) {
      w.fpart[gwarp()] = dp;
      w.fpart[P.nfpart + gwarp()] = gd;
    }
  }
}

__global__ void __launch_bounds__(kThreads) fac_wl_kernel(DevProblem P, Work w, const double* Wpar,
                                                         const double* lam) {
  extern __shared__ double wq_s[];
  fac_wq(P, lam, wq_s, kThreads);
  __syncthreads();
  fac_wl(P, w, Wpar, wq_s);
}

}  // namespace rapdb
