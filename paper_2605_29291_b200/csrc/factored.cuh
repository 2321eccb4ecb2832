// factored.cuh -- the sparse factored path (BASELINE config 3): Q_i = R_i^T R_i.
//
// The U-cache of the dense path becomes a W-cache: W = R x for the stacked R
// (65 x 1e5 rows at C3, 52 MB), from which
//   g_i(x)      = 1/2 |W_i|^2 + c_i . x + d_i                (x'Q_i x = |R_i x|^2)
//   grad_x Phi  = sum_i w_i (R_i^T W_i + c_i) + A^T mu       (w_0 = 1, w_i = lam_i)
// and the linear block A x <= b enters as orthant constraints with Q = 0
// (g = A x - b, multipliers mu = lam[mq:]).
//
// Kernels (host-launched at a stop of the persistent kernel; the same
// arithmetic also exists in-kernel for RAPDB_FAC_HOST=0):
//   gradient     fac_grad_kernel: warps in two roles -- 8 lanes per column
//                walk its R^T entries (gather w_blk(r) W[r]) and A^T mu,
//                while every 4th warp streams the block-weighted c_i part;
//                fac_grad_fin_kernel combines them into grad_x Phi and, in a
//                fused yx trial, takes the primal step x_new = clip(x_k -
//                tau grad) with the D_p / <grad, dx> partials
//   row pass     fac_row_kernel: warps in two roles -- W = R x (+ |W_i|^2
//                partials per 128-row chunk) and A x - b, and the c_i . x
//                chunk partials -- so the pure HBM stream over C runs beside
//                the gather-bound CSR rows
// The CSR passes are bound by the L2 request rate of their 8-byte gathers
// (~65 M per pass at C3; tools/csr_probe2.cu), not by HBM bytes: fusing the
// dense C streams into them costs little and saves a pass and a stop.
// Per yx trial ~2.2 GB (R and R^T 780 MB each, C 520 MB, A, A^T) and one
// stop of the persistent kernel.  Every reduction has a fixed order.
#pragma once
#include "solver_kernel.cuh"

namespace rapdb {

__device__ __forceinline__ long long gwarp() { return (long long)blockIdx.x * kWarps + (threadIdx.x >> 5); }
__device__ __forceinline__ long long nwarps() { return (long long)gridDim.x * kWarps; }

constexpr int kWChunk = 128;    // rows of W per |W_i|^2 partial (inside one block)
constexpr int kCxCols = 1024;   // columns per c_i . x partial
constexpr int kGxLanes = 8;     // lanes per column in the gradient

// sum_k val[k] * x[col[k]] over CSR row r, in stored order, no FMA (the
// operation order of scipy's csr_matvec, so W = R x matches the factored
// restatement bit for bit); evict-first streams keep the gathered x in L2
__device__ __forceinline__ double csr_row_dot(const long long* __restrict__ ptr, const int* __restrict__ col,
                                              const double* __restrict__ val, const double* x, long long r,
                                              uint64_t ef) {
  long long k = __ldg(ptr + r);
  const long long k1 = __ldg(ptr + r + 1);
  double s = 0.0;
  for (; k + 8 <= k1; k += 8) {
    int c[8];
    double v[8], xv[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) { c[t] = ld_stream(col + k + t, ef); v[t] = ld_stream(val + k + t, ef); }
#pragma unroll
    for (int t = 0; t < 8; ++t) xv[t] = ldcg(x + c[t]);
#pragma unroll
    for (int t = 0; t < 8; ++t) s = __dadd_rn(s, __dmul_rn(v[t], xv[t]));
  }
  for (; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(ld_stream(val + k, ef), ldcg(x + ld_stream(col + k, ef))));
  return s;
}

// The same row sums with coalesced CSR loads (standalone kernel): a warp
// takes 32 consecutive rows [r0, min(r0 + 32, rend)), copies their
// contiguous (val, col) range into its shared-memory buffer (CAP entries per
// pass, evict-first), then each lane sums its own row in stored order
// without FMA from shared memory, 4 gathers in flight -- the bits of
// csr_row_dot.  The fastest of the C3 row-pass variants measured
// (tools/csr_probe.cu, tools/csr_probe2.cu: 0.30 ms for R x).
constexpr int kStageCap = 320;
__device__ __forceinline__ double csr_group32(const long long* __restrict__ ptr, const int* __restrict__ col,
                                              const double* __restrict__ val, const double* x, long long r0,
                                              long long rend, double* sv, int* sc, uint64_t ef) {
  const int lane = threadIdx.x & 31;
  const long long r = r0 + lane;
  const long long kb = __ldg(ptr + r0);
  const long long ke = __ldg(ptr + min(r0 + 32, rend));
  long long k = r < rend ? __ldg(ptr + r) : ke;
  const long long k1 = r < rend ? __ldg(ptr + r + 1) : ke;
  double s = 0.0;
  for (long long base = kb; base < ke; base += kStageCap) {
    const long long lim = min(base + kStageCap, ke);
    for (long long e = base + lane; e < lim; e += 32) {
      sv[e - base] = ld_stream(val + e, ef);
      sc[e - base] = ld_stream(col + e, ef);
    }
    __syncwarp();
    const long long kend = min(k1, lim);
    for (; k + 4 <= kend; k += 4) {
      double xv[4], vv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        vv[t] = sv[k + t - base];
        xv[t] = ldcg(x + sc[k + t - base]);
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) s = __dadd_rn(s, __dmul_rn(vv[t], xv[t]));
    }
    for (; k < kend; ++k) s = __dadd_rn(s, __dmul_rn(sv[k - base], ldcg(x + sc[k - base])));
    __syncwarp();
  }
  return s;
}

// rows [r0, r1) of W chunk c (wch[i] = first chunk of local block i)
__device__ __forceinline__ void wchunk_rows(const DevProblem& P, long long c, long long& r0, long long& r1) {
  int lo = 0, hi = P.fnb;                 // local block of chunk c: wch[lo] <= c < wch[lo+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(P.wch + mid) <= c) lo = mid; else hi = mid;
  }
  r0 = __ldg(P.rblk + lo) + (c - __ldg(P.wch + lo)) * kWChunk;
  r1 = min(r0 + kWChunk, __ldg(P.rblk + lo + 1));
}

// c_i . x over columns [ch*1024, +1024): lane-strided fma chain, butterfly
// (the partial of item it = i * nchx + ch)
__device__ __forceinline__ double cx_item(const DevProblem& P, const double* x, long long it) {
  const int lane = threadIdx.x & 31;
  const long long n = P.n;
  const long long i = it / P.nchx, ch = it - i * P.nchx;
  const long long j0 = ch * kCxCols, j1 = min(j0 + kCxCols, n);
  const double* ci = P.q + i * n;
  double s = 0.0;
  for (long long j = j0 + lane; j < j1; j += 32) s = fma(__ldg(ci + j), ldcg(x + j), s);
  return warp_sum(s);
}

// ---------------------------------------------------------------- gradient
__device__ __forceinline__ void fac_wq(const DevProblem& P, const double* lam, double* wq, int nthreads) {
  for (int i = threadIdx.x; i < P.fnb; i += nthreads) {
    const int gi = P.fb0 + i;             // global block id (0 = objective)
    wq[i] = gi == 0 ? 1.0 : ldcg(lam + (gi - 1));
  }
}

constexpr int kRtTagShift = 23;
constexpr int kRtRowMask = (1 << kRtTagShift) - 1;

// w_blk(r) W[r] of one R^T entry (tagged rows), or the weighted W-cache
template <bool TAG>
__device__ __forceinline__ double rt_weighted(const double* Wsrc, const double* wq, int idx) {
  if (TAG) return wq[idx >> kRtTagShift] * ldcg(Wsrc + (idx & kRtRowMask));
  return ldcg(Wsrc + idx);
}

// Wl[r] = w_blk(r) W[r] (untagged R^T only)
__device__ __forceinline__ void fac_wl(const DevProblem& P, const Work& w, const double* Wpar, const double* wq) {
  const uint64_t ef = evict_first_policy();
  const uint64_t el = sym::evict_last_policy();
  for (long long r = gtid(); r < P.nr; r += gstride())
    st_keep(w.wl + r, wq[ld_stream(P.rmat + r, ef)] * ldcg(Wpar + r), el);
}

// grad_x Phi column j = (acc + s) + t, every path the same bits:
//   acc  sum_i w_i c_ij over the blocks in order, skipping zero weights
//        (one thread per column: a plain HBM stream over C);
//   s    the R^T gather sum_r v w_blk(r) W[r]: the 8 lanes sub = 0..7 of a
//        lane group fold entries k0 + sub, + 8, ... with fma (two in flight)
//        over the row phases in order, then an xor tree over the 8 lanes;
//   t    A^T mu the same way.
__device__ __forceinline__ double fac_c_acc(const DevProblem& P, const double* wq, long long j, uint64_t ef) {
  const long long n = P.n;
  double acc = 0.0;
  int i = 0;
  for (; i + 8 <= P.fnb; i += 8) {        // 8 independent loads in flight
    double c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = ld_stream(P.q + (long long)(i + k) * n + j, ef);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double l = wq[i + k];
      acc = (l != 0.0) ? acc + l * c[k] : acc;
    }
  }
  for (; i < P.fnb; ++i) {
    const double l = wq[i];
    const double c = ld_stream(P.q + (long long)i * n + j, ef);
    acc = (l != 0.0) ? acc + l * c : acc;
  }
  return acc;
}

template <bool TAG>
__device__ __forceinline__ void fac_gather_col(const DevProblem& P, const double* Wsrc, const double* wq,
                                               const double* lam, long long j, int sub, uint64_t ef,
                                               double& s, double& t) {
  const long long n = P.n;
  s = 0.0;
  t = 0.0;
  if (j < n) {
    for (int ph = 0; ph < P.rt_nph; ++ph) {
      const long long* ptr = P.rt_ptr + (long long)ph * (n + 1);
      const long long k1 = __ldg(ptr + j + 1);
      long long k = __ldg(ptr + j) + sub;
      for (; k + kGxLanes < k1; k += 2 * kGxLanes) {
        const int r0 = ld_stream(P.rt_row + k, ef), r1 = ld_stream(P.rt_row + k + kGxLanes, ef);
        const double v0 = ld_stream(P.rt_val + k, ef), v1 = ld_stream(P.rt_val + k + kGxLanes, ef);
        const double w0 = rt_weighted<TAG>(Wsrc, wq, r0), w1 = rt_weighted<TAG>(Wsrc, wq, r1);
        s = fma(v0, w0, s);
        s = fma(v1, w1, s);
      }
      if (k < k1) s = fma(ld_stream(P.rt_val + k, ef), rt_weighted<TAG>(Wsrc, wq, ld_stream(P.rt_row + k, ef)), s);
    }
    const long long a0 = __ldg(P.at_ptr + j), a1 = __ldg(P.at_ptr + j + 1);
    for (long long k = a0 + sub; k < a1; k += kGxLanes)
      t = fma(ld_stream(P.at_val + k, ef), ldcg(lam + P.mq + P.l0 + ld_stream(P.at_row + k, ef)), t);
  }
#pragma unroll
  for (int o = kGxLanes / 2; o >= 1; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    t += __shfl_xor_sync(0xffffffffu, t, o);
  }
}

// In-kernel version (RAPDB_FAC_HOST=0): the same lane groups over the
// persistent grid, lane sub == 0 adds its column's c_i part.
template <bool TAG>
__device__ __forceinline__ void fac_gx_cols(const DevProblem& P, const double* Wsrc, const double* wq,
                                            const double* lam, double* out) {
  const int lane = threadIdx.x & 31;
  const int sub = lane & (kGxLanes - 1), grp = lane / kGxLanes;
  const uint64_t ef = evict_first_policy();
  for (long long jb = gwarp() * (32 / kGxLanes); jb < P.n; jb += nwarps() * (32 / kGxLanes)) {
    const long long j = jb + grp;
    double s, t;
    fac_gather_col<TAG>(P, Wsrc, wq, lam, j, sub, ef, s, t);
    if (j < P.n && sub == 0) out[j] = (fac_c_acc(P, wq, j, ef) + s) + t;
  }
}

__device__ __noinline__ bool recombine_factored(const KArgs& K, Sm& S, const double* Wpar, const double* lam,
                                                double* out) {
  double* wq = S.stage;
  __syncthreads();
  fac_wq(K.P, lam, wq, kThreads);
  __syncthreads();
  if (K.P.rt_tag) {
    fac_gx_cols<true>(K.P, Wpar, wq, lam, out);
    return true;
  }
  fac_wl(K.P, K.w, Wpar, wq);
  if (!gsync(K, S)) return false;
  fac_gx_cols<false>(K.P, K.w.wl, wq, lam, out);
  return true;
}

// ---------------------------------------------------------------- in-kernel sweep
// "Sweep" at x into parity par, part A: W = R x (thread per row), A x - b
// into the linear part of gval[par], the c_i . x chunk partials (warp per
// item).  Part B (after a grid barrier): the |W_i|^2 chunk partials.  Used
// when the persistent kernel runs the factored path itself (RAPDB_FAC_HOST=0).
__device__ __forceinline__ void fac_sweep_a(const DevProblem& P, const Work& w, const double* x, int par) {
  double* W = w.W + (long long)par * P.nr;
  const uint64_t ef = evict_first_policy();
  const uint64_t el = sym::evict_last_policy();
  for (long long r = gtid(); r < P.nr; r += gstride())
    st_keep(W + r, csr_row_dot(P.r_ptr, P.r_col, P.r_val, x, r, ef), el);
  double* gv = w.gval + (long long)par * (P.m + 1);
  for (long long j = gtid(); j < P.Lloc; j += gstride())
    gv[1 + P.mq + P.l0 + j] = csr_row_dot(P.a_ptr, P.a_col, P.a_val, x, j, ef) - __ldg(P.b + j);
  const long long items = (long long)P.fnb * P.nchx;
  for (long long it = gwarp(); it < items; it += nwarps()) {
    const double s = cx_item(P, x, it);
    if ((threadIdx.x & 31) == 0) w.pcx[it] = s;
  }
}

// |W_i|^2 over chunk c: lane r0 + lane, + 32, ... with fma, then the butterfly
__device__ __forceinline__ double w2_chunk(const double* W, long long r0, long long r1) {
  double s = 0.0;
  for (long long r = r0 + (threadIdx.x & 31); r < r1; r += 32) {
    const double v = ldcg(W + r);
    s = fma(v, v, s);
  }
  return warp_sum(s);
}

__device__ __forceinline__ void fac_sweep_b(const DevProblem& P, const Work& w, int par) {
  const double* W = w.W + (long long)par * P.nr;
  const long long nch = __ldg(P.wch + P.fnb);
  for (long long c = gwarp(); c < nch; c += nwarps()) {
    long long r0, r1;
    wchunk_rows(P, c, r0, r1);
    const double s = w2_chunk(W, r0, r1);
    if ((threadIdx.x & 31) == 0) w.pw2[c] = s;
  }
}

__device__ __noinline__ bool sweep_factored(const KArgs& K, Sm& S, const double* x, int par) {
  fac_sweep_a(K.P, K.w, x, par);
  if (!gsync(K, S)) return false;
  fac_sweep_b(K.P, K.w, par);
  return gsync(K, S);
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
// items (1024-column chunks of each c_i row: a pure HBM stream); the others
// take the W chunks (128 rows of R as 4 staged 32-row groups, W stored with
// an evict-last hint for the next gradient's gather, lane-ordered |W|^2 fma
// chain and a butterfly -- w2_chunk's bits) and then the 32-row groups of A.
__global__ void __launch_bounds__(kThreads, 4) fac_row_kernel(DevProblem P, Work w, const double* x, int par) {
  __shared__ double sv[kWarps][kStageCap];
  __shared__ int sc[kWarps][kStageCap];
  const uint64_t ef = evict_first_policy();
  const uint64_t el = sym::evict_last_policy();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const long long gw = gwarp(), nw = nwarps();
  if ((gw & 3) == 3) {                       // c_i . x role
    const long long items = (long long)P.fnb * P.nchx;
    for (long long it = gw >> 2; it < items; it += nw >> 2) {
      const double s = cx_item(P, x, it);
      if (lane == 0) w.pcx[it] = s;
    }
    return;
  }
  // row-role warps are numbered densely: 3 of every 4 (the grid is a multiple of 4 warps)
  const long long me = (gw >> 2) * 3 + (gw & 3), nrole = (nw >> 2) * 3;
  double* W = w.W + (long long)par * P.nr;
  double* gv = w.gval + (long long)par * (P.m + 1) + 1 + P.mq + P.l0;
  const long long nch = __ldg(P.wch + P.fnb);
  const long long items = nch + (P.Lloc + 31) / 32;
  for (long long it = me; it < items; it += nrole) {
    if (it < nch) {
      long long r0, r1;
      wchunk_rows(P, it, r0, r1);
      double s2 = 0.0;
      for (long long g0 = r0; g0 < r1; g0 += 32) {
        const double v = csr_group32(P.r_ptr, P.r_col, P.r_val, x, g0, r1, sv[wp], sc[wp], ef);
        if (g0 + lane < r1) {
          st_keep(W + g0 + lane, v, el);
          s2 = fma(v, v, s2);
        }
      }
      s2 = warp_sum(s2);
      if (lane == 0) w.pw2[it] = s2;
    } else {
      const long long a0 = (it - nch) * 32, a1 = min(a0 + 32, (long long)P.Lloc);
      const double v = csr_group32(P.a_ptr, P.a_col, P.a_val, x, a0, a1, sv[wp], sc[wp], ef);
      if (a0 + lane < a1) gv[a0 + lane] = v - __ldg(P.b + a0 + lane);
    }
  }
}

// Gradient part 1 (lam = the trial multipliers) at the W-cache Wsrc, two warp
// roles in one launch so the HBM stream over C runs beside the gather-bound
// R^T walk: warps with gwarp % 4 == 3 form acc (thread per column) into aux;
// the others form s into out and t into aux2.  Dynamic shared memory: wq [fnb].
template <bool TAG>
__global__ void __launch_bounds__(kThreads, 8) fac_grad_kernel(DevProblem P, Work w, const double* Wsrc,
                                                               const double* lam, double* out) {
  extern __shared__ double wq[];
  fac_wq(P, lam, wq, kThreads);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t ef = evict_first_policy();
  const long long n = P.n;
  const long long gw = gwarp(), nw = nwarps();
  if ((gw & 3) == 3) {
    for (long long j = (gw >> 2) * 32 + lane; j < n; j += (nw >> 2) * 32) w.aux[j] = fac_c_acc(P, wq, j, ef);
    return;
  }
  const int sub = lane & (kGxLanes - 1), grp = lane / kGxLanes;
  const long long me = (gw >> 2) * 3 + (gw & 3), nrole = (nw >> 2) * 3;
  for (long long jb = me * (32 / kGxLanes); jb < n; jb += nrole * (32 / kGxLanes)) {
    const long long j = jb + grp;
    double s, t;
    fac_gather_col<TAG>(P, Wsrc, wq, lam, j, sub, ef, s, t);
    if (j < n && sub == 0) {
      out[j] = s;
      w.aux2[j] = t;
    }
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
