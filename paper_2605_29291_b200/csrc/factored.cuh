// factored.cuh -- the sparse factored path (BASELINE config 3): Q_i = R_i^T R_i.
//
// The U-cache of the dense path becomes a W-cache: W = R x for the stacked R
// (65 x 1e5 rows at C3, 52 MB), from which
//   g_i(x)      = 1/2 |W_i|^2 + c_i . x + d_i                (x'Q_i x = |R_i x|^2)
//   grad_x Phi  = sum_i w_i (R_i^T W_i + c_i) + A^T mu       (w_0 = 1, w_i = lam_i)
// and the linear block A x <= b enters as orthant constraints with Q = 0
// (g = A x - b, multipliers mu = lam[mq:]).  Per trial the device reads
// R (sweep), R^T (recombination), C twice and A, A^T once: ~2.66 GB at C3.
// Sparse products are gathers over CSR (R, and a separate CSR of R^T / A^T so
// the transposed products need no atomics); every reduction has a fixed order.
#pragma once
#include "solver_kernel.cuh"

namespace rapdb {

__device__ __forceinline__ long long gwarp() { return (long long)blockIdx.x * kWarps + (threadIdx.x >> 5); }
__device__ __forceinline__ long long nwarps() { return (long long)gridDim.x * kWarps; }

// sum_k val[k] * x[col[k]] over CSR row r, in stored order, no FMA; the CSR
// arrays stream with an evict-first policy so the gathered x stays in L2
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
  for (; k + 4 <= k1; k += 4) {
    const int c0 = ld_stream(col + k, ef), c1 = ld_stream(col + k + 1, ef);
    const int c2 = ld_stream(col + k + 2, ef), c3 = ld_stream(col + k + 3, ef);
    const double v0 = ld_stream(val + k, ef), v1 = ld_stream(val + k + 1, ef);
    const double v2 = ld_stream(val + k + 2, ef), v3 = ld_stream(val + k + 3, ef);
    const double x0 = ldcg(x + c0), x1 = ldcg(x + c1), x2 = ldcg(x + c2), x3 = ldcg(x + c3);
    s = __dadd_rn(s, __dmul_rn(v0, x0));
    s = __dadd_rn(s, __dmul_rn(v1, x1));
    s = __dadd_rn(s, __dmul_rn(v2, x2));
    s = __dadd_rn(s, __dmul_rn(v3, x3));
  }
  for (; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(ld_stream(val + k, ef), ldcg(x + ld_stream(col + k, ef))));
  return s;
}

// The same row sums with coalesced CSR loads (standalone kernel): a warp
// takes 32 consecutive rows, copies their contiguous (val, col) range into
// its shared-memory buffer (CAP entries per pass, evict-first), then each lane
// sums its own row in stored order without FMA from shared memory -- the bits
// of csr_row_dot.  C3's R x: 0.41 -> 0.30 ms (tools/csr_probe.cu, warpstage320).
constexpr int kStageCap = 320;
template <typename Store>
__device__ __forceinline__ void csr_rows_staged(const long long* __restrict__ ptr, const int* __restrict__ col,
                                                const double* __restrict__ val, const double* x, long long rows,
                                                double (*sv)[kStageCap], int (*sc)[kStageCap], uint64_t ef,
                                                Store store) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long long r0 = gwarp() * 32; r0 < rows; r0 += nwarps() * 32) {
    const long long r = r0 + lane;
    const long long kb = __ldg(ptr + r0);
    const long long ke = __ldg(ptr + min(r0 + 32, rows));
    long long k = r < rows ? __ldg(ptr + r) : ke;
    const long long k1 = r < rows ? __ldg(ptr + r + 1) : ke;
    double s = 0.0;
    for (long long base = kb; base < ke; base += kStageCap) {
      const long long lim = min(base + kStageCap, ke);
      for (long long e = base + lane; e < lim; e += 32) {
        sv[w][e - base] = ld_stream(val + e, ef);
        sc[w][e - base] = ld_stream(col + e, ef);
      }
      __syncwarp();
      const long long kend = min(k1, lim);
      for (; k + 4 <= kend; k += 4) {
        double xv[4], vv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          vv[t] = sv[w][k + t - base];
          xv[t] = ldcg(x + sc[w][k + t - base]);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) s = __dadd_rn(s, __dmul_rn(vv[t], xv[t]));
      }
      for (; k < kend; ++k) s = __dadd_rn(s, __dmul_rn(sv[w][k - base], ldcg(x + sc[w][k - base])));
      __syncwarp();
    }
    if (r < rows) store(r, s);
  }
}

// "Sweep" at x into parity par, part A: W = R x (thread per row), A x - b
// into the linear part of gval[par], chunk partials of c_i . x (warp per 1024
// columns).  Part B (after a grid barrier / kernel boundary): chunk partials
// of |W_i|^2 (warp per 1024 rows).  Both run inside the persistent kernel
// (sweep_factored) or as high-occupancy standalone kernels launched by the
// host at a stop (fac_sweep_*_kernel, the default: the gathers are latency
// bound and 8 warps per SM starve them -- tools/csr_probe.cu).
__device__ __forceinline__ void fac_sweep_a(const DevProblem& P, const Work& w, const double* x, int par) {
  const long long n = P.n;
  const int lane = threadIdx.x & 31;
  double* W = w.W + (long long)par * P.nr;
  // thread per CSR row, products summed in stored order without FMA (the
  // operation order of scipy's csr_matvec, so W = R x matches the restatement
  // bit for bit); the row's loads are issued in batches for MLP
  const uint64_t ef = evict_first_policy();
  const uint64_t el = sym::evict_last_policy();
  for (long long r = gtid(); r < P.nr; r += gstride())
    st_keep(W + r, csr_row_dot(P.r_ptr, P.r_col, P.r_val, x, r, ef), el);
  double* gv = w.gval + (long long)par * (P.m + 1);
  for (long long j = gtid(); j < P.Lloc; j += gstride())
    gv[1 + P.mq + P.l0 + j] = csr_row_dot(P.a_ptr, P.a_col, P.a_val, x, j, ef) - __ldg(P.b + j);
  const long long items = (long long)P.fnb * P.nchx;
  for (long long it = gwarp(); it < items; it += nwarps()) {
    const long long i = it / P.nchx, ch = it - i * P.nchx;
    const long long j0 = ch * 1024, j1 = min(j0 + 1024, n);
    const double* ci = P.q + i * n;
    double s = 0.0;
    for (long long j = j0 + lane; j < j1; j += 32) s = fma(__ldg(ci + j), ldcg(x + j), s);
    s = warp_sum(s);
    if (lane == 0) w.pcx[it] = s;
  }
}

__device__ __forceinline__ void fac_sweep_b(const DevProblem& P, const Work& w, int par) {
  const int lane = threadIdx.x & 31;
  const double* W = w.W + (long long)par * P.nr;
  const long long nchw = __ldg(P.wch + P.fnb);
  for (long long c = gwarp(); c < nchw; c += nwarps()) {
    int lo = 0, hi = P.fnb;               // local block of chunk c: wch[lo] <= c < wch[lo+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(P.wch + mid) <= c) lo = mid; else hi = mid;
    }
    const long long r0 = __ldg(P.rblk + lo) + (c - __ldg(P.wch + lo)) * 1024;
    const long long r1 = min(r0 + 1024, __ldg(P.rblk + lo + 1));
    double s = 0.0;
    for (long long r = r0 + lane; r < r1; r += 32) {
      const double v = ldcg(W + r);
      s = fma(v, v, s);
    }
    s = warp_sum(s);
    if (lane == 0) w.pw2[c] = s;
  }
}

__device__ __noinline__ bool sweep_factored(const KArgs& K, Sm& S, const double* x, int par) {
  fac_sweep_a(K.P, K.w, x, par);
  if (!gsync(K, S)) return false;
  fac_sweep_b(K.P, K.w, par);
  return gsync(K, S);
}

// g_i (i = 0..mq, 0 = f) at parity par from the chunk partials: one warp per
// local block; a sharded rank writes 0 for the entries it does not own (the
// all-reduce of g is then exact: disjoint supports)
__device__ void g_factored(const KArgs& K, int par) {
  const DevProblem& P = K.P;
  const int lane = threadIdx.x & 31;
  double* gv = K.w.gval + (long long)par * (P.m + 1);
  for (long long i = gwarp(); i < P.fnb; i += nwarps()) {
    double sw = 0.0, sc = 0.0;
    for (long long c = __ldg(P.wch + i) + lane; c < __ldg(P.wch + i + 1); c += 32) sw += ldcg(K.w.pw2 + c);
    for (long long c = lane; c < P.nchx; c += 32) sc += ldcg(K.w.pcx + i * P.nchx + c);
    sw = warp_sum(sw);
    sc = warp_sum(sc);
    if (lane == 0) gv[P.fb0 + i] = 0.5 * sw + sc + __ldg(P.r + i);
  }
  if (P.fnb < P.mq + 1 || P.Lloc < P.L) {
    for (long long idx = gtid(); idx <= P.m; idx += gstride()) {
      const bool mine = idx <= P.mq ? (idx >= P.fb0 && idx < P.fb0 + P.fnb)
                                    : (idx - 1 - P.mq >= P.l0 && idx - 1 - P.mq < P.l0 + P.Lloc);
      if (!mine) gv[idx] = 0.0;
    }
  }
}

// out = sum_i w_i (R_i^T W_i + c_i) + A^T mu with w = (1, lam_1..lam_mq),
// mu = lam[mq..]; lam is a global m-vector.  Part A (element-parallel) adds
// the dense c_i terms and scales the W-cache by its block weight,
// Wl[r] = w_{blk(r)} W[r]; part B gathers R^T Wl and A^T mu (2 lanes per
// column).  wq: the fnb block weights, staged in shared memory by the caller.
__device__ __forceinline__ void fac_wq(const DevProblem& P, const double* lam, double* wq, int nthreads) {
  for (int i = threadIdx.x; i < P.fnb; i += nthreads) {
    const int gi = P.fb0 + i;             // global block id (0 = objective)
    wq[i] = gi == 0 ? 1.0 : ldcg(lam + (gi - 1));
  }
}

__device__ __forceinline__ void fac_gx_a(const DevProblem& P, const Work& w, const double* Wpar, const double* wq,
                                         double* out) {
  const long long n = P.n;
  const uint64_t ef = evict_first_policy();
  const uint64_t el = sym::evict_last_policy();
  for (long long j = gtid(); j < n; j += gstride()) {
    double acc = 0.0;
    int i = 0;
    for (; i + 16 <= P.fnb; i += 16) {   // 16 independent loads in flight per thread
      double c[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) c[k] = ld_stream(P.q + (long long)(i + k) * n + j, ef);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const double l = wq[i + k];
        acc = (l != 0.0) ? acc + l * c[k] : acc;
      }
    }
    for (; i + 4 <= P.fnb; i += 4) {
      double c[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) c[k] = ld_stream(P.q + (long long)(i + k) * n + j, ef);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double l = wq[i + k];
        acc = (l != 0.0) ? acc + l * c[k] : acc;
      }
    }
    for (; i < P.fnb; ++i) {
      const double l = wq[i];
      if (l != 0.0) acc = acc + l * ld_stream(P.q + (long long)i * n + j, ef);
    }
    out[j] = acc;
  }
  for (long long r = gtid(); r < P.nr; r += gstride())
    st_keep(w.wl + r, wq[ld_stream(P.rmat + r, ef)] * ldcg(Wpar + r), el);
}

// LW lanes per column: 2 is best at the persistent kernel's 8 warps per SM,
// 8 in a standalone kernel with 8 CTAs per SM (tools/csr_probe.cu)
template <int LW>
__device__ __forceinline__ void fac_gx_b(const DevProblem& P, const Work& w, const double* lam, double* out) {
  const long long n = P.n;
  const int lane = threadIdx.x & 31;
  const uint64_t ef = evict_first_policy();
  const double* Wl = w.wl;
  const int sub = lane & (LW - 1), grp = lane / LW;
  for (long long jb = gwarp() * (32 / LW); jb < n; jb += nwarps() * (32 / LW)) {
    const long long j = jb + grp;
    double s = 0.0, t = 0.0;
    if (j < n) {
      const long long k0 = __ldg(P.rt_ptr + j), k1 = __ldg(P.rt_ptr + j + 1);
      long long k = k0 + sub;
      for (; k + LW < k1; k += 2 * LW) {
        const int r0 = ld_stream(P.rt_row + k, ef), r1 = ld_stream(P.rt_row + k + LW, ef);
        const double v0 = ld_stream(P.rt_val + k, ef), v1 = ld_stream(P.rt_val + k + LW, ef);
        const double w0 = ldcg(Wl + r0), w1 = ldcg(Wl + r1);
        s = fma(v0, w0, s);
        s = fma(v1, w1, s);
      }
      if (k < k1) s = fma(ld_stream(P.rt_val + k, ef), ldcg(Wl + ld_stream(P.rt_row + k, ef)), s);
      const long long a0 = __ldg(P.at_ptr + j), a1 = __ldg(P.at_ptr + j + 1);
      for (long long k = a0 + sub; k < a1; k += LW)
        t = fma(ld_stream(P.at_val + k, ef), ldcg(lam + P.mq + P.l0 + ld_stream(P.at_row + k, ef)), t);
    }
#pragma unroll
    for (int o = LW / 2; o >= 1; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    if (j < n && sub == 0) out[j] = (ldcg(out + j) + s) + t;
  }
}

__device__ __noinline__ bool recombine_factored(const KArgs& K, Sm& S, const double* Wpar, const double* lam,
                                                double* out) {
  double* wq = S.stage;
  __syncthreads();
  fac_wq(K.P, lam, wq, kThreads);
  __syncthreads();
  fac_gx_a(K.P, K.w, Wpar, wq, out);
  if (!gsync(K, S)) return false;
  fac_gx_b<2>(K.P, K.w, lam, out);
  return true;
}

// ---- standalone kernels the host launches at a factored stop (fq requests):
// same device code, any grid (blockDim = kThreads), many CTAs per SM
__device__ __forceinline__ void fac_sweep_a_staged(const DevProblem& P, const Work& w, const double* x, int par) {
  __shared__ double sv[kWarps][kStageCap];
  __shared__ int sc[kWarps][kStageCap];
  const uint64_t ef = evict_first_policy();
  const uint64_t el = sym::evict_last_policy();
  double* W = w.W + (long long)par * P.nr;
  csr_rows_staged(P.r_ptr, P.r_col, P.r_val, x, P.nr, sv, sc, ef,
                  [&](long long r, double v) { st_keep(W + r, v, el); });
  double* gv = w.gval + (long long)par * (P.m + 1) + 1 + P.mq + P.l0;
  csr_rows_staged(P.a_ptr, P.a_col, P.a_val, x, P.Lloc, sv, sc, ef,
                  [&](long long j, double v) { gv[j] = v - __ldg(P.b + j); });
  const int lane = threadIdx.x & 31;
  const long long n = P.n;
  const long long items = (long long)P.fnb * P.nchx;
  for (long long it = gwarp(); it < items; it += nwarps()) {
    const long long i = it / P.nchx, ch = it - i * P.nchx;
    const long long j0 = ch * 1024, j1 = min(j0 + 1024, n);
    const double* ci = P.q + i * n;
    double s = 0.0;
    for (long long j = j0 + lane; j < j1; j += 32) s = fma(__ldg(ci + j), ldcg(x + j), s);
    s = warp_sum(s);
    if (lane == 0) w.pcx[it] = s;
  }
}
__global__ void __launch_bounds__(kThreads) fac_sweep_a_kernel(DevProblem P, Work w, const double* x, int par) {
  fac_sweep_a_staged(P, w, x, par);
}
__global__ void __launch_bounds__(kThreads) fac_sweep_b_kernel(DevProblem P, Work w, int par) {
  fac_sweep_b(P, w, par);
}
__global__ void __launch_bounds__(kThreads) fac_gx_a_kernel(DevProblem P, Work w, const double* Wpar,
                                                           const double* lam, double* out) {
  extern __shared__ double wq_s[];
  fac_wq(P, lam, wq_s, kThreads);
  __syncthreads();
  fac_gx_a(P, w, Wpar, wq_s, out);
}
__global__ void __launch_bounds__(kThreads) fac_gx_b_kernel(DevProblem P, Work w, const double* lam, double* out) {
  fac_gx_b<8>(P, w, lam, out);
}

}  // namespace rapdb
