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

// "Sweep" at x into parity par: W = R x (thread per row), A x - b into the
// linear part of gval[par], chunk partials of c_i . x (warp per 1024 columns),
// then (after a grid barrier) chunk partials of |W_i|^2 (warp per 1024 rows).
__device__ bool sweep_factored(const KArgs& K, Sm& S, const double* x, int par) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  const long long n = P.n;
  const int lane = threadIdx.x & 31;
  double* W = w.W + (long long)par * P.nr;
  for (long long r = gtid(); r < P.nr; r += gstride()) {
    const long long k0 = __ldg(P.r_ptr + r), k1 = __ldg(P.r_ptr + r + 1);
    double s = 0.0;
    for (long long k = k0; k < k1; ++k) s = fma(__ldg(P.r_val + k), ldcg(x + __ldg(P.r_col + k)), s);
    W[r] = s;
  }
  double* gv = w.gval + (long long)par * (P.m + 1);
  for (long long j = gtid(); j < P.L; j += gstride()) {
    const long long k0 = __ldg(P.a_ptr + j), k1 = __ldg(P.a_ptr + j + 1);
    double s = 0.0;
    for (long long k = k0; k < k1; ++k) s = fma(__ldg(P.a_val + k), ldcg(x + __ldg(P.a_col + k)), s);
    gv[1 + P.mq + j] = s - __ldg(P.b + j);
  }
  const long long items = (long long)(P.mq + 1) * P.nchx;
  for (long long it = gwarp(); it < items; it += nwarps()) {
    const long long i = it / P.nchx, ch = it - i * P.nchx;
    const long long j0 = ch * 1024, j1 = min(j0 + 1024, n);
    const double* ci = P.q + i * n;
    double s = 0.0;
    for (long long j = j0 + lane; j < j1; j += 32) s = fma(__ldg(ci + j), ldcg(x + j), s);
    s = warp_sum(s);
    if (lane == 0) w.pcx[it] = s;
  }
  if (!gsync(K, S)) return false;
  const long long nchw = __ldg(P.wch + P.mq + 1);
  for (long long c = gwarp(); c < nchw; c += nwarps()) {
    int lo = 0, hi = P.mq + 1;            // block of chunk c: wch[lo] <= c < wch[lo+1]
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
  return gsync(K, S);
}

// g_i (i = 0..mq, 0 = f) at parity par from the chunk partials: one warp per i
__device__ void g_factored(const KArgs& K, int par) {
  const DevProblem& P = K.P;
  const int lane = threadIdx.x & 31;
  double* gv = K.w.gval + (long long)par * (P.m + 1);
  for (long long i = gwarp(); i <= P.mq; i += nwarps()) {
    double sw = 0.0, sc = 0.0;
    for (long long c = __ldg(P.wch + i) + lane; c < __ldg(P.wch + i + 1); c += 32) sw += ldcg(K.w.pw2 + c);
    for (long long c = lane; c < P.nchx; c += 32) sc += ldcg(K.w.pcx + i * P.nchx + c);
    sw = warp_sum(sw);
    sc = warp_sum(sc);
    if (lane == 0) gv[i] = 0.5 * sw + sc + __ldg(P.r + i);
  }
}

// out = sum_i w_i (R_i^T W_i + c_i) + A^T mu with w = (1, lam_1..lam_mq),
// mu = lam[mq..]; lam is a global m-vector.  Pass 1 (column-parallel) adds
// the dense c_i terms, pass 2 (warp per column) the R^T and A^T gathers.
// The result is complete after the caller's grid barrier.
__device__ bool recombine_factored(const KArgs& K, Sm& S, const double* Wpar, const double* lam, double* out) {
  const DevProblem& P = K.P;
  const long long n = P.n;
  const int lane = threadIdx.x & 31;
  double* wq = S.stage;
  __syncthreads();
  for (int i = threadIdx.x; i <= P.mq; i += kThreads) wq[i] = i == 0 ? 1.0 : ldcg(lam + (i - 1));
  __syncthreads();
  for (long long j = gtid(); j < n; j += gstride()) {
    double acc = 0.0;
    int i = 0;
    for (; i + 3 <= P.mq; i += 4) {
      double c[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) c[k] = __ldg(P.q + (long long)(i + k) * n + j);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double l = wq[i + k];
        acc = (l != 0.0) ? acc + l * c[k] : acc;
      }
    }
    for (; i <= P.mq; ++i) {
      const double l = wq[i];
      if (l != 0.0) acc = acc + l * __ldg(P.q + (long long)i * n + j);
    }
    out[j] = acc;
  }
  if (!gsync(K, S)) return false;
  for (long long j = gwarp(); j < n; j += nwarps()) {
    const long long k0 = __ldg(P.rt_ptr + j), k1 = __ldg(P.rt_ptr + j + 1);
    double s = 0.0;
    for (long long k = k0 + lane; k < k1; k += 32) {
      const int r = __ldg(P.rt_row + k);
      const double l = wq[__ldg(P.rmat + r)];
      s = fma(__ldg(P.rt_val + k) * ldcg(Wpar + r), l, s);
    }
    double t = 0.0;
    const long long a0 = __ldg(P.at_ptr + j), a1 = __ldg(P.at_ptr + j + 1);
    for (long long k = a0 + lane; k < a1; k += 32) t = fma(__ldg(P.at_val + k), ldcg(lam + P.mq + __ldg(P.at_row + k)), t);
    s = warp_sum(s);
    t = warp_sum(t);
    if (lane == 0) out[j] = (ldcg(out + j) + s) + t;
  }
  return true;
}

}  // namespace rapdb
