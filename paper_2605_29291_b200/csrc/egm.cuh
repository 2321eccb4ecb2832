// egm.cuh -- the extragradient baseline (egm.py:37-77) on the device, built
// from the rAPDB path's pieces (U-cache recombination, fused sweep, g
// combination, ball projection, fixed-order reductions):
//
//   z~ = Pi(z - s F(z)),  z+ = Pi(z - s F(z~)),   F = (grad_x Phi, -grad_y Phi)
//
// with Pi the product projection (box, orthant, dual ball).  The current point
// z lives at parity `cur` with its caches (U, g, A x - b) valid; z~ and then z+
// are formed at parity cur^1 (two sweeps per iteration), and cur flips at the
// end.  Ergodic sums (weight 1) go to xcum / ycum with st.T = iterations, so
// op_get(average) returns egm.py's average.  Divergence: |z| > 1e8 (1 + |z0|).
#pragma once
#include "solver_ops.cuh"

namespace rapdb {

// |x|^2, |v|^2, |lam|^2 of the point at parity par -> partial slots
__device__ __forceinline__ void egm_norm_partials(const KArgs& K, Sm& S, int par) {
  const DevProblem& P = K.P;
  const int n = P.n, p = P.p, np = p + P.m;
  const double* x = K.w.x + (long long)par * n;
  const double* y = K.w.y + (long long)par * np;
  double sx = 0.0, sv = 0.0, sl = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) { const double t = ldcg(x + j); sx += t * t; }
  for (long long j = gtid(); j < np; j += gstride()) {
    const double t = ldcg(y + j);
    if (j < p) sv += t * t; else sl += t * t;
  }
  const double v3[3] = {sx, sv, sl};
  const int sl3[3] = {S_EGM_X, S_EGM_V, S_EGM_L};
  put_partials(K, S, v3, sl3);
}

// z - s F(w) from the point z (parity zc) and F's pieces at w (parity wc,
// gradient gx in w.gxs, multipliers of w staged in smem for A^T v): primal
// part into x[dst]; dual part (before the ball) into ytr, ball-norm partials
__device__ void egm_step_point(const KArgs& K, Sm& S, int zc, int wc, int dst) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  const int n = P.n, p = P.p, m = P.m, np = p + m;
  const double s = K.rc.egm_s;
  double* v_s = S.stage;
  double* lam_s = S.stage + p;
  stage_dual(K, w.y + (long long)wc * np, BallScale{1.0, 1.0, 0, 0}, v_s, lam_s);
  const double* xz = w.x + (long long)zc * n;
  double* xd = w.x + (long long)dst * n;
  for (long long j = gtid(); j < n; j += gstride()) {
    double gx = ldcg(w.gxs + j);
    if (p > 0) gx = gx + atv(K, v_s, j);
    xd[j] = clipd(ldcg(xz + j) - s * gx, __ldg(P.lo + j), __ldg(P.hi + j));
  }
  const double* yz = w.y + (long long)zc * np;
  const double* eqw = w.eqv + (long long)wc * p;
  const double* gvw = w.gval + (long long)wc * (m + 1);
  double nv = 0.0, nl = 0.0;
  for (long long j = gtid(); j < np; j += gstride()) {
    const double gy = j < p ? ldcg(eqw + j) : ldcg(gvw + (j - p + 1));
    double t = ldcg(yz + j) + s * gy;
    if (j >= p) t = fmax(t, 0.0);
    w.ytr[j] = t;
    if (j < p) nv += t * t; else nl += t * t;
  }
  const double v2[2] = {nv, nl};
  const int sl[2] = {S_BALL_V, S_BALL_L};
  put_partials(K, S, v2, sl);
}

// ytr -> y[dst] through the dual ball (geometry.py:263-311)
__device__ __forceinline__ void egm_ball(const KArgs& K, Sm& S, int dst) {
  const int p = K.P.p, np = p + K.P.m;
  const BallScale bs = ball_from_slots(K, S, S_BALL_V, S_BALL_L);
  double* yd = K.w.y + (long long)dst * np;
  for (long long j = gtid(); j < np; j += gstride()) {
    const double v = ldcg(K.w.ytr + j);
    yd[j] = j < p ? (bs.av ? bs.sv * v : v) : (bs.al ? bs.sl * v : v);
  }
}

// grad_x Phi partial at parity par (multipliers of that point) -> w.gxs
__device__ __forceinline__ bool egm_gx(const KArgs& K, Sm& S, int par) {
  const DevProblem& P = K.P;
  const double* y = K.w.y + (long long)par * (P.p + P.m);
  double* v_s = S.stage;
  double* lam_s = S.stage + P.p;
  stage_dual(K, y, BallScale{1.0, 1.0, 0, 0}, v_s, lam_s);
  return gx_part(K, S, par, y + P.p, lam_s, K.w.gxs);
}

__device__ __noinline__ int egm_step(const KArgs& K, Sm& S, int step, int& xk) {
  SolverState& st = *S.st;
  const Work& w = K.w;
  const int n = K.P.n, np = K.P.p + K.P.m;
  switch (step) {
    case E_INIT: {   // |z0| (egm.py:52), zero the sums
      egm_norm_partials(K, S, st.cur);
      for (long long j = gtid(); j < n; j += gstride()) w.xcum[j] = 0.0;
      for (long long j = gtid(); j < np; j += gstride()) w.ycum[j] = 0.0;
      if (!gsync(K, S)) return kAbort;
      const int sl3[3] = {S_EGM_X, S_EGM_V, S_EGM_L};
      get_totals(K, S, sl3);
      if (threadIdx.x == 0) {
        st.gap[0] = sqrt((S.tot[S_EGM_X] + S.tot[S_EGM_V]) + S.tot[S_EGM_L]);   // |z0|
        st.call_done = 0;
        st.T = 0.0;
        st.fail_iter = 0;   // 1 once diverged
      }
      __syncthreads();
      return E_GX;
    }
    case E_GX:       // F(z): grad_x at z (the U-cache at cur)
      if (!egm_gx(K, S, st.cur)) return kAbort;
      xk = X_GX;
      return E_HALF;
    case E_HALF:     // z~ = Pi(z - s F(z)) -> parity cur^1
      egm_step_point(K, S, st.cur, st.cur, st.cur ^ 1);
      return gsync(K, S) ? E_HSWEEP : kAbort;
    case E_HSWEEP:
      egm_ball(K, S, st.cur ^ 1);
      return sweep_sync(K, S, w.x + (long long)(st.cur ^ 1) * n, st.cur ^ 1) ? E_HGLOC : kAbort;
    case E_HGLOC:
      g_local(K, st.cur ^ 1);
      xk = X_G;
      return E_GXH;
    case E_GXH:      // F(z~): grad_x at z~
      if (!egm_gx(K, S, st.cur ^ 1)) return kAbort;
      xk = X_GX;
      return E_PLUS;
    case E_PLUS:     // z+ = Pi(z - s F(z~)) -> parity cur^1 (z~ is no longer needed)
      egm_step_point(K, S, st.cur, st.cur ^ 1, st.cur ^ 1);
      return gsync(K, S) ? E_PSWEEP : kAbort;
    case E_PSWEEP:
      egm_ball(K, S, st.cur ^ 1);
      return sweep_sync(K, S, w.x + (long long)(st.cur ^ 1) * n, st.cur ^ 1) ? E_PGLOC : kAbort;
    case E_PGLOC:
      g_local(K, st.cur ^ 1);
      xk = X_G;
      return E_POST;
    case E_POST: {   // accept z+, ergodic sums, divergence test, trace (egm.py:64-73)
      const int nxt = st.cur ^ 1;
      const double* x = w.x + (long long)nxt * n;
      const double* y = w.y + (long long)nxt * np;
      for (long long j = gtid(); j < n; j += gstride()) w.xcum[j] += ldcg(x + j);
      for (long long j = gtid(); j < np; j += gstride()) w.ycum[j] += ldcg(y + j);
      egm_norm_partials(K, S, nxt);
      if (!gsync(K, S)) return kAbort;
      const int sl3[3] = {S_EGM_X, S_EGM_V, S_EGM_L};
      get_totals(K, S, sl3);
      if (threadIdx.x == 0) {
        st.cur = nxt;
        st.call_done += 1;
        st.T = (double)st.call_done;
        const double zn = sqrt((S.tot[S_EGM_X] + S.tot[S_EGM_V]) + S.tot[S_EGM_L]);
        if (zn > 1e8 * (1.0 + st.gap[0])) st.fail_iter = 1;
        const int te = K.rc.egm_trace_every;
        if (blockIdx.x == 0 && !st.fail_iter && te > 0 && st.call_done % te == 0 && K.w.trace) {
          const long long row = st.call_done / te - 1;
          K.w.trace[row * 2] = (double)st.call_done;
          K.w.trace[row * 2 + 1] = zn;
        }
      }
      __syncthreads();
      return (st.fail_iter || st.call_done >= K.rc.egm_K) ? DONE : E_GX;
    }
    default:
      return kAbort;
  }
}

}  // namespace rapdb
