// solver_ops.cuh -- phases of the rAPDB iteration on top of solver_kernel.cuh.
//
// Per backtracking trial (APDB-yx, engine.py:181-194 + :151-163):
//   P1 dual momentum + orthant projection          -> ytr          (+ball norms)
//   P2 ball scale, grad_x Phi(x_k, y_new) from the U-cache, primal step + box
//      projection, partials of D_p, <gx, dx>, D_d, Phi(z_mix) terms
//   P3 fused Q sweep at x_new                       -> U_new, segment sums
//   P4 g(x_new), Ax_new-b, gy_new, partials of |dgy|^2 and Phi(z_new) terms
//   P5 every CTA: fixed-order totals -> E and the acceptance test (engine.py:219)
// APDB-xy (engine.py:167-179 + :140-149) runs primal step / sweep / dual step /
// two gradient recombinations / decide in the same five-phase shape.
#pragma once
#include "solver_kernel.cuh"

namespace rapdb {

__device__ __forceinline__ bool sweep_sync(const KArgs& K, Sm& S, const double* xsrc, int par) {
  unsigned long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) t0 = globaltimer();
  sweep(K, S, xsrc, par);
  const bool ok = gsync(K, S);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long t1 = globaltimer();
    if (t1 > t0) S.st->sweep_ns += (double)(t1 - t0);   // skip a driver re-sync jump
    S.st->sweeps += 1;
  }
  return ok;
}

// ------------------------------------------------------------------ reinit
// engine.py:102-136: project the point, reset the stepsize recursion, refresh
// the caches at the (new) point with one sweep, zero the ergodic sums.
__device__ bool dev_reinit(const KArgs& K, Sm& S, int src, int warm_tau) {
  const DevProblem& P = K.P;
  const DevParams& prm = K.prm;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m, np = p + m;
  const int cur = st.cur, nxt = cur ^ 1;
  const bool avg = (src == 2) && st.T > 0.0;
  const double T = st.T;
  const double* xc = w.x + (long long)cur * n;
  const double* yc = w.y + (long long)cur * np;
  double* xn = w.x + (long long)nxt * n;
  for (long long j = gtid(); j < n; j += gstride()) {
    const double v = src == 0 ? ldcg(K.rc.in_x + j) : (avg ? ldcg(w.xcum + j) / T : ldcg(xc + j));
    xn[j] = clipd(v, __ldg(P.lo + j), __ldg(P.hi + j));
  }
  double nv = 0.0, nl = 0.0;
  for (long long j = gtid(); j < np; j += gstride()) {
    double v = src == 0 ? (j < p ? ldcg(K.rc.in_v + j) : ldcg(K.rc.in_lam + (j - p)))
                        : (avg ? ldcg(w.ycum + j) / T : ldcg(yc + j));
    if (j >= p) v = fmax(v, 0.0);
    w.ytr[j] = v;
    if (j < p) nv += v * v; else nl += v * v;
  }
  {
    const double v2[2] = {nv, nl};
    const int sl[2] = {S_AVG_V, S_AVG_L};
    put_partials(K, S, v2, sl);
  }
  if (!gsync(K, S)) return false;
  {
    const int sl[2] = {S_AVG_V, S_AVG_L};
    get_totals(K, S, sl);
  }
  const BallScale bs = ball_scale(prm, S.tot[S_AVG_V], S.tot[S_AVG_L]);
  double* yn = w.y + (long long)nxt * np;
  for (long long j = gtid(); j < np; j += gstride()) {
    const double v = ldcg(w.ytr + j);
    yn[j] = j < p ? (bs.av ? bs.sv * v : v) : (bs.al ? bs.sl * v : v);
  }
  if (!sweep_sync(K, S, xn, nxt)) return false;
  double pv = 0.0, pl = 0.0;
  double* gvn = w.gval + (long long)nxt * (m + 1);
  for (long long idx = gtid(); idx <= np; idx += gstride()) {
    if (idx < np) {
      double gyv;
      if (idx < p) {
        gyv = ldcg(w.eqv + (long long)nxt * p + idx);
      } else {
        gyv = g_combine(K, (int)(idx - p + 1));
        gvn[idx - p + 1] = gyv;
      }
      if (prm.mode == 0) {
        w.gy[(long long)st.ig_cur * np + idx] = gyv;
        w.gy[(long long)st.ig_prev * np + idx] = gyv;
      }
      const double yv = ldcg(yn + idx);
      if (idx < p) pv += yv * gyv; else pl += yv * gyv;
    } else {
      gvn[0] = g_combine(K, 0);
    }
  }
  for (long long j = gtid(); j < n; j += gstride()) w.xcum[j] = 0.0;
  for (long long j = gtid(); j < np; j += gstride()) w.ycum[j] = 0.0;
  {
    const double v2[2] = {pv, pl};
    const int sl[2] = {S_PHIV, S_PHIL};
    put_partials(K, S, v2, sl);
  }
  if (!gsync(K, S)) return false;
  if (prm.mode == 1) {   // xy caches: gx_cur = gx_prev = grad_x Phi(z)
    double* v_s = S.stage;
    double* lam_s = S.stage + p;
    stage_dual(K, yn, BallScale{1.0, 1.0, 0, 0}, v_s, lam_s);
    const double* Un = w.U + (long long)nxt * P.nloc * n;
    for (long long j = gtid(); j < n; j += gstride()) {
      const double gx = recombine(K, Un, lam_s, v_s, j);
      w.gxb[(long long)st.ig_cur * n + j] = gx;
      w.gxb[(long long)st.ig_prev * n + j] = gx;
    }
    if (!gsync(K, S)) return false;
  }
  {
    const int sl[2] = {S_PHIV, S_PHIL};
    get_totals(K, S, sl);
  }
  if (threadIdx.x == 0) {
    st.cur = nxt;
    double phi = ldcg(gvn);
    if (p > 0) phi += S.tot[S_PHIV];
    if (m > 0) phi += S.tot[S_PHIL];
    st.phi_k = phi;
    const double tau0 = warm_tau ? st.tau_cand : prm.tau_bar;
    st.tau_cand = tau0;
    st.tau_prev = tau0;
    st.gamma = prm.gamma0;
    st.sigma_prev = prm.gamma0 * tau0;
    if (prm.mode == 1) {
      st.alpha = prm.c_alpha / tau0;
      st.beta = prm.c_beta / tau0;
    } else {
      st.alpha = prm.c_alpha / st.sigma_prev;
      st.beta = 0.0;
    }
    st.has_sigma0 = 0;
    st.sigma0 = 0.0;
    st.T = 0.0;
  }
  __syncthreads();
  return true;
}

// --------------------------------------------------------------------- KKT
// diagnostics.py:96-113 (orthant cone): stat = |x - Pi_X(x - grad_x Phi)|,
// eq = |Ax-b|, comp = |min(lam, -g)|, infeas = sqrt(|Ax-b|^2 + |max(g,0)|^2).
__device__ bool dev_kkt(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m, np = p + m;
  const int cur = st.cur;
  const double* yc = w.y + (long long)cur * np;
  double* v_s = S.stage;
  double* lam_s = S.stage + p;
  stage_dual(K, yc, BallScale{1.0, 1.0, 0, 0}, v_s, lam_s);
  const double* Uc = w.U + (long long)cur * P.nloc * n;
  const double* xc = w.x + (long long)cur * n;
  const double* gvc = w.gval + (long long)cur * (m + 1);
  double s_st = 0.0, s_eq = 0.0, s_comp = 0.0, s_gp2 = 0.0, s_gp1 = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) {
    const double gx = recombine(K, Uc, lam_s, v_s, j);
    const double xj = ldcg(xc + j);
    const double d = xj - clipd(xj - gx, __ldg(P.lo + j), __ldg(P.hi + j));
    s_st += d * d;
  }
  for (long long idx = gtid(); idx < np; idx += gstride()) {
    if (idx < p) {
      const double e = ldcg(w.eqv + (long long)cur * p + idx);
      s_eq += e * e;
    } else {
      const double g = ldcg(gvc + (idx - p + 1));
      const double c = fmin(lam_s[idx - p], -g);
      s_comp += c * c;
      const double gp = fmax(g, 0.0);
      s_gp2 += gp * gp;
      s_gp1 += gp;
    }
  }
  {
    const double v5[5] = {s_st, s_eq, s_comp, s_gp2, s_gp1};
    const int sl[5] = {S_STAT, S_EQ2, S_COMP, S_GPOS2, S_GPOS1};
    put_partials(K, S, v5, sl);
    if (!gsync(K, S)) return false;
    get_totals(K, S, sl);
  }
  if (threadIdx.x == 0) {
    const double stat = sqrt(S.tot[S_STAT]);
    const double eq = sqrt(S.tot[S_EQ2]);
    const double comp = m > 0 ? sqrt(S.tot[S_COMP]) : 0.0;
    const double infeas = sqrt(S.tot[S_EQ2] + S.tot[S_GPOS2]);
    const double mpv = m > 0 ? S.tot[S_GPOS1] / (double)m : 0.0;
    const double f = ldcg(gvc);
    st.metrics[0] = (stat + eq) + comp;
    st.metrics[1] = stat;
    st.metrics[2] = eq;
    st.metrics[3] = comp;
    st.metrics[4] = infeas;
    st.metrics[5] = f;
    st.metrics[6] = mpv;
    st.metrics[7] = K.rc.has_f_star ? f - K.rc.f_star : __longlong_as_double(0x7ff8000000000000ll);
    st.has_metrics = 1;
  }
  __syncthreads();
  return true;
}

// check_termination (diagnostics.py:252-263)
__device__ __forceinline__ bool terminated(const RunCfg& rc, const double* met) {
  if (rc.criterion == 2 && rc.has_f_star) {
    const double rel = fabs(met[5] - rc.f_star) / (1.0 + fabs(rc.f_star));
    return fmax(rel, met[6]) <= rc.eps;
  }
  return met[0] <= rc.eps_kkt && met[4] <= rc.eps_feas;
}

// ------------------------------------------------------------- yx trial
// returns 1 accept, 0 reject, -1 abort; accepted-step values in S.tot[NSLOT..]
struct TrialOut { double sigma, alpha_n, beta_n, phi_new; };

__device__ int trial_yx(const KArgs& K, Sm& S, double tau, double slack, TrialOut& out) {
  const DevProblem& P = K.P;
  const DevParams& prm = K.prm;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m, np = p + m;
  const int cur = st.cur, nxt = cur ^ 1;
  const double sigma = st.gamma * tau;
  const double alpha_n = prm.c_alpha / sigma;
  const double theta = st.sigma_prev / sigma;
  const double* yc = w.y + (long long)cur * np;
  const double* gc = w.gy + (long long)st.ig_cur * np;
  const double* gp = w.gy + (long long)st.ig_prev * np;
  // P1: y_trial = y + sigma*((1+theta) gy_cur - theta gy_prev); lam <- max(., 0)
  double nv = 0.0, nl = 0.0;
  for (long long j = gtid(); j < np; j += gstride()) {
    const double t1 = (1.0 + theta) * ldcg(gc + j);
    const double t2 = theta * ldcg(gp + j);
    double yt = ldcg(yc + j) + sigma * (t1 - t2);
    if (j >= p) yt = fmax(yt, 0.0);
    w.ytr[j] = yt;
    if (j < p) nv += yt * yt; else nl += yt * yt;
  }
  if (prm.ball) {
    const double v2[2] = {nv, nl};
    const int sl[2] = {S_BALL_V, S_BALL_L};
    put_partials(K, S, v2, sl);
  }
  if (!gsync(K, S)) return -1;
  // P2
  BallScale bs{1.0, 1.0, 0, 0};
  if (prm.ball) {
    const int sl[2] = {S_BALL_V, S_BALL_L};
    get_totals(K, S, sl);
    bs = ball_scale(prm, S.tot[S_BALL_V], S.tot[S_BALL_L]);
  }
  double* v_s = S.stage;
  double* lam_s = S.stage + p;
  stage_dual(K, w.ytr, bs, v_s, lam_s);
  const double* Uc = w.U + (long long)cur * P.nloc * n;
  const double* xc = w.x + (long long)cur * n;
  double* xn = w.x + (long long)nxt * n;
  double s_dp = 0.0, s_gd = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) {
    const double gx = recombine(K, Uc, lam_s, v_s, j);
    w.gxs[j] = gx;
    const double xj = ldcg(xc + j);
    const double xnj = clipd(xj - tau * gx, __ldg(P.lo + j), __ldg(P.hi + j));
    xn[j] = xnj;
    const double d = xnj - xj;
    s_dp += d * d;
    s_gd += gx * d;
  }
  double s_dd = 0.0, s_mv = 0.0, s_ml = 0.0;
  double* yn = w.y + (long long)nxt * np;
  const double* gvc = w.gval + (long long)cur * (m + 1);
  for (long long j = gtid(); j < np; j += gstride()) {
    const double yv = j < p ? v_s[j] : lam_s[j - p];
    yn[j] = yv;
    const double d = yv - ldcg(yc + j);
    s_dd += d * d;
    if (j < p) s_mv += yv * ldcg(w.eqv + (long long)cur * p + j);
    else s_ml += yv * ldcg(gvc + (j - p + 1));
  }
  {
    const double v5[5] = {s_dp, s_gd, s_dd, s_mv, s_ml};
    const int sl[5] = {S_DP, S_GXDX, S_DD, S_MIXV, S_MIXL};
    put_partials(K, S, v5, sl);
  }
  if (!gsync(K, S)) return -1;
  // P3: sweep at x_new
  if (!sweep_sync(K, S, xn, nxt)) return -1;
  // P4: g(x_new), gy_new, |gy_new - gy_cur|^2, Phi(z_new) terms
  double s_dg = 0.0, s_nv = 0.0, s_nl = 0.0;
  double* gvn = w.gval + (long long)nxt * (m + 1);
  double* gnew = w.gy + (long long)st.ig_new * np;
  for (long long idx = gtid(); idx <= np; idx += gstride()) {
    if (idx < np) {
      double gyv;
      if (idx < p) {
        gyv = ldcg(w.eqv + (long long)nxt * p + idx);
      } else {
        gyv = g_combine(K, (int)(idx - p + 1));
        gvn[idx - p + 1] = gyv;
      }
      gnew[idx] = gyv;
      const double d = gyv - ldcg(gc + idx);
      s_dg += d * d;
      const double yv = ldcg(yn + idx);
      if (idx < p) s_nv += yv * gyv; else s_nl += yv * gyv;
    } else {
      gvn[0] = g_combine(K, 0);
    }
  }
  {
    const double v3[3] = {s_dg, s_nv, s_nl};
    const int sl[3] = {S_DGY, S_NEWV, S_NEWL};
    put_partials(K, S, v3, sl);
  }
  if (!gsync(K, S)) return -1;
  // P5: decide (identically in every CTA)
  {
    const int sl[8] = {S_DP, S_GXDX, S_DD, S_MIXV, S_MIXL, S_DGY, S_NEWV, S_NEWL};
    get_totals(K, S, sl);
  }
  if (threadIdx.x == 0) {
    const double D_p = 0.5 * S.tot[S_DP];
    const double D_d = 0.5 * S.tot[S_DD];
    double phi_new = ldcg(gvn);
    if (p > 0) phi_new += S.tot[S_NEWV];
    if (m > 0) phi_new += S.tot[S_NEWL];
    double phi_mix = ldcg(gvc);
    if (p > 0) phi_mix += S.tot[S_MIXV];
    if (m > 0) phi_mix += S.tot[S_MIXL];
    const double lin = (phi_new - phi_mix) - S.tot[S_GXDX];
    const double nrm = sqrt(S.tot[S_DGY]);
    const double E = ((lin - D_p / tau) + (nrm * nrm) / (2.0 * alpha_n))
                     - (1.0 / sigma - theta * st.alpha) * D_d;
    const double rhs = ((-(prm.delta / tau)) * D_p - (prm.delta / sigma) * D_d) + slack;
    S.flag[1] = (E <= rhs) ? 1 : 0;
    S.tot[NSLOT] = phi_new;   // scratch slot (S_AVG_L unused here)
  }
  __syncthreads();
  out.sigma = sigma;
  out.alpha_n = alpha_n;
  out.beta_n = 0.0;
  out.phi_new = S.tot[NSLOT];
  return S.flag[1];
}

// ------------------------------------------------------------- xy trial
__device__ int trial_xy(const KArgs& K, Sm& S, double tau, double slack, TrialOut& out) {
  const DevProblem& P = K.P;
  const DevParams& prm = K.prm;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m, np = p + m;
  const int cur = st.cur, nxt = cur ^ 1;
  const double sigma = st.gamma * tau;
  const double alpha_n = prm.c_alpha / tau;
  const double beta_n = prm.gamma0 * prm.c_beta / sigma;
  const double theta = st.sigma_prev / sigma;
  const double* gc = w.gxb + (long long)st.ig_cur * n;
  const double* gp = w.gxb + (long long)st.ig_prev * n;
  const double* xc = w.x + (long long)cur * n;
  double* xn = w.x + (long long)nxt * n;
  // P1: x_new = Pi_X(x - tau*((1+theta) gx_cur - theta gx_prev))
  double s_dp = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) {
    const double t1 = (1.0 + theta) * ldcg(gc + j);
    const double t2 = theta * ldcg(gp + j);
    const double xj = ldcg(xc + j);
    const double xnj = clipd(xj - tau * (t1 - t2), __ldg(P.lo + j), __ldg(P.hi + j));
    xn[j] = xnj;
    const double d = xnj - xj;
    s_dp += d * d;
  }
  {
    const double v1[1] = {s_dp};
    const int sl[1] = {S_DP};
    put_partials(K, S, v1, sl);
  }
  if (!gsync(K, S)) return -1;
  // P2: sweep at x_new
  if (!sweep_sync(K, S, xn, nxt)) return -1;
  // P3: dual step with g(x_new)
  const double* yc = w.y + (long long)cur * np;
  double* gvn = w.gval + (long long)nxt * (m + 1);
  double nv = 0.0, nl = 0.0;
  for (long long idx = gtid(); idx <= np; idx += gstride()) {
    if (idx < np) {
      double gyv;
      if (idx < p) {
        gyv = ldcg(w.eqv + (long long)nxt * p + idx);
      } else {
        gyv = g_combine(K, (int)(idx - p + 1));
        gvn[idx - p + 1] = gyv;
      }
      double yt = ldcg(yc + idx) + sigma * gyv;
      if (idx >= p) yt = fmax(yt, 0.0);
      w.ytr[idx] = yt;
      if (idx < p) nv += yt * yt; else nl += yt * yt;
    } else {
      gvn[0] = g_combine(K, 0);
    }
  }
  if (prm.ball) {
    const double v2[2] = {nv, nl};
    const int sl[2] = {S_BALL_V, S_BALL_L};
    put_partials(K, S, v2, sl);
  }
  if (!gsync(K, S)) return -1;
  // P4: two recombinations at x_new (y_k and y_new), D_d, Phi(z_new) terms
  BallScale bs{1.0, 1.0, 0, 0};
  if (prm.ball) {
    const int sl[2] = {S_BALL_V, S_BALL_L};
    get_totals(K, S, sl);
    bs = ball_scale(prm, S.tot[S_BALL_V], S.tot[S_BALL_L]);
  }
  double* v_n = S.stage;
  double* lam_n = S.stage + p;
  double* v_k = S.stage + np;
  double* lam_k = S.stage + np + p;
  stage_dual(K, w.ytr, bs, v_n, lam_n);
  stage_dual(K, yc, BallScale{1.0, 1.0, 0, 0}, v_k, lam_k);
  const double* Un = w.U + (long long)nxt * P.nloc * n;
  double* gnew = w.gxb + (long long)st.ig_new * n;
  double s1 = 0.0, s2 = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) {
    const double gyk = recombine(K, Un, lam_k, v_k, j);
    const double gn = recombine(K, Un, lam_n, v_n, j);
    w.gxs[j] = gyk;
    gnew[j] = gn;
    const double d1 = gn - gyk;
    s1 += d1 * d1;
    const double d2 = gyk - ldcg(gc + j);
    s2 += d2 * d2;
  }
  double s_dd = 0.0, s_nv = 0.0, s_nl = 0.0;
  double* yn = w.y + (long long)nxt * np;
  for (long long j = gtid(); j < np; j += gstride()) {
    const double yv = j < p ? v_n[j] : lam_n[j - p];
    yn[j] = yv;
    const double d = yv - ldcg(yc + j);
    s_dd += d * d;
    if (j < p) s_nv += yv * ldcg(w.eqv + (long long)nxt * p + j);
    else s_nl += yv * ldcg(gvn + (j - p + 1));
  }
  {
    const double v5[5] = {s1, s2, s_dd, s_nv, s_nl};
    const int sl[5] = {S_GXD1, S_GXD2, S_DD, S_NEWV, S_NEWL};
    put_partials(K, S, v5, sl);
  }
  if (!gsync(K, S)) return -1;
  // P5: decide
  {
    const int sl[6] = {S_DP, S_GXD1, S_GXD2, S_DD, S_NEWV, S_NEWL};
    get_totals(K, S, sl);
  }
  if (threadIdx.x == 0) {
    const double D_p = 0.5 * S.tot[S_DP];
    const double D_d = 0.5 * S.tot[S_DD];
    const double n1 = sqrt(S.tot[S_GXD1]);
    const double n2 = sqrt(S.tot[S_GXD2]);
    const double E = (((n1 * n1) / (2.0 * alpha_n) - D_d / sigma) + (n2 * n2) / (2.0 * beta_n))
                     - (1.0 / tau - theta * (st.alpha + st.beta)) * D_p;
    const double rhs = ((-(prm.delta / tau)) * D_p - (prm.delta / sigma) * D_d) + slack;
    double phi_new = ldcg(gvn);
    if (p > 0) phi_new += S.tot[S_NEWV];
    if (m > 0) phi_new += S.tot[S_NEWL];
    S.flag[1] = (E <= rhs) ? 1 : 0;
    S.tot[NSLOT] = phi_new;
  }
  __syncthreads();
  out.sigma = sigma;
  out.alpha_n = alpha_n;
  out.beta_n = beta_n;
  out.phi_new = S.tot[NSLOT];
  return S.flag[1];
}

// ---------------------------------------------------- accepted-step roll
// engine.py:228-249: stepsize recursion, cache rotation, ergodic sums.
__device__ void roll(const KArgs& K, Sm& S, double tau, int evals, const TrialOut& o) {
  const DevParams& prm = K.prm;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = K.P.n, np = K.P.p + K.P.m;
  if (threadIdx.x == 0) {
    const double g_next = st.gamma * (1.0 + K.P.mu * tau);
    const double tau_next = tau * sqrt((st.gamma / g_next) * (1.0 + (prm.c_nm * tau) / st.tau_prev));
    const int ip = st.ig_prev;
    st.ig_prev = st.ig_cur;
    st.ig_cur = st.ig_new;
    st.ig_new = ip;
    st.cur ^= 1;
    st.alpha = o.alpha_n;
    st.beta = o.beta_n;
    st.tau_prev = tau;
    st.tau_cand = tau_next;
    st.sigma_prev = o.sigma;
    st.gamma = g_next;
    if (!st.has_sigma0) {
      st.sigma0 = o.sigma;
      st.has_sigma0 = 1;
    }
    const double t_k = o.sigma / st.sigma0;
    st.T += t_k;
    S.tot[NSLOT + 1] = t_k;
    st.phi_k = o.phi_new;
    st.iters += 1;
    st.evals_total += evals;
    st.inner += 1;
  }
  __syncthreads();
  const double t_k = S.tot[NSLOT + 1];
  const double* xk = w.x + (long long)st.cur * n;
  const double* yk = w.y + (long long)st.cur * np;
  for (long long j = gtid(); j < n; j += gstride()) w.xcum[j] += t_k * ldcg(xk + j);
  for (long long j = gtid(); j < np; j += gstride()) w.ycum[j] += t_k * ldcg(yk + j);
}

}  // namespace rapdb
