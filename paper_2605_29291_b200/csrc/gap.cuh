// gap.cuh -- the self-centred smoothed duality gap G_xi(z) on device
// (diagnostics.py:120-163), used by the adaptive restart rule
// (restarts.py:136-161).
//
//   1. candidate z = (x_c, v_c, lam_c) and (Ax_c - b, g(x_c)) -- cached for
//      the current iterate, else one fused Q sweep;
//   2. closed-form dual maximiser y_hat = Pi(y_c + (Ax-b, g)/(2 xi)) and the
//      dual term Phi(x_c, y_hat) - 2 xi D_d(y_hat, y_c);
//   3. H = Q_0 + sum_{lam_i != 0} lam_i Q_i in one pass over the stack (i-order
//      accumulation per entry, as diagnostics.py:145-148);
//   4. L = ||H|| + 2 xi by power iteration (problem.py:47-68, start cos(k+1/2),
//      <= 200 iterations, tolerance 1e-10, x1.01);
//   5. APG with function-value restart (subsolve.py:27-62) on
//      F(z) = 1/2 z'Hz + (c_bar + A'v)'z + (r_bar - v'b) + 2 xi * 1/2 |z - x_c|^2,
//      c_bar = q_0 + sum lam_i q_i, r_bar = r_0 + sum lam_i r_i -- one
//      H-matvec per function/gradient evaluation instead of the reference's
//      full stack re-evaluation.
// Every CTA keeps full copies of the n-vectors in shared memory and computes
// the element-wise updates and the vector dots redundantly (identical code and
// order, hence identical bits); only the matvecs are distributed (one warp
// per row of H) and separated by grid barriers.
#pragma once
#include "solver_ops.cuh"

namespace rapdb {

// total of one value per thread, fixed order, returned to every thread
__device__ __forceinline__ double block_sum(Sm& S, double v) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) S.red[w] = v;
  __syncthreads();
  double s = S.red[0];
  for (int i = 1; i < kWarps; ++i) s += S.red[i];
  return s;
}

// out[r] = (H v)_r for this CTA's rows (one warp per row, v in shared memory);
// returns this thread's share of v'(Hv) (nonzero on lane 0 only)
__device__ double matvec_rows(const KArgs& K, const double* H, const double* v, double* out) {
  const int n = K.P.n;
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const long long nw = (long long)gridDim.x * kWarps;
  double quad = 0.0;
  for (long long r = gw; r < n; r += nw) {
    const double* row = H + r * n;
    double a0 = 0.0, a1 = 0.0;
    int c = lane;
    for (; c + 32 < n; c += 64) {
      a0 = fma(ldcg(row + c), v[c], a0);
      a1 = fma(ldcg(row + c + 32), v[c + 32], a1);
    }
    if (c < n) a0 = fma(ldcg(row + c), v[c], a0);
    const double s = warp_sum(a0 + a1);
    if (lane == 0) {
      out[r] = s;
      quad += v[r] * s;
    }
  }
  return quad;
}

struct GapScratch {
  double *xc, *xa, *yk, *xn, *lin;   // shared-memory n-vectors
};

// F(z) after a matvec: quad total comes from the grid reduction
__device__ __forceinline__ double gap_value(const KArgs& K, Sm& S, const GapScratch& g, const double* z,
                                            double quad, double cst, double xi) {
  const int n = K.P.n;
  double sl = 0.0, sd = 0.0;
  for (int j = threadIdx.x; j < n; j += kThreads) {
    sl += g.lin[j] * z[j];
    const double d = z[j] - g.xc[j];
    sd += d * d;
  }
  const double lin = block_sum(S, sl);
  const double dd = block_sum(S, sd);
  return ((0.5 * quad + lin) + cst) + 2.0 * xi * (0.5 * dd);
}

// distributed z -> H z (into hz) followed by a grid barrier; returns z'Hz
__device__ bool gap_matvec(const KArgs& K, Sm& S, const double* H, const double* z, double* hz, double& quad) {
  const double qp = matvec_rows(K, H, z, hz);
  const double v1[1] = {qp};
  const int sl[1] = {S_GAPQ};
  put_partials(K, S, v1, sl);
  if (!gsync(K, S)) return false;
  get_totals(K, S, sl);
  quad = S.tot[S_GAPQ];
  return true;
}

// dst = clip(src - step * (Hsrc + lin + 2 xi (src - xc)))  (all in shared memory but Hsrc)
__device__ __forceinline__ void gap_pgrad(const KArgs& K, const GapScratch& g, const double* src,
                                          const double* hsrc, double step, double xi, double* dst) {
  const int n = K.P.n;
  for (int j = threadIdx.x; j < n; j += kThreads) {
    const double gr = (ldcg(hsrc + j) + g.lin[j]) + 2.0 * xi * (src[j] - g.xc[j]);
    dst[j] = clipd(src[j] - step * gr, __ldg(K.P.lo + j), __ldg(K.P.hi + j));
  }
}

// G_CAND: choose the candidate parity (st.pad); a point that is not the current
// iterate gets one sweep (its g is then exchanged at G_GLOCAL)
__device__ int g_cand(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, np = p + P.m;
  const int nxt = st.cur ^ 1;
  const bool fresh = K.rc.src != 1 && !(K.rc.src == 2 && !(st.T > 0.0));
  if (threadIdx.x == 0) st.pad = fresh ? nxt : st.cur;
  __syncthreads();
  if (!fresh) return G_HPART;
  const bool avg = K.rc.src == 2;
  for (long long j = gtid(); j < n; j += gstride())
    w.x[(long long)nxt * n + j] = avg ? ldcg(w.xcum + j) / st.T : ldcg(K.rc.in_x + j);
  for (long long j = gtid(); j < np; j += gstride())
    w.y[(long long)nxt * np + j] = avg ? ldcg(w.ycum + j) / st.T
                                        : (j < p ? ldcg(K.rc.in_v + j) : ldcg(K.rc.in_lam + (j - p)));
  if (!gsync(K, S)) return kAbort;
  return sweep_sync(K, S, w.x + (long long)nxt * n, nxt) ? G_GLOCAL : kAbort;
}

// G_HPART: dual term (needs the full g) and this rank's share of H      [X_H]
__device__ int g_hpart(const KArgs& K, Sm& S, int& xk) {
  const DevProblem& P = K.P;
  const DevParams& prm = K.prm;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m, np = p + m;
  const double xi = K.rc.xi;
  const int cp = st.pad;
  const double* xcand = w.x + (long long)cp * n;
  const double* ycand = w.y + (long long)cp * np;
  const double* gvc = w.gval + (long long)cp * (m + 1);
  const double* eqc = w.eqv + (long long)cp * p;
  if (K.rc.out_x)
    for (long long j = gtid(); j < n; j += gstride()) K.rc.out_x[j] = ldcg(xcand + j);

  // ---- 2. dual closed form (every CTA, redundantly, in shared memory)
  double* vh = S.stage;            // (v_hat, lam_hat) raw then projected: np doubles
  double nv = 0.0, nl = 0.0;
  for (int j = threadIdx.x; j < np; j += kThreads) {
    const double gy = j < p ? ldcg(eqc + j) : ldcg(gvc + (j - p + 1));
    double t = ldcg(ycand + j) + gy / (2.0 * xi);
    if (j >= p) t = fmax(t, 0.0);
    vh[j] = t;
    if (j < p) nv += t * t; else nl += t * t;
  }
  const double tv = block_sum(S, nv), tl = block_sum(S, nl);
  const BallScale bs = ball_scale(prm, tv, tl);
  double s_v = 0.0, s_l = 0.0, s_d = 0.0;
  for (int j = threadIdx.x; j < np; j += kThreads) {
    double t = vh[j];
    if (j < p) { if (bs.av) t = bs.sv * t; } else if (bs.al) t = bs.sl * t;
    const double gy = j < p ? ldcg(eqc + j) : ldcg(gvc + (j - p + 1));
    if (j < p) s_v += t * gy; else s_l += t * gy;
    const double d = t - ldcg(ycand + j);
    s_d += d * d;
  }
  const double dv = block_sum(S, s_v), dl = block_sum(S, s_l), ddd = block_sum(S, s_d);
  double phi_hat = ldcg(gvc);
  if (p > 0) phi_hat += dv;
  if (m > 0) phi_hat += dl;
  const double dual_term = phi_hat - 2.0 * xi * (0.5 * ddd);

  // ---- 3. H = Q0 + sum lam_i Q_i (lam = candidate multipliers), one pass
  double* H = w.H;
  {
    const long long ld = P.ld;
    double* lam_s = S.stage;     // staged multipliers (m) -- vh no longer needed
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += kThreads) lam_s[i] = ldcg(ycand + p + i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long gw = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * kWarps;
    constexpr int KC = 16;                  // columns per lane per pass: 16 loads in flight
    // this rank's share: Q0 if held (and not all-zero), then its local Q_i
    const bool q0 = P.k0 == 0 && __ldg(P.mat_slot) >= 0;
    const int i_lo = P.k0 == 0 ? 1 : P.k0;
    if (K.sp.layout == 1) {
      // packed stack: one stored 32 x 32 sub-tile per warp (lane l = column l),
      // the mirrored lower sub-tile written through a per-warp shared transpose
      const sym::Geom& g = K.sp.geom;
      const long long mat_doubles = g.spm * sym::kTD;
      const long long toff = ((long long)m * 8 + 255) / 256 * 256;
      double* tb = reinterpret_cast<double*>(S.ring + toff) + (threadIdx.x >> 5) * (32 * 33);
      for (long long it = gw; it < g.spm; it += nw) {
        int lo = 0, hi = g.upm - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (K.sp.units[mid].off <= it) lo = mid; else hi = mid - 1;
        }
        const sym::Unit un = K.sp.units[lo];
        int rs, cs, sr, sc;
        sym::unit_subtiles(g, un.bi, un.bj, rs, cs);
        sym::unit_sub(un.bi == un.bj, cs, (int)(it - un.off), sr, sc);
        const int R0 = (2 * un.bi + sr) * 32, C0 = (2 * un.bj + sc) * 32;
        double h[32];
        if (q0) {
          const double* t = P.Q + it * sym::kTD + lane;
#pragma unroll
          for (int r = 0; r < 32; ++r) h[r] = __ldg(t + r * 32);
        } else {
#pragma unroll
          for (int r = 0; r < 32; ++r) h[r] = 0.0;
        }
        for (int i = i_lo; i < P.k1; ++i) {
          const double l = lam_s[i - 1];
          if (l == 0.0 || __ldg(P.mat_slot + (i - P.k0)) < 0) continue;   // diagnostics.py:146
          const double* t = P.Q + (long long)(i - P.k0) * mat_doubles + it * sym::kTD + lane;
          double qv[32];
#pragma unroll
          for (int r = 0; r < 32; ++r) qv[r] = __ldg(t + r * 32);
#pragma unroll
          for (int r = 0; r < 32; ++r) h[r] = h[r] + l * qv[r];
        }
        const int c = C0 + lane;
#pragma unroll
        for (int r = 0; r < 32; ++r)
          if (R0 + r < n && c < n) H[(long long)(R0 + r) * n + c] = h[r];
        if (R0 != C0) {
#pragma unroll
          for (int r = 0; r < 32; ++r) tb[r * 33 + lane] = h[r];
          __syncwarp();
          for (int rr = 0; rr < 32; ++rr)
            if (C0 + rr < n && R0 + lane < n) H[(long long)(C0 + rr) * n + R0 + lane] = tb[lane * 33 + rr];
          __syncwarp();
        }
      }
    }
    for (long long r = gw; r < n && K.sp.layout == 0; r += nw) {
      for (int cb = 0; cb < n; cb += 32 * KC) {
        double h[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const int c = cb + lane + 32 * k;
          h[k] = (q0 && c < n) ? __ldg(P.Q + r * ld + c) : 0.0;
        }
        for (int i = i_lo; i < P.k1; ++i) {
          const double l = lam_s[i - 1];
          if (l == 0.0 || __ldg(P.mat_slot + (i - P.k0)) < 0) continue;   // diagnostics.py:146
          const double* qi = P.Q + ((long long)(i - P.k0) * n + r) * ld;
          double qv[KC];
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const int c = cb + lane + 32 * k;
            qv[k] = c < n ? __ldg(qi + c) : 0.0;
          }
#pragma unroll
          for (int k = 0; k < KC; ++k) h[k] = h[k] + l * qv[k];
        }
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const int c = cb + lane + 32 * k;
          if (c < n) H[r * n + c] = h[k];
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) st.gap[5] = dual_term;
  __syncthreads();
  xk = X_H;
  return G_SOLVE;
}

// G_SOLVE: ||H|| by power iteration, then the APG subsolver; writes st.gap
__device__ int g_solve(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m;
  const double xi = K.rc.xi;
  const int cp = st.pad;
  const double* xcand = w.x + (long long)cp * n;
  const double* ycand = w.y + (long long)cp * (p + m);
  const double dual_term = st.gap[5];
  double* H = w.H;
  // c_bar + A'v (shared), r_bar - v'b (scalar); q, r are replicated on every rank
  double* V = reinterpret_cast<double*>(S.xs);   // xs + ring: >= 5n doubles (checked at bind)
  GapScratch g{V, V + n, V + 2 * n, V + 3 * n, V + 4 * n};
  double* lam_s = S.stage + 5 * n;               // after the five vectors
  for (int i = threadIdx.x; i < m; i += kThreads) lam_s[i] = ldcg(ycand + p + i);
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += kThreads) {
    double c = __ldg(P.q + j);
    for (int i = 1; i <= m; ++i) {
      const double l = lam_s[i - 1];
      if (l != 0.0) c = c + l * __ldg(P.q + (long long)i * n + j);
    }
    if (p > 0) {
      double t = 0.0;
      for (int l2 = 0; l2 < p; ++l2) t = t + __ldg(P.A + (long long)l2 * n + j) * ldcg(ycand + l2);
      c = c + t;
    }
    g.lin[j] = c;
    g.xc[j] = ldcg(xcand + j);
  }
  double cst = __ldg(P.r);
  for (int i = 1; i <= m; ++i) {
    const double l = lam_s[i - 1];
    if (l != 0.0) cst = cst + l * __ldg(P.r + i);
  }
  if (p > 0) {
    double vb = 0.0;
    for (int l2 = 0; l2 < p; ++l2) vb += ldcg(ycand + l2) * __ldg(P.b + l2);
    cst = cst - vb;
  }
  __syncthreads();

  // ---- 4. power iteration on H'H (H symmetric): L = 1.01 * sqrt(|H H v|)
  double* T = w.hx;      // scratch n-vectors in global memory
  double* W2 = w.hxn;
  double prev = 0.0;
  {
    double* pv = g.xa;
    double* tv2 = g.yk;
    double s = 0.0;
    for (int j = threadIdx.x; j < n; j += kThreads) {
      const double c = cos((double)j + 0.5);
      pv[j] = c;
      s += c * c;
    }
    const double nv0 = sqrt(block_sum(S, s));
    for (int j = threadIdx.x; j < n; j += kThreads) pv[j] = pv[j] / nv0;
    __syncthreads();
    for (int it = 0; it < 200; ++it) {
      double q;
      if (!gap_matvec(K, S, H, pv, T, q)) return kAbort;
      for (int j = threadIdx.x; j < n; j += kThreads) tv2[j] = ldcg(T + j);
      __syncthreads();
      if (!gap_matvec(K, S, H, tv2, W2, q)) return kAbort;
      double s2 = 0.0;
      for (int j = threadIdx.x; j < n; j += kThreads) {
        const double wj = ldcg(W2 + j);
        s2 += wj * wj;
      }
      const double nrm = sqrt(block_sum(S, s2));
      if (nrm == 0.0) { prev = 0.0; break; }
      for (int j = threadIdx.x; j < n; j += kThreads) pv[j] = ldcg(W2 + j) / nrm;
      __syncthreads();
      const double est = sqrt(nrm);
      const bool done = fabs(est - prev) <= 1e-10 * fmax(est, 1.0);
      prev = est;
      if (done) break;
    }
  }
  const double L = 1.01 * prev + 2.0 * xi;

  // ---- 5. APG with function-value restart (subsolve.py:44-62)
  const double step = 1.0 / L;
  const double tol = K.rc.tol;
  const int max_iter = 50000;
  double* hx = w.hx;     // H x   (current APG x)
  double* hxn = w.hxn;   // H x_new
  double* hy = w.hy;     // H yk
  for (int j = threadIdx.x; j < n; j += kThreads) {
    const double x0 = K.rc.warm ? ldcg(K.rc.warm + j) : g.xc[j];
    const double xv = clipd(x0, __ldg(P.lo + j), __ldg(P.hi + j));
    g.xa[j] = xv;
    g.yk[j] = xv;
  }
  __syncthreads();
  double quad;
  if (!gap_matvec(K, S, H, g.xa, hx, quad)) return kAbort;
  double fx = gap_value(K, S, g, g.xa, quad, cst, xi);
  const double* hyk = hx;   // yk == x at the start
  double t = 1.0, residual = 0.0;
  int its = max_iter, conv = 0;
  bool finished = false;
  for (int it = 1; it <= max_iter; ++it) {
    gap_pgrad(K, g, g.yk, hyk, step, xi, g.xn);
    __syncthreads();
    if (!gap_matvec(K, S, H, g.xn, hxn, quad)) return kAbort;
    double fn = gap_value(K, S, g, g.xn, quad, cst, xi);
    if (fn > fx + 1e-12 * (1.0 + fabs(fx))) {
      gap_pgrad(K, g, g.xa, hx, step, xi, g.xn);
      __syncthreads();
      if (!gap_matvec(K, S, H, g.xn, hxn, quad)) return kAbort;
      fn = gap_value(K, S, g, g.xn, quad, cst, xi);
      t = 1.0;
    }
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    const double mom = (t - 1.0) / tn;
    for (int j = threadIdx.x; j < n; j += kThreads) {
      const double xnj = g.xn[j];
      g.yk[j] = xnj + mom * (xnj - g.xa[j]);
      g.xa[j] = xnj;
    }
    __syncthreads();
    {
      double* tmp = hx; hx = hxn; hxn = tmp;   // H x follows x (identical in every CTA)
    }
    fx = fn;
    t = tn;
    if (it % 10 == 0 || it == max_iter) {
      double sr = 0.0;
      for (int j = threadIdx.x; j < n; j += kThreads) {
        const double gr = (ldcg(hx + j) + g.lin[j]) + 2.0 * xi * (g.xa[j] - g.xc[j]);
        const double d = g.xa[j] - clipd(g.xa[j] - step * gr, __ldg(P.lo + j), __ldg(P.hi + j));
        sr += d * d;
      }
      residual = sqrt(block_sum(S, sr));
      if (residual <= tol) {
        its = it;
        conv = 1;
        finished = true;
        break;
      }
    }
    if (!gap_matvec(K, S, H, g.yk, hy, quad)) return kAbort;
    hyk = hy;
  }
  if (!finished) {
    its = max_iter;
    conv = residual <= tol ? 1 : 0;
  }
  // primal_term = value(x_sol) == fx (same arithmetic on the same point)
  if (threadIdx.x == 0) {
    st.gap[0] = dual_term - fx;
    st.gap[1] = (double)its;
    st.gap[2] = residual;
    st.gap[3] = (double)conv;
    st.gap[4] = L;
    st.gap[5] = dual_term;
  }
  __syncthreads();
  return DONE;
}

}  // namespace rapdb
