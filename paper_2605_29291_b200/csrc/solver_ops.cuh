// solver_ops.cuh -- the rAPDB iteration as a resumable state machine.
//
// Per backtracking trial (APDB-yx, engine.py:181-194 + :151-163):
//   TY_DUAL    dual momentum + orthant projection -> ytr (+ ball norms)
//   TY_GXPART  this rank's share of grad_x Phi(x_k, y_new) from the U-cache   [X_GX]
//   TY_PRIMAL  + A'v, primal step + box projection, partials of D_p, <gx,dx>,
//              D_d and the Phi(z_mix) terms
//   TY_SWEEP   fused Q sweep at x_new (local matrices)
//   TY_GLOCAL  g_i(x_new) for the local matrices, zero elsewhere               [X_G]
//   TY_GY      gy_new, |gy_new - gy_cur|^2 and Phi(z_new) partials
//   TY_DECIDE  every CTA: fixed-order totals -> E and the test (engine.py:219)
// APDB-xy (engine.py:167-179 + :140-149): TX_PRIMAL / TX_SWEEP / TX_GLOCAL [X_G] /
// TX_DUAL / TX_GXPART [X_GX2] / TX_NORMS / TX_DECIDE.
//
// [X_*] marks an exchange point: with constraints sharded over ranks the host
// all-reduces (sums) the named buffer and relaunches the kernel, which resumes
// at the next step (all loop state lives in SolverState).  With one rank the
// partial already is the total and the kernel just continues (a grid barrier
// where the consumer mapping differs).  Single-GPU dense runs never leave the
// kernel; factored runs also stop at each sweep / gradient so the host can run
// them as high-occupancy kernels (SolverState::fq, factored.cuh).
#pragma once
#include "factored.cuh"

namespace rapdb {

__device__ __forceinline__ bool sweep_sync(const KArgs& K, Sm& S, const double* xsrc, int par) {
  unsigned long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) t0 = globaltimer();
  bool ok;
  if (K.P.kind == 1) {   // the host runs the row-pass kernel at the next stop (factored.cuh)
    if (threadIdx.x == 0) {
      SolverState& st = *S.st;
      st.fq[0] = 1;
      st.fq[1] = par;
      st.fq[2] = xsrc == K.rc.in_x ? 1 : 0;
    }
    __syncthreads();
    ok = true;
  } else {
    sweep(K, S, xsrc, par);
    ok = gsync(K, S);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long t1 = globaltimer();
    if (t1 > t0) S.st->sweep_ns += (double)(t1 - t0);   // skip a driver re-sync jump
    S.st->sweeps += 1;
  }
  return ok;
}

constexpr int kAbort = -1;

// ---------------------------------------------------------------- peer exchange
// The in-kernel replacement of the host all-reduce at an exchange point
// (sharded dense runs with peer regions attached, KArgs::px): push this
// rank's partial into slot `rank` of every peer over NVLink, fence, signal
// every peer's flag `rank` with the generation, wait for all R flags of the
// own region, then sum the R slots in rank order (identical bits on every
// rank).  Double-buffered by generation parity: a rank can be at most one
// exchange ahead of any peer (it cannot finish exchange k+1 before every peer
// has signalled k+1, i.e. finished reading exchange k).
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ bool peer_exchange(const KArgs& K, Sm& S, int xk) {
  const PeerX& px = K.px;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const long long n = K.P.n, m = K.P.m;
  double* b0 = w.gxs;
  long long n0 = n;
  double* b1 = nullptr;
  long long n1 = 0;
  if (xk == X_G) { b0 = w.gval + (long long)(st.cur ^ 1) * (m + 1); n0 = m + 1; }
  else if (xk == X_GX2) { b1 = w.gxb + (long long)st.ig_new * n; n1 = n; }
  const long long tot = n0 + n1;
  if (!gsync(K, S)) return false;                 // the partial is complete on this rank
  if (threadIdx.x == 0) st.xgen += 1;
  __syncthreads();
  const unsigned long long gen = st.xgen;
  const long long set = (long long)(gen & 1ull) * px.R * px.S;
  for (long long j = gtid(); j < tot; j += gstride()) {
    const double v = j < n0 ? ldcg(b0 + j) : ldcg(b1 + (j - n0));
    for (int r = 0; r < px.R; ++r) px.slots[r][set + (long long)px.rank * px.S + j] = v;
  }
  __threadfence_system();
  if (!gsync(K, S)) return false;                 // every CTA's pushes are fenced
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int r = 0; r < px.R; ++r) st_release_sys(px.flags[r] + (long long)px.rank * 16, gen);
  if (threadIdx.x == 0) {                         // wait for every peer's push of this generation
    const long long t0 = clock64();
    for (int r = 0; r < px.R; ++r) {
      while (ld_acquire_sys(px.flags[px.rank] + (long long)r * 16) < gen) {
        if (*(volatile int*)K.w.abort_flag) { S.flag[0] = 1; break; }
        if (clock64() - t0 > 60000000000ll) { atomicExch(K.w.abort_flag, 5); S.flag[0] = 1; break; }
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
  if (S.flag[0]) return false;
  const double* mine = px.slots[px.rank] + set;
  for (long long j = gtid(); j < tot; j += gstride()) {
    double s = ldcg(mine + j);
    for (int r = 1; r < px.R; ++r) s += ldcg(mine + (long long)r * px.S + j);
    if (j < n0) b0[j] = s; else b1[j - n0] = s;
  }
  return gsync(K, S);                             // consumers read the sums next
}

__device__ __forceinline__ BallScale ball_from_slots(const KArgs& K, Sm& S, int sv, int sl) {
  if (!K.prm.ball) return BallScale{1.0, 1.0, 0, 0};
  const int s2[2] = {sv, sl};
  get_totals(K, S, s2);
  return ball_scale(K.prm, S.tot[sv], S.tot[sl]);
}

// g_i at parity `par` for this rank's matrices, 0 for the others (summed across ranks: exact)
__device__ __forceinline__ void g_local(const KArgs& K, int par) {
  if (K.P.kind == 1) {   // quadratic rows from the W-cache partials; linear rows came with the sweep
    g_factored(K, par);
    return;
  }
  const DevProblem& P = K.P;
  double* gv = K.w.gval + (long long)par * (P.m + 1);
  const long long gw = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const long long nw = (long long)gridDim.x * kWarps;
  for (long long i = gw; i <= P.m; i += nw) {     // one warp per matrix
    const double v = (i >= P.k0 && i < P.k1) ? g_combine_warp(K, (int)i) : 0.0;
    if ((threadIdx.x & 31) == 0) gv[i] = v;
  }
}

// This rank's share of sum_i lam_i grad g_i(x) + grad f(x) at the cached point
// of parity `par` into out.  Dense: from the U-cache with the staged
// multipliers lam_s; factored: from the W-cache with the global lam_g.
__device__ __forceinline__ bool gx_part(const KArgs& K, Sm& S, int par, const double* lam_g, const double* lam_s,
                                        double* out) {
  const DevProblem& P = K.P;
  if (P.kind == 1) {   // queue it for the host (factored.cuh, fac_grad_*)
    if (threadIdx.x == 0) {
      SolverState& st = *S.st;
      const int np = P.p + P.m;
      const int lid = lam_g == K.w.ytr + P.p ? 0 : lam_g == K.w.y + P.p ? 1 : lam_g == K.w.y + np + P.p ? 2 : 3;
      const int oid = out == K.w.gxs ? 0 : 1;
      const int k = st.fq[0] == 2 ? st.fq[1] : 0;
      st.fq[0] = 2;
      st.fq[1] = k + 1;
      st.fq[2 + 3 * k] = par;
      st.fq[3 + 3 * k] = lid;
      st.fq[4 + 3 * k] = oid;
    }
    __syncthreads();
    return true;
  }
  const double* U = K.w.U + (long long)par * P.nloc * P.n;
  if (K.sp.rc_cols) recombine_cols(K, S, U, lam_s, out);
  else for (long long j = gtid(); j < P.n; j += gstride()) out[j] = recombine_local(K, U, lam_s, j);
  return true;
}

// multiplier j of a dual vector: staged copy (dense) or global y (factored;
// a dual ball has already scaled it there: ball_in_place_fac)
__device__ __forceinline__ double dual_at(const KArgs& K, const double* v_s, const double* lam_s, const double* yg,
                                          long long j) {
  if (K.P.kind == 1) return ldcg(yg + j);
  return j < K.P.p ? v_s[j] : lam_s[j - K.P.p];
}

// ----------------------------------- long-vector variants (factored path)
// C3's vectors are 10^6 (x) and 5 * 10^5 (multipliers) long, and the
// persistent kernel runs 8 warps per SM: the plain grid-stride loops are
// latency bound.  These variants issue four strides' loads before using them
// -- the same per-thread element order, so the same partial sums -- and live
// out of line so the dense path's inlined steps keep their registers.  The
// factored path has p = 0 and reads its multipliers from global memory (a
// dual ball scales them there: ball_in_place_fac).
constexpr int kLV = 4;

// Factored dual ball (geometry.py:263-311; p = 0, so only the multiplier
// block): once the trial multipliers' squared-norm partials are published
// (and a grid barrier passed), every thread scales the entries it wrote
// itself -- the same grid-stride elements -- so the global y~ that the
// gradient gather, the primal step and the test read is already final.
__device__ __noinline__ bool ball_in_place_fac(const KArgs& K, Sm& S) {
  if (!K.prm.ball) return true;
  const BallScale bs = ball_from_slots(K, S, S_BALL_V, S_BALL_L);
  if (!bs.al) return true;
  for (long long j = gtid(); j < K.P.m; j += gstride()) K.w.ytr[j] = bs.sl * K.w.ytr[j];
  return gsync(K, S);
}

__device__ __noinline__ int ty_dual_fac(const KArgs& K, Sm& S) {
  const Work& w = K.w;
  SolverState& st = *S.st;
  if (threadIdx.x == 0) {
    st.sigma = st.gamma * st.tau;
    st.alpha_n = K.prm.c_alpha / st.sigma;
    st.beta_n = 0.0;
    st.theta = st.sigma_prev / st.sigma;
  }
  __syncthreads();
  const long long np = K.P.m;
  const double sigma = st.sigma, theta = st.theta;
  const double* yc = w.y + (long long)st.cur * np;
  const double* gc = w.gy + (long long)st.ig_cur * np;
  const double* gp = w.gy + (long long)st.ig_prev * np;
  const long long G = gstride();
  double nl = 0.0;
  for (long long j0 = gtid(); j0 < np; j0 += kLV * G) {
    double a[kLV], b[kLV], c[kLV];
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < np) { a[t] = ldcg(gc + j); b[t] = ldcg(gp + j); c[t] = ldcg(yc + j); }
    }
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < np) {
        const double t1 = (1.0 + theta) * a[t];
        const double t2 = theta * b[t];
        const double yt = fmax(c[t] + sigma * (t1 - t2), 0.0);
        w.ytr[j] = yt;
        nl += yt * yt;
      }
    }
  }
  if (K.prm.ball) {
    const double v2[2] = {0.0, nl};
    const int sl[2] = {S_BALL_V, S_BALL_L};
    put_partials(K, S, v2, sl);
  }
  if (!gsync(K, S)) return kAbort;
  return ball_in_place_fac(K, S) ? TY_GXPART : kAbort;
}

__device__ __noinline__ int ty_primal_fac(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const long long n = P.n, m = P.m;
  const int cur = st.cur, nxt = cur ^ 1;
  const double tau = st.tau;
  const double* xc = w.x + (long long)cur * n;
  double* xn = w.x + (long long)nxt * n;
  const long long G = gstride();
  double s_dp = 0.0, s_gd = 0.0;
  for (long long j0 = gtid(); j0 < n; j0 += kLV * G) {
    double gx[kLV], xj[kLV], lo[kLV], hi[kLV];
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < n) { gx[t] = ldcg(w.gxs + j); xj[t] = ldcg(xc + j); lo[t] = __ldg(P.lo + j); hi[t] = __ldg(P.hi + j); }
    }
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < n) {
        const double xnj = clipd(xj[t] - tau * gx[t], lo[t], hi[t]);
        xn[j] = xnj;
        const double d = xnj - xj[t];
        s_dp += d * d;
        s_gd += gx[t] * d;
      }
    }
  }
  double s_dd = 0.0, s_ml = 0.0;
  const double* yc = w.y + (long long)cur * m;
  double* yn = w.y + (long long)nxt * m;
  const double* gvc = w.gval + (long long)cur * (m + 1);
  for (long long j0 = gtid(); j0 < m; j0 += kLV * G) {
    double yv[kLV], yo[kLV], gv[kLV];
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < m) { yv[t] = ldcg(w.ytr + j); yo[t] = ldcg(yc + j); gv[t] = ldcg(gvc + (j + 1)); }
    }
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < m) {
        yn[j] = yv[t];
        const double d = yv[t] - yo[t];
        s_dd += d * d;
        s_ml += yv[t] * gv[t];
      }
    }
  }
  const double v5[5] = {s_dp, s_gd, s_dd, 0.0, s_ml};
  const int sl[5] = {S_DP, S_GXDX, S_DD, S_MIXV, S_MIXL};
  put_partials(K, S, v5, sl);
  return gsync(K, S) ? TY_SWEEP : kAbort;
}

// after the fused trial's kernels (x_new, gx, W / g parts at x_new are in
// place): the dual side of ty_primal_fac plus the gradient kernel's per-warp
// partials of D_p and <gx, dx>, dealt to the persistent grid's threads in a
// fixed pattern and reduced with the other partials (fixed order); the
// sweep already ran, so the trial continues at TY_GLOCAL.
__device__ __noinline__ int ty_primal_fac_fused(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const long long m = P.m;
  const int cur = st.cur, nxt = cur ^ 1;
  // thread t of CTA b takes the gradient kernel's warps b + G t, b + G (t + 256), ...
  double s_dp = 0.0, s_gd = 0.0;
  for (long long c = blockIdx.x + (long long)gridDim.x * threadIdx.x; c < P.nfpart; c += gstride()) {
    s_dp += ldcg(w.fpart + c);
    s_gd += ldcg(w.fpart + P.nfpart + c);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) st.sweeps += 1;
  const long long G = gstride();
  double s_dd = 0.0, s_ml = 0.0;
  const double* yc = w.y + (long long)cur * m;
  double* yn = w.y + (long long)nxt * m;
  const double* gvc = w.gval + (long long)cur * (m + 1);
  for (long long j0 = gtid(); j0 < m; j0 += kLV * G) {
    double yv[kLV], yo[kLV], gv[kLV];
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < m) { yv[t] = ldcg(w.ytr + j); yo[t] = ldcg(yc + j); gv[t] = ldcg(gvc + (j + 1)); }
    }
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < m) {
        yn[j] = yv[t];
        const double d = yv[t] - yo[t];
        s_dd += d * d;
        s_ml += yv[t] * gv[t];
      }
    }
  }
  const double v5[5] = {s_dp, s_gd, s_dd, 0.0, s_ml};
  const int sl[5] = {S_DP, S_GXDX, S_DD, S_MIXV, S_MIXL};
  put_partials(K, S, v5, sl);
  return gsync(K, S) ? TY_GLOCAL : kAbort;
}

__device__ __noinline__ int ty_gy_fac(const KArgs& K, Sm& S) {
  const Work& w = K.w;
  SolverState& st = *S.st;
  const long long m = K.P.m;
  const int nxt = st.cur ^ 1;
  const double* gvn = w.gval + (long long)nxt * (m + 1);
  const double* gc = w.gy + (long long)st.ig_cur * m;
  double* gnew = w.gy + (long long)st.ig_new * m;
  const double* yn = w.y + (long long)nxt * m;
  const long long G = gstride();
  double s_dg = 0.0, s_nl = 0.0;
  for (long long j0 = gtid(); j0 < m; j0 += kLV * G) {
    double a[kLV], b[kLV], c[kLV];
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < m) { a[t] = ldcg(gvn + (j + 1)); b[t] = ldcg(gc + j); c[t] = ldcg(yn + j); }
    }
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < m) {
        gnew[j] = a[t];
        const double d = a[t] - b[t];
        s_dg += d * d;
        s_nl += c[t] * a[t];
      }
    }
  }
  const double v3[3] = {s_dg, 0.0, s_nl};
  const int sl[3] = {S_DGY, S_NEWV, S_NEWL};
  put_partials(K, S, v3, sl);
  return gsync(K, S) ? TY_DECIDE : kAbort;
}

// the ergodic sums of roll() for long vectors
__device__ __noinline__ void roll_sums_long(const KArgs& K, double t_k, const double* xk, const double* yk) {
  const Work& w = K.w;
  const long long n = K.P.n, np = K.P.p + K.P.m;
  const long long G = gstride();
  for (long long j0 = gtid(); j0 < n; j0 += kLV * G) {
    double a[kLV], c[kLV];
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < n) { a[t] = ldcg(xk + j); c[t] = ldcg(w.xcum + j); }
    }
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < n) w.xcum[j] = c[t] + t_k * a[t];
    }
  }
  for (long long j0 = gtid(); j0 < np; j0 += kLV * G) {
    double a[kLV], c[kLV];
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < np) { a[t] = ldcg(yk + j); c[t] = ldcg(w.ycum + j); }
    }
#pragma unroll
    for (int t = 0; t < kLV; ++t) {
      const long long j = j0 + t * G;
      if (j < np) w.ycum[j] = c[t] + t_k * a[t];
    }
  }
}

// ------------------------------------------- CTA-local yx dual step (dense)
// With few multipliers every CTA forms the whole trial y~ itself straight into
// its shared staging area (the same bits in every CTA: same inputs, same
// order, the ball sums in a fixed block-level order), so the dual step needs
// no grid barrier and the gradient and primal steps no re-staging.  CTA 0
// also writes y~ (before the ball) to global memory; a sharded run that left
// the kernel at the gradient exchange re-stages from it with the saved sums.
constexpr int kLocalNp = 2048;
__device__ __forceinline__ bool dual_cta_local(const KArgs& K) {
  return K.P.kind == 0 && K.P.p + K.P.m <= kLocalNp;
}
__device__ __forceinline__ bool dual_restage(const KArgs& K) { return K.rc.split && !K.rc.p2p; }

__device__ int ty_dual_local(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const DevParams& prm = K.prm;
  const Work& w = K.w;
  SolverState& st = *S.st;
  if (threadIdx.x == 0) {
    st.sigma = st.gamma * st.tau;
    st.alpha_n = prm.c_alpha / st.sigma;
    st.beta_n = 0.0;
    st.theta = st.sigma_prev / st.sigma;
  }
  __syncthreads();
  const int p = P.p, np = P.p + P.m;
  const double sigma = st.sigma, theta = st.theta;
  const double* yc = w.y + (long long)st.cur * np;
  const double* gc = w.gy + (long long)st.ig_cur * np;
  const double* gp = w.gy + (long long)st.ig_prev * np;
  double* stg = S.stage;   // [v_s | lam_s]
  double nv = 0.0, nl = 0.0;
  for (int j = threadIdx.x; j < np; j += kThreads) {
    const double t1 = (1.0 + theta) * ldcg(gc + j);
    const double t2 = theta * ldcg(gp + j);
    double yt = ldcg(yc + j) + sigma * (t1 - t2);
    if (j >= p) yt = fmax(yt, 0.0);
    stg[j] = yt;
    if (blockIdx.x == 0) w.ytr[j] = yt;
    if (j < p) nv += yt * yt; else nl += yt * yt;
  }
  if (prm.ball) {
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const double a = warp_sum(nv), b = warp_sum(nl);
    if (lane == 0) { S.red[wp * 8] = a; S.red[wp * 8 + 1] = b; }
    __syncthreads();
    if (threadIdx.x < 2) {
      double t = S.red[threadIdx.x];
      for (int i = 1; i < kWarps; ++i) t += S.red[i * 8 + threadIdx.x];
      S.tot[threadIdx.x == 0 ? S_BALL_V : S_BALL_L] = t;
    }
    __syncthreads();
    const BallScale bs = ball_scale(prm, S.tot[S_BALL_V], S.tot[S_BALL_L]);
    if (threadIdx.x == 0) { st.ball_nv = S.tot[S_BALL_V]; st.ball_nl = S.tot[S_BALL_L]; }
    for (int j = threadIdx.x; j < np; j += kThreads) {
      if (j < p) { if (bs.av) stg[j] = bs.sv * stg[j]; }
      else if (bs.al) stg[j] = bs.sl * stg[j];
    }
  }
  __syncthreads();
  return TY_GXPART;
}

// the staged trial duals for the gradient / primal steps of a CTA-local trial
__device__ __forceinline__ void dual_local_stage(const KArgs& K, Sm& S, bool after_relaunch) {
  if (!after_relaunch) return;   // still in shared memory from ty_dual_local
  const BallScale bs = K.prm.ball ? ball_scale(K.prm, S.st->ball_nv, S.st->ball_nl) : BallScale{1.0, 1.0, 0, 0};
  stage_dual(K, K.w.ytr, bs, S.stage, S.stage + K.P.p);
}

// =========================================================== APDB-yx trial

__device__ int ty_dual(const KArgs& K, Sm& S) {
  if (K.P.kind == 1) return ty_dual_fac(K, S);
  if (dual_cta_local(K)) return ty_dual_local(K, S);
  const DevProblem& P = K.P;
  const DevParams& prm = K.prm;
  const Work& w = K.w;
  SolverState& st = *S.st;
  if (threadIdx.x == 0) {
    st.sigma = st.gamma * st.tau;
    st.alpha_n = prm.c_alpha / st.sigma;
    st.beta_n = 0.0;
    st.theta = st.sigma_prev / st.sigma;
  }
  __syncthreads();
  const int p = P.p, np = P.p + P.m;
  const double sigma = st.sigma, theta = st.theta;
  const double* yc = w.y + (long long)st.cur * np;
  const double* gc = w.gy + (long long)st.ig_cur * np;
  const double* gp = w.gy + (long long)st.ig_prev * np;
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
  return gsync(K, S) ? TY_GXPART : kAbort;
}

// The fused factored yx trial (unsharded, host-launched kernels): one stop
// per trial runs the gradient, the primal step, c_i . x_new (one pass over
// C) and the row pass at x_new (factored.cuh fac_trial_kernel /
// fac_row_kernel); ty_primal_fac_fused then adds the dual-side partials.
__device__ __forceinline__ bool fac_fused_trial(const KArgs& K) {
  return K.P.kind == 1 && !K.rc.split && K.prm.mode == 0;
}

__device__ int ty_gxpart(const KArgs& K, Sm& S, int& xk) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  if (fac_fused_trial(K)) {
    if (threadIdx.x == 0) {
      st.fq[0] = 3;
      st.fq[1] = st.cur;
    }
    __syncthreads();
    return TY_PRIMAL;
  }
  double* v_s = S.stage;
  double* lam_s = S.stage + P.p;
  if (dual_cta_local(K)) {
    dual_local_stage(K, S, false);
  } else {
    const BallScale bs = ball_from_slots(K, S, S_BALL_V, S_BALL_L);
    stage_dual(K, w.ytr, bs, v_s, lam_s);
  }
  if (!gx_part(K, S, st.cur, w.ytr + P.p, lam_s, w.gxs)) return kAbort;
  xk = X_GX;
  return TY_PRIMAL;
}

__device__ int ty_primal(const KArgs& K, Sm& S) {
  if (fac_fused_trial(K)) return ty_primal_fac_fused(K, S);
  if (K.P.kind == 1) return ty_primal_fac(K, S);
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m, np = p + m;
  const int cur = st.cur, nxt = cur ^ 1;
  double* v_s = S.stage;
  double* lam_s = S.stage + p;
  if (dual_cta_local(K)) {
    dual_local_stage(K, S, dual_restage(K));
  } else {
    const BallScale bs = ball_from_slots(K, S, S_BALL_V, S_BALL_L);
    stage_dual(K, w.ytr, bs, v_s, lam_s);
  }
  const double tau = st.tau;
  const double* xc = w.x + (long long)cur * n;
  double* xn = w.x + (long long)nxt * n;
  double s_dp = 0.0, s_gd = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) {
    double gx = ldcg(w.gxs + j);
    if (p > 0) gx = gx + atv(K, v_s, j);
    w.gxs[j] = gx;
    const double xj = ldcg(xc + j);
    const double xnj = clipd(xj - tau * gx, __ldg(P.lo + j), __ldg(P.hi + j));
    xn[j] = xnj;
    const double d = xnj - xj;
    s_dp += d * d;
    s_gd += gx * d;
  }
  double s_dd = 0.0, s_mv = 0.0, s_ml = 0.0;
  const double* yc = w.y + (long long)cur * np;
  double* yn = w.y + (long long)nxt * np;
  const double* gvc = w.gval + (long long)cur * (m + 1);
  for (long long j = gtid(); j < np; j += gstride()) {
    const double yv = dual_at(K, v_s, lam_s, w.ytr, j);
    yn[j] = yv;
    const double d = yv - ldcg(yc + j);
    s_dd += d * d;
    if (j < p) s_mv += yv * ldcg(w.eqv + (long long)cur * p + j);
    else s_ml += yv * ldcg(gvc + (j - p + 1));
  }
  const double v5[5] = {s_dp, s_gd, s_dd, s_mv, s_ml};
  const int sl[5] = {S_DP, S_GXDX, S_DD, S_MIXV, S_MIXL};
  put_partials(K, S, v5, sl);
  return gsync(K, S) ? TY_SWEEP : kAbort;
}

__device__ int ty_gy(const KArgs& K, Sm& S) {
  if (K.P.kind == 1) return ty_gy_fac(K, S);
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int p = P.p, m = P.m, np = p + m;
  const int nxt = st.cur ^ 1;
  const double* gvn = w.gval + (long long)nxt * (m + 1);
  const double* gc = w.gy + (long long)st.ig_cur * np;
  double* gnew = w.gy + (long long)st.ig_new * np;
  const double* yn = w.y + (long long)nxt * np;
  double s_dg = 0.0, s_nv = 0.0, s_nl = 0.0;
  for (long long idx = gtid(); idx < np; idx += gstride()) {
    const double gyv = idx < p ? ldcg(w.eqv + (long long)nxt * p + idx) : ldcg(gvn + (idx - p + 1));
    gnew[idx] = gyv;
    const double d = gyv - ldcg(gc + idx);
    s_dg += d * d;
    const double yv = ldcg(yn + idx);
    if (idx < p) s_nv += yv * gyv; else s_nl += yv * gyv;
  }
  const double v3[3] = {s_dg, s_nv, s_nl};
  const int sl[3] = {S_DGY, S_NEWV, S_NEWL};
  put_partials(K, S, v3, sl);
  return gsync(K, S) ? TY_DECIDE : kAbort;
}

// ---------------------------------------------- accepted-step roll (shared)
// engine.py:228-249: stepsize recursion, cache rotation, ergodic sums.
__device__ void roll(const KArgs& K, Sm& S) {
  const DevParams& prm = K.prm;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = K.P.n, np = K.P.p + K.P.m;
  if (threadIdx.x == 0) {
    const double tau = st.tau;
    const double g_next = st.gamma * (1.0 + K.P.mu * tau);
    const double tau_next = tau * sqrt((st.gamma / g_next) * (1.0 + (prm.c_nm * tau) / st.tau_prev));
    const int ip = st.ig_prev;
    st.ig_prev = st.ig_cur;
    st.ig_cur = st.ig_new;
    st.ig_new = ip;
    st.cur ^= 1;
    st.alpha = st.alpha_n;
    st.beta = st.beta_n;
    st.tau_prev = tau;
    st.tau_cand = tau_next;
    st.sigma_prev = st.sigma;
    st.gamma = g_next;
    if (!st.has_sigma0) {
      st.sigma0 = st.sigma;
      st.has_sigma0 = 1;
    }
    const double t_k = st.sigma / st.sigma0;
    st.T += t_k;
    S.tot[NSLOT + 1] = t_k;
    st.phi_k = st.phi_new;
    st.iters += 1;
    st.evals_total += st.evals;
    st.inner += 1;
    st.call_done += 1;
  }
  __syncthreads();
  const double t_k = S.tot[NSLOT + 1];
  const double* xk = w.x + (long long)st.cur * n;
  const double* yk = w.y + (long long)st.cur * np;
  if (K.P.kind == 1) {
    roll_sums_long(K, t_k, xk, yk);
    return;
  }
  for (long long j = gtid(); j < n; j += gstride()) w.xcum[j] += t_k * ldcg(xk + j);
  for (long long j = gtid(); j < np; j += gstride()) w.ycum[j] += t_k * ldcg(yk + j);
}

// after a trial: accept -> roll, else shrink tau or give up (engine.py:205-226)
__device__ int after_trial(const KArgs& K, Sm& S, bool accept, int retry_step) {
  SolverState& st = *S.st;
  if (accept) {
    if (threadIdx.x == 0) st.evals += 1;
    __syncthreads();
    roll(K, S);
    return A_POST;
  }
  if (threadIdx.x == 0) {
    st.evals += 1;
    st.tau *= K.prm.eta;
    if (st.evals > K.prm.max_bt) {
      st.fail_tau = st.tau;
      st.fail_gamma = st.gamma;
      st.fail_iter = st.iters;
      st.status = ST_NONCONV;
    }
  }
  __syncthreads();
  return st.status == ST_NONCONV ? DONE : retry_step;
}

__device__ int ty_decide(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const DevParams& prm = K.prm;
  SolverState& st = *S.st;
  const int sl[8] = {S_DP, S_GXDX, S_DD, S_MIXV, S_MIXL, S_DGY, S_NEWV, S_NEWL};
  get_totals(K, S, sl);
  if (threadIdx.x == 0) {
    const int p = P.p, m = P.m, nxt = st.cur ^ 1;
    const double tau = st.tau, sigma = st.sigma, theta = st.theta;
    const double D_p = 0.5 * S.tot[S_DP];
    const double D_d = 0.5 * S.tot[S_DD];
    double phi_new = ldcg(K.w.gval + (long long)nxt * (m + 1));
    if (p > 0) phi_new += S.tot[S_NEWV];
    if (m > 0) phi_new += S.tot[S_NEWL];
    double phi_mix = ldcg(K.w.gval + (long long)st.cur * (m + 1));
    if (p > 0) phi_mix += S.tot[S_MIXV];
    if (m > 0) phi_mix += S.tot[S_MIXL];
    const double lin = (phi_new - phi_mix) - S.tot[S_GXDX];
    const double nrm = sqrt(S.tot[S_DGY]);
    const double E = ((lin - D_p / tau) + (nrm * nrm) / (2.0 * st.alpha_n))
                     - (1.0 / sigma - theta * st.alpha) * D_d;
    const double rhs = ((-(prm.delta / tau)) * D_p - (prm.delta / sigma) * D_d) + st.slack;
    S.flag[1] = (E <= rhs) ? 1 : 0;
    st.phi_new = phi_new;
  }
  __syncthreads();
  return after_trial(K, S, S.flag[1] != 0, TY_DUAL);
}

// =========================================================== APDB-xy trial

__device__ int tx_primal(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const DevParams& prm = K.prm;
  const Work& w = K.w;
  SolverState& st = *S.st;
  if (threadIdx.x == 0) {
    st.sigma = st.gamma * st.tau;
    st.alpha_n = prm.c_alpha / st.tau;
    st.beta_n = prm.gamma0 * prm.c_beta / st.sigma;
    st.theta = st.sigma_prev / st.sigma;
  }
  __syncthreads();
  const int n = P.n;
  const double tau = st.tau, theta = st.theta;
  const double* gc = w.gxb + (long long)st.ig_cur * n;
  const double* gp = w.gxb + (long long)st.ig_prev * n;
  const double* xc = w.x + (long long)st.cur * n;
  double* xn = w.x + (long long)(st.cur ^ 1) * n;
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
  const double v1[1] = {s_dp};
  const int sl[1] = {S_DP};
  put_partials(K, S, v1, sl);
  return gsync(K, S) ? TX_SWEEP : kAbort;
}

__device__ int tx_dual(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int p = P.p, m = P.m, np = p + m;
  const int nxt = st.cur ^ 1;
  const double sigma = st.sigma;
  const double* yc = w.y + (long long)st.cur * np;
  const double* gvn = w.gval + (long long)nxt * (m + 1);
  double nv = 0.0, nl = 0.0;
  for (long long idx = gtid(); idx < np; idx += gstride()) {
    const double gyv = idx < p ? ldcg(w.eqv + (long long)nxt * p + idx) : ldcg(gvn + (idx - p + 1));
    double yt = ldcg(yc + idx) + sigma * gyv;
    if (idx >= p) yt = fmax(yt, 0.0);
    w.ytr[idx] = yt;
    if (idx < p) nv += yt * yt; else nl += yt * yt;
  }
  if (K.prm.ball) {
    const double v2[2] = {nv, nl};
    const int sl[2] = {S_BALL_V, S_BALL_L};
    put_partials(K, S, v2, sl);
  }
  return gsync(K, S) ? TX_GXPART : kAbort;
}

__device__ int tx_gxpart(const KArgs& K, Sm& S, int& xk) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, np = p + P.m;
  if (P.kind == 1 && !ball_in_place_fac(K, S)) return kAbort;   // factored: y~ scaled in global memory
  const BallScale bs = ball_from_slots(K, S, S_BALL_V, S_BALL_L);
  double* v_n = S.stage;
  double* lam_n = S.stage + p;
  double* v_k = S.stage + np;
  double* lam_k = S.stage + np + p;
  stage_dual(K, w.ytr, bs, v_n, lam_n);
  stage_dual(K, w.y + (long long)st.cur * np, BallScale{1.0, 1.0, 0, 0}, v_k, lam_k);
  const double* Un = w.U + (long long)(st.cur ^ 1) * P.nloc * n;
  double* gnew = w.gxb + (long long)st.ig_new * n;
  if (P.kind == 1) {
    if (!gx_part(K, S, st.cur ^ 1, w.y + (long long)st.cur * np + p, lam_k, w.gxs)) return kAbort;
    if (!gx_part(K, S, st.cur ^ 1, w.ytr + p, lam_n, gnew)) return kAbort;
  } else if (K.sp.rc_cols) {
    recombine_cols(K, S, Un, lam_k, w.gxs);
    recombine_cols(K, S, Un, lam_n, gnew);
  } else {
    for (long long j = gtid(); j < n; j += gstride()) {
      w.gxs[j] = recombine_local(K, Un, lam_k, j);
      gnew[j] = recombine_local(K, Un, lam_n, j);
    }
  }
  xk = X_GX2;
  return TX_NORMS;
}

__device__ int tx_norms(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m, np = p + m;
  const int nxt = st.cur ^ 1;
  const BallScale bs = ball_from_slots(K, S, S_BALL_V, S_BALL_L);
  double* v_n = S.stage;
  double* lam_n = S.stage + p;
  double* v_k = S.stage + np;
  double* lam_k = S.stage + np + p;
  const double* yc = w.y + (long long)st.cur * np;
  stage_dual(K, w.ytr, bs, v_n, lam_n);
  stage_dual(K, yc, BallScale{1.0, 1.0, 0, 0}, v_k, lam_k);
  const double* gc = w.gxb + (long long)st.ig_cur * n;
  double* gnew = w.gxb + (long long)st.ig_new * n;
  double s1 = 0.0, s2 = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) {
    double gyk = ldcg(w.gxs + j);
    double gn = ldcg(gnew + j);
    if (p > 0) {
      gyk = gyk + atv(K, v_k, j);
      gn = gn + atv(K, v_n, j);
    }
    w.gxs[j] = gyk;
    gnew[j] = gn;
    const double d1 = gn - gyk;
    s1 += d1 * d1;
    const double d2 = gyk - ldcg(gc + j);
    s2 += d2 * d2;
  }
  double s_dd = 0.0, s_nv = 0.0, s_nl = 0.0;
  double* yn = w.y + (long long)nxt * np;
  const double* gvn = w.gval + (long long)nxt * (m + 1);
  for (long long j = gtid(); j < np; j += gstride()) {
    const double yv = dual_at(K, v_n, lam_n, w.ytr, j);
    yn[j] = yv;
    const double d = yv - ldcg(yc + j);
    s_dd += d * d;
    if (j < p) s_nv += yv * ldcg(w.eqv + (long long)nxt * p + j);
    else s_nl += yv * ldcg(gvn + (j - p + 1));
  }
  const double v5[5] = {s1, s2, s_dd, s_nv, s_nl};
  const int sl[5] = {S_GXD1, S_GXD2, S_DD, S_NEWV, S_NEWL};
  put_partials(K, S, v5, sl);
  return gsync(K, S) ? TX_DECIDE : kAbort;
}

__device__ int tx_decide(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const DevParams& prm = K.prm;
  SolverState& st = *S.st;
  const int sl[6] = {S_DP, S_GXD1, S_GXD2, S_DD, S_NEWV, S_NEWL};
  get_totals(K, S, sl);
  if (threadIdx.x == 0) {
    const int p = P.p, m = P.m, nxt = st.cur ^ 1;
    const double tau = st.tau, sigma = st.sigma, theta = st.theta;
    const double D_p = 0.5 * S.tot[S_DP];
    const double D_d = 0.5 * S.tot[S_DD];
    const double n1 = sqrt(S.tot[S_GXD1]);
    const double n2 = sqrt(S.tot[S_GXD2]);
    const double E = (((n1 * n1) / (2.0 * st.alpha_n) - D_d / sigma) + (n2 * n2) / (2.0 * st.beta_n))
                     - (1.0 / tau - theta * (st.alpha + st.beta)) * D_p;
    const double rhs = ((-(prm.delta / tau)) * D_p - (prm.delta / sigma) * D_d) + st.slack;
    double phi_new = ldcg(K.w.gval + (long long)nxt * (m + 1));
    if (p > 0) phi_new += S.tot[S_NEWV];
    if (m > 0) phi_new += S.tot[S_NEWL];
    S.flag[1] = (E <= rhs) ? 1 : 0;
    st.phi_new = phi_new;
  }
  __syncthreads();
  return after_trial(K, S, S.flag[1] != 0, TX_PRIMAL);
}

// ====================================================================== KKT
// diagnostics.py:96-113 (orthant cone): stat = |x - Pi_X(x - grad_x Phi)|,
// eq = |Ax-b|, comp = |min(lam, -g)|, infeas = sqrt(|Ax-b|^2 + |max(g,0)|^2).

__device__ int k_gxpart(const KArgs& K, Sm& S, int& xk) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  double* v_s = S.stage;
  double* lam_s = S.stage + P.p;
  const double* yc = w.y + (long long)st.cur * (P.p + P.m);
  stage_dual(K, yc, BallScale{1.0, 1.0, 0, 0}, v_s, lam_s);
  if (!gx_part(K, S, st.cur, yc + P.p, lam_s, w.gxs)) return kAbort;
  xk = X_GX;
  return K_FINISH;
}

__device__ int k_finish(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m, np = p + m;
  const int cur = st.cur;
  double* v_s = S.stage;
  double* lam_s = S.stage + p;
  stage_dual(K, w.y + (long long)cur * np, BallScale{1.0, 1.0, 0, 0}, v_s, lam_s);
  const double* xc = w.x + (long long)cur * n;
  const double* gvc = w.gval + (long long)cur * (m + 1);
  double s_st = 0.0, s_eq = 0.0, s_comp = 0.0, s_gp2 = 0.0, s_gp1 = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) {
    double gx = ldcg(w.gxs + j);
    if (p > 0) gx = gx + atv(K, v_s, j);
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
      const double c = fmin(dual_at(K, v_s, lam_s, w.y + (long long)cur * np, idx), -g);
      s_comp += c * c;
      const double gp = fmax(g, 0.0);
      s_gp2 += gp * gp;
      s_gp1 += gp;
    }
  }
  const double v5[5] = {s_st, s_eq, s_comp, s_gp2, s_gp1};
  const int sl[5] = {S_STAT, S_EQ2, S_COMP, S_GPOS2, S_GPOS1};
  put_partials(K, S, v5, sl);
  if (!gsync(K, S)) return kAbort;
  get_totals(K, S, sl);
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
  return st.kret;
}

// kkt_residual and coupling_value at an explicit point (OP_KKTAT, after the
// probe sweep, g and the gradient at rc.in_x): the k_finish formulas with
// x, v, lam from the caller, plus Phi = (f + v.(Ax - b)) + lam.g
// (problem.py:196-204).  No projection of the point (diagnostics.py:96-113
// evaluates where it is given).
__device__ int p_kkt(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  const RunCfg& rc = K.rc;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m;
  const int par = st.cur ^ 1;
  double* v_s = S.stage;
  if (P.kind == 0 && p > 0) {
    __syncthreads();
    for (int j = threadIdx.x; j < p; j += kThreads) v_s[j] = ldcg(rc.in_v + j);
    __syncthreads();
  }
  const double* gv = w.gval + (long long)par * (m + 1);
  double s_st = 0.0, s_eq = 0.0, s_comp = 0.0, s_gp2 = 0.0, s_gp1 = 0.0, s_pv = 0.0, s_pl = 0.0;
  for (long long j = gtid(); j < n; j += gstride()) {
    double gx = ldcg(w.gxs + j);
    if (p > 0) gx = gx + atv(K, v_s, j);
    const double xj = ldcg(rc.in_x + j);
    const double d = xj - clipd(xj - gx, __ldg(P.lo + j), __ldg(P.hi + j));
    s_st += d * d;
  }
  for (long long idx = gtid(); idx < p + m; idx += gstride()) {
    if (idx < p) {
      const double e = ldcg(w.eqv + (long long)par * p + idx);
      s_eq += e * e;
      s_pv += ldcg(rc.in_v + idx) * e;
    } else {
      const double g = ldcg(gv + (idx - p + 1));
      const double l = ldcg(rc.in_lam + (idx - p));
      const double c = fmin(l, -g);
      s_comp += c * c;
      const double gp = fmax(g, 0.0);
      s_gp2 += gp * gp;
      s_gp1 += gp;
      s_pl += l * g;
    }
  }
  const double v7[7] = {s_st, s_eq, s_comp, s_gp2, s_gp1, s_pv, s_pl};
  const int sl[7] = {S_STAT, S_EQ2, S_COMP, S_GPOS2, S_GPOS1, S_MIXV, S_MIXL};
  put_partials(K, S, v7, sl);
  if (!gsync(K, S)) return kAbort;
  get_totals(K, S, sl);
  if (threadIdx.x == 0) {
    const double stat = sqrt(S.tot[S_STAT]);
    const double eq = sqrt(S.tot[S_EQ2]);
    const double comp = m > 0 ? sqrt(S.tot[S_COMP]) : 0.0;
    const double f = ldcg(gv);
    st.metrics[0] = (stat + eq) + comp;
    st.metrics[1] = stat;
    st.metrics[2] = eq;
    st.metrics[3] = comp;
    st.metrics[4] = sqrt(S.tot[S_EQ2] + S.tot[S_GPOS2]);
    st.metrics[5] = f;
    st.metrics[6] = m > 0 ? S.tot[S_GPOS1] / (double)m : 0.0;
    st.metrics[7] = rc.has_f_star ? f - rc.f_star : __longlong_as_double(0x7ff8000000000000ll);
    st.phi_at = (f + (p > 0 ? S.tot[S_MIXV] : 0.0)) + (m > 0 ? S.tot[S_MIXL] : 0.0);
    st.has_metrics = 1;
  }
  __syncthreads();
  return DONE;
}

// check_termination (diagnostics.py:252-263)
__device__ __forceinline__ bool terminated(const RunCfg& rc, const double* met) {
  if (rc.criterion == 2 && rc.has_f_star) {
    const double rel = fabs(met[5] - rc.f_star) / (1.0 + fabs(rc.f_star));
    return fmax(rel, met[6]) <= rc.eps;
  }
  return met[0] <= rc.eps_kkt && met[4] <= rc.eps_feas;
}

// =================================================================== reinit
// engine.py:102-136: project the point, reset the stepsize recursion, refresh
// the caches at the (new) point with one sweep, zero the ergodic sums.

__device__ int r_point(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, np = p + P.m;
  const int src = st.rsrc, cur = st.cur, nxt = cur ^ 1;
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
  const double v2[2] = {nv, nl};
  const int sl[2] = {S_AVG_V, S_AVG_L};
  put_partials(K, S, v2, sl);
  return gsync(K, S) ? R_SWEEP : kAbort;
}

__device__ int r_sweep(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int np = P.p + P.m, nxt = st.cur ^ 1;
  const int sl[2] = {S_AVG_V, S_AVG_L};
  get_totals(K, S, sl);
  const BallScale bs = ball_scale(K.prm, S.tot[S_AVG_V], S.tot[S_AVG_L]);
  double* yn = w.y + (long long)nxt * np;
  for (long long j = gtid(); j < np; j += gstride()) {
    const double v = ldcg(w.ytr + j);
    yn[j] = j < P.p ? (bs.av ? bs.sv * v : v) : (bs.al ? bs.sl * v : v);
  }
  return sweep_sync(K, S, w.x + (long long)nxt * P.n, nxt) ? R_GLOCAL : kAbort;
}

__device__ int r_cache(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, p = P.p, m = P.m, np = p + m, nxt = st.cur ^ 1;
  const double* gvn = w.gval + (long long)nxt * (m + 1);
  const double* yn = w.y + (long long)nxt * np;
  double pv = 0.0, pl = 0.0;
  for (long long idx = gtid(); idx < np; idx += gstride()) {
    const double gyv = idx < p ? ldcg(w.eqv + (long long)nxt * p + idx) : ldcg(gvn + (idx - p + 1));
    if (K.prm.mode == 0) {
      w.gy[(long long)st.ig_cur * np + idx] = gyv;
      w.gy[(long long)st.ig_prev * np + idx] = gyv;
    }
    const double yv = ldcg(yn + idx);
    if (idx < p) pv += yv * gyv; else pl += yv * gyv;
  }
  for (long long j = gtid(); j < n; j += gstride()) w.xcum[j] = 0.0;
  for (long long j = gtid(); j < np; j += gstride()) w.ycum[j] = 0.0;
  const double v2[2] = {pv, pl};
  const int sl[2] = {S_PHIV, S_PHIL};
  put_partials(K, S, v2, sl);
  if (!gsync(K, S)) return kAbort;
  return K.prm.mode == 1 ? R_GXPART : R_FINISH;
}

__device__ int r_gxpart(const KArgs& K, Sm& S, int& xk) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int nxt = st.cur ^ 1;
  double* v_s = S.stage;
  double* lam_s = S.stage + P.p;
  const double* yn = w.y + (long long)nxt * (P.p + P.m);
  stage_dual(K, yn, BallScale{1.0, 1.0, 0, 0}, v_s, lam_s);
  if (!gx_part(K, S, nxt, yn + P.p, lam_s, w.gxs)) return kAbort;
  xk = X_GX;
  return R_GXCACHE;
}

__device__ int r_gxcache(const KArgs& K, Sm& S) {
  const DevProblem& P = K.P;
  const Work& w = K.w;
  SolverState& st = *S.st;
  const int n = P.n, nxt = st.cur ^ 1;
  double* v_s = S.stage;
  double* lam_s = S.stage + P.p;
  stage_dual(K, w.y + (long long)nxt * (P.p + P.m), BallScale{1.0, 1.0, 0, 0}, v_s, lam_s);
  for (long long j = gtid(); j < n; j += gstride()) {
    double gx = ldcg(w.gxs + j);
    if (P.p > 0) gx = gx + atv(K, v_s, j);
    w.gxb[(long long)st.ig_cur * n + j] = gx;
    w.gxb[(long long)st.ig_prev * n + j] = gx;
  }
  return gsync(K, S) ? R_FINISH : kAbort;
}

__device__ int r_finish(const KArgs& K, Sm& S) {
  const DevParams& prm = K.prm;
  SolverState& st = *S.st;
  const int p = K.P.p, m = K.P.m, nxt = st.cur ^ 1;
  const int sl[2] = {S_PHIV, S_PHIL};
  get_totals(K, S, sl);
  if (threadIdx.x == 0) {
    st.cur = nxt;
    double phi = ldcg(K.w.gval + (long long)nxt * (m + 1));
    if (p > 0) phi += S.tot[S_PHIV];
    if (m > 0) phi += S.tot[S_PHIL];
    st.phi_k = phi;
    const double tau0 = st.rwarm ? st.tau_cand : prm.tau_bar;
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
  return st.ret;
}

}  // namespace rapdb
