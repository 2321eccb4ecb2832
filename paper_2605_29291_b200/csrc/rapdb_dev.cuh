// rapdb_dev.cuh -- device data structures and primitives of the B200 rAPDB path.
//
// Layout in HBM (one context, single rank shard [k0, k1) of the m+1 matrices):
//   Q     [nloc][n][ld]   fp64, row-major, ld even (16-B rows for bulk copies), or
//         [nloc][spm][32][32] packed upper block triangle (layout 1, symsweep.cuh)
//   q     [m+1][n], r [m+1], A [p][n], b [p], lower/upper [n]
//   x     [2][n]          parity `cur` = accepted x_k, `cur^1` = trial x_new
//   U     [2][nloc][n]    u_i = Q_i x for both parities (the U-cache)
//   gval  [2][m+1]        f (index 0) and g_i at both parities
//   eqv   [2][p]          A x - b
//   y     [2][p+m]        (v, lam) at both parities
//   ytr   [p+m]           dual trial point before the dual-ball projection
//   gy    [3][p+m]        yx caches gy_prev / gy_cur / gy_new (rotating indices)
//   gxb   [3][n]          xy caches gx_prev / gx_cur / gx_new (rotating indices)
//   gxs   [n]             scratch gradient (gx_mixed, KKT gradient, gx at y_k)
//   xcum  [n], ycum [p+m] ergodic accumulators (engine.py:244-249)
//   part  [NSLOT][G]      per-CTA partial sums (fixed-order grid reductions)
//   segxu/segqx [G][8][segmax]  per-(CTA, warp, matrix-segment) x.u and q.x sums
//               (packed layout: [nact][nbB] per-(matrix, 64-row block) sums)
//   Pt    [nact][nbB][nbB][64]  packed layout: unit partial products (symsweep.cuh)
//
// All arithmetic is IEEE binary64.  The file is compiled with -fmad=false so
// scalar control reproduces the reference's Python-float operation order
// exactly; dot products request FMA explicitly with fma().
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "symsweep.cuh"

namespace rapdb {

constexpr int kThreads = 256;      // 7 consumer warps + 1 bulk-copy producer warp (2 warps per SMSP: 255-register cap)
constexpr int kConsumerWarps = 7;
constexpr int kWarps = 8;
constexpr int kMaxTR = 32;         // rows per tile upper bound

enum Slot {
  S_BALL_V = 0, S_BALL_L,                       // dual-ball norms of the trial dual
  S_DP, S_GXDX, S_DD, S_MIXV, S_MIXL,           // yx phase 2 / xy phase 1+4
  S_DGY, S_NEWV, S_NEWL,                        // yx phase 4 / xy phase 4
  S_GXD1, S_GXD2,                               // xy: |gx_new-gx_yk|^2, |gx_yk-gx_cur|^2
  S_STAT, S_EQ2, S_COMP, S_GPOS2, S_GPOS1,      // KKT
  S_PHIV, S_PHIL,                               // Phi at a (re)start point
  S_AVG_V, S_AVG_L,                             // ball norms of an average point
  S_GAPQ,                                       // z'Hz in the smoothed-gap subsolver
  S_EGM_X, S_EGM_V, S_EGM_L,                    // EGM: |x|^2, |v|^2, |lam|^2 of a point
  NSLOT
};

enum Op { OP_RUN = 0, OP_REINIT = 1, OP_KKT = 2, OP_GET = 3, OP_PROBE = 4, OP_GAP = 5, OP_GRAD = 6, OP_EGM = 7,
           OP_KKTAT = 8 };
enum RunStatus { ST_LIMIT = 0, ST_CONVERGED = 1, ST_BUDGET = 2, ST_CHECK_DUE = 3,
                 ST_FIXED_DUE = 4, ST_NONCONV = 5, ST_ABORT = 6, ST_EXCHANGE = 7, ST_RUNNING = 8 };

struct SolverState {
  double tau_cand, tau_prev, gamma, sigma_prev, alpha, beta, sigma0, T, phi_k;
  double fail_tau, fail_gamma;
  double metrics[8];
  double phi_at;           // OP_KKTAT: coupling_value at the given point
  double gap[6];           // gap, subsolver iterations, residual, converged, L, dual term
  double sweep_ns;
  long long iters, evals_total, inner, fail_iter, sweeps;
  int cur, ig_prev, ig_cur, ig_new, has_sigma0, status, has_metrics, pad;
  // resumable control (the kernel may exit at an exchange point and resume)
  double tau, tau_start, slack, sigma, alpha_n, beta_n, phi_new, theta;
  long long call_done;     // accepted iterations in the current rapdb_run call
  unsigned long long xgen; // in-kernel peer exchanges done by this context (generation counter)
  int step, ret, kret, xkind, evals, rsrc, rwarm, pad2;
  // factored, host-assisted: request for the host to run the high-occupancy
  // factored kernels at this stop: fq[0] = 0 none, 1 sweep (fq[1] = parity,
  // fq[2] = x source: 0 w.x[par], 1 rc.in_x), 2 gradient(s) (fq[1] = count,
  // then per request: parity, multiplier id, output id; factored.cuh)
  int fq[8];
  double ball_nv, ball_nl; // CTA-local yx dual step: |v~|^2, |lam~|^2 of the trial (re-staging after a relaunch)
  double step_ns[64];      // device time per state-machine step (CTA 0, globaltimer); 60..62: sweep sub-phases
  long long step_cnt[64];
};

// steps of the resumable op state machine
enum Step {
  T_BEGIN = 0,
  TY_DUAL, TY_GXPART, TY_PRIMAL, TY_SWEEP, TY_GLOCAL, TY_GY, TY_DECIDE,
  TX_PRIMAL, TX_SWEEP, TX_GLOCAL, TX_DUAL, TX_GXPART, TX_NORMS, TX_DECIDE,
  A_POST, K_GXPART, K_FINISH, A_RESTART, A_END,
  R_POINT, R_SWEEP, R_GLOCAL, R_CACHE, R_GXPART, R_GXCACHE, R_FINISH,
  G_CAND, G_GLOCAL, G_HPART, G_SOLVE,
  P_SWEEP, P_OUT, P_GRAD, P_GFIN, P_KKT,
  E_INIT, E_GX, E_HALF, E_HSWEEP, E_HGLOC, E_GXH, E_PLUS, E_PSWEEP, E_PGLOC, E_POST,
  DONE
};
// exchange kinds: what the host must all-reduce (sum) across ranks before resuming
enum Xkind { X_NONE = 0, X_GX = 1, X_G = 2, X_GX2 = 3, X_H = 4 };

// Sliced ELLPACK with slices of 32 slots (one warp, lane = slot): entry t of
// slot s lives at sp[s >> 5] + 32 t + (s & 31), so a warp's t-th loads of val
// and idx are one coalesced 256 / 128 byte access and every slot folds its own
// entries in stored order.  A slice is as wide as its longest slot.
struct Sell {
  long long nslots;      // multiple of 32
  long long entries;     // sp[nslots / 32]: stored entries incl. padding
  const long long* sp;   // [nslots / 32 + 1] entry offset of each slice
  const int* idx;        // gathered index of each entry
  const double* val;
  const int* len;        // [nslots] entries of each slot
  const int* map;        // [nslots] output index of each slot (-1: padding); null = the slot itself
};
constexpr int kMaxRtPhases = 8;
constexpr int kSellR = 0, kSellA = 1, kSellAt = 2, kSellRt = 3;   // DevProblem::sell slots

struct DevProblem {
  int n, m, p, k0, k1, nloc, nact, nzero;
  long long ld;
  const double* Q; const double* q; const double* r; const double* A; const double* b;
  const double* lo; const double* hi;
  double mu;
  const int* act;        // [nact]  local index of each streamed (non-zero) matrix
  const int* zero_list;  // [nzero] local index of each all-zero matrix
  const int* seg_lo;     // [nact]  first CTA whose row range touches active matrix a
  const int* seg_hi;     // [nact]  last CTA (inclusive)
  const int* cta_a0;     // [G]     first active matrix of each CTA's row range
  const int* mat_slot;   // [nloc]  active index a >= 0, or -(zero index)-1
  // ---- factored instances (kind 1, BASELINE config 3): Q_i = R_i^T R_i ----
  int kind;              // 0 dense Q stack, 1 factored
  int mq;                // quadratic constraints (factored matrices 0..mq)
  long long nr;          // rows of the stacked R
  int L;                 // linear rows A x <= b (orthant constraints with Q = 0)
  int nchx;              // chunks of kCxCols columns for c_i . x (factored.cuh)
  int nfpart;            // warps of a fused-trial gradient launch (its D_p / <gx, dx> partials)
  // The sparse operands are held as sliced ELLPACK (Sell, slice height 32):
  //   sr   R   [nr x n]: slot = 128 * (W chunk) + row inside the chunk, so every
  //        chunk of a block (wch / rblk) is 4 slices and no slice spans two blocks
  //   sa   A   [Lloc x n]: slot = local row
  //   srt  R^T [n x nr] in rt_nph ROW PHASES (rows [rt_b[p], rt_b[p+1]) of the
  //        stacked R): one Sell per phase over the columns sorted by their
  //        entry count in that phase (map = column of the slot); entries of a
  //        column in row order, so walking the phases walks each column in
  //        sorted row order; rt_tag: idx holds r | (local block of r) << 23
  //        (the gather weights W on the fly)
  //   sat  A^T [n x Lloc], columns sorted by entry count (map = column)
  // (a device table, so a phase can be indexed at run time without a local copy)
  const Sell* sell;      // [kSellRt + rt_nph]: R, A, A^T, then the phases of R^T
  int rt_nph, rt_tag;
  int sym;               // the blocks are the symmetric Q_i themselves (n rows each), not factors R_i:
                         // W = Q x is the U-cache, g_i = 1/2 x . W_i + ..., grad = sum w_i (W_i + c_i), no R^T
  const int* rmat;                                                  // [nr] block of each R row
  const long long* rblk;                                            // [mq+2] first row of block i
  const long long* wch;  // [fnb+1] prefix count of 1024-row chunks of W per local block
  // constraint sharding of a factored instance: this rank holds blocks
  // [fb0, fb0+fnb) of the mq+1 (R, C, d local, rmat local ids) and linear rows
  // [l0, l0+Lloc) of the L (A, A^T, b local); mq and L stay the global counts
  int fb0, fnb, l0, Lloc;
};

struct DevParams {
  int mode;              // 0 yx, 1 xy
  int max_bt, ball;      // ball 0 none, 1 joint, 2 split
  int pad;
  double c_alpha, c_beta, delta, eta, tau_bar, gamma0, c_nm, r1, r2;
};

struct SweepPlan {
  int TR;                // rows per tile (power of two <= 32)
  int nstages;
  int segmax;
  int ncw;               // consumer warps used by the sweep (<= nstages)
  int cpr;               // column chunks per row (> 1: rows wider than a stage)
  int chunk;             // doubles per chunk (== ld when cpr == 1)
  int rc_cols;           // gradient recombination by CTA column blocks (many matrices)
  int pad3;
  long long stage_bytes; // per ring slot (multiple of 128)
  long long rows_total;  // nact * n
  long long xs_bytes;    // x staging bytes (multiple of 128)
  int layout;            // 0 row-major stack [nloc][n][ld], 1 packed symmetric (symsweep.cuh)
  int pad4;
  sym::Geom geom;        // layout 1: unit geometry of one matrix
  int nchunk;            // layout 1: matrix chunks reduced during the stream (0: all in phase B)
  int xglobal;           // layout 1: x too long for shared memory -- per-warp 128-entry x blocks
  const sym::Unit* units;  // layout 1: [upm] unit table (device)
};

struct Work {
  double *x, *U, *gval, *eqv, *y, *ytr, *gy, *gxb, *gxs, *xcum, *ycum, *part,
         *segxu, *segqx, *zq, *aux, *aux2;
  double *H, *hx, *hxn, *hy;   // smoothed gap: dense H (n x n) and H-products
  double *W;                   // factored: [2][nr] W = R x at both parities
  double *pw2, *pcx;           // factored: chunk partials of |W_i|^2 and c_i . x
  double *wl;                  // factored: [nr] block-weighted W-cache of the recombination
  double *fpart;               // factored fused trial: [2][nfpart] per-warp partials of D_p, <gx, dx>
  unsigned *fctr;              // factored row kernel: [2] work-item / finished-CTA counters
  double *Pt;                  // layout 1: per-unit partial products [nact][nbB][nbB][64]
  unsigned* ccnt;              // layout 1: [64] consumer warps done with each matrix chunk
  int* idone;                  // layout 1: [nact*nbB] phase-B items already reduced during the stream
  double* trace;
  SolverState* st;
  unsigned long long* bar;
  int* abort_flag;
};

struct RunCfg {
  long long max_iters, budget, stop_total;
  int metrics_every, criterion, has_f_star, fixed_period, fixed_point, warm_tau, stop_at_fixed;
  int op, src, reset_inner, reps;
  int split;               // exit at exchange points (sharded runs) instead of continuing
  int fac_host;            // factored: sweeps / gradients run as host-launched kernels (stops)
  int p2p;                 // sharded dense: exchanges in-kernel over peer memory (PeerX)
  int resume;              // continue the saved op at st.step

  double eps, eps_kkt, eps_feas, f_star;
  double xi, tol;                  // smoothed gap
  double egm_s;                    // EGM stepsize
  long long egm_K;                 // EGM iterations
  int egm_trace_every, egm_pad;
  const double* warm;              // smoothed gap subsolver warm start (or null)
  const double* in_x; const double* in_v; const double* in_lam;   // explicit points
  double* out_x; double* out_v; double* out_lam; double* out_u; double* out_g;
};

// In-kernel constraint-shard exchange over NVLink peer memory: every rank
// owns a region [2 sets][R slots][S doubles] + [R flags]; rank r pushes its
// partial into slot r of set (gen & 1) of every peer, signals flag r of every
// peer with the generation, waits for all R flags of its own region, and sums
// its R slots in rank order -- the same bits on every rank.
struct PeerX {
  double* const* slots;            // [R] base of each rank's region (device pointers, peers mapped)
  unsigned long long* const* flags; // [R] each rank's flag array (R x 16 words apart)
  long long S;                     // doubles per slot
  int rank, R;
};

struct KArgs {
  DevProblem P;
  DevParams prm;
  SweepPlan sp;
  Work w;
  RunCfg rc;
  PeerX px;
};

// ---------------------------------------------------------------- primitives

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile("{\n\t.reg .pred p;\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

// spin on an mbarrier phase; after ~10 s raise the device abort flag and give
// up (a protocol bug then surfaces as RAPDB_EDEVICE instead of a hung GPU)
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, unsigned parity, int* abort_flag) {
  if (mbar_try_wait(bar, parity)) return true;
  // SM cycle counter, not %globaltimer: the driver re-synchronises globaltimer
  // with host time and it can jump (a backward jump wrapped the unsigned delta
  // and fired this watchdog spuriously)
  const long long t0 = clock64();
  for (unsigned spins = 1;; ++spins) {
    if (mbar_try_wait(bar, parity)) return true;
    if ((spins & 1023u) == 0) {
      if (*(volatile int*)abort_flag) return false;
      const long long el = (clock64() - t0) / 2;   // ~ns at ~2 GHz
      if (el > 20000000000ll) {
        if (atomicExch(abort_flag, 2) == 0) {   // 2: mbarrier (bulk-copy pipeline) timeout
          abort_flag[1] = blockIdx.x;
          abort_flag[2] = threadIdx.x;
          abort_flag[3] = (int)parity;
          abort_flag[4] = (int)(el / 1000000ll);
          abort_flag[5] = (int)(smem_u32(bar) & 0x3ffff);
        }
        return false;
      }
    }
  }
}

// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier (UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;"
      :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void named_bar_consumers() {
  asm volatile("bar.sync 1, 256;" ::: "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // butterfly: every lane holds the same bits
}

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// streaming read-only loads that ask L2 to evict the line first (big
// once-per-pass streams must not push small gathered vectors out of L2)
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(p), "d"(v), "l"(pol) : "memory");
}

}  // namespace rapdb
