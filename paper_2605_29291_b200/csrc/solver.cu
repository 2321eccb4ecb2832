// solver.cu -- kernel entry (op dispatch + the accepted-iteration loop) and
// the C ABI declared in include/rapdb_b200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.cuh"
#include "egm.cuh"
#include "gap.cuh"
#include "spectral.cuh"
#include "rapdb_b200.h"
#include "solver_ops.cuh"

namespace rapdb {

__device__ __forceinline__ void trace_put(const KArgs& K, long long row, int col, double v) {
  if (K.w.trace) K.w.trace[row * RAPDB_TRACE_COLS + col] = v;
}

// One step of the resumable op state machine (see solver_ops.cuh).  Returns the
// next step; `xk` is set at exchange points.
__device__ int run_step(const KArgs& K, Sm& S, int step, int& xk) {
  SolverState& st = *S.st;
  const RunCfg& rc = K.rc;
  switch (step) {
    case T_BEGIN:   // ApdbEngine.step entry (engine.py:199-204)
      if (threadIdx.x == 0) {
        st.tau = st.tau_cand;
        st.tau_start = st.tau;
        st.slack = 1e-13 * (1.0 + fabs(st.phi_k));
        st.evals = 0;
      }
      __syncthreads();
      return K.prm.mode == 1 ? TX_PRIMAL : TY_DUAL;
    case TY_DUAL: return ty_dual(K, S);
    case TY_GXPART: return ty_gxpart(K, S, xk);
    case TY_PRIMAL: return ty_primal(K, S);
    case TY_SWEEP: return sweep_sync(K, S, K.w.x + (long long)(st.cur ^ 1) * K.P.n, st.cur ^ 1) ? TY_GLOCAL : kAbort;
    case TY_GLOCAL: g_local(K, st.cur ^ 1); xk = X_G; return TY_GY;
    case TY_GY: return ty_gy(K, S);
    case TY_DECIDE: return ty_decide(K, S);
    case TX_PRIMAL: return tx_primal(K, S);
    case TX_SWEEP: return sweep_sync(K, S, K.w.x + (long long)(st.cur ^ 1) * K.P.n, st.cur ^ 1) ? TX_GLOCAL : kAbort;
    case TX_GLOCAL: g_local(K, st.cur ^ 1); xk = X_G; return TX_DUAL;
    case TX_DUAL: return tx_dual(K, S);
    case TX_GXPART: return tx_gxpart(K, S, xk);
    case TX_NORMS: return tx_norms(K, S);
    case TX_DECIDE: return tx_decide(K, S);
    case A_POST: {  // trace row; KKT cadence (restarts.py:115-124)
      const long long total = st.iters, row = st.call_done - 1;
      if (blockIdx.x == 0 && threadIdx.x == 0 && K.w.trace) {
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
        double* tr = K.w.trace + row * RAPDB_TRACE_COLS;
        tr[0] = (double)total; tr[1] = st.tau_start; tr[2] = st.tau; tr[3] = st.sigma; tr[4] = st.gamma;
        tr[5] = (double)st.evals; tr[6] = (double)st.evals_total; tr[7] = qnan; tr[8] = qnan; tr[9] = qnan;
        tr[10] = 0.0;
      }
      if (rc.criterion != 0 && rc.metrics_every > 0 && (total % rc.metrics_every == 0 || total == rc.budget)) {
        if (threadIdx.x == 0) st.kret = A_RESTART;
        __syncthreads();
        return K_GXPART;
      }
      return A_RESTART;
    }
    case K_GXPART: return k_gxpart(K, S, xk);
    case K_FINISH: {
      const int nx = k_finish(K, S);
      if (nx == A_RESTART) {   // inside a run: record and test termination
        const long long row = st.call_done - 1;
        if (blockIdx.x == 0 && threadIdx.x == 0 && K.w.trace) {
          double* tr = K.w.trace + row * RAPDB_TRACE_COLS;
          tr[7] = st.metrics[0]; tr[8] = st.metrics[4]; tr[9] = st.metrics[7];
        }
        if (terminated(rc, st.metrics)) {
          if (threadIdx.x == 0) st.status = ST_CONVERGED;
          __syncthreads();
          return DONE;
        }
      }
      return nx;
    }
    case A_RESTART: {   // FixedRestart (restarts.py:126-135)
      const long long total = st.iters;
      const bool due = rc.fixed_period > 0 && st.inner >= rc.fixed_period && total < rc.budget;
      __syncthreads();   // every thread has read st.inner before thread 0 resets it below
      if (due) {
        if (rc.stop_at_fixed) {
          if (threadIdx.x == 0) st.status = ST_FIXED_DUE;
          __syncthreads();
          return DONE;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0 && K.w.trace)
          K.w.trace[(st.call_done - 1) * RAPDB_TRACE_COLS + 10] = 1.0;
        if (threadIdx.x == 0) {
          st.rsrc = rc.fixed_point ? 2 : 1;
          st.rwarm = rc.warm_tau;
          st.ret = A_END;
          st.inner = 0;
        }
        __syncthreads();
        return gsync(K, S) ? R_POINT : kAbort;
      }
      return A_END;
    }
    case A_END: {
      const long long total = st.iters;
      int status = -1;
      if (rc.stop_total > 0 && total == rc.stop_total && total < rc.budget) status = ST_CHECK_DUE;
      else if (total >= rc.budget) status = ST_BUDGET;
      else if (st.call_done >= rc.max_iters) status = ST_LIMIT;
      if (status < 0) return T_BEGIN;
      if (threadIdx.x == 0) st.status = status;
      __syncthreads();
      return DONE;
    }
    case R_POINT: return r_point(K, S);
    case R_SWEEP: return r_sweep(K, S);
    case R_GLOCAL: g_local(K, st.cur ^ 1); xk = X_G; return R_CACHE;
    case R_CACHE: return r_cache(K, S);
    case R_GXPART: return r_gxpart(K, S, xk);
    case R_GXCACHE: return r_gxcache(K, S);
    case R_FINISH: return r_finish(K, S);
    case G_CAND: return g_cand(K, S);
    case G_GLOCAL: g_local(K, st.cur ^ 1); xk = X_G; return G_HPART;
    case G_HPART: return g_hpart(K, S, xk);
    case G_SOLVE: return g_solve(K, S);
    case P_SWEEP: {
      for (int r = 0; r < max(1, rc.reps); ++r)
        if (!sweep_sync(K, S, rc.in_x, st.cur ^ 1)) return kAbort;
      return P_OUT;
    }
    case P_OUT: {   // g (and the cache row(s): U, or W = R x when factored) at rc.in_x
      const DevProblem& P = K.P;
      const int par = st.cur ^ 1;
      const int nxt = (rc.op == OP_GRAD || rc.op == OP_KKTAT) ? P_GRAD : DONE;
      if (P.kind == 1) {
        g_factored(K, par);
        if (!gsync(K, S)) return kAbort;
        const double* gv = K.w.gval + (long long)par * (P.m + 1);
        if (rc.out_g)
          for (long long i = gtid(); i <= P.m; i += gstride()) rc.out_g[i] = ldcg(gv + i);
        const double* Wp = K.w.W + (long long)par * P.nr;
        if (rc.out_u)
          for (long long j = gtid(); j < P.nr; j += gstride()) rc.out_u[j] = ldcg(Wp + j);
        return nxt;
      }
      if (rc.out_v && rc.op == OP_PROBE)   // A x - b at the probed point (eq_residual)
        for (long long i = gtid(); i < P.p; i += gstride()) rc.out_v[i] = ldcg(K.w.eqv + (long long)par * P.p + i);
      if (rc.out_g) {
        for (long long i = gtid(); i <= P.m; i += gstride())
          rc.out_g[i] = (i >= P.k0 && i < P.k1) ? g_combine(K, (int)i) : 0.0;
      } else if (nxt != DONE) {   // keep g at the probed point for the KKT / gradient steps
        double* gv = K.w.gval + (long long)par * (P.m + 1);
        for (long long i = gtid(); i <= P.m; i += gstride())
          gv[i] = (i >= P.k0 && i < P.k1) ? g_combine(K, (int)i) : 0.0;
        if (!gsync(K, S)) return kAbort;
      }
      const double* Up = K.w.U + (long long)par * P.nloc * P.n;
      const long long tot = (long long)P.nloc * P.n;
      if (rc.out_u)
        for (long long j = gtid(); j < tot; j += gstride()) rc.out_u[j] = ldcg(Up + j);
      return nxt;
    }
    case P_GRAD: {  // grad_x Phi(x, v, lam) at the probed point (problem.py:207-217)
      const DevProblem& P = K.P;
      double* v_s = S.stage;
      double* lam_s = S.stage + P.p;
      if (P.kind == 0) {
        for (int j = threadIdx.x; j < P.p + P.m; j += kThreads) {
          if (j < P.p) v_s[j] = ldcg(rc.in_v + j);
          else lam_s[j - P.p] = ldcg(rc.in_lam + (j - P.p));
        }
        __syncthreads();
      }
      if (!gx_part(K, S, st.cur ^ 1, rc.in_lam, lam_s, K.w.gxs)) return kAbort;
      xk = X_GX;
      return rc.op == OP_KKTAT ? P_KKT : P_GFIN;
    }
    case P_KKT: return p_kkt(K, S);
    case P_GFIN: {
      const DevProblem& P = K.P;
      double* v_s = S.stage;
      if (P.kind == 0 && P.p > 0) {
        __syncthreads();
        for (int j = threadIdx.x; j < P.p; j += kThreads) v_s[j] = ldcg(rc.in_v + j);
        __syncthreads();
      }
      for (long long j = gtid(); j < P.n; j += gstride()) {
        double gx = ldcg(K.w.gxs + j);
        if (P.p > 0) gx = gx + atv(K, v_s, j);
        rc.out_x[j] = gx;
      }
      return DONE;
    }
    case E_INIT: case E_GX: case E_HALF: case E_HSWEEP: case E_HGLOC:
    case E_GXH: case E_PLUS: case E_PSWEEP: case E_PGLOC: case E_POST:
      return egm_step(K, S, step, xk);
    default:
      return kAbort;
  }
}

// Run the state machine until DONE, an abort, or (sharded runs) an exchange.
__device__ void drive(const KArgs& K, Sm& S) {
  SolverState& st = *S.st;
  for (;;) {
    const int step = st.step;
    // All shared state (st, in shared memory) is written by thread 0 only, and
    // every write is separated from the other threads' reads by a barrier: here,
    // nobody may overwrite st.step (end of this iteration) before all threads
    // have read it -- a step without an internal barrier let thread 0 race
    // ahead and split the CTA across two steps (a bar.sync deadlock).
    __syncthreads();
    if (step == DONE) return;
    int xk = X_NONE;
    unsigned long long t0 = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) t0 = globaltimer();
    if (threadIdx.x == 0) {   // progress beacon, readable by the host while the kernel runs
      volatile int* bcn = K.w.abort_flag + 32 + 4 * blockIdx.x;
      bcn[0] = step;
      bcn[1] = (int)S.gen;
      bcn[2] = (int)st.call_done;
      bcn[3] = (int)S.pseq;
    }
    const int next = run_step(K, S, step, xk);
    if (blockIdx.x == 0 && threadIdx.x == 0 && step < 60) {
      const unsigned long long t1 = globaltimer();
      if (t1 > t0) st.step_ns[step] += (double)(t1 - t0);
      st.step_cnt[step] += 1;
    }
    __syncthreads();   // the step's reads of st are done before thread 0 writes below
    if (next == kAbort) {
      if (threadIdx.x == 0) { st.status = ST_ABORT; st.step = DONE; }
      __syncthreads();
      return;
    }
    if (threadIdx.x == 0) st.step = next;
    __syncthreads();
    if (st.fq[0] != 0) {   // host-assisted factored work (and maybe an exchange) at this stop
      if (threadIdx.x == 0) { st.xkind = K.rc.split ? xk : X_NONE; st.status = ST_EXCHANGE; }
      __syncthreads();
      return;
    }
    if (xk != X_NONE && K.rc.p2p && xk != X_H) {   // in-kernel exchange over NVLink peer memory
      if (!peer_exchange(K, S, xk)) {
        if (threadIdx.x == 0) { st.status = ST_ABORT; st.step = DONE; }
        __syncthreads();
        return;
      }
      continue;
    }
    if (xk != X_NONE) {
      if (K.rc.split) {   // the host all-reduces the buffer and relaunches
        if (threadIdx.x == 0) { st.xkind = xk; st.status = ST_EXCHANGE; }
        __syncthreads();
        return;
      }
      // one rank: the partial is the total; G/H (and column-block gradients) are
      // read by other threads next
      if ((xk == X_G || xk == X_H || K.sp.rc_cols) && !gsync(K, S)) {
        if (threadIdx.x == 0) { st.status = ST_ABORT; st.step = DONE; }
        __syncthreads();
        return;
      }
    }
  }
}

__device__ void op_get(const KArgs& K, Sm& S) {
  const SolverState& st = *S.st;
  const Work& w = K.w;
  const int n = K.P.n, p = K.P.p, m = K.P.m, np = p + m;
  const bool avg = K.rc.src == 2 && st.T > 0.0;
  const double* xc = w.x + (long long)st.cur * n;
  const double* yc = w.y + (long long)st.cur * np;
  for (long long j = gtid(); j < n; j += gstride())
    K.rc.out_x[j] = avg ? ldcg(w.xcum + j) / st.T : ldcg(xc + j);
  for (long long j = gtid(); j < np; j += gstride()) {
    const double v = avg ? ldcg(w.ycum + j) / st.T : ldcg(yc + j);
    if (j < p) K.rc.out_v[j] = v; else K.rc.out_lam[j - p] = v;
  }
}

}  // namespace rapdb

using namespace rapdb;

extern "C" __global__ void __launch_bounds__(kThreads, 1) rapdb_solver_kernel(const __grid_constant__ KArgs K) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ double s_red[kWarps * 8];
  __shared__ double s_tot[NSLOT + 4];
  __shared__ SolverState s_st;
  __shared__ int s_flag[4];
  __shared__ unsigned s_prog[kConsumerWarps];
  __shared__ unsigned s_tag[32], s_rel[32];
  Sm S;
  S.prog = s_prog;
  S.tag = s_tag;
  S.rel = s_rel;
  if (threadIdx.x < kConsumerWarps) s_prog[threadIdx.x] = 0;
  S.xs = reinterpret_cast<double*>(dsm);
  S.ring = dsm + K.sp.xs_bytes;
  S.full = reinterpret_cast<uint64_t*>(S.ring + (long long)K.sp.nstages * K.sp.stage_bytes);
  S.empty = S.full + K.sp.nstages;
  S.stage = reinterpret_cast<double*>(S.ring);
  S.rc = reinterpret_cast<double(*)[32]>(S.ring + (long long)K.sp.nstages * K.sp.stage_bytes - kWarps * 32 * 8);
  S.red = s_red;
  S.tot = s_tot;
  S.st = &s_st;
  S.flag = s_flag;
  S.gen = 0;
  S.pseq = 0;
  if (threadIdx.x == 0) {
    s_st = *K.w.st;
    s_st.fq[0] = 0;   // the host served the previous stop's request
    for (int s = 0; s < K.sp.nstages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);   // each ring slot is consumed by exactly one warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (!K.rc.resume) {   // a new op: initial step
      s_st.status = ST_RUNNING;
      s_st.xkind = X_NONE;
      switch (K.rc.op) {
        case OP_RUN: s_st.step = T_BEGIN; s_st.call_done = 0; break;
        case OP_REINIT:
          s_st.step = R_POINT; s_st.ret = DONE; s_st.rsrc = K.rc.src; s_st.rwarm = K.rc.warm_tau;
          if (K.rc.reset_inner) s_st.inner = 0;
          break;
        case OP_KKT: s_st.step = K_GXPART; s_st.kret = DONE; break;
        case OP_GAP: s_st.step = G_CAND; break;
        case OP_PROBE: case OP_GRAD: case OP_KKTAT: s_st.step = P_SWEEP; break;
        case OP_EGM: s_st.step = E_INIT; break;
        default: s_st.step = DONE; break;
      }
    } else {
      s_st.status = ST_RUNNING;
    }
  }
  __syncthreads();
  if (K.rc.op == OP_GET) op_get(K, S);
  else drive(K, S);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (s_st.status == ST_RUNNING) s_st.status = ST_LIMIT;   // op completed
    *K.w.st = s_st;
  }
}

// ========================================================================
// host side
// ========================================================================

struct rapdb_ctx {
  int device = 0, rank = 0, nranks = 1;
  cudaStream_t stream = nullptr;
  std::string err;
  int nsm = 0, G = 0;
  size_t optin = 0, dyn_smem = 0;
  bool bound = false, have_params = false, have_ws = false;
  DevProblem P{};
  DevParams prm{};
  SweepPlan sp{};
  Work w{};
  int* d_ints = nullptr;
  long long* d_ll = nullptr;   // factored: rblk and W-chunk prefix tables
  Sell* d_sell = nullptr;      // factored: the Sell descriptors (DevProblem::sell)
  Sell h_sell[kSellRt + kMaxRtPhases];
  long long grad_bytes = 0;    // factored: bytes one gradient streams (R^T, A^T, C, column partials)
  sym::Unit* d_units = nullptr;  // packed layout: unit table
  SolverState* h_state = nullptr;  // page-locked copy of the device state (+ abort flag)
  long long ws_bytes = 0;
  long long stage_cap = 0;  // doubles available in the staging area
  bool gap_ok = false;      // dense H + shared n-vectors fit (smoothed gap available)
  long long sweep_bytes = 0;  // algorithmic bytes of one sweep (the roofline numerator)
  long long nchw = 0;       // factored: kWChunk-row chunks of W over all blocks
  int split = 0;            // sharded: stop at exchange points
  int fac_host = 0;         // factored: sweeps / gradients as host-launched high-occupancy kernels
  int p2p = 0;              // sharded dense: in-kernel exchanges over peer memory
  PeerX px{};
  void* d_px = nullptr;     // device tables of the peer region pointers
  rapdb_exchange_fn xcb = nullptr;
  void* xuser = nullptr;
  rapdb_comm* comm = nullptr;        // native rank-ordered NCCL exchange (instead of xcb)
  rcomm::Scratch xscratch;      // its gather / reduce-scatter scratch
  long long exchanges = 0;
  SolverState last_st{};
  int guard = 0;                     // RAPDB_GUARD: guard zones in the workspace (fixed at bind)
  char* ws_base = nullptr;
};

// One NCCL communicator per process and device, shared by every context of
// a sharded run (comm.cuh: rank-ordered sums, NCCL moves bytes only).
struct rapdb_comm {
  ncclComm_t nccl = nullptr;
  int device = 0, rank = 0, nranks = 1;
};

namespace {

int fail(rapdb_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(rapdb_ctx* c, cudaError_t e, const char* where) {
  return fail(c, RAPDB_EDEVICE, std::string(where) + ": " + cudaGetErrorString(e));
}

// Owns the CUDA events a host entry point creates, so every early return
// (CK, a failed launch, an exchange-callback error) releases them.
struct EventGuard {
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~EventGuard() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
};

#define CK(call)                                   \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, #call); \
  } while (0)

long long align_up(long long v, long long a) { return (v + a - 1) / a * a; }

// Small per-context device tables are stream-ordered allocations (no device
// synchronisation on free: a context is created and destroyed per solve), and
// the page-locked state readback buffers are pooled across contexts.
cudaError_t table_alloc(void** p, size_t bytes, cudaStream_t s) { return cudaMallocAsync(p, bytes, s); }
void table_free(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

std::mutex g_pin_mu;
std::vector<void*> g_pin_pool;

void* pinned_get(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_pool.empty()) {
      void* p = g_pin_pool.back();
      g_pin_pool.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, std::max<size_t>(bytes, 4096)) != cudaSuccess) return nullptr;
  return p;
}

void pinned_put(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_pool.push_back(p);
}

constexpr int B_COUNT_MAX = 32;

struct Layout {
  long long off[B_COUNT_MAX];
  long long end[B_COUNT_MAX];   // first byte past buffer i's payload (guard zone up to the next)
  long long total;
};

// RAPDB_GUARD=1: a 4 KB guard zone after every workspace buffer, filled with
// a byte pattern at bind time and verified by rapdb_check_guards -- the
// out-of-bounds-write check that stands in for compute-sanitizer (closed on
// the test pool).
constexpr long long kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;
bool guards_on() {
  const char* e = std::getenv("RAPDB_GUARD");
  return e && e[0] == '1';
}

enum WsBuf { B_X, B_U, B_GVAL, B_EQV, B_Y, B_YTR, B_GY, B_GXB, B_GXS, B_XCUM, B_YCUM, B_PART,
             B_SEGXU, B_SEGQX, B_ZQ, B_AUX, B_AUX2, B_ST, B_BAR, B_ABORT, B_H, B_HX, B_HXN, B_HY,
             B_W, B_PW2, B_PCX, B_PT, B_WL, B_EARLY, B_FPART, B_FCTR, B_COUNT };
static_assert(B_COUNT <= B_COUNT_MAX, "Layout::off too small");

// chunk counters + per-item flags of the packed sweep's early reduction
long long early_bytes(const rapdb_ctx* c) {
  return c->sp.layout == 1 ? 256 + 4LL * std::max(1LL, (long long)c->P.nact * c->sp.geom.nbB) : 256;
}

Layout layout_of(const rapdb_ctx* c) {
  const long long n = c->P.n, m = c->P.m, p = c->P.p, np = n > 0 ? p + m : 0;
  const long long G = c->G, nloc = c->P.nloc;
  long long sz[B_COUNT];
  sz[B_X] = 2 * n * 8;
  sz[B_U] = 2 * nloc * n * 8;
  sz[B_GVAL] = 2 * (m + 1) * 8;
  sz[B_EQV] = 2 * std::max(p, 1LL) * 8;
  sz[B_Y] = 2 * std::max(np, 1LL) * 8;
  sz[B_YTR] = std::max(np, 1LL) * 8;
  sz[B_GY] = 3 * std::max(np, 1LL) * 8;
  sz[B_GXB] = 3 * n * 8;
  sz[B_GXS] = n * 8;
  sz[B_XCUM] = n * 8;
  sz[B_YCUM] = std::max(np, 1LL) * 8;
  sz[B_PART] = (long long)NSLOT * G * 8;
  const bool packed = c->sp.layout == 1;
  const long long nseg = packed ? std::max(1LL, (long long)c->P.nact * c->sp.geom.nbB)
                                : G * kConsumerWarps * c->sp.segmax;
  sz[B_SEGXU] = nseg * 8;
  sz[B_SEGQX] = nseg * 8;
  sz[B_ZQ] = std::max(c->P.nzero, 1) * 8LL;
  sz[B_AUX] = n * 8;
  sz[B_AUX2] = n * 8;
  sz[B_H] = c->gap_ok ? n * n * 8 : 8;
  sz[B_HX] = n * 8;
  sz[B_HXN] = n * 8;
  sz[B_HY] = n * 8;
  sz[B_ST] = sizeof(SolverState);
  sz[B_BAR] = 64;
  sz[B_ABORT] = 128 + 16LL * G;   // flag + diagnostics + per-CTA progress beacons
  const bool fac = c->P.kind == 1;
  sz[B_W] = fac ? 2 * c->P.nr * 8 : 8;
  sz[B_PW2] = fac ? std::max(c->nchw, 1LL) * 8 : 8;
  sz[B_PCX] = fac ? (long long)std::max(c->P.fnb, 1) * c->P.nchx * 8 : 8;
  sz[B_PT] = packed ? std::max(1LL, (long long)c->P.nact) * c->sp.geom.nbB * c->sp.geom.nbB * sym::kB * 8 : 8;
  sz[B_WL] = fac ? std::max(c->P.nr, 1LL) * 8 : 8;
  sz[B_EARLY] = early_bytes(c);
  sz[B_FPART] = fac ? 2LL * std::max(c->P.nfpart, 1) * 8 : 8;
  sz[B_FCTR] = 64;
  Layout L;
  long long o = 0;
  const long long guard = c->guard ? kGuardBytes : 0;
  for (int i = 0; i < B_COUNT; ++i) {
    L.off[i] = o;
    L.end[i] = o + sz[i];
    o += align_up(sz[i], 256) + guard;
  }
  L.total = o;
  return L;
}

long long g_launches = 0;

int read_state(rapdb_ctx* c, SolverState* st);

int launch_once(rapdb_ctx* c, const RunCfg& rc) {
  KArgs K;
  K.P = c->P;
  K.prm = c->prm;
  K.sp = c->sp;
  K.w = c->w;
  K.rc = rc;
  K.px = c->px;
  // grid-barrier word and watchdog flag: neighbours in the workspace (one
  // memset unless guard zones sit between them)
  {
    const char* b0 = reinterpret_cast<const char*>(c->w.bar);
    const char* a0 = reinterpret_cast<const char*>(c->w.abort_flag);
    if (!c->guard && a0 > b0 && a0 - b0 <= 1024) {
      CK(cudaMemsetAsync(c->w.bar, 0, (size_t)(a0 - b0) + 128, c->stream));
    } else {
      CK(cudaMemsetAsync(c->w.bar, 0, 64, c->stream));
      CK(cudaMemsetAsync(c->w.abort_flag, 0, 128, c->stream));
    }
  }
  // an aborted launch can leave the early-reduction counters mid-sweep
  if (c->sp.layout == 1) CK(cudaMemsetAsync(c->w.ccnt, 0, early_bytes(c), c->stream));
  void* args[] = {&K};
  CK(cudaLaunchCooperativeKernel((const void*)rapdb_solver_kernel, dim3(c->G), dim3(kThreads), args,
                                 c->dyn_smem, c->stream));
  CK(cudaGetLastError());
  ++g_launches;
  return RAPDB_OK;
}

// The max-dynamic-shared-memory attribute is per function and process-wide:
// only ever raise it, so a context bound later with a smaller need cannot
// invalidate the launches of an earlier one.
std::mutex g_attr_mu;
cudaError_t raise_smem_attr(const void* f, int bytes) {
  static std::vector<std::pair<const void*, int>> seen;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  for (auto& e : seen)
    if (e.first == f) {
      if (bytes <= e.second) return cudaSuccess;
      const cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (r == cudaSuccess) e.second = bytes;
      return r;
    }
  const cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (r == cudaSuccess) seen.emplace_back(f, bytes);
  return r;
}

// A factored stop: run the requested sweep / gradient(s) / fused trial as
// standalone kernels (several CTAs per SM) on the context's stream, then the
// op resumes.  Dynamic shared memory of the factored kernels:
// opt the factored kernels into their shared memory (the per-block weight
// table rides in dynamic shared memory)
int fac_kernel_attrs(rapdb_ctx* c) {
  const DevProblem& P = c->P;
  const int wq = std::max(P.fnb, 1) * 8;
  const void* ks[] = {(const void*)fac_grad_kernel<true>, (const void*)fac_grad_kernel<false>,
                      (const void*)fac_wl_kernel};
  for (const void* f : ks) {
    cudaFuncAttributes fa{};
    CK(cudaFuncGetAttributes(&fa, f));
    if ((long long)fa.sharedSizeBytes + wq > (long long)c->optin)
      return fail(c, RAPDB_ECONFIG, "too many quadratic blocks for the factored kernels' shared memory");
    CK(raise_smem_attr(f, wq));
  }
  return RAPDB_OK;
}

// the gradient at W-cache Wpar with multipliers lam into out; TRIAL also
// takes the fused yx trial's primal step (exactly P.nfpart warps)
int fac_gradient(rapdb_ctx* c, const Work& w, const double* Wpar, const double* lam, double* out, bool trial,
                 double tau, int cur) {
  const DevProblem& P = c->P;
  const size_t wq = (size_t)std::max(P.fnb, 1) * 8;
  const double* Wsrc = Wpar;
  if (!P.rt_tag && !P.sym) {   // block-weighted W-cache first (a symmetric stack has no R^T to gather for)
    fac_wl_kernel<<<c->nsm * 8, kThreads, wq, c->stream>>>(P, w, Wpar, lam);
    Wsrc = w.wl;
    ++g_launches;
  }
  for (int ph = 0; ph < P.rt_nph; ++ph) {   // one launch per row phase: its slice of the W-cache stays in L2
    if (P.rt_tag) fac_grad_kernel<true><<<c->nsm * kGradCtas, kThreads, wq, c->stream>>>(P, w, Wsrc, lam, out, ph);
    else fac_grad_kernel<false><<<c->nsm * kGradCtas, kThreads, wq, c->stream>>>(P, w, Wsrc, lam, out, ph);
    ++g_launches;
  }
  const int fgrid = P.nfpart / kWarps;
  if (trial) fac_grad_fin_kernel<true><<<fgrid, kThreads, 0, c->stream>>>(P, w, out, tau, cur);
  else fac_grad_fin_kernel<false><<<fgrid, kThreads, 0, c->stream>>>(P, w, out, tau, cur);
  ++g_launches;
  return RAPDB_OK;
}

// the row pass at x into parity par
static void launch_row_pass(rapdb_ctx* c, const double* x, int par) {
  fac_row_kernel<<<c->nsm * kRowCtas, kThreads, 0, c->stream>>>(c->P, c->w, x, par);
  ++g_launches;
}

int serve_factored(rapdb_ctx* c, const RunCfg& rc, const SolverState& st) {
  const DevProblem& P = c->P;
  const Work& w = c->w;
  const long long n = P.n, np = (long long)P.p + P.m;
  if (st.fq[0] == 1) {
    const int par = st.fq[1];
    const double* x = st.fq[2] ? rc.in_x : w.x + (long long)par * n;
    launch_row_pass(c, x, par);
  } else if (st.fq[0] == 2) {
    for (int k = 0; k < st.fq[1] && k < 2; ++k) {
      const int par = st.fq[2 + 3 * k], lid = st.fq[3 + 3 * k], oid = st.fq[4 + 3 * k];
      const double* lam = lid == 0 ? w.ytr + P.p : lid == 1 ? w.y + P.p : lid == 2 ? w.y + np + P.p : rc.in_lam;
      double* out = oid == 0 ? w.gxs : w.gxb + (long long)st.ig_new * n;
      fac_gradient(c, w, w.W + (long long)par * P.nr, lam, out, false, 0.0, 0);
    }
  } else if (st.fq[0] == 3) {
    // the fused yx trial (unsharded): gradient + primal step, then the row
    // pass (W, |W|^2, A x - b, c_i . x) at x_new
    const int cur = st.fq[1];
    fac_gradient(c, w, w.W + (long long)cur * P.nr, w.ytr + P.p, w.gxs, true, st.tau, cur);
    launch_row_pass(c, w.x + (long long)(cur ^ 1) * n, cur ^ 1);
  } else {
    return fail(c, RAPDB_EDEVICE, "unknown factored request");
  }
  CK(cudaGetLastError());
  return RAPDB_OK;
}

// The buffers of exchange `kind` summed across ranks in rank order on the
// context's stream (no host synchronisation: the relaunch queues behind it).
int comm_exchange(rapdb_ctx* c, int kind) {
  double *b0 = nullptr, *b1 = nullptr;
  long long n0 = 0, n1 = 0;
  int r = rapdb_exchange_buffers(c, kind, &b0, &n0, &b1, &n1);
  if (r) return r;
  const rapdb_comm* m = c->comm;
  const char* what = "";
  for (int v = 0; v < 2; ++v) {
    double* b = v ? b1 : b0;
    const long long n = v ? n1 : n0;
    if (!b || n <= 0) continue;
    const int e = rcomm::ordered_allreduce(m->nccl, m->rank, m->nranks, b, n, c->xscratch, c->stream,
                                                c->nsm, &what);
    if (e) return fail(c, RAPDB_EDEVICE, std::string("rank-ordered exchange: ") + what);
  }
  return RAPDB_OK;
}

// Launch an op.  Single-rank contexts run it to completion in one launch
// (asynchronous).  Sharded contexts ("split") stop at every exchange point:
// the registered callback all-reduces the buffer rapdb_exchange_buffers names
// (NCCL over NVLink in the Python binding) and the op resumes in a new launch.
int launch(rapdb_ctx* c, RunCfg rc) {
  if (!c->bound || !c->have_params || !c->have_ws) return fail(c, RAPDB_ECONFIG, "context not fully bound");
  if (c->P.kind == 1 && c->P.rt_nph < 1)
    return fail(c, RAPDB_ECONFIG, "factored context has no R^T / A^T (rapdb_set_factored_transpose)");
  rc.split = c->split;
  rc.fac_host = c->fac_host;
  rc.p2p = c->p2p;
  rc.resume = 0;
  int r = launch_once(c, rc);
  if (r || (!c->split && !c->fac_host)) return r;
  for (;;) {
    r = read_state(c, &c->last_st);
    if (r) return r;
    if (c->last_st.status != ST_EXCHANGE) return RAPDB_OK;
    if (c->last_st.fq[0] != 0) {
      r = serve_factored(c, rc, c->last_st);
      if (r) return r;
    }
    if (c->split && c->last_st.xkind != X_NONE) {
      if (c->comm) {
        r = comm_exchange(c, c->last_st.xkind);
        if (r) return r;
      } else {
        if (!c->xcb) return fail(c, RAPDB_ECONFIG, "sharded context has no exchange callback");
        if (c->xcb(c->xuser, c->last_st.xkind) != 0) return fail(c, RAPDB_EDEVICE, "exchange callback failed");
      }
      ++c->exchanges;
    }
    rc.resume = 1;
    r = launch_once(c, rc);
    if (r) return r;
  }
}

// The host side of the watchdog: if an op does not finish within 120 s, read
// the per-CTA progress beacons over a non-blocking stream (the kernel is still
// resident) and fail with them instead of blocking forever.
int wait_stream(rapdb_ctx* c) {
  EventGuard eg;
  CK(cudaEventCreateWithFlags(&eg.ev[0], cudaEventDisableTiming));
  cudaEvent_t ev = eg.ev[0];
  CK(cudaEventRecord(ev, c->stream));
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return cuda_fail(c, q, "kernel");
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
      cudaStream_t ds;
      std::vector<int> b(4 * c->G + 32, -1);
      if (cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking) == cudaSuccess) {
        cudaMemcpyAsync(b.data(), c->w.abort_flag, b.size() * sizeof(int), cudaMemcpyDeviceToHost, ds);
        cudaStreamSynchronize(ds);
      }
      std::string msg = "op did not finish within 120 s (device hang); per-CTA step/gen/iter/pseq:";
      for (int i = 0; i < c->G; ++i) {
        const int* v = b.data() + 32 + 4 * i;
        char t[64];
        std::snprintf(t, sizeof t, " %d:%d/%d/%d/%d", i, v[0], v[1], v[2], v[3]);
        msg += t;
      }
      std::fprintf(stderr, "[rapdb] %s\n", msg.c_str());
      c->err = msg;
      return RAPDB_EDEVICE;
    }
    // spin for the first 2 ms (a sharded run comes back here at every
    // exchange point, typically after tens of microseconds), then back off
    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(2))
      std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
  return RAPDB_OK;
}

int read_state(rapdb_ctx* c, SolverState* st) {
  int ab = 0;
  {
    const int wr = wait_stream(c);   // poll first: a pageable D2H copy would block behind a hung kernel
    if (wr) return wr;
  }
  if (!c->h_state) {
    static_assert(sizeof(SolverState) + 64 <= 4096, "pinned state buffer");
    c->h_state = static_cast<SolverState*>(pinned_get(sizeof(SolverState) + 64));
    if (!c->h_state) return fail(c, RAPDB_EDEVICE, "cudaMallocHost failed");
  }
  int* h_ab = reinterpret_cast<int*>(reinterpret_cast<char*>(c->h_state) + sizeof(SolverState));
  CK(cudaMemcpyAsync(c->h_state, c->w.st, sizeof(SolverState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *st = *c->h_state;
  // a stop on the way (exchange point / factored request) left through the
  // normal exit: every abort path sets ST_ABORT, so the watchdog flag is only
  // fetched when the op ended -- one copy less per stop
  if (st->status != ST_EXCHANGE) {
    CK(cudaMemcpyAsync(h_ab, c->w.abort_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    ab = *h_ab;
  }
  if (ab) {
    int info[20] = {0};
    cudaMemcpy(info, c->w.abort_flag, sizeof(info), cudaMemcpyDeviceToHost);
    char buf[512];
    std::snprintf(buf, sizeof buf, "device watchdog fired (%s): cta=%d thread=%d parity=%d waited_ms=%d bar=0x%x "
                  "issued=%d slot=%d use=%d ntiles=%d base=%d prog=[%d %d %d %d %d %d %d %d]",
                  ab == 2 ? "bulk-copy pipeline timeout" : ab == 1 ? "grid barrier timeout" :
                  ab == 3 ? "ring slot holds another tile (seq/slot/tag/use/base in issued..base)" :
                  ab == 4 ? "ring slot released by another tile (seq/slot/rel in issued..use)" : "abort flag corrupted",
                  info[1], info[2], info[3], info[4], info[5], info[6], info[7], info[8], info[9], info[10],
                  info[11], info[12], info[13], info[14], info[15], info[16], info[17], info[18]);
    return fail(c, RAPDB_EDEVICE, buf);
  }
  return RAPDB_OK;
}

}  // namespace

extern "C" {

int rapdb_abi_version(void) { return 1; }

long long rapdb_launch_count(void) { return g_launches; }

int rapdb_set_exchange(rapdb_ctx* c, rapdb_exchange_fn fn, void* user, int force_split) {
  if (!c) return RAPDB_EINPUT;
  c->xcb = fn;
  c->xuser = user;
  c->split = (c->nranks > 1 || force_split) ? 1 : 0;
  return RAPDB_OK;
}

int rapdb_exchange_buffers(rapdb_ctx* c, int kind, double** b0, long long* n0, double** b1, long long* n1) {
  if (!c || !b0 || !n0 || !b1 || !n1 || !c->have_ws) return RAPDB_EINPUT;
  const SolverState& st = c->last_st;
  const long long n = c->P.n, m = c->P.m;
  *b1 = nullptr;
  *n1 = 0;
  switch (kind) {
    case X_GX: *b0 = c->w.gxs; *n0 = n; break;
    case X_G: *b0 = c->w.gval + (long long)(st.cur ^ 1) * (m + 1); *n0 = m + 1; break;
    case X_GX2:
      *b0 = c->w.gxs; *n0 = n;
      *b1 = c->w.gxb + (long long)st.ig_new * n; *n1 = n;
      break;
    case X_H: *b0 = c->w.H; *n0 = n * n; break;
    default: return fail(c, RAPDB_EINPUT, "unknown exchange kind");
  }
  return RAPDB_OK;
}

long long rapdb_exchange_count(const rapdb_ctx* c) { return c ? c->exchanges : -1; }

int rapdb_comm_unique_id(unsigned char* id128) {
  if (!id128) return RAPDB_EINPUT;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return RAPDB_EDEVICE;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof(id));
  return RAPDB_OK;
}

int rapdb_comm_create(int device, const unsigned char* id128, int rank, int nranks, rapdb_comm** out) {
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return RAPDB_EINPUT;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return RAPDB_EDEVICE;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  rapdb_comm* m = new rapdb_comm();
  m->device = device;
  m->rank = rank;
  m->nranks = nranks;
  if (ncclCommInitRank(&m->nccl, nranks, id, rank) != ncclSuccess) {
    delete m;
    return RAPDB_EDEVICE;
  }
  *out = m;
  return RAPDB_OK;
}

void rapdb_comm_destroy(rapdb_comm* m) {
  if (!m) return;
  if (m->nccl) ncclCommDestroy(m->nccl);
  delete m;
}

int rapdb_comm_allreduce_ordered(rapdb_comm* m, double* buf, long long count, void* stream) {
  if (!m || (!buf && count > 0) || count < 0) return RAPDB_EINPUT;
  rcomm::Scratch sc;
  const char* what = "";
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rcomm::ordered_allreduce(m->nccl, m->rank, m->nranks, buf, count, sc, s, nsm, &what)) return RAPDB_EDEVICE;
  // the scratch is freed on return: finish the queued work first
  return cudaStreamSynchronize(s) == cudaSuccess ? RAPDB_OK : RAPDB_EDEVICE;
}

int rapdb_set_comm_exchange(rapdb_ctx* c, rapdb_comm* m, int force_split) {
  if (!c || !m) return RAPDB_EINPUT;
  if (m->nranks != c->nranks || m->rank != c->rank)
    return fail(c, RAPDB_ECONFIG, "communicator rank/size differ from the context's");
  if (m->device != c->device) return fail(c, RAPDB_ECONFIG, "communicator is on another device");
  c->comm = m;
  c->xcb = nullptr;
  c->split = (c->nranks > 1 || force_split) ? 1 : 0;
  return RAPDB_OK;
}

// ---- in-kernel peer exchange (sharded dense contexts) ---------------------
namespace {
long long peer_slot_doubles(const rapdb_ctx* c) { return 2LL * c->P.n + c->P.m + 1; }
}

long long rapdb_peer_region_bytes(rapdb_ctx* c) {
  if (!c || !c->bound || c->P.kind != 0) return -1;
  const long long R = c->nranks, S = peer_slot_doubles(c);
  return 2 * R * S * 8 + R * 16 * 8;
}

int rapdb_region_alloc(long long bytes, void** out) {
  if (bytes <= 0 || !out) return RAPDB_EINPUT;
  if (cudaMalloc(out, (size_t)bytes) != cudaSuccess) return RAPDB_EDEVICE;
  if (cudaMemset(*out, 0, (size_t)bytes) != cudaSuccess) return RAPDB_EDEVICE;
  return cudaDeviceSynchronize() == cudaSuccess ? RAPDB_OK : RAPDB_EDEVICE;
}

int rapdb_region_free(void* p) {
  if (!p) return RAPDB_EINPUT;
  return cudaFree(p) == cudaSuccess ? RAPDB_OK : RAPDB_EDEVICE;
}

int rapdb_ipc_handle(const void* dptr, unsigned char* out) {
  if (!dptr || !out) return RAPDB_EINPUT;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)) != cudaSuccess) return RAPDB_EDEVICE;
  static_assert(sizeof(h) <= 64, "ipc handle");
  std::memcpy(out, &h, sizeof(h));
  return RAPDB_OK;
}

int rapdb_ipc_open(const unsigned char* handle, void** out) {
  if (!handle || !out) return RAPDB_EINPUT;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? RAPDB_OK : RAPDB_EDEVICE;
}

int rapdb_ipc_close(void* p) {
  if (!p) return RAPDB_EINPUT;
  return cudaIpcCloseMemHandle(p) == cudaSuccess ? RAPDB_OK : RAPDB_EDEVICE;
}

int rapdb_set_peer_exchange(rapdb_ctx* c, void* const* regions) {
  if (!c || !regions) return RAPDB_EINPUT;
  if (!c->bound || c->P.kind != 0) return fail(c, RAPDB_ECONFIG, "peer exchange needs a bound dense context");
  const int R = c->nranks;
  const long long S = peer_slot_doubles(c);
  std::vector<void*> tab(2 * (size_t)R);
  for (int r = 0; r < R; ++r) {
    if (!regions[r] || (reinterpret_cast<uintptr_t>(regions[r]) & 127)) return fail(c, RAPDB_EINPUT, "bad peer region");
    tab[r] = regions[r];
    tab[R + r] = static_cast<char*>(regions[r]) + 2 * R * S * 8;
  }
  table_free(c->d_px, c->stream);
  c->d_px = nullptr;
  CK(table_alloc(&c->d_px, tab.size() * sizeof(void*), c->stream));
  CK(cudaMemcpyAsync(c->d_px, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  PeerX px{};
  px.slots = reinterpret_cast<double* const*>(c->d_px);
  px.flags = reinterpret_cast<unsigned long long* const*>(static_cast<void**>(c->d_px) + R);
  px.S = S;
  px.rank = c->rank;
  px.R = R;
  c->px = px;
  c->p2p = 1;
  return RAPDB_OK;
}

int rapdb_step_profile(rapdb_ctx* c, double* ns, long long* counts, int nsteps) {
  if (!c || !ns || !counts || !c->have_ws) return RAPDB_EINPUT;
  SolverState st;
  int r = read_state(c, &st);
  if (r) return r;
  for (int i = 0; i < nsteps && i < 64; ++i) {
    ns[i] = st.step_ns[i];
    counts[i] = st.step_cnt[i];
  }
  return RAPDB_OK;
}

int rapdb_create(int device, int rank, int nranks, rapdb_ctx** out) {
  if (!out) return RAPDB_EINPUT;
  *out = nullptr;
  rapdb_ctx* c = new rapdb_ctx();
  c->device = device;
  c->rank = rank;
  c->nranks = nranks;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete c;
    return RAPDB_EDEVICE;
  }
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  c->nsm = v;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  c->optin = (size_t)v;
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  if (!coop || c->nsm <= 0) {
    delete c;
    return RAPDB_EDEVICE;
  }
  *out = c;
  return RAPDB_OK;
}

void rapdb_destroy(rapdb_ctx* c) {
  if (!c) return;
  table_free(c->d_ints, c->stream);
  table_free(c->d_ll, c->stream);
  table_free(c->d_sell, c->stream);
  table_free(c->d_units, c->stream);
  table_free(c->d_px, c->stream);
  pinned_put(c->h_state);
  delete c;
}

int rapdb_last_error(const rapdb_ctx* c, char* buf, int size) {
  if (!c || !buf || size <= 0) return RAPDB_EINPUT;
  std::snprintf(buf, (size_t)size, "%s", c->err.c_str());
  return RAPDB_OK;
}

int rapdb_set_stream(rapdb_ctx* c, void* s) {
  if (!c) return RAPDB_EINPUT;
  c->stream = static_cast<cudaStream_t>(s);
  return RAPDB_OK;
}

namespace {
int bind_dense_impl(rapdb_ctx* c, int layout, int n, int m, int p, int k0, int k1, long long ld, const double* Q,
                    const double* q, const double* r, const double* A, const double* b,
                    const double* lower, const double* upper, double mu, const unsigned char* zero_flags);
}

int rapdb_bind_dense(rapdb_ctx* c, int n, int m, int p, int k0, int k1, long long ld, const double* Q,
                     const double* q, const double* r, const double* A, const double* b,
                     const double* lower, const double* upper, double mu, const unsigned char* zero_flags) {
  return bind_dense_impl(c, 0, n, m, p, k0, k1, ld, Q, q, r, A, b, lower, upper, mu, zero_flags);
}

int rapdb_bind_dense_packed(rapdb_ctx* c, int n, int m, int p, int k0, int k1, const double* Qp,
                            const double* q, const double* r, const double* A, const double* b,
                            const double* lower, const double* upper, double mu, const unsigned char* zero_flags) {
  return bind_dense_impl(c, 1, n, m, p, k0, k1, n + (n & 1), Qp, q, r, A, b, lower, upper, mu, zero_flags);
}

long long rapdb_packed_doubles(int n) {
  if (n <= 0) return -1;
  return sym::make_geom(n).spm * sym::kTD;
}

int rapdb_pack_symmetric(int n, long long count, const double* src, long long ld, long long mat_stride,
                         double* dst, void* stream) {
  if (n <= 0 || count < 0 || ld < n || mat_stride < (long long)n * ld - (ld - n) || !src || !dst) return RAPDB_EINPUT;
  if (count == 0) return RAPDB_OK;
  const sym::Geom g = sym::make_geom(n);
  std::vector<sym::Unit> hu(g.upm);
  sym::fill_units(g, hu.data());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  sym::Unit* du = nullptr;
  if (cudaMallocAsync(&du, hu.size() * sizeof(sym::Unit), st) != cudaSuccess) return RAPDB_EDEVICE;
  if (cudaMemcpyAsync(du, hu.data(), hu.size() * sizeof(sym::Unit), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return RAPDB_EDEVICE;
  for (long long a0 = 0; a0 < count; a0 += 65535) {
    const int cnt = (int)std::min(65535LL, count - a0);
    sym::pack_kernel<<<dim3(g.upm, cnt), 256, 0, st>>>(g, du, src + a0 * mat_stride, ld, mat_stride,
                                                         dst + a0 * g.spm * sym::kTD);
    ++g_launches;
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(du, st);
  if (e != cudaSuccess) return RAPDB_EDEVICE;
  return cudaStreamSynchronize(st) == cudaSuccess ? RAPDB_OK : RAPDB_EDEVICE;
}

namespace {
int bind_dense_impl(rapdb_ctx* c, int layout, int n, int m, int p, int k0, int k1, long long ld, const double* Q,
                    const double* q, const double* r, const double* A, const double* b,
                    const double* lower, const double* upper, double mu, const unsigned char* zero_flags) {
  if (!c) return RAPDB_EINPUT;
  if (n <= 0 || m < 0 || p < 0) return fail(c, RAPDB_EINPUT, "need n > 0, m >= 0, p >= 0");
  if (k0 < 0 || k1 > m + 1 || k1 <= k0) return fail(c, RAPDB_EINPUT, "bad local matrix range");
  if (ld < n || (ld & 1)) return fail(c, RAPDB_EINPUT, "ld must be even and >= n");
  if (layout == 1 && n > 32767 * 64) return fail(c, RAPDB_EINPUT, "n too large for the packed layout");
  if (c->nranks == 1 && (k0 != 0 || k1 != m + 1) && !c->split)
    return fail(c, RAPDB_EINPUT, "a single-rank context must hold all m+1 matrices (or be split)");
  if (c->nranks > 1) c->split = 1;
  if (!Q || !q || !r || !lower || !upper || (p > 0 && (!A || !b)))
    return fail(c, RAPDB_EINPUT, "null data pointer");
  if ((reinterpret_cast<uintptr_t>(Q) & 15) != 0) return fail(c, RAPDB_EINPUT, "Q must be 16-byte aligned");
  const int nloc = k1 - k0;
  std::vector<int> act, zl, slot(nloc);
  for (int i = 0; i < nloc; ++i) {
    if (zero_flags && zero_flags[i]) {
      slot[i] = -(int)zl.size() - 1;
      zl.push_back(i);
    } else {
      slot[i] = (int)act.size();
      act.push_back(i);
    }
  }
  // sweep plan: rows per tile, ring depth, shared memory
  const long long row_bytes = ld * 8;
  // ~16 KB bulk copies (whole rows up to 48 KB), 12-16-deep ring: measured at
  // ~6.9 TB/s for the C1 sweep on B200 (tools/profile_sweep.py); env knobs
  // RAPDB_TILE_BYTES / RAPDB_STAGES / RAPDB_ROW_TILE_MAX exist for tuning runs.
  const char* env_tile = std::getenv("RAPDB_TILE_BYTES");
  const char* env_st = std::getenv("RAPDB_STAGES");
  const char* env_rt = std::getenv("RAPDB_ROW_TILE_MAX");
  const long long tile_target = env_tile ? std::max(1024LL, std::atoll(env_tile)) : 16384;
  const long long max_stages = std::min(32LL, env_st ? std::max(2LL, std::atoll(env_st)) : 16LL);
  const long long row_tile_max = env_rt ? std::atoll(env_rt) : 49152;
  SweepPlan sp{};
  if (row_bytes > tile_target && row_bytes <= row_tile_max) {   // one whole row per tile
    sp.TR = 1;
    sp.cpr = 1;
    sp.chunk = (int)ld;
    sp.stage_bytes = align_up(row_bytes, 128);
  } else if (row_bytes <= tile_target) {
    int TR = 1;
    while (TR * 2 <= kMaxTR && (long long)(TR * 2) * row_bytes <= tile_target) TR *= 2;
    sp.TR = TR;
    sp.cpr = 1;
    sp.chunk = (int)ld;
    sp.stage_bytes = align_up((long long)TR * row_bytes, 128);
  } else {
    sp.TR = 1;
    sp.chunk = (int)(tile_target / 16 * 2);          // even number of doubles
    sp.cpr = (int)((ld + sp.chunk - 1) / sp.chunk);
    sp.stage_bytes = align_up((long long)sp.chunk * 8, 128);
  }
  sp.xs_bytes = align_up(row_bytes, 128);
  sp.layout = layout;
  if (layout == 1) {
    // packed symmetric stack: one unit (<= 4 sub-tiles, 32 KB) per ring slot,
    // x staged zero-padded to whole 64-row blocks
    sp.geom = sym::make_geom(n);
    sp.TR = 1;
    sp.cpr = 1;
    sp.chunk = (int)ld;
    sp.stage_bytes = 4LL * sym::kTD * 8;
    sp.xs_bytes = align_up((long long)sp.geom.nbB * sym::kB * 8, 128);
    // x does not fit next to a 2-slot ring (n > ~19 500), or forced: every
    // consumer warp loads its unit's two 64-entry x blocks instead
    const long long budget0 = (long long)c->optin - 16384 - 2048;
    const char* env_xg = std::getenv("RAPDB_XGLOBAL");
    sp.xglobal = (env_xg && env_xg[0] == '1') || sp.xs_bytes + 2 * sp.stage_bytes + 256 > budget0;
    if (sp.xglobal) sp.xs_bytes = align_up((long long)kConsumerWarps * 128 * 8, 128);
  }
  const char* env_rc = std::getenv("RAPDB_RC_COLS");
  sp.rc_cols = env_rc ? std::atoi(env_rc) : (k1 - k0 >= 24 ? 1 : 0);
  cudaFuncAttributes fa{};
  long long static_smem = 16384;
  if (cudaFuncGetAttributes(&fa, (const void*)rapdb_solver_kernel) == cudaSuccess)
    static_smem = (long long)fa.sharedSizeBytes;
  // dynamic = x staging + ring + 2 mbarriers per slot, within the per-block opt-in
  long long ns = ((long long)c->optin - static_smem - sp.xs_bytes - 128) / (sp.stage_bytes + 16);
  ns = std::min(ns, layout == 1 ? std::min(max_stages, 8LL) : max_stages);
  if (ns < 2) return fail(c, RAPDB_ECONFIG, "n too large for the dense path (x does not fit in shared memory)");
  // consumer warp k owns every ncw-th slot use and waits on the slot's full
  // mbarrier by phase parity: every use of a slot must go to the same warp,
  // so the stage count is a multiple of the consumer-warp count
  if (ns > kConsumerWarps) ns -= ns % kConsumerWarps;
  sp.nstages = (int)ns;
  sp.ncw = (int)std::min<long long>(kConsumerWarps, ns);
  if (sp.nstages % sp.ncw != 0) return fail(c, RAPDB_ECONFIG, "ring stages not a multiple of the consumer warps");
  // packed sweep: the consumer warp without a ring slot reduces the unit
  // partials of finished matrix chunks while later chunks stream
  // (RAPDB_EARLY_CHUNKS, 0 = everything after the stream)
  if (layout == 1 && sp.ncw < kConsumerWarps) {
    const char* env_ec = std::getenv("RAPDB_EARLY_CHUNKS");
    // default with enough matrices to spread (C1, C2): chunks of <= ~24 MB of
    // unit partials, so a chunk's partials are still in L2 when reduced (C2:
    // 43 chunks, 5.80 -> 5.43 ms per sweep; C1: 8, 0.538 -> 0.509 ms); with
    // a handful of matrices (C4: 4) the mid-stream fences cost more than phase B
    const long long pt_bytes = (long long)act.size() * sp.geom.nbB * sp.geom.nbB * sym::kB * 8;
    const long long by_l2 = (pt_bytes + (24LL << 20) - 1) / (24LL << 20);
    const int want = env_ec ? std::atoi(env_ec) : (act.size() >= 16 ? (int)std::max(8LL, by_l2) : 0);
    sp.nchunk = (int)std::max(0LL, std::min<long long>({(long long)want, 64LL, (long long)act.size()}));
    if (sp.nchunk == 1) sp.nchunk = 0;
  }
  c->dyn_smem = (size_t)(sp.xs_bytes + ns * sp.stage_bytes + 2 * ns * 8);
  c->stage_cap = ns * sp.stage_bytes / 8;
  // smoothed gap: five shared n-vectors + staged multipliers in xs+ring, and a
  // dense n x n H in the workspace (skipped for very large n)
  c->gap_ok = (5LL * n + m + p + m + 64) * 8 <= sp.xs_bytes + ns * sp.stage_bytes && n <= 16384;
  if (layout == 1)   // per-warp 32 x 33 transpose buffers after the staged multipliers (gap.cuh)
    c->gap_ok = c->gap_ok && align_up((long long)m * 8, 256) + kWarps * 32LL * 33 * 8 <= ns * sp.stage_bytes;
  // the staged duals and the recombination scratch at the ring's end must not meet
  if (2LL * (p + m) + kWarps * 32 > c->stage_cap)
    return fail(c, RAPDB_ECONFIG, "too many multipliers for the shared-memory dual staging area");
  cudaError_t e = raise_smem_attr((const void*)rapdb_solver_kernel, (int)c->dyn_smem);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaFuncSetAttribute");
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)rapdb_solver_kernel, kThreads, c->dyn_smem);
  if (e != cudaSuccess) return cuda_fail(c, e, "occupancy");
  if (occ < 1) return fail(c, RAPDB_EDEVICE, "solver kernel cannot be resident");
  c->G = c->nsm * occ;
  if (c->G > 256) c->G = 256;   // get_totals keeps <= 8 partials per lane
  if (const char* eg = std::getenv("RAPDB_GRID")) {   // experiment knob: fewer CTAs
    const int g = std::atoi(eg);
    if (g >= 1 && g < c->G) c->G = g;
  }
  const int G = c->G;
  // row partition of the streamed rows over CTAs and the segment tables
  const long long R = (long long)act.size() * n;
  sp.rows_total = R;
  std::vector<int> cta_a0(G, 0), seg_lo(std::max<size_t>(act.size(), 1), 0), seg_hi(std::max<size_t>(act.size(), 1), -1);
  int segmax = 1;
  for (int bb = 0; bb < G; ++bb) {
    const long long rs = (long long)bb * R / G, re = (long long)(bb + 1) * R / G;
    if (rs >= re) {
      cta_a0[bb] = -1;
      continue;
    }
    const int a_lo = (int)(rs / n), a_hi = (int)((re - 1) / n);
    cta_a0[bb] = a_lo;
    segmax = std::max(segmax, a_hi - a_lo + 1);
    for (int a = a_lo; a <= a_hi; ++a) {
      if (seg_hi[a] < 0) seg_lo[a] = bb;
      seg_hi[a] = bb;
    }
  }
  sp.segmax = segmax;
  std::vector<int> ints;
  auto put = [&](const std::vector<int>& v) {
    size_t o = ints.size();
    ints.insert(ints.end(), v.begin(), v.end());
    if (v.empty()) ints.push_back(0);
    return o;
  };
  const size_t o_act = put(act), o_zl = put(zl), o_lo = put(seg_lo), o_hi = put(seg_hi),
               o_a0 = put(cta_a0), o_slot = put(slot);
  table_free(c->d_ints, c->stream);
  c->d_ints = nullptr;
  CK(table_alloc(reinterpret_cast<void**>(&c->d_ints), ints.size() * sizeof(int), c->stream));
  CK(cudaMemcpyAsync(c->d_ints, ints.data(), ints.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  DevProblem P{};
  P.n = n; P.m = m; P.p = p; P.k0 = k0; P.k1 = k1; P.nloc = nloc;
  P.nact = (int)act.size(); P.nzero = (int)zl.size(); P.ld = ld;
  P.Q = Q; P.q = q; P.r = r; P.A = A; P.b = b; P.lo = lower; P.hi = upper; P.mu = mu;
  P.act = c->d_ints + o_act; P.zero_list = c->d_ints + o_zl; P.seg_lo = c->d_ints + o_lo;
  P.seg_hi = c->d_ints + o_hi; P.cta_a0 = c->d_ints + o_a0; P.mat_slot = c->d_ints + o_slot;
  c->P = P;
  c->sp = sp;
  c->sweep_bytes = R * (long long)n * 8;
  c->fac_host = 0;
  if (layout == 1) {
    // the unit table rides in its own allocation (8-byte entries)
    table_free(c->d_units, c->stream);
    c->d_units = nullptr;
    std::vector<sym::Unit> hu(sp.geom.upm);
    sym::fill_units(sp.geom, hu.data());
    CK(table_alloc(reinterpret_cast<void**>(&c->d_units), hu.size() * sizeof(sym::Unit), c->stream));
    CK(cudaMemcpyAsync(c->d_units, hu.data(), hu.size() * sizeof(sym::Unit), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->sp.units = c->d_units;
    c->sweep_bytes = (long long)act.size() * sp.geom.spm * sym::kTD * 8;   // packed bytes streamed
  }
  c->nchw = 0;
  c->bound = true;
  c->have_ws = false;
  return RAPDB_OK;
}
}  // namespace

int rapdb_bind_factored(rapdb_ctx* c, int n, int mq, int L, long long nr, const rapdb_sell* R, const int* rmat,
                        const long long* rblk, const double* C, const double* d, const rapdb_sell* A,
                        const double* b, const double* lower, const double* upper, double mu) {
  return rapdb_bind_factored_range(c, n, mq, L, 0, mq + 1, 0, L, nr, R, rmat, rblk, C, d, A, b, lower, upper, mu);
}

// a caller's Sell descriptor checked against the expected slot count; the
// entry total (sp[last]) is read back for the byte accounting
static int take_sell(rapdb_ctx* c, const rapdb_sell* in, long long want_slots, bool need_map, const char* name,
                     Sell* out, long long* entries) {
  *out = Sell{};
  *entries = 0;
  if (!in) return fail(c, RAPDB_EINPUT, std::string("null Sell descriptor: ") + name);
  if (in->nslots != want_slots || (in->nslots & 31))
    return fail(c, RAPDB_EINPUT, std::string("Sell slot count mismatch: ") + name);
  if (!in->sp || (in->nslots > 0 && (!in->len || (need_map && !in->map))))
    return fail(c, RAPDB_EINPUT, std::string("null Sell array: ") + name);
  CK(cudaMemcpy(entries, in->sp + (in->nslots >> 5), 8, cudaMemcpyDeviceToHost));
  if (*entries < 0 || (*entries & 31) || (*entries > 0 && (!in->idx || !in->val)))
    return fail(c, RAPDB_EINPUT, std::string("bad Sell entry arrays: ") + name);
  out->nslots = in->nslots; out->entries = *entries; out->sp = in->sp; out->idx = in->idx; out->val = in->val;
  out->len = in->len; out->map = in->map;
  return RAPDB_OK;
}

int rapdb_bind_factored_range(rapdb_ctx* c, int n, int mq, int L, int fb0, int fb1, int l0, int l1, long long nr,
                              const rapdb_sell* R, const int* rmat, const long long* rblk, const double* C,
                              const double* d, const rapdb_sell* A, const double* b,
                              const double* lower, const double* upper, double mu) {
  if (!c) return RAPDB_EINPUT;
  if (n <= 0 || mq < 0 || L < 0 || nr < 0) return fail(c, RAPDB_EINPUT, "need n > 0, mq >= 0, L >= 0, nr >= 0");
  if (fb0 < 0 || fb1 > mq + 1 || fb1 < fb0 || l0 < 0 || l1 > L || l1 < l0)
    return fail(c, RAPDB_EINPUT, "bad local block / linear-row range");
  const int fnb = fb1 - fb0, Lloc = l1 - l0;
  const bool whole = fnb == mq + 1 && Lloc == L;
  if (c->nranks == 1 && !whole && !c->split)
    return fail(c, RAPDB_EINPUT, "a single-rank context must hold the whole instance (or be split)");
  if (c->nranks > 1) c->split = 1;
  if (!rblk || (fnb > 0 && (!C || !d)) || !lower || !upper || (nr > 0 && !rmat) || (Lloc > 0 && !b))
    return fail(c, RAPDB_EINPUT, "null data pointer");
  if (rblk[0] != 0 || rblk[fnb] != nr) return fail(c, RAPDB_EINPUT, "rblk must run from 0 to nr");
  // d_ll: [fnb+1] local block row offsets, then [fnb+1] prefix counts of W chunks
  std::vector<long long> ll(2 * (size_t)(fnb + 1));
  for (int i = 0; i < fnb; ++i) {
    if (rblk[i + 1] < rblk[i]) return fail(c, RAPDB_EINPUT, "rblk must be nondecreasing");
    ll[i] = rblk[i];
    ll[fnb + 1 + i + 1] = ll[fnb + 1 + i] + (rblk[i + 1] - rblk[i] + kWChunk - 1) / kWChunk;   // W chunks
  }
  ll[fnb] = nr;
  const long long nchw = ll[2 * (fnb + 1) - 1];
  table_free(c->d_ll, c->stream);
  c->d_ll = nullptr;
  CK(table_alloc(reinterpret_cast<void**>(&c->d_ll), ll.size() * sizeof(long long), c->stream));
  CK(cudaMemcpyAsync(c->d_ll, ll.data(), ll.size() * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  table_free(c->d_ints, c->stream);
  c->d_ints = nullptr;
  CK(table_alloc(reinterpret_cast<void**>(&c->d_ints), 16, c->stream));
  CK(cudaMemsetAsync(c->d_ints, 0, 16, c->stream));
  long long nnz_r = 0, nnz_a = 0;   // stored entries incl. slice padding: the bytes actually streamed
  Sell sr{}, sa{};
  {
    int e = take_sell(c, R, nchw * kWChunk, false, "R", &sr, &nnz_r);
    if (e) return e;
    e = take_sell(c, A, ((long long)Lloc + 31) / 32 * 32, false, "A", &sa, &nnz_a);
    if (e) return e;
  }
  // no streamed sweep: the ring degenerates to the multiplier staging area
  SweepPlan sp{};
  sp.TR = 1; sp.cpr = 1; sp.chunk = 2; sp.nstages = 1; sp.ncw = 1; sp.segmax = 1;
  sp.rc_cols = 1;   // the recombination ends warp-per-column: barrier before the primal step
  sp.stage_bytes = align_up((long long)(kWarps + 1) * std::max(fnb, 1) * 8, 128);   // wq / c_i . x sums
  sp.xs_bytes = 0;
  sp.rows_total = 0;
  c->dyn_smem = (size_t)(sp.stage_bytes + 16);
  c->stage_cap = sp.stage_bytes / 8;
  c->gap_ok = false;
  if ((long long)c->dyn_smem + 4096 > (long long)c->optin)
    return fail(c, RAPDB_ECONFIG, "too many quadratic constraints for the staging area");
  cudaError_t e = raise_smem_attr((const void*)rapdb_solver_kernel, (int)c->dyn_smem);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaFuncSetAttribute");
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)rapdb_solver_kernel, kThreads, c->dyn_smem);
  if (e != cudaSuccess) return cuda_fail(c, e, "occupancy");
  if (occ < 1) return fail(c, RAPDB_EDEVICE, "solver kernel cannot be resident");
  c->G = c->nsm * 1;   // one CTA per SM: grid barriers stay cheap
  DevProblem P{};
  const int m = mq + L;
  P.n = n; P.m = m; P.p = 0; P.k0 = 0; P.k1 = m + 1; P.nloc = 0; P.nact = 0; P.nzero = 0; P.ld = n;
  P.Q = nullptr; P.q = C; P.r = d; P.A = nullptr; P.b = b; P.lo = lower; P.hi = upper; P.mu = mu;
  P.act = P.zero_list = P.seg_lo = P.seg_hi = P.cta_a0 = P.mat_slot = c->d_ints;
  P.kind = 1; P.mq = mq; P.nr = nr; P.L = L; P.nchx = (n + kCxCols - 1) / kCxCols;
  P.nfpart = c->nsm * 4 * kWarps;   // fused-trial gradient grid: 4 CTAs per SM
  P.fb0 = fb0; P.fnb = fnb; P.l0 = l0; P.Lloc = Lloc;
  // the Sell descriptors live in a device table (DevProblem::sell); R^T / A^T
  // arrive with rapdb_set_factored_transpose (required before any op)
  std::memset(c->h_sell, 0, sizeof c->h_sell);
  c->h_sell[kSellR] = sr; c->h_sell[kSellA] = sa;
  table_free(c->d_sell, c->stream);
  c->d_sell = nullptr;
  CK(table_alloc(reinterpret_cast<void**>(&c->d_sell), sizeof c->h_sell, c->stream));
  CK(cudaMemcpyAsync(c->d_sell, c->h_sell, sizeof c->h_sell, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  P.sell = c->d_sell;
  P.sym = 0;
  P.rt_nph = 0; P.rt_tag = 0;
  P.rmat = rmat; P.rblk = c->d_ll; P.wch = c->d_ll + (fnb + 1);
  c->P = P;
  c->sp = sp;
  c->nchw = nchw;
  c->fac_host = 1;   // every factored sweep / gradient is a stop served by standalone kernels
  // one factored sweep: R (12 B/nnz + row pointers) streamed, W written and
  // re-read, C and A (+ b) read, x gathered once
  c->sweep_bytes = 12 * nnz_r + 4 * sr.nslots + 16 * nr + 8LL * fnb * n + 12 * nnz_a + 4 * sa.nslots + 16LL * Lloc +
                   8LL * n;
  {
    const int ra = fac_kernel_attrs(c);
    if (ra) return ra;
  }
  c->bound = true;
  c->have_ws = false;
  return RAPDB_OK;
}

int rapdb_spectral_norm(const double* M, long long rows, long long cols, long long ld, int iters, double tol,
                        void* stream, double* out) {
  if (!M || !out || rows < 0 || cols < 0 || ld < cols || iters < 0) return RAPDB_EINPUT;
  *out = 0.0;
  if (rows == 0 || cols == 0) return RAPDB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double *v = nullptr, *w1 = nullptr, *w = nullptr, *nr = nullptr, *h = nullptr;
  const size_t bytes = (size_t)(2 * cols + rows + 2) * sizeof(double);
  if (cudaMallocAsync(reinterpret_cast<void**>(&v), bytes, s) != cudaSuccess) return RAPDB_EDEVICE;
  w = v + cols;
  w1 = w + cols;
  nr = w1 + rows;
  int rc = RAPDB_OK;
  if (cudaMallocHost(reinterpret_cast<void**>(&h), sizeof(double)) != cudaSuccess) rc = RAPDB_EDEVICE;
  const int blocks = (int)std::min<long long>(1184, (cols + 255) / 256);
  const int rblocks = (int)std::min<long long>(1184, (rows * 32 + 255) / 256);
  if (!rc) {
    rapdb_spec::init_v<<<blocks, 256, 0, s>>>(v, cols);
    rapdb_spec::norm_normalize<<<1, 1024, 0, s>>>(v, v, cols, nr, 1);    // v /= |v|
    g_launches += 2;
    double prev = 0.0;
    for (int it = 0; it < iters; ++it) {
      rapdb_spec::mv_rows<<<rblocks, 256, 0, s>>>(M, rows, cols, ld, v, w1);
      rapdb_spec::mv_cols<<<blocks, 256, 0, s>>>(M, rows, cols, ld, w1, w);
      rapdb_spec::norm_normalize<<<1, 1024, 0, s>>>(w, v, cols, nr, 1);
      g_launches += 3;
      if (cudaMemcpyAsync(h, nr, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess) { rc = RAPDB_EDEVICE; break; }
      const double nrm = *h;
      if (nrm == 0.0) { prev = 0.0; break; }
      const double est = std::sqrt(nrm);
      const bool done = std::fabs(est - prev) <= tol * std::max(est, 1.0);
      prev = est;
      if (done) break;
    }
    *out = 1.01 * prev;
  }
  if (h) cudaFreeHost(h);
  cudaFreeAsync(v, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) rc = RAPDB_EDEVICE;
  return rc;
}

int rapdb_set_factored_transpose(rapdb_ctx* c, int nph, const long long* ph_bounds, const rapdb_sell* RT,
                                 const rapdb_sell* AT, int tagged) {
  if (!c) return RAPDB_EINPUT;
  if (!c->bound || c->P.kind != 1) return fail(c, RAPDB_ECONFIG, "bind a factored instance first");
  DevProblem& P = c->P;
  if (nph < 1 || nph > kMaxRtPhases || !ph_bounds || !RT || !AT)
    return fail(c, RAPDB_EINPUT, "need 1..8 row phases of R^T and A^T");
  if (ph_bounds[0] != 0 || ph_bounds[nph] != P.nr) return fail(c, RAPDB_EINPUT, "phase bounds must run from 0 to nr");
  for (int i = 0; i < nph; ++i)
    if (ph_bounds[i + 1] < ph_bounds[i]) return fail(c, RAPDB_EINPUT, "phase bounds must be nondecreasing");
  if (tagged && (P.nr > kRtRowMask + 1LL || P.fnb > (1 << (31 - kRtTagShift))))
    return fail(c, RAPDB_EINPUT, "tagged R^T rows need nr <= 2^23 and at most 256 local blocks");
  const long long cols = ((long long)P.n + 31) / 32 * 32;
  long long ent = 0;
  c->grad_bytes = 8LL * P.fnb * P.n + 24LL * P.n;   // C once, the three column partials
  for (int ph = 0; ph < nph; ++ph) {
    const int e = take_sell(c, RT + ph, cols, true, "R^T phase", &c->h_sell[kSellRt + ph], &ent);
    if (e) return e;
    c->grad_bytes += 12 * ent + 8 * cols;
  }
  const int e = take_sell(c, AT, cols, true, "A^T", &c->h_sell[kSellAt], &ent);
  if (e) return e;
  c->grad_bytes += 12 * ent + 8 * cols;
  CK(cudaMemcpyAsync(c->d_sell, c->h_sell, sizeof c->h_sell, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  P.rt_nph = nph; P.rt_tag = tagged ? 1 : 0;
  return RAPDB_OK;
}

int rapdb_set_factored_symmetric(rapdb_ctx* c, int symmetric) {
  if (!c) return RAPDB_EINPUT;
  if (!c->bound || c->P.kind != 1) return fail(c, RAPDB_ECONFIG, "bind a factored instance first");
  if (symmetric && c->P.nr != (long long)c->P.fnb * c->P.n)
    return fail(c, RAPDB_EINPUT, "a symmetric stack needs n rows per block");
  c->P.sym = symmetric ? 1 : 0;
  return RAPDB_OK;
}

int rapdb_set_params(rapdb_ctx* c, int mode, double c_alpha, double c_beta, double delta, double eta,
                     double tau_bar, double gamma0, int nonmonotone, int max_backtracks, int ball_kind,
                     double r1, double r2) {
  if (!c) return RAPDB_EINPUT;
  if (mode != 0 && mode != 1) return fail(c, RAPDB_ECONFIG, "unknown mode");
  if (!(eta > 0.0 && eta < 1.0)) return fail(c, RAPDB_ECONFIG, "eta must lie in (0, 1)");
  if (tau_bar <= 0 || gamma0 <= 0) return fail(c, RAPDB_ECONFIG, "tau_bar and gamma0 must be positive");
  if (max_backtracks < 0) return fail(c, RAPDB_ECONFIG, "max_backtracks must be >= 0");
  if (ball_kind < 0 || ball_kind > 2) return fail(c, RAPDB_ECONFIG, "unknown dual ball");
  DevParams d{};
  d.mode = mode; d.c_alpha = c_alpha; d.c_beta = c_beta; d.delta = delta; d.eta = eta;
  d.tau_bar = tau_bar; d.gamma0 = gamma0; d.c_nm = nonmonotone ? 1.0 : 0.0; d.max_bt = max_backtracks;
  d.ball = ball_kind; d.r1 = r1; d.r2 = r2;
  c->prm = d;
  c->have_params = true;
  return RAPDB_OK;
}

long long rapdb_workspace_bytes(rapdb_ctx* c) {
  if (!c || !c->bound) return -1;
  c->guard = guards_on() ? 1 : 0;
  return layout_of(c).total;
}

int rapdb_check_guards(rapdb_ctx* c, char* report, int size) {
  if (!c || !c->have_ws) return -1;
  if (!c->guard) return 0;
  const Layout L = layout_of(c);
  int bad = 0;
  std::string rep;
  std::vector<unsigned char> h;
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return -1;
  for (int i = 0; i < B_COUNT; ++i) {
    const long long g0 = L.end[i], g1 = (i + 1 < B_COUNT ? L.off[i + 1] : L.total);
    h.assign((size_t)(g1 - g0), 0);
    if (cudaMemcpy(h.data(), c->ws_base + g0, h.size(), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    long long nb = 0, first = -1;
    for (size_t k = 0; k < h.size(); ++k)
      if (h[k] != kGuardByte) { ++nb; if (first < 0) first = (long long)k; }
    if (nb) {
      ++bad;
      char t[96];
      std::snprintf(t, sizeof t, "buffer %d: %lld guard bytes overwritten (first at +%lld); ", i, nb, first);
      rep += t;
    }
  }
  if (report && size > 0) std::snprintf(report, (size_t)size, "%s", rep.c_str());
  return bad;
}

int rapdb_bind_workspace(rapdb_ctx* c, void* dptr, long long bytes) {
  if (!c || !c->bound) return RAPDB_EINPUT;
  const Layout L = layout_of(c);
  if (!dptr || bytes < L.total) return fail(c, RAPDB_EINPUT, "workspace too small");
  if ((reinterpret_cast<uintptr_t>(dptr) & 255) != 0) return fail(c, RAPDB_EINPUT, "workspace must be 256-byte aligned");
  char* base = static_cast<char*>(dptr);
  auto D = [&](int i) { return reinterpret_cast<double*>(base + L.off[i]); };
  Work w{};
  w.x = D(B_X); w.U = D(B_U); w.gval = D(B_GVAL); w.eqv = D(B_EQV); w.y = D(B_Y); w.ytr = D(B_YTR);
  w.gy = D(B_GY); w.gxb = D(B_GXB); w.gxs = D(B_GXS); w.xcum = D(B_XCUM); w.ycum = D(B_YCUM);
  w.part = D(B_PART); w.segxu = D(B_SEGXU); w.segqx = D(B_SEGQX); w.zq = D(B_ZQ); w.aux = D(B_AUX);
  w.aux2 = D(B_AUX2);
  w.H = D(B_H);
  w.hx = D(B_HX);
  w.hxn = D(B_HXN);
  w.hy = D(B_HY);
  w.W = D(B_W);
  w.pw2 = D(B_PW2);
  w.pcx = D(B_PCX);
  w.Pt = D(B_PT);
  w.wl = D(B_WL);
  w.fpart = D(B_FPART);
  w.fctr = reinterpret_cast<unsigned*>(base + L.off[B_FCTR]);
  w.ccnt = reinterpret_cast<unsigned*>(base + L.off[B_EARLY]);
  w.idone = reinterpret_cast<int*>(base + L.off[B_EARLY] + 256);
  w.trace = nullptr;
  w.st = reinterpret_cast<SolverState*>(base + L.off[B_ST]);
  w.bar = reinterpret_cast<unsigned long long*>(base + L.off[B_BAR]);
  w.abort_flag = reinterpret_cast<int*>(base + L.off[B_ABORT]);
  c->w = w;
  c->ws_base = base;
  CK(cudaMemsetAsync(dptr, 0, (size_t)L.total, c->stream));
  if (c->guard)
    for (int i = 0; i < B_COUNT; ++i) {
      const long long g0 = L.end[i], g1 = (i + 1 < B_COUNT ? L.off[i + 1] : L.total);
      CK(cudaMemsetAsync(base + g0, kGuardByte, (size_t)(g1 - g0), c->stream));
    }
  SolverState st{};
  st.ig_prev = 0; st.ig_cur = 1; st.ig_new = 2;
  CK(cudaMemcpyAsync(w.st, &st, sizeof(st), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->have_ws = true;
  return RAPDB_OK;
}

int rapdb_reinit(rapdb_ctx* c, int source, const double* x, const double* v, const double* lam, int warm_tau,
                 int reset_inner) {
  if (!c) return RAPDB_EINPUT;
  if (source < 0 || source > 2) return fail(c, RAPDB_EINPUT, "bad reinit source");
  if (source == 0 && (!x || (c->P.p > 0 && !v) || (c->P.m > 0 && !lam)))
    return fail(c, RAPDB_EINPUT, "explicit reinit needs x, v, lam");
  RunCfg rc{};
  rc.op = OP_REINIT;
  rc.src = source;
  rc.warm_tau = warm_tau;
  rc.reset_inner = reset_inner;
  rc.in_x = x; rc.in_v = v; rc.in_lam = lam;
  int r = launch(c, rc);
  if (r) return r;
  SolverState st;
  return read_state(c, &st);
}

int rapdb_egm(rapdb_ctx* c, double stepsize, long long K, int trace_every, double* trace, long long* iterations,
              int* diverged) {
  if (!c || !iterations || !diverged) return RAPDB_EINPUT;
  if (!(stepsize >= 0.0)) return fail(c, RAPDB_ECONFIG, "stepsize must be nonnegative");
  if (K < 1) return fail(c, RAPDB_ECONFIG, "need K >= 1");
  if (trace_every < 0 || (trace_every > 0 && !trace)) return fail(c, RAPDB_EINPUT, "trace_every needs a trace buffer");
  RunCfg rc{};
  rc.op = OP_EGM;
  rc.egm_s = stepsize;
  rc.egm_K = K;
  rc.egm_trace_every = trace_every;
  Work saved = c->w;
  c->w.trace = trace_every > 0 ? trace : nullptr;
  int r = launch(c, rc);
  c->w = saved;
  if (r) return r;
  SolverState st;
  r = read_state(c, &st);
  if (r) return r;
  if (st.status == ST_ABORT) return fail(c, RAPDB_EDEVICE, "EGM op aborted");
  *iterations = st.call_done;
  *diverged = st.fail_iter ? 1 : 0;
  return RAPDB_OK;
}

int rapdb_run(rapdb_ctx* c, const rapdb_run_args* a, double* trace, rapdb_run_result* out) {
  if (!c || !a || !out) return RAPDB_EINPUT;
  if (a->max_iters < 1) return fail(c, RAPDB_ECONFIG, "need max_iters >= 1");
  RunCfg rc{};
  rc.op = OP_RUN;
  rc.max_iters = a->max_iters; rc.budget = a->budget; rc.stop_total = a->stop_total;
  rc.metrics_every = a->metrics_every; rc.criterion = a->criterion;
  rc.eps = a->eps; rc.eps_kkt = a->eps_kkt; rc.eps_feas = a->eps_feas;
  rc.f_star = a->f_star; rc.has_f_star = a->has_f_star;
  rc.fixed_period = a->fixed_period; rc.fixed_point = a->fixed_point; rc.warm_tau = a->warm_tau;
  rc.stop_at_fixed = a->stop_at_fixed;
  Work saved = c->w;
  c->w.trace = trace;
  SolverState before;
  int r = read_state(c, &before);
  EventGuard eg;
  cudaEvent_t& e0 = eg.ev[0];
  cudaEvent_t& e1 = eg.ev[1];
  if (!r) {
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, c->stream));
    r = launch(c, rc);
    if (!r) CK(cudaEventRecord(e1, c->stream));
  }
  c->w = saved;
  if (r) return r;
  SolverState st;
  r = read_state(c, &st);
  if (r) return r;
  float kms = 0.0f;
  cudaEventElapsedTime(&kms, e0, e1);
  std::memset(out, 0, sizeof(*out));
  out->status = st.status;
  out->iters_done = st.iters - before.iters;
  out->total = st.iters;
  out->inner = st.inner;
  out->evals_total = st.evals_total;
  out->tau_cand = st.tau_cand; out->tau_prev = st.tau_prev; out->gamma = st.gamma;
  out->sigma_prev = st.sigma_prev; out->T = st.T;
  out->fail_tau = st.fail_tau; out->fail_gamma = st.fail_gamma; out->fail_iter = st.fail_iter;
  for (int i = 0; i < 8; ++i) out->metrics[i] = st.metrics[i];
  out->has_metrics = st.has_metrics;
  out->sweep_ns = st.sweep_ns - before.sweep_ns;
  out->sweeps = st.sweeps - before.sweeps;
  out->kernel_ms = (double)kms;
  out->sweep_bytes = c->sweep_bytes;
  if (st.status == ST_ABORT) return fail(c, RAPDB_EDEVICE, "device watchdog fired");
  if (st.status == ST_NONCONV) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "backtracking failed after %d shrinkages (tau=%.3e); check data validity / Lipschitz regime",
                  c->prm.max_bt, st.fail_tau);
    c->err = buf;
    return RAPDB_ENONCONV;
  }
  return RAPDB_OK;
}

int rapdb_kkt(rapdb_ctx* c, int has_f_star, double f_star, double* out) {
  if (!c || !out) return RAPDB_EINPUT;
  RunCfg rc{};
  rc.op = OP_KKT;
  rc.has_f_star = has_f_star;
  rc.f_star = f_star;
  int r = launch(c, rc);
  if (r) return r;
  SolverState st;
  r = read_state(c, &st);
  if (r) return r;
  for (int i = 0; i < 8; ++i) out[i] = st.metrics[i];
  return RAPDB_OK;
}

int rapdb_get_iterate(rapdb_ctx* c, int which, double* x, double* v, double* lam) {
  if (!c || !x || (c->P.p > 0 && !v) || (c->P.m > 0 && !lam)) return RAPDB_EINPUT;
  RunCfg rc{};
  rc.op = OP_GET;
  rc.src = which == 1 ? 2 : 1;
  rc.out_x = x; rc.out_v = v; rc.out_lam = lam;
  int r = launch(c, rc);
  if (r) return r;
  SolverState st;
  return read_state(c, &st);
}

int rapdb_probe_sweep(rapdb_ctx* c, const double* x, double* u, double* g, int reps, float* ms) {
  if (!c || !x || !u || !g) return RAPDB_EINPUT;
  RunCfg rc{};
  rc.op = OP_PROBE;
  rc.in_x = x; rc.out_u = u; rc.out_g = g;
  rc.reps = reps < 1 ? 1 : reps;
  EventGuard eg;
  cudaEvent_t& e0 = eg.ev[0];
  cudaEvent_t& e1 = eg.ev[1];
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, c->stream));
  int r = launch(c, rc);
  CK(cudaEventRecord(e1, c->stream));
  if (r) return r;
  SolverState st;
  r = read_state(c, &st);
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  if (ms) *ms = t / (float)rc.reps;
  return r;
}

int rapdb_grad_x(rapdb_ctx* c, const double* x, const double* v, const double* lam, double* gx, double* g) {
  if (!c || !x || !gx || !g || (c->P.p > 0 && !v) || (c->P.m > 0 && !lam)) return RAPDB_EINPUT;
  if (c->split) return fail(c, RAPDB_ECONFIG, "rapdb_grad_x needs an unsharded context");
  RunCfg rc{};
  rc.op = OP_GRAD;
  rc.in_x = x; rc.in_v = v; rc.in_lam = lam;
  rc.out_x = gx; rc.out_g = g; rc.out_u = nullptr;
  rc.reps = 1;
  int r = launch(c, rc);
  if (r) return r;
  SolverState st;
  return read_state(c, &st);
}

int rapdb_eq_residual(rapdb_ctx* c, const double* x, double* eq) {
  if (!c || !x || (c->P.p > 0 && !eq)) return RAPDB_EINPUT;
  if (c->P.p == 0) return RAPDB_OK;
  RunCfg rc{};
  rc.op = OP_PROBE;
  rc.in_x = x;
  rc.out_v = eq;
  rc.out_g = nullptr;
  rc.out_u = nullptr;
  rc.reps = 1;
  int r = launch(c, rc);
  if (r) return r;
  SolverState st;
  return read_state(c, &st);
}

int rapdb_kkt_at(rapdb_ctx* c, const double* x, const double* v, const double* lam, int has_f_star, double f_star,
                 double* out) {
  if (!c || !x || !out || (c->P.p > 0 && !v) || (c->P.m > 0 && !lam)) return RAPDB_EINPUT;
  if (c->split) return fail(c, RAPDB_ECONFIG, "rapdb_kkt_at needs an unsharded context");
  RunCfg rc{};
  rc.op = OP_KKTAT;
  rc.in_x = x; rc.in_v = v; rc.in_lam = lam;
  rc.out_g = nullptr;      // g at x stays in the workspace (gval)
  rc.out_u = nullptr;
  rc.has_f_star = has_f_star ? 1 : 0;
  rc.f_star = f_star;
  rc.reps = 1;
  int r = launch(c, rc);
  if (r) return r;
  SolverState st;
  r = read_state(c, &st);
  if (r) return r;
  for (int i = 0; i < 8; ++i) out[i] = st.metrics[i];
  out[8] = st.phi_at;
  return RAPDB_OK;
}

int rapdb_smoothed_gap(rapdb_ctx* c, int source, const double* x, const double* v, const double* lam,
                       double xi, double tol, const double* x_warm, double* x_cand, double* out) {
  if (!c || !out) return RAPDB_EINPUT;
  if (!(xi > 0.0)) return fail(c, RAPDB_ECONFIG, "xi must be positive");
  if (!(tol > 0.0)) return fail(c, RAPDB_ECONFIG, "need tol > 0");
  if (source < 0 || source > 2) return fail(c, RAPDB_EINPUT, "bad smoothed_gap source");
  if (source == 0 && (!x || (c->P.p > 0 && !v) || (c->P.m > 0 && !lam)))
    return fail(c, RAPDB_EINPUT, "explicit smoothed_gap point needs x, v, lam");
  if (!c->gap_ok)
    return fail(c, RAPDB_ECONFIG, "smoothed gap needs the dense H (n too large for this instance layout)");
  RunCfg rc{};
  rc.op = OP_GAP;
  rc.src = source;
  rc.in_x = x; rc.in_v = v; rc.in_lam = lam;
  rc.xi = xi;
  rc.tol = tol;
  rc.warm = x_warm;
  rc.out_x = x_cand;
  int r = launch(c, rc);
  if (r) return r;
  SolverState st;
  r = read_state(c, &st);
  if (r) return r;
  for (int i = 0; i < 6; ++i) out[i] = st.gap[i];
  return RAPDB_OK;
}

}  // extern "C"
