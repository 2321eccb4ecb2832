// solver_kernel.cuh -- the persistent, cooperative rAPDB kernel (sm_100a, fp64).
//
// One CTA per SM (256 threads: 7 consumer warps + 1 TMA-bulk producer warp --
// two warps per SM sub-partition, so the register cap is 255 and the sweeps do
// not spill; ~210 KB of shared memory for the Q-tile ring).  A launch executes
// one "op":
//   OP_RUN    accepted iterations with device-side backtracking, KKT cadence,
//             termination and fixed restarts  (engine.py:198-259 inside
//             restarts.py:111-161);
//   OP_REINIT ApdbEngine.reinit from an explicit / last / average point
//             (engine.py:102-136);
//   OP_KKT    kkt_residual at the current iterate (diagnostics.py:96-113);
//   OP_GET    engine.last / engine.average() (engine.py:262-272);
//   OP_PROBE  one (or reps) fused Q sweeps at a given x, for KATs and timing;
//   OP_GAP    the smoothed duality gap (gap.cuh); OP_GRAD grad_x Phi at a point;
//   OP_EGM    extragradient iterations (egm.cuh).
//
// Phases inside an op are separated by a software grid barrier (the launch is
// cooperative, so all CTAs are co-resident).  Every cross-CTA sum is a
// two-level fixed-order reduction (warp butterfly -> per-CTA partial -> every
// CTA sums the G partials in CTA order), so results are bitwise reproducible
// and every CTA derives the same accept/reject decision without a broadcast.
#pragma once
#include "rapdb_dev.cuh"

namespace rapdb {

struct Sm {
  double* xs;              // staged x (ld doubles, zero padded)
  unsigned char* ring;     // nstages * stage_bytes bulk-copy ring
  uint64_t* full;          // [nstages] TMA-complete barriers
  uint64_t* empty;         // [nstages] consumer-release barriers
  double* stage;           // the ring reused as a dual-vector staging area outside sweeps
  double* red;             // [kWarps*8] block-reduction scratch
  double* tot;             // [NSLOT] grid totals
  SolverState* st;
  int* flag;
  volatile unsigned* prog; // [8] units consumed per consumer warp in the current sweep
  volatile unsigned* tag;  // [32] sequence number of the tile last issued into each slot
  volatile unsigned* rel;  // [32] sequence number of the tile last released from each slot
  double (*rc)[32];        // [kWarps][32] chunk partials of recombine_cols (the ring's last
                           // 2 KB: used outside sweeps only, after the staged duals)
  unsigned long long gen;  // grid-barrier generation (thread 0)
  unsigned pseq;           // pipeline sequence (producer lane / consumers)
};

// ------------------------------------------------------------ grid barrier

// Arrival is one acq_rel atomic (release: the CTA's writes, ordered before it
// by the CTA barrier; acquire: invalidates L1), the wait an acquire-load spin
// -- 1.14 us per barrier on 148 CTAs against 1.50 us for fence + atomic +
// volatile spin + fence (tools/bar_probe.cu).
__device__ __noinline__ bool gsync(const KArgs& K, Sm& S) {
  __syncthreads();
  if (threadIdx.x == 0) {
    S.gen += gridDim.x;
    unsigned long long r;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(r) : "l"(K.w.bar) : "memory");
    r += 1;
    volatile int* va = K.w.abort_flag;
    const long long t0 = clock64();   // monotonic per SM (see mbar_wait)
    int ab = 0;
    while (r < S.gen) {
      if (*va) { ab = 1; break; }
      if (clock64() - t0 > 60000000000ll) {   // ~30 s watchdog
        atomicExch(K.w.abort_flag, 1);   // 1: grid-barrier timeout
        ab = 1;
        break;
      }
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(K.w.bar) : "memory");
    }
    S.flag[0] = ab;
  }
  __syncthreads();
  return S.flag[0] == 0;
}

// ------------------------------------------------------ fixed-order sums

template <int NK>
__device__ __forceinline__ void put_partials(const KArgs& K, Sm& S, const double (&v)[NK],
                                             const int (&slots)[NK]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const double t = warp_sum(v[k]);
    if (lane == 0) S.red[w * 8 + k] = t;
  }
  __syncthreads();
  if (threadIdx.x < NK) {
    double s = S.red[threadIdx.x];
    for (int i = 1; i < kWarps; ++i) s += S.red[i * 8 + threadIdx.x];
    K.w.part[(long long)slots[threadIdx.x] * gridDim.x + blockIdx.x] = s;
  }
  __syncthreads();
}

template <int NK>
__device__ __forceinline__ void get_totals(const KArgs& K, Sm& S, const int (&slots)[NK]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = gridDim.x;
  for (int k = w; k < NK; k += kWarps) {
    const double* p = K.w.part + (long long)slots[k] * G;
    // all of a lane's partials in flight at once (G <= 8 * 32), summed in
    // index order: one L2 round trip instead of G / 32 dependent ones
    double v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = (lane + 32 * t < G) ? ldcg(p + lane + 32 * t) : 0.0;
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += v[t];
    s = warp_sum(s);
    if (lane == 0) S.tot[slots[k]] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ long long gtid() { return (long long)blockIdx.x * kThreads + threadIdx.x; }
__device__ __forceinline__ long long gstride() { return (long long)gridDim.x * kThreads; }

__device__ __forceinline__ double clipd(double w, double lo, double hi) { return fmin(fmax(w, lo), hi); }

// ---------------------------------------------------------------- sweep

__device__ __forceinline__ double rowdot(const double* row, const double* xs, long long npairs,
                                         int start, int step) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
  const double2* x2 = reinterpret_cast<const double2*>(xs);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  long long k = start;
  for (; k + step < npairs; k += 2 * step) {
    const double2 q0 = r2[k], x0 = x2[k], q1 = r2[k + step], x1 = x2[k + step];
    a0 = fma(q0.x, x0.x, a0);
    a1 = fma(q0.y, x0.y, a1);
    a2 = fma(q1.x, x1.x, a2);
    a3 = fma(q1.y, x1.y, a3);
  }
  if (k < npairs) {
    const double2 q0 = r2[k], x0 = x2[k];
    a0 = fma(q0.x, x0.x, a0);
    a1 = fma(q0.y, x0.y, a1);
  }
  return warp_sum((a0 + a1) + (a2 + a3));
}

// One fused pass over the streamed (non-zero) local matrices at x:
//   U[par][lm][j] = (Q_lm x)_j, per-(CTA, warp, matrix-segment) sums of x_j u_j
//   and q_j x_j, eqv[par] = A x - b, zq = q.x for all-zero matrices.
// The CTA's contiguous row range is cut into ~8 KB tiles: TR whole rows when a
// row fits (small n), else one column chunk of one row (cpr chunks per row).
// Tile t is streamed by a 1-D TMA bulk copy into ring slot (pseq+t) % nstages
// and consumed by ONE consumer warp -- the warp that owns its row unit -- which
// dots it with the staged x and releases the slot.  There is no CTA-wide
// barrier per tile, so the ring keeps nstages*stage_bytes of HBM reads in
// flight per SM; chunk partials of a row are summed in chunk order.
// equality rows (A x - b) and q.x of skipped all-zero matrices: one warp each
// Items are dealt round-robin starting at it0 with stride istride (a warp id
// in the grid); the default is every warp of every CTA.
__device__ __forceinline__ void sweep_tail(const KArgs& K, Sm& S, int par, const double* xg = nullptr,
                                           long long it0 = -1, long long istride = 0) {
  const DevProblem& P = K.P;
  const int n = P.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long items = (long long)P.p + P.nzero;
  if (it0 < 0) {
    it0 = (long long)blockIdx.x * kWarps + warp;
    istride = (long long)gridDim.x * kWarps;
  }
  for (long long it = it0; it < items; it += istride) {
    const double* vec = it < P.p ? P.A + it * n : P.q + (long long)(P.k0 + __ldg(P.zero_list + (it - P.p))) * n;
    // 4 independent chains per lane (8 loads in flight), combined in fixed order
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = lane;
    // x from shared memory, or from global memory when it is too long (xg)
    auto xv = [&](int jj) { return xg ? ldcg(xg + jj) : S.xs[jj]; };
    // four 128-strides' loads in flight at once, the same chains and order
    for (; j + 480 < n; j += 512) {
      double a[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) a[t] = __ldg(vec + j + 32 * t);
#pragma unroll
      for (int t = 0; t < 16; t += 4) {
        s0 = fma(a[t], xv(j + 32 * t), s0);
        s1 = fma(a[t + 1], xv(j + 32 * t + 32), s1);
        s2 = fma(a[t + 2], xv(j + 32 * t + 64), s2);
        s3 = fma(a[t + 3], xv(j + 32 * t + 96), s3);
      }
    }
    for (; j + 96 < n; j += 128) {
      const double a0 = __ldg(vec + j), a1 = __ldg(vec + j + 32), a2 = __ldg(vec + j + 64), a3 = __ldg(vec + j + 96);
      s0 = fma(a0, xv(j), s0);
      s1 = fma(a1, xv(j + 32), s1);
      s2 = fma(a2, xv(j + 64), s2);
      s3 = fma(a3, xv(j + 96), s3);
    }
    for (; j < n; j += 32) s0 = fma(__ldg(vec + j), xv(j), s0);
    double s = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) {
      if (it < P.p) K.w.eqv[(long long)par * P.p + it] = s - __ldg(P.b + it);
      else K.w.zq[it - P.p] = s;
    }
  }
}

// sub-phase timing of the packed sweep on CTA 0 (step-profile slots 60..62:
// x staging, stream, reduce+tail)
__device__ __forceinline__ void sub_time(Sm& S, int slot, unsigned long long& t) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long now = globaltimer();
    if (now > t) S.st->step_ns[slot] += (double)(now - t);
    S.st->step_cnt[slot] += 1;
    t = now;
  }
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

#ifndef RAPDB_EARLY_POLL_NS
#define RAPDB_EARLY_POLL_NS 1000
#endif
constexpr unsigned kEarlyPollNs = RAPDB_EARLY_POLL_NS;

// streamed matrix a's chunk for the early reduction (monotone in a)
__device__ __forceinline__ int chunk_of(long long a, int nch, int nact) { return (int)(a * nch / nact); }

// One phase-B item (streamed matrix a, 64-row block B), by one warp:
// u = sum_K Pt[a][B][K] in K order into the U-cache row segment, the block's
// x.u and q.x sums, and the item's partial lines dropped from L2.  The same
// bits whichever warp runs it (during the stream or after it).
__device__ __forceinline__ void reduce_item(const KArgs& K, const double* xs, const double* xsrc, double* U,
                                            long long it) {
  const DevProblem& P = K.P;
  const int n = P.n;
  const int lane = threadIdx.x & 31;
  const int nbB = K.sp.geom.nbB;
  const bool xglobal = K.sp.xglobal;
  const int a = (int)(it / nbB);
  const int B = (int)(it - (long long)a * nbB);
  const double2* pp = reinterpret_cast<const double2*>(K.w.Pt + ((long long)a * nbB + B) * nbB * sym::kB) + lane;
  double sx = 0.0, sy = 0.0;
  // up to 32 x 512 B in flight per warp: ceil(nbB / 32) dependent rounds
  // (predicated, so a ragged nbB does not fall into short batches)
  for (int kk = 0; kk < nbB; kk += 32) {
    double2 t[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) t[q] = kk + q < nbB ? __ldcg(pp + (kk + q) * 32) : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (kk + q < nbB) { sx += t[q].x; sy += t[q].y; }
  }
  // the item's partials are dead until the next sweep rewrites them: drop
  // the L2 lines without writing them back to DRAM
  __syncwarp();
  {
    const char* base = reinterpret_cast<const char*>(K.w.Pt + ((long long)a * nbB + B) * nbB * sym::kB);
    for (int L = lane; L < nbB * 4; L += 32)
      asm volatile("discard.global.L2 [%0], 128;" :: "l"(base + (long long)L * 128) : "memory");
  }
  const int lm = __ldg(P.act + a);
  const double* qa = P.q + (long long)(P.k0 + lm) * n;
  const int r = B * sym::kB + 2 * lane;
  double xu = 0.0, qx = 0.0;
  if (r < n) {
    const double x0 = xglobal ? ldcg(xsrc + r) : xs[r];
    U[(long long)lm * n + r] = sx;
    xu = x0 * sx;
    qx = __ldg(qa + r) * x0;
  }
  if (r + 1 < n) {
    const double x1 = xglobal ? ldcg(xsrc + r + 1) : xs[r + 1];
    U[(long long)lm * n + r + 1] = sy;
    xu = xu + x1 * sy;
    qx = qx + __ldg(qa + r + 1) * x1;
  }
  xu = warp_sum(xu);
  qx = warp_sum(qx);
  if (lane == 0) {
    K.w.segxu[it] = xu;
    K.w.segqx[it] = qx;
  }
}

// The packed-symmetric sweep (layout 1, symsweep.cuh): stream the upper block
// triangle of every streamed matrix (round-robin units over the CTAs, TMA
// bulk copies into the ring, one consumer warp per unit) into the unit
// partials Pt; grid barrier; then reduce Pt in fixed order into the U-cache
// and the per-(matrix, 64-row block) x.u and q.x sums that g_combine adds.
__device__ __noinline__ void sweep_sym(const KArgs& K, Sm& S, const double* xsrc, int par) {
  const DevProblem& P = K.P;
  const SweepPlan& sp = K.sp;
  const sym::Geom& g = sp.geom;
  const int n = P.n;
  const int xlen = g.nbB * sym::kB;
  unsigned long long tsub = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) tsub = globaltimer();
  // stage x (zero padded): all of a thread's loads in flight at once; with a
  // very long x (sp.xglobal) each consumer warp loads its unit's two x blocks
  for (int j0 = threadIdx.x; j0 < (sp.xglobal ? 0 : xlen); j0 += 8 * kThreads) {
    double v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = j0 + t * kThreads;
      v[t] = (j < n) ? ldcg(xsrc + j) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = j0 + t * kThreads;
      if (j < xlen) S.xs[j] = v[t];
    }
  }
  if (threadIdx.x == 0) S.flag[2] = 0;   // consumer warps finished with the stream
  // generic-proxy use of the ring (dual staging) before the bulk copies below
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  sub_time(S, 60, tsub);
  const int G = gridDim.x, b = blockIdx.x;
  const long long total = (long long)P.nact * g.upm;
  const long long mine = total > b ? (total - 1 - b) / G + 1 : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncw = sp.ncw;
  const unsigned base = S.pseq;
  const unsigned ns = (unsigned)sp.nstages;
  const long long mat_doubles = g.spm * sym::kTD;
  const long long pstride = (long long)g.nbB * g.nbB * sym::kB;
  const int upm = g.upm;
  // hoisted into registers: S is a by-reference local (stack) object and every
  // S.field access in the loops below would otherwise be a local-memory load
  unsigned char* const ring = S.ring;
  uint64_t* const fullb = S.full;
  uint64_t* const emptyb = S.empty;
  const double* const xs = S.xs;
  int* const abort_flag = K.w.abort_flag;
  double* const Pt = K.w.Pt;
  const sym::Unit* const units = sp.units;
  const long long stage_bytes = sp.stage_bytes;
  const int* const act = P.act;
  const double* const Qst = P.Q;
  const sym::Geom gg = g;
  const int nch = sp.nchunk;
  double* const U = K.w.U + (long long)par * P.nloc * n;
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      long long a = b / upm;
      int u = (int)(b - a * upm);
      unsigned s = base % ns, use = base / ns;
      for (long long k = 0; k < mine; ++k) {
        if (use > 0 && !mbar_wait(&emptyb[s], (use - 1) & 1, abort_flag)) break;
        const sym::Unit un = units[u];
        int rs, cs;
        const unsigned bytes = (unsigned)sym::unit_subtiles(gg, un.bi, un.bj, rs, cs) * sym::kTD * 8u;
        mbar_expect_tx(&fullb[s], bytes);
        bulk_g2s(ring + (long long)s * stage_bytes,
                 Qst + (long long)__ldg(act + a) * mat_doubles + (long long)un.off * sym::kTD, bytes,
                 &fullb[s], pol);
        u += G;
        while (u >= upm) { u -= upm; ++a; }
        if (++s == ns) { s = 0; ++use; }
      }
    }
  } else if (warp < ncw) {
    const long long gi = b + (long long)warp * G;
    long long a = gi / upm;
    int u = (int)(gi - a * upm);
    unsigned s = (base + warp) % ns, use = (base + warp) / ns;
    const int adv = ncw * G;
    const uint64_t keep = sym::evict_last_policy();
    // early reduction: tell the grid once this warp is past a matrix chunk
    // (its partial stores made visible first)
    int cch = 0;
    auto pass_chunk = [&]() {
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(K.w.ccnt + cch, 1u);
      ++cch;
    };
    for (long long k = warp; k < mine; k += ncw) {
      if (nch) {
        const int ch = min(chunk_of(a, nch, P.nact), nch - 1);
        while (cch < ch) pass_chunk();
      }
      if (!mbar_wait(&fullb[s], use & 1, abort_flag)) break;
      const sym::Unit un = units[u];
      if (sp.xglobal) {   // this unit's x blocks into the warp's 128-entry buffer
        double* xw = S.xs + warp * 128;
        const int r0 = un.bi * sym::kB, c0 = un.bj * sym::kB;
        xw[lane] = r0 + lane < n ? ldcg(xsrc + r0 + lane) : 0.0;
        xw[32 + lane] = r0 + 32 + lane < n ? ldcg(xsrc + r0 + 32 + lane) : 0.0;
        xw[64 + lane] = c0 + lane < n ? ldcg(xsrc + c0 + lane) : 0.0;
        xw[96 + lane] = c0 + 32 + lane < n ? ldcg(xsrc + c0 + 32 + lane) : 0.0;
        __syncwarp();
        sym::consume_unit_x(gg, reinterpret_cast<const double*>(ring + (long long)s * stage_bytes), xw, xw + 64,
                            un.bi, un.bj, Pt + a * pstride, keep, &emptyb[s]);
        __syncwarp();
      } else {   // the slot is handed back inside, right after the last tile read
        sym::consume_unit(gg, reinterpret_cast<const double*>(ring + (long long)s * stage_bytes), xs,
                          un.bi, un.bj, Pt + a * pstride, keep, &emptyb[s]);
      }
      u += adv;
      while (u >= upm) { u -= upm; ++a; }
      s += ncw;
      while (s >= ns) { s -= ns; ++use; }
    }
    while (cch < nch - 1) pass_chunk();   // the last chunk is reduced in phase B: no signal
    if (lane == 0) atomicAdd(S.flag + 2, 1);
  } else if (warp == ncw) {
    // a consumer warp without a ring slot: the equality rows and the q.x of
    // all-zero matrices (independent of the stream), then the phase-B items
    // of every matrix chunk all consumer warps of the grid are past, until
    // this CTA's own consumers finish (the last chunk is left to phase B)
    sweep_tail(K, S, par, sp.xglobal ? xsrc : nullptr, b, G);
    if (nch) {
      const unsigned target = (unsigned)(G * ncw);
      const long long items = (long long)P.nact * gg.nbB;
      for (long long it = b; it < items; it += G) {
        const int ch = chunk_of(it / gg.nbB, nch, P.nact);
        if (ch >= nch - 1) break;
        int ok = 0;
        if (lane == 0) {
          volatile int* cdone = S.flag + 2;
          while (true) {
            if (*cdone >= ncw) break;
            if (ld_acquire_gpu(K.w.ccnt + ch) >= target) { ok = 1; break; }
            __nanosleep(kEarlyPollNs);
          }
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) break;
        reduce_item(K, xs, xsrc, U, it);
        if (lane == 0) K.w.idone[it] = 1;
      }
    }
  }
  S.pseq = base + (unsigned)mine;
  if (!gsync(K, S)) return;   // aborted: the caller's barrier reports it
  sub_time(S, 61, tsub);
  // phase B: u = sum_K Pt[a][B][K] (K order), U-cache rows, block x.u and q.x
  // for the items not already reduced during the stream
  const long long items = (long long)P.nact * g.nbB;
  if (nch && b == 0 && threadIdx.x < nch) K.w.ccnt[threadIdx.x] = 0u;
  // warp-major item order: a handful of items still spreads over all SMs
  for (long long it = (long long)warp * G + b; it < items; it += (long long)G * kWarps) {
    if (nch && __ldcg(K.w.idone + it)) {
      __syncwarp();
      if (lane == 0) K.w.idone[it] = 0;
      continue;
    }
    reduce_item(K, xs, xsrc, U, it);
  }
  if (ncw == kConsumerWarps) sweep_tail(K, S, par, sp.xglobal ? xsrc : nullptr);
  __syncthreads();
  sub_time(S, 62, tsub);
}

__device__ __noinline__ void sweep(const KArgs& K, Sm& S, const double* xsrc, int par) {
  if (K.sp.layout == 1) {
    sweep_sym(K, S, xsrc, par);
    return;
  }
  const DevProblem& P = K.P;
  const SweepPlan& sp = K.sp;
  const int n = P.n;
  const long long ld = P.ld;
  for (long long j = threadIdx.x; j < ld; j += kThreads) S.xs[j] = (j < n) ? ldcg(xsrc + j) : 0.0;
  // the ring doubles as a generic-proxy staging area between sweeps: order
  // those accesses before the async-proxy (bulk copy) writes below
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  const int G = gridDim.x, b = blockIdx.x;
  const long long rs = ((long long)b * sp.rows_total) / G;
  const long long re = ((long long)(b + 1) * sp.rows_total) / G;
  const bool chunked = sp.cpr > 1;
  const long long nunits = chunked ? (re - rs) : (re - rs + sp.TR - 1) / sp.TR;
  const long long ntiles = chunked ? nunits * sp.cpr : nunits;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncw = sp.ncw;
  const unsigned base = S.pseq;
  double* U = K.w.U + (long long)par * P.nloc * n;

  if (warp == kConsumerWarps) {
    if (lane == 0) {
      // Single issuing thread: all tile addressing is incremental (no 64-bit
      // divisions on the issue path -- they capped the issue rate at ~1 tile
      // per 0.5 us).  Ring slot / phase advance as counters.
      const uint64_t pol = evict_first_policy();
      const int ns = sp.nstages;
      unsigned s = base % ns, use = base / ns;
      unsigned issued = 0;
      auto next_slot = [&](unsigned bytes) -> unsigned char* {
        const unsigned seq = base + issued;
        if (use > 0 && !mbar_wait(&S.empty[s], (use - 1) & 1, K.w.abort_flag)) {
          int* f = K.w.abort_flag;   // diagnostics of a stalled ring (host prints them)
          f[6] = (int)issued;
          f[7] = (int)s;
          f[8] = (int)use;
          f[9] = (int)ntiles;
          f[10] = (int)base;
          for (int w = 0; w < kConsumerWarps; ++w) f[11 + w] = (int)S.prog[w];
        } else if (use > 0 && S.rel[s] != seq - (unsigned)ns) {
          int* f = K.w.abort_flag;   // protocol check: slot released by the wrong tile
          if (atomicExch(f, 4) == 0) {
            f[1] = blockIdx.x; f[2] = threadIdx.x; f[6] = (int)seq; f[7] = (int)s; f[8] = (int)S.rel[s];
          }
        }
        ++issued;
        S.tag[s] = seq;
        unsigned char* dst = S.ring + (long long)s * sp.stage_bytes;
        mbar_expect_tx(&S.full[s], bytes);
        return dst;
      };
      auto advance = [&]() { if (++s == (unsigned)ns) { s = 0; ++use; } };
      if (rs < re) {
        int a = (int)(rs / n);
        long long jr = rs - (long long)a * n;
        const double* qa = P.Q + (long long)__ldg(P.act + a) * n * ld;
        if (chunked) {
          // stream order: groups of ncw rows, chunk-major inside a group, so
          // every consumer warp's consecutive tiles are exactly ncw apart (a
          // wider gap than nstages would alias the slot's mbarrier parity)
          for (long long g0 = 0; g0 < nunits; g0 += ncw) {
            const int width = (int)min((long long)ncw, nunits - g0);
            for (int c = 0; c < sp.cpr; ++c) {
              const long long c0 = (long long)c * sp.chunk;
              const unsigned bytes = (unsigned)(min((long long)sp.chunk, ld - c0) * 8);
              int ar = a;
              long long jj = jr;
              const double* qr = qa;
              for (int rr = 0; rr < width; ++rr) {
                unsigned char* dst = next_slot(bytes);
                bulk_g2s(dst, qr + jj * ld + c0, bytes, &S.full[s], pol);
                advance();
                if (++jj == n && rr + 1 < width) {
                  jj = 0;
                  ++ar;
                  qr = P.Q + (long long)__ldg(P.act + ar) * n * ld;
                }
              }
            }
            jr += width;
            while (jr >= n && g0 + width < nunits) {
              jr -= n;
              ++a;
              qa = P.Q + (long long)__ldg(P.act + a) * n * ld;
            }
          }
        } else {
          for (long long r0 = rs; r0 < re; r0 += sp.TR) {
            const long long r1 = min(r0 + sp.TR, re);
            unsigned char* dst = next_slot((unsigned)((r1 - r0) * ld * 8));
            long long row = r0;
            while (row < r1) {             // one bulk copy per matrix the tile touches
              const long long cnt = min(r1 - row, (long long)n - jr);
              bulk_g2s(dst, qa + jr * ld, (unsigned)(cnt * ld * 8), &S.full[s], pol);
              dst += cnt * ld * 8;
              row += cnt;
              jr += cnt;
              if (jr == n && row < re) {
                jr = 0;
                ++a;
                qa = P.Q + (long long)__ldg(P.act + a) * n * ld;
              }
            }
            advance();
          }
        }
      }
    }
  } else if (warp < ncw) {
    const int a0 = __ldg(P.cta_a0 + b);
    const long long segbase = ((long long)b * kConsumerWarps + warp) * sp.segmax;
    // q.x over this CTA's row range while the first tiles are in flight
    if (rs < re) {
      const int alo = (int)(rs / n), ahi = (int)((re - 1) / n);
      for (int a = alo; a <= ahi; ++a) {
        const long long j0 = max(rs, (long long)a * n) - (long long)a * n;
        const long long j1 = min(re, (long long)(a + 1) * n) - (long long)a * n;
        const double* qa = P.q + (long long)(P.k0 + __ldg(P.act + a)) * n;
        double s = 0.0;
        for (long long j = j0 + warp * 32 + lane; j < j1; j += (long long)ncw * 32)
          s = fma(__ldg(qa + j), S.xs[j], s);
        s = warp_sum(s);
        if (lane == 0) K.w.segqx[segbase + (a - a0)] = s;
      }
    }
    // per-warp x.u sums for every matrix segment alo..ahi of the CTA range
    // (segments this warp never touches are written as 0)
    const int alo = rs < re ? (int)(rs / n) : 0;
    const int ahi = rs < re ? (int)((re - 1) / n) : -1;
    int next_a = alo, cur_a = -1;
    double accx = 0.0;
    // The warp's current row (active matrix ra, row rj) and ring position
    // (slot rs_s, phase use) advance incrementally: no divisions per tile.
    int ra = 0;
    long long rj = 0;
    const unsigned ns = (unsigned)sp.nstages;
    unsigned slot = 0, use = 0;
    auto seek = [&](long long row, unsigned seq) {
      ra = (int)(row / n);
      rj = row - (long long)ra * n;
      slot = seq % ns;
      use = seq / ns;
    };
    auto step_rows = [&](long long d) {
      rj += d;
      while (rj >= n) { rj -= n; ++ra; }
    };
    auto step_seq = [&](unsigned d) {    // d <= nstages
      slot += d;
      if (slot >= ns) { slot -= ns; ++use; }
    };
    auto emit = [&](double u) {          // u = (Q x)_row: U-cache + segment sum
      const int j = (int)rj;
      if (ra != cur_a) {
        if (cur_a >= 0) {
          if (lane == 0) K.w.segxu[segbase + (cur_a - a0)] = accx;
          next_a = cur_a + 1;
        }
        for (; next_a < ra; ++next_a)
          if (lane == 0) K.w.segxu[segbase + (next_a - a0)] = 0.0;
        cur_a = ra;
        accx = 0.0;
      }
      accx += S.xs[j] * u;
      if (lane == 0) U[(long long)__ldg(P.act + ra) * n + j] = u;
    };
    if (chunked) {
      const long long full = nunits / ncw, rem = nunits - full * ncw;
      if (warp < nunits) seek(rs + warp, base + (unsigned)warp);
      for (long long k = warp; k < nunits; k += ncw) {
        const unsigned width = (unsigned)(k / ncw < full ? ncw : rem);   // rows in this group
        double u = 0.0;
        const unsigned gseq = base + (unsigned)((k / ncw) * sp.cpr * ncw) + (unsigned)warp;
        for (int c = 0; c < sp.cpr; ++c) {
          if (c > 0) step_seq(width);
          const unsigned expect = gseq + (unsigned)c * width;
          if (mbar_wait(&S.full[slot], use & 1, K.w.abort_flag) && S.tag[slot] != expect) {
            int* f = K.w.abort_flag;
            if (lane == 0 && atomicExch(f, 3) == 0) {
              f[1] = blockIdx.x; f[2] = threadIdx.x; f[6] = (int)expect; f[7] = (int)slot;
              f[8] = (int)S.tag[slot]; f[9] = (int)use; f[10] = (int)base;
            }
          }
          const double* tile = reinterpret_cast<const double*>(S.ring + (long long)slot * sp.stage_bytes);
          const long long c0 = (long long)c * sp.chunk;
          const long long len = min((long long)sp.chunk, ld - c0);
          u += rowdot(tile, S.xs + c0, len / 2, lane, 32);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            S.rel[slot] = expect;
            mbar_arrive(&S.empty[slot]);
          }
        }
        emit(u);
        step_rows(ncw);
        step_seq((unsigned)ncw);
      }
    } else {
      if (warp < nunits) seek(rs + (long long)warp * sp.TR, base + (unsigned)warp);
      for (long long k = warp; k < nunits; k += ncw) {
        const unsigned expect = base + (unsigned)k;
        if (mbar_wait(&S.full[slot], use & 1, K.w.abort_flag) && S.tag[slot] != expect) {
          int* f = K.w.abort_flag;   // protocol check: slot holds another tile
          if (lane == 0 && atomicExch(f, 3) == 0) {
            f[1] = blockIdx.x; f[2] = threadIdx.x; f[6] = (int)expect; f[7] = (int)slot;
            f[8] = (int)S.tag[slot]; f[9] = (int)use; f[10] = (int)base;
          }
        }
        const double* tile = reinterpret_cast<const double*>(S.ring + (long long)slot * sp.stage_bytes);
        const long long r0 = rs + k * sp.TR;
        const int cnt = (int)(min(r0 + sp.TR, re) - r0);
        for (int rr = 0; rr < cnt; ++rr) {
          emit(rowdot(tile + rr * ld, S.xs, ld / 2, lane, 32));
          step_rows(1);
        }
        // generic-proxy reads of the slot must be ordered before the producer's
        // next async-proxy (bulk copy) write into it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          S.rel[slot] = expect;
          mbar_arrive(&S.empty[slot]);
          S.prog[warp] = (unsigned)(k + 1);
        }
        step_rows((long long)ncw * sp.TR - cnt);
        step_seq((unsigned)ncw);
      }
    }
    if (cur_a >= 0) {
      if (lane == 0) K.w.segxu[segbase + (cur_a - a0)] = accx;
      next_a = cur_a + 1;
    }
    for (; next_a <= ahi; ++next_a)
      if (lane == 0) K.w.segxu[segbase + (next_a - a0)] = 0.0;
  }
  S.pseq = base + (unsigned)ntiles;
  __syncthreads();
  sweep_tail(K, S, par);
}

// g_i (i = 0..m, i = 0 is f) from the sweep's segment sums: 0.5*x.u + q.x + r
// (problem.py:166-177 operation order).
__device__ __forceinline__ double g_combine(const KArgs& K, int i) {
  const DevProblem& P = K.P;
  const int lm = i - P.k0;
  const int slot = __ldg(P.mat_slot + lm);
  double sxu, sqx;
  if (slot < 0) {
    sxu = 0.0;
    sqx = ldcg(K.w.zq + (-slot - 1));
  } else if (K.sp.layout == 1) {
    const int nbB = K.sp.geom.nbB;
    sxu = 0.0;
    sqx = 0.0;
    for (int B = 0; B < nbB; ++B) {
      sxu += ldcg(K.w.segxu + (long long)slot * nbB + B);
      sqx += ldcg(K.w.segqx + (long long)slot * nbB + B);
    }
  } else {
    const int lo = __ldg(P.seg_lo + slot), hi = __ldg(P.seg_hi + slot);
    sxu = 0.0;
    sqx = 0.0;
    for (int b = lo; b <= hi; ++b) {
      const int a0 = __ldg(P.cta_a0 + b);
      if (a0 < 0) continue;  // CTA with an empty row range (fewer rows than CTAs)
      for (int w = 0; w < K.sp.ncw; ++w) {
        const long long at = ((long long)b * kConsumerWarps + w) * K.sp.segmax + (slot - a0);
        sxu += ldcg(K.w.segxu + at);
        sqx += ldcg(K.w.segqx + at);
      }
    }
  }
  return 0.5 * sxu + sqx + __ldg(P.r + i);
}

// The same value computed by a whole warp (every lane gets it): the (CTA, warp)
// segment partials are spread over the lanes and butterfly-reduced -- a fixed
// order, so the bits do not depend on timing.
__device__ __forceinline__ double g_combine_warp(const KArgs& K, int i) {
  const DevProblem& P = K.P;
  const int lane = threadIdx.x & 31;
  const int slot = __ldg(P.mat_slot + (i - P.k0));
  double sxu = 0.0, sqx = 0.0;
  if (slot < 0) {
    sqx = ldcg(K.w.zq + (-slot - 1));
  } else if (K.sp.layout == 1) {
    const int nbB = K.sp.geom.nbB;
    double ax = 0.0, aq = 0.0;
    for (int B = lane; B < nbB; B += 32) {
      ax += ldcg(K.w.segxu + (long long)slot * nbB + B);
      aq += ldcg(K.w.segqx + (long long)slot * nbB + B);
    }
    sxu = warp_sum(ax);
    sqx = warp_sum(aq);
  } else {
    const int lo = __ldg(P.seg_lo + slot), hi = __ldg(P.seg_hi + slot);
    const int ncw = K.sp.ncw;
    const int cnt = (hi - lo + 1) * ncw;
    double ax = 0.0, aq = 0.0;
    for (int e = lane; e < cnt; e += 32) {
      const int b = lo + e / ncw, w = e - (e / ncw) * ncw;
      const int a0 = __ldg(P.cta_a0 + b);
      if (a0 < 0) continue;
      const long long at = ((long long)b * kConsumerWarps + w) * K.sp.segmax + (slot - a0);
      ax += ldcg(K.w.segxu + at);
      aq += ldcg(K.w.segqx + at);
    }
    sxu = warp_sum(ax);
    sqx = warp_sum(aq);
  }
  return 0.5 * sxu + sqx + __ldg(P.r + i);
}

// grad_x Phi(x, (v, lam)) at coordinate j from the U-cache (problem.py:207-217):
// (u_0 + q_0) then, in i order, + lam_i (u_i + q_i) for lam_i != 0, then + A^T v.
// This rank's share of sum_i w_i (u_i + q_i) over its local matrices
// [k0, k1) (w_0 = 1, w_i = lam_i); the rank holding Q_0 starts from u_0 + q_0.
// With one rank this is the whole sum in the reference's i order.
__device__ __forceinline__ double recombine_local(const KArgs& K, const double* Upar, const double* lam_s,
                                                  long long j) {
  const DevProblem& P = K.P;
  const long long n = P.n;
  double acc = 0.0;
  int i = P.k0;
  if (i == 0) {
    acc = ldcg(Upar + j) + __ldg(P.q + j);
    i = 1;
  }
  for (; i + 3 < P.k1; i += 4) {
    double u[4], qq[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u[k] = ldcg(Upar + (long long)(i + k - P.k0) * n + j);
      qq[k] = __ldg(P.q + (long long)(i + k) * n + j);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double l = lam_s[i + k - 1];
      const double t = l * (u[k] + qq[k]);
      acc = (l != 0.0) ? acc + t : acc;
    }
  }
  for (; i < P.k1; ++i) {
    const double l = lam_s[i - 1];
    if (l != 0.0) acc = acc + l * (ldcg(Upar + (long long)(i - P.k0) * n + j) + __ldg(P.q + (long long)i * n + j));
  }
  return acc;
}

// recombine_local for every column, for many matrices: each CTA takes 32-column
// blocks, its 8 warps take contiguous chunks of the local matrices, and warp 0
// adds the chunk partials in warp order (fixed order -> deterministic).  The
// per-thread variant above leaves all but n threads idle and is latency-bound
// for m in the hundreds (C1: 24 us -> ~4 us per trial).
__device__ void recombine_cols(const KArgs& K, Sm& S, const double* Upar, const double* lam_s, double* out) {
  const DevProblem& P = K.P;
  const long long n = P.n;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nl = P.k1 - P.k0;
  const int l0 = (w * nl) / kWarps, l1 = ((w + 1) * nl) / kWarps;
  const long long nblk = (n + 31) / 32;
  for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const long long j = blk * 32 + lane;
    double acc = 0.0;
    if (j < n) {
      int lm = l0;
      if (lm == 0 && P.k0 == 0 && l1 > 0) {
        acc = ldcg(Upar + j) + __ldg(P.q + j);
        lm = 1;
      }
      for (; lm + 7 < l1; lm += 8) {     // 16 loads in flight per lane
        double u[8], qq[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          u[k] = ldcg(Upar + (long long)(lm + k) * n + j);
          qq[k] = __ldg(P.q + (long long)(P.k0 + lm + k) * n + j);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double l = lam_s[P.k0 + lm + k - 1];
          const double t = l * (u[k] + qq[k]);
          acc = (l != 0.0) ? acc + t : acc;
        }
      }
      for (; lm + 3 < l1; lm += 4) {
        double u[4], qq[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          u[k] = ldcg(Upar + (long long)(lm + k) * n + j);
          qq[k] = __ldg(P.q + (long long)(P.k0 + lm + k) * n + j);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double l = lam_s[P.k0 + lm + k - 1];
          const double t = l * (u[k] + qq[k]);
          acc = (l != 0.0) ? acc + t : acc;
        }
      }
      for (; lm < l1; ++lm) {
        const double l = lam_s[P.k0 + lm - 1];
        if (l != 0.0) acc = acc + l * (ldcg(Upar + (long long)lm * n + j) + __ldg(P.q + (long long)(P.k0 + lm) * n + j));
      }
    }
    S.rc[w][lane] = acc;
    __syncthreads();
    if (w == 0 && j < n) {
      double t = S.rc[0][lane];
      for (int k = 1; k < kWarps; ++k) t += S.rc[k][lane];
      out[j] = t;
    }
    __syncthreads();
  }
}

// (A^T v)_j, added after the cross-rank sum (problem.py:215-216)
__device__ __forceinline__ double atv(const KArgs& K, const double* v_s, long long j) {
  double t = 0.0;
  for (int l = 0; l < K.P.p; ++l) t = t + __ldg(K.P.A + (long long)l * K.P.n + j) * v_s[l];
  return t;
}

// full grad_x Phi for a single rank (no exchange): recombination then A^T v
__device__ __forceinline__ double recombine(const KArgs& K, const double* Upar, const double* lam_s,
                                            const double* v_s, long long j) {
  double acc = recombine_local(K, Upar, lam_s, j);
  if (K.P.p > 0) acc = acc + atv(K, v_s, j);
  return acc;
}

// dual-ball radial scaling factors from the two squared norms (geometry.py:263-311)
struct BallScale { double sv, sl; int av, al; };

__device__ __forceinline__ BallScale ball_scale(const DevParams& prm, double vv, double ll) {
  BallScale r{1.0, 1.0, 0, 0};
  if (prm.ball == 1) {
    const double nrm = sqrt(vv + ll);
    if (!(nrm <= prm.r1)) { r.sv = r.sl = prm.r1 / nrm; r.av = r.al = 1; }
  } else if (prm.ball == 2) {
    const double nv = sqrt(vv), nl = sqrt(ll);
    if (nv > prm.r1) { r.sv = prm.r1 / nv; r.av = 1; }
    if (nl > prm.r2) { r.sl = prm.r2 / nl; r.al = 1; }
  }
  return r;
}

// stage (v, lam) = ball(src) into shared memory: v_s[0..p), lam_s[0..m)
__device__ __forceinline__ void stage_dual(const KArgs& K, const double* src, BallScale bs,
                                           double* v_s, double* lam_s) {
  if (K.P.kind == 1) return;   // factored: multipliers are read from global (dual_at)
  const int p = K.P.p, m = K.P.m;
  for (int j = threadIdx.x; j < p + m; j += kThreads) {
    double yv = ldcg(src + j);
    if (j < p) v_s[j] = bs.av ? bs.sv * yv : yv;
    else lam_s[j - p] = bs.al ? bs.sl * yv : yv;
  }
  __syncthreads();
}

}  // namespace rapdb
