/*
 * rapdb_b200.h -- C ABI of the B200-native rAPDB hot path.
 *
 * The reference (arxiv 2605.29291, package `rapdb`, pure Python) has no FFI;
 * its operator seam is the set of Python functions the engine calls
 * (pkg/src/rapdb/problem.py:196-223 coupling_value / grad_x_coupling /
 * grad_y_coupling, geometry.py:144-148 project_set, problem.py:182-186
 * project_dual_cone) driven by ApdbEngine.step (engine.py:198-259) and
 * run_restarted (restarts.py:82-170).  This library replaces that whole
 * per-iteration path: the host binding (paper_2605_29291_b200/_capi.py,
 * ctypes) calls these entry points from the drop-in Python API.
 *
 * Conventions
 *  - Every large buffer (Q stack, q, r, A, b, bounds, workspace, trace) is a
 *    caller-owned DEVICE allocation (a PyTorch CUDA tensor); the library never
 *    frees caller memory.  Scalars and small result structs are host memory.
 *  - Return codes: 0 ok, 1 input (InputError), 2 configuration
 *    (ConfigurationError), 3 backtracking exhausted (NonConvergence), 4
 *    CUDA/device.  rapdb_last_error() returns the message of the last failure.
 *  - One context per (process, device); not thread-safe; all work is enqueued
 *    on the stream given to rapdb_set_stream (default: legacy stream) and the
 *    calls that return results synchronise that stream.
 */
#ifndef RAPDB_B200_H
#define RAPDB_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define RAPDB_OK 0
#define RAPDB_EINPUT 1
#define RAPDB_ECONFIG 2
#define RAPDB_ENONCONV 3
#define RAPDB_EDEVICE 4

/* run status codes (rapdb_run_result.status) */
#define RAPDB_RUN_LIMIT 0        /* max_iters accepted iterations done           */
#define RAPDB_RUN_CONVERGED 1    /* check_termination fired (diagnostics.py:252)  */
#define RAPDB_RUN_BUDGET 2       /* total == budget (restarts.py:105, :166)       */
#define RAPDB_RUN_CHECK_DUE 3    /* adaptive-restart gap check due (host side)    */
#define RAPDB_RUN_FIXED_DUE 4    /* fixed restart due and caller wants the point  */
#define RAPDB_RUN_NONCONV 5      /* backtracking exhausted (engine.py:222-226)    */
#define RAPDB_RUN_ABORT 6        /* device watchdog fired                         */

#define RAPDB_TRACE_COLS 11      /* iter,tau_start,tau,sigma,gamma,evals_iter,
                                    evals_total,kkt,infeas,subopt,restart_flag  */

typedef struct rapdb_ctx rapdb_ctx;

typedef struct {
  long long max_iters;     /* accepted iterations to run in this call (>= 1)       */
  long long budget;        /* run_restarted budget: KKT forced at total == budget  */
  long long stop_total;    /* return CHECK_DUE when total reaches it (<=0: never)  */
  int metrics_every;       /* KKT cadence (restarts.py:115); <= 0: no KKT          */
  int criterion;           /* 0 none, 1 conic, 2 paper51 (diagnostics.py:252-263) */
  double eps, eps_kkt, eps_feas, f_star;
  int has_f_star;
  int fixed_period;        /* FixedRestart period, 0 = no fixed restarts           */
  int fixed_point;         /* 0 last, 1 average                                    */
  int warm_tau;            /* reinit keeps tau (engine.py:111)                     */
  int stop_at_fixed;       /* return FIXED_DUE instead of restarting on device     */
} rapdb_run_args;

typedef struct {
  int status;
  long long iters_done;    /* accepted iterations performed by this call          */
  long long total;         /* == engine.iters (cumulative accepted iterations)    */
  long long inner;         /* iterations since the last restart                   */
  long long evals_total;
  double tau_cand, tau_prev, gamma, sigma_prev, T;
  double fail_tau, fail_gamma;
  long long fail_iter;
  double metrics[8];       /* kkt, stationarity, primal_eq, complementarity,
                              infeas, f_value, mean_pos_violation, subopt_abs     */
  int has_metrics;
  double sweep_ns;         /* device time spent in Q sweeps (globaltimer)         */
  long long sweeps;        /* number of Q sweeps                                  */
  double kernel_ms;        /* CUDA-event time of this call's solver launch        */
  long long sweep_bytes;   /* algorithmic bytes of one sweep (streamed Q rows)    */
} rapdb_run_result;

/* process-wide number of kernel launches issued by this library */
long long rapdb_launch_count(void);

/* ---- constraint sharding ---------------------------
 * Rank r binds only its matrices [k0, k1) of the m+1 stack (rapdb_bind_dense);
 * x, (v, lam), q, r, A, b and the bounds are replicated.  A sharded context
 * ("split", set automatically when nranks > 1, or forced for testing) stops at
 * every exchange point and calls `fn(user, kind)`; the callback must sum the
 * buffer(s) returned by rapdb_exchange_buffers(kind) across all ranks
 * (all-reduce, identical result on every rank) and return 0; the op then
 * resumes.  Exchange kinds: 1 partial grad_x Phi (n), 2 constraint values
 * g (m+1, exact: disjoint supports), 3 two gradients (n + n, APDB-xy),
 * 4 H (n*n, smoothed gap).  Per yx trial: one n-vector and one (m+1)-vector. */
typedef int (*rapdb_exchange_fn)(void* user, int kind);
int rapdb_set_exchange(rapdb_ctx* ctx, rapdb_exchange_fn fn, void* user, int force_split);
int rapdb_exchange_buffers(rapdb_ctx* ctx, int kind, double** buf0, long long* count0,
                           double** buf1, long long* count1);
/* number of exchanges performed by this context so far */
long long rapdb_exchange_count(const rapdb_ctx* ctx);

/* Native exchange over NCCL (the default of the Python binding's
 * nccl_shard): one communicator per process and GPU, bootstrapped from a
 * 128-byte ncclUniqueId that rank 0 creates and the caller distributes.  A
 * context given a communicator sums its exchange buffers itself, on its
 * stream, without calling back into the host: NCCL only moves bytes
 * (all-gather, or send/recv + all-gather for long buffers) and a kernel of
 * this library adds the R partials in rank order, so every rank -- and the
 * emulated / peer-memory paths -- gets the same bits whatever algorithm NCCL
 * picks (fixed reduction order).                               */
typedef struct rapdb_comm rapdb_comm;
int rapdb_comm_unique_id(unsigned char* id128);
int rapdb_comm_create(int device, const unsigned char* id128, int rank, int nranks, rapdb_comm** out);
void rapdb_comm_destroy(rapdb_comm* comm);
/* rank-ordered in-place all-reduce of a device buffer (synchronises stream) */
int rapdb_comm_allreduce_ordered(rapdb_comm* comm, double* buf, long long count, void* stream);
/* use `comm` for this context's exchanges (replaces rapdb_set_exchange)     */
int rapdb_set_comm_exchange(rapdb_ctx* ctx, rapdb_comm* comm, int force_split);

/* In-kernel exchange over NVLink peer memory (dense shards; opt-in): each
 * rank allocates a zeroed device region of rapdb_peer_region_bytes(ctx)
 * bytes (rapdb_region_alloc), shares it with the other ranks (CUDA IPC handles:
 * rapdb_ipc_handle / rapdb_ipc_open / rapdb_ipc_close), and passes the R
 * device pointers (regions[rank] = its own) to rapdb_set_peer_exchange.  The
 * per-trial gradient / g exchanges then run inside the persistent kernel:
 * push the partial into slot `rank` of every peer, release-signal every peer,
 * acquire all R signals, sum the R slots in rank order -- no host round trip.
 * The smoothed gap's H still goes through the exchange callback.          */
long long rapdb_peer_region_bytes(rapdb_ctx* ctx);
/* a zeroed device allocation of its own (an IPC handle names a whole
 * allocation, so the region must not live inside a pooled block)           */
int rapdb_region_alloc(long long bytes, void** dptr);
int rapdb_region_free(void* dptr);
int rapdb_ipc_handle(const void* dptr, unsigned char* handle64);
int rapdb_ipc_open(const unsigned char* handle64, void** dptr);
int rapdb_ipc_close(void* dptr);
int rapdb_set_peer_exchange(rapdb_ctx* ctx, void* const* regions);

/* cumulative device time (ns, CTA 0 globaltimer) and call counts per step of
 * the op state machine (step ids: rapdb_dev.cuh enum Step), for profiling */
int rapdb_step_profile(rapdb_ctx* ctx, double* ns, long long* counts, int nsteps);

/* problem.spectral_norm (problem.py:47-68) of a dense device matrix M
 * [rows][ld] (ld >= cols): power iteration on M'M from cos(k + 1/2), at most
 * iters steps, stop when |est - prev| <= tol max(est, 1); *out = 1.01 est.
 * Runs on `stream` and synchronises it.                                     */
int rapdb_spectral_norm(const double* M, long long rows, long long cols, long long ld, int iters, double tol,
                        void* stream, double* out);

/* Debug: with RAPDB_GUARD=1 in the environment when the workspace size is
 * queried, every workspace buffer is followed by a 4 KB guard zone filled
 * with a byte pattern; this returns the number of buffers whose guard was
 * written (report: which), 0 when all are intact or guards are off.        */
int rapdb_check_guards(rapdb_ctx* ctx, char* report, int size);

/* version of the ABI (bumped on incompatible change) */
int rapdb_abi_version(void);

/* context ------------------------------------------------------------------ */
int rapdb_create(int device, int rank, int nranks, rapdb_ctx** out);
void rapdb_destroy(rapdb_ctx* ctx);
int rapdb_last_error(const rapdb_ctx* ctx, char* buf, int size);
int rapdb_set_stream(rapdb_ctx* ctx, void* cuda_stream);

/* problem data: replaces ProblemInstance's Q/q/r/A/b/primal_set storage
 * (problem.py:109-162, _as_operator problem.py:31-40).  Q is the local shard
 * of the (m+1)-matrix stack, matrices k0..k1-1, laid out [k1-k0][n][ld] with
 * ld even and ld >= n (zero padded).  q is [(m+1)][n], r [m+1], A [p][n],
 * b [p], lower/upper [n] (+-inf allowed).  zero_flags (HOST, k1-k0 bytes)
 * marks all-zero local matrices that the sweep skips.                         */
int rapdb_bind_dense(rapdb_ctx* ctx, int n, int m, int p, int k0, int k1, long long ld,
                     const double* Q, const double* q, const double* r,
                     const double* A, const double* b,
                     const double* lower, const double* upper, double mu,
                     const unsigned char* zero_flags);

/* Packed symmetric layout of the same stack (the default of the Python
 * binding).  Every Q_i is symmetric (the reference validates it at load time,
 * problem.py:142-144), so only the upper block triangle is stored and
 * streamed: half the HBM bytes of the row-major stack.  Qp is the local shard
 * [k1-k0][rapdb_packed_doubles(n)] built by rapdb_pack_symmetric; every other
 * argument is as for rapdb_bind_dense.  Layout: 32 x 32 row-major sub-tiles in
 * 64 x 64 units, units block-row-major over Bi <= Bj, diagonal units storing
 * (0,0), (0,1), (1,1) (paper_2605_29291_b200/csrc/symsweep.cuh).             */
int rapdb_bind_dense_packed(rapdb_ctx* ctx, int n, int m, int p, int k0, int k1,
                            const double* Qp, const double* q, const double* r,
                            const double* A, const double* b,
                            const double* lower, const double* upper, double mu,
                            const unsigned char* zero_flags);

/* doubles of one packed n x n matrix (upper block triangle incl. zero padding) */
long long rapdb_packed_doubles(int n);

/* Pack `count` dense n x n matrices (row stride ld, matrix stride mat_stride
 * doubles) into the packed layout at dst (device).  src may be device memory
 * or page-locked host memory (read through the unified address space, so only
 * the upper triangle crosses PCIe).  Runs on `stream` and synchronises it.  */
int rapdb_pack_symmetric(int n, long long count, const double* src, long long ld,
                         long long mat_stride, double* dst, void* stream);

/* Sliced ELLPACK (slice height 32) of a sparse operand, all arrays on the
 * device: slots are grouped 32 to a slice (one warp, lane = slot); entry t of
 * slot s lives at sp[s / 32] + 32 t + s % 32, a slice being as wide as its
 * longest slot (shorter slots are padded; len says where each stops).  Every
 * slot's entries are in the operand's stored order, which is the order they
 * are summed in (no FMA: the bits of scipy's csr_matvec).                   */
typedef struct rapdb_sell {
  long long nslots;      /* multiple of 32                                   */
  const long long* sp;   /* [nslots / 32 + 1] entry offset of each slice     */
  const int* idx;        /* [sp[nslots / 32]] gathered index of each entry   */
  const double* val;     /* [sp[nslots / 32]]                                */
  const int* len;        /* [nslots] entries of each slot                    */
  const int* map;        /* [nslots] output index of each slot, -1 = padding;
                            NULL where the slot number is the output index   */
} rapdb_sell;

/* Factored sparse problem data (BASELINE config 3): replaces a ProblemInstance
 * whose Q_i are sparse operators (_as_operator problem.py:31-40 keeps them as
 * CSR) with Q_i = R_i^T R_i, plus L linear inequality rows a_j x <= b_j that
 * the reference would hold as Q = 0 orthant constraints (problem.py:38-39:
 * an all-zero Q becomes an empty CSR).  Constraint order: m = mq + L, rows
 * 1..mq quadratic (q = C[1..mq], r = d[1..mq]), rows mq+1..m linear.
 *   R     [nr x n], the stacked R_0..R_mq; block i owns rows rblk[i]..rblk[i+1].
 *         Sell with idx = column and the slots laid out per block in chunks
 *         of 128 rows: slot = 128 * (chunks of the earlier blocks) + row
 *         inside the block, each block padded to a multiple of 128 slots
 *         (nslots = 128 * sum_i ceil(rows_i / 128)), map = NULL
 *   rmat  [nr] block id of each stacked row (int32)
 *   rblk  HOST [mq+2] row offsets of the blocks (rblk[0] = 0, rblk[mq+1] = nr)
 *   C     [(mq+1) x n] linear terms, d [mq+1] constants
 *   A     [L x n], Sell with idx = column, slot = row, nslots = L rounded up
 *         to 32, map = NULL; b [L]
 * All other pointers are device pointers.  R^T and A^T follow with
 * rapdb_set_factored_transpose (required before any op).  No equality block
 * (p = 0), and the smoothed gap is not available (its n x n H does not fit at
 * this n): adaptive restarts need a dense instance.  Dual balls are supported
 * (the trial multipliers are scaled in place after one norm reduction).
 * Equivalent to rapdb_bind_factored_range over the whole instance.          */
int rapdb_bind_factored(rapdb_ctx* ctx, int n, int mq, int L, long long nr,
                        const rapdb_sell* R, const int* rmat, const long long* rblk,
                        const double* C, const double* d, const rapdb_sell* A,
                        const double* b, const double* lower, const double* upper, double mu);

/* The same, holding only a constraint shard: blocks
 * [fb0, fb1) of the mq+1 quadratic blocks (R rows, rblk with fb1-fb0+1
 * entries, rmat LOCAL block ids, C and d rows fb0..fb1-1) and linear rows
 * [l0, l1) of the L (A with local row ids, b).  mq and L are the global
 * counts; x and the m multipliers are replicated.  The context exchanges the
 * gradient partial (n) and g (m+1, zero outside this rank's rows) per trial. */
int rapdb_bind_factored_range(rapdb_ctx* ctx, int n, int mq, int L, int fb0, int fb1, int l0, int l1,
                              long long nr, const rapdb_sell* R, const int* rmat, const long long* rblk,
                              const double* C, const double* d, const rapdb_sell* A,
                              const double* b, const double* lower, const double* upper, double mu);

/* The transposed operands of the gradient gather grad_x Phi = sum_i w_i
 * (R_i^T W_i + c_i) + A^T mu (no atomics, fixed summation order), after a
 * factored bind.  The stacked rows of R are split into nph <= 8 ROW PHASES
 * ph_bounds[0..nph] (HOST, 0 .. nr) so that each phase gathers from an
 * L2-sized slice of the W-cache; RT[ph] is the Sell of (rows of phase ph of
 * R)^T: nslots = n rounded up to 32, the columns sorted by their entry count
 * in the phase (map[slot] = column, every column exactly once), entries of a
 * column in row order with idx = stacked row -- or, `tagged`, row | (local
 * block of the row) << 23, which lets the gather weight W on the fly (needs
 * nr <= 2^23 and at most 256 local blocks).  AT is the Sell of A^T (local
 * rows) over the same kind of column slots.                                 */
int rapdb_set_factored_transpose(rapdb_ctx* ctx, int nph, const long long* ph_bounds, const rapdb_sell* RT,
                                 const rapdb_sell* AT, int tagged);

/* Sparse symmetric Q stack (the reference keeps a Q_i below 25 % density as
 * CSR, _as_operator problem.py:31-40): bind the stacked Q_0..Q_m through
 * rapdb_bind_factored as the "R" operand with n rows per block (mq = m,
 * C = q, d = r), pass empty transposes, and set this flag.  The blocks are
 * then applied as Q_i themselves: the W-cache holds u_i = Q_i x (each row
 * summed in CSR order: the bits of scipy's csr_matvec the reference calls),
 * g_i = 1/2 x . u_i + q_i . x + r_i, and grad_x Phi = sum_i w_i (u_i + q_i)
 * + A^T mu in the reference's operation order (problem.py:205-214).        */
int rapdb_set_factored_symmetric(rapdb_ctx* ctx, int symmetric);

/* SolverConfig.resolved() (engine.py:33-63); mode 0 = yx, 1 = xy;
 * ball_kind 0/1/2 = Unbounded / JointBall(r1) / SplitBall(r1=v, r2=lam)       */
int rapdb_set_params(rapdb_ctx* ctx, int mode, double c_alpha, double c_beta, double delta,
                     double eta, double tau_bar, double gamma0, int nonmonotone,
                     int max_backtracks, int ball_kind, double r1, double r2);

/* workspace: size query after bind+params, then a caller-owned device buffer */
long long rapdb_workspace_bytes(rapdb_ctx* ctx);
int rapdb_bind_workspace(rapdb_ctx* ctx, void* dptr, long long bytes);

/* ApdbEngine.reinit (engine.py:102-136).  source 0: explicit point (device
 * pointers x[n], v[p], lam[m]); 1: current iterate; 2: ergodic average.
 * reset_inner zeroes the since-restart counter (run_restarted's `inner`).     */
int rapdb_reinit(rapdb_ctx* ctx, int source, const double* x, const double* v,
                 const double* lam, int warm_tau, int reset_inner);

/* Accepted iterations with device-side backtracking, KKT cadence, termination
 * and fixed restarts (engine.py:198-259 inside restarts.py:111-161).  trace is
 * a device buffer of max_iters * RAPDB_TRACE_COLS doubles (row-major).        */
int rapdb_run(rapdb_ctx* ctx, const rapdb_run_args* args, double* trace, rapdb_run_result* out);

/* Extragradient baseline (egm.py:37-77) from the
 * current point (set it with rapdb_reinit: the projection Pi of egm.py:52):
 * K iterations of z~ = Pi(z - s F(z)), z+ = Pi(z - s F(z~)), two sweeps each,
 * stopping early when |z| > 1e8 (1 + |z0|).  Afterwards rapdb_get_iterate
 * returns the last point (which 0) and the plain average (which 1).  trace:
 * device buffer of (K / trace_every) rows (iter, |z|), or NULL with
 * trace_every = 0.                                                          */
int rapdb_egm(rapdb_ctx* ctx, double stepsize, long long K, int trace_every, double* trace,
              long long* iterations, int* diverged);

/* kkt_residual at the current iterate (diagnostics.py:96-113); out[8] host   */
int rapdb_kkt(rapdb_ctx* ctx, int has_f_star, double f_star, double* out);

/* kkt_residual (diagnostics.py:96-113) and coupling_value (problem.py:196-204)
 * at an explicit point (device x[n], v[p], lam[m]; evaluated where given, no
 * projection): one fused sweep at x, g, grad_x Phi, the residual norms.
 * out[9] host = kkt, stationarity, primal_eq, complementarity, infeas,
 * f_value, mean_pos_violation, subopt_abs (NaN without f_star), Phi.
 * Unsharded contexts only.                                                   */
/* eq_residual (problem.py:175-177): A x - b at device x into device eq[p]    */
int rapdb_eq_residual(rapdb_ctx* ctx, const double* x, double* eq);

int rapdb_kkt_at(rapdb_ctx* ctx, const double* x, const double* v, const double* lam, int has_f_star, double f_star,
                 double* out);

/* engine.last / engine.average() (engine.py:262-272) into device buffers     */
int rapdb_get_iterate(rapdb_ctx* ctx, int which, double* x, double* v, double* lam);

/* One fused sweep at x (device): u[(k1-k0)][n] (factored: W = R x, [nr]) and
 * g[m+1] (index 0 = f) into device buffers; reps > 1 repeats it (timing);
 * *ms = mean device ms/sweep.  g_value/f_value (problem.py:166-180).          */
int rapdb_probe_sweep(rapdb_ctx* ctx, const double* x, double* u, double* g, int reps, float* ms);

/* grad_x_coupling (problem.py:207-217) and g (problem.py:172-180) at an
 * arbitrary point: gx[n] = grad_x Phi(x, v, lam), g[m+1] (index 0 = f); all
 * device pointers; unsharded contexts only.                                  */
int rapdb_grad_x(rapdb_ctx* ctx, const double* x, const double* v, const double* lam, double* gx, double* g);

/* smoothed_gap(z, xi) (diagnostics.py:120-163) at an explicit point (source 0:
 * device x[n], v[p], lam[m], used as given -- no projection), the current
 * iterate (1) or the ergodic average (2): closed-form dual step, dense
 * H = Q0 + sum lam_i Q_i built in one pass over the stack, power iteration for
 * ||H|| (problem.py:47-68), accelerated projected gradient with function-value
 * restart on Phi(., y) + xi |. - x|^2 (subsolve.py:27-62), all in one device
 * launch.  x_warm: device pointer or NULL.  x_cand (device, n) receives the
 * candidate's x for the next warm start (restarts.py:148).
 * out[6] host = gap, subsolver iterations, residual, converged, L, dual_term. */
int rapdb_smoothed_gap(rapdb_ctx* ctx, int source, const double* x, const double* v, const double* lam,
                       double xi, double tol, const double* x_warm, double* x_cand, double* out);

#ifdef __cplusplus
}
#endif
#endif
