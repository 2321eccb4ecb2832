"""ctypes binding of the C ABI (include/rapdb_b200.h) -- no CPU fallback.

``load()`` opens ``_rapdb_b200.so`` built in-tree by ``csrc/Makefile``; if the
library or a CUDA device is missing every solver entry point raises
``DeviceError`` instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from .errors import ConfigurationError, DeviceError, InputError, NonConvergence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RAPDB_LIB") or os.path.join(_HERE, "_rapdb_b200.so")   # RAPDB_LIB: A/B builds (tools/)

TRACE_COLS = 11
RUN_LIMIT, RUN_CONVERGED, RUN_BUDGET, RUN_CHECK_DUE, RUN_FIXED_DUE, RUN_NONCONV, RUN_ABORT = range(7)


class RunArgs(C.Structure):
    _fields_ = [("max_iters", C.c_longlong), ("budget", C.c_longlong), ("stop_total", C.c_longlong),
                ("metrics_every", C.c_int), ("criterion", C.c_int),
                ("eps", C.c_double), ("eps_kkt", C.c_double), ("eps_feas", C.c_double),
                ("f_star", C.c_double), ("has_f_star", C.c_int), ("fixed_period", C.c_int),
                ("fixed_point", C.c_int), ("warm_tau", C.c_int), ("stop_at_fixed", C.c_int)]


class RunResult(C.Structure):
    _fields_ = [("status", C.c_int), ("iters_done", C.c_longlong), ("total", C.c_longlong),
                ("inner", C.c_longlong), ("evals_total", C.c_longlong),
                ("tau_cand", C.c_double), ("tau_prev", C.c_double), ("gamma", C.c_double),
                ("sigma_prev", C.c_double), ("T", C.c_double),
                ("fail_tau", C.c_double), ("fail_gamma", C.c_double), ("fail_iter", C.c_longlong),
                ("metrics", C.c_double * 8), ("has_metrics", C.c_int),
                ("sweep_ns", C.c_double), ("sweeps", C.c_longlong),
                ("kernel_ms", C.c_double), ("sweep_bytes", C.c_longlong)]


_lib = None
EXPORTS = ["rapdb_abi_version", "rapdb_create", "rapdb_destroy", "rapdb_last_error", "rapdb_set_stream",
           "rapdb_bind_dense", "rapdb_set_params", "rapdb_workspace_bytes", "rapdb_bind_workspace",
           "rapdb_reinit", "rapdb_run", "rapdb_kkt", "rapdb_get_iterate", "rapdb_probe_sweep",
           "rapdb_smoothed_gap", "rapdb_launch_count", "rapdb_set_exchange", "rapdb_exchange_buffers",
           "rapdb_exchange_count", "rapdb_step_profile", "rapdb_bind_factored", "rapdb_grad_x",
           "rapdb_bind_dense_packed", "rapdb_packed_doubles", "rapdb_pack_symmetric",
           "rapdb_bind_factored_range", "rapdb_egm", "rapdb_peer_region_bytes", "rapdb_ipc_handle",
           "rapdb_ipc_open", "rapdb_ipc_close", "rapdb_set_peer_exchange", "rapdb_region_alloc",
           "rapdb_region_free", "rapdb_comm_unique_id", "rapdb_comm_create", "rapdb_comm_destroy",
           "rapdb_comm_allreduce_ordered", "rapdb_set_comm_exchange", "rapdb_set_factored_transpose", "rapdb_set_factored_symmetric",
           "rapdb_spectral_norm", "rapdb_kkt_at", "rapdb_eq_residual",
           "rapdb_check_guards"]

_STEPS = ["T_BEGIN", "TY_DUAL", "TY_GXPART", "TY_PRIMAL", "TY_SWEEP", "TY_GLOCAL", "TY_GY", "TY_DECIDE",
          "TX_PRIMAL", "TX_SWEEP", "TX_GLOCAL", "TX_DUAL", "TX_GXPART", "TX_NORMS", "TX_DECIDE",
          "A_POST", "K_GXPART", "K_FINISH", "A_RESTART", "A_END",
          "R_POINT", "R_SWEEP", "R_GLOCAL", "R_CACHE", "R_GXPART", "R_GXCACHE", "R_FINISH",
          "G_CAND", "G_GLOCAL", "G_HPART", "G_SOLVE", "P_SWEEP", "P_OUT", "P_GRAD", "P_GFIN", "P_KKT",
          "E_INIT", "E_GX", "E_HALF", "E_HSWEEP", "E_HGLOC", "E_GXH", "E_PLUS", "E_PSWEEP", "E_PGLOC",
          "E_POST", "DONE"]            # enum Step (csrc/rapdb_dev.cuh), in order
# SolverState::step_ns has 64 slots: the steps, then the packed sweep's
# sub-phases at 60, 61, 62 (sub_time in csrc/solver_kernel.cuh)
STEP_NAMES = _STEPS + [""] * (60 - len(_STEPS)) + ["sweep:stage_x", "sweep:stream", "sweep:reduce", ""]
assert len(STEP_NAMES) == 64 and STEP_NAMES[60] == "sweep:stage_x"

EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int)
X_GX, X_G, X_GX2, X_H = 1, 2, 3, 4


def launch_count() -> int:
    """Kernel launches issued by the native library in this process."""
    return int(load().rapdb_launch_count())


def packed_doubles(n: int) -> int:
    """Doubles of one packed (upper block triangle) n x n matrix."""
    return int(load().rapdb_packed_doubles(int(n)))


def pack_symmetric(n: int, count: int, src_ptr: int, ld: int, mat_stride: int, dst_ptr: int, stream_ptr: int):
    """Pack `count` dense matrices (device or page-locked host memory) into the
    packed symmetric layout at dst (device); synchronises the stream."""
    code = load().rapdb_pack_symmetric(int(n), int(count), C.c_void_p(src_ptr), int(ld), int(mat_stride),
                                       C.c_void_p(dst_ptr), C.c_void_p(stream_ptr))
    if code != 0:
        raise DeviceError(f"rapdb_pack_symmetric failed (code {code})")


def ipc_handle(dptr: int) -> bytes:
    buf = C.create_string_buffer(64)
    if load().rapdb_ipc_handle(C.c_void_p(int(dptr)), buf) != 0:
        raise DeviceError("cudaIpcGetMemHandle failed")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    out = C.c_void_p()
    if load().rapdb_ipc_open(handle, C.byref(out)) != 0:
        raise DeviceError("cudaIpcOpenMemHandle failed")
    return int(out.value)


def ipc_close(dptr: int) -> None:
    load().rapdb_ipc_close(C.c_void_p(int(dptr)))


class PeerRegion:
    """A zeroed cudaMalloc'd region (freed with the object)."""

    def __init__(self, nbytes: int):
        out = C.c_void_p()
        if load().rapdb_region_alloc(int(nbytes), C.byref(out)) != 0:
            raise DeviceError("peer region allocation failed")
        self.ptr = int(out.value)

    def __del__(self):
        try:
            if self.ptr:
                load().rapdb_region_free(C.c_void_p(self.ptr))
        except Exception:   # interpreter shutdown
            pass


def spectral_norm(M, iters: int, tol: float) -> float:
    """rapdb_spectral_norm of a float64 CUDA tensor [rows][cols] (row stride = stride(0))."""
    import torch
    if M.dtype != torch.float64 or not M.is_cuda or M.dim() != 2 or M.stride(1) != 1:
        raise InputError("need a row-major float64 CUDA matrix")
    out = C.c_double()
    code = load().rapdb_spectral_norm(C.c_void_p(M.data_ptr()), M.shape[0], M.shape[1], M.stride(0), int(iters),
                                      float(tol), C.c_void_p(torch.cuda.current_stream(M.device).cuda_stream),
                                      C.byref(out))
    if code != 0:
        raise DeviceError(f"rapdb_spectral_norm failed (code {code})")
    return float(out.value)


def comm_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for rapdb_comm_create."""
    buf = C.create_string_buffer(128)
    if load().rapdb_comm_unique_id(buf) != 0:
        raise DeviceError("ncclGetUniqueId failed")
    return buf.raw


class Comm:
    """Native NCCL communicator (rapdb_comm): the library's rank-ordered
    exchange for sharded contexts.  Collective: every rank constructs it with
    the same unique id."""

    def __init__(self, device_index: int, unique_id: bytes, rank: int, nranks: int):
        if len(unique_id) != 128:
            raise InputError("an ncclUniqueId is 128 bytes")
        self.lib = load()
        self.rank, self.nranks, self.device_index = rank, nranks, device_index
        h = C.c_void_p()
        if self.lib.rapdb_comm_create(int(device_index), unique_id, int(rank), int(nranks), C.byref(h)) != 0:
            raise DeviceError(f"ncclCommInitRank failed (rank {rank} of {nranks})")
        self.h = h

    def allreduce_ordered(self, t, stream_ptr: int = 0):
        """In-place rank-ordered sum of a contiguous float64 CUDA tensor."""
        if t.dtype.itemsize != 8 or not t.is_contiguous() or not t.is_cuda:
            raise InputError("need a contiguous float64 CUDA tensor")
        if self.lib.rapdb_comm_allreduce_ordered(self.h, C.c_void_p(t.data_ptr()), t.numel(),
                                                 C.c_void_p(stream_ptr)) != 0:
            raise DeviceError("rank-ordered all-reduce failed")

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.rapdb_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter shutdown
            pass


def load(path: str = LIB_PATH):
    """Open the native library (raises DeviceError when it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(f"native library {path} is missing; run `make -C paper_2605_29291_b200/csrc` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    P, D, I, LL = C.c_void_p, C.c_double, C.c_int, C.c_longlong
    lib.rapdb_abi_version.restype = I
    lib.rapdb_create.argtypes = [I, I, I, C.POINTER(P)]
    lib.rapdb_destroy.argtypes = [P]
    lib.rapdb_destroy.restype = None
    lib.rapdb_last_error.argtypes = [P, C.c_char_p, I]
    lib.rapdb_set_stream.argtypes = [P, P]
    lib.rapdb_bind_dense.argtypes = [P, I, I, I, I, I, LL, P, P, P, P, P, P, P, D, P]
    lib.rapdb_bind_dense_packed.argtypes = [P, I, I, I, I, I, P, P, P, P, P, P, P, D, P]
    lib.rapdb_packed_doubles.argtypes = [I]
    lib.rapdb_packed_doubles.restype = LL
    lib.rapdb_pack_symmetric.argtypes = [I, LL, P, LL, LL, P, P]
    lib.rapdb_set_params.argtypes = [P, I, D, D, D, D, D, D, I, I, I, D, D]
    lib.rapdb_workspace_bytes.argtypes = [P]
    lib.rapdb_workspace_bytes.restype = LL
    lib.rapdb_bind_workspace.argtypes = [P, P, LL]
    lib.rapdb_reinit.argtypes = [P, I, P, P, P, I, I]
    lib.rapdb_run.argtypes = [P, C.POINTER(RunArgs), P, C.POINTER(RunResult)]
    lib.rapdb_kkt.argtypes = [P, I, D, C.POINTER(D)]
    lib.rapdb_get_iterate.argtypes = [P, I, P, P, P]
    lib.rapdb_probe_sweep.argtypes = [P, P, P, P, I, C.POINTER(C.c_float)]
    lib.rapdb_smoothed_gap.argtypes = [P, I, P, P, P, D, D, P, P, C.POINTER(D)]
    lib.rapdb_launch_count.restype = LL
    lib.rapdb_set_exchange.argtypes = [P, EXCHANGE_FN, P, I]
    lib.rapdb_exchange_buffers.argtypes = [P, I, C.POINTER(C.c_void_p), C.POINTER(LL),
                                           C.POINTER(C.c_void_p), C.POINTER(LL)]
    lib.rapdb_exchange_count.argtypes = [P]
    lib.rapdb_exchange_count.restype = LL
    lib.rapdb_step_profile.argtypes = [P, C.POINTER(D), C.POINTER(LL), I]
    lib.rapdb_bind_factored.argtypes = [P, I, I, I, LL] + [P] * 9 + [D]
    lib.rapdb_bind_factored_range.argtypes = [P, I, I, I, I, I, I, I, LL] + [P] * 9 + [D]
    lib.rapdb_egm.argtypes = [P, D, LL, I, P, C.POINTER(LL), C.POINTER(I)]
    lib.rapdb_peer_region_bytes.argtypes = [P]
    lib.rapdb_peer_region_bytes.restype = LL
    lib.rapdb_ipc_handle.argtypes = [P, C.c_char_p]
    lib.rapdb_ipc_open.argtypes = [C.c_char_p, C.POINTER(P)]
    lib.rapdb_ipc_close.argtypes = [P]
    lib.rapdb_region_alloc.argtypes = [LL, C.POINTER(P)]
    lib.rapdb_region_free.argtypes = [P]
    lib.rapdb_set_peer_exchange.argtypes = [P, C.POINTER(P)]
    lib.rapdb_grad_x.argtypes = [P, P, P, P, P, P]
    lib.rapdb_comm_unique_id.argtypes = [C.c_char_p]
    lib.rapdb_comm_create.argtypes = [I, C.c_char_p, I, I, C.POINTER(P)]
    lib.rapdb_comm_destroy.argtypes = [P]
    lib.rapdb_comm_destroy.restype = None
    lib.rapdb_comm_allreduce_ordered.argtypes = [P, P, LL, P]
    lib.rapdb_set_comm_exchange.argtypes = [P, P, I]
    lib.rapdb_set_factored_transpose.argtypes = [P, I, P, P, P, I]
    lib.rapdb_set_factored_symmetric.argtypes = [P, I]
    lib.rapdb_spectral_norm.argtypes = [P, LL, LL, LL, I, D, P, C.POINTER(D)]
    lib.rapdb_kkt_at.argtypes = [P, P, P, P, I, D, C.POINTER(D)]
    lib.rapdb_eq_residual.argtypes = [P, P, P]
    lib.rapdb_check_guards.argtypes = [P, C.c_char_p, I]
    _lib = lib
    return lib


class SellDescriptor(C.Structure):
    """``rapdb_sell`` of include/rapdb_b200.h (device pointers)."""
    _fields_ = [("nslots", C.c_longlong), ("sp", C.c_void_p), ("idx", C.c_void_p), ("val", C.c_void_p),
                ("len", C.c_void_p), ("map", C.c_void_p)]


def _ptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


class Context:
    """One device solver context bound to a device instance (see problem.DeviceData)."""

    def __init__(self, device_index: int = 0, rank: int = 0, nranks: int = 1):
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the rAPDB path runs only on the GPU (no CPU fallback)")
        self.lib = load()
        self.torch = torch
        self.device = torch.device("cuda", device_index)
        h = C.c_void_p()
        self._check(self.lib.rapdb_create(device_index, rank, nranks, C.byref(h)), ctx=None)
        self.h = h
        self.ws = None
        self.data = None

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and self.h.value:
                self.lib.rapdb_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # -- error mapping (rapdb_b200.h return codes) --------------------------
    def _msg(self):
        buf = C.create_string_buffer(512)
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.rapdb_last_error(self.h, buf, 512)
        return buf.value.decode(errors="replace")

    def _check(self, code, ctx="self", state=None):
        if code == 0:
            return
        msg = self._msg() if ctx is not None else f"rapdb_create failed ({code})"
        if code == 1:
            raise InputError(msg)
        if code == 2:
            raise ConfigurationError(msg)
        if code == 3:
            raise NonConvergence(msg, state=state)
        raise DeviceError(msg)

    def stream(self):
        return self.torch.cuda.current_stream(self.device)

    def _set_stream(self):
        self.lib.rapdb_set_stream(self.h, C.c_void_p(self.stream().cuda_stream))

    # -- sharding ----------------------------------------------------------
    def set_exchange(self, fn, force_split=False):
        """fn(kind) -> None must all-reduce (sum) self.exchange_views(kind) across
        ranks.  Must be called before bind()."""
        def _cb(user, kind):
            try:
                fn(int(kind))
                return 0
            except Exception as exc:  # surfaced as DeviceError by the C side
                self._cb_error = exc
                return 1
        self._cb = EXCHANGE_FN(_cb)      # keep the thunk alive
        self._check(self.lib.rapdb_set_exchange(self.h, self._cb, None, 1 if force_split else 0))

    def set_comm_exchange(self, comm: "Comm", force_split=False):
        """Exchanges summed by the library itself over `comm` (no host callback)."""
        self._comm = comm      # keep the communicator alive with the context
        self._check(self.lib.rapdb_set_comm_exchange(self.h, comm.h, 1 if force_split else 0))

    def exchange_views(self, kind):
        """float64 views into the workspace of the buffer(s) to all-reduce."""
        b0, b1 = C.c_void_p(), C.c_void_p()
        n0, n1 = C.c_longlong(), C.c_longlong()
        self._check(self.lib.rapdb_exchange_buffers(self.h, kind, C.byref(b0), C.byref(n0),
                                                    C.byref(b1), C.byref(n1)))
        base = self.ws.data_ptr()
        out = []
        for b, cnt in ((b0, n0), (b1, n1)):
            if b.value and cnt.value > 0:
                off = b.value - base
                out.append(self.ws[off:off + 8 * cnt.value].view(self.torch.float64))
        return out

    def peer_region_bytes(self) -> int:
        return int(self.lib.rapdb_peer_region_bytes(self.h))

    def set_peer_exchange(self, regions):
        """regions: R device pointers (ints), this rank's own at index rank."""
        arr = (C.c_void_p * len(regions))(*[C.c_void_p(int(r)) for r in regions])
        self._check(self.lib.rapdb_set_peer_exchange(self.h, arr))

    def exchange_count(self):
        return int(self.lib.rapdb_exchange_count(self.h))

    def step_profile(self):
        """{step name: (total device ms, calls)} accumulated since bind."""
        ns = (C.c_double * 64)()
        cnt = (C.c_longlong * 64)()
        self._check(self.lib.rapdb_step_profile(self.h, ns, cnt, 64))
        return {name: (ns[i] / 1e6, int(cnt[i])) for i, name in enumerate(STEP_NAMES) if cnt[i]}

    # -- binding -----------------------------------------------------------
    def bind(self, data, cfg, k0=0, k1=None):
        """data: problem.DeviceData (data.Q holds matrices k0..k1-1) or
        factored.FactoredDeviceData; cfg: resolved SolverConfig."""
        self._set_stream()
        if getattr(data, "factored", False):
            rblk = np.ascontiguousarray(data.rblk, dtype=np.int64)
            self._check(self.lib.rapdb_bind_factored_range(
                self.h, data.n, data.mq, data.L, data.k0, data.k1, data.l0, data.l1, data.nr,
                C.byref(data.sell_R.descriptor()), _ptr(data.rmat), rblk.ctypes.data_as(C.c_void_p),
                _ptr(data.C), _ptr(data.d), C.byref(data.sell_A.descriptor()),
                _ptr(data.b), _ptr(data.lower), _ptr(data.upper), float(data.mu)))
            bounds = np.ascontiguousarray(data.rt_bounds, dtype=np.int64)
            rt = (SellDescriptor * int(data.rt_nph))(*[t.descriptor() for t in data.sell_RT])
            self._check(self.lib.rapdb_set_factored_transpose(
                self.h, int(data.rt_nph), bounds.ctypes.data_as(C.c_void_p), rt,
                C.byref(data.sell_AT.descriptor()), int(data.rt_tag)))
            if getattr(data, "sym", False):
                self._check(self.lib.rapdb_set_factored_symmetric(self.h, 1))
        else:
            k1 = data.m + 1 if k1 is None else k1
            zero = np.ascontiguousarray(data.zero_flags, dtype=np.uint8)
            tail = (_ptr(data.q), _ptr(data.r), _ptr(data.A) if data.p else None,
                    _ptr(data.b) if data.p else None, _ptr(data.lower), _ptr(data.upper), float(data.mu),
                    zero.ctypes.data_as(C.c_void_p))
            if getattr(data, "layout", "rows") == "packed":
                self._check(self.lib.rapdb_bind_dense_packed(
                    self.h, data.n, data.m, data.p, k0, k1, _ptr(data.Q), *tail))
            else:
                self._check(self.lib.rapdb_bind_dense(
                    self.h, data.n, data.m, data.p, k0, k1, data.ld, _ptr(data.Q), *tail))
        self._set_params(cfg)
        nbytes = int(self.lib.rapdb_workspace_bytes(self.h))
        if nbytes <= 0:
            raise DeviceError("workspace size query failed")
        self.ws = self.torch.empty(nbytes + 256, dtype=self.torch.uint8, device=self.device)
        base = self.ws.data_ptr()
        off = (-base) % 256
        self._check(self.lib.rapdb_bind_workspace(self.h, C.c_void_p(base + off), nbytes))
        self.data = data

    def _set_params(self, cfg):
        from .geometry import ball_code
        kind, r1, r2 = ball_code(cfg.dual_ball)
        self._check(self.lib.rapdb_set_params(
            self.h, 1 if cfg.mode == "xy" else 0, float(cfg.c_alpha), float(cfg.c_beta), float(cfg.delta),
            float(cfg.eta), float(cfg.tau_bar), float(cfg.gamma0), 1 if cfg.nonmonotone else 0,
            int(cfg.max_backtracks), kind, r1, r2))

    # -- ops -----------------------------------------------------------------
    def reinit(self, source: int, x=None, v=None, lam=None, warm_tau=False, reset_inner=False):
        self._set_stream()
        self._check(self.lib.rapdb_reinit(self.h, source, _ptr(x), _ptr(v), _ptr(lam),
                                          1 if warm_tau else 0, 1 if reset_inner else 0))

    def run(self, args: RunArgs, trace_tensor):
        self._set_stream()
        res = RunResult()
        code = self.lib.rapdb_run(self.h, C.byref(args), _ptr(trace_tensor), C.byref(res))
        state = None
        if code == 3:
            state = {"tau": res.fail_tau, "gamma": res.fail_gamma, "iter": int(res.fail_iter)}
        self._check(code, state=state)
        return res

    def kkt(self, f_star=None):
        self._set_stream()
        out = (C.c_double * 8)()
        self._check(self.lib.rapdb_kkt(self.h, 0 if f_star is None else 1,
                                       0.0 if f_star is None else float(f_star), out))
        return list(out)

    def check_guards(self):
        """(number of workspace buffers whose guard zone was written, report)."""
        buf = C.create_string_buffer(4096)
        n = int(self.lib.rapdb_check_guards(self.h, buf, 4096))
        if n < 0:
            raise DeviceError("guard check failed")
        return n, buf.value.decode(errors="replace")

    def eq_residual(self, x, out):
        self._set_stream()
        self._check(self.lib.rapdb_eq_residual(self.h, _ptr(x), _ptr(out)))

    def kkt_at(self, x, v, lam, f_star=None):
        """[kkt, stationarity, primal_eq, complementarity, infeas, f, mpv,
        subopt, Phi] at an explicit device point (rapdb_kkt_at)."""
        self._set_stream()
        out = (C.c_double * 9)()
        self._check(self.lib.rapdb_kkt_at(self.h, _ptr(x), _ptr(v), _ptr(lam), 0 if f_star is None else 1,
                                          0.0 if f_star is None else float(f_star), out))
        return list(out)

    def egm(self, stepsize: float, K: int, trace_every: int = 0):
        """Extragradient iterations from the current point (egm.py:37-77);
        returns (iterations, diverged, trace rows (iter, |z|) as a host array)."""
        torch = self.torch
        rows = (K // trace_every) if trace_every > 0 else 0
        tr = torch.zeros((max(rows, 1), 2), dtype=torch.float64, device=self.device)
        it = C.c_longlong()
        dv = C.c_int()
        self._set_stream()
        self._check(self.lib.rapdb_egm(self.h, float(stepsize), int(K), int(trace_every),
                                       _ptr(tr) if rows else None, C.byref(it), C.byref(dv)))
        return int(it.value), bool(dv.value), tr[:rows].cpu().numpy()

    def get_iterate(self, which: int):
        torch = self.torch
        d = self.data
        x = torch.empty(d.n, dtype=torch.float64, device=self.device)
        v = torch.empty(max(d.p, 1), dtype=torch.float64, device=self.device)
        lam = torch.empty(max(d.m, 1), dtype=torch.float64, device=self.device)
        self._set_stream()
        self._check(self.lib.rapdb_get_iterate(self.h, which, _ptr(x), _ptr(v), _ptr(lam)))
        return x, v[:d.p], lam[:d.m]

    def probe_sweep(self, x, reps=1):
        torch = self.torch
        d = self.data
        if getattr(d, "factored", False):
            u = torch.empty(max(d.nr, 1), dtype=torch.float64, device=self.device)
        else:
            u = torch.empty((d.m + 1, d.n), dtype=torch.float64, device=self.device)
        g = torch.empty(d.m + 1, dtype=torch.float64, device=self.device)
        ms = C.c_float()
        self._set_stream()
        self._check(self.lib.rapdb_probe_sweep(self.h, _ptr(x), _ptr(u), _ptr(g), int(reps), C.byref(ms)))
        return u, g, float(ms.value)

    def grad_x(self, x, v, lam):
        """(grad_x Phi(x, v, lam), g(x)) on the device (x, v, lam device tensors)."""
        torch = self.torch
        d = self.data
        gx = torch.empty(d.n, dtype=torch.float64, device=self.device)
        g = torch.empty(d.m + 1, dtype=torch.float64, device=self.device)
        self._set_stream()
        self._check(self.lib.rapdb_grad_x(self.h, _ptr(x), _ptr(v), _ptr(lam), _ptr(gx), _ptr(g)))
        return gx, g

    def smoothed_gap(self, source: int, xi: float, tol: float, x_warm=None, x_cand=None, point=None):
        """point = (x, v, lam) device tensors for source 0."""
        out = (C.c_double * 6)()
        x, v, lam = point if point is not None else (None, None, None)
        self._set_stream()
        self._check(self.lib.rapdb_smoothed_gap(self.h, source, _ptr(x), _ptr(v), _ptr(lam), float(xi),
                                                float(tol), _ptr(x_warm), _ptr(x_cand), out))
        return list(out)
