"""Python mirror of the reference's streaming API over the product C ABI.

Same names, argument meaning and error behaviour as the reference's
``tucker::`` streaming interface (proj/include/tucker/streaming.hpp):

    stream_init(x_init, tau)                -> StreamingState   (streaming.hpp:55)
    stream_update(state, y)                                      (streaming.hpp:63)
    process_nonstreaming_mode(state, y, mode, delta) -> (res, y) (streaming.hpp:69-70)
    estimate_relative_error(state)          -> float            (streaming.hpp:79)
    assemble_streaming_state(model_state)   -> StreamingState   (streaming.hpp:85-87)

Every call goes through ``libtsg.so`` (include/tsg.h), which runs the whole
update on the B200. There is no CPU fallback: if the library or a CUDA
device is missing, calls raise.

Errors: ``InvalidArgument`` (a ``ValueError``) mirrors std::invalid_argument,
``CouplingDrift`` mirrors the std::runtime_error on core/ISVD drift,
``DeviceError`` reports CUDA failures.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtsg.so")
MAXD = 8
MEM_HOST, MEM_DEVICE = 0, 1
ASYNC, PROFILE, PROFILE_MODE0 = 1, 2, 4

_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)


class TsgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[tsg {code}] {msg}")
        self.code = code


class InvalidArgument(TsgError, ValueError):
    pass


class CouplingDrift(TsgError):
    pass


class IoError(TsgError, OSError):
    """Checkpoint file errors (tucker::IoError, io.hpp:24-33)."""


class DeviceError(TsgError):
    pass


def _raise(code: int, msg: str):
    if code == 1:
        raise InvalidArgument(code, msg)
    if code == 2:
        raise CouplingDrift(code, msg)
    if code == 4:
        raise DeviceError(code, msg)
    if code == 5:
        raise IoError(code, msg)
    raise TsgError(code, msg)


class TsgConfig(C.Structure):
    _fields_ = [("device", C.c_int32), ("flags", C.c_int32), ("rank_capacity", C.c_int64),
                ("row_capacity", C.c_int64), ("reorthogonalize_every", C.c_int64)]


class TsgDims(C.Structure):
    _fields_ = [
        ("order", C.c_int32), ("n_d", C.c_int64), ("rank", C.c_int64), ("insertions", C.c_int64),
        ("core_dims", C.c_int64 * MAXD), ("slice_dims", C.c_int64 * MAXD),
        ("tau", C.c_double), ("squared_error", C.c_double), ("total_input_sq", C.c_double),
        ("nonstream_discarded_sq", C.c_double),
    ]


class TsgExchange(C.Structure):
    """tsg_exchange (include/tsg.h): one collective request of a sharded update
    (op 0: allgather, op 1: all-reduce sum)."""
    _fields_ = [("pending", C.c_int32), ("op", C.c_int32), ("count", C.c_int64),
                ("send", C.c_void_p), ("recv", C.c_void_p)]


XCHG_ALLGATHER, XCHG_ALLREDUCE_SUM = 0, 1


class TsgAddRowResult(C.Structure):
    """tsg_add_row_result (AddRowResult, isvd.hpp:97-104, without inner_left)."""
    _fields_ = [("r_old", C.c_int64), ("r_new", C.c_int64), ("degenerate", C.c_int32),
                ("added_error_sq", C.c_double)]


class TsgMetrics(C.Structure):
    _fields_ = [
        ("slice_index", C.c_int64), ("ranks", C.c_int64 * MAXD),
        ("slice_norm", C.c_double), ("projected_norm", C.c_double), ("error_estimate", C.c_double),
        ("mode_residuals", C.c_double * MAXD), ("expanded_mask", C.c_int32),
        ("peak_bytes", C.c_int64), ("wall_ms", C.c_double), ("trunc_margin", C.c_double),
        ("jacobi_sweeps", C.c_int32),
    ]


EXPORTED = [
    "tsg_create", "tsg_destroy", "tsg_last_error", "tsg_init", "tsg_update", "tsg_synchronize",
    "tsg_process_mode", "tsg_query", "tsg_export_state", "tsg_import_state",
    "tsg_estimate_relative_error", "tsg_metrics_count", "tsg_metrics_at", "tsg_last_metrics",
    "tsg_kernel_launches", "tsg_cuda_stream", "tsg_slice_buffer", "tsg_sym_eig_desc",
    "tsg_small_svd_truncated", "tsg_mode_subspace", "tsg_ttm", "tsg_profile",
    "tsg_measure_fp64_peaks", "tsg_readback_bytes_per_update", "tsg_debug_project",
    "tsg_add_row", "tsg_shard_setup", "tsg_shard_setup_mode", "tsg_shard_begin", "tsg_shard_continue", "tsg_reconstruct",
    "tsg_error_sums", "tsg_profile_timeline", "tsg_save_checkpoint", "tsg_load_checkpoint",
]

_LIB = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libtsg.so (raises if it was not built: no fallback exists)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing; build it with `make -C {HERE}` "
                          "(or __graft_entry__.build()) — there is no CPU fallback")
    L = C.CDLL(path)
    L.tsg_create.argtypes = [C.POINTER(TsgConfig), C.POINTER(C.c_void_p)]
    L.tsg_save_checkpoint.argtypes = [C.c_void_p, C.c_char_p]
    L.tsg_load_checkpoint.argtypes = [C.c_void_p, C.c_char_p]
    L.tsg_destroy.argtypes = [C.c_void_p]
    L.tsg_last_error.argtypes = [C.c_void_p]
    L.tsg_last_error.restype = C.c_char_p
    L.tsg_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, _i64p, C.c_double, C.c_int32]
    L.tsg_update.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
    L.tsg_synchronize.argtypes = [C.c_void_p]
    L.tsg_process_mode.argtypes = [C.c_void_p, _dp, _i64p, C.c_int32, C.c_double, _dp, C.c_int64,
                                   _i64p, _dp]
    L.tsg_query.argtypes = [C.c_void_p, C.POINTER(TsgDims)]
    L.tsg_export_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
    L.tsg_import_state.argtypes = [C.c_void_p, C.POINTER(TsgDims), _dp, _dp, _dp, _dp, _dp]
    L.tsg_estimate_relative_error.argtypes = [C.c_void_p]
    L.tsg_estimate_relative_error.restype = C.c_double
    L.tsg_metrics_count.argtypes = [C.c_void_p]
    L.tsg_metrics_count.restype = C.c_int64
    L.tsg_metrics_at.argtypes = [C.c_void_p, C.c_int64, C.POINTER(TsgMetrics)]
    L.tsg_last_metrics.argtypes = [C.c_void_p, C.POINTER(TsgMetrics)]
    L.tsg_kernel_launches.argtypes = [C.c_void_p]
    L.tsg_kernel_launches.restype = C.c_int64
    L.tsg_cuda_stream.argtypes = [C.c_void_p]
    L.tsg_cuda_stream.restype = C.c_void_p
    L.tsg_slice_buffer.argtypes = [C.c_void_p, C.c_int32]
    L.tsg_slice_buffer.restype = C.c_void_p
    L.tsg_sym_eig_desc.argtypes = [C.c_int64, _dp, _dp, _dp]
    L.tsg_small_svd_truncated.argtypes = [C.c_int64, C.c_int64, _dp, C.c_double, _dp, _dp, _dp,
                                          _i64p, _dp]
    L.tsg_mode_subspace.argtypes = [_dp, C.c_int32, _i64p, C.c_int32, C.c_double, _dp, _i64p,
                                    _dp, _dp]
    L.tsg_ttm.argtypes = [_dp, C.c_int32, _i64p, C.c_int32, _dp, C.c_int64, C.c_int64, C.c_int32,
                          _dp]
    L.tsg_profile.argtypes = [C.c_void_p, _dp, C.c_int32, C.c_int32]
    L.tsg_measure_fp64_peaks.argtypes = [C.c_int32, _dp, _dp]
    L.tsg_readback_bytes_per_update.argtypes = []
    L.tsg_readback_bytes_per_update.restype = C.c_int64
    L.tsg_shard_setup.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _i64p]
    L.tsg_add_row.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_double,
                              C.POINTER(TsgAddRowResult)]
    L.tsg_shard_setup_mode.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, _i64p]
    L.tsg_shard_begin.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(TsgExchange)]
    L.tsg_shard_continue.argtypes = [C.c_void_p, C.POINTER(TsgExchange)]
    L.tsg_profile_timeline.argtypes = [C.c_void_p, _dp, C.c_int64]
    L.tsg_profile_timeline.restype = C.c_int64
    L.tsg_reconstruct.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int32]
    L.tsg_error_sums.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32, _dp, _dp]
    _LIB = L
    return L


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _flat(t) -> tuple[np.ndarray, list]:
    """numpy tensor indexed t[i0, i1, ...] -> colexicographic buffer + dims."""
    t = np.asarray(t, dtype=np.float64)
    return np.ascontiguousarray(t.transpose().ravel()), list(t.shape)


def _unflat(buf: np.ndarray, dims) -> np.ndarray:
    return np.ascontiguousarray(buf.reshape(list(dims)[::-1]).transpose())


@dataclass
class State:
    """Exported state in the reference's layouts (StreamingState)."""
    order: int
    n_d: int
    rank: int
    insertions: int
    core_dims: tuple
    slice_dims: tuple
    tau: float
    squared_error: float
    total_input_sq: float
    nonstream_discarded_sq: float
    core: np.ndarray = field(repr=False)    # flat colexicographic R_0..R_{d-1}
    factors: list = field(repr=False)       # N_k x R_k, k < d-1
    sigma: np.ndarray = field(repr=False)
    left: np.ndarray = field(repr=False)    # n_d x r (streaming_factor())
    right: np.ndarray = field(repr=False)   # n x r

    def core_tensor(self) -> np.ndarray:
        return _unflat(self.core, self.core_dims)


def metrics_dict(m: TsgMetrics, d: int) -> dict:
    return {
        "slice_index": m.slice_index,
        "ranks": tuple(m.ranks[k] for k in range(d)),
        "slice_norm": m.slice_norm,
        "projected_norm": m.projected_norm,
        "error_estimate": m.error_estimate,
        "mode_residuals": tuple(m.mode_residuals[k] for k in range(d - 1)),
        "expanded_mask": m.expanded_mask,
        "peak_bytes": m.peak_bytes,
        "wall_ms": m.wall_ms,
        "trunc_margin": m.trunc_margin,
        "jacobi_sweeps": m.jacobi_sweeps,
    }


class StreamingState:
    """Owns one device-resident streaming state (a tsg_stream handle)."""

    def __init__(self, device: int = 0, asynchronous: bool = False, rank_capacity: int = 0,
                 row_capacity: int = 0, profile: bool | str = False,
                 reorthogonalize_every: int = 0):
        """profile: False, True (all phases) or "mode0" (the mode-0 kernel only).
        reorthogonalize_every: ISVDOptions (isvd.hpp:62-67), 0 = off."""
        self.L = load_library()
        prof = PROFILE_MODE0 if profile == "mode0" else (PROFILE if profile else 0)
        flags = (ASYNC if asynchronous else 0) | prof
        cfg = TsgConfig(device, flags, rank_capacity, row_capacity, int(reorthogonalize_every))
        h = C.c_void_p()
        code = self.L.tsg_create(C.byref(cfg), C.byref(h))
        if code:
            _raise(code, self.L.tsg_last_error(None).decode())
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.tsg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, code: int):
        if code:
            _raise(code, self.L.tsg_last_error(self.h).decode())

    # -- reference API --
    def init_flat(self, x_flat, dims, tau: float):
        dims = np.asarray(dims, dtype=np.int64)
        ptr, kind = _pointer(x_flat)
        self._check(self.L.tsg_init(self.h, ptr, len(dims), dims.ctypes.data_as(_i64p), float(tau), kind))

    def stream_update(self, y):
        """y: numpy tensor (indexed y[i0, ...]), flat colexicographic numpy
        buffer, or a CUDA torch tensor holding the flat colexicographic slice."""
        if isinstance(y, np.ndarray) and y.ndim > 1:
            y, _ = _flat(y)
        ptr, kind = _pointer(y)
        # the pipelined engine may read a slice again until two further updates
        # have returned (include/tsg.h): keep the last inputs alive here
        live = getattr(self, "_live", None)
        if live is None:
            live = self._live = []
        live.append(y)
        del live[:-4]
        self._check(self.L.tsg_update(self.h, ptr, kind))

    def add_row(self, b, abs_tol: float, slice_norm_sq: float = 0.0) -> dict:
        """add_row (isvd.hpp:110-111) on the device ISVD plus the core rotation of
        stream_update (streaming.cpp:199-222): b = vec(projected slice), n doubles
        (numpy or CUDA torch). Returns r_old, r_new, degenerate, added_error_sq."""
        if isinstance(b, np.ndarray):
            b = np.ascontiguousarray(b.ravel(order="F"), dtype=np.float64)
        ptr, kind = _pointer(b)
        res = TsgAddRowResult()
        self._check(self.L.tsg_add_row(self.h, ptr, kind, float(abs_tol), float(slice_norm_sq),
                                       C.byref(res)))
        return {"r_old": int(res.r_old), "r_new": int(res.r_new),
                "degenerate": bool(res.degenerate), "added_error_sq": float(res.added_error_sq)}

    def update_device_ptr(self, ptr: int):
        self._check(self.L.tsg_update(self.h, C.c_void_p(ptr), MEM_DEVICE))

    def save_checkpoint(self, path: str):
        """save_checkpoint (io.cpp:303-324): TUCKCKPT v1, written atomically."""
        self._check(self.L.tsg_save_checkpoint(self.h, os.fsencode(path)))

    def synchronize(self):
        self._check(self.L.tsg_synchronize(self.h))
        if getattr(self, "_live", None):
            self._live.clear()

    def process_nonstreaming_mode(self, y: np.ndarray, mode: int, delta: float):
        x, dims = _flat(y)
        q = self.query()
        cap = int(np.prod(dims)) // max(dims[mode], 1) * q["slice_dims"][mode] + 16
        out = np.zeros(cap)
        d = np.array(dims, dtype=np.int64)
        od = np.zeros(MAXD, dtype=np.int64)
        res = C.c_double()
        self._check(self.L.tsg_process_mode(self.h, _p(x), d.ctypes.data_as(_i64p), mode,
                                            float(delta), _p(out), cap,
                                            od.ctypes.data_as(_i64p), C.byref(res)))
        odims = [int(v) for v in od[: len(dims)]]
        return res.value, _unflat(out[: int(np.prod(odims))], odims)

    def query(self) -> dict:
        dm = TsgDims()
        self._check(self.L.tsg_query(self.h, C.byref(dm)))
        d = dm.order
        return {
            "order": d, "n_d": dm.n_d, "rank": dm.rank, "insertions": dm.insertions,
            "core_dims": tuple(dm.core_dims[k] for k in range(d)),
            "slice_dims": tuple(dm.slice_dims[k] for k in range(d - 1)),
            "tau": dm.tau, "squared_error": dm.squared_error,
            "total_input_sq": dm.total_input_sq,
            "nonstream_discarded_sq": dm.nonstream_discarded_sq,
        }

    def export(self) -> State:
        q = self.query()
        d, cd, sd, r = q["order"], q["core_dims"], q["slice_dims"], q["rank"]
        n = int(np.prod(cd[:-1]))
        core = np.zeros(max(int(np.prod(cd)), 1))
        fsz = [sd[k] * cd[k] for k in range(d - 1)]
        fac = np.zeros(max(sum(fsz), 1))
        sig = np.zeros(max(r, 1))
        left = np.zeros(max(q["n_d"] * r, 1))
        right = np.zeros(max(n * r, 1))
        self._check(self.L.tsg_export_state(self.h, _p(core), _p(fac), _p(sig), _p(left), _p(right)))
        factors, off = [], 0
        for k in range(d - 1):
            factors.append(fac[off: off + fsz[k]].reshape(sd[k], cd[k], order="F").copy())
            off += fsz[k]
        return State(order=d, n_d=q["n_d"], rank=r, insertions=q["insertions"], core_dims=cd,
                     slice_dims=sd, tau=q["tau"], squared_error=q["squared_error"],
                     total_input_sq=q["total_input_sq"],
                     nonstream_discarded_sq=q["nonstream_discarded_sq"],
                     core=core[: int(np.prod(cd))].copy(), factors=factors, sigma=sig[:r].copy(),
                     left=left[: q["n_d"] * r].reshape(q["n_d"], r, order="F").copy(),
                     right=right[: n * r].reshape(n, r, order="F").copy())

    def metrics(self) -> list:
        d = self.query()["order"]
        out = []
        for i in range(self.L.tsg_metrics_count(self.h)):
            m = TsgMetrics()
            self._check(self.L.tsg_metrics_at(self.h, i, C.byref(m)))
            out.append(metrics_dict(m, d))
        return out

    def last_metrics(self) -> dict:
        m = TsgMetrics()
        self._check(self.L.tsg_last_metrics(self.h, C.byref(m)))
        return metrics_dict(m, self.query()["order"])

    def estimate_relative_error(self) -> float:
        return float(self.L.tsg_estimate_relative_error(self.h))

    def reconstruct(self, t0: int = 0, count: int | None = None, out=None):
        """Slices [t0, t0+count) of full_model() (reconstruct, sthosvd.cpp:135-146),
        flat colexicographic. `out` may be a CUDA torch tensor (filled on the
        device); otherwise a numpy array is returned."""
        q = self.query()
        if count is None:
            count = q["n_d"] - t0
        n = int(np.prod(q["slice_dims"])) * count
        if out is None:
            out = np.zeros(max(n, 1))
            ptr, kind = _pointer(out)
            self._check(self.L.tsg_reconstruct(self.h, t0, count, ptr, kind))
            return out[:n]
        ptr, kind = _pointer(out)
        self._check(self.L.tsg_reconstruct(self.h, t0, count, ptr, kind))
        return out

    def error_sums(self, x, t0: int, count: int) -> tuple[float, float]:
        """(||x - X||^2, ||x||^2) over slices [t0, t0+count) for the caller's
        flat slices x (numpy or CUDA torch)."""
        ptr, kind = _pointer(x)
        a, b = C.c_double(), C.c_double()
        self._check(self.L.tsg_error_sums(self.h, ptr, t0, count, kind, C.byref(a), C.byref(b)))
        return a.value, b.value

    def profile(self, reset: bool = False) -> dict:
        out = np.zeros(6)
        self._check(self.L.tsg_profile(self.h, _p(out), 6, int(reset)))
        n = max(out[0], 1.0)
        return {"updates": int(out[0]), "mode0_ms": out[1] / n, "rest_proj_ms": out[2] / n,
                "isvd_ms": out[3] / n, "host_gap_ms": out[4] / n}

    def timeline(self, cap: int = 4096) -> np.ndarray:
        """(slices x 5) ms: mode-0 start, mode-0 end, decision, insertion
        start, insertion end of the profiled slices since the last reset."""
        out = np.zeros(5 * cap)
        n = int(self.L.tsg_profile_timeline(self.h, _p(out), cap))
        if n < 0:
            self._check(4)
        return out[: 5 * n].reshape(n, 5)

    def kernel_launches(self) -> int:
        return int(self.L.tsg_kernel_launches(self.h))

    def cuda_stream(self) -> int:
        return int(self.L.tsg_cuda_stream(self.h) or 0)

    def slice_buffer(self, which: int = 0) -> int:
        return int(self.L.tsg_slice_buffer(self.h, which) or 0)


def _pointer(x):
    """(pointer, mem_kind) for a numpy array or a CUDA torch tensor."""
    if isinstance(x, np.ndarray):
        if x.dtype != np.float64 or not x.flags.c_contiguous:
            raise InvalidArgument(1, "host buffers must be C-contiguous float64")
        return x.ctypes.data_as(C.c_void_p), MEM_HOST
    mod = type(x).__module__
    if mod.startswith("torch"):
        import torch
        if x.dtype != torch.float64 or not x.is_contiguous():
            raise InvalidArgument(1, "tensors must be contiguous float64")
        if x.is_cuda:
            return C.c_void_p(x.data_ptr()), MEM_DEVICE
        return C.c_void_p(x.data_ptr()), MEM_HOST
    raise InvalidArgument(1, f"unsupported buffer type {type(x)!r}")


# ---------------------------------------------------------------- free API
def stream_init(x_init, tau: float, dims=None, device: int = 0, asynchronous: bool = False,
                **kw) -> StreamingState:
    """Batch ST-HOSVD of the initial block + ISVD setup (streaming.cpp:83-124).
    x_init: numpy tensor indexed x[i0, ..., i_{d-1}] (streaming mode last), or
    a flat colexicographic buffer (numpy / CUDA torch) with explicit dims."""
    st = StreamingState(device=device, asynchronous=asynchronous, **kw)
    if dims is None:
        flat, dims = _flat(x_init)
    else:
        flat = x_init
    st.init_flat(flat, dims, tau)
    return st


def stream_update(state: StreamingState, y) -> None:
    state.stream_update(y)


def process_nonstreaming_mode(state: StreamingState, y, mode: int, delta: float):
    return state.process_nonstreaming_mode(y, mode, delta)


def relative_error(x, state: StreamingState) -> float:
    """relative_error(x, state.full_model()) (sthosvd.cpp:148-160) for the
    whole stream x (flat colexicographic, n_d slices; numpy or CUDA torch)."""
    q = state.query()
    per = int(np.prod(q["slice_dims"]))
    if len(x) != per * q["n_d"]:
        raise InvalidArgument(1, "relative_error: shape mismatch")
    num, den = state.error_sums(x, 0, q["n_d"])
    if den == 0.0:
        if num == 0.0:
            return 0.0
        raise InvalidArgument(1, "relative_error: zero-norm input with nonzero reconstruction")
    return float(np.sqrt(num) / np.sqrt(den))


def estimate_relative_error(state: StreamingState) -> float:
    return state.estimate_relative_error()


def assemble_streaming_state(st: State, device: int = 0, asynchronous: bool = False,
                             reorthogonalize_every: int = 0) -> StreamingState:
    """assemble_streaming_state (streaming.cpp:242-263) from exported pieces."""
    out = StreamingState(device=device, asynchronous=asynchronous,
                         reorthogonalize_every=reorthogonalize_every)
    dm = TsgDims()
    dm.order, dm.n_d, dm.rank, dm.insertions = st.order, st.n_d, st.rank, st.insertions
    for k, v in enumerate(st.core_dims):
        dm.core_dims[k] = v
    for k, v in enumerate(st.slice_dims):
        dm.slice_dims[k] = v
    dm.tau, dm.squared_error = st.tau, st.squared_error
    dm.total_input_sq, dm.nonstream_discarded_sq = st.total_input_sq, st.nonstream_discarded_sq
    fac = np.concatenate([np.asfortranarray(f).ravel(order="F") for f in st.factors])
    core = np.ascontiguousarray(st.core, dtype=np.float64)
    sig = np.ascontiguousarray(st.sigma, dtype=np.float64)
    left = np.asfortranarray(st.left).ravel(order="F")
    right = np.asfortranarray(st.right).ravel(order="F")
    out._check(out.L.tsg_import_state(out.h, C.byref(dm), _p(core), _p(fac), _p(sig), _p(left),
                                      _p(right)))
    return out


def save_checkpoint(path: str, state: StreamingState) -> None:
    state.save_checkpoint(path)


def load_checkpoint(path: str, device: int = 0, asynchronous: bool = False,
                    reorthogonalize_every: int = 0) -> StreamingState:
    """from_checkpoint(load_checkpoint(path)) (io.cpp:326-423) on the device."""
    st = StreamingState(device=device, asynchronous=asynchronous,
                        reorthogonalize_every=reorthogonalize_every)
    st._check(st.L.tsg_load_checkpoint(st.h, os.fsencode(path)))
    return st


def readback_bytes_per_update() -> int:
    return int(load_library().tsg_readback_bytes_per_update())


def measure_fp64_peaks(device: int = 0) -> tuple[float, float]:
    L = load_library()
    a, b = C.c_double(), C.c_double()
    code = L.tsg_measure_fp64_peaks(device, C.byref(a), C.byref(b))
    if code:
        _raise(code, L.tsg_last_error(None).decode())
    return a.value, b.value


# ------------------------------------------------------------ building blocks
def sym_eig_desc(g: np.ndarray):
    L = load_library()
    n = g.shape[0]
    gf = np.asfortranarray(g, dtype=np.float64).ravel(order="F")
    ev, vec = np.zeros(max(n, 1)), np.zeros(max(n * n, 1))
    code = L.tsg_sym_eig_desc(n, _p(gf), _p(ev), _p(vec))
    if code:
        _raise(code, L.tsg_last_error(None).decode())
    return ev[:n], vec[: n * n].reshape(n, n, order="F")


def small_svd_truncated(a: np.ndarray, thr: float):
    L = load_library()
    m, n = a.shape
    af = np.asfortranarray(a, dtype=np.float64).ravel(order="F")
    left, sig, right = np.zeros(max(m * n, 1)), np.zeros(max(n, 1)), np.zeros(max(n * n, 1))
    rk, disc = C.c_int64(), C.c_double()
    code = L.tsg_small_svd_truncated(m, n, _p(af), float(thr), _p(left), _p(sig), _p(right),
                                     C.byref(rk), C.byref(disc))
    if code:
        _raise(code, L.tsg_last_error(None).decode())
    r = rk.value
    return (left[: m * r].reshape(m, r, order="F"), sig[:r].copy(),
            right[: n * r].reshape(n, r, order="F"), disc.value)


def mode_subspace(t: np.ndarray, mode: int, delta: float):
    L = load_library()
    x, dims = _flat(t)
    nk = dims[mode]
    basis, ev = np.zeros(nk * nk), np.zeros(nk)
    rk, disc = C.c_int64(), C.c_double()
    d = np.array(dims, dtype=np.int64)
    code = L.tsg_mode_subspace(_p(x), len(dims), d.ctypes.data_as(_i64p), mode, float(delta),
                               _p(basis), C.byref(rk), _p(ev), C.byref(disc))
    if code:
        _raise(code, L.tsg_last_error(None).decode())
    r = rk.value
    return basis[: nk * r].reshape(nk, r, order="F"), ev, disc.value


def ttm(t: np.ndarray, mode: int, a: np.ndarray, transpose_a: bool = False) -> np.ndarray:
    L = load_library()
    x, dims = _flat(t)
    af = np.asfortranarray(a, dtype=np.float64).ravel(order="F")
    od = list(dims)
    od[mode] = a.shape[1] if transpose_a else a.shape[0]
    out = np.zeros(max(int(np.prod(od)), 1))
    d = np.array(dims, dtype=np.int64)
    code = L.tsg_ttm(_p(x), len(dims), d.ctypes.data_as(_i64p), mode, _p(af), a.shape[0],
                     a.shape[1], int(transpose_a), _p(out))
    if code:
        _raise(code, L.tsg_last_error(None).decode())
    return _unflat(out[: int(np.prod(od))], od)
