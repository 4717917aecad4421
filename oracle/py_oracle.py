"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the two CPU checkers.

* ``load_oracle()``    -> this repo's C restatement (oracle/liboracle.so, prefix tko_)
* ``load_reference()`` -> the reference's own sources compiled in place
                          (oracle/_ref/libtucker_ref.so, prefix tkr_)

Both expose oracle_abi.h. Only tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline leg import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MAXD = 8
_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)


class OrcDims(C.Structure):
    _fields_ = [
        ("order", C.c_int32),
        ("n_d", C.c_int64),
        ("rank", C.c_int64),
        ("insertions", C.c_int64),
        ("core_dims", C.c_int64 * MAXD),
        ("slice_dims", C.c_int64 * MAXD),
        ("tau", C.c_double),
        ("squared_error", C.c_double),
        ("total_input_sq", C.c_double),
        ("nonstream_discarded_sq", C.c_double),
    ]


class OrcMetrics(C.Structure):
    _fields_ = [
        ("slice_index", C.c_int64),
        ("ranks", C.c_int64 * MAXD),
        ("slice_norm", C.c_double),
        ("projected_norm", C.c_double),
        ("error_estimate", C.c_double),
        ("mode_residuals", C.c_double * MAXD),
        ("expanded_mask", C.c_int32),
    ]


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(CheckerError, ValueError):
    pass


class CouplingDrift(CheckerError):
    pass


def _raise(code: int, msg: str):
    if code == 1:
        raise InvalidArgument(code, msg)
    if code == 2:
        raise CouplingDrift(code, msg)
    raise CheckerError(code, msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


@dataclass
class State:
    """Exported streaming state in the reference's layouts."""
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
    core: np.ndarray = field(repr=False)       # colexicographic, flat
    factors: list = field(repr=False)          # N_k x R_k (k < d-1)
    sigma: np.ndarray = field(repr=False)
    left: np.ndarray = field(repr=False)       # n_d x r
    right: np.ndarray = field(repr=False)      # n x r

    def core_tensor(self) -> np.ndarray:
        return self.core.reshape(self.core_dims[::-1]).transpose()


def metrics_dict(m: OrcMetrics, d: int) -> dict:
    return {
        "slice_index": m.slice_index,
        "ranks": tuple(m.ranks[k] for k in range(d)),
        "slice_norm": m.slice_norm,
        "projected_norm": m.projected_norm,
        "error_estimate": m.error_estimate,
        "mode_residuals": tuple(m.mode_residuals[k] for k in range(d - 1)),
        "expanded_mask": m.expanded_mask,
    }


class Checker:
    """Drives one CPU checker library through oracle_abi.h."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle all ref`)")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        L = self.lib
        f = lambda n: getattr(L, prefix + n)
        self._init = f("stream_init"); self._init.argtypes = [_dp, C.c_int32, _i64p, C.c_double, C.POINTER(C.c_void_p)]
        self._upd = f("stream_update"); self._upd.argtypes = [C.c_void_p, _dp]
        self._pm = f("process_mode"); self._pm.argtypes = [C.c_void_p, _dp, _i64p, C.c_int32, C.c_double, _dp, C.c_int64, _i64p, _dp]
        self._q = f("query"); self._q.argtypes = [C.c_void_p, C.POINTER(OrcDims)]
        self._ex = f("export_state"); self._ex.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
        self._mc = f("metrics_count"); self._mc.argtypes = [C.c_void_p]; self._mc.restype = C.c_int64
        self._ma = f("metrics_at"); self._ma.argtypes = [C.c_void_p, C.c_int64, C.POINTER(OrcMetrics)]
        self._as = f("assemble"); self._as.argtypes = [C.POINTER(OrcDims), _dp, _dp, _dp, _dp, _dp, C.POINTER(C.c_void_p)]
        self._de = f("destroy"); self._de.argtypes = [C.c_void_p]
        self._sro = f("set_reorthogonalize_every"); self._sro.argtypes = [C.c_void_p, C.c_int64]
        self._le = f("last_error"); self._le.restype = C.c_char_p
        self._eig = f("sym_eig_desc"); self._eig.argtypes = [C.c_int64, _dp, _dp, _dp]
        self._tr = f("truncation_rank"); self._tr.argtypes = [C.c_int64, _dp, C.c_double]; self._tr.restype = C.c_int64
        self._ssvd = f("small_svd_truncated"); self._ssvd.argtypes = [C.c_int64, C.c_int64, _dp, C.c_double, _dp, _dp, _dp, _i64p, _dp]
        self._ms = f("mode_subspace"); self._ms.argtypes = [_dp, C.c_int32, _i64p, C.c_int32, C.c_double, _dp, _i64p, _dp, _dp]
        self._ttm = f("ttm"); self._ttm.argtypes = [_dp, C.c_int32, _i64p, C.c_int32, _dp, C.c_int64, C.c_int64, C.c_int32, _dp]
        self._ss = f("sum_of_squares"); self._ss.argtypes = [_dp, C.c_int64]; self._ss.restype = C.c_double

    def _check(self, code: int):
        if code:
            _raise(code, self._le().decode())

    # ---- streaming API (streaming.hpp) ----
    def stream_init(self, x: np.ndarray, tau: float) -> "Handle":
        """x: a d-way tensor given in colexicographic order via its dims."""
        x, dims = _flat(x)
        h = C.c_void_p()
        d = np.array(dims, dtype=np.int64)
        self._check(self._init(_p(x), len(dims), d.ctypes.data_as(_i64p), float(tau), C.byref(h)))
        return Handle(self, h)

    def assemble(self, st: State) -> "Handle":
        dm = _dims_struct(st)
        h = C.c_void_p()
        fac = np.concatenate([np.asfortranarray(f).ravel(order="F") for f in st.factors]) if st.factors else np.zeros(1)
        core = np.ascontiguousarray(st.core, dtype=np.float64)
        sig = np.ascontiguousarray(st.sigma, dtype=np.float64)
        left = np.asfortranarray(st.left).ravel(order="F")
        right = np.asfortranarray(st.right).ravel(order="F")
        self._check(self._as(C.byref(dm), _p(core), _p(fac), _p(sig), _p(left), _p(right), C.byref(h)))
        return Handle(self, h)

    # ---- building blocks ----
    def sym_eig_desc(self, g: np.ndarray):
        n = g.shape[0]
        gf = np.asfortranarray(g, dtype=np.float64).ravel(order="F")
        ev = np.zeros(n); vec = np.zeros(n * n)
        self._check(self._eig(n, _p(gf), _p(ev), _p(vec)))
        return ev, vec.reshape(n, n, order="F")

    def truncation_rank(self, ev: np.ndarray, delta: float) -> int:
        ev = np.ascontiguousarray(ev, dtype=np.float64)
        r = self._tr(len(ev), _p(ev), float(delta))
        if r < 0:
            _raise(1, self._le().decode())
        return int(r)

    def small_svd_truncated(self, a: np.ndarray, thr: float):
        m, n = a.shape
        af = np.asfortranarray(a, dtype=np.float64).ravel(order="F")
        left = np.zeros(max(m * n, 1)); sig = np.zeros(max(n, 1)); right = np.zeros(max(n * n, 1))
        rk = C.c_int64(); disc = C.c_double()
        self._check(self._ssvd(m, n, _p(af), float(thr), _p(left), _p(sig), _p(right), C.byref(rk), C.byref(disc)))
        r = rk.value
        return (left[: m * r].reshape(m, r, order="F"), sig[:r].copy(),
                right[: n * r].reshape(n, r, order="F"), disc.value)

    def mode_subspace(self, t: np.ndarray, mode: int, delta: float):
        x, dims = _flat(t)
        nk = dims[mode]
        basis = np.zeros(nk * nk); ev = np.zeros(nk)
        rk = C.c_int64(); disc = C.c_double()
        d = np.array(dims, dtype=np.int64)
        self._check(self._ms(_p(x), len(dims), d.ctypes.data_as(_i64p), mode, float(delta), _p(basis), C.byref(rk), _p(ev), C.byref(disc)))
        r = rk.value
        return basis[: nk * r].reshape(nk, r, order="F"), ev, disc.value

    def ttm(self, t: np.ndarray, mode: int, a: np.ndarray, transpose_a: bool = False) -> np.ndarray:
        x, dims = _flat(t)
        af = np.asfortranarray(a, dtype=np.float64).ravel(order="F")
        od = list(dims)
        od[mode] = a.shape[1] if transpose_a else a.shape[0]
        out = np.zeros(int(np.prod(od)))
        d = np.array(dims, dtype=np.int64)
        self._check(self._ttm(_p(x), len(dims), d.ctypes.data_as(_i64p), mode, _p(af), a.shape[0], a.shape[1], int(transpose_a), _p(out)))
        return _unflat(out, od)

    def load_checkpoint(self, path: str) -> "Handle":
        """from_checkpoint(load_checkpoint(path)) (reference library only)."""
        f = self.lib.tkr_load_checkpoint
        f.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        h = C.c_void_p()
        self._check(f(path.encode(), C.byref(h)))
        return Handle(self, h)

    def sum_of_squares(self, x: np.ndarray) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64).ravel()
        return self._ss(_p(x), x.size)


class Handle:
    """One StreamingState owned by a checker library."""

    def __init__(self, checker: Checker, h: C.c_void_p):
        self.c = checker
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.c._de(self.h)
                self.h = None
        except Exception:
            pass

    def stream_update(self, y: np.ndarray):
        y, _ = _flat(y)
        self.c._check(self.c._upd(self.h, _p(y)))

    def save_checkpoint(self, path: str):
        """save_checkpoint(path, state) (reference library only)."""
        f = self.c.lib.tkr_save_checkpoint
        f.argtypes = [C.c_void_p, C.c_char_p]
        self.c._check(f(self.h, path.encode()))

    def set_reorthogonalize_every(self, k: int):
        """ISVDOptions::reorthogonalize_every of this state (isvd.hpp:62-67)."""
        self.c._check(self.c._sro(self.h, int(k)))

    def update_flat(self, y: np.ndarray):
        y = np.ascontiguousarray(y, dtype=np.float64)
        self.c._check(self.c._upd(self.h, _p(y)))

    def process_nonstreaming_mode(self, y: np.ndarray, mode: int, delta: float):
        x, dims = _flat(y)
        st = self.query()
        cap = int(np.prod(dims)) * 2 + int(np.prod(dims)) // max(dims[mode], 1) * (st["slice_dims"][mode] + 1)
        out = np.zeros(cap)
        od = np.zeros(MAXD, dtype=np.int64)
        res = C.c_double()
        d = np.array(dims, dtype=np.int64)
        self.c._check(self.c._pm(self.h, _p(x), d.ctypes.data_as(_i64p), mode, float(delta), _p(out), cap, od.ctypes.data_as(_i64p), C.byref(res)))
        odims = [int(v) for v in od[: len(dims)]]
        return res.value, _unflat(out[: int(np.prod(odims))], odims)

    def query(self) -> dict:
        dm = OrcDims()
        self.c._check(self.c._q(self.h, C.byref(dm)))
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
        d = q["order"]
        cd, sd = q["core_dims"], q["slice_dims"]
        r = q["rank"]
        n = int(np.prod(cd[:-1]))
        core = np.zeros(max(int(np.prod(cd)), 1))
        fsz = [sd[k] * cd[k] for k in range(d - 1)]
        fac = np.zeros(max(sum(fsz), 1))
        sig = np.zeros(max(r, 1)); left = np.zeros(max(q["n_d"] * r, 1)); right = np.zeros(max(n * r, 1))
        self.c._check(self.c._ex(self.h, _p(core), _p(fac), _p(sig), _p(left), _p(right)))
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
        for i in range(self.c._mc(self.h)):
            m = OrcMetrics()
            self.c._check(self.c._ma(self.h, i, C.byref(m)))
            out.append(metrics_dict(m, d))
        return out

    def estimate_relative_error(self) -> float:
        q = self.query()
        if q["total_input_sq"] <= 0:
            return 0.0
        return float(np.sqrt(max(q["squared_error"] + q["nonstream_discarded_sq"], 0.0) / q["total_input_sq"]))


def _flat(t: np.ndarray):
    """numpy array (indexed t[i0, i1, ...]) -> colexicographic flat buffer + dims."""
    t = np.asarray(t, dtype=np.float64)
    dims = list(t.shape)
    return np.ascontiguousarray(t.transpose().ravel()), dims


def _unflat(buf: np.ndarray, dims) -> np.ndarray:
    return np.ascontiguousarray(buf.reshape(list(dims)[::-1]).transpose())


def _dims_struct(st: State) -> OrcDims:
    dm = OrcDims()
    dm.order = st.order
    dm.n_d = st.n_d
    dm.rank = st.rank
    dm.insertions = st.insertions
    for k, v in enumerate(st.core_dims):
        dm.core_dims[k] = v
    for k, v in enumerate(st.slice_dims):
        dm.slice_dims[k] = v
    dm.tau = st.tau
    dm.squared_error = st.squared_error
    dm.total_input_sq = st.total_input_sq
    dm.nonstream_discarded_sq = st.nonstream_discarded_sq
    return dm


def load_oracle() -> Checker:
    return Checker(os.path.join(HERE, "liboracle.so"), "tko_")


def load_reference() -> Checker:
    return Checker(os.path.join(HERE, "_ref", "libtucker_ref.so"), "tkr_")


def reference_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libtucker_ref.so"))
