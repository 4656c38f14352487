"""ctypes binding of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product path
(paper_2410_03969_b200) never imports this module.

The oracle restates the reference accelerated RPCholesky path
(/root/reference/proj/include/rpchol/{rng,oracle,rpcholesky}.hpp); see
oracle/rpc_oracle.c for the per-function file:line citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import weakref
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

KERNELS = {"gaussian": 0, "l1laplace": 1, "laplace": 1, "matern32": 2, "matern52": 3}
DIST = {"direct": 0, "gram": 1}
MODES = {"fixed_rounds": 0, "until_rank": 1}
_ERRS = {1: ValueError, 2: IndexError, 3: RuntimeError, 4: MemoryError}


class _Oracle(C.Structure):
    _fields_ = [
        ("is_dense", C.c_int),
        ("n", C.c_int64),
        ("x", C.c_void_p),
        ("d", C.c_int64),
        ("kind", C.c_int),
        ("sigma", C.c_double),
        ("dist_mode", C.c_int),
        ("sq_norms", C.c_void_p),
        ("a", C.c_void_p),
        ("n_threads", C.c_int),
    ]


class _Cfg(C.Structure):
    _fields_ = [
        ("block_size", C.c_int64),
        ("mode", C.c_int),
        ("rounds", C.c_int64),
        ("target_rank", C.c_int64),
        ("seed", C.c_uint64),
        ("stop_tol", C.c_double),
    ]


class _Res(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("rank", C.c_int64),
        ("factor", C.POINTER(C.c_double)),
        ("pivots", C.POINTER(C.c_int64)),
        ("chol", C.POINTER(C.c_double)),
        ("residual_diag", C.POINTER(C.c_double)),
        ("n_rounds", C.c_int64),
        ("block_size", C.c_int64),
        ("proposed", C.POINTER(C.c_int64)),
        ("accepted_count", C.POINTER(C.c_int64)),
        ("rank_exhausted", C.c_int),
        ("surplus", C.c_int64),
        ("captured_sq", C.c_double),
    ]


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", _HERE, "liboracle.so"], check=True,
                           stdout=subprocess.DEVNULL)
        L = C.CDLL(path)
        L.rpo_splitmix64_draw.restype = C.c_uint64
        L.rpo_splitmix64_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.rpo_u01.restype = C.c_double
        L.rpo_u01.argtypes = [C.c_uint64]
        L.rpo_cumulative_sums.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.rpo_sample_discrete.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.POINTER(C.c_int64)]
        L.rpo_oracle_kernel.argtypes = [C.POINTER(_Oracle), C.c_void_p, C.c_int64, C.c_int64,
                                        C.c_int, C.c_double, C.c_int, C.c_int]
        L.rpo_oracle_dense.argtypes = [C.POINTER(_Oracle), C.c_void_p, C.c_int64]
        L.rpo_oracle_free.argtypes = [C.POINTER(_Oracle)]
        L.rpo_submatrix.argtypes = [C.POINTER(_Oracle), C.c_void_p, C.c_int64, C.c_void_p,
                                    C.c_int64, C.c_void_p]
        L.rpo_rejection_sweep.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64,
                                          C.c_uint64, C.c_void_p, C.c_void_p,
                                          C.POINTER(C.c_int64), C.c_void_p]
        L.rpo_accelerated_rpcholesky_bounded.argtypes = [C.POINTER(_Oracle), C.POINTER(_Cfg),
                                                         C.c_int64, C.POINTER(_Res)]
        L.rpo_accelerated_rpcholesky_lowmem.argtypes = [C.POINTER(_Oracle), C.POINTER(_Cfg),
                                                        C.POINTER(_Res)]
        L.rpo_block_rpcholesky.argtypes = [C.POINTER(_Oracle), C.POINTER(_Cfg), C.POINTER(_Res)]
        L.rpo_simple_rpcholesky.argtypes = [C.POINTER(_Oracle), C.c_int64, C.c_uint64,
                                            C.POINTER(_Res)]
        L.rpo_result_free.argtypes = [C.POINTER(_Res)]
        L.rpo_relative_trace_error.restype = C.c_double
        L.rpo_relative_trace_error.argtypes = [C.POINTER(_Oracle), C.c_void_p, C.c_int64,
                                               C.c_int64]
        L.rpo_last_error.restype = C.c_char_p
        L.rpo_free.argtypes = [C.c_void_p]
        L.rpo_margins_reset.argtypes = [C.c_int]
        L.rpo_margins_get.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        _LIB = L
    return _LIB


def _check(rc: int) -> None:
    if rc:
        raise _ERRS.get(rc, RuntimeError)(lib().rpo_last_error().decode())


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


# ---- rng.hpp -------------------------------------------------------------
def splitmix64_draw(seed: int, n: int) -> int:
    return int(lib().rpo_splitmix64_draw(seed, n))


def u01(z: int) -> float:
    return float(lib().rpo_u01(z))


def cumulative_sums(w: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = np.empty_like(w)
    lib().rpo_cumulative_sums(_p(w), w.size, _p(out))
    return out


def sample_discrete(cumsum: np.ndarray, r01: float) -> int:
    cumsum = np.ascontiguousarray(cumsum, dtype=np.float64)
    idx = C.c_int64()
    _check(lib().rpo_sample_discrete(_p(cumsum), cumsum.size, r01, C.byref(idx)))
    return idx.value


# ---- oracle.hpp ------------------------------------------------------------
class Oracle:
    """KernelOracle (X: N x d, any layout) or DenseOracle (A: N x N)."""

    def __init__(self, *, x=None, kernel="gaussian", sigma=1.0, dist=None, dense=None,
                 n_threads=1):
        self._o = _Oracle()
        L = lib()
        if dense is not None:
            self._a = np.asfortranarray(dense, dtype=np.float64)
            _check(L.rpo_oracle_dense(C.byref(self._o), _p(self._a), self._a.shape[0]))
        else:
            self._x = np.asfortranarray(x, dtype=np.float64)
            kind = KERNELS[kernel]
            if dist is None:
                dist = "direct" if kind == 1 else "gram"   # oracle.hpp:39-42
            _check(L.rpo_oracle_kernel(C.byref(self._o), _p(self._x), self._x.shape[0],
                                       self._x.shape[1], kind, float(sigma), DIST[dist],
                                       int(n_threads)))

    @property
    def n(self) -> int:
        return self._o.n

    def submatrix(self, rows, cols) -> np.ndarray:
        r = np.ascontiguousarray(rows, dtype=np.int64)
        c = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.zeros((r.size, c.size), dtype=np.float64, order="F")
        _check(lib().rpo_submatrix(C.byref(self._o), _p(r), r.size, _p(c), c.size, _p(out)))
        return out

    def columns(self, cols) -> np.ndarray:
        return self.submatrix(np.arange(self.n), cols)

    def __del__(self):
        try:
            lib().rpo_oracle_free(C.byref(self._o))
        except Exception:
            pass


# ---- rpcholesky.hpp --------------------------------------------------------
def rejection_sweep(h: np.ndarray, proposals, seed: int, draw0: int):
    """Returns (accepted ids, positions, chol m x m)."""
    h = np.array(h, dtype=np.float64, order="F", copy=True)
    b = h.shape[0]
    prop = np.ascontiguousarray(proposals, dtype=np.int64)
    acc = np.zeros(b, np.int64)
    pos = np.zeros(b, np.int64)
    chol = np.zeros(b * b, np.float64)
    m = C.c_int64()
    _check(lib().rpo_rejection_sweep(_p(h), b, _p(prop), seed, draw0, _p(acc), _p(pos),
                                     C.byref(m), _p(chol)))
    k = m.value
    return acc[:k].copy(), pos[:k].copy(), chol[: k * k].reshape(k, k, order="F").copy()


@dataclass
class Result:
    factor: np.ndarray          # N x k (Fortran order)
    pivots: np.ndarray          # k int64
    chol: np.ndarray            # k x k lower
    residual_diag: np.ndarray   # N
    proposed: list              # per round, b int64
    accepted: list              # per round, accepted ids (sweep order)
    rank_exhausted: bool
    surplus: int
    captured_sq: float

    @property
    def rank(self) -> int:
        return len(self.pivots)


def _adopt_buffer(ptr, count: int) -> np.ndarray:
    """A numpy view of a C-allocated double buffer that frees it when the last view goes
    (used to keep a multi-GB oracle factor without a second copy)."""
    addr = C.cast(ptr, C.c_void_p).value
    holder = (C.c_double * count).from_address(addr)
    weakref.finalize(holder, lib().rpo_free, addr)
    return np.ctypeslib.as_array(holder)


def _unpack(res, copy_factor: bool = True) -> Result:
    try:
        n, k, b, nr = res.n, res.rank, res.block_size, res.n_rounds
        if not res.factor:
            factor = None  # LowMemResult
        elif k and not copy_factor:
            factor = _adopt_buffer(res.factor, k * n).reshape(n, k, order="F")
            res.factor = C.POINTER(C.c_double)()  # ownership moved to the view
        else:
            factor = np.ctypeslib.as_array(res.factor, shape=(k * n,)).reshape(n, k, order="F").copy() \
                if k else np.zeros((n, 0), order="F")
        pivots = np.ctypeslib.as_array(res.pivots, shape=(k,)).copy() if k else np.zeros(0, np.int64)
        chol = np.ctypeslib.as_array(res.chol, shape=(k * k,)).reshape(k, k, order="F").copy() \
            if k else np.zeros((0, 0))
        resid = np.ctypeslib.as_array(res.residual_diag, shape=(n,)).copy()
        prop = np.ctypeslib.as_array(res.proposed, shape=(nr * b,)).reshape(nr, b).copy() \
            if nr else np.zeros((0, b), np.int64)
        cnt = np.ctypeslib.as_array(res.accepted_count, shape=(nr,)).copy() \
            if nr else np.zeros(0, np.int64)
        accepted, off = [], 0
        for c in cnt:
            accepted.append(pivots[off: off + c].copy())
            off += int(c)
        return Result(factor, pivots, chol, resid, [p for p in prop], accepted,
                      bool(res.rank_exhausted), int(res.surplus), float(res.captured_sq))
    finally:
        lib().rpo_result_free(C.byref(res))


def accelerated_rpcholesky(oracle: Oracle, *, block_size: int, mode: str = "until_rank",
                           rounds: int = 0, target_rank: int = 0, seed: int = 0,
                           stop_tol: float = 0.0, max_rounds: int = -1,
                           copy_factor: bool = True) -> Result:
    """copy_factor=False keeps the C factor buffer behind a numpy view (no second copy of
    a multi-GB factor); it is freed with the last view."""
    cfg = _Cfg(block_size, MODES[mode], rounds, target_rank, seed, stop_tol)
    res = _Res()
    _check(lib().rpo_accelerated_rpcholesky_bounded(C.byref(oracle._o), C.byref(cfg),
                                                    max_rounds, C.byref(res)))
    return _unpack(res, copy_factor)


@dataclass
class Margins:
    """Smallest decision margins seen since margins_reset() (rpc_oracle.c recorder):
    draw = distance of a sampling target to the nearer cumsum bucket edge / total;
    sweep = |u_i r_i - h_ii| / u_i over every accept test."""
    min_draw: float
    min_sweep: float
    n_draws: int
    n_decisions: int


def margins_reset(on: bool = True) -> None:
    lib().rpo_margins_reset(int(on))


def margins_get() -> Margins:
    a, b, c, d = C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
    lib().rpo_margins_get(C.byref(a), C.byref(b), C.byref(c), C.byref(d))
    return Margins(a.value, b.value, c.value, d.value)


def block_rpcholesky(oracle: Oracle, *, block_size: int, mode: str = "until_rank",
                     rounds: int = 0, target_rank: int = 0, seed: int = 0,
                     stop_tol: float = 0.0) -> Result:
    """rpcholesky.hpp:268-333; Result.accepted holds the kept (sorted, distinct) proposals."""
    cfg = _Cfg(block_size, MODES[mode], rounds, target_rank, seed, stop_tol)
    res = _Res()
    _check(lib().rpo_block_rpcholesky(C.byref(oracle._o), C.byref(cfg), C.byref(res)))
    return _unpack(res)


def simple_rpcholesky(oracle: Oracle, k: int, seed: int) -> Result:
    """rpcholesky.hpp:206-246."""
    res = _Res()
    _check(lib().rpo_simple_rpcholesky(C.byref(oracle._o), k, seed, C.byref(res)))
    return _unpack(res)


def accelerated_rpcholesky_lowmem(oracle: Oracle, *, block_size: int, mode: str = "until_rank",
                                  rounds: int = 0, target_rank: int = 0, seed: int = 0,
                                  stop_tol: float = 0.0) -> Result:
    """rpcholesky.hpp:408-485; Result.factor is None (LowMemResult)."""
    cfg = _Cfg(block_size, MODES[mode], rounds, target_rank, seed, stop_tol)
    res = _Res()
    _check(lib().rpo_accelerated_rpcholesky_lowmem(C.byref(oracle._o), C.byref(cfg), C.byref(res)))
    return _unpack(res)


def relative_trace_error(oracle: Oracle, factor: np.ndarray) -> float:
    f = np.asfortranarray(factor, dtype=np.float64)
    return float(lib().rpo_relative_trace_error(C.byref(oracle._o), _p(f), f.shape[0],
                                                f.shape[1]))


# ---- io.hpp:218-293, 336-350: RPCF factor file and pivot-trace CSV (restatement) ----------
def write_rpcf(path: str, factor: np.ndarray, pivots, chol: np.ndarray | None) -> None:
    """write_rpcf (io.hpp:218-256): "RPCF", u32 1, u64 N, u64 k, factor column-major f64 LE,
    k u64 pivots, u64 packed count, chol lower triangle row by row."""
    import struct
    f = np.asarray(factor, dtype="<f8")
    n, k = f.shape
    piv = np.asarray(pivots, dtype="<u8")
    if piv.size != k:
        raise ValueError("write_rpcf: pivot count must match factor columns")
    has_chol = chol is not None and chol.shape == (k, k) and k > 0
    with open(path, "wb") as fh:
        fh.write(b"RPCF" + struct.pack("<IQQ", 1, n, k))
        fh.write(np.asfortranarray(f).tobytes(order="F"))
        fh.write(piv.tobytes())
        fh.write(struct.pack("<Q", k * (k + 1) // 2 if has_chol else 0))
        if has_chol:
            fh.write(np.concatenate([np.asarray(chol, "<f8")[i, : i + 1] for i in range(k)]).tobytes())


def read_rpcf(path: str):
    """read_rpcf (io.hpp:258-293): (factor N x k, pivots int64, chol k x k or None)."""
    import struct
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != b"RPCF":
        raise RuntimeError(f"read_rpcf: bad magic in {path}")
    ver, n, k = struct.unpack_from("<IQQ", data, 4)
    if ver != 1:
        raise RuntimeError("read_rpcf: unsupported version")
    off = 24
    factor = np.frombuffer(data, "<f8", n * k, off).reshape((n, k), order="F").copy()
    off += 8 * n * k
    piv = np.frombuffer(data, "<u8", k, off).astype(np.int64)
    off += 8 * k
    (cnt,) = struct.unpack_from("<Q", data, off)
    off += 8
    chol = None
    if cnt:
        if cnt != k * (k + 1) // 2:
            raise RuntimeError("read_rpcf: unexpected Cholesky payload size")
        vals = np.frombuffer(data, "<f8", cnt, off)
        chol = np.zeros((k, k))
        p = 0
        for i in range(k):
            chol[i, : i + 1] = vals[p: p + i + 1]
            p += i + 1
    return factor, piv, chol


def write_pivot_trace_csv(path: str, proposed, accepted) -> None:
    """write_pivot_trace_csv (io.hpp:336-350)."""
    with open(path, "w") as fh:
        fh.write("round,proposed,accepted,acceptance_rate\n")
        for r, (p, a) in enumerate(zip(proposed, accepted)):
            rate = len(a) / len(p) if len(p) else 0.0
            fh.write(f"{r},{len(p)},{len(a)},{'%.17g' % rate}\n")
