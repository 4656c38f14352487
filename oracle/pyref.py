"""ctypes binding of oracle/_ref/libref_rpchol.so: the REFERENCE's own headers
(/root/reference/proj/include/rpchol) compiled against the Eigen-API shim
(oracle/eigen_shim) by `make -C oracle ref`.

TEST INFRASTRUCTURE ONLY (pins the C restatement; reference arm of bench.py).
The library exists only where /root/reference was present at build time; on
the GPU box it travels as a prebuilt .so.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

import pyoracle as po

_HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(_HERE, "_ref", "libref_rpchol.so")
_L = None


def available() -> bool:
    return os.path.exists(PATH)


def lib():
    global _L
    if _L is None:
        L = C.CDLL(PATH)
        i64, vp, d = C.c_int64, C.c_void_p, C.c_double
        L.ref_last_error.restype = C.c_char_p
        L.ref_accelerated_kernel.argtypes = [vp, i64, i64, C.c_int, d, C.c_int, i64, C.c_int, i64,
                                             i64, C.c_uint64, d, C.POINTER(po._Res)]
        L.ref_lowmem_kernel.argtypes = L.ref_accelerated_kernel.argtypes
        L.ref_read_rpcf.argtypes = [C.c_char_p, C.POINTER(po._Res)]
        L.ref_write_rpcf_kernel.argtypes = [vp, i64, i64, C.c_int, d, C.c_int, i64, i64,
                                            C.c_uint64, C.c_char_p, C.c_char_p]
        L.ref_block_kernel.argtypes = L.ref_accelerated_kernel.argtypes
        L.ref_simple_kernel.argtypes = [vp, i64, i64, C.c_int, d, C.c_int, i64, C.c_uint64,
                                        C.POINTER(po._Res)]
        L.ref_accelerated_dense.argtypes = [vp, i64, i64, C.c_int, i64, i64, C.c_uint64, d,
                                            C.POINTER(po._Res)]
        L.ref_relative_trace_error_kernel.restype = d
        L.ref_relative_trace_error_kernel.argtypes = [vp, i64, i64, C.c_int, d, C.c_int, vp, i64]
        L.ref_kernel_submatrix.argtypes = [vp, i64, i64, C.c_int, d, C.c_int, vp, i64, vp, i64, vp]
        L.ref_sample_discrete.argtypes = [vp, i64, C.c_uint64, C.c_uint64, i64, vp]
        L.ref_rejection_sweep.argtypes = [vp, i64, vp, C.c_uint64, C.c_uint64, vp, vp,
                                          C.POINTER(i64), vp]
        L.ref_result_free.argtypes = [C.POINTER(po._Res)]
        L.ref_kernel_matvec.argtypes = [vp, i64, i64, C.c_int, d, C.c_int, vp, i64, vp]
        L.ref_fit_krr.argtypes = [vp, i64, i64, C.c_int, d, vp, d, i64, i64, C.c_uint64, d, i64,
                                  i64, vp, C.POINTER(d), C.POINTER(i64), C.POINTER(C.c_int), vp,
                                  vp, vp, C.POINTER(i64), vp, i64, vp]
        _L = L
    return _L


def _check(rc):
    if rc:
        raise {1: ValueError, 2: IndexError}.get(rc, RuntimeError)(lib().ref_last_error().decode())


def _unpack(res) -> po.Result:
    try:
        n, k, b, nr = res.n, res.rank, res.block_size, res.n_rounds
        f = (np.ctypeslib.as_array(res.factor, shape=(max(n * k, 1),))[: n * k]
             .reshape(n, k, order="F").copy() if res.factor else None)
        piv = np.ctypeslib.as_array(res.pivots, shape=(max(k, 1),))[:k].copy()
        chol = np.ctypeslib.as_array(res.chol, shape=(max(k * k, 1),))[: k * k].reshape(k, k, order="F").copy()
        resid = np.ctypeslib.as_array(res.residual_diag, shape=(n,)).copy()
        prop = np.ctypeslib.as_array(res.proposed, shape=(max(nr * b, 1),))[: nr * b].reshape(nr, b).copy()
        cnt = np.ctypeslib.as_array(res.accepted_count, shape=(max(nr, 1),))[:nr].copy()
        acc, off = [], 0
        for c in cnt:
            acc.append(piv[off: off + c].copy())
            off += int(c)
        return po.Result(f, piv, chol, resid, list(prop), acc, bool(res.rank_exhausted),
                         int(res.surplus), 0.0)
    finally:
        lib().ref_result_free(C.byref(res))


def accelerated_rpcholesky_kernel(x, kernel, sigma, *, block_size, mode="until_rank", rounds=0,
                                  target_rank=0, seed=0, stop_tol=0.0, dist=None) -> po.Result:
    xf = np.asfortranarray(x, dtype=np.float64)
    kind = po.KERNELS[kernel]
    dm = po.DIST[dist or ("direct" if kind == 1 else "gram")]
    res = po._Res()
    _check(lib().ref_accelerated_kernel(xf.ctypes.data, xf.shape[0], xf.shape[1], kind, sigma, dm,
                                        block_size, po.MODES[mode], rounds, target_rank, seed,
                                        stop_tol, C.byref(res)))
    return _unpack(res)


def accelerated_rpcholesky_lowmem_kernel(x, kernel, sigma, *, block_size, mode="until_rank",
                                         rounds=0, target_rank=0, seed=0, stop_tol=0.0,
                                         dist=None) -> po.Result:
    """accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485); .factor is None."""
    xf = np.asfortranarray(x, dtype=np.float64)
    kind = po.KERNELS[kernel]
    dm = po.DIST[dist or ("direct" if kind == 1 else "gram")]
    res = po._Res()
    _check(lib().ref_lowmem_kernel(xf.ctypes.data, xf.shape[0], xf.shape[1], kind, sigma, dm,
                                   block_size, po.MODES[mode], rounds, target_rank, seed,
                                   stop_tol, C.byref(res)))
    return _unpack(res)


def block_rpcholesky_kernel(x, kernel, sigma, *, block_size, mode="until_rank", rounds=0,
                            target_rank=0, seed=0, stop_tol=0.0, dist=None) -> po.Result:
    """block_rpcholesky (rpcholesky.hpp:268-333)."""
    xf = np.asfortranarray(x, dtype=np.float64)
    kind = po.KERNELS[kernel]
    dm = po.DIST[dist or ("direct" if kind == 1 else "gram")]
    res = po._Res()
    _check(lib().ref_block_kernel(xf.ctypes.data, xf.shape[0], xf.shape[1], kind, sigma, dm,
                                  block_size, po.MODES[mode], rounds, target_rank, seed, stop_tol,
                                  C.byref(res)))
    return _unpack(res)


def simple_rpcholesky_kernel(x, kernel, sigma, k, seed=0, dist=None) -> po.Result:
    """simple_rpcholesky (rpcholesky.hpp:206-246)."""
    xf = np.asfortranarray(x, dtype=np.float64)
    kind = po.KERNELS[kernel]
    dm = po.DIST[dist or ("direct" if kind == 1 else "gram")]
    res = po._Res()
    _check(lib().ref_simple_kernel(xf.ctypes.data, xf.shape[0], xf.shape[1], kind, sigma, dm, k,
                                   seed, C.byref(res)))
    return _unpack(res)


def accelerated_rpcholesky_dense(a, *, block_size, mode="until_rank", rounds=0, target_rank=0,
                                 seed=0, stop_tol=0.0) -> po.Result:
    af = np.asfortranarray(a, dtype=np.float64)
    res = po._Res()
    _check(lib().ref_accelerated_dense(af.ctypes.data, af.shape[0], block_size, po.MODES[mode],
                                       rounds, target_rank, seed, stop_tol, C.byref(res)))
    return _unpack(res)


def relative_trace_error_kernel(x, kernel, sigma, factor, dist=None) -> float:
    xf = np.asfortranarray(x, dtype=np.float64)
    f = np.asfortranarray(factor, dtype=np.float64)
    kind = po.KERNELS[kernel]
    dm = po.DIST[dist or ("direct" if kind == 1 else "gram")]
    return float(lib().ref_relative_trace_error_kernel(xf.ctypes.data, xf.shape[0], xf.shape[1],
                                                       kind, sigma, dm, f.ctypes.data, f.shape[1]))


def kernel_submatrix(x, kernel, sigma, rows, cols, dist=None):
    xf = np.asfortranarray(x, dtype=np.float64)
    kind = po.KERNELS[kernel]
    dm = po.DIST[dist or ("direct" if kind == 1 else "gram")]
    r = np.ascontiguousarray(rows, np.int64)
    c = np.ascontiguousarray(cols, np.int64)
    out = np.zeros((r.size, c.size), order="F")
    _check(lib().ref_kernel_submatrix(xf.ctypes.data, xf.shape[0], xf.shape[1], kind, sigma, dm,
                                      r.ctypes.data, r.size, c.ctypes.data, c.size, out.ctypes.data))
    return out


def sample_discrete(w, seed, draw0, count):
    w = np.ascontiguousarray(w, np.float64)
    out = np.zeros(count, np.int64)
    _check(lib().ref_sample_discrete(w.ctypes.data, w.size, seed, draw0, count, out.ctypes.data))
    return out


def rejection_sweep(h, proposals, seed, draw0):
    h = np.asfortranarray(h, np.float64)
    b = h.shape[0]
    prop = np.ascontiguousarray(proposals, np.int64)
    acc, pos, chol = np.zeros(b, np.int64), np.zeros(b, np.int64), np.zeros(b * b)
    m = C.c_int64()
    _check(lib().ref_rejection_sweep(h.ctypes.data, b, prop.ctypes.data, seed, draw0,
                                     acc.ctypes.data, pos.ctypes.data, C.byref(m), chol.ctypes.data))
    k = m.value
    return acc[:k].copy(), pos[:k].copy(), chol[: k * k].reshape(k, k, order="F").copy()


def kernel_matvec(x, kernel, sigma, v, dist=None, row_block=1024):
    """kernel_matvec (krr.hpp:143-162)."""
    xf = np.asfortranarray(x, dtype=np.float64)
    kind = po.KERNELS[kernel]
    dm = po.DIST[dist or ("direct" if kind == 1 else "gram")]
    vv = np.ascontiguousarray(v, np.float64)
    out = np.zeros(xf.shape[0])
    _check(lib().ref_kernel_matvec(xf.ctypes.data, xf.shape[0], xf.shape[1], kind, sigma, dm,
                                   vv.ctypes.data, row_block, out.ctypes.data))
    return out


def fit_krr(x, targets, kernel, sigma, mu, precond_rank, block_size, seed, tol, max_iters=500,
            materialize_threshold=8192, query=None):
    """fit_krr (krr.hpp:177-224) with RunConfig::until_rank(rank, b, seed), then predict on
    `query` when given.  Returns a dict of the KrrFitResult fields."""
    xf = np.asfortranarray(x, dtype=np.float64)
    n, d = xf.shape
    kind = po.KERNELS[kernel]
    t = np.ascontiguousarray(targets, np.float64)
    coef = np.zeros(n)
    rel, unreg = np.zeros(max(max_iters, 1)), np.zeros(max(max_iters, 1))
    piv = np.zeros(max(precond_rank, 1) + block_size, np.int64)
    mean, iters, conv, k = C.c_double(), C.c_int64(), C.c_int(), C.c_int64()
    qf = np.asfortranarray(query, np.float64) if query is not None else None
    pred = np.zeros(qf.shape[0]) if qf is not None else np.zeros(1)
    _check(lib().ref_fit_krr(xf.ctypes.data, n, d, kind, sigma, t.ctypes.data, mu, precond_rank,
                             block_size, seed, tol, max_iters, materialize_threshold,
                             coef.ctypes.data, C.byref(mean), C.byref(iters), C.byref(conv),
                             rel.ctypes.data, unreg.ctypes.data, piv.ctypes.data, C.byref(k),
                             qf.ctypes.data if qf is not None else None,
                             qf.shape[0] if qf is not None else 0, pred.ctypes.data))
    it = iters.value
    return dict(coefficients=coef, target_mean=mean.value, iterations=it, converged=bool(conv.value),
                relative_residuals=rel[:it].copy(), relative_residuals_unreg=unreg[:it].copy(),
                pivots=piv[:k.value].copy(), predictions=pred if qf is not None else None)


def read_rpcf(path):
    """read_rpcf (io.hpp:258-293): (factor N x k, pivots, chol k x k)."""
    res = po._Res()
    _check(lib().ref_read_rpcf(path.encode(), C.byref(res)))
    r = _unpack(res)
    return r.factor, r.pivots, r.chol


def write_rpcf_kernel(x, kernel, sigma, block_size, target_rank, seed, path, trace_csv=None, dist=None):
    """The reference's accelerated run written by its own write_rpcf / write_pivot_trace_csv."""
    xf = np.asfortranarray(x, dtype=np.float64)
    kind = po.KERNELS[kernel]
    dm = po.DIST[dist or ("direct" if kind == 1 else "gram")]
    _check(lib().ref_write_rpcf_kernel(xf.ctypes.data, xf.shape[0], xf.shape[1], kind, sigma, dm,
                                       block_size, target_rank, seed, path.encode(),
                                       trace_csv.encode() if trace_csv else None))
