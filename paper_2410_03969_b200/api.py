"""Python mirror of the reference's hot-path API over the B200 C-ABI.

Names and argument meaning follow /root/reference/proj/include/rpchol:
  KernelSpec (kernels.hpp:41-51), DistanceMode (oracle.hpp:37),
  KernelOracle (oracle.hpp:243-258), RunConfig (rpcholesky.hpp:36-67),
  accelerated_rpcholesky (rpcholesky.hpp:338-401) -> CholeskyResult (106-110),
  relative_trace_error (577-583).
Errors map to the reference's exception classes: ValueError for
std::invalid_argument, IndexError for std::out_of_range, RuntimeError for
std::runtime_error.  Every call runs on the GPU through librpchol_b200.so;
there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

KERNEL_KINDS = {"gaussian": L.RPC_KERNEL_GAUSSIAN, "l1laplace": L.RPC_KERNEL_L1LAPLACE,
                "laplace": L.RPC_KERNEL_L1LAPLACE, "matern32": L.RPC_KERNEL_MATERN32,
                "matern52": L.RPC_KERNEL_MATERN52}  # kernel_kind_from_name (kernels.hpp:31-37)
DISTANCE_MODES = {None: L.RPC_DIST_DEFAULT, "direct": L.RPC_DIST_DIRECT, "gram": L.RPC_DIST_GRAM}


@dataclass
class KernelSpec:
    kind: str = "gaussian"
    bandwidth: float = 1.0


@dataclass
class RunConfig:
    block_size: int = 1
    mode: str = "until_rank"
    rounds: int = 0
    target_rank: int = 0
    seed: int = 0
    stop_tol: float = 0.0
    replay_scan: bool = False
    fp64_residual: bool = False  # every round's residual GEMM on FP64 DMMA (no int8 digits)

    @staticmethod
    def fixed_rounds(t: int, b: int, seed: int) -> "RunConfig":
        if t < 1 or b < 1:
            raise ValueError("RunConfig: t, b must be >= 1")
        return RunConfig(block_size=b, mode="fixed_rounds", rounds=t, seed=seed)

    @staticmethod
    def until_rank(k: int, b: int, seed: int) -> "RunConfig":
        if k < 1 or b < 1:
            raise ValueError("RunConfig: k, b must be >= 1")
        return RunConfig(block_size=b, mode="until_rank", target_rank=k, seed=seed)

    def to_c(self) -> L.RunConfigC:
        mode = L.RPC_FIXED_ROUNDS if self.mode == "fixed_rounds" else L.RPC_UNTIL_RANK
        return L.RunConfigC(self.block_size, mode, self.rounds, self.target_rank,
                            self.seed & 0xFFFFFFFFFFFFFFFF, self.stop_tol,
                            (L.RPC_FLAG_REPLAY_SCAN if self.replay_scan else 0) |
                            (L.RPC_FLAG_FP64_RESIDUAL if self.fp64_residual else 0))


class Context:
    """One GPU (optionally holding `virtual_shards` row shards), or one rank of
    an NCCL job (`nccl_id`, `nranks`, `rank`), or one rank of a job whose collectives
    run on the host (`host_collectives`, see hostcoll.py; rpc_create_hostcoll)."""

    def __init__(self, device: int = 0, virtual_shards: int = 1, nccl_id: bytes | None = None,
                 nranks: int = 1, rank: int = 0, host_collectives=None):
        lib = L.load()
        h = C.c_void_p()
        if host_collectives is not None:
            self._hc = _host_collectives_c(host_collectives)  # keeps the callbacks alive
            L.check(lib.rpc_create_hostcoll(device, host_collectives.nranks,
                                            host_collectives.rank, C.byref(self._hc), C.byref(h)))
        elif nccl_id is not None:
            L.check(lib.rpc_create_nccl(device, nccl_id, nranks, rank, C.byref(h)))
        elif virtual_shards > 1:
            L.check(lib.rpc_create_virtual(device, virtual_shards, C.byref(h)))
        else:
            L.check(lib.rpc_create(device, C.byref(h)))
        self.handle = h
        self.virtual_shards = virtual_shards
        self._children = weakref.WeakSet()  # results / models that hold device memory

    def _adopt(self, child):
        self._children.add(child)
        return child

    def close(self):
        if self.handle:
            for c in list(self._children):  # release children before the context goes
                c.free()
            L.load().rpc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard_rows(self, n: int, local: int = 0):
        r0, nr = C.c_int64(), C.c_int64()
        L.check(L.load().rpc_shard_rows(self.handle, n, local, C.byref(r0), C.byref(nr)))
        return r0.value, nr.value


def _host_collectives_c(hc) -> L.HostCollectivesC:
    """Wraps an object with allgather(send: uint8 array) -> uint8 array (nranks x bytes) and
    allreduce_or(buf: uint64 array, in place) as rpc_host_collectives callbacks."""

    def allgather(user, send, recv, nbytes):
        try:
            src = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), shape=(nbytes,))
            dst = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)),
                                        shape=(nbytes * hc.nranks,))
            dst[:] = np.asarray(hc.allgather(src.copy()), dtype=np.uint8).reshape(-1)
            return 0
        except Exception:  # reported as RPC_ENCCL by the library
            return 1

    def allreduce_or(user, buf, count):
        try:
            a = np.ctypeslib.as_array(buf, shape=(count,))
            hc.allreduce_or(a)
            return 0
        except Exception:
            return 1

    return L.HostCollectivesC(None, L.ALLGATHER_FN(allgather), L.ALLREDUCE_OR_FN(allreduce_or))


def plan_shards(n: int, n_shards: int, shard: int) -> dict:
    """Host-only shard plan of the C-ABI (rpc_plan_shards); needs no GPU."""
    r0, nr = C.c_int64(), C.c_int64()
    c0, nc, cpr = C.c_int(), C.c_int(), C.c_int()
    L.check(L.load().rpc_plan_shards(n, n_shards, shard, C.byref(r0), C.byref(nr), C.byref(c0),
                                     C.byref(nc), C.byref(cpr)))
    return {"row0": r0.value, "nrows": nr.value, "chunk0": c0.value, "nchunks": nc.value,
            "chunks_per_shard": cpr.value}


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    L.check(L.load().rpc_nccl_unique_id(buf))
    return buf.raw


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class KernelOracle:
    """Implicit kernel matrix over points X (N x d), as oracle.hpp:243-327."""

    def __init__(self, points: np.ndarray, spec: KernelSpec, distance_mode: str | None = None):
        x = np.asarray(points, dtype=np.float64)
        if x.ndim != 2:
            raise ValueError("DataMatrix: need at least one point and one dimension")
        self.points = x
        self.spec = spec
        self.distance_mode = distance_mode

    def dimension(self) -> int:
        return self.points.shape[0]

    def _c_spec(self) -> L.KernelSpecC:
        kind = KERNEL_KINDS.get(self.spec.kind)
        if kind is None:
            raise ValueError("unknown kernel: " + str(self.spec.kind))
        return L.KernelSpecC(kind, float(self.spec.bandwidth), DISTANCE_MODES[self.distance_mode])

    def _host_layout(self):
        x = self.points
        if x.flags.f_contiguous and not x.flags.c_contiguous:
            return x, L.RPC_COL_MAJOR, x.shape[0]
        x = np.ascontiguousarray(x)
        return x, L.RPC_ROW_MAJOR, x.shape[1]

    def columns(self, cols, ctx: Context | None = None, return_ms: bool = False):
        """A(:, cols) via the standalone K5 kernel (PsdOracle::columns)."""
        ctx = ctx or default_context()
        x, lay, ld = self._host_layout()
        c = np.ascontiguousarray(cols, dtype=np.int64)
        n = x.shape[0]
        out = np.zeros((n, c.size), dtype=np.float64, order="F")
        ms = C.c_double()
        L.check(L.load().rpc_kernel_columns(ctx.handle, x.ctypes.data, n, x.shape[1], ld, lay,
                                            self._c_spec(), c.ctypes.data, c.size,
                                            out.ctypes.data, n, C.byref(ms)), ctx.handle)
        return (out, ms.value) if return_ms else out


@dataclass(eq=False)
class CholeskyResult:
    """CholeskyResult (rpcholesky.hpp:106-110) with the factor kept on the device
    until `factor` is first read."""
    _handle: C.c_void_p
    _ctx: Context
    n: int
    pivots: np.ndarray
    proposed: list
    accepted: list
    rank_exhausted: bool
    surplus: int
    captured_sq: float
    relative_trace_error: float
    timing: dict = field(default_factory=dict)
    _factor: np.ndarray | None = None
    _chol: np.ndarray | None = None

    @property
    def rank(self) -> int:
        return int(self.pivots.size)

    @property
    def chol_factor(self) -> np.ndarray:
        """k x k lower-triangular F(pivots, :) (rpcholesky.hpp:140-145)."""
        if self._chol is None:
            k = self.rank
            self._chol = np.zeros((k, k), order="F")
            L.check(L.load().rpc_result_chol_copy(self._handle, self._chol.ctypes.data),
                    self._ctx.handle)
        return self._chol

    def factor_into(self, out: np.ndarray, layout: str = "F") -> np.ndarray:
        lay = L.RPC_COL_MAJOR if layout == "F" else L.RPC_ROW_MAJOR
        ld = out.shape[0] if layout == "F" else out.shape[1]
        L.check(L.load().rpc_result_factor_copy(self._handle, out.ctypes.data, ld, lay),
                self._ctx.handle)
        return out

    @property
    def factor(self) -> np.ndarray:
        if self._factor is None:
            self._factor = self.factor_into(np.zeros((self.n, self.rank), order="F"))
        return self._factor

    @property
    def residual_diag(self) -> np.ndarray:
        out = np.zeros(self.n)
        L.check(L.load().rpc_result_residual_diag_copy(self._handle, out.ctypes.data),
                self._ctx.handle)
        return out

    def write_rpcf(self, path: str) -> None:
        """write_rpcf (io.hpp:218-256), streamed from the device-resident factor."""
        L.check(L.load().rpc_result_write_rpcf(self._handle, path.encode()), self._ctx.handle)

    def write_trace_csv(self, path: str) -> None:
        """write_pivot_trace_csv (io.hpp:336-350)."""
        L.check(L.load().rpc_result_write_trace_csv(self._handle, path.encode()), self._ctx.handle)

    def free(self):
        if self._handle:
            L.load().rpc_result_free(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _wrap_result(h: C.c_void_p, ctx: Context) -> CholeskyResult:
    lib = L.load()
    n = lib.rpc_result_n(h)
    k = lib.rpc_result_rank(h)
    piv = np.zeros(k, np.int64)
    lib.rpc_result_pivots(h, piv.ctypes.data)
    b = lib.rpc_result_block_size(h)
    proposed, accepted = [], []
    for r in range(lib.rpc_result_num_rounds(h)):
        pr = np.zeros(b, np.int64)
        ac = np.zeros(b, np.int64)
        na = C.c_int64()
        L.check(lib.rpc_result_round(h, r, pr.ctypes.data, ac.ctypes.data, C.byref(na)))
        proposed.append(pr)
        accepted.append(ac[: na.value].copy())
    t = L.TimingC()
    lib.rpc_result_timing(h, C.byref(t))
    timing = {f: getattr(t, f) for f, _ in L.TimingC._fields_}
    return ctx._adopt(CholeskyResult(h, ctx, n, piv, proposed, accepted,
                                     bool(lib.rpc_result_rank_exhausted(h)),
                                     int(lib.rpc_result_surplus(h)),
                                     float(lib.rpc_result_captured_sq(h)),
                                     float(lib.rpc_result_relative_trace_error(h)), timing))


def accelerated_rpcholesky(oracle: KernelOracle, cfg: RunConfig,
                           ctx: Context | None = None) -> CholeskyResult:
    """rpchol::accelerated_rpcholesky (rpcholesky.hpp:338-401) on the GPU."""
    if not isinstance(oracle, KernelOracle):
        raise ValueError("accelerated_rpcholesky (B200): only KernelOracle inputs are supported")
    ctx = ctx or default_context()
    x, lay, ld = oracle._host_layout()
    h = C.c_void_p()
    L.check(L.load().rpc_accelerated_rpcholesky(ctx.handle, x.ctypes.data, x.shape[0],
                                                x.shape[1], ld, lay, oracle._c_spec(),
                                                cfg.to_c(), C.byref(h)), ctx.handle)
    return _wrap_result(h, ctx)


def factor_capacity(n: int, cfg: RunConfig) -> int:
    """Columns the factor can reach: min(N, t b) (FixedRounds) or min(N, k + b)."""
    cap = cfg.rounds * cfg.block_size if cfg.mode == "fixed_rounds" else cfg.target_rank + cfg.block_size
    return min(n, cap)


def accelerated_rpcholesky_into(oracle: KernelOracle, cfg: RunConfig, out: np.ndarray | None = None,
                                ctx: Context | None = None) -> CholeskyResult:
    """accelerated_rpcholesky with the factor streamed to host memory while the rounds run
    (rpc_accelerated_rpcholesky_into).  `out`: Fortran-ordered N x >= factor_capacity; the
    result's `factor` is a view of its first rank columns."""
    if not isinstance(oracle, KernelOracle):
        raise ValueError("accelerated_rpcholesky (B200): only KernelOracle inputs are supported")
    ctx = ctx or default_context()
    x, lay, ld = oracle._host_layout()
    n = x.shape[0]
    cap = factor_capacity(n, cfg)
    if out is None:
        out = np.empty((n, cap), order="F")
    if not out.flags.f_contiguous or out.shape[0] != n or out.shape[1] < cap:
        raise ValueError("accelerated_rpcholesky_into: out must be Fortran-ordered N x capacity")
    h = C.c_void_p()
    L.check(L.load().rpc_accelerated_rpcholesky_into(ctx.handle, x.ctypes.data, n, x.shape[1], ld,
                                                     lay, oracle._c_spec(), cfg.to_c(),
                                                     out.ctypes.data, n, out.shape[1], C.byref(h)),
            ctx.handle)
    r = _wrap_result(h, ctx)
    r._factor = out[:, : r.rank]
    return r


def accelerated_rpcholesky_device(x_dev_ptr: int, n: int, d: int, ld: int, layout: int,
                                  spec: KernelSpec, cfg: RunConfig, ctx: Context,
                                  distance_mode: str | None = None) -> CholeskyResult:
    """Same, with this process's shard rows already resident on the device."""
    o = KernelOracle(np.zeros((1, 1)), spec, distance_mode)
    h = C.c_void_p()
    L.check(L.load().rpc_accelerated_rpcholesky_device(ctx.handle, C.c_void_p(x_dev_ptr), n, d,
                                                       ld, layout, o._c_spec(), cfg.to_c(),
                                                       C.byref(h)), ctx.handle)
    return _wrap_result(h, ctx)


def block_rpcholesky(oracle: KernelOracle, cfg: RunConfig,
                     ctx: Context | None = None) -> CholeskyResult:
    """rpchol::block_rpcholesky (rpcholesky.hpp:268-333) on the GPU; `accepted` per round is
    the kept (sorted, distinct) proposal list."""
    if not isinstance(oracle, KernelOracle):
        raise ValueError("block_rpcholesky (B200): only KernelOracle inputs are supported")
    ctx = ctx or default_context()
    x, lay, ld = oracle._host_layout()
    h = C.c_void_p()
    L.check(L.load().rpc_block_rpcholesky(ctx.handle, x.ctypes.data, x.shape[0], x.shape[1], ld,
                                          lay, oracle._c_spec(), cfg.to_c(), C.byref(h)),
            ctx.handle)
    return _wrap_result(h, ctx)


def simple_rpcholesky(oracle: KernelOracle, k: int, seed: int, ctx: Context | None = None,
                      replay_scan: bool = False) -> CholeskyResult:
    """rpchol::simple_rpcholesky (rpcholesky.hpp:206-246) on the GPU."""
    if not isinstance(oracle, KernelOracle):
        raise ValueError("simple_rpcholesky (B200): only KernelOracle inputs are supported")
    ctx = ctx or default_context()
    x, lay, ld = oracle._host_layout()
    h = C.c_void_p()
    L.check(L.load().rpc_simple_rpcholesky(ctx.handle, x.ctypes.data, x.shape[0], x.shape[1], ld,
                                           lay, oracle._c_spec(), k, seed,
                                           L.RPC_FLAG_REPLAY_SCAN if replay_scan else 0,
                                           C.byref(h)), ctx.handle)
    return _wrap_result(h, ctx)


def block_rpcholesky_device(x_dev_ptr: int, n: int, d: int, ld: int, layout: int,
                            spec: KernelSpec, cfg: RunConfig, ctx: Context) -> CholeskyResult:
    o = KernelOracle(np.zeros((1, 1)), spec)
    h = C.c_void_p()
    L.check(L.load().rpc_block_rpcholesky_device(ctx.handle, C.c_void_p(x_dev_ptr), n, d, ld,
                                                 layout, o._c_spec(), cfg.to_c(), C.byref(h)),
            ctx.handle)
    return _wrap_result(h, ctx)


def simple_rpcholesky_device(x_dev_ptr: int, n: int, d: int, ld: int, layout: int,
                             spec: KernelSpec, k: int, seed: int, ctx: Context) -> CholeskyResult:
    o = KernelOracle(np.zeros((1, 1)), spec)
    h = C.c_void_p()
    L.check(L.load().rpc_simple_rpcholesky_device(ctx.handle, C.c_void_p(x_dev_ptr), n, d, ld,
                                                  layout, o._c_spec(), k, seed, 0, C.byref(h)),
            ctx.handle)
    return _wrap_result(h, ctx)


def accelerated_rpcholesky_lowmem(oracle: KernelOracle, cfg: RunConfig,
                                  ctx: Context | None = None) -> CholeskyResult:
    """rpchol::accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485) on the GPU.

    Returns the LowMemResult fields (rpcholesky.hpp:114-119): pivots, chol_factor,
    residual_diag and the trace; `factor` is not stored (reading it raises ValueError).
    """
    if not isinstance(oracle, KernelOracle):
        raise ValueError("accelerated_rpcholesky_lowmem (B200): only KernelOracle inputs are supported")
    ctx = ctx or default_context()
    x, lay, ld = oracle._host_layout()
    h = C.c_void_p()
    L.check(L.load().rpc_accelerated_rpcholesky_lowmem(ctx.handle, x.ctypes.data, x.shape[0],
                                                       x.shape[1], ld, lay, oracle._c_spec(),
                                                       cfg.to_c(), C.byref(h)), ctx.handle)
    return _wrap_result(h, ctx)


def accelerated_rpcholesky_lowmem_device(x_dev_ptr: int, n: int, d: int, ld: int, layout: int,
                                         spec: KernelSpec, cfg: RunConfig, ctx: Context,
                                         distance_mode: str | None = None) -> CholeskyResult:
    """Low-memory variant with this process's shard rows already on the device."""
    o = KernelOracle(np.zeros((1, 1)), spec, distance_mode)
    h = C.c_void_p()
    L.check(L.load().rpc_accelerated_rpcholesky_lowmem_device(
        ctx.handle, C.c_void_p(x_dev_ptr), n, d, ld, layout, o._c_spec(), cfg.to_c(), C.byref(h)),
        ctx.handle)
    return _wrap_result(h, ctx)


def bench_column_throughput(oracle: KernelOracle, block_sizes, seed: int = 0,
                            ctx: Context | None = None) -> list:
    """bench_column_throughput (experiment.hpp:344-387) on the device: one dict per
    (block size, distance mode) with columns, wall_ms (device), columns_per_sec, output_gbs."""
    ctx = ctx or default_context()
    x, lay, ld = oracle._host_layout()
    bs = np.ascontiguousarray(block_sizes, dtype=np.int64)
    rows = (L.ThroughputRowC * (2 * bs.size))()
    nr = C.c_int()
    L.check(L.load().rpc_bench_column_throughput(ctx.handle, x.ctypes.data, x.shape[0], x.shape[1],
                                                 ld, lay, oracle._c_spec(), bs.ctypes.data, bs.size,
                                                 seed, rows, C.byref(nr)), ctx.handle)
    names = {L.RPC_DIST_DIRECT: "direct", L.RPC_DIST_GRAM: "gram"}
    return [dict(block_size=r.block_size, mode=names[r.distance_mode], columns=r.columns,
                 wall_ms=r.wall_ms, columns_per_sec=r.columns_per_sec, output_gbs=r.output_gbs)
            for r in rows[: nr.value]]


def relative_trace_error(oracle: KernelOracle, result: CholeskyResult) -> float:
    """rpcholesky.hpp:577-583, evaluated from the device-resident factor."""
    return result.relative_trace_error


def sample_discrete(u: np.ndarray, b: int, seed: int, draw0: int = 0, replay: bool = False,
                    ctx: Context | None = None) -> np.ndarray:
    """b draws of rng.hpp:80-96 against cumulative_sums(u), on the GPU."""
    ctx = ctx or default_context()
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(b, np.int64)
    L.check(L.load().rpc_sample_discrete(ctx.handle, u.ctypes.data, u.size, b, seed, draw0,
                                         int(replay), out.ctypes.data), ctx.handle)
    return out


def rejection_sample_submatrix(h: np.ndarray, proposals, seed: int, draw0: int,
                               ctx: Context | None = None):
    """rpcholesky.hpp:167-201 on the GPU: (accepted, positions, chol)."""
    ctx = ctx or default_context()
    h = np.asfortranarray(h, dtype=np.float64)
    b = h.shape[0]
    prop = np.ascontiguousarray(proposals, dtype=np.int64)
    acc = np.zeros(b, np.int64)
    pos = np.zeros(b, np.int64)
    chol = np.zeros(b * b)
    m = C.c_int64()
    L.check(L.load().rpc_rejection_sweep(ctx.handle, h.ctypes.data, b, prop.ctypes.data, seed,
                                         draw0, acc.ctypes.data, pos.ctypes.data, C.byref(m),
                                         chol.ctypes.data), ctx.handle)
    k = m.value
    return acc[:k].copy(), pos[:k].copy(), chol[: k * k].reshape(k, k, order="F").copy()


# ---------------------------------------------------------------------------
# Kernel ridge regression (krr.hpp) on the device
# ---------------------------------------------------------------------------
def kernel_matvec(oracle: KernelOracle, v: np.ndarray, ctx: Context | None = None) -> np.ndarray:
    """kernel_matvec (krr.hpp:143-162): A v (or A V for up to 8 columns), A never formed."""
    ctx = ctx or default_context()
    x, lay, ld = oracle._host_layout()
    v = np.asarray(v, dtype=np.float64)
    vv = np.asfortranarray(v.reshape(v.shape[0], -1))
    out = np.zeros(vv.shape, order="F")
    L.check(L.load().rpc_kernel_matvec(ctx.handle, x.ctypes.data, x.shape[0], x.shape[1], ld, lay,
                                       oracle._c_spec(), vv.ctypes.data, vv.shape[1],
                                       out.ctypes.data), ctx.handle)
    return out.reshape(v.shape)


@dataclass
class PcgReport:
    """PcgReport (krr.hpp:80-85)."""
    iterations: int
    relative_residuals: np.ndarray
    relative_residuals_unreg: np.ndarray
    converged: bool


class KrrModel:
    """KrrModel (krr.hpp:125-131): coefficients and training points stay on the device."""

    def __init__(self, handle: C.c_void_p, ctx: Context, n: int, d: int):
        self._h, self._ctx, self.n, self.d = handle, ctx, n, d

    @property
    def coefficients(self) -> np.ndarray:
        out = np.zeros(self.n)
        L.check(L.load().rpc_krr_coefficients(self._h, out.ctypes.data), self._ctx.handle)
        return out

    @property
    def target_mean(self) -> float:
        return float(L.load().rpc_krr_target_mean(self._h))

    def free(self):
        if self._h:
            L.load().rpc_krr_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


@dataclass
class KrrFitResult:
    """KrrFitResult (krr.hpp:164-168); `preconditioner_pivots` are the pivots of the
    accelerated-RPCholesky factor behind the Woodbury preconditioner."""
    model: KrrModel
    report: PcgReport
    preconditioner_pivots: np.ndarray


def fit_krr(points: np.ndarray, targets: np.ndarray, spec: KernelSpec, mu: float,
            precond_rank: int, config: RunConfig, tol: float, max_iters: int = 500,
            ctx: Context | None = None) -> KrrFitResult:
    """fit_krr (krr.hpp:177-224) on the GPU: RPCholesky preconditioner + PCG with fused
    kernel matvecs."""
    ctx = ctx or default_context()
    ko = KernelOracle(points, spec)
    x, lay, ld = ko._host_layout()
    t = np.ascontiguousarray(targets, dtype=np.float64)
    if t.shape[0] != x.shape[0]:
        raise ValueError("fit_krr: targets size mismatch")
    h = C.c_void_p()
    lib = L.load()
    L.check(lib.rpc_krr_fit(ctx.handle, x.ctypes.data, x.shape[0], x.shape[1], ld, lay,
                            ko._c_spec(), t.ctypes.data, mu, precond_rank, config.to_c(), tol,
                            max_iters, C.byref(h)), ctx.handle)
    it = lib.rpc_krr_iterations(h)
    reg, unreg = np.zeros(max(it, 1)), np.zeros(max(it, 1))
    lib.rpc_krr_residuals(h, reg.ctypes.data, unreg.ctypes.data)
    k = lib.rpc_krr_precond_rank(h)
    piv = np.zeros(max(k, 1), np.int64)
    lib.rpc_krr_precond_pivots(h, piv.ctypes.data)
    report = PcgReport(int(it), reg[:it].copy(), unreg[:it].copy(), bool(lib.rpc_krr_converged(h)))
    return KrrFitResult(ctx._adopt(KrrModel(h, ctx, x.shape[0], x.shape[1])), report, piv[:k].copy())


def predict(model: KrrModel, query: np.ndarray) -> np.ndarray:
    """predict (krr.hpp:227-250): sum_i beta_i kappa(x_i, q) + target mean."""
    q = np.asarray(query, dtype=np.float64)
    if q.ndim != 2 or q.shape[1] != model.d:
        raise ValueError("predict: query dimension mismatch")
    if q.flags.f_contiguous and not q.flags.c_contiguous:
        lay, ld = L.RPC_COL_MAJOR, q.shape[0]
    else:
        q = np.ascontiguousarray(q)
        lay, ld = L.RPC_ROW_MAJOR, q.shape[1]
    out = np.zeros(q.shape[0])
    L.check(L.load().rpc_krr_predict(model._h, q.ctypes.data, q.shape[0], q.shape[1], ld, lay,
                                     out.ctypes.data), model._ctx.handle)
    return out
