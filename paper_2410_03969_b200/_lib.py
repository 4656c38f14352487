"""ctypes binding of librpchol_b200.so (the C-ABI declared in include/rpchol_gpu.h).

The library is built in-tree by `python -c "import __graft_entry__ as g; g.build()"`
(or `make -C paper_2410_03969_b200/csrc`).  Loading fails loudly when it is
missing: there is no CPU fallback for the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librpchol_b200.so")

RPC_OK, RPC_EINVAL, RPC_ERANGE, RPC_ENUMERIC, RPC_ECUDA, RPC_ENCCL, RPC_ENOMEM = range(7)
RPC_KERNEL_GAUSSIAN, RPC_KERNEL_L1LAPLACE, RPC_KERNEL_MATERN32, RPC_KERNEL_MATERN52 = 0, 1, 2, 3
RPC_DIST_DIRECT, RPC_DIST_GRAM, RPC_DIST_DEFAULT = 0, 1, -1
RPC_FIXED_ROUNDS, RPC_UNTIL_RANK = 0, 1
RPC_COL_MAJOR, RPC_ROW_MAJOR = 0, 1
RPC_FLAG_REPLAY_SCAN = 1
RPC_FLAG_FP64_RESIDUAL = 2

# Every symbol include/rpchol_gpu.h declares (checked by tests/test_boundary.py).
EXPORTS = [
    "rpc_create", "rpc_create_virtual", "rpc_nccl_unique_id", "rpc_create_nccl", "rpc_destroy",
    "rpc_last_error", "rpc_shard_rows", "rpc_plan_shards", "rpc_accelerated_rpcholesky",
    "rpc_accelerated_rpcholesky_device", "rpc_result_n", "rpc_result_rank", "rpc_result_pivots",
    "rpc_result_factor_copy", "rpc_result_chol_copy", "rpc_result_residual_diag_copy",
    "rpc_result_num_rounds", "rpc_result_block_size", "rpc_result_round",
    "rpc_result_rank_exhausted", "rpc_result_surplus", "rpc_result_captured_sq",
    "rpc_result_relative_trace_error", "rpc_result_factor_device", "rpc_result_timing",
    "rpc_result_free", "rpc_kernel_columns", "rpc_sample_discrete", "rpc_rejection_sweep",
    "rpc_accelerated_rpcholesky_lowmem", "rpc_accelerated_rpcholesky_lowmem_device",
    "rpc_result_is_lowmem", "rpc_kernel_matvec", "rpc_krr_fit", "rpc_krr_iterations",
    "rpc_krr_converged", "rpc_krr_residuals", "rpc_krr_coefficients", "rpc_krr_target_mean",
    "rpc_krr_precond_rank", "rpc_krr_precond_pivots", "rpc_krr_predict", "rpc_krr_free",
    "rpc_block_rpcholesky", "rpc_block_rpcholesky_device", "rpc_simple_rpcholesky",
    "rpc_simple_rpcholesky_device", "rpc_result_write_rpcf", "rpc_result_write_trace_csv",
    "rpc_bench_column_throughput", "rpc_accelerated_rpcholesky_into", "rpc_create_hostcoll",
]

# rpc_host_collectives (include/rpchol_gpu.h): callbacks the library calls for each collective
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
ALLREDUCE_OR_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_size_t)


class HostCollectivesC(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", ALLGATHER_FN),
                ("allreduce_or_u64", ALLREDUCE_OR_FN)]


class KernelSpecC(C.Structure):
    _fields_ = [("kind", C.c_int), ("sigma", C.c_double), ("distance_mode", C.c_int)]


class RunConfigC(C.Structure):
    _fields_ = [
        ("block_size", C.c_int64),
        ("mode", C.c_int),
        ("rounds", C.c_int64),
        ("target_rank", C.c_int64),
        ("seed", C.c_uint64),
        ("stop_tol", C.c_double),
        ("flags", C.c_uint32),
    ]


class ThroughputRowC(C.Structure):
    _fields_ = [("block_size", C.c_int64), ("distance_mode", C.c_int), ("columns", C.c_int64),
                ("wall_ms", C.c_double), ("columns_per_sec", C.c_double),
                ("output_gbs", C.c_double)]


class TimingC(C.Structure):
    _fields_ = [
        ("factorize_ms", C.c_double),
        ("upload_ms", C.c_double),
        ("update_ms", C.c_double),
        ("update_flops", C.c_double),
        ("update_bytes", C.c_double),
        ("update_launches", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("host_total_ms", C.c_double),
        ("host_setup_ms", C.c_double),
        ("host_loop_ms", C.c_double),
        ("host_final_ms", C.c_double),
        ("tc_ms", C.c_double),
        ("tc_int8_ops", C.c_double),
        ("tc_fp64_flops", C.c_double),
        ("tc_slice_ms", C.c_double),
    ]


_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                          "(no CPU fallback exists for this path)")
    L = C.CDLL(LIB_PATH)
    vp, i64, pi64, pd = C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_double)
    sig = {
        "rpc_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "rpc_create_virtual": (C.c_int, [C.c_int, C.c_int, C.POINTER(vp)]),
        "rpc_nccl_unique_id": (C.c_int, [C.c_char_p]),
        "rpc_create_nccl": (C.c_int, [C.c_int, C.c_char_p, C.c_int, C.c_int, C.POINTER(vp)]),
        "rpc_create_hostcoll": (C.c_int, [C.c_int, C.c_int, C.c_int,
                                          C.POINTER(HostCollectivesC), C.POINTER(vp)]),
        "rpc_destroy": (None, [vp]),
        "rpc_last_error": (C.c_char_p, [vp]),
        "rpc_shard_rows": (C.c_int, [vp, i64, C.c_int, pi64, pi64]),
        "rpc_plan_shards": (C.c_int, [i64, C.c_int, C.c_int, pi64, pi64, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "rpc_accelerated_rpcholesky": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC,
                                                 RunConfigC, C.POINTER(vp)]),
        "rpc_accelerated_rpcholesky_device": (C.c_int, [vp, vp, i64, i64, i64, C.c_int,
                                                        KernelSpecC, RunConfigC, C.POINTER(vp)]),
        "rpc_accelerated_rpcholesky_lowmem": (C.c_int, [vp, vp, i64, i64, i64, C.c_int,
                                                        KernelSpecC, RunConfigC, C.POINTER(vp)]),
        "rpc_accelerated_rpcholesky_lowmem_device": (C.c_int, [vp, vp, i64, i64, i64, C.c_int,
                                                               KernelSpecC, RunConfigC,
                                                               C.POINTER(vp)]),
        "rpc_result_is_lowmem": (C.c_int, [vp]),
        "rpc_result_write_rpcf": (C.c_int, [vp, C.c_char_p]),
        "rpc_accelerated_rpcholesky_into": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC,
                                                      RunConfigC, vp, i64, i64, C.POINTER(vp)]),
        "rpc_bench_column_throughput": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC, vp,
                                                  C.c_int, C.c_uint64, vp, C.POINTER(C.c_int)]),
        "rpc_result_write_trace_csv": (C.c_int, [vp, C.c_char_p]),
        "rpc_block_rpcholesky": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC,
                                           RunConfigC, C.POINTER(vp)]),
        "rpc_block_rpcholesky_device": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC,
                                                  RunConfigC, C.POINTER(vp)]),
        "rpc_simple_rpcholesky": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC, i64,
                                            C.c_uint64, C.c_uint32, C.POINTER(vp)]),
        "rpc_simple_rpcholesky_device": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC,
                                                   i64, C.c_uint64, C.c_uint32, C.POINTER(vp)]),
        "rpc_kernel_matvec": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC, vp, i64, vp]),
        "rpc_krr_fit": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC, vp, C.c_double, i64,
                                  RunConfigC, C.c_double, i64, C.POINTER(vp)]),
        "rpc_krr_iterations": (i64, [vp]),
        "rpc_krr_converged": (C.c_int, [vp]),
        "rpc_krr_residuals": (C.c_int, [vp, vp, vp]),
        "rpc_krr_coefficients": (C.c_int, [vp, vp]),
        "rpc_krr_target_mean": (C.c_double, [vp]),
        "rpc_krr_precond_rank": (i64, [vp]),
        "rpc_krr_precond_pivots": (C.c_int, [vp, vp]),
        "rpc_krr_predict": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, vp]),
        "rpc_krr_free": (None, [vp]),
        "rpc_result_n": (i64, [vp]),
        "rpc_result_rank": (i64, [vp]),
        "rpc_result_pivots": (C.c_int, [vp, vp]),
        "rpc_result_factor_copy": (C.c_int, [vp, vp, i64, C.c_int]),
        "rpc_result_chol_copy": (C.c_int, [vp, vp]),
        "rpc_result_residual_diag_copy": (C.c_int, [vp, vp]),
        "rpc_result_num_rounds": (i64, [vp]),
        "rpc_result_block_size": (i64, [vp]),
        "rpc_result_round": (C.c_int, [vp, i64, vp, vp, pi64]),
        "rpc_result_rank_exhausted": (C.c_int, [vp]),
        "rpc_result_surplus": (i64, [vp]),
        "rpc_result_captured_sq": (C.c_double, [vp]),
        "rpc_result_relative_trace_error": (C.c_double, [vp]),
        "rpc_result_factor_device": (vp, [vp, pi64, pi64, pi64]),
        "rpc_result_timing": (C.c_int, [vp, C.POINTER(TimingC)]),
        "rpc_result_free": (None, [vp]),
        "rpc_kernel_columns": (C.c_int, [vp, vp, i64, i64, i64, C.c_int, KernelSpecC, vp, i64,
                                         vp, i64, pd]),
        "rpc_sample_discrete": (C.c_int, [vp, vp, i64, i64, C.c_uint64, C.c_uint64, C.c_int, vp]),
        "rpc_rejection_sweep": (C.c_int, [vp, vp, i64, vp, C.c_uint64, C.c_uint64, vp, vp, pi64,
                                          vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


_EXC = {RPC_EINVAL: ValueError, RPC_ERANGE: IndexError, RPC_ENUMERIC: RuntimeError,
        RPC_ECUDA: RuntimeError, RPC_ENCCL: RuntimeError, RPC_ENOMEM: MemoryError}


def check(rc: int, ctx=None) -> None:
    if rc != RPC_OK:
        msg = load().rpc_last_error(ctx).decode(errors="replace")
        raise _EXC.get(rc, RuntimeError)(msg)
