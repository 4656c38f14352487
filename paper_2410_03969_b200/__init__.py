"""B200-native accelerated randomly pivoted Cholesky (arXiv 2410.03969).

The product is librpchol_b200.so (paper_2410_03969_b200/csrc, C-ABI in
include/rpchol_gpu.h).  `api` mirrors the reference's hot-path API
(KernelOracle, RunConfig, accelerated_rpcholesky) over that C-ABI.
"""
from .api import (CholeskyResult, Context, KernelOracle, KernelSpec, RunConfig,  # noqa: F401
                  accelerated_rpcholesky, accelerated_rpcholesky_device, nccl_unique_id,
                  rejection_sample_submatrix, relative_trace_error, sample_discrete)
