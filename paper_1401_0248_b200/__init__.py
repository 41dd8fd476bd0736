"""B200-native (sm_100a) twofold (value + error) summation and dot product.

Drop-in for the hot path of the reference package `twofold` (arXiv 1401.0248,
pkg/src/twofold/__init__.py): the same Method / Flavor / SumResult /
Twofold types, run_flavor and the ten sum_* / dot_* wrappers, the EFT
primitives and the canary — computed by hand-written CUDA kernels behind a
C ABI (include/twofold_b200.h).  New surface: the "cuda" flavor (grid
reduction, default for the wrappers), batched row-wise sums/dots, seeded
on-device Philox inputs and the contiguous multi-GPU shard layer.
"""

from .api import (
    Flavor,
    Method,
    RowsResult,
    SumResult,
    Twofold,
    dot_direct,
    dot_kahan,
    dot_rows,
    dot_twofold_fast,
    dot_twofold_rigorous,
    dot_wide,
    fast_two_sum,
    leaf_log2_for,
    merge_pairs,
    raw_sum_kernel,
    reduce,
    reduce_rows,
    rounding_canary,
    run_flavor,
    sum_direct,
    sum_kahan,
    sum_rows,
    sum_twofold_fast,
    sum_twofold_rigorous,
    sum_wide,
    two_sum,
    workspace_size,
)
from .dist import combine_in_use, peer_combine_error, rows_range, shard_range, sharded_reduce, sharded_rows, sharded_run
from .exact import ExactValue, exact_dot, exact_sum, relative_error
from .gen import CONFIGS, lcg_fill, make_inputs, philox_fill, philox_fill_host, rows_scaled_normal

__version__ = "0.1.0"

__all__ = [
    "Twofold", "fast_two_sum", "two_sum", "rounding_canary",
    "Method", "Flavor", "SumResult", "RowsResult", "run_flavor", "raw_sum_kernel",
    "sum_direct", "sum_wide", "sum_twofold_fast", "sum_twofold_rigorous", "sum_kahan",
    "dot_direct", "dot_wide", "dot_twofold_fast", "dot_twofold_rigorous", "dot_kahan",
    "reduce", "reduce_rows", "sum_rows", "dot_rows", "merge_pairs", "workspace_size", "leaf_log2_for",
    "shard_range", "sharded_reduce", "sharded_run", "combine_in_use", "peer_combine_error",
    "rows_range", "sharded_rows",
    "ExactValue", "exact_sum", "exact_dot", "relative_error",
    "philox_fill", "philox_fill_host", "lcg_fill", "rows_scaled_normal", "make_inputs", "CONFIGS",
    "__version__",
]
