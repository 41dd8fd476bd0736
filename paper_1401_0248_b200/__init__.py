"""B200-native (sm_100a) twofold (value + error) summation and dot product.

Drop-in for the hot path of the reference package `twofold` (arXiv 1401.0248,
pkg/src/twofold/__init__.py:11-42): the same Method / Flavor / SumResult /
Twofold types, run_flavor and the ten sum_* / dot_* wrappers, the EFT
primitives and the canary, the Expansion oracle API (exact_sum / exact_dot /
expansion_add / relative_error) and the LCG data API (LcgKind, LcgState,
next_raw, uniform01, uniform_sym, fill) — computed by hand-written CUDA
kernels behind a C ABI (include/twofold_b200.h).  New surface: the "cuda"
flavor (grid reduction; the wrappers default to the reference's "seq" bits,
see set_default_flavor), batched row-wise sums/dots, seeded on-device
Philox inputs and the contiguous multi-GPU shard layer.

Like the reference (kernels.py:559-568), importing the package checks strict
rounding: when a CUDA device is visible the device canary runs at import and
a value-unsafe build raises RuntimeError.
"""

from .api import (
    Flavor,
    Method,
    RowsResult,
    SumResult,
    Twofold,
    default_flavor,
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
    set_default_flavor,
    sum_direct,
    sum_kahan,
    sum_rows,
    sum_twofold_fast,
    sum_twofold_rigorous,
    sum_wide,
    two_sum,
    using_flavor,
    workspace_size,
)
from .dist import combine_in_use, peer_combine_error, rows_range, shard_range, sharded_reduce, sharded_rows, sharded_run
from .exact import ExactValue, Expansion, exact_dot, exact_sum, expansion_add, relative_error
from .gen import CONFIGS, lcg_fill, make_inputs, philox_fill, philox_fill_host, rows_scaled_normal
from .lcg import LcgKind, LcgState, fill, next_raw, raw_to_uniform, uniform01, uniform_sym

__version__ = "0.2.0"

__all__ = [
    "Twofold", "fast_two_sum", "two_sum", "rounding_canary",
    "Expansion", "ExactValue", "exact_sum", "exact_dot", "expansion_add", "relative_error",
    "Method", "Flavor", "SumResult", "RowsResult", "run_flavor", "raw_sum_kernel",
    "default_flavor", "set_default_flavor", "using_flavor",
    "sum_direct", "sum_wide", "sum_twofold_fast", "sum_twofold_rigorous", "sum_kahan",
    "dot_direct", "dot_wide", "dot_twofold_fast", "dot_twofold_rigorous", "dot_kahan",
    "LcgKind", "LcgState", "next_raw", "raw_to_uniform", "uniform01", "uniform_sym", "fill",
    "reduce", "reduce_rows", "sum_rows", "dot_rows", "merge_pairs", "workspace_size", "leaf_log2_for",
    "shard_range", "sharded_reduce", "sharded_run", "combine_in_use", "peer_combine_error",
    "rows_range", "sharded_rows",
    "philox_fill", "philox_fill_host", "lcg_fill", "rows_scaled_normal", "make_inputs", "CONFIGS",
    "__version__",
]


def _import_canary() -> None:
    """kernels.py:559-568: refuse to import on a value-unsafe build.  Without a
    CUDA device nothing can run (every compute call raises), so there is
    nothing to check until one is visible; ensure_canary also runs per device
    on first use."""
    import os

    import torch

    from . import _lib
    if torch.cuda.is_available():
        # under torchrun each rank owns GPU LOCAL_RANK: check that one rather than
        # creating a context on device 0 in every rank
        local = os.environ.get("LOCAL_RANK")
        dev = int(local) if local is not None and local.isdigit() and int(local) < torch.cuda.device_count() \
            else torch.cuda.current_device()
        _lib.ensure_canary(dev)


_import_canary()
