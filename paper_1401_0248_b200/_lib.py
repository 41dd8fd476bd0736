"""ctypes binding of the in-tree C-ABI library libtwofold_b200.so.

The library is the only compute path of this package: if it is missing or
the device canary fails, every call raises — there is no CPU fallback.
Status codes map to the reference's exception types (kernels.py:574-584,
:600-601, :559-565): DTYPE -> TypeError, SHAPE/ARG/METHOD -> ValueError,
CANARY/CUDA/WORKSPACE -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# TFB_LIB overrides the path (tuning sweeps over build variants only).
LIB_PATH = os.environ.get("TFB_LIB") or os.path.join(_HERE, "libtwofold_b200.so")

TF_OK = 0
TF_EINVAL_METHOD, TF_EINVAL_DTYPE, TF_EINVAL_SHAPE, TF_EINVAL_ARG = 1, 2, 3, 4
TF_EWORKSPACE, TF_ECUDA, TF_ECANARY = 5, 6, 7

TF_F32, TF_F64 = 0, 1
DIST_UNIFORM01, DIST_UNIFORM_SYM, DIST_NORMAL, DIST_ILLCOND = 0, 1, 2, 3

_lock = threading.Lock()
_lib = None
_canary_ok: set[int] = set()


def _bind(L):
    vp, i64, i32, u64, sz, dbl = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64,
                                  ctypes.c_size_t, ctypes.c_double)
    sig = {
        "tf_version": ([], i32),
        "tf_strerror": ([i32], ctypes.c_char_p),
        "tf_last_cuda_error": ([], ctypes.c_char_p),
        "tf_launch_count": ([], ctypes.c_uint64),
        "tf_canary": ([], i32),
        "tf_leaf_log2": ([i32, i64], i32),
        "tf_set_leaf_split": ([i32], i32),
        "tf_set_loader": ([i32], i32),
        "tf_set_tail": ([i32], i32),
        "tf_set_prefetch": ([i32], i32),
        "tf_set_rows_kernel": ([i32], i32),
        "tf_last_launch": ([], ctypes.c_char_p),
        "tf_workspace_size": ([i32, i32, i64, i64, i32, ctypes.POINTER(sz), ctypes.POINTER(i64),
                               ctypes.POINTER(i64)], i32),
        "tf_reduce": ([i32, i32, vp, vp, i64, i32, vp, vp, sz, vp, i64, vp], i32),
        "tf_reduce_peer": ([i32, i32, vp, vp, i64, i32, vp, vp, sz, vp, i64, vp, ctypes.c_uint32, vp], i32),
        "tf_peer_ctx_size": ([], i32),
        "tf_reduce_rows": ([i32, i32, vp, vp, i64, i64, i64, i64, i32, vp, vp, sz, vp, i64, vp], i32),
        "tf_reduce_leaves": ([i32, i32, vp, vp, i64, i32, vp, vp], i32),
        "tf_merge_tree": ([i32, i32, vp, i64, vp, vp], i32),
        "tf_reduce_seq": ([i32, i32, vp, vp, i64, vp, vp], i32),
        "tf_reduce_lanes": ([i32, i32, vp, vp, i64, i32, vp, vp], i32),
        "tf_eft": ([i32, i32, vp, vp, i64, vp, vp, vp], i32),
        "tf_fill": ([i32, i32, u64, u64, u64, i64, dbl, dbl, dbl, i64, vp, vp], i32),
        "tf_read_roof": ([vp, i64, i32, vp, vp], i32),
        "tf_noread": ([i32, i32, i32, vp, i64, i64, vp, vp], i32),
        "tf_exact_workspace": ([ctypes.POINTER(i64), ctypes.POINTER(sz)], i32),
        "tf_exact": ([i32, vp, vp, i64, i32, vp, vp, vp, sz, vp, vp], i32),
        "tf_fill_host": ([i32, i32, u64, u64, u64, i64, dbl, dbl, dbl, i64, vp, i32], i32),
        "tf_lcg_fill": ([i32, i32, u64, i32, i64, i64, vp, vp], i32),
        "tf_fill_rows_scaled": ([i32, u64, u64, u64, i64, i64, i64, i64, dbl, dbl, vp, vp], i32),
        "tf_host_engine_create": ([i32, i32, sz, ctypes.POINTER(vp)], i32),
        "tf_host_engine_destroy": ([vp], i32),
        "tf_host_engine_threads": ([vp], i32),
        "tf_host_reduce": ([vp, i32, i32, vp, vp, i64, i32, vp, vp], i32),
        "tf_host_reduce_rows": ([vp, i32, i32, vp, vp, i64, i64, i64, i64, i32, vp, vp], i32),
        "tf_host_engine_hybrid": ([vp, i32, sz], i32),
        "tf_host_engine_last_split": ([vp, ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
        "tf_host_leaves": ([i32, i32, vp, vp, i64, i32, i64, i64, vp], i32),
        "tf_host_rows": ([i32, i32, vp, vp, i64, i64, i64, i64, i32, i64, i64, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


def lib():
    """Load the library (no GPU needed to load; compute calls need one)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                        "g.build()'` (or make -C paper_1401_0248_b200/csrc); there is no CPU fallback")
                _lib = _bind(ctypes.CDLL(LIB_PATH))
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == TF_OK:
        return
    L = lib()
    msg = L.tf_strerror(rc).decode()
    if what:
        msg = f"{what}: {msg}"
    if rc == TF_EINVAL_DTYPE:
        raise TypeError(msg)
    if rc in (TF_EINVAL_SHAPE, TF_EINVAL_ARG, TF_EINVAL_METHOD):
        raise ValueError(msg)
    if rc == TF_ECUDA:
        raise RuntimeError(f"{msg} ({L.tf_last_cuda_error().decode()})")
    raise RuntimeError(msg)


def ensure_canary(device_index: int) -> None:
    """Run the device strict-rounding canary once per device (kernels.py:559-568)."""
    if device_index in _canary_ok:
        return
    import torch
    with torch.cuda.device(device_index):
        rc = lib().tf_canary()
    if rc == TF_ECANARY:
        raise RuntimeError(
            "compiled kernels violate strict IEEE rounding (device canary: fast_two_sum(1, 2**-53) "
            "lost its round-off or a product was fused into an FMA); the library is unusable for "
            "error tracking")
    check(rc, "tf_canary")
    _canary_ok.add(device_index)


_engines: dict = {}
_default_engines: dict = {}


def host_split(engine) -> tuple[int, int]:
    """(elements the GPU reduced, elements the host workers reduced) in the engine's last call."""
    a, b = ctypes.c_int64(0), ctypes.c_int64(0)
    check(lib().tf_host_engine_last_split(engine, ctypes.byref(a), ctypes.byref(b)), "tf_host_engine_last_split")
    return a.value, b.value


def host_engine(device_index: int, chunk_bytes: int | None = None, threads: int | None = None):
    """The host-buffer engine (tf_host_engine_create) for one device and
    configuration, created once.  Defaults: TFB_HOST_THREADS (0 = auto) and
    TFB_HOST_CHUNK_MB (0 = 16 MiB per operand per slot)."""
    if chunk_bytes is None and threads is None:
        eng = _default_engines.get(device_index)
        if eng is not None:
            return eng
        eng = host_engine(device_index, int(os.environ.get("TFB_HOST_CHUNK_MB", "0")) << 20,
                          int(os.environ.get("TFB_HOST_THREADS", "0")))
        _default_engines[device_index] = eng
        return eng
    if threads is None:
        threads = int(os.environ.get("TFB_HOST_THREADS", "0"))
    if chunk_bytes is None:
        chunk_bytes = int(os.environ.get("TFB_HOST_CHUNK_MB", "0")) << 20
    key = (device_index, chunk_bytes, threads)
    eng = _engines.get(key)
    if eng is None:
        L = lib()  # load outside _lock: lib() takes the same (non-reentrant) lock on first use
        with _lock:
            eng = _engines.get(key)
            if eng is None:
                eng = ctypes.c_void_p()
                rc = L.tf_host_engine_create(device_index, threads, chunk_bytes, ctypes.byref(eng))
                if rc:
                    raise RuntimeError(f"tf_host_engine_create: {L.tf_strerror(rc).decode()} "
                                       f"({L.tf_last_cuda_error().decode()})")
                _engines[key] = eng
    return eng
