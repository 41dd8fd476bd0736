"""Seeded on-device input generation (Philox4x32-10) for the BASELINE.json configs.

Element i of stream `stream` under key `seed` depends only on (seed, stream,
i), so a rank that owns the global slice [offset, offset+n) produces exactly
the bytes a single GPU would — data is independent of the GPU count.  The
reference generates inputs with LCGs (lcg.py:75-116); BASELINE.json replaces
them with Philox streams.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check, lib

_DIST = {"uniform01": _lib.DIST_UNIFORM01, "uniform_sym": _lib.DIST_UNIFORM_SYM,
         "normal": _lib.DIST_NORMAL, "illcond": _lib.DIST_ILLCOND}


def _dev(device) -> torch.device:
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def philox_fill(dist: str, n: int, *, seed: int, stream: int = 0, offset: int = 0,
                dtype: torch.dtype = torch.float64, device=None, params=(1e8, 9e8, 1e-3),
                total: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Fill n elements [offset, offset+n) of a Philox stream.

    dist: "uniform01" [0,1), "uniform_sym" [-1,1), "normal" N(0,1) (Box-Muller),
    "illcond" (cfg3: a keyed permutation of `total` positions holding +-b_k pairs,
    b_k = p0 + p1*u, and a half of p2*u; the exact sum is the small half's).
    """
    dev = _dev(device)
    if out is None:
        out = torch.empty(n, dtype=dtype, device=dev)
    code = _lib.TF_F32 if out.dtype == torch.float32 else _lib.TF_F64
    tot = total if total is not None else offset + n
    with torch.cuda.device(dev):
        check(lib().tf_fill(_DIST[dist], code, seed, stream, offset, n, params[0], params[1], params[2], tot,
                            out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream), "tf_fill")
    return out


def philox_fill_host(dist: str, n: int, *, seed: int, stream: int = 0, offset: int = 0,
                     dtype: torch.dtype = torch.float64, params=(1e8, 9e8, 1e-3), total: int | None = None,
                     pin_memory: bool = False, nthreads: int = 0) -> torch.Tensor:
    """Host (CPU) twin of philox_fill for the integer-exact distributions:
    bit-identical bytes in a host tensor (optionally pinned, for e2e inputs)."""
    if dist not in ("uniform01", "uniform_sym", "illcond"):
        raise ValueError("the host twin covers uniform01, uniform_sym and illcond")
    out = torch.empty(n, dtype=dtype, pin_memory=pin_memory)
    code = _lib.TF_F32 if dtype == torch.float32 else _lib.TF_F64
    tot = total if total is not None else offset + n
    check(lib().tf_fill_host(_DIST[dist], code, seed, stream, offset, n, params[0], params[1], params[2], tot,
                             out.data_ptr(), nthreads), "tf_fill_host")
    return out


def lcg_fill(kind: str, n: int, seed: int = 1, dtype: torch.dtype = torch.float64, sym: bool = False, *,
             offset: int = 0, device=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """The reference's LCG data on the device, bit-identical to
    twofold.fill(LcgKind(kind), offset + n, seed, dtype, sym)[offset:] (lcg.py:108-116).
    kind: "nr" (Numerical Recipes, 32-bit) or "mmix" (64-bit)."""
    if kind not in ("nr", "mmix"):
        raise ValueError(f"unknown LCG kind {kind!r}")
    dev = _dev(device)
    if out is None:
        out = torch.empty(n, dtype=dtype, device=dev)
    code = _lib.TF_F32 if out.dtype == torch.float32 else _lib.TF_F64
    with torch.cuda.device(dev):
        check(lib().tf_lcg_fill(0 if kind == "nr" else 1, code, seed, 1 if sym else 0, offset, n, out.data_ptr(),
                                torch.cuda.current_stream(dev).cuda_stream), "tf_lcg_fill")
    return out


def rows_scaled_normal(rows: int, cols: int, *, seed: int, stream: int, scale_stream: int = 2,
                       row0: int = 0, lo: float = -4.0, hi: float = 4.0,
                       dtype: torch.dtype = torch.float32, device=None) -> torch.Tensor:
    """cfg4 matrix: N(0,1) entries, row r scaled by 10^U_r, U_r ~ U[lo, hi) drawn once
    per row from `scale_stream` (so x and y of the same row share the scale)."""
    dev = _dev(device)
    out = torch.empty(rows, cols, dtype=dtype, device=dev)
    code = _lib.TF_F32 if dtype == torch.float32 else _lib.TF_F64
    with torch.cuda.device(dev):
        check(lib().tf_fill_rows_scaled(code, seed, stream, scale_stream, row0, rows, cols, cols, lo, hi,
                                        out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
              "tf_fill_rows_scaled")
    return out


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration (the bench workload or a parity case)."""

    name: str
    op: str            # "sum" | "dot" | "rows-dot"
    dtype: torch.dtype
    n: int             # elements (rows*cols for rows configs)
    seed: int
    dist: str
    methods: tuple     # method names run on this config
    rows: int = 0
    cols: int = 0
    note: str = ""


CONFIGS = {
    "cfg1": Config("cfg1", "sum", torch.float64, 1 << 20, 0, "uniform01", ("twofold-fast",),
                   note="fp64 sumtf N=2^20 U[0,1) seed 0 (L2-resident, latency-bound)"),
    "cfg2": Config("cfg2", "dot", torch.float32, 1 << 24, 1, "normal", ("twofold-fast", "twofold-rigorous"),
                   note="fp32 dottf/dott N=2^24 N(0,1) seed 1"),
    "cfg2-small": Config("cfg2-small", "dot", torch.float32, 1 << 16, 1, "normal",
                         ("twofold-fast", "twofold-rigorous"), note="first 2^16 of cfg2's streams"),
    "cfg3": Config("cfg3", "sum", torch.float64, 1 << 28, 2, "illcond", ("twofold-rigorous", "kahan"),
                   note="fp64 sumt/sumk N=2^28 ill-conditioned, exact sum known by construction"),
    "cfg4": Config("cfg4", "rows-dot", torch.float32, 4096 * 65536, 3, "rows-normal", ("twofold-fast",),
                   rows=4096, cols=65536, note="fp32 row-wise dottf 4096x65536, rows scaled by 10^U[-4,4)"),
    "cfg5": Config("cfg5", "dot", torch.float64, 1 << 32, 4, "uniform_sym", ("twofold-fast",),
                   note="fp64 dottf N=2^32 U[-1,1) seed 4, contiguous shards"),
}


def make_inputs(cfg: Config, *, device=None, offset: int = 0, n: int | None = None):
    """Generate (x, y) for a config (y None for sums); `offset`/`n` select a
    contiguous global slice (shards).  Stream ids: x = 0, y = 1, row scales = 2."""
    dev = _dev(device)
    if cfg.op == "rows-dot":
        rows = n // cfg.cols if n is not None else cfg.rows
        row0 = offset // cfg.cols
        x = rows_scaled_normal(rows, cfg.cols, seed=cfg.seed, stream=0, scale_stream=2, row0=row0,
                               dtype=cfg.dtype, device=dev)
        y = rows_scaled_normal(rows, cfg.cols, seed=cfg.seed, stream=1, scale_stream=2, row0=row0,
                               dtype=cfg.dtype, device=dev)
        return x, y
    cnt = cfg.n - offset if n is None else n
    x = philox_fill(cfg.dist, cnt, seed=cfg.seed, stream=0, offset=offset, dtype=cfg.dtype, device=dev,
                    total=cfg.n)
    y = None
    if cfg.op == "dot":
        y = philox_fill(cfg.dist, cnt, seed=cfg.seed, stream=1, offset=offset, dtype=cfg.dtype, device=dev,
                        total=cfg.n)
    return x, y
