"""The reference's measurement harnesses on the GPU path.

* ``table1`` — the paper's Table 1 methodology (bench.py
  run_bench / run_read_baseline / run_noread_baseline, :196-307) on B200:
  elements/s of every method x precision x {sum, dot} at three tiers
  (small: launch/latency bound, medium: L2-resident, large: HBM), the
  read roofs (read1 = direct sum, read2 = direct dot: one add per element,
  the cheapest pass over the data) and the "noread" compute roofs
  (p-functions: the same recurrence fed from registers).
* ``run_accuracy_table`` / ``run_hours100`` / ``run_scaling_study`` —
  accuracy.py:73-173 with the reference's own LCG data generated on the
  device (bit-identical to lcg.fill), the GPU exact oracle and any flavor
  (default "cuda", the grid reduction).

Scores follow accuracy.py:66-70: twofold methods on value + error, the
others on value.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .api import Flavor, Method, _METHOD_ID, _dtype_code, reduce, run_flavor
from .exact import exact_sum, relative_error
from .gen import lcg_fill

_CUDA = Flavor.cuda()
_SEQ = Flavor.sequential()
_TWOFOLD = (Method.TWOFOLD_FAST, Method.TWOFOLD_RIGOROUS)
DTYPES = {"f32": torch.float32, "f64": torch.float64}
TIERS = {"small": 256 << 10, "medium": 32 << 20, "large": 2 << 30}  # bytes per operand


def _graph_time(fn, reps: int) -> float:
    """Seconds per call of fn, from one CUDA-graph replay of `reps` calls."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


@dataclass(frozen=True)
class KernelRow:
    """One Table-1 cell (bench.py KernelReport analogue)."""

    name: str          # paper row name: sumtf, dott, read1, psumt, ...
    method: str
    precision: str
    tier: str
    n: int
    seconds: float
    gelem_s: float     # paper convention: one add per element
    gbytes_s: float


_PAPER = {Method.DIRECT: "", Method.WIDE: "d", Method.TWOFOLD_FAST: "tf", Method.TWOFOLD_RIGOROUS: "t",
          Method.KAHAN: "k"}


def memory_rows(precisions=("f32", "f64"), tiers=("small", "medium", "large"), reps: int = 20,
                methods=tuple(Method), ops=("sum", "dot"), flavor: Flavor = _CUDA, seed: int = 1):
    """bench.run_bench (bench.py:196-247) on the device: every method x precision x
    tier x op, graph-timed; data = the reference's LCG streams (x: NR, y: MMIX)."""
    rows = []
    dev = torch.device("cuda", torch.cuda.current_device())
    for prec in precisions:
        dt = DTYPES[prec]
        item = torch.empty(0, dtype=dt).element_size()
        for tier in tiers:
            n = TIERS[tier] // item
            x = lcg_fill("nr", n, seed, dt, device=dev)
            y = lcg_fill("mmix", n, seed + 1, dt, device=dev) if "dot" in ops else None
            for method in methods:
                if method is Method.WIDE and prec != "f32":
                    continue
                for op, yy in (("sum", None), ("dot", y)):
                    if op not in ops:
                        continue
                    out = torch.empty(2, dtype=torch.float64 if method is Method.WIDE else dt, device=dev)
                    t = _graph_time(lambda: reduce(method, x, yy, flavor=flavor, out=out), reps)
                    nb = n * item * (1 if yy is None else 2)
                    rows.append(KernelRow(f"{op}{_PAPER[method]}", method.value, prec, tier, n, t, n / t / 1e9,
                                          nb / t / 1e9))
            del x, y
    return rows


def read_roofs(rows):
    """read1 / read2 = the direct sum / dot rows (one add per element)."""
    out = []
    for r in rows:
        if r.method == "direct":
            out.append(KernelRow("read1" if r.name == "sum" else "read2", r.method, r.precision, r.tier, r.n,
                                 r.seconds, r.gelem_s, r.gbytes_s))
    return out


def noread_rows(precisions=("f32", "f64"), iters: int = 4096, reps: int = 5, methods=tuple(Method)):
    """p-rows: the recurrence on register-resident addends (compute roof;
    bench.run_noread_baseline, bench.py:281-307)."""
    rows = []
    dev = torch.device("cuda", torch.cuda.current_device())
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks = sms * 8
    for prec in precisions:
        dt = DTYPES[prec]
        seed8 = torch.tensor([1.0 + 2.0 ** -(j + 3) for j in range(8)], dtype=dt, device=dev)
        for method in methods:
            if method is Method.WIDE and prec != "f32":
                continue
            for op, dot in (("sum", 0), ("dot", 1)):
                acc = torch.float64 if method is Method.WIDE else dt
                out = torch.empty(blocks * 256, 2, dtype=acc, device=dev)

                def launch():
                    check(lib().tf_noread(_METHOD_ID[method], _dtype_code(dt), dot, seed8.data_ptr(), iters, blocks,
                                          out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream), "tf_noread")
                _lib.ensure_canary(dev.index)
                t = _graph_time(launch, reps)
                n = blocks * 256 * iters * 8
                rows.append(KernelRow(f"p{op}{_PAPER[method]}", method.value, prec, "noread", n, t, n / t / 1e9, 0.0))
    return rows


def table1(reps: int = 20):
    mem = memory_rows(reps=reps)
    return mem + read_roofs(mem) + noread_rows()


def rows_markdown(rows) -> str:
    """One line per measurement (bench.bench_markdown analogue)."""
    lines = ["| row | method | precision | tier | n | us | Gelem/s | GB/s |", "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r.name} | {r.method} | {r.precision} | {r.tier} | {r.n} | {r.seconds * 1e6:.2f} | "
                     f"{r.gelem_s:.2f} | {r.gbytes_s:.1f} |")
    return "\n".join(lines) + "\n"


def rows_csv(rows) -> str:
    lines = ["row,method,precision,tier,n,seconds,gelem_s,gbytes_s"]
    for r in rows:
        lines.append(f"{r.name},{r.method},{r.precision},{r.tier},{r.n},{r.seconds!r},{r.gelem_s!r},{r.gbytes_s!r}")
    return "\n".join(lines) + "\n"


def run_selftest(pairs32: int = 10_000, pairs64: int = 2_000) -> list[str]:
    """selftest.run_selftest (selftest.py:18-63) against the DEVICE code: the
    strict-rounding canary, EFT exactness on random f32 / f64 pairs (vectorised
    through tf_eft), and the LCG recurrence constants of the device generator.
    Returns failure descriptions; empty means healthy."""
    from fractions import Fraction

    from .api import fast_two_sum, two_sum

    failures = []
    if lib().tf_canary() != _lib.TF_OK:
        failures.append("device canary: fast_two_sum(1, 2**-53) lost its round-off or a product was fused "
                        "into an FMA (value-unsafe code generation)")
    g = np.random.default_rng(12345)
    a32 = (g.uniform(-1, 1, pairs32) * 2.0 ** g.integers(-20, 20, pairs32)).astype(np.float32)
    b32 = (g.uniform(-1, 1, pairs32) * 2.0 ** g.integers(-20, 20, pairs32)).astype(np.float32)
    x, y = two_sum(a32, b32)
    x, y = np.asarray(x), np.asarray(y)
    bad = np.nonzero(x.astype(np.float64) + y.astype(np.float64) != a32.astype(np.float64) + b32.astype(np.float64))[0]
    if bad.size:
        i = int(bad[0])
        failures.append(f"two_sum inexact for f32 pair ({a32[i]!r}, {b32[i]!r})")
    swap = np.abs(a32) < np.abs(b32)
    hi, lo = np.where(swap, b32, a32), np.where(swap, a32, b32)
    xf, yf = (np.asarray(v) for v in fast_two_sum(hi, lo))
    xt, yt = (np.asarray(v) for v in two_sum(hi, lo))
    bad = np.nonzero((xf != xt) | (yf != yt))[0]
    if bad.size:
        i = int(bad[0])
        failures.append(f"fast_two_sum disagrees with two_sum on ({hi[i]!r}, {lo[i]!r})")
    a64 = g.uniform(-1, 1, pairs64) * 2.0 ** g.integers(-300, 300, pairs64)
    b64 = g.uniform(-1, 1, pairs64) * 2.0 ** g.integers(-300, 300, pairs64)
    x, y = (np.asarray(v) for v in two_sum(a64, b64))
    for i in range(pairs64):
        if Fraction(float(x[i])) + Fraction(float(y[i])) != Fraction(float(a64[i])) + Fraction(float(b64[i])):
            failures.append(f"two_sum inexact for f64 pair ({a64[i]!r}, {b64[i]!r})")
            break
    nr = float(lcg_fill("nr", 1, 0, torch.float64)[0])
    mx = float(lcg_fill("mmix", 1, 0, torch.float64)[0])
    if nr != 1013904223 / 2.0 ** 32 or mx != float(1442695040888963407) / 2.0 ** 64:
        failures.append("LCG recurrence constants are wrong")
    return failures


def format_table1(rows) -> str:
    """Markdown in the paper's layout: rows x (f32 small/medium/large, f64 ...) in Gelem/s."""
    cols = [(p, t) for p in ("f32", "f64") for t in ("small", "medium", "large", "noread")]
    names = []
    for r in rows:
        if r.name not in names:
            names.append(r.name)
    cell = {(r.name, r.precision, r.tier): r for r in rows}
    head = "| row | " + " | ".join(f"{p} {t}" for p, t in cols) + " |"
    lines = [head, "|---|" + "---|" * len(cols)]
    for nm in names:
        vals = []
        for p, t in cols:
            r = cell.get((nm, p, t))
            vals.append(f"{r.gelem_s:.1f}" if r else "")
        lines.append(f"| {nm} | " + " | ".join(vals) + " |")
    return "\n".join(lines)


# ---------------------------------------------------------------------------
# Accuracy experiments (accuracy.py:73-173) on device data + the GPU oracle.

@dataclass(frozen=True)
class AccuracyRow:
    precision: str
    generator: str
    interval: str
    method: str
    n: int
    seed: int
    rel_error: float
    valid: bool = True


@dataclass(frozen=True)
class Hours100Row:
    method: str
    result_hours: float
    deviation_hours: float
    estimate_hours: float | None = None


def _score(method: Method, res) -> float:
    if method in _TWOFOLD:
        return float(res.value) + float(res.error)
    return float(res.value)


DEFAULT_METHODS = (Method.DIRECT, Method.KAHAN, Method.TWOFOLD_FAST)


def run_accuracy_table(n: int = 1_000_000, seed: int = 1, methods=DEFAULT_METHODS, precisions=("f32", "f64"),
                       generators=("nr", "mmix"), intervals=("unit", "sym"), flavor: Flavor = _SEQ):
    """accuracy.run_accuracy_table (accuracy.py:73-103) on the GPU.  Default flavor:
    seq, the reference's (accuracy.py:97), so the table reproduces its numbers;
    flavor=Flavor.cuda() scores the grid reduction instead."""
    if n < 1:
        raise ValueError("n must be >= 1")
    rows = []
    for prec in precisions:
        dt = DTYPES[prec]
        for gen in generators:
            for interval in intervals:
                data = lcg_fill(gen, n, seed, dt, interval == "sym")
                ref = exact_sum(data)
                for method in methods:
                    if method is Method.WIDE and prec != "f32":
                        continue
                    res = run_flavor(method, flavor, data)
                    score = _score(method, res)
                    valid = math.isfinite(score) and not ref.is_zero
                    rel = relative_error(score, ref) if valid else math.nan
                    rows.append(AccuracyRow(prec, gen, interval, method.value, n, seed, rel, valid))
    return rows


def run_hours100(flavor: Flavor = Flavor.sequential()):
    """accuracy.run_hours100 (accuracy.py:106-136); seq reproduces the reference's goldens."""
    ticks = 3_600_000
    data = torch.full((ticks,), 0.1, dtype=torch.float32, device="cuda")

    def dev(h):
        return abs(100.0 - h)

    rows = []
    d = run_flavor(Method.DIRECT, flavor, data)
    h = float(d.value) / 3600.0
    rows.append(Hours100Row("direct", h, dev(h)))
    w = run_flavor(Method.WIDE, flavor, data)
    h = float(w.value) / 3600.0
    rows.append(Hours100Row("wide", h, dev(h)))
    k = run_flavor(Method.KAHAN, flavor, data)
    h = float(k.value) / 3600.0
    rows.append(Hours100Row("kahan", h, dev(h)))
    t = run_flavor(Method.TWOFOLD_FAST, flavor, data)
    h = (float(t.value) + float(t.error)) / 3600.0
    rows.append(Hours100Row("twofold-fast", h, dev(h), estimate_hours=float(t.error) / 3600.0))
    return rows


def run_scaling_study(ns=(10 ** 3, 10 ** 4, 10 ** 5, 10 ** 6), trials: int = 100, seed: int = 1,
                      methods=(Method.DIRECT, Method.TWOFOLD_FAST), flavor: Flavor = _SEQ,
                      generator: str = "nr"):
    """Median |relative error| vs N over seeded binary32 trials (trial t draws
    uniform [0,1) data from seed + t) and the fitted log-log slope per method,
    as accuracy.run_scaling_study (accuracy.py:139-173): direct scored on value,
    twofold on value + error, no slope for a method with an exact-zero median.
    Default flavor seq (the reference's, :159)."""
    out = []
    medians = {m: [] for m in methods}
    for n in ns:
        errs = {m: [] for m in methods}
        for t in range(trials):
            data = lcg_fill(generator, n, seed + t, torch.float32)
            ref = exact_sum(data)
            for m in methods:
                errs[m].append(abs(relative_error(_score(m, run_flavor(m, flavor, data)), ref)))
        for m in methods:
            med = float(np.median(errs[m]))
            medians[m].append(med)
            out.append((n, m.value, med))
    slopes = {}
    logn = np.log10(np.asarray(ns, float))
    for m in methods:
        med = np.asarray(medians[m])
        slopes[m.value] = (float(np.polyfit(logn, np.log10(med), 1)[0])
                           if len(ns) >= 2 and np.all(med > 0) else None)
    return out, slopes


__all__ = ["KernelRow", "table1", "memory_rows", "noread_rows", "read_roofs", "format_table1", "rows_markdown",
           "rows_csv", "run_selftest", "AccuracyRow", "Hours100Row", "run_accuracy_table", "run_hours100",
           "run_scaling_study"]
