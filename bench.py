"""Benchmark: twofold sum/dot throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg5]

Default workload: BASELINE.json configs[4] exactly as stated — fp64
twofold-fast dot (dottf) of two N = 2^32 U[-1,1) Philox streams (seed 4),
N fixed and split contiguously over the ranks (rank r of G owns
[r*N/G, (r+1)*N/G), generated at that global offset, so the data never
depends on G).  At --gpus 1 that is the whole 2 x 32 GiB on one B200; at 8
it is 2^29 elements per GPU.  `--config cfg5-weak` keeps 2^29 elements per
rank instead (weak scaling).  A step = one pass of the hot path over the
rank's shard: the fused leaf+tree reduction kernel, and for N>1 the NCCL
all-gather of the 16-byte (v, e) pairs plus the merge kernel.  Inputs are
>= 68x the 126 MB L2 (no flush needed); the small configs (--config
cfg1/cfg2/cfg2-small) rotate over input copies >= 4x L2.

Launch: `--gpus N` without a torchrun environment re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` (the driver's own
launch line), so `python bench.py --gpus 8` runs 8 ranks; under torchrun
(WORLD_SIZE set) it runs as one rank.  Rank 0 prints ONE JSON line: value =
elements/s over all ranks (device-timed with CUDA events, max over ranks),
e2e = the same through the public API from pinned host buffers (H2D + reduce
+ D2H of the pair each step), roofline of the reduction kernel from the same
timed window, cpu_baseline = the oracle's port of the reference recurrence
on this host (the same routine as the reference arm).  --impl reference runs
that CPU port alone on rank 0 (the reference arm).  --dry-run exercises the
launcher and the process group on CPU (gloo) without touching a GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "twofold sum/dot Gelem/s & HBM GB/s vs roofline at 1/2/4/8 B200, fp32/fp64"
UNIT = "Gelem/s"
PER_RANK = 1 << 29          # cfg5-weak: elements per rank (N=8 is cfg5 in full)
CPU_SAMPLE = 1 << 29        # CPU baselines: at most the rank-0 slice of this many elements
SINGLE_CORE_SAMPLE = 1 << 24

WORKLOADS = {
    # name: (config key, method, per-rank layout, needs L2 rotation)
    #   "split": the config's N split evenly over the ranks (strong scaling)
    #   int:     that many elements per rank at offset rank*int (weak scaling)
    #   None:    the whole config on every rank (small single-GPU configs)
    "cfg5": ("cfg5", "twofold-fast", "split", False),
    "cfg5-weak": ("cfg5", "twofold-fast", PER_RANK, False),
    "cfg1": ("cfg1", "twofold-fast", None, True),
    "cfg2": ("cfg2", "twofold-fast", None, True),
    "cfg2-dott": ("cfg2", "twofold-rigorous", None, True),
    "cfg2-small": ("cfg2-small", "twofold-fast", None, True),
    "cfg3": ("cfg3", "twofold-rigorous", None, False),
    "cfg3-sumk": ("cfg3", "kahan", None, False),
    "cfg4": ("cfg4", "twofold-fast", None, False),
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--leaf-log2", type=int, default=0, help="override the auto leaf size (sweeps)")
    ap.add_argument("--graph", action="store_true", help="replay the timed steps from a CUDA graph")
    ap.add_argument("--combine", default="nccl", choices=["nccl", "peer", "auto"],
                    help="cross-rank combine: NCCL all-gather + merge kernel (default), the fused NVLink "
                         "peer combine (tf_reduce_peer), or auto (peer after a one-time self-check)")
    ap.add_argument("--force-collective", action="store_true",
                    help="init NCCL and run the all-gather + merge path even at world size 1 (plumbing check)")
    ap.add_argument("--spawn", action="store_true",
                    help="re-exec under torch.distributed.run even at --gpus 1 (exercises the launcher)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher + process-group plumbing only, on CPU (gloo); no GPU work, value 0")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# Launcher

def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int | None:
    """Without a torchrun environment, `--gpus N` re-executes this script under
    torch.distributed.run with N local ranks (exactly the driver's launch line);
    returns the launcher's exit code, or None to run in this process."""
    if "WORLD_SIZE" in os.environ or "TFB_BENCH_CHILD" in os.environ:
        return None
    if args.gpus <= 1 and not args.spawn:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    env = dict(os.environ, TFB_BENCH_CHILD="1")
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env).returncode


def dist_env() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------------------
# Descriptions shared by both arms (identical `config` dicts)

def layout(name: str, cfg, world: int, rank: int):
    """(elements on this rank, global offset of its slice, elements all ranks process per step)."""
    per = WORKLOADS[name][2]
    if per == "split":
        lo, hi = (rank * cfg.n) // world, ((rank + 1) * cfg.n) // world
        return hi - lo, lo, cfg.n
    if isinstance(per, int):
        return per, rank * per, per * world
    return cfg.n, 0, cfg.n * world


def workload_desc(name, cfg, method, world):
    per = WORKLOADS[name][2]
    n_rank0 = layout(name, cfg, world, 0)[0]
    if per == "split":
        shape = (f"N = 2^{cfg.n.bit_length() - 1} fixed, split contiguously over {world} rank(s): "
                 f"rank r owns [r*N/{world}, (r+1)*N/{world}) at that Philox offset")
    elif isinstance(per, int):
        shape = (f"{per} elements per rank, rank r owns [r*{per}, (r+1)*{per}) of the cfg5 stream "
                 "(weak scaling; N=8 is cfg5 in full)")
    else:
        shape = "the whole config on each rank"
    return {
        "workload": f"{name}: {cfg.note}; {method}; {shape}",
        "op": cfg.op, "method": method, "n_global": layout(name, cfg, world, 0)[2], "n_per_rank": n_rank0,
        "data_dtype": "f64" if str(cfg.dtype).endswith("64") else "f32",
        "generator": f"Philox4x32-10 seed {cfg.seed} (x stream 0, y stream 1)",
        "parallelism": ("single GPU" if world == 1 else
                        (f"dp{world}: contiguous row blocks per rank, no collective" if cfg.op == "rows-dot" else
                         f"dp{world}: contiguous shards + NCCL all-gather of (v,e) pairs + TwoSum merge")),
    }


def scaling_kind(name: str, world: int) -> str:
    per = WORKLOADS[name][2]
    return "strong" if per == "split" or (per is None and world > 1 and name == "cfg4") else "weak"


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # NVML missing: report nothing rather than guess
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def report(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def bind_to_gpu_numa(local: int) -> str | None:
    """Multi-GPU ranks: run on the CPUs NVML reports as local to this GPU, so the
    pinned e2e shard is first-touched on the GPU's NUMA node (its own PCIe root)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * w + b for w, word in enumerate(words) for b in range(64) if (int(word) >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return f"{len(cpus)} GPU-local CPUs"
    except Exception:
        return None
    return None


def _numa_nodes() -> int:
    try:
        return max(1, len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")]))
    except OSError:
        return 1


def measured_peak():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_for(name):
    path = os.path.join(REPO, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(name)
    except Exception:
        return None


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _thp() -> str:
    try:
        with open("/sys/kernel/mm/transparent_hugepage/enabled") as f:
            return f.read().strip()
    except OSError:
        return "unknown"


# ---------------------------------------------------------------------------
# CPU baseline: ONE routine for the reference arm and the cpu_baseline leg

def cpu_sample(name: str, cfg, n_sample: int, nt: int):
    """The bounded CPU sample of the workload as numpy buffers: the rank-0 slice
    [0, n_sample), bit-identical to the device data for the Philox
    distributions (host twin), first-touched by the same pinned threads that
    later stream it (NUMA-local pages).  Normals (cfg2) have no bit-exact
    host twin: a numpy stand-in of the same distribution."""
    from oracle import oracle as O
    O.lib().tfo_set_pin(1)
    dt = np.float64 if str(cfg.dtype).endswith("64") else np.float32
    if cfg.dist in ("uniform01", "uniform_sym"):
        xh = O.philox_fill(cfg.dist, n_sample, cfg.seed, 0, 0, dt, nthreads=nt)
        yh = O.philox_fill(cfg.dist, n_sample, cfg.seed, 1, 0, dt, nthreads=nt) if cfg.op != "sum" else None
        what = f"rank-0 slice [0, {n_sample}) of the workload, Philox host twin (bit-identical to the device data)"
    elif cfg.dist == "illcond":
        xh = O.philox_fill("illcond", n_sample, cfg.seed, 0, 0, dt, total=cfg.n, nthreads=nt)
        yh = None
        what = f"{n_sample} elements of the cfg3 layout, Philox host twin"
    else:
        rng = np.random.default_rng(cfg.seed)
        xh = rng.standard_normal(n_sample).astype(dt)
        yh = rng.standard_normal(n_sample).astype(dt)
        what = f"{n_sample} elements N(0,1) (numpy stand-in with the config's distribution)"
    return xh, yh, what


def cpu_rows_sample(cfg):
    dt = np.float32 if cfg.dtype.__str__().endswith("32") else np.float64
    rng = np.random.default_rng(cfg.seed)
    scale = (10.0 ** rng.uniform(-4, 4, (cfg.rows, 1))).astype(dt)
    X = (rng.standard_normal((cfg.rows, cfg.cols)) * scale).astype(dt)
    Y = (rng.standard_normal((cfg.rows, cfg.cols)) * scale).astype(dt)
    return X, Y


def cpu_steps(mid: int, xh, yh, nt: int, steps: int, warmup: int):
    """W untimed + K timed passes of the reference recurrence on nt pinned threads
    (contiguous shards, each the seq recurrence, shard pairs merged with the
    lane merge).  Returns the per-step seconds."""
    from oracle import oracle as O
    O.lib().tfo_set_pin(1)
    for _ in range(warmup):
        O.threads(mid, xh, yh, nt)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.threads(mid, xh, yh, nt)
        times.append(time.perf_counter() - t0)
    return times


def cpu_rows_steps(mid: int, X, Y, nt: int, steps: int, warmup: int):
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    rows = X.shape[0]
    chunks = [((i * rows) // nt, ((i + 1) * rows) // nt) for i in range(nt)]

    def work(c):
        for r in range(*c):
            O.seq(mid, X[r], None if Y is None else Y[r])

    times = []
    with ThreadPoolExecutor(nt) as ex:
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            list(ex.map(work, chunks))
            if i >= warmup:
                times.append(time.perf_counter() - t0)
    return times


def single_core(mid: int, xh, yh):
    """The reference's own single-thread methodology (bench.py:82-89 pin_to_one_core,
    :104-130 _time_best_of: inner repeats doubled until one sample takes >= 10 ms,
    one warm-up sample, best of 5) on this thread, pinned to the first allowed CPU."""
    from oracle import oracle as O
    n = min(xh.shape[0], SINGLE_CORE_SAMPLE)
    x = xh[:n]
    y = None if yh is None else yh[:n]
    old = os.sched_getaffinity(0)
    try:
        os.sched_setaffinity(0, {min(old)})
        inner = 1
        while True:
            t0 = time.perf_counter()
            for _ in range(inner):
                O.seq(mid, x, y)
            if time.perf_counter() - t0 >= 0.010:
                break
            inner *= 2
        for _ in range(inner):
            O.seq(mid, x, y)
        best = float("inf")
        for _ in range(5):
            t0 = time.perf_counter()
            for _ in range(inner):
                O.seq(mid, x, y)
            best = min(best, (time.perf_counter() - t0) / inner)
    finally:
        os.sched_setaffinity(0, old)
    return n / best / 1e9, n


def cpu_measure(name: str, cfg, method: str, steps: int, warmup: int) -> dict:
    """The reference's CPU path on this host (the oracle's C port of the seq
    recurrence, kernels.py:127-243), all host threads pinned one per CPU, on a
    bounded rank-0 sample: value = sample elements x steps / total seconds."""
    from oracle import oracle as O
    nt = host_threads()
    mid = O.METHODS.index(method)
    if cfg.op == "rows-dot":
        X, Y = cpu_rows_sample(cfg)
        times = cpu_rows_steps(mid, X, Y, nt, steps, warmup)
        n = X.size
        one, n1 = single_core(mid, X[0], Y[0])
        what = (f"the full {cfg.rows}x{cfg.cols} matrix per step (numpy N(0,1) rows scaled by 10^U[-4,4), the "
                f"config's distribution); the reference seq recurrence on every row, rows split over {nt} threads")
    else:
        n = min(layout(name, cfg, 1, 0)[0], CPU_SAMPLE)
        xh, yh, what = cpu_sample(name, cfg, n, nt)
        times = cpu_steps(mid, xh, yh, nt, steps, warmup)
        one, n1 = single_core(mid, xh, yh)
        what += (f"; {nt} threads pinned one per CPU on contiguous shards (first-touched by the same threads), "
                 "each the reference seq recurrence (kernels.py), shard pairs merged with kernels.py:310-317")
    value = n * len(times) / sum(times) / 1e9
    return {"value": value, "unit": UNIT, "cores": nt, "kind": "port",
            "sample": what + f"; {len(times)} timed steps after {warmup} warm-up, value = elements x steps / seconds",
            "step_s": {"median": statistics.median(times), "min": min(times), "max": max(times)},
            "single_core": {"value": one, "unit": UNIT, "elements": n1,
                            "method": "reference bench.py:82-130 (one pinned core, auto-scaled best of 5)"},
            "cpu": cpu_model(), "thp": _thp()}


def cpu_leg(args, steps: int, warmup: int) -> dict:
    """cpu_baseline of our arm: run `bench.py --impl reference` (the reference arm) as a
    child process on this config and K / W and take its cpu_baseline — one code path and
    one kind of process for both CPU figures."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE")}
    env.update(TFB_BENCH_CHILD="1", CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--config", args.config,
           "--steps", str(steps), "--warmup", str(warmup)]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1800)
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    if out.returncode != 0 or not lines:
        raise RuntimeError(f"CPU reference leg failed: {out.stderr[-2000:]}")
    cpu = json.loads(lines[-1])["cpu_baseline"]
    cpu["sample"] += "; measured by the reference arm (bench.py --impl reference) in a child process"
    return cpu


# ---------------------------------------------------------------------------
# Arms

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    # the CPU arm never touches a GPU: hide them, so the package import creates no
    # CUDA context (no driver threads or pinned pools beside the timed CPU work)
    os.environ["CUDA_VISIBLE_DEVICES"] = ""
    from paper_1401_0248_b200.gen import CONFIGS
    cfg_key, method, _, _ = WORKLOADS[args.config]
    cfg = CONFIGS[cfg_key]
    cpu = cpu_measure(args.config, cfg, method, args.steps, args.warmup)
    value = cpu["value"]
    n_sample = cfg.n if cfg.op == "rows-dot" else min(layout(args.config, cfg, 1, 0)[0], CPU_SAMPLE)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * n_sample / (value * 1e9), "higher_is_better": True,
        "scaling": scaling_kind(args.config, world), "vs_baseline": None,
        "dtype": "f64" if str(cfg.dtype).endswith("64") else "f32",
        "data": "synthetic", "impl": "reference",
        "config": workload_desc(args.config, cfg, method, world),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def run_dry(args):
    """Launcher/process-group plumbing on CPU: every rank joins a gloo group,
    barriers, and the max-over-ranks of a host timer reaches rank 0's line."""
    import torch
    import torch.distributed as dist

    from paper_1401_0248_b200.gen import CONFIGS
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg_key, method, _, _ = WORKLOADS[args.config]
    cfg = CONFIGS[cfg_key]
    t0 = time.perf_counter()
    if world > 1:
        dist.barrier()
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    ranks = torch.tensor([rank], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ranks, op=dist.ReduceOp.SUM)
    if rank == 0:
        emit({"metric": METRIC, "value": 0.0, "unit": UNIT, "n_gpus": world, "steps": args.steps,
              "warmup": args.warmup, "ms_per_step": 1e3 * t.item(), "higher_is_better": True,
              "scaling": scaling_kind(args.config, world), "vs_baseline": None, "data": "synthetic",
              "dry_run": True, "rank_sum": int(ranks.item()),
              "config": workload_desc(args.config, cfg, method, world)})
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    numa = bind_to_gpu_numa(local) if world > 1 else None
    torch.cuda.set_device(local)  # before the package import runs its device canary

    import paper_1401_0248_b200 as tfb
    from paper_1401_0248_b200 import _lib as _tl
    from paper_1401_0248_b200.gen import CONFIGS, make_inputs

    if world > 1 and "TFB_HYBRID_THREADS" not in os.environ:
        # the ranks of a node share its host cores: give each rank's hybrid host workers
        # its share of the CPUs it may run on (NUMA-local after the binding above)
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        os.environ["TFB_HYBRID_THREADS"] = str(max(1, len(os.sched_getaffinity(0))
                                                   // max(1, local_world // max(1, _numa_nodes())) - 1))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.force_collective:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    use_dist = dist.is_initialized()

    cfg_key, method_name, _, flush = WORKLOADS[args.config]
    cfg = CONFIGS[cfg_key]
    method = tfb.Method(method_name)
    rows = cfg.op == "rows-dot"
    rows_shard = rows and (world > 1 or args.force_collective)
    n, offset, total_elems = layout(args.config, cfg, world, rank)
    if rows_shard:
        r_lo, r_hi = tfb.rows_range(cfg.rows, rank, world)
        n, offset, total_elems = (r_hi - r_lo) * cfg.cols, r_lo * cfg.cols, cfg.n
    n_global = total_elems if not rows else cfg.n
    x, y = make_inputs(cfg, device=dev, offset=offset, n=n)
    torch.cuda.synchronize()
    item = x.element_size()
    bytes_per_step = n * item * (1 if y is None else 2)
    lg = tfb.leaf_log2_for(x.dtype, n_global if not rows else cfg.cols)
    leaf_arg = args.leaf_log2 or lg

    # Small working sets rotate over R identical copies whose total is >= 4x the
    # 126 MB L2, so every step streams its inputs from HBM with clean L2 lines
    # (a memset "flush" would leave dirty lines whose write-back lands in the
    # timed kernel).  Launch-bound steps are replayed from one CUDA graph.
    R = 1
    if flush:
        R = max(2, -(-(4 * 126 * 10**6) // bytes_per_step))
    copies = [(x, y)] + [(x.clone(), None if y is None else y.clone()) for _ in range(R - 1)]

    combine_desc = "none: contiguous row blocks per rank (dist.sharded_rows)" if rows_shard else args.combine
    if not rows and (world > 1 or args.force_collective):
        acc_dt = torch.float64 if method is tfb.Method.WIDE else x.dtype
        if args.combine == "auto":
            combine_desc = (tfb.combine_in_use(None, dev, acc_dt) if world > 1 else
                            "nccl (world size 1: the peer combine needs peers)")
        combine_desc = {"peer": "fused NVLink peer combine inside the reduction launch (tf_reduce_peer)",
                        "nccl": "NCCL all-gather of (v,e) pairs + tf_merge_tree"}.get(combine_desc, combine_desc)

    stream = torch.cuda.current_stream(dev)
    K = args.steps
    K_eff = max(K, R)  # every timed replay must stream >= 4x L2 of distinct bytes
    use_graph = world == 1 and not args.force_collective and (flush or args.graph)
    collective = not rows and (world > 1 or args.force_collective)
    # per-step events around the local reduction (eager, collective steps only):
    # the kernel's time inside the SAME window as ms_per_step
    kev: list = []

    def local_timed(meth, xs, ys, lg_):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = tfb.reduce(meth, xs, ys, leaf_log2=lg_)
        e1.record(stream)
        kev.append((e0, e1))
        return out

    def step(i, timed_kernel=False):
        xi, yi = copies[i % R]
        if rows_shard:
            return tfb.sharded_rows(method, xi, yi, rows_global=cfg.rows, leaf_log2=args.leaf_log2)
        if rows:
            return tfb.reduce_rows(method, xi, yi, leaf_log2=args.leaf_log2)
        if collective and args.combine == "nccl" and timed_kernel:
            return tfb.sharded_reduce(method, xi, yi, n_global=n_global, leaf_log2=leaf_arg,
                                      force_collective=args.force_collective, combine="nccl",
                                      local_reduce=local_timed)
        return tfb.sharded_reduce(method, xi, yi, n_global=n_global, leaf_log2=leaf_arg,
                                  force_collective=args.force_collective, combine=args.combine)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    def timed(fn):
        """Device time (ms) of K_eff back-to-back calls of fn, CUDA events on the launching stream."""
        if use_graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(K_eff):
                    fn(i)
            torch.cuda.synchronize()
            g.replay()  # untimed replay: first-launch costs of the graph
            torch.cuda.synchronize()
            s = torch.cuda.current_stream(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(K_eff):
            fn(i, True)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    # --- device-timed steps -------------------------------------------------
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    n0 = _tl.lib().tf_launch_count()
    with clocks, torch.cuda.nvtx.range("bench: timed steps"):
        elapsed_ms = timed(step)
    # kernels this library launched for the timed steps (graph mode: counted at capture,
    # i.e. the launches of the one timed replay)
    our_launches = _tl.lib().tf_launch_count() - n0
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms = t.item() / K_eff
    value = total_elems * K_eff / (t.item() * 1e-3) / 1e9

    # --- roofline of the reduction kernel, from the same timed window --------
    if kev:
        kernel_ms = sum(a.elapsed_time(b) for a, b in kev) / len(kev)
        ktiming = "per-step CUDA events around the reduction launch inside the timed window (this rank)"
    else:
        kernel_ms = elapsed_ms / K_eff
        ktiming = ("the timed window itself: each step is the reduction launch alone"
                   + (" (CUDA graph replay)" if use_graph else " (eager launches)"))
    (tfb.reduce_rows(method, x, y, leaf_log2=args.leaf_log2) if rows
     else tfb.reduce(method, x, y, leaf_log2=leaf_arg))
    torch.cuda.synchronize()
    launch_desc = _tl.lib().tf_last_launch().decode()
    peak, peak_src = measured_peak()
    achieved = bytes_per_step / (kernel_ms * 1e-3) / 1e9
    # practical HBM read ceiling, measured live on the same input buffer (the
    # paper's read1 row): XOR-fold streaming kernel, no FP chain
    read_roof = None
    if not rows and x.numel() * item >= (256 << 20):
        sink = torch.zeros(1, dtype=torch.int32, device=dev)
        rr = []
        for unroll in (4, 16):
            fn = (lambda i, u=unroll: _tl.lib().tf_read_roof(x.data_ptr(), x.numel() * item, u, sink.data_ptr(),
                                                              stream.cuda_stream))
            fn(0)
            torch.cuda.synchronize()
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r0.record(stream)
            for i in range(10):
                fn(i)
            r1.record(stream)
            torch.cuda.synchronize()
            rr.append(x.numel() * item * 10 / (r0.elapsed_time(r1) * 1e-3) / 1e9)
        read_roof = max(rr)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic_for(args.config), "peak_source": peak_src,
                "kernel": launch_desc + " (fused leaf + tree, one launch per step)",
                "algorithmic_bytes_per_launch": bytes_per_step, "kernel_ms": kernel_ms,
                "kernel_share_of_step": kernel_ms / step_ms if step_ms else None,
                "timing": ktiming,
                "read_roof_gbs": read_roof,
                "frac_of_read_roof": (achieved / read_roof) if read_roof else None,
                "read_roof_source": "tf_read_roof (XOR-fold 16-byte streaming, best of unroll 4/16) on the x buffer, live"}

    # --- end to end through the public API, pinned host buffers --------------
    e2e = None
    res_dev = step(0).cpu()
    if not args.no_e2e:
        xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        xh.copy_(x)
        yh = None
        if y is not None:
            yh = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
            yh.copy_(y)
        torch.cuda.synchronize()
        ke = args.e2e_steps or max(3, min(K, 10))

        def e2e_step():
            if rows_shard:
                return tfb.sharded_rows(method, xh, yh, rows_global=cfg.rows).cpu()
            if rows:
                r = tfb.dot_rows(method, xh, yh)
                return r.values.cpu()
            return tfb.sharded_run(method, xh, yh, n_global=n_global, leaf_log2=lg)

        r0 = e2e_step()  # warm-up (also allocates the staging buffers)
        if not rows:
            assert float(r0.value) == float(res_dev[0]) and (
                method not in (tfb.Method.TWOFOLD_FAST, tfb.Method.TWOFOLD_RIGOROUS)
                or float(r0.error) == float(res_dev[1])), "e2e result differs from the device path"
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()
        eng = _tl.host_engine(local)
        split = [0, 0]  # elements the GPU / the host workers reduced over the timed e2e steps
        w0 = time.perf_counter()
        with torch.cuda.nvtx.range("bench: e2e steps"):
            for _ in range(ke):
                e2e_step()
                if eng is not None:
                    g_el, h_el = _tl.host_split(eng)
                    split[0] += g_el
                    split[1] += h_el
            torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        if use_dist:
            tw = torch.tensor([wall], dtype=torch.float64, device=dev)
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
            wall = tw.item()
        # bytes that crossed the link: the GPU's share (the hybrid host path reduces the rest
        # of the host-resident shard on the engine's host workers and uploads leaf pairs only)
        gpu_frac = split[0] / max(1, split[0] + split[1])
        h2d = int(round(bytes_per_step * gpu_frac))
        e2e = {"value": total_elems * ke / wall / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 16 if not rows else cfg.rows * item,
               "steps": ke, "ms_per_step": 1e3 * wall / ke,
               "path": (("paper_1401_0248_b200.dot_rows(pinned host matrices) -> C-ABI tf_host_reduce_rows "
                         "(host-buffer engine, hybrid): the GPU takes row blocks from the front (DMA'd straight from "
                         "the pinned matrices on a copy stream, overlapped with the row kernels) while the engine's "
                         "host workers reduce whole rows from the back with the same leaves and row tree "
                         "(csrc/hostleaf.cpp); row pairs stored into mapped host memory")
                        if rows else
                        ("paper_1401_0248_b200.sharded_run(pinned host shard) -> C-ABI tf_host_reduce (host-buffer "
                         "engine, hybrid): the GPU pipeline takes leaf-aligned 16 MiB chunks from the front of the shard "
                         "(DMA'd straight from pinned memory on a copy stream, overlapped with the leaf kernels) while "
                         "the engine's host workers reduce full leaves from the back with the same chains and leaf "
                         "tree (csrc/hostleaf.cpp) and upload only their leaf pairs; one tree kernel over all leaf "
                         "pairs stores the pair into mapped host memory (bit-identical to the device-resident result)"
                         + ("; NCCL all-gather + merge across ranks" if world > 1 else ""))),
               "host_share": split[1] / max(1, split[0] + split[1]),
               "timing": "wall clock around the steps after synchronize, max over ranks",
               **({"host_placement": numa} if numa else {})}
        # The link the e2e path streams over: plain pinned H2D of the same host
        # buffer (up to 1 GiB, best of 3, CUDA events) — the e2e ceiling.
        src = xh.view(-1).view(torch.uint8)[: 1 << 30]
        dst = torch.empty_like(src, device=dev)
        h2d_link = 0.0
        for _ in range(3):
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record()
            dst.copy_(src, non_blocking=True)
            c1.record()
            torch.cuda.synchronize()
            h2d_link = max(h2d_link, src.numel() / (c0.elapsed_time(c1) * 1e-3) / 1e9)
        del dst, src, xh, yh
        _release_pinned(torch)
        e2e["h2d_link_gbs"] = h2d_link
        e2e["frac_of_h2d_link"] = (e2e["h2d_bytes_per_step"] / (1e-3 * e2e["ms_per_step"]) / 1e9) / h2d_link

    # --- CPU baseline (rank 0, N=1 only): the reference arm's own routine -----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        del copies, x, y
        torch.cuda.empty_cache()
        # the reference arm itself, in a fresh process (same routine, same process
        # conditions as `--impl reference`), over the run's K / W (capped: seconds)
        cpu = cpu_leg(args, steps=min(args.steps, 20), warmup=min(args.warmup, 5))

    dtype_name = "f64" if item == 8 else "f32"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": scaling_kind(args.config, world),
        "vs_baseline": None,
        "dtype": dtype_name, "data": "synthetic",
        "config": workload_desc(args.config, cfg, method_name, world),
        "run": {"l2": (f"rotating over {R} input copies ({R * bytes_per_step / 1e6:.0f} MB >= 4x the 126 MB L2)"
                       if R > 1 else f"inputs {bytes_per_step / 2**30:.1f} GiB per rank >> 126 MB L2 (no flush)"),
                "leaf_log2": (leaf_arg if not rows else
                              (args.leaf_log2 or tfb.leaf_log2_for(cfg.dtype, cfg.rows * cfg.cols))),
                "steps_timing": "CUDA graph replay" if use_graph else "eager launches",
                "steps_timed": K_eff, "n_this_rank": n,
                **({"combine": combine_desc} if world > 1 or args.force_collective else {})},
        "hbm_gbs": bytes_per_step * total_elems / n * K_eff / (t.item() * 1e-3) / 1e9,
        "value_per_gpu": value / world,
        "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
        "gpu_launches": int(our_launches),
        "gpu_launches_per_step": our_launches / K_eff,
        "clocks": clocks.report(),
        "result": {"value": float(res_dev[0]) if not rows else None,
                   "error": float(res_dev[1]) if not rows else None},
    }
    if rank == 0:
        emit(line)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _release_pinned(torch) -> None:
    """Return the caching host allocator's pinned blocks to the OS (the e2e shard
    can be 64 GiB; the CPU baseline allocates its own pageable sample next)."""
    f = getattr(torch._C, "_host_emptyCache", None)
    if f is not None:
        try:
            f()
        except Exception:
            pass


def _reserve_stdout():
    """The contract is ONE JSON line on stdout: native libraries (NCCL's version
    banner, driver warnings) write to fd 1, so fd 1 is pointed at stderr for the
    run and the JSON line goes to a saved copy of the real stdout."""
    global _OUT
    real = os.dup(1)
    os.dup2(2, 1)
    _OUT = os.fdopen(real, "w")


_OUT = None


def emit(line: dict) -> None:
    out = _OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    args = parse()
    rc = self_launch(args)
    if rc is not None:
        return rc
    _, world, _ = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting the process group's size",
              file=sys.stderr)
    _reserve_stdout()
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
