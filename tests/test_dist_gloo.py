"""Multi-rank shard/combine plumbing on CPU: world_size 2 (and 4) over gloo.

The product's local reducer and merge are CUDA kernels; here they are
injected with the oracle's bit-exact restatements of those kernels, so the
test exercises exactly dist.py's sharding, all-gather order and merge
placement.  With a power-of-two layout the sharded result must equal the
single-device result bit for bit, on every rank.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, dtype_name, q):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    import paper_1401_0248_b200 as tfb

    dt = np.float32 if dtype_name == "f32" else np.float64
    tdt = torch.float32 if dt == np.float32 else torch.float64
    x = O.lcg_fill("mmix", n, 17, dt, True)
    y = O.lcg_fill("nr", n, 18, dt, True)
    lg = tfb.leaf_log2_for(tdt, n)
    a, b = tfb.shard_range(n, rank, world, lg)
    xs, ys = torch.from_numpy(x[a:b].copy()), torch.from_numpy(y[a:b].copy())

    def local(method, xl, yl, leaf):
        mid = list(tfb.Method).index(method)
        v, e = O.emulate(mid, xl.numpy(), None if yl is None else yl.numpy(), leaf)
        return torch.tensor([float(v), float(e)], dtype=torch.float64 if method is tfb.Method.WIDE else tdt)

    def merge(method, pairs):
        mid = list(tfb.Method).index(method)
        v, e = O.tree(mid, np.float64 if method is tfb.Method.WIDE else dt, pairs[:, 0].numpy(), pairs[:, 1].numpy())
        return torch.tensor([float(v), float(e)], dtype=pairs.dtype)

    out = {}
    for method in tfb.Method:
        if method is tfb.Method.WIDE and dt != np.float32:
            continue
        pair = tfb.sharded_reduce(method, xs, ys, n_global=n, local_reduce=local, merge=merge)
        res = tfb.sharded_run(method, xs, None, n_global=n, local_reduce=local, merge=merge)
        out[method.value] = (pair.tolist(), float(res.value), float(res.error), type(res.value).__name__,
                             res.adds_performed)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, n, dtype_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, dtype_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return results


@pytest.mark.parametrize("world,dtype_name", [(2, "f64"), (2, "f32"), (4, "f64")])
def test_sharded_equals_single_device_tree(oracle, world, dtype_name):
    n = 1 << 18
    results = _run(world, n, dtype_name)
    dt = np.float32 if dtype_name == "f32" else np.float64
    x = oracle.lcg_fill("mmix", n, 17, dt, True)
    y = oracle.lcg_fill("nr", n, 18, dt, True)
    for method_name, (pair, v, e, tname, adds) in results[0].items():
        mid = oracle.METHODS.index(method_name)
        want = oracle.emulate(mid, x, y)
        assert [float(want[0]), float(want[1])] == pair, method_name
        # all ranks hold the identical result
        for r in range(1, world):
            assert results[r][method_name] == results[0][method_name]
        # SumResult conventions: typed like the data (f64 for wide), error 0 for non-twofold
        ws = oracle.emulate(mid, x)
        assert v == float(ws[0])
        assert e == (float(ws[1]) if mid in (2, 3) else 0.0)
        assert tname == ("float64" if mid == 1 else np.dtype(dt).name)
        assert adds == n


def _agree_worker(rank, world, port, q):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1401_0248_b200 import dist as D
    cpu = torch.device("cpu")
    all_ok = D._agree(None, None, cpu)
    one_bad = D._agree("boom" if rank == 1 else None, None, cpu)
    q.put((rank, all_ok, one_bad))
    dist.barrier()
    dist.destroy_process_group()


def test_auto_combine_decision_is_collective():
    """combine="auto": one rank's failed peer self-check moves EVERY rank to NCCL."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = dict((r, (a, b)) for r, a, b in (q.get(timeout=300) for _ in range(3)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(a is None for a, _ in res.values())
    assert res[1][1] == "boom"
    assert res[0][1] == res[2][1] == "peer self-check failed on another rank"


def _peer_fail_worker(rank, world, port, q):
    """Host side of the fused peer combine's failure path, one gloo rank each.
    The device launch is simulated: call 1 succeeds everywhere; in call 2 rank 1
    never publishes, so rank 0's kernel stamps (epoch 2, missing {1}) and yields
    NaN while rank 1 completes (its peers did publish); in call 3 rank 0 has
    retired the peer path, so rank 1's kernel stamps (epoch 3, missing {0})."""
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1401_0248_b200 import dist as D
    import paper_1401_0248_b200 as tfb
    pc = D._PeerCombine.__new__(D._PeerCombine)
    pc.world, pc.rank, pc.epoch, pc.failed = world, rank, 0, None
    pc.error = torch.zeros(2, dtype=torch.int32)

    def launch(pc_, epoch):
        if (epoch == 2 and rank == 0) or (epoch == 3 and rank == 1):
            pc_.error[1] = 1 << (1 - rank)
            pc_.error[0] = epoch
            return torch.full((2,), float("nan"), dtype=torch.float64)
        return torch.tensor([1.0 + rank, 0.0], dtype=torch.float64)

    x = torch.zeros(8, dtype=torch.float64)
    log = []
    for call in (1, 2, 3, 4):
        try:
            out = D._reduce_peer(tfb.Method.TWOFOLD_FAST, x, None, 10, None, False, pc=pc, launch=launch)
            log.append(("ok", float(out[0])))
        except D.PeerTimeout as exc:
            log.append(("timeout", str(exc)))
    # the NCCL/gloo combine still works for every rank after the peer path is retired
    pair = D.sharded_reduce(tfb.Method.TWOFOLD_FAST, torch.tensor([float(rank)]), None, n_global=2,
                            local_reduce=lambda m, xl, yl, lg: torch.tensor([float(xl[0]), 0.0], dtype=torch.float64),
                            merge=lambda m, pairs: pairs.sum(0))
    q.put((rank, log, pair.tolist(), pc.failed))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_timeout_raises_instead_of_nan():
    """a peer timeout must raise on the host (never hand back NaN), is
    stamped per call (not sticky: the stale stamp of call 2 does not fail call 1's
    successor on the other rank), and retires the peer path on the failing rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (log, pair, failed) for r, log, pair, failed in (q.get(timeout=300) for _ in range(2))}
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    log0, pair0, failed0 = res[0]
    log1, pair1, failed1 = res[1]
    assert log0[0] == ("ok", 1.0) and log0[1][0] == "timeout" and "rank(s) [1]" in log0[1][1]
    assert log0[2][0] == log0[3][0] == "timeout" and "retired" in log0[2][1]  # no silent NaN afterwards
    assert log1[0] == ("ok", 2.0) and log1[1] == ("ok", 2.0)  # call 2 completed on the late rank
    assert log1[2][0] == "timeout" and "rank(s) [0]" in log1[2][1] and log1[3][0] == "timeout"
    assert failed0 and failed1
    assert pair0 == pair1 == [1.0, 0.0]


def test_ragged_shards_cover_everything(oracle):
    """Non-power-of-two n: shards are leaf-aligned and the merged pair still tracks the exact sum."""
    n = 300_007
    results = _run(2, n, "f64")
    x = oracle.lcg_fill("mmix", n, 17, np.float64, True)
    y = oracle.lcg_fill("nr", n, 18, np.float64, True)
    S, A = oracle.exact(x, y), oracle.abs_sum(x, y)
    pair = results[0]["twofold-rigorous"][0]
    assert oracle.deviation(pair[0], pair[1], S) <= oracle.bound(3, np.float64, n, A)


def _rows_worker(rank, world, port, rows, cols, dtype_name, q):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    import paper_1401_0248_b200 as tfb

    dt = np.float32 if dtype_name == "f32" else np.float64
    X = O.lcg_fill("mmix", rows * cols, 27, dt, True).reshape(rows, cols)
    Y = O.lcg_fill("nr", rows * cols, 28, dt, True).reshape(rows, cols)
    a, b = tfb.rows_range(rows, rank, world)

    def local(method, xl, yl, leaf):
        mid = list(tfb.Method).index(method)
        v, e = O.emulate_rows(mid, xl.numpy(), None if yl is None else yl.numpy(), leaf)
        t = torch.float64 if method is tfb.Method.WIDE else torch.from_numpy(X[:1]).dtype
        return torch.stack([torch.from_numpy(np.asarray(v, np.float64)), torch.from_numpy(np.asarray(e, np.float64))],
                           1).to(t)

    out = {}
    for method in (tfb.Method.TWOFOLD_FAST, tfb.Method.KAHAN, tfb.Method.DIRECT):
        full = tfb.sharded_rows(method, torch.from_numpy(X[a:b].copy()), torch.from_numpy(Y[a:b].copy()),
                                rows_global=rows, gather=True, local_reduce=local)
        mine = tfb.sharded_rows(method, torch.from_numpy(X[a:b].copy()), None, rows_global=rows, local_reduce=local)
        out[method.value] = (full.numpy().tolist(), mine.numpy().tolist(), (a, b))
    try:
        tfb.sharded_rows(tfb.Method.DIRECT, torch.from_numpy(X[: b - a + 1].copy()), rows_global=rows,
                         local_reduce=local)
        out["bad_block"] = "no error"
    except ValueError:
        out["bad_block"] = "ValueError"
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,dtype_name", [(2, 37, "f32"), (3, 50, "f64")])
def test_sharded_rows_gather_equals_unsharded(oracle, world, rows, dtype_name):
    """Rows sharded by contiguous blocks: each rank's pairs use the whole
    matrix's leaf size, and the gathered table equals the single-device row reduction."""
    cols = 3000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, rows, cols, dtype_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dt = np.float32 if dtype_name == "f32" else np.float64
    X = oracle.lcg_fill("mmix", rows * cols, 27, dt, True).reshape(rows, cols)
    Y = oracle.lcg_fill("nr", rows * cols, 28, dt, True).reshape(rows, cols)
    import paper_1401_0248_b200 as tfb
    tdt = torch.float32 if dt == np.float32 else torch.float64
    lg = tfb.leaf_log2_for(tdt, rows * cols)
    for name in ("twofold-fast", "kahan", "direct"):
        mid = oracle.METHODS.index(name)
        ev, ee = oracle.emulate_rows(mid, X, Y, lg)
        sv, se = oracle.emulate_rows(mid, X, None, lg)
        for r in range(world):
            full, mine, (a, b) = res[r][name]
            assert [p[0] for p in full] == [float(v) for v in ev] and [p[1] for p in full] == [float(v) for v in ee]
            assert [p[0] for p in mine] == [float(v) for v in sv[a:b]]
        assert res[0]["bad_block"] == "ValueError"
