"""Contiguous multi-GPU sharding with one tiny all-gather.

Rank r of G owns the leaf-aligned slice shard_range(n, r, G) of the global
array, reduces it to one raw (value, error) pair with the GLOBAL leaf size,
then the G pairs are all-gathered (NCCL over NVLink: 16·G bytes for binary64)
and every rank merges them with the same balanced TwoSum tree, so all ranks
hold bit-identical results.  NCCL has no TwoSum reduction op and ncclSum
would drop the round-off, hence all-gather + a fixed-order merge.

When every rank owns the same power-of-two number of leaves (e.g. cfg5:
N = 2^32, G in {1,2,4,8}, leaf 2^16) each rank's tree is an exact subtree of
the single-GPU tree, so the G-GPU result is bit-identical to the 1-GPU one.

The local reducer and the merge are injectable so the plumbing can be
exercised with gloo on CPU (tests/test_dist_gloo.py); the defaults are the
CUDA kernels and there is no CPU fallback.

combine="nccl" (the default, the north_star design) is that all-gather
plus the merge kernel.  combine="peer" replaces reduce + NCCL all-gather +
merge by ONE launch (tf_reduce_peer, csrc/peer.cuh): the CTA that builds the
shard's root writes it into every peer's symmetric-memory buffer over
NVLink, waits for the G pairs (system-scope release/acquire flags, epoch
double-buffered, bounded wait) and merges them in-kernel.  It is opt-in: on
this round's single-GPU pool it has only run at world size 1 (self-
publication through the same code).  A peer that does not arrive within the
timeout (TFB_PEER_TIMEOUT_S, default the process group's default timeout)
makes that call raise RuntimeError on the host — never a silent NaN — and
retires the peer combine for the group (later peer calls raise at once;
NCCL keeps working), so ranks cannot drift apart.  combine="auto" uses the
peer path for device-resident shards at world size > 1 after a one-time
self-check against NCCL on every rank.
"""

from __future__ import annotations

import os
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from .api import Method, SumResult, Twofold, _TWOFOLD_METHODS, _acc_dtype, _np_type, leaf_log2_for, merge_pairs

LocalReduce = Callable[[Method, torch.Tensor, "torch.Tensor | None", int], torch.Tensor]
Merge = Callable[[Method, torch.Tensor], torch.Tensor]


def shard_range(n: int, rank: int, world: int, leaf_log2: int) -> tuple[int, int]:
    """Leaf-aligned contiguous slice [start, stop) of rank `rank` (leaves split as evenly as possible)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    L = 1 << leaf_log2
    P = -(-n // L)
    lo = (rank * P) // world
    hi = ((rank + 1) * P) // world
    return min(lo * L, n), min(hi * L, n)


def _default_local(method: Method, x: torch.Tensor, y, leaf_log2: int, track_product: bool = False) -> torch.Tensor:
    from .api import _all_host, _device_for, _on_device, _reduce_grid, _reduce_host
    dev = _device_for(x)
    with torch.cuda.device(dev):
        if _all_host(x, y):
            # host shard: the native host-buffer engine (pinned staging, chunked H2D
            # overlapped with the leaf kernels)
            return _reduce_host(method, x, y, dev, leaf_log2, track_product=track_product)
        return _reduce_grid(method, _on_device(x, dev), _on_device(y, dev), leaf_log2,
                            track_product=track_product)


def _default_merge(method: Method, pairs: torch.Tensor) -> torch.Tensor:
    return merge_pairs(method, pairs)  # enters pairs.device itself


def _peer_timeout_ns() -> int:
    env = os.environ.get("TFB_PEER_TIMEOUT_S")
    if env:
        return int(float(env) * 1e9)
    try:
        from torch.distributed.constants import default_pg_timeout
        return int(default_pg_timeout.total_seconds() * 1e9)
    except Exception:
        return 1800 * 10 ** 9


class PeerTimeout(RuntimeError):
    """A fused peer combine did not hear from every rank within the timeout."""


class _PeerCombine:
    """Symmetric buffers + device PeerCtx for one (group, device, accumulator dtype)."""

    MAX_PEERS = 16

    def __init__(self, group, dev: torch.device, acc: torch.dtype):
        import struct

        import torch.distributed._symmetric_memory as symm

        from . import _lib
        rank, world = _world(group)
        if world > self.MAX_PEERS:
            raise ValueError(f"peer combine supports up to {self.MAX_PEERS} ranks")
        self.world, self.rank = world, rank
        # every rank must be here before the (store-based) rendezvous: one NCCL
        # collective, bounded by the process group's own timeout
        ready = torch.ones(1, dtype=torch.int32, device=dev)
        dist.all_reduce(ready, group=group)
        self.buf = symm.empty(2 * world * 2, dtype=acc, device=dev)      # [2 parities][world] pairs
        self.flags = symm.empty(world, dtype=torch.int32, device=dev)    # epoch of rank g's last publication
        self.flags.zero_()
        self.error = torch.zeros(2, dtype=torch.int32, device=dev)       # [epoch of a timeout, missing mask]
        torch.cuda.synchronize(dev)
        pg = group if group is not None else dist.group.WORLD
        hb = symm.rendezvous(self.buf, pg)
        hf = symm.rendezvous(self.flags, pg)
        dist.barrier(group)
        bufs = list(hb.buffer_ptrs) + [0] * (self.MAX_PEERS - world)
        flags = list(hf.buffer_ptrs) + [0] * (self.MAX_PEERS - world)
        raw = struct.pack("<iiQ16Q16QQ", world, rank, self.error.data_ptr(), *bufs, *flags, _peer_timeout_ns())
        assert len(raw) == _lib.lib().tf_peer_ctx_size(), "PeerCtx layout mismatch"
        self.ctx = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
        self.epoch = 0
        self.failed: str | None = None
        self._handles = (hb, hf)  # keep the mappings alive

    def next_epoch(self) -> int:
        self.epoch += 1
        return self.epoch

    def check(self, epoch: int, error_words) -> None:
        """Raise PeerTimeout if call `epoch` timed out; error_words = (stamped epoch, missing mask)."""
        stamped, missing = int(error_words[0]), int(error_words[1])
        if stamped == epoch:
            ranks = [r for r in range(self.world) if (missing >> r) & 1]
            self.failed = (f"peer combine call {epoch} on rank {self.rank} timed out waiting for rank(s) {ranks}; "
                           "the peer combine is retired for this group (use combine='nccl')")
            raise PeerTimeout(self.failed)


_peer_cache: dict = {}


def _peer_combine_for(group, dev: torch.device, acc: torch.dtype) -> _PeerCombine:
    key = (id(group), dev.index, acc)
    pc = _peer_cache.get(key)
    if pc is None:
        pc = _PeerCombine(group, dev, acc)
        _peer_cache[key] = pc
    return pc


def _reduce_peer(method: Method, x: torch.Tensor, y, leaf_log2: int, group, track_product: bool,
                 pc: _PeerCombine | None = None, launch=None) -> torch.Tensor:
    """One fused reduce + peer combine, then (synchronously) the timeout check.
    `pc` / `launch` are injectable for the CPU tests of the failure path."""
    from . import _lib
    from .api import _acc_dtype, _dtype_code, _mid, _on_device, _ptr, _scratch, _stream_ptr, workspace_size
    dev = x.device
    acc = _acc_dtype(method, x.dtype)
    if pc is None:
        _lib.ensure_canary(dev.index)
        pc = _peer_combine_for(group, dev, acc)
    if pc.failed:
        raise PeerTimeout(pc.failed)
    epoch = pc.next_epoch()
    if launch is not None:
        out = launch(pc, epoch)
    else:
        y = _on_device(y, dev)
        x = x.contiguous()
        out = torch.empty(2, dtype=acc, device=dev)
        pb, cnt, _ = workspace_size(method, x.dtype, 1, x.numel(), leaf_log2)
        parts, ctrs = _scratch.get(dev, pb, cnt)
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().tf_reduce_peer(_mid(method, track_product, y is not None), _dtype_code(x.dtype),
                                                 _ptr(x), _ptr(y), x.numel(), leaf_log2, out.data_ptr(),
                                                 _ptr(parts), pb, _ptr(ctrs), cnt, pc.ctx.data_ptr(), epoch,
                                                 _stream_ptr(dev)),
                       "tf_reduce_peer")
    pc.check(epoch, pc.error.tolist())  # .tolist() waits for the launch
    return out


_auto_cache: dict = {}


def _peer_self_check(group, dev: torch.device, acc: torch.dtype) -> str | None:
    """Run the fused peer combine once on known per-rank data and compare it with
    the NCCL all-gather + merge result; every rank takes the same decision
    (all-reduce MIN of the verdicts).  Returns None if the peer path is usable,
    else the reason."""
    from .api import _reduce_grid
    rank, world = _world(group)
    reason = None
    try:
        n = 3 * 4096 + 17
        dt = torch.float32 if acc == torch.float32 else torch.float64
        g = torch.Generator(device="cpu").manual_seed(1234 + rank)
        x = (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1).to(dt).to(dev)
        lg = leaf_log2_for(dt, n * world)
        method = Method.TWOFOLD_RIGOROUS
        with torch.cuda.device(dev):
            got = _reduce_peer(method, x, None, lg, group, False)
            local = _reduce_grid(method, x, None, lg)
            parts = [torch.empty_like(local) for _ in range(world)]
            dist.all_gather(parts, local, group=group)
            want = _default_merge(method, torch.stack(parts, 0))
            if not torch.equal(got.view(torch.int64 if dt == torch.float64 else torch.int32),
                               want.view(torch.int64 if dt == torch.float64 else torch.int32)):
                reason = "peer self-check result differs from the NCCL combine"
    except PeerTimeout as exc:
        reason = f"peer self-check: {exc}"
    except Exception as exc:  # no symmetric memory / P2P on this box
        reason = f"peer combine unavailable: {type(exc).__name__}: {exc}"
    return _agree(reason, group, dev)


def _agree(reason: str | None, group, dev: torch.device) -> str | None:
    """Every rank adopts the peer combine only if every rank's check passed."""
    ok = torch.tensor([0 if reason else 1], dtype=torch.int32, device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if reason is None and int(ok.item()) == 0:
        reason = "peer self-check failed on another rank"
    return reason


def combine_in_use(group=None, dev: torch.device | None = None, acc: torch.dtype = torch.float64) -> str:
    """The cross-rank combine `combine="auto"` picks for this group/device/accumulator:
    "peer" (fused NVLink combine, self-checked against NCCL once) or "nccl (<reason>)"."""
    dev = dev or torch.device("cuda", torch.cuda.current_device())
    key = (id(group), dev.index, acc)
    if key not in _auto_cache:
        _auto_cache[key] = _peer_self_check(group, dev, acc)
    reason = _auto_cache[key]
    return "peer" if reason is None else f"nccl ({reason})"


def peer_combine_error(group=None) -> str | None:
    """Why the peer combine was retired for this group on this rank (a timeout), else None."""
    for (gid, _, _), pc in _peer_cache.items():
        if gid == id(group) and pc.failed:
            return pc.failed
    return None


def _world(group) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def sharded_reduce(method: Method, x_local: torch.Tensor, y_local: torch.Tensor | None = None, *,
                   n_global: int, leaf_log2: int = 0, group=None,
                   local_reduce: LocalReduce | None = None, merge: Merge | None = None,
                   track_product: bool = False, force_collective: bool = False,
                   combine: str = "nccl") -> torch.Tensor:
    """Raw (value, error) pair of the global array, identical on every rank.

    x_local / y_local: this rank's shard (CUDA tensors for the default
    reducer).  leaf_log2 = 0 uses the global array's auto leaf size, so the
    partition does not depend on G.  combine: "peer" (fused NVLink combine
    inside the reduction launch; synchronous, raises PeerTimeout if a peer
    never arrives), "nccl" (default: all-gather + merge kernel), or "auto"
    (peer for device-resident shards at world size > 1 once a one-time
    self-check against NCCL passed on every rank and no timeout retired it,
    else nccl).
    """
    if combine not in ("nccl", "peer", "auto"):
        raise ValueError("combine must be 'auto', 'nccl' or 'peer'")
    lg = leaf_log2 or leaf_log2_for(x_local.dtype, n_global)
    distributed = dist.is_available() and dist.is_initialized()
    # The peer combine's epoch is a host counter baked into each launch, so a
    # captured CUDA graph would replay a stale epoch: never inside a capture.
    capturing = x_local.is_cuda and torch.cuda.is_current_stream_capturing()
    if combine == "auto":
        combine = "nccl"
        if (distributed and local_reduce is None and merge is None and x_local.is_cuda and not capturing
                and _world(group)[1] > 1
                and combine_in_use(group, x_local.device, _acc_dtype(method, x_local.dtype)) == "peer"
                and not peer_combine_error(group)):
            combine = "peer"
    if combine == "peer" and distributed and local_reduce is None:
        if not x_local.is_cuda:
            raise ValueError("the peer combine reduces device-resident shards")
        if capturing:
            raise ValueError("the peer combine is not CUDA-graph capturable (host-side epochs); "
                             "use combine='auto' or 'nccl' inside a capture")
        return _reduce_peer(method, x_local, y_local, lg, group, track_product)
    if local_reduce is None:
        local = _default_local(method, x_local, y_local, lg, track_product)
    else:
        local = local_reduce(method, x_local, y_local, lg)
    _, world = _world(group)
    if world == 1 and not (force_collective and dist.is_available() and dist.is_initialized()):
        return local  # force_collective exercises the all-gather + merge path at world size 1
    local = local.contiguous()
    if local.is_cuda and dist.get_backend(group) == "nccl":
        # one NCCL all-gather straight into the (world, 2) pair table
        gathered = torch.empty((world, 2), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(gathered, local, group=group)
    else:
        # any other backend (gloo: CPU tensors only): the 8/16-byte pairs travel through host
        # memory and the merge runs where the shards live
        send = local.cpu() if local.is_cuda else local
        parts = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(parts, send, group=group)
        gathered = torch.stack(parts, 0).to(local.device)
    return (merge or _default_merge)(method, gathered)


def sharded_run(method: Method, x_local, y_local=None, *, n_global: int, leaf_log2: int = 0, group=None,
                local_reduce: LocalReduce | None = None, merge: Merge | None = None,
                track_product: bool = False) -> SumResult:
    """SumResult of the global sum / dot (reference result conventions)."""
    if not isinstance(x_local, torch.Tensor):
        x_local = torch.as_tensor(x_local)
    if y_local is not None and not isinstance(y_local, torch.Tensor):
        y_local = torch.as_tensor(y_local)
    if (local_reduce is None and merge is None and not x_local.is_cuda and (y_local is None or not y_local.is_cuda)
            and _world(group)[1] == 1):
        # one rank, host-resident shard: the host-buffer engine already returns the pair in
        # host memory — no bounce through a device tensor (two small copies and a sync less)
        from .api import _device_for, _host_pair
        lg = leaf_log2 or leaf_log2_for(x_local.dtype, n_global)
        dev = _device_for(x_local)
        with torch.cuda.device(dev):
            v, e = _host_pair(method, x_local, y_local, dev, lg, track_product).tolist()
    else:
        pair = sharded_reduce(method, x_local, y_local, n_global=n_global, leaf_log2=leaf_log2, group=group,
                              local_reduce=local_reduce, merge=merge, track_product=track_product)
        v, e = pair.cpu().tolist()
    t = np.float64 if method is Method.WIDE else _np_type(x_local.dtype)
    if method in _TWOFOLD_METHODS:
        return SumResult(Twofold(t(v), t(e)), n_global)
    return SumResult(Twofold(t(v), t(0)), n_global)


def rows_range(rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row block [start, stop) of rank `rank` (rows split as evenly as possible)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return (rank * rows) // world, ((rank + 1) * rows) // world


LocalRows = Callable[[Method, torch.Tensor, "torch.Tensor | None", int], torch.Tensor]


def sharded_rows(method: Method, X_local, Y_local=None, *, rows_global: int, leaf_log2: int = 0, group=None,
                 gather: bool = False, local_reduce: LocalRows | None = None,
                 track_product: bool = False) -> torch.Tensor:
    """Row-wise reduction of a matrix sharded by rows (rows shard with no
    collective).  X_local / Y_local: this rank's contiguous row block rows_range(rows_global,
    rank, world).  Every row is reduced with the WHOLE matrix's leaf size, so each row's pair
    is bit-identical to reduce_rows on the unsharded matrix.  Returns this rank's (rows, 2)
    pairs, or with gather=True all rows_global pairs in row order on every rank (one
    all-gather of the padded blocks)."""
    from .api import _as_rows, reduce_rows
    x = _as_rows(X_local)
    rows_l, cols = x.shape
    rank, world = _world(group)
    lo, hi = rows_range(rows_global, rank, world)
    if rows_l != hi - lo:
        raise ValueError(f"X_local has {rows_l} rows; rank {rank} of {world} owns rows [{lo}, {hi})")
    lg = leaf_log2 or leaf_log2_for(x.dtype, rows_global * cols)
    if local_reduce is None:
        pairs = reduce_rows(method, X_local, Y_local, leaf_log2=lg, track_product=track_product)
    else:
        pairs = local_reduce(method, x, None if Y_local is None else _as_rows(Y_local), lg)
    if not gather or world == 1:
        return pairs
    block = -(-rows_global // world)  # padded block: ragged blocks all-gather as equal sizes
    padded = torch.zeros((block, 2), dtype=pairs.dtype, device=pairs.device)
    padded[:rows_l] = pairs
    if padded.is_cuda and dist.get_backend(group) == "nccl":
        table = torch.empty((world * block, 2), dtype=pairs.dtype, device=pairs.device)
        dist.all_gather_into_tensor(table, padded, group=group)
        parts = list(table.split(block))
    else:
        send = padded.cpu() if padded.is_cuda else padded  # gloo: through host memory
        parts = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(parts, send, group=group)
        parts = [p.to(padded.device) for p in parts]
    return torch.cat([parts[r][: rows_range(rows_global, r, world)[1] - rows_range(rows_global, r, world)[0]]
                      for r in range(world)], 0)


__all__ = ["shard_range", "sharded_reduce", "sharded_run", "peer_combine_error", "PeerTimeout", "rows_range",
           "sharded_rows"]
