"""torchrun entry: the shard layer with REAL kernels at world size > 1 on ONE GPU.

Every rank selects cuda:0 and a gloo process group carries the 8/16-byte pairs (NCCL refuses
two ranks on one device); the ranks' kernels are independent launches that never wait on one
another.  Checked, bit for bit: every rank holds the same pair; with equal power-of-two
leaf counts per rank the pair equals the single-GPU reduction of the whole array; otherwise
it equals the merge tree over the per-shard reductions; sharded rows equal the unsharded
reduce_rows; the host-resident path (sharded_run on pinned shards) agrees."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402


def merge_tree(method, pairs):
    from paper_1401_0248_b200.dist import _default_merge
    return _default_merge(method, pairs)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo")
    checked = 0
    for dt in (torch.float32, torch.float64):
        for n_global in (world << 20, 3 * (1 << 20) + 12345, 70_001, 5, 0):
            lg = tfb.leaf_log2_for(dt, max(n_global, 1))
            a, b = tfb.shard_range(n_global, rank, world, lg)
            x = tfb.philox_fill("uniform_sym", b - a, seed=9, stream=0, offset=a, dtype=dt, device=dev, total=n_global)
            y = tfb.philox_fill("normal", b - a, seed=9, stream=1, offset=a, dtype=dt, device=dev, total=n_global)
            xf = tfb.philox_fill("uniform_sym", n_global, seed=9, stream=0, dtype=dt, device=dev)
            yf = tfb.philox_fill("normal", n_global, seed=9, stream=1, dtype=dt, device=dev)
            assert torch.equal(x, xf[a:b]) and torch.equal(y, yf[a:b])  # shard data independent of the layout
            leaves = -(-n_global // (1 << lg)) if n_global else 0
            aligned = n_global > 0 and leaves % world == 0 and (leaves // world) & (leaves // world - 1) == 0 \
                and n_global % (1 << lg) == 0
            for m in tfb.Method:
                if m is tfb.Method.WIDE and dt != torch.float32:
                    continue
                for dot in (False, True):
                    got = tfb.sharded_reduce(m, x, y if dot else None, n_global=n_global).cpu()
                    # every rank holds the same bits
                    table = [torch.empty_like(got) for _ in range(world)]
                    dist.all_gather(table, got)
                    for t in table:
                        assert torch.equal(t, got) or (torch.isnan(t).all() and torch.isnan(got).all()), (dt, n_global, m, table)
                    # == the merge tree over the per-shard reductions, computed by this rank alone
                    parts = []
                    for r in range(world):
                        ra, rb = tfb.shard_range(n_global, r, world, lg)
                        parts.append(tfb.reduce(m, xf[ra:rb], yf[ra:rb] if dot else None, leaf_log2=lg))
                    want = merge_tree(m, torch.stack(parts, 0)).cpu()
                    assert torch.equal(got, want), (dt, n_global, m, dot, got, want)
                    if aligned:  # exact subtrees: the G-rank result is the 1-GPU result
                        whole = tfb.reduce(m, xf, yf if dot else None, leaf_log2=lg).cpu()
                        assert torch.equal(got, whole), (dt, n_global, m, dot, got, whole)
                    checked += 1
        # rows shard by contiguous row blocks, no collective (gather=True all-gathers the blocks)
        rows_g, cols = 37, 70_001
        lo, hi = tfb.rows_range(rows_g, rank, world)
        X = tfb.rows_scaled_normal(rows_g, cols, seed=3, stream=0, dtype=dt)
        Y = tfb.rows_scaled_normal(rows_g, cols, seed=3, stream=1, dtype=dt)
        full = tfb.reduce_rows(tfb.Method.TWOFOLD_RIGOROUS, X, Y).cpu()
        mine = tfb.sharded_rows(tfb.Method.TWOFOLD_RIGOROUS, X[lo:hi], Y[lo:hi], rows_global=rows_g).cpu()
        assert torch.equal(mine, full[lo:hi])
        every = tfb.sharded_rows(tfb.Method.TWOFOLD_RIGOROUS, X[lo:hi], Y[lo:hi], rows_global=rows_g, gather=True).cpu()
        assert torch.equal(every, full)
        checked += 2
    # host-resident shards through the host-buffer engine (hybrid host path) at world size > 1
    n_global = world << 22
    lg = tfb.leaf_log2_for(torch.float64, n_global)
    a, b = tfb.shard_range(n_global, rank, world, lg)
    xh = tfb.philox_fill_host("uniform_sym", b - a, seed=4, stream=0, offset=a, dtype=torch.float64, pin_memory=True)
    yh = tfb.philox_fill_host("uniform_sym", b - a, seed=4, stream=1, offset=a, dtype=torch.float64, pin_memory=True)
    r = tfb.sharded_run(tfb.Method.TWOFOLD_FAST, xh, yh, n_global=n_global)
    whole = tfb.reduce(tfb.Method.TWOFOLD_FAST,
                       tfb.philox_fill("uniform_sym", n_global, seed=4, stream=0, dtype=torch.float64, device=dev),
                       tfb.philox_fill("uniform_sym", n_global, seed=4, stream=1, dtype=torch.float64, device=dev),
                       leaf_log2=lg).cpu()
    assert float(r.value) == float(whole[0]) and float(r.error) == float(whole[1]), (r, whole)
    checked += 1
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(f"gloo shard layer ok: {checked} checks, world {world}, launches {_lib.lib().tf_launch_count()}")


if __name__ == "__main__":
    main()
