"""torchrun entry: the fused peer combine (tf_reduce_peer) == NCCL all-gather + merge
== single-device result, bit for bit, over repeated epochs (run with --nproc-per-node G)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import dist as tdist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    checked = 0
    for dt in (torch.float32, torch.float64):
        for n in (0, 5, 100_003, 1 << 22):
            n_global = n * world
            lg = tfb.leaf_log2_for(dt, max(n_global, 1))
            a, b = tfb.shard_range(n_global, rank, world, lg)
            x = tfb.philox_fill("uniform_sym", b - a, seed=8, stream=0, offset=a, dtype=dt, device=dev, total=n_global)
            y = tfb.philox_fill("uniform_sym", b - a, seed=8, stream=1, offset=a, dtype=dt, device=dev, total=n_global)
            for m in tfb.Method:
                if m is tfb.Method.WIDE and dt != torch.float32:
                    continue
                ref = tfb.sharded_reduce(m, x, y, n_global=n_global, force_collective=True, combine="nccl").cpu()
                for _ in range(3):  # several epochs through both parities
                    got = tfb.sharded_reduce(m, x, y, n_global=n_global, combine="peer").cpu()
                    assert torch.equal(got, ref) or (torch.isnan(got).all() and torch.isnan(ref).all()), (dt, n, m, got, ref)
                    checked += 1
            if world == 1 and n > 0:
                whole = tfb.reduce(tfb.Method.TWOFOLD_FAST, x, y, leaf_log2=lg).cpu()
                assert torch.equal(tfb.sharded_reduce(tfb.Method.TWOFOLD_FAST, x, y, n_global=n_global,
                                                      combine="peer").cpu(), whole)
    got = tfb.sharded_reduce(tfb.Method.TWOFOLD_RIGOROUS, x, y, n_global=n_global, combine="peer",
                             track_product=True).cpu()
    ref = tfb.sharded_reduce(tfb.Method.TWOFOLD_RIGOROUS, x, y, n_global=n_global, force_collective=True,
                             track_product=True).cpu()
    assert torch.equal(got, ref)
    # the TMA loader finishes the combine inside its own single launch: force it
    from paper_1401_0248_b200 import _lib
    for loader in (2, 3, 6, 7):
        _lib.lib().tf_set_loader(loader)
        got = tfb.sharded_reduce(tfb.Method.TWOFOLD_FAST, x, y, n_global=n_global, combine="peer").cpu()
        ref = tfb.sharded_reduce(tfb.Method.TWOFOLD_FAST, x, y, n_global=n_global, combine="nccl",
                                 force_collective=True).cpu()
        assert torch.equal(got, ref), (loader, got, ref)
        checked += 1
    _lib.lib().tf_set_loader(0)
    assert not tdist.peer_combine_error()
    # combine="auto": the one-time self-check (peer vs NCCL on known data) passes on every rank
    for acc in (torch.float32, torch.float64):
        used = tfb.combine_in_use(None, dev, acc)
        assert used == "peer", used
    if world > 1:  # auto then routes device shards through the fused kernel
        got = tfb.sharded_reduce(tfb.Method.TWOFOLD_FAST, x, y, n_global=n_global, combine="auto").cpu()
        ref = tfb.sharded_reduce(tfb.Method.TWOFOLD_FAST, x, y, n_global=n_global, combine="nccl").cpu()
        assert torch.equal(got, ref)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(f"peer combine ok: {checked} checks, world {world}")


if __name__ == "__main__":
    main()
