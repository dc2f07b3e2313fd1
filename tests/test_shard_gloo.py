"""World-size-2 gloo test of the multi-GPU sharding logic on CPU.

Each rank takes its contiguous (b,h) range of a global problem (tkb_shard_range, the same
call bench.py makes), computes its shard with the CPU oracle, and the gathered result must
equal the single-process result bit for bit: shards are independent, no collective touches
the data path (the all_gather here is verification only).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, H, N, D, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    from oracle import oracle as orc
    from paper_2410_20399_b200 import attention as A

    q, k, v = orc.qkv(77, B, H, N, D)
    units = B * H
    b, e = A.shard_range(units, rank, world)
    flat = lambda x: x.reshape(units, N, D)  # noqa: E731
    o, lse = orc.attn_fwd(flat(q)[b:e], flat(k)[b:e], flat(v)[b:e], causal=True, nthreads=1)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([e - b]))
    maxn = int(max(s.item() for s in sizes))
    mine = torch.zeros(maxn, N, D, dtype=torch.float64)
    mine[: e - b] = torch.from_numpy(o)
    got = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(got, mine)
    if rank == 0:
        full = torch.cat([g[: int(s.item())] for g, s in zip(got, sizes)]).numpy()
        np.save(os.path.join(out_dir, "sharded.npy"), full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_bh_sharding_matches_single_process(tmp_path, world):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    from oracle import oracle as orc

    B, H, N, D = 2, 3, 96, 64
    mp.spawn(_worker, args=(world, _free_port(), B, H, N, D, str(tmp_path)), nprocs=world, join=True)
    q, k, v = orc.qkv(77, B, H, N, D)
    ref, _ = orc.attn_fwd(q.reshape(-1, N, D), k.reshape(-1, N, D), v.reshape(-1, N, D), causal=True)
    assert np.array_equal(np.load(tmp_path / "sharded.npy"), ref)
