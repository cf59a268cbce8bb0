"""Multi-GPU path on the CPU: world_size-2 gloo processes exercise the batch
partitioner and the max-over-ranks step timing used by bench.py.  The data
path itself has no collective (batched transforms are independent); each rank
runs the CPU oracle on its shard here as the stand-in for its GPU and the
concatenated shards must equal the single-process result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_00567_b200.distributed import shard_range


def test_shard_ranges_cover_batch():
    for batch in (0, 1, 2, 7, 1 << 20, 1000003):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and b >= a
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, batch, out_dir):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2604_00567_b200.distributed import max_over_ranks, shard_range

    orc = oracle.load_oracle()
    x = orc.random_buffer(n, 99, batch=batch)
    x = orc.round_to(x.view(np.float64), "fp32").view(np.complex128).reshape(batch, n)
    a, b = shard_range(batch, rank, world)
    y = orc.forward(x[a:b], "dual", "fp32", threads=1)
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), y)
    # control plane only: the step time is the slowest rank's
    t = max_over_ranks(0.5 + rank)
    assert t == 0.5 + (world - 1)
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([b - a]))
    assert sum(int(c) for c in counts) == batch
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_batch(tmp_path, orc):
    world, n, batch = 2, 256, 9
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, batch, str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"shard{r}.npy") for r in range(world)])
    x = orc.random_buffer(n, 99, batch=batch)
    x = orc.round_to(x.view(np.float64), "fp32").view(np.complex128).reshape(batch, n)
    want = orc.forward(x, "dual", "fp32")
    assert got.tobytes() == want.tobytes()
