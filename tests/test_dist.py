"""Multi-process (gloo, world_size 2, CPU) tests of the stream sharding + final gather.

The GPU compute is stood in for by the CPU oracle (test infrastructure): each
rank generates its shard with noise keyed by the global stream id, and the
gathered result must equal the single-process run -- the sharding invariance
the multi-GPU bench relies on.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_09482_b200.distributed import gather_sequences, shard_streams


def test_shard_streams_partition():
    for total in (1, 7, 64, 4096, 4097):
        for world in (1, 2, 3, 8):
            if world > total:
                continue
            shards = [shard_streams(total, world, r) for r in range(world)]
            assert sum(s.count for s in shards) == total
            assert shards[0].offset == 0
            for a, b in zip(shards, shards[1:]):
                assert b.offset == a.offset + a.count
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1
    assert shard_streams(4096, 8, 3).count == 512 and shard_streams(4096, 8, 3).offset == 1536
    with pytest.raises(ValueError):
        shard_streams(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cell as oc
        from paper_1611_09482_b200.cell import CellConfig, build_cell_model

        m = build_cell_model(CellConfig(1, 3, 8, 8, 16, classes=16, init_seed=4))
        o = oc.CellOracle(m, exact=False)
        sh = shard_streams(total, world, rank)
        primer = (np.arange(total) % 16)[sh.offset:sh.offset + sh.count].reshape(1, -1)
        out, _ = oc.generate(o, primer, steps, 2, seed=9, stream_offset=sh.offset)
        full = gather_sequences(torch.as_tensor(out, dtype=torch.int32), sh, total)
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [8, 7])
def test_gloo_sharded_generation_equals_single_process(total):
    from oracle import cell as oc
    from paper_1611_09482_b200.cell import CellConfig, build_cell_model

    steps, world = 12, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = build_cell_model(CellConfig(1, 3, 8, 8, 16, classes=16, init_seed=4))
    ref, _ = oc.generate(oc.CellOracle(m, exact=False), (np.arange(total) % 16).reshape(1, -1),
                         steps, 2, seed=9)
    for r in range(world):
        assert np.array_equal(results[r], ref)
