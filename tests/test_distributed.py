"""Multi-process sharding of independent meshes (BASELINE configs[4]) over
torch.distributed with the gloo backend, world size 2, on CPU.  The worker is
a host-side stand-in (mesh generation and topology summary need no GPU); on
the box the same code runs `shard.run_item` per rank over NCCL."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_13168_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _host_worker(spec):
    import paper_2105_13168_b200 as dt
    info = dt.TriangleMesh.generate(spec).info()
    return {"spec": spec, "V": info["V"], "genus": info["genus"], "pid": os.getpid()}


def _rank_main(rank, world, port, items, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = shard.run_sharded(items, rank, world, _host_worker, dist)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_shard_slices_partition():
    items = list(range(13))
    parts = [shard.shard(items, r, 4) for r in range(4)]
    assert sorted(x for p in parts for x in p) == items
    assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        shard.shard(items, 4, 4)


def test_batch_specs_cover_genera():
    specs = shard.batch_specs(64, 32)
    assert len(specs) == 64 and {int(s.split(":")[1]) for s in specs} == set(range(1, 33))


def test_gloo_world2_gathers_all_items_in_order():
    items = shard.batch_specs(6, 3, resolution=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, items, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    merged = results[0]
    assert [r["spec"] for r in merged] == items
    assert [r["genus"] for r in merged] == [1, 2, 3, 1, 2, 3]
    # the two ranks really split the work
    assert len({r["pid"] for r in merged}) == 2
    assert [r["spec"] for r in results[1]] == items[1::2]
