"""Multi-process host logic of KV-head sharding on CPU (gloo, world size 2).

The per-layer collectives need GPUs (tests/test_gpu_sharded.py runs the
sharded arithmetic on one B200 through the loopback communicator); here the
host side is checked with real processes: the NCCL-id rendezvous over
torch.distributed, the head / row partitions every rank applies, and that a
sharded context refuses to start without a GPU."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2602_23592_b200 as kb


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_23592_b200.dist import share_nccl_id, sharded_context
        nid = share_nccl_id()
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        heads = kb.shard_heads(40, 5120, world, rank)
        rows = {n: kb.shard_rows(n, world, rank) for n in (0, 1, 7, 8, 8450, 16280)}
        err = None
        try:
            sharded_context(2, 40, 5120, 13824, 1024, 7, kb.FAST)
        except kb.KeepError as e:
            err = e.kind
        q.put((rank, len(nid), ids, heads, rows, err))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_nccl_id_rendezvous(results):
    ids0 = results[0][2]
    assert all(r[1] == 128 for r in results)
    assert ids0[0] == ids0[1] and all(r[2] == ids0 for r in results)


def test_head_partition(results):
    heads = [r[3] for r in results]
    assert [h[0] for h in heads] == [0, 20] and all(h[1] == 20 for h in heads)
    assert [h[2] for h in heads] == [0, 2560] and all(h[3] == 2560 for h in heads)


def test_row_blocks_cover_rows(results):
    for n in (0, 1, 7, 8, 8450, 16280):
        blocks = [r[4][n] for r in results]
        covered = []
        for r0, m in blocks:
            covered += list(range(r0, r0 + m))
        assert covered == list(range(n)), (n, blocks)


def test_sharded_context_fails_loudly_without_gpu(results):
    assert all(r[5] in ("CudaError", "ConfigError") for r in results)


def test_partition_errors():
    with pytest.raises(kb.KeepError):
        kb.shard_heads(40, 5120, 3, 0)  # 40 heads do not split 3 ways
    with pytest.raises(kb.KeepError):
        kb.shard_rows(10, 2, 2)
