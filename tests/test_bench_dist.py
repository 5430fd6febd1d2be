"""Multi-rank plumbing of bench.py on CPU (gloo, world size 2): the timed
region is reduced as the max over ranks and replicas aggregate their units
(replicas only, no data-path collective)."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    t = bench.max_over_ranks(1.0 + rank * 0.5, world, device="cpu")
    q.put((rank, t, bench.replica_value(1000.0, world, t)))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_replica_value_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank sees the slowest rank's time; value = all ranks' units / that time
    assert [t for _, t, _ in res] == [1.5, 1.5]
    assert all(abs(v - 2000.0 / 1.5) < 1e-9 for _, _, v in res)


def test_single_rank_identity():
    import bench
    assert bench.max_over_ranks(0.25, 1) == 0.25
    assert bench.replica_value(10.0, 1, 0.5) == 20.0
