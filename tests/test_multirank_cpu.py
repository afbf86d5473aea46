"""The N>1 bench path on CPU: two ranks over gloo (world_size 2).

bench.py runs replicas (each rank the full detection on its own copy of the
graph, no collective on the data path); the only cross-rank step is the
max-over-ranks of the device time and the whole-job aggregation, exercised
here with the same functions bench.py calls."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    local_ms = [12.0, 20.0][rank]
    ms = bench.reduce_max(local_ms, world)
    value = bench.whole_job_gteps(1_000_000_000, ms, world)
    out[rank] = (ms, value)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_max_and_whole_job_value():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for rank in (0, 1):
        ms, value = out[rank]
        assert ms == 20.0
        assert value == pytest.approx(2 * 1e9 / 0.020 / 1e9)


def test_single_rank_is_identity():
    import bench

    assert bench.reduce_max(3.5, 1) == 3.5
    assert bench.whole_job_gteps(10**9, 1000.0, 1) == pytest.approx(1.0)
