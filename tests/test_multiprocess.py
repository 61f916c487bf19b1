"""N > 1 host logic of bench.py (replicas only, no data-path collective), on CPU
with the gloo backend and world size 2: the job time is the max over ranks and the value
counts every rank's queries; the reference arm runs on rank 0 only."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ws, r, local = bench.dist_env()
    assert (ws, r, local) == (world, rank, rank)
    # rank 1 is the slow one
    t, e = bench.max_over_ranks([100.0 + 50.0 * rank, 200.0 - 30.0 * rank], "cpu")
    out[rank] = (t, e, bench.weak_scaling_value(ws, 10000, 10, t))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_weak_scaling_gloo():
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for rank in (0, 1):
        t, e, v = out[rank]
        assert t == 150.0 and e == 200.0
        assert v == pytest.approx(2 * 10000 * 10 / 0.150)


def test_single_process_is_identity():
    import bench
    assert bench.max_over_ranks([1.5, 2.5], "cpu") == [1.5, 2.5]
    assert bench.weak_scaling_value(1, 100, 2, 10.0) == pytest.approx(20000.0)


def test_reference_arm_runs_on_rank0_only(monkeypatch):
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")

    class A:
        config, ef, steps, warmup, gpus = "C1", 0, 1, 1, 2
    assert bench.reference_arm(A()) == 0  # returns before building any workload


def test_operating_point_is_smallest_ef_reaching_the_target():
    import bench
    sweep = {16: {"recall": 0.79}, 128: {"recall": 0.949}, 136: {"recall": 0.9513}, 160: {"recall": 0.9562},
             256: {"recall": 0.967}}
    assert bench.operating_ef(sweep) == 136
    assert bench.operating_ef(sweep, 0.96) == 256
    assert bench.operating_ef({32: {"recall": 0.2}, 64: {"recall": 0.3}}) == 64  # target out of reach


def test_operating_point_needs_every_query_set():
    # the aggregate 0.95 at ef 130 is not enough when one timed query set sits below it
    import bench
    sweep = {128: {"recall": 0.94956, "recall_per_set": [0.949, 0.9503, 0.9493, 0.9497]},
             130: {"recall": 0.95, "recall_per_set": [0.9495, 0.9506, 0.9498, 0.9501]},
             132: {"recall": 0.95056, "recall_per_set": [0.9502, 0.9512, 0.9503, 0.9506]}}
    assert bench.operating_ef(sweep) == 132
