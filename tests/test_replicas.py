"""Multi-process (world size 2, gloo, CPU) checks of the replica host logic
used by bench.py --gpus N: distinct per-rank inputs, max-over-ranks timing,
whole-job throughput, column splitting."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

import mht_inputs as mi
from paper_2605_21828_b200 import replicas


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = mi.WORKLOADS["c1"]
    c = replicas.rank_coefficients(w, 2, rank)
    y = replicas.rank_adjoint_inputs(w, 2, rank)
    my_time = 1.0 + rank  # rank 1 is the slowest
    replicas.barrier(world)
    t = replicas.allreduce_max(my_time, world)
    out.put((rank, float(c[0, 0].real), float(y[0, 0].real), t,
             replicas.job_throughput(66, world, t)))
    dist.destroy_process_group()


def test_world2_gloo_replicas():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, c0, y0, t0, v0), (r1, c1, y1, t1, v1) = res
    assert c0 != c1 and y0 != y1                 # replicas transform different columns
    assert t0 == t1 == 2.0                       # max over ranks
    assert v0 == v1 == pytest.approx(66 * 2 / 2.0)
    # rank 0 reproduces the single-GPU inputs
    w = mi.WORKLOADS["c1"]
    assert np.array_equal(replicas.rank_coefficients(w, 2, 0), mi.workload_coefficients(w, 2))


@pytest.mark.parametrize("total,world", [(32, 2), (33, 4), (5, 8), (64, 3)])
def test_split_columns_partition(total, world):
    spans = [replicas.split_columns(total, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == total
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and b >= a
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1
