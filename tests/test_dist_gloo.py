"""Multi-rank host path on CPU (gloo, world_size 2): each rank owns the
queries [rank*Q, (rank+1)*Q) of the stream (weak scaling, no data-path
collective), bench.Dist reduces times with MAX and counts with SUM, and the
gathered verdicts equal a single-process run of the whole stream.  The C
oracle stands in for the device here (host logic only; the GPU path is covered
by the gpu-marked tests)."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

from conftest import ROOT

Q = 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as td

    import bench
    from oracle import oracle
    from paper_2601_21552_b200 import synth

    d = bench.Dist(world, rank, backend="gloo")
    fb = synth.generate("c3", Q, first=rank * Q, names=False)
    res = oracle.solve_flat(fb, 30.0)
    t_max = d.max(float(rank + 1))
    n_sum = d.sum(float(Q))
    gathered = [None] * world
    td.all_gather_object(gathered, res["verdict"].tolist())
    if rank == 0:
        out.put((t_max, n_sum, sum(gathered, [])))
    d.close()


def test_two_rank_sharding_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    t_max, n_sum, verdicts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t_max == 2.0 and n_sum == 2 * Q
    from oracle import oracle
    from paper_2601_21552_b200 import synth
    whole = oracle.solve_flat(synth.generate("c3", 2 * Q, names=False), 30.0)
    assert np.array_equal(np.array(verdicts, dtype=np.int8), whole["verdict"])
