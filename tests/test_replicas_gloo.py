"""Multi-rank harness logic of bench.py on CPU (gloo, world_size 2): disjoint per-rank query batches,
max-over-ranks timing and the whole-job throughput.  The path itself runs one index per GPU as
independent replicas by default: no data-path collective on this path; the document-sharded
protocol and its all-gathers are covered by tests/test_sharded_gloo.py."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    import datagen
    cfg = datagen.CONFIGS["tiny"]
    nb = 3
    starts = [bench.query_batch_start(rank, nb, b, 16) for b in range(nb)]
    firsts = [datagen.queries(cfg, st, 16)[1][:3].tolist() for st in starts]
    my_ms = 10.0 + 5.0 * rank                        # rank 1 is the slow one
    mx = bench.max_over_ranks(my_ms, ws)
    dist.barrier()
    out[rank] = (starts, firsts, mx, bench.job_qps(16, 4, ws, mx))
    dist.destroy_process_group()


def test_two_ranks_disjoint_batches_and_max_time():
    ws, port = 2, _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    s0, f0, m0, q0 = out[0]
    s1, f1, m1, q1 = out[1]
    assert not set(s0) & set(s1)                      # disjoint query rows per rank
    assert f0 != f1                                   # hence different batches
    assert m0 == m1 == 15.0                           # both ranks report the slowest rank's time
    assert q0 == q1 == pytest.approx(16 * 4 * 2 / 0.015)  # all ranks' queries / max time
