"""The N > 1 path of bench.py on CPU (gloo, world_size 2): replicas only — every
rank builds its own copy of the workload, the job's step time is the max over ranks, value = n * ws / max, and
the reference arm prints on rank 0 only."""
import io
import os
import sys
from contextlib import redirect_stdout

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, ws, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        import bench
        import synth

        assert bench.dist_env() == (ws, rank, rank)
        ms_max, value = bench.job_throughput(10.0 + rank, 1000, ws)
        # replicas: each rank generates an independent instance (seed = rank)
        cfg = synth.C1.scaled(300)
        a = synth.gen_points(cfg, seed=rank)
        buf = io.StringIO()

        class A:
            ref_sample, warmup, steps = 200, 0, 1

        with redirect_stdout(buf):
            bench.run_reference(A, cfg)
        q.put((rank, ms_max, value, a[:4].tolist(), buf.getvalue()))
    finally:
        dist.destroy_process_group()


def test_replicas_rank_max_and_reference_on_rank0():
    ws, port = 2, 29613
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(ws):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(ws):
        _, ms_max, value, _, out = res[r]
        assert ms_max == 11.0  # the slowest rank's step time, on every rank
        assert value == pytest.approx(1000 * ws / 0.011)
    assert res[0][3] != res[1][3]  # independent replicas
    assert '"impl": "reference"' in res[0][4] and res[1][4] == ""  # rank 0 alone runs and prints the oracle arm
