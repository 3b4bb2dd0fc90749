"""N>1 host path (replicas) on CPU with gloo, world size 2.

bench.py --gpus N runs one independent IRK trajectory per GPU; the only
cross-rank operations are the barrier and the max-over-ranks timing.  Here two
gloo ranks check that aggregation and that the reference arm's rank != 0
exits without work.
"""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    from paper_2010_11377_b200 import replicas
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, lr, w = replicas.world()
    assert (r, lr, w) == (rank, rank, world)
    replicas.barrier()
    local_ms = 100.0 + 50.0 * rank  # rank 1 is the slow one
    mx = replicas.max_over_ranks(local_ms)
    out[rank] = (mx, replicas.whole_job_throughput(10, world, mx))
    dist.destroy_process_group()


def test_gloo_world2_max_and_throughput():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0] == res[1]
    mx, thr = res[0]
    assert mx == 150.0
    assert thr == pytest.approx(2 * 10 / 0.150)


def test_throughput_rejects_nonpositive_time():
    sys.path.insert(0, str(ROOT))
    from paper_2010_11377_b200 import replicas
    with pytest.raises(ValueError):
        replicas.whole_job_throughput(1, 1, 0.0)


def test_reference_arm_nonzero_rank_exits_without_work():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0
    assert r.stdout.strip() == ""
