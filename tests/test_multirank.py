"""CPU tests of bench.py's multi-rank plumbing (world_size 2 over gloo) and of its
reference arm.  The spin path itself shards as independent replicas:
the only cross-rank operations are the barrier and the max-over-ranks timing."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    bench.dist_init("gloo")
    t = bench.allreduce_max(float(rank * 10 + 1))
    s = bench.allreduce_sum(float(rank + 1))
    bench.barrier()
    cen = bench.rank_centres(3, 1_000_000, rank)[:1000]
    strong = bench.rank_centres(1, 2000, rank, world, strong=True)

    class FakeDealer:            # the IPC calls need a GPU; the handle exchange does not
        def __init__(self, h=b"H" * 64):
            self.h = h

        def ipc_handle(self):
            return self.h

        @classmethod
        def open(cls, h):
            return cls(b"opened:" + h[:8])

    class FakeSpin:
        Dealer = FakeDealer

    d = bench.share_dealer(FakeSpin, rank, world)
    q.put((rank, t, cen.tolist(), s, strong.tolist(), d.h))
    dist.destroy_process_group()


def test_gloo_two_ranks_max_and_distinct_shards():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] == 11.0          # max over ranks
    assert res[0][3] == res[1][3] == 3.0           # sum over ranks (pairs, images)
    a, b = np.asarray(res[0][2]), np.asarray(res[1][2])
    assert not np.array_equal(a, b)               # ranks run distinct images
    # strong scaling: the configured centres split into disjoint contiguous shards
    s0, s1 = res[0][4], res[1][4]
    assert s0 + s1 == list(range(2000)) and len(s0) == len(s1) == 1000
    # shared dealer: rank 0 owns the counter, rank 1 maps rank 0's handle
    assert res[0][5] == b"H" * 64 and res[1][5] == b"opened:HHHHHHHH"


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "1", "--steps", "2", "--warmup", "1", "--cpu-seconds", "2"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "pair-evals/s"
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""
