"""GPU test of the shared dealer: one schedule dealt to two
processes through a counter mapped with CUDA IPC.  Run on one GPU (both processes share
it; neither waits on the other: each CTA only grabs chunks until the table is
exhausted), it exercises the same dealing and partial-output contract a multi-GPU run
uses (the paper's master dealing to workers on many nodes).  The partial
images of the two processes must sum to the ORACLE's images (NEAREST counts: exact), every
chunk dealt exactly once."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCHEDS = ("SS", "STATIC", "GSS", "FAC")
PRUNES = ("brute", "cells")


def _worker(rank, handle, barrier, q):
    sys.path.insert(0, ROOT)
    import torch
    from paper_1811_00901_b200 import spin
    from synth import clouds
    torch.cuda.set_device(0)
    P, Nn = clouds.bumpy_sphere(20000, 41)
    cen = torch.arange(20000, dtype=torch.int32, device="cuda")
    eng = spin.SpinEngine(torch.from_numpy(P).cuda(), torch.from_numpy(Nn).cuda())
    dealer = spin.Dealer.open(handle)
    res = {}
    for prune in PRUNES:
        for sched in SCHEDS:
            barrier.wait()                      # the parent has reset the counter
            out = torch.zeros((20000, 16, 16), dtype=torch.float32, device="cuda")
            _, st = eng.generate(cen, 16, 0.02, 0.5, schedule=sched, mode="nearest", out=out,
                                 prune=prune, P=2 * 148, grid=148, cta_offset=rank * 148,
                                 shared_counter=dealer.ptr, stats=True, cta_capacity=148)
            torch.cuda.synchronize()
            res[(prune, sched)] = (out.cpu().numpy(), int(st["cta_units"].sum()), st["G"])
            barrier.wait()
    dealer.close()
    eng.close()
    q.put((rank, res))


def test_shared_dealer_two_processes():
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    from paper_1811_00901_b200 import spin
    from synth import clouds
    from oracle import spin_oracle_cpp as OC
    P, Nn = clouds.bumpy_sphere(20000, 41)
    eng = spin.SpinEngine(torch.from_numpy(P).cuda(), torch.from_numpy(Nn).cuda())
    # the expected images come from the oracle (Alg. 1), not from the GPU
    ref = OC.generate(P, Nn, np.arange(20000), 16, 0.02, 0.5, OC.NEAREST).astype(np.float32)
    dealer = spin.Dealer()
    ctx = mp.get_context("spawn")
    barrier, q = ctx.Barrier(3), ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, dealer.ipc_handle(), barrier, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        for _ in range(len(PRUNES) * len(SCHEDS)):
            dealer.reset()
            torch.cuda.synchronize()
            barrier.wait()                  # workers start this schedule
            barrier.wait()                  # workers done
        res = dict(q.get(timeout=300) for _ in range(2))
    finally:
        for p in procs:
            p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    for key in res[0]:
        a, ua, G = res[0][key]
        b, ub, _ = res[1][key]
        np.testing.assert_array_equal(a + b, ref, err_msg=str(key))
        assert ua + ub == -(-20000 // G), (key, ua, ub)
        # disjoint: an image written by both would double its counts
        assert not np.any((a.reshape(20000, -1).sum(1) > 0) & (b.reshape(20000, -1).sum(1) > 0))
    dealer.close()
    eng.close()


def test_bench_torchrun_shared_dealer_two_ranks():
    """bench.py under torchrun with two ranks and the shared dealer (the
    paper's master dealing one schedule to every worker): both ranks on
    cuda:0 (this pool has one GPU per call; the ranks never wait on each other), gloo for
    the barrier and the max-over-ranks timing.  Rank 0 prints one parseable JSON line with
    the whole job's pairs."""
    import json
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--config", "1", "--dealer", "shared", "--steps", "3", "--warmup", "3",
           "--dist-backend", "gloo", "--same-device", "--no-cpu-baseline", "--no-e2e", "--no-dls"]
    r = subprocess.run(cmd, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["pairs"]["visited"] == 2000 * 2000          # one schedule of C1 over both ranks
    assert "shared counter" in d["config"]["parallelism"]
    assert d["value"] > 0 and d["ms_per_step"] > 0
