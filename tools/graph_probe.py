"""Probe: capture spin_generate (C1, the launch-bound configuration) in a CUDA graph and
replay it; checks the images and times direct calls against graph replays."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_00901_b200 import spin  # noqa: E402
from synth import clouds  # noqa: E402

P, Nn = clouds.make_cloud(1)
cen = torch.arange(P.shape[0], dtype=torch.int32, device="cuda")
eng = spin.SpinEngine(torch.from_numpy(P).cuda(), torch.from_numpy(Nn).cuda())
kw = dict(schedule="SS", mode="bilinear")
out = torch.empty((P.shape[0], 8, 8), dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
res = {}
with torch.cuda.stream(s):
    for _ in range(3):
        eng.generate(cen, 8, 0.05, 0.5, out=out, **kw)   # warm-up: chunk table, attributes
    torch.cuda.synchronize()
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            eng.generate(cen, 8, 0.05, 0.5, out=out, **kw)
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        res["graph_equal"] = bool(torch.equal(out, ref))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 200
        e0.record(s)
        for _ in range(n):
            eng.generate(cen, 8, 0.05, 0.5, out=out, **kw)
        e1.record(s)
        torch.cuda.synchronize()
        res["direct_us"] = 1e3 * e0.elapsed_time(e1) / n
        e0.record(s)
        for _ in range(n):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        res["graph_us"] = 1e3 * e0.elapsed_time(e1) / n
    except Exception as ex:  # report, do not crash the probe
        res["error"] = repr(ex)
eng.close()
# CELLS: the centre ordering kernels and the grid are part of the captured call
P3, N3 = clouds.make_cloud(3, n=200000)
cen3 = torch.from_numpy(np.arange(0, 200000, 97, dtype=np.int32)).cuda()
eng3 = spin.SpinEngine(torch.from_numpy(P3).cuda(), torch.from_numpy(N3).cuda())
out3 = torch.empty((cen3.shape[0], 16, 16), dtype=torch.float32, device="cuda")
with torch.cuda.stream(s):
    for _ in range(2):
        eng3.generate(cen3, 16, 0.01, 0.5, out=out3, schedule="SS", prune="cells", mode="nearest")
    torch.cuda.synchronize()
    ref3 = out3.clone()
    try:
        g3 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g3, stream=s):
            eng3.generate(cen3, 16, 0.01, 0.5, out=out3, schedule="SS", prune="cells", mode="nearest")
        out3.zero_()
        g3.replay()
        torch.cuda.synchronize()
        res["cells_graph_equal"] = bool(torch.equal(out3, ref3))
    except Exception as ex:
        res["cells_error"] = repr(ex)
eng3.close()
print(json.dumps(res))
