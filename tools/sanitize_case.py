"""Small spin_generate workload for compute-sanitizer runs (memcheck / racecheck / synccheck)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1811_00901_b200 import spin
from synth import clouds

P, Nn = clouds.bumpy_sphere(5000, 2)
eng = spin.SpinEngine(torch.from_numpy(P).cuda(), torch.from_numpy(Nn).cuda())
cen = torch.arange(0, 5000, 37, dtype=torch.int32, device="cuda")
for mode in ("nearest", "bilinear"):
    for prune in ("brute", "cells"):
        for sched in ("STATIC", "FAC"):
            eng.generate(cen, 16, 0.02, 0.5, mode=mode, prune=prune, schedule=sched)
Pc, Nc = clouds.clustered(8000, 3)
eng.load_cloud(torch.from_numpy(Pc).cuda(), torch.from_numpy(Nc).cuda())
cen = torch.arange(0, 8000, 53, dtype=torch.int32, device="cuda")
eng.generate(cen, 8, 0.01, 0.5, mode="nearest", prune="cells", schedule="SS")
eng.generate(cen, 8, 0.01, 0.5, mode="bilinear", prune="brute", schedule="GSS")
torch.cuda.synchronize()
print("sanitize case ok")
