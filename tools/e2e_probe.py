import time, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1811_00901_b200 import spin
from synth import clouds
P, Nn = clouds.make_cloud(2); cen = clouds.make_centres(2, 100000)
hP = torch.from_numpy(P).pin_memory(); hN = torch.from_numpy(Nn).pin_memory()
hC = torch.from_numpy(cen).pin_memory(); hO = torch.empty((100000, 16, 16), dtype=torch.float32).pin_memory()
eng = spin.SpinEngine(hP.cuda(), hN.cuda())
for _ in range(3):
    eng.load_cloud(hP, hN); eng.generate_host(hC.numpy(), 16, 0.02, 0.5, schedule="SS", mode="bilinear", out=hO.numpy())
torch.cuda.synchronize()
for what in ("load", "gen", "both"):
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        if what in ("load", "both"): eng.load_cloud(hP, hN)
        if what in ("gen", "both"): eng.generate_host(hC.numpy(), 16, 0.02, 0.5, schedule="SS", mode="bilinear", out=hO.numpy())
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(what, round(1e3 * np.median(ts), 3), "ms")
_, st = eng.generate(torch.from_numpy(cen).cuda(), 16, 0.02, 0.5, schedule="SS", mode="bilinear", stats=True)
print("kernel", round(st["elapsed_ms"], 3))
