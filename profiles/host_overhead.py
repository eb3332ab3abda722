"""Host-side cost of enqueuing one frame through the public API (run on the GPU box).

The enqueue of a few frames is timed without waiting for the GPU (fewer launches than the
driver's queue holds, so the host never blocks on a full queue); cProfile shows where the
host time goes."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2412_00578_b200 import synth
from paper_2412_00578_b200.raster import DeviceScene, Rasterizer, camera_struct

scene, cams = synth.make_workload("mnr360-3m", n=200000)
rz = Rasterizer(DeviceScene.from_host(scene), cams[0].width, cams[0].height)
rz.ensure_capacity(cams[0])
cs = [camera_struct(c) for c in cams[:8]]
out = torch.empty((3, cams[0].height, cams[0].width), device="cuda")
for _ in range(3):
    for c in cs:
        rz.prepare(c)
        rz.render(out=out)
torch.cuda.synchronize()
best = 1e9
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c in cs:
        rz.prepare(c)
        rz.render(out=out)
    best = min(best, (time.perf_counter() - t0) / len(cs))
    torch.cuda.synchronize()
print(f"host enqueue per frame: {best * 1e6:.1f} us (best of 5, 8 frames each)")
for name, fn in [("preprocess", lambda c: rz.preprocess(c)), ("bin", lambda c: rz.bin(c)),
                 ("sort", lambda c: rz.sort()), ("render", lambda c: rz.render(out=out))]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c in cs:
        fn(c)
    print(f"  {name:10s} host us/call {(time.perf_counter() - t0) / len(cs) * 1e6:8.1f}")
    torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for c in cs:
    rz.prepare(c)
    rz.render(out=out)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
