"""Experiment: frames/s with 1, 2, 3 concurrent frame workspaces on separate streams."""
import time
import torch
from paper_2412_00578_b200 import synth
from paper_2412_00578_b200.raster import DeviceScene, Rasterizer, camera_struct

scene, cams = synth.make_workload("mnr360-3m")
ds = DeviceScene.from_host(scene)
W, H = cams[0].width, cams[0].height
views = list(range(64))
cs = [camera_struct(cams[v]) for v in views]
for nst in (1, 2, 3, 4):
    rzs = [Rasterizer(ds, W, H, capacity=12_000_000) for _ in range(nst)]
    sts = [torch.cuda.Stream() for _ in range(nst)]
    outs = [torch.empty((3, H, W), device="cuda") for _ in range(nst)]
    def run():
        cur = torch.cuda.current_stream()
        e0 = torch.cuda.Event()
        e0.record(cur)
        for s in sts:
            s.wait_stream(cur)
        for j, c in enumerate(cs):
            k = j % nst
            with torch.cuda.stream(sts[k]):
                rzs[k].prepare(c, sts[k])
                rzs[k].render(out=outs[k], stream=sts[k])
        for s in sts:
            cur.wait_stream(s)
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"streams={nst}: {5 * len(cs) / (ms / 1e3):.1f} frames/s", flush=True)
