"""Per-tile list-length statistics of one view per workload (diagnostic, GPU)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2412_00578_b200 import synth
from paper_2412_00578_b200.raster import DeviceScene, Rasterizer

for name, mode in [("mnr360-3m", "accutile"), ("mnr360-3m", "3sigma"), ("truck", "accutile"),
                   ("garden", "accutile"), ("playroom", "accutile")]:
    scene, cams = synth.make_workload(name)
    rz = Rasterizer(DeviceScene.from_host(scene), cams[0].width, cams[0].height, mode=mode)
    for v in (0, len(cams) // 2):
        rz.ensure_capacity(cams[v])
        rz.render_frame(cams[v])
        r = rz.ranges().cpu().numpy().astype(np.int64)
        L = r[:, 1] - r[:, 0]
        q = np.percentile(L, [50, 90, 99, 100])
        print(f"{name:10s} {mode:8s} v{v:3d} P={L.sum():9d} tiles={len(L)} mean={L.mean():7.0f} "
              f"p50/p90/p99/max={q.astype(int).tolist()} >2048:{(L > 2048).sum()} >4096:{(L > 4096).sum()} "
              f">8192:{(L > 8192).sum()} pairs_in_>4096={L[L > 4096].sum() / max(1, L.sum()):.3f}", flush=True)
    del rz
    torch.cuda.empty_cache()
