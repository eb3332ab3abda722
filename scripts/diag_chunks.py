"""Pairs and 4x4-super-tile entries per chunk of 4096 depth-ordered Gaussians (diagnostic, GPU)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2412_00578_b200 import synth
from paper_2412_00578_b200.raster import DeviceScene, Rasterizer

for name in ["mnr360-3m", "garden", "truck"]:
    scene, cams = synth.make_workload(name)
    cam = cams[0]
    ds = DeviceScene.from_host(scene)
    out = {}
    for mode in ("snugbox", "accutile"):
        rz = Rasterizer(ds, cam.width, cam.height, mode=mode)
        rz.ensure_capacity(cam)
        rz.render_frame(cam)
        nv = rz.totals()["n_visible"]
        order = rz.order().cpu().numpy()[:nv]
        er = rz.emit_records().cpu().numpy().view(np.uint32)[order]
        out[mode] = (order, er)
        del rz
    order, er_s = out["snugbox"]
    _, er_a = out["accutile"]
    cnt = er_a[:, 0].astype(np.int64)
    pr = er_s[:, 6]
    x0, x1 = pr & 0xFF, (pr & 0xFF) + ((pr >> 8) & 0xFF) + 1
    y0, y1 = (pr >> 16) & 0xFF, ((pr >> 16) & 0xFF) + (pr >> 24) + 1
    ent = ((x1 - 1) // 4 - x0 // 4 + 1).astype(np.int64) * ((y1 - 1) // 4 - y0 // 4 + 1)
    C = 4096
    nck = (len(cnt) + C - 1) // C
    pc = np.add.reduceat(cnt, np.arange(0, len(cnt), C))
    ec = np.add.reduceat(ent, np.arange(0, len(cnt), C))
    print(f"{name}: nv={len(cnt)} P={cnt.sum()} E~{ent.sum()} chunks={nck}")
    print("  pairs/chunk  mean %.0f max %.0f  first8 %s" % (pc.mean(), pc.max(), pc[:8].tolist()))
    print("  entries/chunk mean %.0f max %.0f first8 %s" % (ec.mean(), ec.max(), ec[:8].tolist()))
    print("  max pairs per Gaussian %d, max entries %d, Gaussians > 256 pairs: %d" % (cnt.max(), ent.max(), (cnt > 256).sum()))
    del ds
    torch.cuda.empty_cache()
