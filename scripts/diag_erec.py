"""Emission-record types of one frame (diagnostic, GPU)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2412_00578_b200 import synth
from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
scene, cams = synth.make_workload("mnr360-3m")
rz = Rasterizer(DeviceScene.from_host(scene), cams[0].width, cams[0].height)
rz.ensure_capacity(cams[0]); rz.render_frame(cams[0])
er = rz.emit_records().cpu().numpy().view(np.uint32)
vis = rz.depth_keys().cpu().numpy().view(np.uint32) != 0xFFFFFFFF
info = er[vis, 1]
spn = (info & 0x800) != 0; ent = (info & 0x100) != 0; big = ~spn & ~ent
ne = info >> 12
print("visible", vis.sum(), "span-inline", spn.sum(), "entry-inline", ent.sum(), "big", big.sum())
print("entries total", ne.sum(), "big entries", ne[big].sum(), "max", ne.max())
print("spans per span-inline:", np.bincount(info[spn] & 0xFF))
print("entries per Gaussian hist:", np.bincount(np.minimum(ne, 20)))
