"""A small end-to-end run of every libss call for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): tiny scene, all three tile modes, a frame through the 2-stream pipeline
(one-call and graph paths), the pruning score, the backward, one training step's kernels and
the prune step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_00578_b200 import synth  # noqa: E402
from paper_2412_00578_b200.raster import DeviceScene, FramePipeline, Rasterizer, prune  # noqa: E402
from paper_2412_00578_b200.train import AdamConfig, Trainer  # noqa: E402

scene, cams = synth.make_workload("tiny")
cam = cams[0]
ds = DeviceScene.from_host(scene)
for mode in ("3sigma", "snugbox", "accutile"):
    rz = Rasterizer(ds, cam.width, cam.height, mode=mode)
    img, T, nc = rz.render_frame(cam, (0.1, 0.2, 0.3), want_T=True, want_ncontrib=True)
    s = torch.zeros(ds.n, dtype=torch.float64, device="cuda")
    rz.prune_score(s, (0.1, 0.2, 0.3))
    g2 = rz.render_backward(torch.ones_like(img), T, nc, bg=(0.1, 0.2, 0.3))
    rz.preprocess_backward(cam, g2)
    rz.finalize_colours()
    rz.render_stats()
    rz.sorted_keys()
cams2 = synth.orbit_cameras(3, 96, 64)
sc2, _ = synth.make_workload("mnr360-3m", n=4000)
ds2 = DeviceScene.from_host(sc2)
pipe = FramePipeline(ds2, 96, 64, n_streams=2)
pipe.ensure_capacity(cams2)
pipe.render_views(cams2)
pipe.capture(cams2)
pipe.render_views(cams2, graphs=True)
sc = torch.zeros(ds2.n, dtype=torch.float64, device="cuda")
pipe.score_views(cams2, sc)
pruned, keep = prune(ds2, sc, 0.5)
targets = [torch.rand((3, 64, 96), device="cuda") for _ in cams2]
tr = Trainer(DeviceScene(ds2.mean_opac.clone(), ds2.scale.clone(), ds2.rot.clone(), ds2.sh.clone(), ds2.sh_degree),
             cams2, targets, adam=AdamConfig())
for j in range(3):
    tr.step(j)
tr.prune(0.3)
tr.step(0)
torch.cuda.synchronize()
print("sanitize run ok", pruned.n)
