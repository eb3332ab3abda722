"""k_render's TMA staging variant (SS_RENDER_STAGING=tma: cp.async.bulk.tensor tile::gather4 of the
record rows, mbarrier-tracked) gives the same images and n_contrib as the default cp.async staging,
bitwise, on tiny scenes and a ragged multi-block view (run in a subprocess: the variant is selected
from the environment at launch)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2412_00578_b200 import synth
from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
out = {}
for name in ("tiny", "tiny-lowsigma"):
    scene, cams = synth.make_workload(name)
    ds = DeviceScene.from_host(scene)
    rz = Rasterizer(ds, cams[0].width, cams[0].height)
    img, T, nc = rz.render_frame(cams[0], (0.1, 0.2, 0.3), want_T=True, want_ncontrib=True)
    out[name] = (img.cpu().numpy(), nc.cpu().numpy())
scene = synth.orbit_scene(30000, 5)
cams = synth.orbit_cameras(3, 200, 136)
ds = DeviceScene.from_host(scene)
rz = Rasterizer(ds, 200, 136)
for j, c in enumerate(cams):
    rz.ensure_capacity(c)
    img, T, nc = rz.render_frame(c, (0.0, 0.0, 0.0), want_T=True, want_ncontrib=True)
    out["orbit%%d" %% j] = (img.cpu().numpy(), nc.cpu().numpy())
np.savez(sys.argv[1], **{k + "_img": v[0] for k, v in out.items()}, **{k + "_nc": v[1] for k, v in out.items()})
'''


def _run(tmp_path, staging):
    path = str(tmp_path / f"{staging}.npz")
    env = dict(os.environ, SS_RENDER_STAGING=staging)
    subprocess.run([sys.executable, "-c", SCRIPT % ROOT, path], check=True, env=env, timeout=600)
    import numpy as np
    return dict(np.load(path))


def test_tma_staging_equals_cp_async(tmp_path):
    import numpy as np
    a = _run(tmp_path, "cp_async")
    b = _run(tmp_path, "tma")
    assert a.keys() == b.keys() and len(a) >= 10
    for k in a:
        assert np.array_equal(a[k], b[k]), k
