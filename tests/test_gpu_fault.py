"""Fault injection: a build of libss with the AccuTile tangent-point row
test dropped (-DSS_FAULT_SKIP_TANGENT_ROW, in both the float32 and float64 tile geometry) must
be caught by the parity checks -- its tile counts differ from the oracle's on the tiny scene --
while the normal build matches.  The variant is built into libss_fault.so and loaded in a
subprocess (SS_LIB_PATH), so the normal library is untouched."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHECK = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import oracle
from paper_2412_00578_b200 import synth
from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
bad = 0
for name in ("tiny", "tiny-lowsigma"):
    scene, cams = synth.make_workload(name)
    rz = Rasterizer(DeviceScene.from_host(scene), cams[0].width, cams[0].height, mode="accutile")
    rz.render_frame(cams[0])
    f = oracle.frame(scene, cams[0], "accutile", render=False)
    bad += int((rz.counts().cpu().numpy().view(np.uint32) != f.counts).sum())
print("MISMATCHES", bad)
'''


def _mismatches(env):
    out = subprocess.run([sys.executable, "-c", CHECK % ROOT], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return int(out.stdout.strip().split()[-1])


def test_fault_build_is_caught():
    env = dict(os.environ, SS_BUILD_TAG="fault", NVCC_APPEND_FLAGS="-DSS_FAULT_SKIP_TANGENT_ROW")
    subprocess.run([sys.executable, "-m", "paper_2412_00578_b200.build"], cwd=ROOT, env=env, check=True,
                   capture_output=True, timeout=1200)
    fault = dict(os.environ, SS_LIB_PATH=os.path.join(ROOT, "paper_2412_00578_b200", "libss_fault.so"))
    assert _mismatches(fault) > 0
    assert _mismatches(dict(os.environ)) == 0
