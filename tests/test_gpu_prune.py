"""GPU prune step (NEXT-1: select + compact) versus the oracle's plain selection."""
import numpy as np
import pytest

import oracle
from paper_2412_00578_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ratio", [0.0, 0.3, 0.8, 1.0])
def test_prune_select_and_compact(ratio):
    from paper_2412_00578_b200.raster import DeviceScene, prune
    scene, _ = synth.make_workload("mnr360-3m", n=50000)
    rng = np.random.default_rng(11)
    # many exact ties (integers) plus a continuous part and zeros: every tie-break path
    s = np.where(rng.random(scene.n) < 0.3, 0.0, rng.integers(0, 200, scene.n) * rng.uniform(0.1, 3.0, scene.n))
    s[rng.integers(0, scene.n, 5000)] = 7.0
    ds = DeviceScene.from_host(scene)
    out, keep = prune(ds, torch.from_numpy(s).cuda(), ratio)
    torch.cuda.synchronize()
    want, k = oracle.prune_select(s, ratio)
    assert np.array_equal(keep.cpu().numpy(), want)
    idx = np.nonzero(want)[0]
    assert out.n == len(idx) == scene.n - k
    assert np.array_equal(out.mean_opac.cpu().numpy(), scene.mean_opac[idx])
    assert np.array_equal(out.rot.cpu().numpy(), scene.rot[idx])
    assert np.array_equal(out.scale.cpu().numpy(), scene.scale[idx])
    assert np.array_equal(out.sh.cpu().numpy(), np.transpose(scene.sh[:, idx], (1, 0, 2)))


def test_score_then_prune_renders():
    """Score over views -> prune 90% -> the pruned scene renders through the same path and
    matches the oracle rendering the same pruned scene (the pruned-regime workload)."""
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer, prune
    scene, _ = synth.make_workload("mnr360-3m", n=30000)
    cams = synth.orbit_cameras(12, 320, 208)
    ds = DeviceScene.from_host(scene)
    rz = Rasterizer(ds, 320, 208)
    score = torch.zeros(scene.n, dtype=torch.float64, device="cuda")
    for c in cams:
        rz.render_frame(c)
        rz.prune_score(score)
    out, keep = prune(ds, score, 0.9)
    kept = np.nonzero(keep.cpu().numpy())[0]
    pruned = scene.subset(kept)
    rz2 = Rasterizer(out, 320, 208)
    img = rz2.render_frame(cams[3]).cpu().numpy()
    f = oracle.frame(pruned, cams[3], "accutile")
    assert np.abs(img - f.image).max() <= 1e-4
