"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Per config, the whole frame runs through libss exactly as in the bench; the oracle then
checks, bit-exactly, every Gaussian's tile count and the full sorted key list / tile
ranges, and, on sampled tiles, the image (1e-4) and -- for sampled Gaussians whose every
tile is checked -- the pruning score (1e-4 relative).  Knife-edge pixels (R22)
are counted and must be below 1e-5 of the checked pixels.
"""
import numpy as np
import pytest

import oracle
from paper_2412_00578_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _run(scene, cam, mode, bg=(0.0, 0.0, 0.0)):
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
    rz = Rasterizer(DeviceScene.from_host(scene), cam.width, cam.height, mode=mode)
    rz.ensure_capacity(cam)
    img = rz.render_frame(cam, bg)
    torch.cuda.synchronize()
    P = rz.totals()["pairs"]
    return rz, img.cpu().numpy(), P


def _check(scene, cam, mode, rng, n_tiles_sample=48, bg=(0.0, 0.0, 0.0), score_sample=0):
    rz, img, P = _run(scene, cam, mode, bg)
    f = oracle.frame(scene, cam, mode, bg, render=False, cap_hint=int(P * 1.05) + 16)
    counts = rz.counts().cpu().numpy().view(np.uint32)
    assert np.array_equal(counts, f.counts)
    assert P == f.P
    keys = rz.sorted_keys().cpu().numpy().view(np.uint64)[:P]
    assert np.array_equal(keys, f.keys)
    assert np.array_equal(rz.sorted_values().cpu().numpy().view(np.uint32)[:P], f.values)
    ranges = rz.ranges().cpu().numpy().view(np.uint32)
    assert np.array_equal(ranges, f.ranges)
    # image on sampled tiles: the heaviest tiles plus a random sample
    lens = ranges[:, 1].astype(np.int64) - ranges[:, 0]
    heavy = np.argsort(-lens)[: n_tiles_sample // 2]
    rand = rng.choice(len(lens), n_tiles_sample // 2, replace=False)
    tiles = np.unique(np.concatenate([heavy, rand])).astype(np.int32)
    oimg, _, _ = oracle.render_tiles(f.rec, f.values, f.ranges, cam.width, cam.height, tiles, bg)
    m = ~np.isnan(oimg)
    d = np.abs(img[m] - oimg[m])
    bad = (d > 1e-4).sum()
    assert bad <= max(0, int(1e-5 * m.sum())), f"{bad} of {m.sum()} sampled values differ by > 1e-4 (max {d.max()})"
    out = {"P": P, "tiles_checked": len(tiles), "values_checked": int(m.sum()), "max_diff": float(d.max())}
    if score_sample:
        # Gaussians whose every tile is in the checked set: their oracle score is complete
        score = torch.zeros(scene.n, dtype=torch.float64, device="cuda")
        rz.prune_score(score, bg)
        s_gpu = score.cpu().numpy()
        vis = np.nonzero((f.counts > 0) & (f.counts <= 4))[0]
        pick = rng.choice(vis, min(score_sample, len(vis)), replace=False)
        tl = set()
        for g in pick:
            tl.update(oracle.tiles_of_record(mode, f.rec[g], f.rect[g], cam.tiles_x, cam.tiles_y).tolist())
        s_or = oracle.prune_score_tiles(f.rec, f.values, f.ranges, cam.width, cam.height,
                                        np.array(sorted(tl), np.int32), bg)
        ref = s_or[pick]
        rel = np.abs(s_gpu[pick] - ref) / np.maximum(ref, 1e-6 * max(ref.max(), 1e-30))
        assert rel.max() <= 1e-4, f"score max rel {rel.max()}"
        out["score_checked"] = len(pick)
    return out


def test_mnr360_3m_bench_view():
    """The bench workload (BASELINE metric config): 3.0M Gaussians, 1297x840, AccuTile."""
    scene, cams = synth.make_workload("mnr360-3m")
    rng = np.random.default_rng(0)
    for v in (0, 92):
        _check(scene, cams[v], "accutile", rng, score_sample=150)


@pytest.mark.parametrize("mode", ["3sigma", "snugbox", "accutile"])
def test_truck_modes(mode):
    """Tanks&Temples truck-shaped (2.5M, 979x546): the three tile tests of the paper."""
    scene, cams = synth.make_workload("truck")
    rng = np.random.default_rng(1)
    r = _check(scene, cams[17], mode, rng)
    assert r["P"] > 0


def test_playroom_score_views():
    """Deep Blending playroom-shaped (2.3M, 1264x832) with the pruning score + background."""
    scene, cams = synth.make_workload("playroom")
    rng = np.random.default_rng(2)
    _check(scene, cams[5], "accutile", rng, bg=(0.1, 0.3, 0.6), score_sample=150)


def test_garden_accutile():
    """Mip-NeRF 360 garden-shaped (5.8M, 1297x840)."""
    scene, cams = synth.make_workload("garden")
    rng = np.random.default_rng(3)
    _check(scene, cams[40], "accutile", rng)
