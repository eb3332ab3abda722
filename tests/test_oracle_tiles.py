"""Pins of the oracle's tile sets (3-sigma, SnugBox, AccuTile) against the exact
continuous-cell definition, brute force per-pixel scans, Appendix A cases and the
containment chain (Sec. 4.1, Alg. 1, App. A)."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2412_00578_b200 import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = json.load(open(os.path.join(GOLDEN, "accutile_cases.json")))["cases"]
SIGMA_STAR = math.exp(4.5) / 255.0  # t = 9: SnugBox half-extent sqrt(t Sxx) vs 3 sqrt(lmax)


def _case_conic(c):
    if "conic" in c:
        a, b, cc = c["conic"]
        return a, b, cc, c["t"], None
    l1, l2, th = c["cov_diag_theta"]
    th = math.radians(th)
    R = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
    S = R @ np.diag([l1, l2]) @ R.T
    Ci = np.linalg.inv(S)
    return Ci[0, 0], Ci[0, 1], Ci[1, 1], oracle.threshold(c["sigma"]), S


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_accutile_fixture_cases(case):
    tx, ty = case.get("grid", [16, 16])
    a, b, c, t, S = _case_conic(case)
    mx, my = case["mu"]
    acc, n_solves = oracle.accutile(mx, my, a, b, c, t, tx, ty)
    exact = oracle.tiles_exact(mx, my, a, b, c, t, tx, ty)
    assert np.array_equal(acc, exact), "AccuTile != continuous-cell definition"
    r = oracle.rect_snugbox(mx, my, a, b, c, t, tx, ty)
    snug = (r[1] - r[0]) * (r[3] - r[2])
    if "tiles" in case:
        want = sorted(int(rw) * tx + int(cl) for rw, cl in case["tiles"])
        assert acc.tolist() == want
    if "count_accutile" in case:
        assert len(acc) == case["count_accutile"]
    for key in ("snugbox", "count_snugbox"):
        if key in case:
            assert snug == case[key]
    if "count_3sigma" in case:
        D = a * c - b * b
        r3 = oracle.rect_3sigma(mx, my, c / D, -b / D, a / D, tx, ty)
        assert (r3[1] - r3[0]) * (r3[3] - r3[2]) == case["count_3sigma"]
    # cost bound: "counts tiles in time proportional to the shorter side"
    assert n_solves <= min(r[1] - r[0], r[3] - r[2]) + 1
    if "max_solves" in case:
        assert n_solves <= case["max_solves"]
    # rows and columns sweeps give the same set (App. A symmetry)
    for d in (0, 1):
        alt, _ = oracle.accutile(mx, my, a, b, c, t, tx, ty, force_dir=d)
        assert np.array_equal(alt, acc)


def _pixel_hits(mx, my, a, b, c, t, tx, ty, rect):
    """Brute force over integer pixel centres (R3) inside the rect's tiles: the tiles
    holding at least one pixel with q <= t (alpha >= 1/255)."""
    x0, x1, y0, y1 = rect
    xs = np.arange(x0 * 16, x1 * 16, dtype=np.float64)
    ys = np.arange(y0 * 16, y1 * 16, dtype=np.float64)
    X, Y = np.meshgrid(xs, ys)
    xd, yd = X - mx, Y - my
    q = a * xd * xd + 2 * b * xd * yd + c * yd * yd
    hit = (q <= t) & (X < tx * 16) & (Y < ty * 16)
    tiles = np.unique((Y[hit] // 16).astype(np.int64) * tx + (X[hit] // 16).astype(np.int64))
    return tiles.astype(np.uint32)


def test_random_battery_exactness_and_containment():
    """F6 battery: random conics, cond <= 1e3, sigma in (1/255, 1), means on a
    40x40-tile grid (with off-grid margins).  Checks per conic:
      AccuTile == exact continuous-cell set (App. A)
      AccuTile subset of SnugBox rect; SnugBox rect subset of 3-sigma rect iff sigma <= sigma*
      per-pixel alpha >= 1/255 hits subset of AccuTile (R23)
      line solves <= shorter side + 1; rows sweep == columns sweep."""
    n = 100000
    T = 40
    mx, my, cxx, cxy, cyy, sig = synth.random_conics(n, seed=5, tiles=T)
    viol_low = viol_high = 0
    phantom = total = 0
    for i in range(n):
        D = cxx[i] * cyy[i] - cxy[i] * cxy[i]
        a, b, c = cyy[i] / D, -cxy[i] / D, cxx[i] / D
        t = oracle.threshold(float(sig[i]))
        acc, ns = oracle.accutile(mx[i], my[i], a, b, c, t, T, T)
        ex = oracle.tiles_exact(mx[i], my[i], a, b, c, t, T, T)
        assert np.array_equal(acc, ex), i
        r = oracle.rect_snugbox(mx[i], my[i], a, b, c, t, T, T)
        rx = acc % T
        ry = acc // T
        assert np.all((rx >= r[0]) & (rx < r[1]) & (ry >= r[2]) & (ry < r[3]))
        assert ns <= min(r[1] - r[0], r[3] - r[2]) + 1 or len(acc) == 0
        r3 = oracle.rect_3sigma(mx[i], my[i], cxx[i], cxy[i], cyy[i], T, T)
        inside = (r[0] >= r3[0] and r[1] <= r3[1] and r[2] >= r3[2] and r[3] <= r3[3]) or len(acc) == 0
        if sig[i] <= SIGMA_STAR * (1 - 1e-9):
            viol_low += not inside
        else:
            viol_high += not inside
        if i % 10 == 0:
            alt, _ = oracle.accutile(mx[i], my[i], a, b, c, t, T, T, force_dir=1 - (len(acc) % 2))
            assert np.array_equal(alt, acc)
            if len(acc):
                hits = _pixel_hits(mx[i], my[i], a, b, c, t, T, T, r)
                assert np.all(np.isin(hits, acc))
                phantom += len(acc) - len(hits)
                total += len(acc)
    assert viol_low == 0, "SnugBox must be inside the 3-sigma square when t <= 9 (R17)"
    assert viol_high > 0, "above sigma* the 3-sigma square must miss real extent somewhere (R17)"
    # phantom tiles (continuous cell hit, no pixel centre hit) exist but are a minority (R23)
    assert 0 < phantom < 0.25 * total


def test_accutile_count_equals_emit_on_scene():
    """Count mode == emit mode ("once to count ... once to populate"), on a scene."""
    scene, cams = synth.make_workload("tiny")
    cam = cams[0]
    for mode in ("3sigma", "snugbox", "accutile"):
        rec, rect, cnt = oracle.project(scene, cam, mode)
        for i in range(scene.n):
            tl = oracle.tiles_of_record(mode, rec[i], rect[i], cam.tiles_x, cam.tiles_y)
            assert len(tl) == cnt[i]
            assert len(np.unique(tl)) == len(tl)


def test_mode_containment_on_scene():
    """Per Gaussian of the tiny scene: AccuTile set subset of SnugBox set; SnugBox rect
    subset of 3-sigma rect whenever sigma <= sigma* (R17)."""
    scene, cams = synth.make_workload("tiny")
    cam = cams[0]
    recA, rectA, cA = oracle.project(scene, cam, "accutile")
    recS, rectS, cS = oracle.project(scene, cam, "snugbox")
    rec3, rect3, c3 = oracle.project(scene, cam, "3sigma")
    assert np.array_equal(recA, recS)
    assert np.all(cA <= cS)
    for i in range(scene.n):
        if cA[i] == 0:
            continue
        ta = set(oracle.tiles_of_record("accutile", recA[i], rectA[i], cam.tiles_x, cam.tiles_y).tolist())
        ts = set(oracle.tiles_of_record("snugbox", recS[i], rectS[i], cam.tiles_x, cam.tiles_y).tolist())
        assert ta <= ts
        if scene.mean_opac[i, 3] <= SIGMA_STAR * (1 - 1e-6):
            t3 = set(oracle.tiles_of_record("3sigma", rec3[i], rect3[i], cam.tiles_x, cam.tiles_y).tolist())
            assert ts <= t3
