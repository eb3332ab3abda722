"""Pins of the oracle's scan / sort / ranges / render / score (Sec. 3.2,
Eqs. 5-7, Sec. 4.2.1 Eqs. 20-21) against printed examples, library
routines, brute force and finite differences."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2412_00578_b200 import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RS = json.load(open(os.path.join(GOLDEN, "render_score_examples.json")))


def test_scan_examples():
    """[1,0,3] -> offsets [0,1,1], total 4; [] -> 0; random vs cumsum."""
    off, tot = oracle.exclusive_scan(np.array([1, 0, 3]))
    assert off.tolist() == [0, 1, 1] and tot == 4
    off, tot = oracle.exclusive_scan(np.zeros(0, np.uint32))
    assert tot == 0
    rng = np.random.default_rng(0)
    c = rng.integers(0, 50, 100000).astype(np.uint32)
    off, tot = oracle.exclusive_scan(c)
    ref = np.concatenate([[0], np.cumsum(c.astype(np.uint64))])
    assert np.array_equal(off, ref[:-1]) and tot == ref[-1]


def test_sort_is_stable_and_matches_library():
    """P:174 'sorts the key array, ordering Gaussian indices by tile and then depth';
    stable (R14).  Examples S:298-300 and numpy's stable argsort as the library routine."""
    d2, d1 = int(np.float32(2.0).view(np.uint32)), int(np.float32(1.0).view(np.uint32))
    k, v = oracle.sort_pairs(np.array([(5 << 32) | d2, (5 << 32) | d1], np.uint64),
                             np.array([0, 1], np.uint32))
    assert v.tolist() == [1, 0]
    rng = np.random.default_rng(1)
    keys = (rng.integers(0, 300, 200000).astype(np.uint64) << np.uint64(32)) | \
        rng.integers(0, 50, 200000).astype(np.uint64)  # many equal keys
    vals = np.arange(200000, dtype=np.uint32)
    k, v = oracle.sort_pairs(keys, vals)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(k, keys[order]) and np.array_equal(v, vals[order])
    k2, v2 = oracle.sort_pairs(k, v)   # already sorted: unchanged
    assert np.array_equal(k2, k) and np.array_equal(v2, v)


def test_tile_ranges():
    """P:175; all keys in tile 5 -> [0,n); empty tiles (0,0); vs searchsorted."""
    keys = np.array([5 << 32] * 7, np.uint64)
    r = oracle.tile_ranges(keys, 16)
    assert r[5].tolist() == [0, 7] and r.sum() == 7
    rng = np.random.default_rng(2)
    keys = np.sort((rng.integers(0, 1000, 50000).astype(np.uint64) << np.uint64(32)))
    r = oracle.tile_ranges(keys, 1200)
    tiles = (keys >> np.uint64(32)).astype(np.int64)
    lo = np.searchsorted(tiles, np.arange(1200), "left")
    hi = np.searchsorted(tiles, np.arange(1200), "right")
    empty = lo == hi
    assert np.array_equal(r[~empty, 0], lo[~empty]) and np.array_equal(r[~empty, 1], hi[~empty])
    assert np.all(r[empty] == 0)


def _coincident_records(sigmas, colors, px=8.0, py=8.0):
    """Records placed exactly at pixel (px, py): q = 0 there, so alpha = min(0.99, sigma)."""
    n = len(sigmas)
    rec = np.zeros((n, oracle.R_NF), np.float32)
    for i, (s, c) in enumerate(zip(sigmas, colors)):
        rec[i, :] = [px, py, 1.0 + i, 1.0, 0.0, 1.0, s, oracle.threshold(np.float32(s)), c[0], c[1], c[2], 1.0]
    return rec


def _single_tile_inputs(n):
    values = np.arange(n, dtype=np.uint32)
    ranges = np.zeros((1, 2), np.uint32)
    ranges[0] = [0, n]
    return values, ranges


@pytest.mark.parametrize("case", RS["render"], ids=lambda c: c["cite"][:20])
def test_render_printed_examples(case):
    rec = _coincident_records(case["sigmas"], case["colors"])
    values, ranges = _single_tile_inputs(len(rec))
    img, T, nc = oracle.render(rec, values, ranges, 16, 16, bg=case.get("bg", (0.0, 0.0, 0.0)))
    assert np.allclose(img[:, 8, 8], case["C"], atol=2e-7)
    assert abs(T[8, 8] - case["T"]) < 1e-7
    if "ncontrib" in case:
        assert nc[8, 8] == case["ncontrib"]


def test_render_binned_equals_unbinned_and_3sigma_loss():
    """R17 / P:44 'identical renders': AccuTile- and SnugBox-binned renders equal the
    unbinned render bitwise; the 3-sigma render does too when every sigma <= sigma*, but
    not in general (a sigma = 0.99 Gaussian reaches 3.3 sigma, beyond Eq. 8's square)."""
    for name in ("tiny", "tiny-lowsigma", "tiny-deg0"):
        scene, cams = synth.make_workload(name)
        cam = cams[0]
        fa = oracle.frame(scene, cam, "accutile")
        ub = oracle.render_unbinned(fa.rec, cam.width, cam.height)
        assert np.array_equal(fa.image, ub), name
        fs = oracle.frame(scene, cam, "snugbox")
        assert np.array_equal(fs.image, ub)
        if name == "tiny-lowsigma":
            f3 = oracle.frame(scene, cam, "3sigma")
            assert np.array_equal(f3.image, ub)
    # hand-built 3-sigma counterexample: cov I, sigma 0.99 at (12.9, 8): the square
    # [9.9, 15.9] stays in tile 0 while pixel (16, 8) (tile 1, q = 9.61 <= t = 11.06) is lit
    _, cam = synth.tiny_scene(4, 0)
    rec = np.zeros((1, oracle.R_NF), np.float32)
    rec[0] = [12.9, 8.0, 1.0, 1.0, 0.0, 1.0, 0.99, oracle.threshold(np.float32(0.99)), 1, 1, 1, 1]
    ub = oracle.render_unbinned(rec, 32, 16)
    assert ub[0, 8, 16] > 0.004
    keys3 = np.array([0 << 32], np.uint64)      # 3-sigma: tile 0 only
    r3 = oracle.tile_ranges(keys3, 2)
    img3, _, _ = oracle.render(rec, np.zeros(1, np.uint32), r3, 32, 16)
    assert img3[0, 8, 16] == 0.0
    tl, _ = oracle.accutile(12.9, 8.0, 1.0, 0.0, 1.0, oracle.threshold(np.float32(0.99)), 2, 1)
    assert tl.tolist() == [0, 1]


@pytest.mark.parametrize("case", RS["score"], ids=lambda c: c["cite"][:20])
def test_score_printed_examples(case):
    rec = _coincident_records(case["sigmas"], case["colors"])
    values, ranges = _single_tile_inputs(len(rec))
    s = oracle.prune_score(rec, values, ranges, 16, 16, window=(8, 9, 8, 9))
    assert np.allclose(s, case["U"], rtol=1e-6, atol=1e-12)


def test_score_matches_finite_differences():
    """dC/dg_i = sigma_i dC/dalpha_i (Eq. 5) against central differences of
    the plain compositing of Eq. 7 (or_composite_alphas) for 20 coincident Gaussians with
    alpha in (0.05, 0.5) and a non-black background."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        K = 20
        sig = rng.uniform(0.05, 0.5, K).astype(np.float32)
        col = rng.uniform(0, 1, (K, 3)).astype(np.float32)
        bg = rng.uniform(0, 1, 3).astype(np.float32)
        rec = _coincident_records(sig, col)
        values, ranges = _single_tile_inputs(K)
        s = oracle.prune_score(rec, values, ranges, 16, 16, bg=bg, window=(8, 9, 8, 9))
        alpha = sig.astype(np.float64)
        h = 1e-6
        for i in range(K):
            ap, am = alpha.copy(), alpha.copy()
            ap[i] += h
            am[i] -= h
            d = (oracle.composite_alphas(ap, col, bg) - oracle.composite_alphas(am, col, bg)) / (2 * h)
            U = float(np.sum((alpha[i] * d) ** 2))    # sigma_i = alpha_i here (q = 0)
            assert abs(s[i] - U) <= 1e-6 * max(U, 1e-12), (trial, i, s[i], U)


def test_score_additive_over_views_and_nonnegative():
    """Score is a sum over poses (P:384 'sum over phi'): U(A+B) = U(A) + U(B); U >= 0."""
    scene, cams = synth.make_workload("mnr360-3m", n=600)
    cams = [synth.orbit_cameras(185, 160, 104)[k] for k in (0, 40)]
    sa = oracle.score_views(scene, cams[:1])
    sb = oracle.score_views(scene, cams[1:])
    sab = oracle.score_views(scene, cams)
    assert np.allclose(sab, sa + sb, rtol=1e-12, atol=0)
    assert np.all(sab >= 0) and sab.max() > 0


def test_prune_select_examples_and_invariants():
    """Prune step (P:381 'removing a set percentage with the lowest sensitivities'); printed
    examples S:389-392 and the argsort invariance of P:416 (log is monotone)."""
    keep, k = oracle.prune_select(np.arange(10, dtype=np.float64), 0.3)
    assert k == 3 and keep.sum() == 7 and keep[:3].sum() == 0
    keep, k = oracle.prune_select(np.ones(10), 0.5)          # ties: the last 5 by index go
    assert keep.tolist() == [1] * 5 + [0] * 5
    keep, k = oracle.prune_select(np.array([5.0, 1.0, 3.0, 0.0]), 0.5)
    assert keep.tolist() == [1, 0, 1, 0]
    rng = np.random.default_rng(7)
    s = rng.integers(0, 50, 10000).astype(np.float64) * rng.uniform(0.5, 2.0)  # many ties
    for ratio in (0.0, 0.1, 0.3, 0.8, 1.0):
        keep, k = oracle.prune_select(s, ratio)
        assert k == int(np.floor(ratio * len(s))) and keep.sum() == len(s) - k
        order = np.lexsort((-np.arange(len(s)), s))            # library: (score asc, index desc)
        want = np.ones(len(s), np.uint8)
        want[order[:k]] = 0
        assert np.array_equal(keep, want)
        keep2, _ = oracle.prune_select(s * 37.5, ratio)      # positive scaling: same set
        assert np.array_equal(keep, keep2)
