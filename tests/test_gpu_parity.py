"""GPU parity: libss (through the C-ABI binding) versus the CPU oracle, element by element.

Bar (BASELINE.json north_star): bit-exact records, tile counts, depth order, sorted keys,
values and tile ranges; images within 1e-4 absolute per channel; pruning scores within
1e-4 relative (|dU| / max(U, 1e-6 max U)).  Knife-edge exemptions (R22) are
counted, and must be zero on the small configs.
"""
import numpy as np
import pytest

import oracle
from paper_2412_00578_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MODES = ("3sigma", "snugbox", "accutile")
IMG_TOL = 1e-4
SCORE_TOL = 1e-4


def _rz(scene, cam, mode, capacity=None):
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
    ds = DeviceScene.from_host(scene)
    return Rasterizer(ds, cam.width, cam.height, mode=mode, capacity=capacity)


def _gpu_frame(scene, cam, mode, bg=(0.0, 0.0, 0.0), capacity=None):
    rz = _rz(scene, cam, mode, capacity)
    img, T, nc = rz.render_frame(cam, bg, want_T=True, want_ncontrib=True)
    rz.finalize_colours()   # colours the render did not need (never gathered) are still pending
    torch.cuda.synchronize()
    tot = rz.totals()
    P = tot["pairs"]
    out = dict(
        rz=rz, img=img.cpu().numpy(), T=T.cpu().numpy(), nc=nc.cpu().numpy().astype(np.uint32),
        rec=rz.records().cpu().numpy(), counts=rz.counts().cpu().numpy().view(np.uint32),
        erec=rz.emit_records().cpu().numpy().view(np.uint32),
        depth_key=rz.depth_keys().cpu().numpy().view(np.uint32),
        order=rz.order().cpu().numpy().view(np.uint32)[:tot["n_visible"]],
        values=rz.sorted_values().cpu().numpy().view(np.uint32)[:P],
        keys=rz.sorted_keys().cpu().numpy().view(np.uint64)[:P],
        ranges=rz.ranges().cpu().numpy().view(np.uint32), P=P, n_visible=tot["n_visible"],
        overflow=tot["overflow"])
    return out


def _check_frame(scene, cam, mode, bg=(0.0, 0.0, 0.0), capacity=None, image=True):
    g = _gpu_frame(scene, cam, mode, bg, capacity)
    f = oracle.frame(scene, cam, mode, bg, render=image)
    assert g["overflow"] == 0
    cnt = g["counts"]
    assert np.array_equal(cnt, f.counts), "tile counts differ"
    vis = cnt > 0
    # records (bit-exact): GPU (x,y,a,b | c,t,sigma,hx | hy,r,g,b); oracle (x,y,depth,a,b,c,sigma,t,r,g,b,vis)
    gr, orr = g["rec"][vis], f.rec[vis]
    assert np.all(gr[:, 8] == 1.0), "colour flags"   # every colour computed (lazily or by finalize)
    pairs = [(0, 0), (1, 1), (2, 3), (3, 4), (4, 5), (5, 7), (6, 6), (9, 8), (10, 9), (11, 10)]
    for gi, oi in pairs:
        assert np.array_equal(gr[:, gi].view(np.uint32), orr[:, oi].view(np.uint32)), f"record field {gi}"
    assert np.array_equal(g["depth_key"][vis], orr[:, 2].view(np.uint32)), "depth keys"
    assert np.all(g["depth_key"][~vis] == 0xFFFFFFFF)
    er = g["erec"][vis]
    big = (er[:, 1] & 0x900) == 0  # records holding aux (neither spans nor entries inline)
    if mode == "accutile":  # aux = t as float64 bits: 2 log(255 sigma) of the stored sigma
        t64 = er[big, 2:4].copy().view(np.float64)[:, 0]
        t_or = np.array([oracle.threshold(s) for s in orr[big, 6]])
        assert np.all(np.abs(t64 - t_or) <= 4.5e-16 * np.abs(t_or))  # CUDA log vs glibc log (R2)
        # line spans stored by the count = the oracle's AccuTile set, Gaussian by Gaussian
        spn = np.nonzero((er[:, 1] & 0x800) != 0)[0][:300]
        for j in spn:
            gi = np.nonzero(vis)[0][j]
            cols = (er[j, 1] & 0x200) != 0
            tiles = set()
            for w in er[j, 2:2 + (er[j, 1] & 0xFF)]:
                lo, hi, line = w & 0x1FF, (w >> 9) & 0x1FF, w >> 18
                for u in range(lo, hi):
                    tiles.add(u * cam.tiles_x + line if cols else line * cam.tiles_x + u)
            want = oracle.tiles_of_record(mode, f.rec[gi], f.rect[gi], cam.tiles_x, cam.tiles_y)
            assert tiles == set(want.tolist()), f"spans of Gaussian {gi}"
    else:  # the packed tile rect
        pr = er[big, 2]
        x0, y0 = pr & 0xFF, (pr >> 16) & 0xFF
        rect = np.stack([x0, x0 + ((pr >> 8) & 0xFF) + 1, y0, y0 + (pr >> 24) + 1], 1)
        assert np.array_equal(rect.astype(np.int32), f.rect[vis][big])
    # depth order of the visible Gaussians: (depth bits, index) -- numpy's lexsort on the oracle records
    idx = np.nonzero(vis)[0]
    dbits = f.rec[idx, 2].view(np.uint32)
    want_order = idx[np.lexsort((idx, dbits))]
    assert g["n_visible"] == len(idx)
    assert np.array_equal(g["order"], want_order.astype(np.uint32))
    # pairs, keys, ranges (bit-exact)
    assert g["P"] == f.P
    assert np.array_equal(g["values"], f.values)
    assert np.array_equal(g["keys"], f.keys)
    assert np.array_equal(g["ranges"], f.ranges)
    if image:
        d = np.abs(g["img"] - f.image)
        assert d.max() <= IMG_TOL, f"image max |diff| {d.max()}"
        assert np.abs(g["T"] - f.T).max() <= IMG_TOL
        assert (g["nc"] != f.ncontrib).sum() == 0
    return g, f


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", ["tiny", "tiny-lowsigma", "tiny-deg0", "tiny-deg1", "tiny-deg2"])
def test_tiny_parity(name, mode):
    scene, cams = synth.make_workload(name)
    _check_frame(scene, cams[0], mode)


@pytest.mark.parametrize("mode", MODES)
def test_medium_multiblock_parity(mode):
    """Spans many sort tiles (>4096 keys), two tile-sort passes (1200 tiles), a ragged
    image edge (W, H not multiples of 16) and SH degree 3."""
    scene, _ = synth.make_workload("mnr360-3m", n=40000)
    cam = synth.orbit_cameras(185, 630, 470)[11]
    _check_frame(scene, cam, mode, bg=(0.1, 0.2, 0.3))


@pytest.mark.parametrize("mode", ["3sigma", "accutile"])
def test_dense_ties_and_long_tiles(mode):
    """Sort stress: central tiles hold more than 4096 pairs each and half the Gaussians share
    one depth, so equal (tile, depth) keys are frequent; they must come out in index order,
    bit-exactly like the oracle's stable sort."""
    scene, cam = synth.dense_scene()
    g, f = _check_frame(scene, cam, mode)
    lens = f.ranges[:, 1] - f.ranges[:, 0]
    assert lens.max() > 4096
    assert (np.diff(g["keys"]) == 0).sum() > 1000


def test_binned_renders_equal_on_gpu():
    """R17 on the device: AccuTile and SnugBox renders are bitwise identical; the 3-sigma
    render equals them when every sigma <= sigma* (tiny-lowsigma)."""
    for name in ("tiny", "tiny-lowsigma"):
        scene, cams = synth.make_workload(name)
        imgs = {m: _gpu_frame(scene, cams[0], m)["img"] for m in MODES}
        assert np.array_equal(imgs["accutile"], imgs["snugbox"])
        if name == "tiny-lowsigma":
            assert np.array_equal(imgs["accutile"], imgs["3sigma"])


def test_prune_score_parity():
    for name, n, W, H in [("tiny", None, None, None), ("mnr360-3m", 20000, 320, 208)]:
        if n is None:
            scene, cams = synth.make_workload(name)
            cam = cams[0]
        else:
            scene, _ = synth.make_workload(name, n=n)
            cam = synth.orbit_cameras(185, W, H)[3]
        bg = (0.2, 0.5, 0.7)
        g = _gpu_frame(scene, cam, "accutile", bg)
        score = torch.zeros(scene.n, dtype=torch.float64, device="cuda")
        g["rz"].prune_score(score, bg)
        s_gpu = score.cpu().numpy()
        f = oracle.frame(scene, cam, "accutile", bg, render=False)
        s_or = oracle.prune_score(f.rec, f.values, f.ranges, cam.width, cam.height, bg)
        denom = np.maximum(s_or, 1e-6 * s_or.max())
        rel = np.abs(s_gpu - s_or) / denom
        assert rel.max() <= SCORE_TOL, f"{name}: max rel {rel.max()}"
        assert (s_or > 0).sum() > 100


def test_edge_cases():
    """Empty scene, everything culled, one Gaussian, capacity overflow + regrow."""
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
    scene, cams = synth.make_workload("tiny")
    cam = cams[0]
    # n = 0
    empty = scene.subset(np.zeros(0, np.int64))
    rz = Rasterizer(DeviceScene.from_host(empty), cam.width, cam.height, capacity=16)
    img = rz.render_frame(cam, (0.25, 0.5, 0.75))
    assert torch.allclose(img[:, 0, 0].cpu(), torch.tensor([0.25, 0.5, 0.75]))
    # all behind the camera
    behind = scene.subset(np.arange(100))
    behind.mean_opac[:, 2] = -5.0
    g = _gpu_frame(behind, cam, "accutile", capacity=16)
    assert g["P"] == 0 and g["n_visible"] == 0 and np.all(g["img"] == 0)
    # one Gaussian
    _check_frame(scene.subset(np.array([123])), cam, "accutile")
    # overflow: tiny capacity, then render_frame regrows and re-runs
    _check_frame(scene, cam, "accutile", capacity=8)


@pytest.mark.parametrize("name", ["tiny", "tiny-lowsigma"])
def test_phantom_pairs_invariant(name):
    """ss_render_stats' phantom pairs (a Gaussian's tile with alpha < 1/255 at every pixel
    centre): the pairs that DO hit a pixel centre are the same set in every mode whose tile sets
    contain every pixel-hit tile -- SnugBox and AccuTile (R23: pixel-hit <= AccuTile <=
    SnugBox) -- so P - phantom is equal for both, and AccuTile has no more phantoms."""
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
    scene, cams = synth.make_workload(name)
    cam = cams[0]
    ds = DeviceScene.from_host(scene)
    res = {}
    for mode in ("snugbox", "accutile"):
        rz = Rasterizer(ds, cam.width, cam.height, mode=mode)
        rz.render_frame(cam)
        st = rz.render_stats()
        res[mode] = (rz.totals()["pairs"], st["phantom_pairs"])
    (ps, fs), (pa, fa) = res["snugbox"], res["accutile"]
    assert 0 <= fa <= fs and fa < pa
    assert ps - fs == pa - fa, res


@pytest.mark.parametrize("mode", ["snugbox", "accutile"])
@pytest.mark.parametrize("seed", [11, 12, 13, "tangent-21", "tangent-22"])
def test_knife_edge_tile_decisions(mode, seed):
    """synth.knife_scene: means on / within 1e-5 px of tile lines, axis ratios up to 1e3,
    t ~ 0 and near-1 opacities, clipped giants.  Every count, sorted key and range equals the
    oracle's float64 tile sets bit-exactly; the float32-certified path must have handed some
    Gaussians to the float64 fallback here (pre_deferred > 0), so both paths are exercised."""
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
    if isinstance(seed, str):  # swept-axis extremes on tile lines (near-tangent Algorithm-1 lines)
        scene, cam = synth.tangent_scene(seed=int(seed.split("-")[1]))
    else:
        scene, cam = synth.knife_scene(seed=seed)
    rz = Rasterizer(DeviceScene.from_host(scene), cam.width, cam.height, mode=mode)
    rz.ensure_capacity(cam)
    rz.render_frame(cam)
    torch.cuda.synchronize()
    t = rz.totals()
    f = oracle.frame(scene, cam, mode, render=False, cap_hint=t["pairs"] + 16)
    assert np.array_equal(rz.counts().cpu().numpy().view(np.uint32), f.counts)
    assert t["pairs"] == f.P
    assert np.array_equal(rz.sorted_keys().cpu().numpy().view(np.uint64)[:f.P], f.keys)
    assert np.array_equal(rz.ranges().cpu().numpy().view(np.uint32), f.ranges)
    assert t["deferred"] > 0, "the float64 fallback was not exercised"


def test_maximum_image_size():
    """At the limits include/ss.h states: a 4096 x 4096 view is 256 x 256 = 65,536 tiles (the
    tile maximum, 256 per axis) and 64 x 64 = 4,096 super-tiles (the level-1 maximum).  150k
    Gaussians of the MNR360 recipe: records, counts, sorted keys, ranges bit-exact and the whole
    image within 1e-4 of the oracle (the full _check_frame battery)."""
    scene, _ = synth.make_workload("mnr360-3m", n=150000)
    cam = synth.orbit_cameras(1, 4096, 4096)[0]
    assert cam.tiles_x * cam.tiles_y == 65536
    _check_frame(scene, cam, "accutile", bg=(0.1, 0.2, 0.3))


@pytest.mark.parametrize("name", ["tiny", "tiny-lowsigma", "orbit", "dense"])
def test_plain_and_ncontrib_forward_equal(name):
    """The plain forward (the bench's frame path) and the n_contrib forward (the score's first
    walk) are separate instantiations of k_render; their images and T must be bitwise equal.  (It
    also guarded the batch-level culling experiment of NEXT-4: culled vs not.)"""
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
    if name == "orbit":
        scene, cams = synth.orbit_scene(30000, 5), synth.orbit_cameras(3, 200, 136)
    elif name == "dense":
        scene, cam = synth.dense_scene()
        cams = [cam]
    else:
        scene, cams = synth.make_workload(name)
    ds = DeviceScene.from_host(scene)
    for cam in cams:
        rz = Rasterizer(ds, cam.width, cam.height)
        rz.ensure_capacity(cam)
        bg = (0.1, 0.3, 0.2)
        img_c, T_c, _ = rz.render_frame(cam, bg, want_T=True)
        img_c, T_c = img_c.clone(), T_c.clone()
        img_n, T_n, _ = rz.render_frame(cam, bg, want_T=True, want_ncontrib=True)
        torch.cuda.synchronize()
        assert torch.equal(img_c, img_n) and torch.equal(T_c, T_n)


@pytest.mark.parametrize("variant", ["no-clip", "anisotropic-offcentre", "far-near-plane"])
@pytest.mark.parametrize("mode", ["3sigma", "accutile"])
def test_camera_variants(variant, mode):
    """Camera parameters the synthetic workloads keep fixed: the J clamp disabled (clip = 0,
    R5), fx != fy with the principal point off the image centre (R3), and a near plane at 1.0
    instead of 0.2 (R4).  The full record / count / key / range / image battery vs the oracle on
    a 20k-Gaussian orbit scene at 200 x 136 (ragged tiles)."""
    import dataclasses
    scene = synth.orbit_scene(20000, 7)
    cam = synth.orbit_cameras(2, 200, 136)[1]
    if variant == "no-clip":
        cam = dataclasses.replace(cam, clip=0.0)
    elif variant == "anisotropic-offcentre":
        cam = dataclasses.replace(cam, fy=float(np.float32(cam.fx * 1.37)), cx=81.25, cy=77.5)
    else:
        cam = dataclasses.replace(cam, z_near=1.0)
    _check_frame(scene, cam, mode, bg=(0.05, 0.1, 0.15))
