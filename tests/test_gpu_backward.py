"""GPU parity of the backward: ss_render_backward and
ss_preprocess_backward through the C-ABI binding versus the float64 oracle
(oracle/ss_oracle_bwd.c, pinned by tests/test_oracle_backward.py).

Tolerances (DESIGN.md §5 "backward"):
  * render backward: every entry of grad2d within 1e-4 of the sum of the absolute values of
    its per-pixel terms (gabs, computed by the oracle) -- float32 terms carry ~K eps relative
    error (T recovered by K divisions) and float32 atomics add ~n eps of the absolute sum;
    plus 1e-7 absolute;
  * preprocess backward (same float32 grad2d fed to both sides): within 2e-3 relative of the
    largest entry of the same parameter group of that Gaussian (float32 chain through the
    conic inverse and Sigma_3D = M M^T; 1e-3 measured worst case is the conic's 1/det^2
    amplification for the thinnest ellipses).
"""
import numpy as np
import pytest

import oracle
from paper_2412_00578_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RENDER_TOL = 1e-4
PRE_TOL = 2e-3


def _setup(scene, cam, bg, seed=3, capacity=None):
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
    rz = Rasterizer(DeviceScene.from_host(scene), cam.width, cam.height, mode="accutile", capacity=capacity)
    rz.ensure_capacity(cam)
    img, T, nc = rz.render_frame(cam, bg, want_T=True, want_ncontrib=True)
    rng = np.random.default_rng(seed)
    dimg = rng.uniform(-1.0, 1.0, (3, cam.height, cam.width)).astype(np.float32)
    g2d = rz.render_backward(torch.from_numpy(dimg).cuda(), T, nc, bg=bg)
    torch.cuda.synchronize()
    return rz, dimg, g2d.cpu().numpy(), T, nc


def _check_render(g_gpu, g_or, gabs, vis):
    d = np.abs(g_gpu[:, :9].astype(np.float64) - g_or)
    lim = RENDER_TOL * gabs + 1e-7
    bad = d > lim
    assert not bad.any(), (f"{bad.sum()} grad2d entries outside tolerance; worst ratio "
                           f"{(d / lim).max():.3g} at {np.unravel_index(np.argmax(d / lim), d.shape)}")
    assert np.all(g_gpu[~vis] == 0.0)
    assert np.all(g_gpu[:, 9:] == 0.0)


def _check_pre(name, a_gpu, a_or):
    a_gpu = a_gpu.astype(np.float64)
    scale = np.abs(a_or).max(axis=-1, keepdims=True)
    d = np.abs(a_gpu - a_or)
    ok = d <= PRE_TOL * scale + 1e-9
    assert ok.all(), f"{name}: {(~ok).sum()} entries off; worst {(d / (scale + 1e-30)).max():.3g}"


@pytest.mark.parametrize("case", ["grad72x40", "tiny", "tiny-deg0"])
def test_render_and_preprocess_backward_parity(case):
    if case == "grad72x40":
        scene, cam = synth.grad_scene(n=40, width=72, height=40, seed=7, yaw_deg=20.0)
        bg = (0.1, 0.2, 0.3)
    else:
        scene, cams = synth.make_workload(case)
        cam = cams[0]
        bg = (0.0, 0.0, 0.0) if case == "tiny" else (0.3, 0.1, 0.2)
    rz, dimg, g_gpu, T, nc = _setup(scene, cam, bg)
    f = oracle.frame(scene, cam, "accutile", bg)
    vis = f.counts > 0
    # the forward the backward starts from: same blended sets
    assert np.array_equal(nc.cpu().numpy().astype(np.uint32), f.ncontrib)
    g_or, gabs = oracle.render_backward(f.rec, f.values, f.ranges, cam.width, cam.height, dimg, bg)
    _check_render(g_gpu, g_or, gabs, vis)
    # preprocess backward on the same float32 grad2d
    g32 = g_gpu[:, :9].astype(np.float64)
    dmo, ds, dr, dsh = oracle.project_backward(scene, cam, g32)
    grads = rz.preprocess_backward(cam, torch.from_numpy(g_gpu).cuda())
    torch.cuda.synchronize()
    _check_pre("mean xyz", grads.mean_opac.cpu().numpy()[:, :3], dmo[:, :3])
    _check_pre("opacity", grads.mean_opac.cpu().numpy()[:, 3:], dmo[:, 3:])
    _check_pre("scale", grads.scale.cpu().numpy()[:, :3], ds[:, :3])
    assert np.all(grads.scale.cpu().numpy()[:, 3] == 0.0)
    _check_pre("rot", grads.rot.cpu().numpy(), dr)
    sh_gpu = grads.host_sh_planes()                      # [B][N][4] like the oracle's
    nb3 = (scene.sh_degree + 1) ** 2 * 3
    flat_g = sh_gpu.transpose(1, 0, 2).reshape(scene.n, -1)[:, :nb3]
    flat_o = dsh.transpose(1, 0, 2).reshape(scene.n, -1)[:, :nb3]
    _check_pre("sh", flat_g, flat_o)


def test_backward_accumulates_and_is_idempotent():
    """grad2d and the parameter gradients accumulate (+=): two identical calls give exactly 2x
    one call's per-Gaussian sums up to float32 atomics order; zero dL/dC gives zero."""
    scene, cam = synth.grad_scene(n=40, width=72, height=40, seed=7)
    rz, dimg, g1, T, nc = _setup(scene, cam, (0.0, 0.0, 0.0))
    g = torch.from_numpy(g1).cuda()
    rz.render_backward(torch.from_numpy(dimg).cuda(), T, nc, grad2d=g)
    g2 = g.cpu().numpy()
    assert np.allclose(g2, 2 * g1, rtol=1e-5, atol=1e-7)
    z = rz.render_backward(torch.zeros((3, cam.height, cam.width), device="cuda"), T, nc)
    assert float(z.abs().max()) == 0.0
    gr = rz.preprocess_backward(cam, z)
    assert float(gr.mean_opac.abs().max()) == 0.0 and float(gr.sh.abs().max()) == 0.0


def test_backward_edge_cases():
    """n = 0, and every Gaussian culled: calls succeed and write nothing."""
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer
    scene, cam = synth.grad_scene(n=40, width=72, height=40, seed=7)
    empty = scene.subset(np.zeros(0, np.int64))
    rz = Rasterizer(DeviceScene.from_host(empty), cam.width, cam.height)
    img, T, nc = rz.render_frame(cam, want_T=True, want_ncontrib=True)
    g = rz.render_backward(torch.ones((3, cam.height, cam.width), device="cuda"), T, nc)
    assert g.numel() == 0
    rz.preprocess_backward(cam, g)
    behind = scene.subset(np.arange(scene.n))
    behind.mean_opac = behind.mean_opac.copy()
    behind.mean_opac[:, 2] = -5.0
    rz = Rasterizer(DeviceScene.from_host(behind), cam.width, cam.height)
    img, T, nc = rz.render_frame(cam, want_T=True, want_ncontrib=True)
    g = rz.render_backward(torch.ones((3, cam.height, cam.width), device="cuda"), T, nc)
    gr = rz.preprocess_backward(cam, g)
    torch.cuda.synchronize()
    assert float(g.abs().max()) == 0.0 and float(gr.mean_opac.abs().max()) == 0.0


@pytest.mark.parametrize("workload,view,bg", [("mnr360-3m", 0, (0.0, 0.0, 0.0)), ("garden", 40, (0.0, 0.0, 0.0)),
                                               ("playroom", 5, (0.1, 0.3, 0.6)), ("truck", 17, (0.0, 0.0, 0.0))])
def test_fullsize_backward_sampled(workload, view, bg):
    """BASELINE.json's full-size scenes (MNR360-3M = the bench workload, garden 5.8M, playroom
    2.3M with background, truck 2.5M), AccuTile, in the bench's launch configuration: grad2d of
    150 sampled Gaussians whose every tile is checked by the oracle (their oracle sums are
    complete), and their parameter gradients."""
    scene, cams = synth.make_workload(workload)
    cam = cams[view]
    rz, dimg, g_gpu, T, nc = _setup(scene, cam, bg, seed=4)
    P = rz.totals()["pairs"]
    f = oracle.frame(scene, cam, "accutile", bg, render=False, cap_hint=int(P * 1.05) + 16)
    rng = np.random.default_rng(0)
    small = (f.counts > 0) & (f.counts <= 4)
    # most Gaussians with tiles are never blended (behind saturated pixels): sample 100 among
    # those the GPU reports blended and 50 among all (the expected values are the oracle's)
    blended = np.nonzero(small & np.any(g_gpu[:, :9] != 0, axis=1))[0]
    pick = np.unique(np.concatenate([rng.choice(blended, min(100, len(blended)), replace=False),
                                     rng.choice(np.nonzero(small)[0], 50, replace=False)]))
    assert len(blended) >= 100
    tl = set()
    for gi in pick:
        tl.update(oracle.tiles_of_record("accutile", f.rec[gi], f.rect[gi], cam.tiles_x, cam.tiles_y).tolist())
    g_or, gabs = oracle.render_backward(f.rec, f.values, f.ranges, cam.width, cam.height, dimg, bg,
                                        tiles=np.array(sorted(tl), np.int32))
    d = np.abs(g_gpu[pick, :9].astype(np.float64) - g_or[pick])
    assert np.all(d <= RENDER_TOL * gabs[pick] + 1e-7), f"worst {(d / (RENDER_TOL * gabs[pick] + 1e-7)).max()}"
    grads = rz.preprocess_backward(cam, torch.from_numpy(g_gpu).cuda())
    torch.cuda.synchronize()
    sub = scene.subset(pick)
    dmo, ds, dr, dsh = oracle.project_backward(sub, cam, g_gpu[pick, :9].astype(np.float64))
    _check_pre("mean xyz", grads.mean_opac.cpu().numpy()[pick, :3], dmo[:, :3])
    _check_pre("scale", grads.scale.cpu().numpy()[pick, :3], ds[:, :3])
    _check_pre("rot", grads.rot.cpu().numpy()[pick], dr)
