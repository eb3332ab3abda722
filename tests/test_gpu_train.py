"""GPU parity and behaviour of the NEXT-3 training pieces (ss_l1_loss_grad, ss_adam_step)
and of pruning-in-the-loop training on synthetic targets (paper_2412_00578_b200/train.py).

Parity against the oracle (oracle/ss_oracle_bwd.c, pinned by tests/test_oracle_train.py):
  * L1 gradient bit-exact (both sides round sign / count to float32 the same way), the loss
    sum within 1e-6 relative (float32 partial sums);
  * Adam: three steps on every scene array; raw parameters within 1e-6 |raw| + 1e-4 lr of the
    float64 oracle, m within 1e-5 relative of its scale, activated parameters within 1e-5
    relative (float32 state, one rounding per operation).
Behaviour: training decreases the L1 loss; pruning 50% by the efficient score Ũ keeps a
higher PSNR than pruning the same number at random (the paper's premise).
"""
import numpy as np
import pytest

import oracle
from paper_2412_00578_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_l1_parity():
    import ctypes as C
    from paper_2412_00578_b200._abi import check, lib
    rng = np.random.default_rng(0)
    img = rng.uniform(0, 1, (3, 37, 53)).astype(np.float32)      # count not a multiple of 4
    gt = rng.uniform(0, 1, (3, 37, 53)).astype(np.float32)
    gt[1, 5] = img[1, 5]
    L, g = oracle.l1_loss_grad(img, gt)
    ti, tg = torch.from_numpy(img).cuda(), torch.from_numpy(gt).cuda()
    out = torch.empty_like(ti)
    ls = torch.zeros(1, dtype=torch.float64, device="cuda")
    check(lib().ss_l1_loss_grad(ti.numel(), C.c_void_p(ti.data_ptr()), C.c_void_p(tg.data_ptr()),
                                C.c_void_p(out.data_ptr()), C.c_void_p(ls.data_ptr()), None), "l1")
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), g)
    assert abs(ls.item() / img.size - L) <= 1e-6 * L


def _oracle_layout(scene, cfg):
    """Per-element activation / learning rate of each scene array (the kernel's grouping)."""
    n, deg = scene.n, scene.sh_degree
    B = synth.SH_PLANES[deg]
    nb3 = (deg + 1) ** 2 * 3
    act_mo = np.tile([0, 0, 0, 2], (n, 1))
    lr_mo = np.tile([cfg.lr_mean * cfg.extent] * 3 + [cfg.lr_opacity], (n, 1))
    act_sc = np.ones((n, 4), np.int32)
    lr_sc = np.full((n, 4), cfg.lr_scale)
    coef = np.arange(4 * B).reshape(B, 4)
    lr_sh = np.where(coef < 3, cfg.lr_sh_dc, cfg.lr_sh_rest)[None].repeat(n, 0)
    used_sh = (coef < nb3)[None].repeat(n, 0)
    return act_mo, lr_mo, act_sc, lr_sc, lr_sh, used_sh


def test_adam_parity():
    from paper_2412_00578_b200.raster import DeviceScene
    from paper_2412_00578_b200.train import AdamConfig, Trainer
    import ctypes as C
    from paper_2412_00578_b200._abi import check, lib
    scene, cam = synth.grad_scene(n=40, width=72, height=40, seed=7)
    cfg = AdamConfig(extent=2.0)
    ds = DeviceScene.from_host(scene)
    tr = Trainer(ds, [cam], [torch.zeros((3, 40, 72), device="cuda")], adam=cfg)
    act_mo, lr_mo, act_sc, lr_sc, lr_sh, used_sh = _oracle_layout(scene, cfg)
    mo = scene.mean_opac.astype(np.float64)
    raw_mo = mo.copy()
    raw_mo[:, 3] = np.log(mo[:, 3] / (1 - mo[:, 3]))
    raw_sc = np.log(np.maximum(scene.scale.astype(np.float64), 1e-30))
    raw_rot = scene.rot.astype(np.float64).copy()
    raw_sh = np.transpose(scene.sh, (1, 0, 2)).astype(np.float64).copy()          # [n][B][4]
    state = {k: (np.zeros_like(a), np.zeros_like(a)) for k, a in
             (("mo", raw_mo), ("sc", raw_sc), ("rot", raw_rot), ("sh", raw_sh))}
    rng = np.random.default_rng(3)
    for t in range(1, 4):
        g_mo = rng.normal(0, 1, raw_mo.shape).astype(np.float32)
        g_sc = rng.normal(0, 1, raw_sc.shape).astype(np.float32)
        g_sc[:, 3] = 0
        g_rot = rng.normal(0, 1, raw_rot.shape).astype(np.float32)
        g_sh = (rng.normal(0, 1, raw_sh.shape) * used_sh).astype(np.float32)
        grads = DeviceScene(*(torch.from_numpy(a).cuda() for a in (g_mo, g_sc, g_rot, g_sh)), scene.sh_degree)
        out = DeviceScene(ds.mean_opac, ds.scale, ds.rot, ds.sh, ds.sh_degree)
        check(lib().ss_adam_step(C.byref(grads.struct()), C.byref(tr.raw.struct()), C.byref(tr.m.struct()),
                                 C.byref(tr.v.struct()), C.byref(out.struct()), C.byref(cfg.struct(t)), None), "adam")
        a_mo = oracle.adam_step(g_mo, raw_mo, *state["mo"], act_mo, lr_mo, eps=cfg.eps, t=t)
        sc_used = raw_sc[:, :3].copy()
        m_sc, v_sc = (np.ascontiguousarray(x[:, :3]) for x in state["sc"])
        a_sc = oracle.adam_step(g_sc[:, :3], sc_used, m_sc, v_sc, 1, cfg.lr_scale, eps=cfg.eps, t=t)
        raw_sc[:, :3] = sc_used
        state["sc"][0][:, :3], state["sc"][1][:, :3] = m_sc, v_sc
        a_rot = oracle.adam_step(g_rot, raw_rot, *state["rot"], 0, cfg.lr_rot, eps=cfg.eps, t=t)
        a_sh = oracle.adam_step(g_sh, raw_sh, *state["sh"], 0, lr_sh, eps=cfg.eps, t=t)
    torch.cuda.synchronize()

    def close(name, gpu, ref, lr):
        gpu = gpu.astype(np.float64)
        d = np.abs(gpu - ref)
        ok = d <= 1e-6 * np.abs(ref) + 1e-4 * lr
        assert ok.all(), f"{name}: worst {(d / (1e-6 * np.abs(ref) + 1e-4 * lr)).max()}"

    close("raw mean_opac", tr.raw.mean_opac.cpu().numpy(), raw_mo, lr_mo)
    close("raw scale", tr.raw.scale.cpu().numpy()[:, :3], raw_sc[:, :3], cfg.lr_scale)
    close("raw rot", tr.raw.rot.cpu().numpy(), raw_rot, cfg.lr_rot)
    sh_gpu = tr.raw.sh.cpu().numpy()
    close("raw sh", sh_gpu[used_sh], raw_sh[used_sh], lr_sh[used_sh])
    assert np.array_equal(sh_gpu[~used_sh], raw_sh[~used_sh].astype(np.float32))   # padding untouched
    for name, gpu, ref in (("mean_opac", ds.mean_opac, a_mo), ("scale", ds.scale[:, :3], a_sc), ("rot", ds.rot, a_rot)):
        g = gpu.cpu().numpy().astype(np.float64)
        assert np.allclose(g, ref, rtol=1e-5, atol=1e-7), name
    m_gpu = tr.m.mean_opac.cpu().numpy()
    assert np.allclose(m_gpu, state["mo"][0], rtol=1e-5, atol=1e-6)


def _small_orbit(n=20000, seed=5, views=8, W=192, H=128):
    scene = synth.orbit_scene(n, seed)
    cams = synth.orbit_cameras(views, W, H)
    return scene, cams


def _mean_l1(tr):
    tot = 0.0
    for v in range(len(tr.cams)):
        img = tr.render_view(v)
        tot += float((img - tr.targets[v]).abs().mean())
    return tot / len(tr.cams)


def test_training_reduces_l1():
    from paper_2412_00578_b200.raster import DeviceScene
    from paper_2412_00578_b200.train import AdamConfig, Trainer, render_targets
    gt, cams = _small_orbit()
    targets = render_targets(DeviceScene.from_host(gt), cams)
    init = synth.perturb(gt, seed=1)
    tr = Trainer(DeviceScene.from_host(init), cams, targets, adam=AdamConfig(extent=4.0), seed=0)
    l0 = _mean_l1(tr)
    tr.fit(300)
    l1 = _mean_l1(tr)
    assert l1 < 0.8 * l0, (l0, l1)
    assert np.isfinite(tr.scene.mean_opac.cpu().numpy()).all()


@pytest.mark.parametrize("seed", [5, 6, 7])
def test_score_pruning_beats_random(seed):
    """Prune 50% of a scene by U~ vs 50% uniformly at random: the score keeps more PSNR."""
    from paper_2412_00578_b200.raster import DeviceScene
    from paper_2412_00578_b200.train import Trainer, render_targets
    gt, cams = _small_orbit(seed=seed)
    targets = render_targets(DeviceScene.from_host(gt), cams)
    a = Trainer(DeviceScene.from_host(gt), cams, targets)
    a.prune(0.5)
    p_score = a.psnr()
    b = Trainer(DeviceScene.from_host(gt), cams, targets)
    rng = np.random.default_rng(seed)
    keep = np.ones(gt.n, np.uint8)
    keep[rng.choice(gt.n, gt.n // 2, replace=False)] = 0
    b.prune_mask(torch.from_numpy(keep).cuda(), int(keep.sum()))
    p_rand = b.psnr()
    assert a.n == b.n
    assert p_score > p_rand + 1.0, (p_score, p_rand)


def test_schedule_prunes_inside_training():
    """The scaled paper schedule (one soft event at 80%, hard 30% events) inside fit()."""
    from paper_2412_00578_b200.raster import DeviceScene
    from paper_2412_00578_b200.train import Trainer, render_targets, scaled_schedule
    gt, cams = _small_orbit(n=8000, views=6, W=128, H=96)
    targets = render_targets(DeviceScene.from_host(gt), cams)
    sched = scaled_schedule(200, soft_ratio=0.8, hard_ratio=0.3)
    assert list(sched.values())[0] == 0.8 and len(sched) == 6
    tr = Trainer(DeviceScene.from_host(synth.perturb(gt, seed=2)), cams, targets)
    hist = tr.fit(200, sched)
    n = gt.n
    for it, ratio, k, n_after in hist["events"]:
        assert k == int(np.floor(ratio * n)) and n_after == n - k
        n = n_after
    assert tr.n == n and len(hist["events"]) == len(sched)


def test_prune_keeps_optimizer_state_aligned():
    """After a prune event the Adam state rows belong to the surviving Gaussians: raw = the
    inverse activation of the (compacted) scene, and m / v are the compacted pre-prune rows."""
    from paper_2412_00578_b200.raster import DeviceScene
    from paper_2412_00578_b200.train import Trainer, render_targets
    gt, cams = _small_orbit(n=6000, views=4, W=128, H=96)
    targets = render_targets(DeviceScene.from_host(gt), cams)
    tr = Trainer(DeviceScene.from_host(synth.perturb(gt, seed=3)), cams, targets)
    tr.fit(20)
    m_before = tr.m.mean_opac.cpu().numpy().copy()
    score = tr.score()
    from paper_2412_00578_b200.raster import prune_select
    keep, k = prune_select(score, 0.5)
    tr.prune_mask(keep, tr.n - k)
    kept = np.nonzero(keep.cpu().numpy())[0]
    assert tr.n == len(kept)
    assert np.array_equal(tr.m.mean_opac.cpu().numpy(), m_before[kept])
    mo, raw = tr.scene.mean_opac.cpu().numpy(), tr.raw.mean_opac.cpu().numpy()
    assert np.array_equal(mo[:, :3], raw[:, :3])
    assert np.allclose(mo[:, 3], 1.0 / (1.0 + np.exp(-raw[:, 3].astype(np.float64))), rtol=1e-6)
    sc, rs = tr.scene.scale.cpu().numpy()[:, :3], tr.raw.scale.cpu().numpy()[:, :3]
    assert np.allclose(sc, np.exp(rs.astype(np.float64)), rtol=1e-6)
    tr.fit(5)   # training continues on the pruned scene
    assert np.isfinite(tr.scene.mean_opac.cpu().numpy()).all()


def test_assign_backward_and_flagged_adam_equal_the_dense_path():
    """ss_preprocess_backward_assign writes exactly what ss_preprocess_backward accumulates into
    zeroed arrays, flags exactly the Gaussians with a non-zero grad2d row and leaves the others'
    entries untouched; ss_adam_step_flagged then equals ss_adam_step on the zero-filled gradients."""
    import ctypes as C
    from paper_2412_00578_b200._abi import check, lib
    from paper_2412_00578_b200.raster import DeviceScene, Rasterizer, camera_struct
    from paper_2412_00578_b200.train import AdamConfig
    scene, cams = _small_orbit(n=8000, views=2, W=128, H=96)
    ds = DeviceScene.from_host(scene)
    rz = Rasterizer(ds, 128, 96)
    rz.ensure_capacity(cams[0])
    img, T, nc = rz.render_frame(cams[0], want_T=True, want_ncontrib=True)
    dimg = torch.empty_like(img).uniform_(-1, 1)
    g2d = rz.render_backward(dimg, T, nc)
    dense = rz.preprocess_backward(cams[0], g2d)                      # += into zeros
    stale = ds.zeros_like()
    for t in (stale.mean_opac, stale.scale, stale.rot, stale.sh):
        t.fill_(123.0)
    flags = torch.zeros(scene.n, dtype=torch.uint8, device="cuda")
    check(lib().ss_preprocess_backward_assign(C.byref(ds.struct()), C.byref(camera_struct(cams[0])),
                                              C.c_void_p(g2d.data_ptr()), C.byref(stale.struct()),
                                              C.c_void_p(flags.data_ptr()), None), "assign")
    torch.cuda.synchronize()
    f = flags.cpu().numpy().astype(bool)
    assert np.array_equal(f, (g2d.cpu().numpy()[:, :9] != 0).any(1))
    assert f.sum() > 100
    for a, b in ((stale.mean_opac, dense.mean_opac), (stale.scale, dense.scale), (stale.rot, dense.rot),
                 (stale.sh, dense.sh)):
        an, bn = a.cpu().numpy(), b.cpu().numpy()
        # same chain rule; the two template instantiations may contract the SH-basis polynomials
        # into FMAs differently (a few float32 ulps)
        assert np.allclose(an[f], bn[f], rtol=1e-6, atol=1e-12)
        assert np.all(an[~f] == 123.0)
    # flagged Adam on gradients whose unflagged rows are stale == dense Adam on zero-filled rows
    fl = torch.from_numpy(f).cuda()
    for t_stale, t_dense in ((stale.mean_opac, dense.mean_opac), (stale.scale, dense.scale), (stale.rot, dense.rot),
                             (stale.sh, dense.sh)):
        t_stale[fl] = t_dense[fl]
    cfg = AdamConfig(extent=4.0).struct(1)
    outs = []
    for flagged in (False, True):
        sc = DeviceScene(ds.mean_opac.clone(), ds.scale.clone(), ds.rot.clone(), ds.sh.clone(), ds.sh_degree)
        raw, m, v = sc.zeros_like(), sc.zeros_like(), sc.zeros_like()
        check(lib().ss_adam_init(C.byref(sc.struct()), C.byref(raw.struct()), C.byref(m.struct()), C.byref(v.struct()),
                                 None), "init")
        if flagged:
            check(lib().ss_adam_step_flagged(C.byref(stale.struct()), C.byref(raw.struct()), C.byref(m.struct()),
                                             C.byref(v.struct()), C.byref(sc.struct()), C.byref(cfg),
                                             C.c_void_p(flags.data_ptr()), None), "flagged")
        else:
            check(lib().ss_adam_step(C.byref(dense.struct()), C.byref(raw.struct()), C.byref(m.struct()),
                                     C.byref(v.struct()), C.byref(sc.struct()), C.byref(cfg), None), "dense")
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in (sc.mean_opac, sc.scale, sc.rot, sc.sh, m.sh, v.mean_opac)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
