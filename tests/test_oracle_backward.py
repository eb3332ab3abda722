"""Pins of the oracle's render backward and preprocess backward (SURVEY §8(f) NEXT-2
"the per-pixel gradients from the render kernel are ... aggregated to the 2D mu_2D and
Sigma_2D parameters, which are then parallelized across Gaussians to compute gradients for
mu and s"; DESIGN.md §3 reading R27).

The backward is pinned against things other than itself:
  * central finite differences of the float64 forward (or_loss_f64 / or_project_f64),
  * the float64 forward pinned to the float32 forward of ss_oracle.c (itself pinned by
    test_oracle_pipeline.py / test_oracle_geometry.py),
  * closed forms for one Gaussian over one pixel (C = c alpha + bg (1 - alpha)).
"""
import numpy as np
import pytest

import oracle
from paper_2412_00578_b200 import synth

REC_TO_64 = [0, 1, 2, 3, 4, 5, 6, 8, 9, 10, 11]   # f32 record fields -> rec64 fields
G_TO_64 = [0, 1, 3, 4, 5, 6, 7, 8, 9]             # g2d column -> rec64 field


def rec64_of(rec):
    return np.ascontiguousarray(rec[:, REC_TO_64].astype(np.float64))


def central_difference(fn, set_x, x0, h0):
    """Central difference of fn (returning (value, blend-set hash)) at x0, with a step that
    leaves the blended (pixel, Gaussian) set unchanged (the loss jumps where a pixel crosses
    alpha = 1/255, R27); None when no step down to h0/16^3 does."""
    set_x(x0)
    _, h_mid = fn()
    h = h0
    for _ in range(4):
        set_x(x0 + h)
        fp, hp = fn()
        set_x(x0 - h)
        fm, hm = fn()
        set_x(x0)
        if hp == h_mid == hm:
            return (fp - fm) / (2 * h)
        h /= 16
    return None


def weights(cam, seed=3):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, (3, cam.height, cam.width)).astype(np.float32)


@pytest.fixture(scope="module")
def grad_case():
    sc, cam = synth.grad_scene(n=40, width=72, height=40, seed=7, yaw_deg=20.0)
    f = oracle.frame(sc, cam, "accutile", (0.1, 0.2, 0.3))
    return sc, cam, f


def test_project_f64_equals_float32_forward(grad_case):
    """or_project_f64 = or_project (pinned float32 contract) to float32 rounding."""
    sc, cam, f = grad_case
    r64 = oracle.project_f64(sc, cam)
    vis = f.rec[:, 11] > 0
    assert np.array_equal(vis, r64[:, 10] > 0)
    a, b = r64[vis][:, :10], rec64_of(f.rec)[vis][:, :10]
    assert np.all(np.abs(a - b) <= 1e-5 * np.maximum(np.abs(a), 1.0))


def test_loss_f64_equals_float32_render(grad_case):
    """Sum w * C of the float64 unbinned render = the same weighted sum of the float32 binned
    render of ss_oracle.c (equal up to float32 rounding, R17)."""
    sc, cam, f = grad_case
    w = weights(cam)
    L64 = oracle.loss_f64(oracle.project_f64(sc, cam), cam.width, cam.height, w.astype(np.float64), f.bg)
    L32 = float((w.astype(np.float64) * f.image.astype(np.float64)).sum())
    assert abs(L64 - L32) <= 1e-5 * np.abs(w).sum()


def test_single_gaussian_closed_form():
    """One Gaussian, one pixel, no clamp: C = c alpha + bg (1 - alpha), alpha = sigma G(q):
    dC/dc = alpha, dC/dsigma = G (c - bg), dC/dq = -alpha/2 (c - bg), dq/da = dx^2,
    dq/db = 2 dx dy, dq/dc = dy^2, dq/dx2d = -2 (a dx + b dy)."""
    a, b, c, sig, x2d, y2d = 0.05, 0.01, 0.08, 0.6, 3.3, 2.6
    q = a * 3.3 ** 2 + 2 * b * 3.3 * 2.6 + c * 2.6 ** 2   # pixel (0, 0): dx = -3.3, dy = -2.6
    t = 2 * np.log(255 * sig)
    rec = np.zeros((1, 12), np.float32)
    rec[0] = [x2d, y2d, 1.0, a, b, c, sig, t, 0.7, 0.2, 0.4, 1.0]
    values = np.zeros(1, np.uint32)
    ranges = np.array([[0, 1]], np.uint32)
    bg = np.array([0.1, 0.5, 0.3], np.float32)
    dimg = np.zeros((3, 1, 1), np.float32)
    r32 = rec[0].astype(np.float64)
    dx, dy = -r32[0], -r32[1]
    G = np.exp(-0.5 * (r32[3] * dx * dx + 2 * r32[4] * dx * dy + r32[5] * dy * dy))
    alpha = r32[6] * G
    assert alpha < 0.99 and q <= t
    for ch in range(3):
        dimg[:] = 0
        dimg[ch] = 1.0
        g, _ = oracle.render_backward(rec, values, ranges, 1, 1, dimg, bg)
        col = r32[8 + ch]
        dCdq = -0.5 * alpha * (col - bg[ch])
        want = np.zeros(9)
        want[6 + ch] = alpha
        want[5] = G * (col - bg[ch])
        want[0] = dCdq * (-2 * (r32[3] * dx + r32[4] * dy))
        want[1] = dCdq * (-2 * (r32[4] * dx + r32[5] * dy))
        want[2], want[3], want[4] = dCdq * dx * dx, dCdq * 2 * dx * dy, dCdq * dy * dy
        assert np.allclose(g[0], want, rtol=1e-12, atol=1e-15)


def test_clamped_alpha_passes_no_gradient():
    """R27: alpha = min(0.99, sigma G) at the clamp has zero derivative w.r.t. sigma and the
    2-D geometry; the colour derivative alpha T remains."""
    rec = np.zeros((1, 12), np.float32)
    rec[0] = [0.0, 0.0, 1.0, 0.05, 0.0, 0.05, 0.999, 2 * np.log(255 * 0.999), 0.7, 0.2, 0.4, 1.0]
    dimg = np.ones((3, 1, 1), np.float32)
    g, _ = oracle.render_backward(rec, np.zeros(1, np.uint32), np.array([[0, 1]], np.uint32), 1, 1, dimg)
    assert np.all(g[0, :6] == 0.0)
    assert np.allclose(g[0, 6:], 0.99)


def test_render_backward_finite_differences(grad_case):
    """dL/d(x2d, y2d, a, b, c, sigma, r, g, b) of every Gaussian = central differences of the
    float64 unbinned loss over the records (AccuTile-binned backward, ragged 72x40 image,
    background)."""
    sc, cam, f = grad_case
    w = weights(cam)
    g, gabs = oracle.render_backward(f.rec, f.values, f.ranges, cam.width, cam.height, w, f.bg)
    r64 = rec64_of(f.rec)
    w64 = w.astype(np.float64)
    checked = skipped = 0
    r = r64.copy()
    fn = lambda: oracle.loss_f64(r, cam.width, cam.height, w64, f.bg, with_hash=True)  # noqa: E731
    for i in np.nonzero(f.rec[:, 11] > 0)[0]:
        for col, field in enumerate(G_TO_64):
            def set_x(v, i=i, field=field):
                r[i, field] = v
            fd = central_difference(fn, set_x, r64[i, field], 1e-6 * max(1.0, abs(r64[i, field])))
            if fd is None:
                skipped += 1
                continue
            assert abs(fd - g[i, col]) <= 1e-5 * max(gabs[i].max(), 1e-3), (i, col, fd, g[i, col])
            checked += 1
    assert checked >= 300 and skipped <= checked // 50
    assert np.all(np.abs(g) <= gabs + 1e-12)


def _param_views(scene64):
    """(array, column list) of every differentiable parameter of a float64 scene."""
    nb = (scene64.sh_degree + 1) ** 2 * 3
    out = [("mean_opac", list(range(4))), ("scale", [0, 1, 2]), ("rot", [0, 1, 2, 3])]
    return out, nb


def _scene64(sc):
    return synth.Scene(sc.mean_opac.astype(np.float64), sc.scale.astype(np.float64), sc.rot.astype(np.float64),
                       sc.sh.astype(np.float64), sc.sh_degree, sc.name)


@pytest.mark.parametrize("deg,yaw,margin", [(3, 20.0, 8.0), (1, 0.0, 60.0), (0, -35.0, 8.0)])
def test_project_backward_finite_differences(deg, yaw, margin):
    """dL/d(mu, sigma, s, q, h) for L = sum_i u_i . rec64_i(params) with random cotangents u
    (x2d, y2d, a, b, c, sigma, r, g, b) = central differences of or_project_f64.  The wide
    margin puts Gaussians beyond the J clamp (R5: |x/z| > 1.3 W/2 / fx); degree 0 with
    strongly negative DC makes some colours clamp at 0."""
    sc, cam = synth.grad_scene(n=24, width=72, height=40, seed=11 + deg, yaw_deg=yaw, margin=margin,
                               sh_degree=deg)
    if deg == 0:
        sc.sh[0, :6, :3] = -3.0   # clamped colours: c = max(0, .) = 0
    s64 = _scene64(sc)
    rng = np.random.default_rng(5)
    u = rng.normal(0, 1, (sc.n, 9))
    r0 = oracle.project_f64(s64, cam)
    vis = r0[:, 10] > 0
    u[~vis] = 0.0
    dmo, ds, dr, dsh = oracle.project_backward(s64, cam, u)

    def F(s):
        r = oracle.project_f64(s, cam)
        return float((u * r[:, G_TO_64]).sum())

    if margin > 30:
        tx = np.abs((r0[vis, 0] - cam.cx) / cam.fx)
        assert np.any(tx > 1.3 * (cam.width / 2) / cam.fx), "no clamped J in the case"
    grads = {"mean_opac": dmo, "scale": ds, "rot": dr}
    for i in np.nonzero(vis)[0]:
        for name, cols in [("mean_opac", range(4)), ("scale", range(3)), ("rot", range(4))]:
            for k in cols:
                arr = getattr(s64, name)
                x0 = arr[i, k]
                h = 1e-6 * max(1.0, abs(x0))
                arr[i, k] = x0 + h
                fp = F(s64)
                arr[i, k] = x0 - h
                fm = F(s64)
                arr[i, k] = x0
                fd = (fp - fm) / (2 * h)
                g = grads[name][i, k]
                assert abs(fd - g) <= 1e-5 * max(1.0, abs(fd)), (name, i, k, fd, g)
        nb = (deg + 1) ** 2 * 3
        for coef in range(nb):
            pl, comp = coef // 4, coef % 4
            x0 = s64.sh[pl, i, comp]
            h = 1e-6
            s64.sh[pl, i, comp] = x0 + h
            fp = F(s64)
            s64.sh[pl, i, comp] = x0 - h
            fm = F(s64)
            s64.sh[pl, i, comp] = x0
            fd = (fp - fm) / (2 * h)
            assert abs(fd - dsh[pl, i, comp]) <= 1e-6 * max(1.0, abs(fd)), ("sh", i, coef, fd, dsh[pl, i, comp])
    if deg == 0:
        assert np.all(dsh[0, :6, :3] == 0.0)   # clamped colours pass nothing to their SH


def test_end_to_end_finite_differences(grad_case):
    """Composition: project_backward(render_backward(dL/dC)) = central differences of
    L(params) = sum w * C(project_f64(params)) for a sample of parameters."""
    sc, cam, f = grad_case
    w = weights(cam, seed=9)
    g2d, _ = oracle.render_backward(f.rec, f.values, f.ranges, cam.width, cam.height, w, f.bg)
    s64 = _scene64(sc)
    dmo, ds, dr, dsh = oracle.project_backward(s64, cam, g2d)
    w64 = w.astype(np.float64)

    def L():
        return oracle.loss_f64(oracle.project_f64(s64, cam), cam.width, cam.height, w64, f.bg, with_hash=True)

    rng = np.random.default_rng(2)
    vis = np.nonzero(f.rec[:, 11] > 0)[0]
    checked = 0
    for i in rng.choice(vis, 12, replace=False):
        for arr, idx, g in [(s64.mean_opac, (i, 0), dmo[i, 0]), (s64.mean_opac, (i, 2), dmo[i, 2]),
                            (s64.mean_opac, (i, 3), dmo[i, 3]), (s64.scale, (i, 1), ds[i, 1]),
                            (s64.rot, (i, 2), dr[i, 2]), (s64.sh, (0, i, 1), dsh[0, i, 1])]:
            def set_x(v, arr=arr, idx=idx):
                arr[idx] = v
            x0 = arr[idx]
            fd = central_difference(L, set_x, x0, 1e-6 * max(1.0, abs(x0)))
            if fd is None:
                continue
            # float32 records feed the analytic side (R22), float64 the differences
            assert abs(fd - g) <= 2e-4 * max(1.0, abs(fd)), (idx, fd, g)
            checked += 1
    assert checked >= 60
