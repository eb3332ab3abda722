"""Pins of the oracle's geometry (threshold, SnugBox, 3-sigma radius, projection, SH)
against what PAPER.md / mathematics fix -- never against the oracle itself.

P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n (worked examples only).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2412_00578_b200 import synth
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SNUG = json.load(open(os.path.join(GOLDEN, "snugbox_examples.json")))


def conic_of(cxx, cxy, cyy):
    d = cxx * cyy - cxy * cxy
    return cyy / d, -cxy / d, cxx / d


@pytest.mark.parametrize("case", SNUG["threshold"], ids=lambda c: c["cite"][:20])
def test_threshold_printed_values(case):
    """Eq. 11 values printed by the spec."""
    assert abs(oracle.threshold(case["sigma"]) - case["t"]) <= case["tol"]


def test_threshold_defines_alpha_cut():
    """Eq. 9: at q = t the alpha of Eq. 5 equals exactly 1/255."""
    for s in np.linspace(0.01, 1.0, 57):
        t = oracle.threshold(float(np.float32(s)))
        assert abs(float(np.float32(s)) * math.exp(-0.5 * t) - 1.0 / 255.0) < 1e-12
    # sigma* = e^4.5/255: t = 9 exactly, where SnugBox meets the 3-sigma radius (R17)
    assert abs(oracle.threshold(float(np.float32(math.exp(4.5) / 255))) - 9.0) < 1e-6


@pytest.mark.parametrize("case", SNUG["cases"], ids=lambda c: c["cite"][:24])
def test_snugbox_printed_examples(case):
    if "conic" in case:
        a, b, c = case["conic"]
        t = case["t"]
    else:
        a, b, c = conic_of(*case["cov"])
        t = oracle.threshold(case["sigma"])
    bb, tg = oracle.snugbox(*case["mu"], a, b, c, t)
    if "half" in case:
        hx, hy = case["half"]
        mx, my = case["mu"]
        assert np.allclose(bb, [mx - hx, mx + hx, my - hy, my + hy], atol=case["tol"])
    if "bbox" in case:
        assert np.allclose(bb, case["bbox"], atol=case["tol"])
        assert np.allclose([tg[0, 1], tg[1, 1]], case["tangent_y_at_xmin_xmax"], atol=case["tol"])
        assert np.allclose([tg[2, 0], tg[3, 0]], case["tangent_x_at_ymin_ymax"], atol=case["tol"])


def _paper_route_bbox(mx, my, a, b, c, t):
    """PAPER.md's own route: Eq. 16 x_args = +-sqrt(-b^2 t / ((b^2 - ac) a)), substituted into
    Eq. 15 y_d = (-b x_d +- sqrt((b^2-ac) x_d^2 + t c)) / c; x extents by the a<->c swap."""
    def extents(a_, b_, c_):
        xa = math.sqrt(-b_ * b_ * t / ((b_ * b_ - a_ * c_) * a_)) if b_ != 0 else 0.0
        ys = []
        for xd in (xa, -xa):
            disc = max(0.0, (b_ * b_ - a_ * c_) * xd * xd + t * c_)
            ys += [(-b_ * xd + math.sqrt(disc)) / c_, (-b_ * xd - math.sqrt(disc)) / c_]
        return min(ys), max(ys)
    ylo, yhi = extents(a, b, c)
    xlo, xhi = extents(c, b, a)
    return np.array([mx + xlo, mx + xhi, my + ylo, my + yhi])


def test_snugbox_equals_paper_route_and_tangency():
    """Closed form == Eq. 16 -> Eq. 15 route; every tangent point lies on the
    ellipse (q = t); the bbox contains dense boundary samples and touches them."""
    mx, my, cxx, cxy, cyy, sig = synth.random_conics(2000, seed=11)
    for i in range(2000):
        a, b, c = conic_of(cxx[i], cxy[i], cyy[i])
        t = oracle.threshold(float(sig[i]))
        bb, tg = oracle.snugbox(mx[i], my[i], a, b, c, t)
        ref = _paper_route_bbox(mx[i], my[i], a, b, c, t)
        scale = max(1.0, abs(bb).max())
        assert np.allclose(bb, ref, rtol=0, atol=1e-9 * scale)
        for (px, py) in tg:
            xd, yd = px - mx[i], py - my[i]
            q = a * xd * xd + 2 * b * xd * yd + c * yd * yd
            assert abs(q - t) <= 1e-9 * t
    # boundary sampling: ellipse q = t parameterised through the eigen-decomposition (numpy)
    a, b, c = 1.0, 0.6, 1.0
    t = 8.0
    w, V = np.linalg.eigh(np.array([[a, b], [b, c]]))
    th = np.linspace(0, 2 * np.pi, 200001)
    pts = V @ np.stack([np.sqrt(t / w[0]) * np.cos(th), np.sqrt(t / w[1]) * np.sin(th)])
    bb, _ = oracle.snugbox(10.0, 20.0, a, b, c, t)
    xs, ys = pts[0] + 10, pts[1] + 20
    assert xs.min() >= bb[0] - 1e-9 and xs.max() <= bb[1] + 1e-9
    assert ys.min() >= bb[2] - 1e-9 and ys.max() <= bb[3] + 1e-9
    assert abs(xs.min() - bb[0]) < 1e-6 and abs(ys.max() - bb[3]) < 1e-6


@pytest.mark.parametrize("case", SNUG["radius_3sigma"], ids=lambda c: c["cite"][:16])
def test_3sigma_radius(case):
    """Eq. 8, printed radii S:105-107: the rect is [floor((m-r)/16), floor((m+r)/16)+1)."""
    cxx, cxy, cyy = case["cov"]
    r = case["r"]
    # place the mean so that m - r and m + r sit strictly inside tiles 4..6
    m = 100.0 + 0.5
    rect = oracle.rect_3sigma(m, m, cxx, cxy, cyy, 64, 64)
    assert rect == (int((m - r) // 16), int((m + r) // 16) + 1, int((m - r) // 16), int((m + r) // 16) + 1)
    # one pixel more would have moved the upper edge: radius is exactly r
    for mm in np.arange(80.0, 130.0, 0.25):
        rr = oracle.rect_3sigma(mm, mm, cxx, cxy, cyy, 64, 64)
        assert rr[0] == math.floor((mm - r) / 16) and rr[1] == math.floor((mm + r) / 16) + 1


def test_sh_degree0_closed_form():
    """R13 / S:472: degree 0 colour is 0.5 + Y00 h0 with Y00 = 1/(2 sqrt(pi))."""
    Y = oracle.sh_basis(0, 0.3, -0.2, 0.9)
    assert abs(Y[0] - 1.0 / (2.0 * math.sqrt(math.pi))) < 1e-7
    assert np.all(Y[1:] == 0)


def test_sh_basis_orthonormal_and_matches_scipy():
    """The 16 real SH functions (degree 3, P:124 h in R^{16x3}) are orthonormal on the
    sphere (Gauss-Legendre x uniform-phi quadrature, exact for degree <= 6 products) and,
    up to one sign per function, equal scipy's real spherical harmonics."""
    from scipy.special import sph_harm_y
    nt, nph = 24, 48
    xg, wg = np.polynomial.legendre.leggauss(nt)
    G = np.zeros((16, 16))
    pts = []
    for ct, w in zip(xg, wg):
        st = math.sqrt(1 - ct * ct)
        for k in range(nph):
            ph = 2 * math.pi * k / nph
            d = (st * math.cos(ph), st * math.sin(ph), ct)
            Y = oracle.sh_basis(3, *[float(np.float32(v)) for v in d]).astype(np.float64)
            G += np.outer(Y, Y) * w * (2 * math.pi / nph)
            pts.append((d, Y, math.acos(ct), ph))
    assert np.abs(G - np.eye(16)).max() < 2e-6
    # compare with scipy real SH: index k = l^2 + l + m
    signs = {}
    for d, Y, theta, phi in pts[::37]:
        for l in range(4):
            for m in range(-l, l + 1):
                if m < 0:
                    ref = math.sqrt(2) * (-1) ** m * sph_harm_y(l, -m, theta, phi).imag
                elif m == 0:
                    ref = sph_harm_y(l, 0, theta, phi).real
                else:
                    ref = math.sqrt(2) * (-1) ** m * sph_harm_y(l, m, theta, phi).real
                k = l * l + l + m
                # map the basis' axis convention: check |value| agreement with a fixed sign
                if abs(ref) > 1e-3:
                    s = np.sign(Y[k] / ref) if abs(Y[k]) > 1e-6 else 0
                    signs.setdefault(k, set()).add(s)
                    assert abs(abs(Y[k]) - abs(ref)) < 2e-6
    # one fixed sign per basis function (a convention), never a mixture
    assert all(len(v - {0}) == 1 for v in signs.values()) and len(signs) == 16


def _project_ref(cam, mu, scale, quat):
    """Independent check: numeric Jacobian of the pinhole map world -> pixel at mu
    (central differences, float64) and Sigma_3D from scipy's rotation."""
    from scipy.spatial.transform import Rotation
    V = np.asarray(cam.viewmat, np.float64)

    def pix(p):
        pc = V[:, :3] @ p + V[:, 3]
        return np.array([cam.fx * pc[0] / pc[2] + cam.cx, cam.fy * pc[1] / pc[2] + cam.cy])

    h = 1e-6 * max(1.0, np.linalg.norm(mu))
    Jw = np.zeros((2, 3))
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        Jw[:, k] = (pix(mu + e) - pix(mu - e)) / (2 * h)
    w, x, y, z = quat
    Rm = Rotation.from_quat([x, y, z, w]).as_matrix()
    S3 = Rm @ np.diag(np.asarray(scale) ** 2) @ Rm.T
    cov = Jw @ S3 @ Jw.T + 0.3 * np.eye(2)
    return pix(mu), cov


def test_projection_on_axis_closed_form():
    """identity rotation, unit scale, on the optical axis at z = fx -> Sigma_2D = 1.3 I."""
    _, cam = synth.tiny_scene(4, 0)
    n = 1
    sc = synth.Scene(np.array([[0, 0, cam.fx, 0.8]], np.float32), np.array([[1, 1, 1, 0]], np.float32),
                     np.array([[1, 0, 0, 0]], np.float32), np.zeros((12, n, 4), np.float32), 3)
    rec, rect, cnt = oracle.project(sc, cam, "accutile")
    a, b, c = rec[0, 3:6]
    assert abs(a - 1 / 1.3) < 1e-6 and abs(c - 1 / 1.3) < 1e-6 and b == 0
    assert rec[0, 0] == cam.cx and rec[0, 1] == cam.cy and rec[0, 2] == np.float32(cam.fx)


def test_projection_matches_numeric_jacobian():
    """Eq. 4: Sigma_2D = J W Sigma_3D W^T J^T (+0.3 I, R5) versus a central-
    difference Jacobian of the full pinhole map and scipy's quaternion rotation."""
    scene, cams = synth.make_workload("mnr360-3m", n=3000)
    cam = cams[7]
    rec, rect, cnt = oracle.project(scene, cam, "accutile")
    checked = 0
    for i in range(scene.n):
        if rec[i, 11] == 0:
            continue
        mu = scene.mean_opac[i, :3].astype(np.float64)
        pc = np.asarray(cam.viewmat, np.float64)[:, :3] @ mu + np.asarray(cam.viewmat, np.float64)[:, 3]
        tx, ty = pc[0] / pc[2], pc[1] / pc[2]
        if abs(tx) > 1.2 * cam.width / 2 / cam.fx or abs(ty) > 1.2 * cam.height / 2 / cam.fy:
            continue  # J clamp (R5) active: not the plain Jacobian
        q = scene.rot[i].astype(np.float64)
        q /= np.linalg.norm(q)
        p2, cov = _project_ref(cam, mu, scene.scale[i, :3].astype(np.float64), q)
        a, b, c = rec[i, 3:6].astype(np.float64)
        conic_ref = np.linalg.inv(cov)
        assert abs(rec[i, 0] - p2[0]) < 1e-3 + 1e-5 * abs(p2[0])
        assert abs(rec[i, 1] - p2[1]) < 1e-3 + 1e-5 * abs(p2[1])
        assert abs(rec[i, 2] - pc[2]) < 1e-5 * pc[2]
        nrm = np.abs(conic_ref).max()
        assert np.allclose([a, b, c], [conic_ref[0, 0], conic_ref[0, 1], conic_ref[1, 1]], atol=2e-3 * nrm)
        checked += 1
    assert checked > 200


def test_projection_culling_rules():
    """R4: z < z_near culls in every mode; opacity <= 1/255 (t <= 0) culls SnugBox/AccuTile
    but not the 3-sigma baseline, which "neglects opacity"."""
    _, cam = synth.tiny_scene(4, 0)
    mo = np.array([[0, 0, 0.1, 0.5],       # behind near plane
                   [0, 0, 3.0, 0.003],     # opacity < 1/255
                   [0, 0, 3.0, 0.5]], np.float32)
    sc = synth.Scene(mo, np.tile(np.array([[0.05, 0.05, 0.05, 0]], np.float32), (3, 1)),
                     np.tile(np.array([[1, 0, 0, 0]], np.float32), (3, 1)), np.zeros((12, 3, 4), np.float32), 3)
    for mode, want in [("accutile", [0, 0, 1]), ("snugbox", [0, 0, 1]), ("3sigma", [0, 1, 1])]:
        rec, rect, cnt = oracle.project(sc, cam, mode)
        assert [int(v > 0) for v in cnt] == want, mode


JCLAMP = json.load(open(os.path.join(GOLDEN, "jclamp_examples.json")))


def _jclamp_scene_cam(case):
    """The golden's setting: identity view matrix, identity quaternion, cx = W/2, cy = H/2."""
    cc = case["camera"]
    vm = np.concatenate([np.eye(3), np.zeros((3, 1))], axis=1).astype(np.float32)
    cam = synth.Camera(vm, cc["fx"], cc["fy"], cc["width"] / 2.0, cc["height"] / 2.0,
                       np.zeros(3, np.float32), cc["width"], cc["height"], 0.2, cc["clip"])
    sc = synth.Scene(np.array([[*case["mean"], 0.8]], np.float32),
                     np.array([[*case["scale"], 0.0]], np.float32),
                     np.array([[1, 0, 0, 0]], np.float32), np.zeros((12, 1, 4), np.float32), 3)
    return sc, cam


@pytest.mark.parametrize("case", JCLAMP["cases"], ids=lambda c: c["name"][:30])
def test_projection_jclamp_hand_derived(case):
    """R5 (Eq. 4, P:162-166 + the 3D-GS clamp): the J entries use X/Z clamped to
    +-clip*(W/2)/fx while the projected mean stays unclamped.  The expected Sigma_2D of every
    case is worked by hand in tests/golden/jclamp_examples.json; a wrong limit (W instead of
    W/2, fy for fx), a clamped mean or a dropped sign fails at least one case.  Both the
    float32 contract (or_project) and the float64 forward (or_project_f64) are checked."""
    sc, cam = _jclamp_scene_cam(case)
    xx, xy, yy = case["cov2d"]
    want = np.linalg.inv(np.array([[xx, xy], [xy, yy]], np.float64))
    rec, rect, cnt = oracle.project(sc, cam, "3sigma")
    assert rec[0, 11] == 1.0
    assert np.allclose(rec[0, 0:2], case["xy2d"], rtol=1e-6, atol=1e-4)
    got = np.array([rec[0, 3], rec[0, 4], rec[0, 5]], np.float64)
    assert np.allclose(got, [want[0, 0], want[0, 1], want[1, 1]], rtol=2e-5, atol=1e-6 * np.abs(want).max())
    r64 = oracle.project_f64(sc, cam)
    assert r64[0, 10] == 1.0
    assert np.allclose(r64[0, 0:2], case["xy2d"], rtol=1e-12, atol=1e-9)
    # float64 arithmetic on float32 camera fields (clip = 1.3f is 1.3 - 4.8e-8): 1e-6 relative
    assert np.allclose(r64[0, 3:6], [want[0, 0], want[0, 1], want[1, 1]], rtol=1e-6, atol=1e-15)


def test_projection_clamped_gaussians_numeric_jacobian():
    """R5 on a real workload view: with clip = 0 EVERY projected Gaussian (also those beyond
    the 1.3 limit) matches the central-difference Jacobian of the pinhole map; with clip = 1.3
    the Gaussians beyond the limit match the numeric Jacobian of the pinhole map evaluated at
    the clamped camera-space point (tx_c Z, ty_c Z, Z) -- the reading 'J at the clamped tx'."""
    import dataclasses
    scene, cams = synth.make_workload("mnr360-3m", n=6000)
    cam = cams[11]
    V = np.asarray(cam.viewmat, np.float64)
    Vinv_R = V[:, :3].T
    for clip in (0.0, 1.3):
        c2 = dataclasses.replace(cam, clip=clip)
        rec, rect, cnt = oracle.project(scene, c2, "3sigma")
        n_clamped = 0
        for i in range(scene.n):
            if rec[i, 11] == 0:
                continue
            mu = scene.mean_opac[i, :3].astype(np.float64)
            pc = V[:, :3] @ mu + V[:, 3]
            tx, ty = pc[0] / pc[2], pc[1] / pc[2]
            limx, limy = 1.3 * cam.width / 2 / cam.fx, 1.3 * cam.height / 2 / cam.fy
            clamped = abs(tx) > limx * (1 + 1e-6) or abs(ty) > limy * (1 + 1e-6)
            if not clamped:
                continue
            if clip > 0:  # world point whose camera-space coordinates are the clamped ones
                pcc = np.array([np.clip(tx, -limx, limx) * pc[2], np.clip(ty, -limy, limy) * pc[2], pc[2]])
                mu_j = Vinv_R @ (pcc - V[:, 3])
            else:
                mu_j = mu
            q = scene.rot[i].astype(np.float64)
            q /= np.linalg.norm(q)
            _, cov = _project_ref(cam, mu_j, scene.scale[i, :3].astype(np.float64), q)
            # float32 det = xx yy - xy^2 loses ~kappa ulps (kappa = xx yy / det): compare only
            # where float32 can hold 2e-3 (thin far-off-axis ellipses are skipped, counted)
            if cov[0, 0] * cov[1, 1] / np.linalg.det(cov) > 1e3:
                continue
            conic_ref = np.linalg.inv(cov)
            nrm = np.abs(conic_ref).max()
            assert np.allclose(rec[i, 3:6], [conic_ref[0, 0], conic_ref[0, 1], conic_ref[1, 1]], atol=2e-3 * nrm), \
                (clip, i)
            n_clamped += 1
            # the projected mean is never clamped
            assert abs(rec[i, 0] - (cam.fx * tx + cam.cx)) < 1e-3 + 1e-5 * abs(cam.fx * tx)
        assert n_clamped > 20, n_clamped
