"""Seeded synthetic scenes and cameras shared by the CUDA path, the oracle and the bench.

This module holds NONE of the method's arithmetic (no projection, no binning, no
blending, no score).  It only draws random numbers (numpy PCG64, fixed seeds) and
lays them out in the SoA float32 planes both sides read, plus the camera poses.
The workload recipes follow SURVEY.md §8(d) and are restated in DESIGN.md
("Input recipe").

Scene layout (Eq. 1: G = {mu, s, r, h, sigma}):
  mean_opac  float32 [N,4]   x, y, z, opacity sigma in (0,1) (activated)
  scale      float32 [N,4]   linear (activated) scales sx, sy, sz, 0
  rot        float32 [N,4]   quaternion (w, x, y, z), unit norm
  sh         float32 [P,N,4] P = ceil((deg+1)^2*3/4) coefficient-major planes;
                             coefficient k = basis*3 + channel lives in plane k//4,
                             component k%4 (SH h_i in R^{16x3})
Camera ("camera poses", "viewing transform W and a perspective projection"):
  viewmat float32 [3,4] world->camera (rows: right, down, forward | translation)
  fx, fy, cx, cy pixels; campos world centre; width, height; z_near; clip.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SH_PLANES = {0: 1, 1: 3, 2: 7, 3: 12}


@dataclass
class Scene:
    mean_opac: np.ndarray  # [N,4] f32
    scale: np.ndarray      # [N,4] f32
    rot: np.ndarray        # [N,4] f32
    sh: np.ndarray         # [P,N,4] f32
    sh_degree: int
    name: str = "scene"

    @property
    def n(self) -> int:
        return int(self.mean_opac.shape[0])

    def subset(self, idx: np.ndarray) -> "Scene":
        idx = np.asarray(idx)
        return Scene(np.ascontiguousarray(self.mean_opac[idx]), np.ascontiguousarray(self.scale[idx]),
                     np.ascontiguousarray(self.rot[idx]), np.ascontiguousarray(self.sh[:, idx]),
                     self.sh_degree, self.name + "-subset")


@dataclass
class Camera:
    viewmat: np.ndarray            # [3,4] f32 world->camera
    fx: float
    fy: float
    cx: float
    cy: float
    campos: np.ndarray             # [3] f32
    width: int
    height: int
    z_near: float = 0.2
    clip: float = 1.3

    @property
    def tiles_x(self) -> int:
        return (self.width + 15) // 16

    @property
    def tiles_y(self) -> int:
        return (self.height + 15) // 16

    @property
    def n_tiles(self) -> int:
        return self.tiles_x * self.tiles_y


@dataclass
class Workload:
    name: str
    n: int
    width: int
    height: int
    n_views: int
    seed: int
    kind: str                  # "tiny" | "orbit" | "room"
    fovx_deg: float = 60.0
    extra: dict = field(default_factory=dict)


# Workloads of BASELINE.json "configs" (SURVEY.md §8(a) table, §8(d) recipe).
WORKLOADS = {
    "tiny": Workload("tiny", 1000, 256, 256, 1, 0, "tiny"),
    "tiny-lowsigma": Workload("tiny-lowsigma", 1000, 256, 256, 1, 0, "tiny", extra={"low_sigma": True}),
    "tiny-deg0": Workload("tiny-deg0", 1000, 256, 256, 1, 0, "tiny", extra={"sh_degree": 0}),
    "tiny-deg1": Workload("tiny-deg1", 1000, 256, 256, 1, 0, "tiny", extra={"sh_degree": 1}),
    "tiny-deg2": Workload("tiny-deg2", 1000, 256, 256, 1, 0, "tiny", extra={"sh_degree": 2}),
    "truck": Workload("truck", 2_500_000, 979, 546, 251, 1, "orbit"),
    "garden": Workload("garden", 5_800_000, 1297, 840, 185, 2, "orbit"),
    "playroom": Workload("playroom", 2_300_000, 1264, 832, 225, 3, "room", fovx_deg=65.0),
    "mnr360-3m": Workload("mnr360-3m", 3_000_000, 1297, 840, 185, 4, "orbit"),
}


def _haar_quaternions(rng: np.random.Generator, n: int) -> np.ndarray:
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q.astype(np.float32)


def _sh_planes(rng: np.random.Generator, n: int, deg: int) -> np.ndarray:
    n_coef = (deg + 1) ** 2 * 3
    coef = np.zeros((n, SH_PLANES[deg] * 4), np.float32)
    coef[:, 0:3] = rng.normal(0.0, 0.5, (n, 3))             # DC band
    if n_coef > 3:
        coef[:, 3:n_coef] = rng.normal(0.0, 0.05, (n, n_coef - 3))
    return np.ascontiguousarray(coef.reshape(n, SH_PLANES[deg], 4).transpose(1, 0, 2))


def _opacity_u_shaped(rng: np.random.Generator, n: int) -> np.ndarray:
    z = rng.normal(-0.5, 2.5, n)
    s = 1.0 / (1.0 + np.exp(-z))
    return np.clip(s, 1.0 / 255.0 + 1e-3, 0.999)


def look_at(pos, target, width, height, fovx_deg, up=(0.0, 1.0, 0.0), z_near=0.2, clip=1.3) -> Camera:
    """Pinhole camera at `pos` looking at `target`; image x right, y down (right-handed)."""
    pos = np.asarray(pos, np.float64)
    f = np.asarray(target, np.float64) - pos
    f /= np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, np.float64))
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f])
    t = -R @ pos
    vm = np.concatenate([R, t[:, None]], axis=1).astype(np.float32)
    fx = width / (2.0 * math.tan(math.radians(fovx_deg) / 2.0))
    return Camera(vm, float(np.float32(fx)), float(np.float32(fx)), width / 2.0, height / 2.0,
                  pos.astype(np.float32), width, height, z_near, clip)


def tiny_scene(n=1000, seed=0, low_sigma=False, sh_degree=3) -> tuple[Scene, Camera]:
    """SURVEY §8(d) 'Tiny': one 256x256 camera at the origin looking +z, 60 deg FOV.

    Means are drawn in pixel space (u, v in [-32, 288]) and depth z in [2, 8], then
    un-projected; projected 1-sigma extents are ~0.5-30 px; a few special Gaussians
    exercise culling (behind the near plane, opacity <= 1/255) and very large
    footprints (many tile rows).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    W = H = 256
    cam = look_at((0, 0, 0), (0, 0, 1), W, H, 60.0, up=(0, -1, 0))
    # look_at with up=-y gives rows (right=+x, down=+y, fwd=+z): identity world->camera.
    fx = cam.fx
    u = rng.uniform(-32, W + 32, n)
    v = rng.uniform(-32, H + 32, n)
    z = rng.uniform(2.0, 8.0, n)
    x = (u - cam.cx) * z / fx
    y = (v - cam.cy) * z / fx
    px_sigma = np.exp(rng.normal(math.log(4.0), 0.8, (n, 3))).clip(0.5, 30.0)
    scale = px_sigma * z[:, None] / fx
    opac = rng.uniform(0.05, 0.35 if low_sigma else 0.95, n)
    k = max(1, n // 50)
    # special cases: near-plane culls, sub-threshold opacity, huge footprints
    z[:k] = rng.uniform(-1.0, 0.19, k)
    if not low_sigma:
        opac[k:2 * k] = rng.uniform(1e-4, 1.0 / 255.0, k)
    scale[2 * k:2 * k + k // 2] = (rng.uniform(40, 90, (k // 2, 3)) * z[2 * k:2 * k + k // 2, None] / fx)
    mean_opac = np.stack([x, y, z, opac], 1).astype(np.float32)
    sc = np.concatenate([scale, np.zeros((n, 1))], 1).astype(np.float32)
    scene = Scene(mean_opac, sc, _haar_quaternions(rng, n), _sh_planes(rng, n, sh_degree), sh_degree, "tiny")
    return scene, cam


def knife_scene(n=20000, seed=11, sh_degree=0) -> tuple[Scene, Camera]:
    """Stress scene for the tile decisions (the float32-certified geometry of ss_preprocess and
    its float64 fallback): the tiny camera; means on or within 1e-5..1e-1 px of tile lines and
    tile corners, extreme anisotropy (axis ratios up to 1e3, Haar rotations: thin, strongly
    correlated conics), opacities from just above 1/255 (t ~ 0: tiny ellipses) to 0.999,
    footprints from sub-pixel to several hundred pixels (clipped at the image border)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    W = H = 256
    cam = look_at((0, 0, 0), (0, 0, 1), W, H, 60.0, up=(0, -1, 0))
    fx = cam.fx
    line = lambda m: 16.0 * rng.integers(-2, 19, m)
    off = lambda m: rng.choice([0.0, 1e-5, -1e-5, 1e-3, -1e-3, 0.1, -0.1], m) * rng.uniform(0.5, 1.5, m)
    u = np.where(rng.uniform(size=n) < 0.7, line(n) + off(n), rng.uniform(-32, W + 32, n))
    v = np.where(rng.uniform(size=n) < 0.7, line(n) + off(n), rng.uniform(-32, H + 32, n))
    z = rng.uniform(1.0, 10.0, n)
    x = (u - cam.cx) * z / fx
    y = (v - cam.cy) * z / fx
    big = np.exp(rng.uniform(math.log(0.3), math.log(200.0), n))          # px, the long axis
    ratio = np.exp(rng.uniform(0.0, math.log(1e3), (n, 2)))
    px = np.stack([big, big / ratio[:, 0], big / ratio[:, 1]], 1)
    scale = px * z[:, None] / fx
    opac = np.where(rng.uniform(size=n) < 0.3, 1.0 / 255.0 + rng.uniform(1e-7, 1e-3, n),
                    rng.uniform(0.05, 0.999, n))
    mean_opac = np.stack([x, y, z, opac], 1).astype(np.float32)
    sc = np.concatenate([scale, np.zeros((n, 1))], 1).astype(np.float32)
    scene = Scene(mean_opac, sc, _haar_quaternions(rng, n), _sh_planes(rng, n, sh_degree), sh_degree, "knife")
    return scene, cam


def tangent_scene(n=20000, seed=21, sh_degree=0) -> tuple[Scene, Camera]:
    """Stress scene for the swept-axis extremes (the float32-certified geometry's near-tangent
    lines, R28): Gaussians flat along the optical axis and rotated about it by 0 or a
    small-to-moderate angle, placed so that an extreme of their SnugBox, mu_y -+ h_y (or
    mu_x -+ h_x), lands on or within 1e-5..1e-1 px of a tile line -- the Algorithm-1 boundary
    line next to the extreme then grazes the ellipse (discriminant near 0).  h is the
    closed-form half-extent sqrt(t Sigma_2D) of the camera's projection near the image centre
    (the exact float32 value differs slightly, which spreads the distances further)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    W = H = 256
    cam = look_at((0, 0, 0), (0, 0, 1), W, H, 60.0, up=(0, -1, 0))
    f = cam.fx
    z = rng.uniform(2.0, 8.0, n)
    sx_px = np.exp(rng.uniform(math.log(0.5), math.log(60.0), n))
    sy_px = sx_px * np.exp(rng.uniform(math.log(0.05), math.log(20.0), n))
    theta = np.where(rng.uniform(size=n) < 0.3, 0.0, rng.uniform(-0.6, 0.6, n))
    opac = rng.uniform(0.02, 0.999, n)
    t = 2.0 * np.log(255.0 * opac)
    c2, s2 = np.cos(theta) ** 2, np.sin(theta) ** 2
    sxx = c2 * sx_px ** 2 + s2 * sy_px ** 2 + 0.3
    syy = s2 * sx_px ** 2 + c2 * sy_px ** 2 + 0.3
    hx, hy = np.sqrt(t * sxx), np.sqrt(t * syy)
    delta = rng.choice([0.0, 1e-5, -1e-5, 1e-3, -1e-3, 0.1, -0.1], n) * rng.uniform(0.5, 1.5, n)
    line = 16.0 * rng.integers(1, 16, n)
    side = np.where(rng.uniform(size=n) < 0.5, -1.0, 1.0)
    on_y = rng.uniform(size=n) < 0.5
    u = np.where(on_y, rng.uniform(16, 240, n), line - side * hx + delta)
    v = np.where(on_y, line - side * hy + delta, rng.uniform(16, 240, n))
    x = (u - cam.cx) * z / f
    y = (v - cam.cy) * z / f
    scale = np.stack([sx_px * z / f, sy_px * z / f, np.full(n, 1e-4) * z / f], 1)
    quat = np.stack([np.cos(theta / 2), np.zeros(n), np.zeros(n), np.sin(theta / 2)], 1)
    mean_opac = np.stack([x, y, z, opac], 1).astype(np.float32)
    sc = np.concatenate([scale, np.zeros((n, 1))], 1).astype(np.float32)
    scene = Scene(mean_opac, sc, quat.astype(np.float32), _sh_planes(rng, n, sh_degree), sh_degree, "tangent")
    return scene, cam


def dense_scene(n=12000, seed=5, tie_frac=0.5, sh_degree=1) -> tuple[Scene, Camera]:
    """Tile-sort stress case on the tiny camera: means packed into a 64x64 px window at the
    image centre, so the central tiles' lists are longer than one shared-memory sort
    (ss_sort's global-memory path), and a fraction `tie_frac` of the Gaussians share the
    exact depth 5.0 (equal keys, ordered by index)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    W = H = 256
    cam = look_at((0, 0, 0), (0, 0, 1), W, H, 60.0, up=(0, -1, 0))
    fx = cam.fx
    u = rng.uniform(96, 160, n)
    v = rng.uniform(96, 160, n)
    z = rng.uniform(2.0, 8.0, n)
    z[rng.uniform(0, 1, n) < tie_frac] = 5.0
    x = (u - cam.cx) * z / fx
    y = (v - cam.cy) * z / fx
    px_sigma = np.exp(rng.normal(math.log(6.0), 0.6, (n, 3))).clip(1.0, 30.0)
    scale = px_sigma * z[:, None] / fx
    opac = rng.uniform(0.02, 0.3, n)
    mean_opac = np.stack([x, y, z, opac], 1).astype(np.float32)
    sc = np.concatenate([scale, np.zeros((n, 1))], 1).astype(np.float32)
    scene = Scene(mean_opac, sc, _haar_quaternions(rng, n), _sh_planes(rng, n, sh_degree), sh_degree, "dense")
    return scene, cam


def orbit_scene(n, seed, object_frac=0.6, mu_s=-5.75, sd_s=1.0, sh_degree=3, name="orbit") -> Scene:
    """SURVEY §8(d) Mip-NeRF-360-shaped 'object + unbounded background' scene."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n_obj = int(round(object_frac * n))
    obj = rng.normal(0.0, 0.6, (n_obj, 3))
    d = rng.standard_normal((n - n_obj, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:, 1] = np.abs(d[:, 1]) * 0.5                       # flattened upper hemisphere
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rad = np.exp(rng.uniform(math.log(2.0), math.log(20.0), n - n_obj))
    mu = np.concatenate([obj, d * rad[:, None]], 0)
    mu = mu[rng.permutation(n)]
    s = np.exp(rng.normal(mu_s, sd_s, (n, 3))) * np.maximum(1.0, np.linalg.norm(mu, axis=1))[:, None]
    opac = _opacity_u_shaped(rng, n)
    mean_opac = np.concatenate([mu, opac[:, None]], 1).astype(np.float32)
    sc = np.concatenate([s, np.zeros((n, 1))], 1).astype(np.float32)
    return Scene(mean_opac, sc, _haar_quaternions(rng, n), _sh_planes(rng, n, sh_degree), sh_degree, name)


def orbit_cameras(n_views, width, height, radius=4.0, height_y=0.8, fovx_deg=60.0) -> list[Camera]:
    cams = []
    for k in range(n_views):
        a = 2.0 * math.pi * k / n_views
        pos = (radius * math.cos(a), height_y, radius * math.sin(a))
        cams.append(look_at(pos, (0.0, 0.0, 0.0), width, height, fovx_deg))
    return cams


def room_scene(n, seed, sh_degree=3, name="room") -> Scene:
    """SURVEY §8(d) Deep-Blending-playroom-shaped indoor scene: 70% wall-aligned
    Gaussians on a box shell of half-extent (3, 1.5, 4), 30% in 8 furniture clusters."""
    rng = np.random.Generator(np.random.PCG64(seed))
    half = np.array([3.0, 1.5, 4.0])
    n_wall = int(round(0.7 * n))
    face = rng.integers(0, 6, n_wall)
    axis = face // 2
    sign = np.where(face % 2 == 0, -1.0, 1.0)
    p = rng.uniform(-1, 1, (n_wall, 3)) * half
    p[np.arange(n_wall), axis] = sign * half[axis]
    centres = rng.uniform(-1, 1, (8, 3)) * half * 0.7
    c = centres[rng.integers(0, 8, n - n_wall)] + rng.normal(0, 0.35, (n - n_wall, 3))
    mu = np.concatenate([p, c], 0)
    s = np.exp(rng.normal(-5.5, 1.0, (n, 3)))
    s[np.arange(n_wall), axis] *= 0.1
    q = _haar_quaternions(rng, n)
    q[:n_wall] = np.array([1, 0, 0, 0], np.float32)
    perm = rng.permutation(n)
    opac = _opacity_u_shaped(rng, n)
    mean_opac = np.concatenate([mu, opac[:, None]], 1)[perm].astype(np.float32)
    sc = np.concatenate([s, np.zeros((n, 1))], 1)[perm].astype(np.float32)
    sh = _sh_planes(rng, n, sh_degree)[:, perm]
    return Scene(mean_opac, sc, np.ascontiguousarray(q[perm]), np.ascontiguousarray(sh), sh_degree, name)


def room_cameras(n_views, width, height, seed, fovx_deg=65.0) -> list[Camera]:
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    cams = []
    for k in range(n_views):
        pos = rng.uniform(-1, 1, 3) * np.array([1.5, 0.5, 2.0])
        yaw = 2.0 * math.pi * k / n_views + rng.uniform(-0.3, 0.3)
        pitch = rng.uniform(-0.2, 0.2)
        fwd = np.array([math.cos(pitch) * math.cos(yaw), math.sin(pitch), math.cos(pitch) * math.sin(yaw)])
        cams.append(look_at(pos, pos + fwd, width, height, fovx_deg))
    return cams


def make_workload(name: str, n: int | None = None) -> tuple[Scene, list[Camera]]:
    """Scene + camera list for a named workload; `n` overrides the Gaussian count."""
    w = WORKLOADS[name]
    n = w.n if n is None else n
    if w.kind == "tiny":
        sc, cam = tiny_scene(n, w.seed, low_sigma=w.extra.get("low_sigma", False),
                             sh_degree=w.extra.get("sh_degree", 3))
        sc.name = name
        return sc, [cam]
    if w.kind == "orbit":
        sc = orbit_scene(n, w.seed, name=name)
        return sc, orbit_cameras(w.n_views, w.width, w.height, fovx_deg=w.fovx_deg)
    sc = room_scene(n, w.seed, name=name)
    return sc, room_cameras(w.n_views, w.width, w.height, w.seed, fovx_deg=w.fovx_deg)


def random_conics(n, seed, tiles=40, cond_max=1e3, sigma_range=(1.0 / 255.0 + 1e-6, 1.0)):
    """Random positive-definite 2-D covariances / opacities / means on a `tiles`x`tiles`
    grid (SURVEY F6 battery: cond <= 1e3, sigma in (1/255,1)).  Returns float64 arrays
    (mx, my, cov_xx, cov_xy, cov_yy, sigma); the conic is derived by the caller."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lam1 = np.exp(rng.uniform(math.log(0.5), math.log(400.0), n))
    cond = np.exp(rng.uniform(0.0, math.log(cond_max), n))
    lam2 = np.maximum(lam1 / cond, 0.3)
    th = rng.uniform(0, math.pi, n)
    c, s = np.cos(th), np.sin(th)
    cxx = c * c * lam1 + s * s * lam2
    cyy = s * s * lam1 + c * c * lam2
    cxy = c * s * (lam1 - lam2)
    mx = rng.uniform(-20, tiles * 16 + 20, n)
    my = rng.uniform(-20, tiles * 16 + 20, n)
    sig = rng.uniform(sigma_range[0], sigma_range[1], n)
    return mx, my, cxx, cxy, cyy, sig


def grad_scene(n=40, width=72, height=40, seed=7, opac=(0.05, 0.5), px_sigma=(1.0, 6.0), sh_degree=3,
               margin=8.0, yaw_deg=0.0) -> tuple[Scene, Camera]:
    """Small scene for the backward pins and parity tests: `n` Gaussians in
    front of a width x height camera (ragged tiles when the sides are not multiples of 16),
    means uniform in pixel space (-margin .. side+margin) at depth z in [2, 6], projected
    1-sigma extents log-uniform in `px_sigma`, opacity uniform in `opac` (the default upper
    bound keeps transmittance far from the 1e-4 stop), Haar quaternions, SH as the tiny
    scene.  `yaw_deg` turns the camera so the world->camera rotation is not the identity."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cam0 = look_at((0, 0, 0), (0, 0, 1), width, height, 60.0, up=(0, -1, 0))
    u = rng.uniform(-margin, width + margin, n)
    v = rng.uniform(-margin, height + margin, n)
    z = rng.uniform(2.0, 6.0, n)
    x = (u - cam0.cx) * z / cam0.fx
    y = (v - cam0.cy) * z / cam0.fy
    pxs = np.exp(rng.uniform(math.log(px_sigma[0]), math.log(px_sigma[1]), (n, 3)))
    scale = pxs * z[:, None] / cam0.fx
    o = rng.uniform(opac[0], opac[1], n)
    p_cam = np.stack([x, y, z], 1)
    if yaw_deg:
        a = math.radians(yaw_deg)
        pos = np.array([0.3, -0.2, 0.1])
        fwd = np.array([math.sin(a), 0.0, math.cos(a)])
        cam = look_at(pos, pos + fwd, width, height, 60.0, up=(0, -1, 0))
        Rm = cam.viewmat[:, :3].astype(np.float64)
        world = (p_cam - cam.viewmat[:, 3].astype(np.float64)) @ Rm  # R^T (p - t)
    else:
        cam, world = cam0, p_cam
    mean_opac = np.concatenate([world, o[:, None]], 1).astype(np.float32)
    sc = np.concatenate([scale, np.zeros((n, 1))], 1).astype(np.float32)
    q = rng.standard_normal((n, 4))
    q *= rng.uniform(0.5, 2.0, (n, 1)) / np.linalg.norm(q, axis=1, keepdims=True)  # non-unit: normalised in-kernel
    return Scene(mean_opac, sc, q.astype(np.float32), _sh_planes(rng, n, sh_degree), sh_degree, "grad"), cam


def perturb(scene: Scene, seed=1, mean_sd=0.01, logit_sd=0.5, dc_sd=0.2, log_scale_sd=0.2) -> Scene:
    """A noisy copy of `scene` (NEXT-3 training init): means + N(0, mean_sd), opacity logits
    + N(0, logit_sd), SH DC + N(0, dc_sd), log-scales + N(0, log_scale_sd)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = scene.n
    mo = scene.mean_opac.astype(np.float64).copy()
    mo[:, :3] += rng.normal(0, mean_sd, (n, 3))
    o = np.clip(mo[:, 3], 1e-4, 1 - 1e-4)
    logit = np.log(o / (1 - o)) + rng.normal(0, logit_sd, n)
    mo[:, 3] = 1.0 / (1.0 + np.exp(-logit))
    sc = scene.scale.astype(np.float64).copy()
    sc[:, :3] *= np.exp(rng.normal(0, log_scale_sd, (n, 3)))
    sh = scene.sh.copy()
    sh[0, :, :3] += rng.normal(0, dc_sd, (n, 3)).astype(np.float32)
    return Scene(mo.astype(np.float32), sc.astype(np.float32), scene.rot.copy(), sh, scene.sh_degree,
                 scene.name + "-perturbed")
