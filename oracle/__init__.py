"""CPU oracle for the Speedy-Splat forward hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import this package.  The product path (paper_2412_00578_b200) never imports,
links or executes it; the two share no code.  The arithmetic lives in ss_oracle.c
(plain C, -ffp-contract=off); this module only marshals numpy arrays through ctypes.
See ss_oracle.c's header for the precision contract and the citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ss_oracle.c")
_SRC_BWD = os.path.join(_HERE, "ss_oracle_bwd.c")  # render / preprocess backward (NEXT-2)
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

MODES = {"3sigma": 0, "snugbox": 1, "accutile": 2}
R_NF = 12
REC_FIELDS = ["x", "y", "depth", "a", "b", "c", "sigma", "t", "r", "g", "b_", "vis"]

GCC_FLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-Wall", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain C; the checker, not the product)."""
    srcs = [_SRC, _SRC_BWD]
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(f) for f in srcs):
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", _LIB_PATH, *srcs, "-lm"])
    return _LIB_PATH


class OrCamera(C.Structure):
    _fields_ = [("viewmat", C.c_float * 12), ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float),
                ("cy", C.c_float), ("campos", C.c_float * 3), ("width", C.c_int32), ("height", C.c_int32),
                ("z_near", C.c_float), ("clip", C.c_float)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, f, i, u32, u64, vp = C.c_double, C.c_float, C.c_int, C.c_uint32, C.c_uint64, C.c_void_p
        sig = {
            "or_sh_basis": (None, [i, f, f, f, vp]),
            "or_threshold": (d, [f]),
            "or_snugbox": (None, [d, d, d, d, d, d, vp, vp]),
            "or_rect_snugbox": (None, [d, d, d, d, d, d, i, i, vp]),
            "or_rect_3sigma": (None, [d, d, d, d, d, i, i, vp]),
            "or_accutile": (u32, [d, d, d, d, d, d, i, i, vp, u32, vp, i]),
            "or_tiles_exact": (u32, [d, d, d, d, d, d, i, i, vp]),
            "or_project": (None, [i, i, vp, vp, vp, vp, vp, i, vp, vp, vp]),
            "or_tiles_of_record": (u32, [i, vp, vp, i, i, vp, u32]),
            "or_exclusive_scan": (u64, [i, vp, vp]),
            "or_duplicate_with_keys": (u64, [i, i, vp, vp, vp, vp, i, i, vp, vp]),
            "or_sort_pairs": (None, [u64, vp, vp]),
            "or_tile_ranges": (None, [u64, vp, i, vp]),
            "or_render": (None, [vp, vp, vp, i, i, vp, vp, vp, vp]),
            "or_global_order": (None, [i, vp, vp, vp]),
            "or_render_unbinned": (None, [vp, vp, u32, i, i, vp, i, i, i, i, vp]),
            "or_prune_score": (None, [vp, vp, vp, i, vp, vp, i, i, i, i]),
            "or_composite_alphas": (None, [i, vp, vp, vp, vp]),
            "or_render_tiles": (None, [vp, vp, vp, i, i, vp, vp, i, vp, vp, vp]),
            "or_prune_score_tiles": (None, [vp, vp, vp, i, i, vp, vp, vp, i]),
            "or_prune_select": (C.c_int64, [i, vp, d, vp]),
            "or_project_f64": (None, [i, i, vp, vp, vp, vp, vp, vp]),
            "or_loss_f64": (d, [i, vp, i, i, vp, vp, i, i, i, i, vp]),
            "or_render_backward": (None, [vp, vp, vp, i, i, vp, vp, i, i, i, i, vp, vp]),
            "or_render_backward_tiles": (None, [vp, vp, vp, i, i, vp, vp, vp, i, vp, vp]),
            "or_project_backward": (None, [i, i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "or_l1_loss_grad": (d, [C.c_int64, vp, vp, vp]),
            "or_adam_step": (None, [C.c_int64, vp, vp, vp, vp, vp, vp, vp, d, d, d, C.c_int32]),
            "or_frame": (u64, [i, i, vp, vp, vp, vp, vp, i, vp, vp, vp, vp, vp, vp, vp, u64, vp, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def camera(cam) -> OrCamera:
    oc = OrCamera()
    oc.viewmat[:] = [float(v) for v in np.asarray(cam.viewmat, np.float32).reshape(-1)]
    oc.fx, oc.fy, oc.cx, oc.cy = cam.fx, cam.fy, cam.cx, cam.cy
    oc.campos[:] = [float(v) for v in np.asarray(cam.campos, np.float32)]
    oc.width, oc.height, oc.z_near, oc.clip = cam.width, cam.height, cam.z_near, cam.clip
    return oc


# ---- geometry -------------------------------------------------------------------------

def sh_basis(deg: int, x: float, y: float, z: float) -> np.ndarray:
    out = np.zeros(16, np.float32)
    lib().or_sh_basis(deg, x, y, z, _p(out))
    return out


def threshold(sigma: float) -> float:
    return lib().or_threshold(sigma)


def snugbox(mx, my, a, b, c, t):
    bb = np.zeros(4)
    tg = np.zeros(8)
    lib().or_snugbox(mx, my, a, b, c, t, _p(bb), _p(tg))
    return bb, tg.reshape(4, 2)


def rect_snugbox(mx, my, a, b, c, t, tiles_x, tiles_y):
    r = np.zeros(4, np.int32)
    lib().or_rect_snugbox(mx, my, a, b, c, t, tiles_x, tiles_y, _p(r))
    return tuple(int(v) for v in r)


def rect_3sigma(mx, my, cxx, cxy, cyy, tiles_x, tiles_y):
    r = np.zeros(4, np.int32)
    lib().or_rect_3sigma(mx, my, cxx, cxy, cyy, tiles_x, tiles_y, _p(r))
    return tuple(int(v) for v in r)


def accutile(mx, my, a, b, c, t, tiles_x, tiles_y, force_dir=-1):
    """Returns (sorted tile-id array, n_line_solves)."""
    cap = tiles_x * tiles_y + 1
    out = np.zeros(cap, np.uint32)
    ns = C.c_int32(0)
    n = lib().or_accutile(mx, my, a, b, c, t, tiles_x, tiles_y, _p(out), cap, C.byref(ns), force_dir)
    return np.sort(out[:n]), ns.value


def tiles_exact(mx, my, a, b, c, t, tiles_x, tiles_y) -> np.ndarray:
    mask = np.zeros(tiles_x * tiles_y, np.uint8)
    lib().or_tiles_exact(mx, my, a, b, c, t, tiles_x, tiles_y, _p(mask))
    return np.nonzero(mask)[0].astype(np.uint32)


# ---- pipeline -------------------------------------------------------------------------

def project(scene, cam, mode: str):
    n = scene.n
    rec = np.zeros((n, R_NF), np.float32)
    rect = np.zeros((n, 4), np.int32)
    cnt = np.zeros(n, np.uint32)
    lib().or_project(n, scene.sh_degree, _p(scene.mean_opac), _p(scene.scale), _p(scene.rot), _p(scene.sh),
                     C.byref(camera(cam)), MODES[mode], _p(rec), _p(rect), _p(cnt))
    return rec, rect, cnt


def tiles_of_record(mode: str, rec_row: np.ndarray, rect_row: np.ndarray, tiles_x, tiles_y) -> np.ndarray:
    rec_row = np.ascontiguousarray(rec_row, np.float32)
    rect_row = np.ascontiguousarray(rect_row, np.int32)
    cap = tiles_x * tiles_y + 1
    out = np.zeros(cap, np.uint32)
    n = lib().or_tiles_of_record(MODES[mode], _p(rec_row), _p(rect_row), tiles_x, tiles_y, _p(out), cap)
    return out[:n].copy()


def exclusive_scan(counts: np.ndarray):
    counts = np.ascontiguousarray(counts, np.uint32)
    off = np.zeros(len(counts), np.uint64)
    total = lib().or_exclusive_scan(len(counts), _p(counts), _p(off))
    return off, int(total)


def sort_pairs(keys: np.ndarray, values: np.ndarray):
    k = np.ascontiguousarray(keys, np.uint64).copy()
    v = np.ascontiguousarray(values, np.uint32).copy()
    lib().or_sort_pairs(len(k), _p(k), _p(v))
    return k, v


def tile_ranges(sorted_keys: np.ndarray, n_tiles: int) -> np.ndarray:
    k = np.ascontiguousarray(sorted_keys, np.uint64)
    r = np.zeros((n_tiles, 2), np.uint32)
    lib().or_tile_ranges(len(k), _p(k), n_tiles, _p(r))
    return r


class Frame:
    """Every intermediate of one oracle view (CS3)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def frame(scene, cam, mode: str = "accutile", bg=(0.0, 0.0, 0.0), render=True, cap_hint=None) -> Frame:
    n = scene.n
    rec = np.zeros((n, R_NF), np.float32)
    rect = np.zeros((n, 4), np.int32)
    cnt = np.zeros(n, np.uint32)
    off = np.zeros(n, np.uint64)
    n_tiles = cam.tiles_x * cam.tiles_y
    ranges = np.zeros((n_tiles, 2), np.uint32)
    bgv = np.asarray(bg, np.float32)
    oc = camera(cam)
    cap = int(cap_hint) if cap_hint else 0
    keys = np.zeros(max(cap, 1), np.uint64)
    vals = np.zeros(max(cap, 1), np.uint32)
    img = np.zeros((3, cam.height, cam.width), np.float32) if render else None
    T = np.zeros((cam.height, cam.width), np.float32) if render else None
    nc = np.zeros((cam.height, cam.width), np.uint32) if render else None
    for _ in range(2):
        P = lib().or_frame(n, scene.sh_degree, _p(scene.mean_opac), _p(scene.scale), _p(scene.rot),
                           _p(scene.sh), C.byref(oc), MODES[mode], _p(bgv), _p(rec), _p(rect), _p(cnt),
                           _p(off), _p(keys), _p(vals), cap, _p(ranges), _p(img), _p(T), _p(nc))
        if P <= cap:
            break
        cap = int(P)
        keys = np.zeros(max(cap, 1), np.uint64)
        vals = np.zeros(max(cap, 1), np.uint32)
    P = int(P)
    return Frame(rec=rec, rect=rect, counts=cnt, offsets=off, P=P, keys=keys[:P], values=vals[:P],
                 ranges=ranges, image=img, T=T, ncontrib=nc, mode=mode, bg=bgv)


def render(rec, values, ranges, width, height, bg=(0.0, 0.0, 0.0)):
    img = np.zeros((3, height, width), np.float32)
    T = np.zeros((height, width), np.float32)
    nc = np.zeros((height, width), np.uint32)
    bgv = np.asarray(bg, np.float32)
    lib().or_render(_p(np.ascontiguousarray(rec, np.float32)), _p(np.ascontiguousarray(values, np.uint32)),
                    _p(np.ascontiguousarray(ranges, np.uint32)), width, height, _p(bgv), _p(img), _p(T), _p(nc))
    return img, T, nc


def render_unbinned(rec, width, height, bg=(0.0, 0.0, 0.0), window=None):
    rec = np.ascontiguousarray(rec, np.float32)
    order = np.zeros(len(rec), np.uint32)
    nv = C.c_uint32(0)
    lib().or_global_order(len(rec), _p(rec), _p(order), C.byref(nv))
    img = np.zeros((3, height, width), np.float32)
    x0, x1, y0, y1 = window if window else (0, width, 0, height)
    bgv = np.asarray(bg, np.float32)
    lib().or_render_unbinned(_p(rec), _p(order), nv.value, width, height, _p(bgv), x0, x1, y0, y1, _p(img))
    return img


def prune_score(rec, values, ranges, width, height, bg=(0.0, 0.0, 0.0), score=None, window=None):
    rec = np.ascontiguousarray(rec, np.float32)
    if score is None:
        score = np.zeros(len(rec), np.float64)
    x0, x1, y0, y1 = window if window else (0, width, 0, height)
    bgv = np.asarray(bg, np.float32)
    lib().or_prune_score(_p(rec), _p(np.ascontiguousarray(values, np.uint32)),
                         _p(np.ascontiguousarray(ranges, np.uint32)), width, _p(bgv), _p(score),
                         x0, x1, y0, y1)
    return score


def composite_alphas(alpha, rgb, bg=(0.0, 0.0, 0.0)) -> np.ndarray:
    alpha = np.ascontiguousarray(alpha, np.float64)
    rgb = np.ascontiguousarray(rgb, np.float64)
    out = np.zeros(3)
    lib().or_composite_alphas(len(alpha), _p(alpha), _p(rgb), _p(np.asarray(bg, np.float64)), _p(out))
    return out


def score_views(scene, cams, mode="accutile", bg=(0.0, 0.0, 0.0)) -> np.ndarray:
    """U~ summed over a list of views (oracle side of the multi-view score)."""
    s = np.zeros(scene.n, np.float64)
    for cam in cams:
        f = frame(scene, cam, mode, bg, render=False)
        prune_score(f.rec, f.values, f.ranges, cam.width, cam.height, bg, s)
    return s


def render_tiles(rec, values, ranges, width, height, tiles, bg=(0.0, 0.0, 0.0)):
    """Oracle render of a list of tiles only; pixels outside those tiles are NaN."""
    img = np.full((3, height, width), np.nan, np.float32)
    T = np.full((height, width), np.nan, np.float32)
    nc = np.zeros((height, width), np.uint32)
    tl = np.ascontiguousarray(tiles, np.int32)
    lib().or_render_tiles(_p(np.ascontiguousarray(rec, np.float32)), _p(np.ascontiguousarray(values, np.uint32)),
                          _p(np.ascontiguousarray(ranges, np.uint32)), width, height,
                          _p(np.asarray(bg, np.float32)), _p(tl), len(tl), _p(img), _p(T), _p(nc))
    return img, T, nc


def prune_score_tiles(rec, values, ranges, width, height, tiles, bg=(0.0, 0.0, 0.0), score=None):
    rec = np.ascontiguousarray(rec, np.float32)
    if score is None:
        score = np.zeros(len(rec), np.float64)
    tl = np.ascontiguousarray(tiles, np.int32)
    lib().or_prune_score_tiles(_p(rec), _p(np.ascontiguousarray(values, np.uint32)),
                               _p(np.ascontiguousarray(ranges, np.uint32)), width, height,
                               _p(np.asarray(bg, np.float32)), _p(score), _p(tl), len(tl))
    return score


def prune_select(score: np.ndarray, ratio: float):
    """keep mask (uint8) and k = floor(ratio * N) removed (lowest scores, higher index first on ties)."""
    score = np.ascontiguousarray(score, np.float64)
    keep = np.zeros(len(score), np.uint8)
    k = lib().or_prune_select(len(score), _p(score), float(ratio), _p(keep))
    return keep, int(k)


# ---- backward (ss_oracle_bwd.c) ----------------------------------------
G_FIELDS = ["x", "y", "a", "b", "c", "sigma", "r", "g", "b_"]   # g2d columns
F_NF = 11                                                        # or_project_f64 record width


def project_f64(scene, cam) -> np.ndarray:
    """float64 projection (parameters read as float64; scene arrays may be float64) rec64[n][11] = (x2d, y2d, depth, a, b, c, sigma, r, g, b, visible)."""
    out = np.zeros((scene.n, F_NF), np.float64)
    mo, sc, ro, sh = (np.ascontiguousarray(a, np.float64) for a in (scene.mean_opac, scene.scale, scene.rot, scene.sh))
    lib().or_project_f64(scene.n, scene.sh_degree, _p(mo), _p(sc), _p(ro), _p(sh), C.byref(camera(cam)), _p(out))
    return out


def loss_f64(rec64, width, height, weights, bg=(0.0, 0.0, 0.0), window=None, with_hash=False):
    """L = sum w * C of the float64 unbinned render of rec64 (weights float64 [3][H][W]);
    with_hash: also the hash of the blended (pixel, Gaussian) set."""
    rec64 = np.ascontiguousarray(rec64, np.float64)
    w = np.ascontiguousarray(weights, np.float64)
    x0, x1, y0, y1 = window if window else (0, width, 0, height)
    h = C.c_uint64(0)
    L = lib().or_loss_f64(len(rec64), _p(rec64), width, height, _p(np.asarray(bg, np.float64)), _p(w),
                          x0, x1, y0, y1, C.byref(h))
    return (L, h.value) if with_hash else L


def render_backward(rec, values, ranges, width, height, dimg, bg=(0.0, 0.0, 0.0), window=None,
                    tiles=None, g2d=None, gabs=None):
    """dL/d(x2d, y2d, a, b, c, sigma, r, g, b) per Gaussian (float64 [n][9], accumulated) and
    the sums of absolute per-pixel terms (same shape).  dimg = dL/dC float32 [3][H][W]."""
    rec = np.ascontiguousarray(rec, np.float32)
    n = len(rec)
    if g2d is None:
        g2d = np.zeros((n, 9), np.float64)
    if gabs is None:
        gabs = np.zeros((n, 9), np.float64)
    dimg = np.ascontiguousarray(dimg, np.float32)
    bgv = np.asarray(bg, np.float32)
    v = np.ascontiguousarray(values, np.uint32)
    r = np.ascontiguousarray(ranges, np.uint32)
    if tiles is not None:
        tl = np.ascontiguousarray(tiles, np.int32)
        lib().or_render_backward_tiles(_p(rec), _p(v), _p(r), width, height, _p(bgv), _p(dimg), _p(tl), len(tl),
                                       _p(g2d), _p(gabs))
    else:
        x0, x1, y0, y1 = window if window else (0, width, 0, height)
        lib().or_render_backward(_p(rec), _p(v), _p(r), width, height, _p(bgv), _p(dimg), x0, x1, y0, y1,
                                 _p(g2d), _p(gabs))
    return g2d, gabs


def project_backward(scene, cam, g2d):
    """Accumulated float64 parameter gradients (dmean_opac [n][4], dscale [n][4], drot [n][4],
    dsh like scene.sh) from g2d float64 [n][9]."""
    n = scene.n
    dmo = np.zeros((n, 4), np.float64)
    ds = np.zeros((n, 4), np.float64)
    dr = np.zeros((n, 4), np.float64)
    dsh = np.zeros(scene.sh.shape, np.float64)
    g2d = np.ascontiguousarray(g2d, np.float64)
    mo, sc, ro, sh = (np.ascontiguousarray(a, np.float64) for a in (scene.mean_opac, scene.scale, scene.rot, scene.sh))
    lib().or_project_backward(n, scene.sh_degree, _p(mo), _p(sc), _p(ro), _p(sh), C.byref(camera(cam)), _p(g2d),
                              _p(dmo), _p(ds), _p(dr), _p(dsh))
    return dmo, ds, dr, dsh


# ---- NEXT-3: L1 loss gradient and the Adam step (ss_oracle_bwd.c) -----------------------
def l1_loss_grad(img, gt):
    """(L, dL/dimg float32) for L = mean |img - gt|."""
    img = np.ascontiguousarray(img, np.float32)
    gt = np.ascontiguousarray(gt, np.float32)
    g = np.zeros_like(img)
    L = lib().or_l1_loss_grad(img.size, _p(img), _p(gt), _p(g))
    return L, g


def adam_step(grad_act, raw, m, v, act_of, lr_of, b1=0.9, b2=0.999, eps=1e-15, t=1):
    """One Adam step on float64 arrays (raw, m, v updated in place); returns the activated
    parameters.  act_of: 0 identity, 1 exp, 2 sigmoid (per element); lr_of per element."""
    arrs = [np.ascontiguousarray(a, np.float64) for a in (grad_act, raw, m, v)]
    for a, src in zip(arrs[1:], (raw, m, v)):
        assert a is src, "raw / m / v must be C-contiguous float64 (updated in place)"
    out = np.zeros_like(arrs[1])
    act = np.ascontiguousarray(np.broadcast_to(act_of, arrs[1].shape), np.int32)
    lr = np.ascontiguousarray(np.broadcast_to(lr_of, arrs[1].shape), np.float64)
    lib().or_adam_step(arrs[1].size, _p(arrs[0]), _p(arrs[1]), _p(arrs[2]), _p(arrs[3]), _p(out), _p(act), _p(lr),
                       b1, b2, eps, t)
    return out
