"""ctypes binding of libss.so (include/ss.h).  Argument marshalling only: every step of
the path runs in libss's CUDA kernels.  There is NO fallback: if libss.so cannot be loaded
the import raises."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SS_LIB_PATH") or os.path.join(HERE, "libss.so")  # SS_LIB_PATH: a variant build

SS_OK, SS_ERR_INVALID_ARG, SS_ERR_CAPACITY, SS_ERR_CUDA, SS_ERR_UNSUPPORTED = range(5)
MODES = {"3sigma": 0, "snugbox": 1, "accutile": 2}

EXPORTS = ["ss_frame_workspace_size", "ss_workspace_size", "ss_frame_layout", "ss_preprocess", "ss_bin", "ss_sort", "ss_sorted_keys",
           "ss_render", "ss_render_stats", "ss_finalize_colours", "ss_prune_score", "ss_render_frame",
           "ss_prune_workspace_size", "ss_prune_count", "ss_prune_select", "ss_compact_scene",
           "ss_render_backward", "ss_preprocess_backward", "ss_l1_loss_grad", "ss_adam_init", "ss_adam_step",
           "ss_preprocess_backward_assign", "ss_adam_step_flagged", "ss_status_string", "ss_last_cuda_error", "ss_version"]


class SsScene(C.Structure):
    _fields_ = [("n", C.c_int32), ("sh_degree", C.c_int32), ("mean_opac", C.c_void_p), ("scale", C.c_void_p),
                ("rot", C.c_void_p), ("sh", C.c_void_p)]


class SsCamera(C.Structure):
    _fields_ = [("viewmat", C.c_float * 12), ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float),
                ("cy", C.c_float), ("campos", C.c_float * 3), ("width", C.c_int32), ("height", C.c_int32),
                ("z_near", C.c_float), ("clip", C.c_float)]


class SsFrame(C.Structure):
    _fields_ = [("ws", C.c_void_p), ("ws_bytes", C.c_size_t), ("n", C.c_int32), ("capacity", C.c_uint32),
                ("width", C.c_int32), ("height", C.c_int32)]


class SsLayout(C.Structure):
    _fields_ = [(k, C.c_size_t) for k in ("rec", "erec", "depth_key", "order", "sorted_value", "tile_count", "ranges", "n_visible", "total_pairs",
                                          "overflow", "overflow_count", "pre_deferred", "scratch", "total_bytes")] + \
               [(k, C.c_int32) for k in ("tiles_x", "tiles_y", "n_tiles", "tile_bits")]


class SsAdamConfig(C.Structure):
    _fields_ = [(k, C.c_float) for k in ("lr_mean", "lr_opacity", "lr_scale", "lr_rot", "lr_sh_dc", "lr_sh_rest",
                                         "beta1", "beta2", "eps")] + [("step", C.c_int32)]


class SsError(RuntimeError):
    pass


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SsError(f"libss.so not built ({LIB_PATH}); run `python -m paper_2412_00578_b200.build`")
        _lib = C.CDLL(LIB_PATH)
        vp, st = C.c_void_p, C.c_int
        P = C.POINTER
        sig = {
            "ss_frame_workspace_size": (C.c_size_t, [C.c_int32, C.c_uint32, C.c_int32, C.c_int32]),
            "ss_frame_layout": (st, [C.c_int32, C.c_uint32, C.c_int32, C.c_int32, P(SsLayout)]),
            "ss_workspace_size": (st, [st, C.c_int32, C.c_uint32, C.c_int32, C.c_int32, P(C.c_size_t)]),
            "ss_preprocess": (st, [P(SsScene), P(SsCamera), st, P(SsFrame), vp]),
            "ss_bin": (st, [P(SsCamera), st, P(SsFrame), vp]),
            "ss_sort": (st, [P(SsFrame), vp]),
            "ss_sorted_keys": (st, [P(SsFrame), vp, vp]),
            "ss_render": (st, [P(SsFrame), P(C.c_float), vp, vp, vp, vp]),
            "ss_render_stats": (st, [P(SsFrame), vp, vp]),
            "ss_finalize_colours": (st, [P(SsFrame), vp]),
            "ss_prune_score": (st, [P(SsFrame), P(C.c_float), vp, vp]),
            "ss_render_frame": (st, [P(SsScene), P(SsCamera), st, P(SsFrame), P(C.c_float), vp, vp, vp, vp]),
            "ss_prune_workspace_size": (C.c_size_t, [C.c_int32]),
            "ss_prune_count": (C.c_uint32, [C.c_int32, C.c_double]),
            "ss_prune_select": (st, [vp, C.c_int32, C.c_double, vp, vp, C.c_size_t, vp]),
            "ss_compact_scene": (st, [P(SsScene), vp, P(SsScene), vp, vp, C.c_size_t, vp]),
            "ss_render_backward": (st, [P(SsFrame), P(C.c_float), vp, vp, vp, vp, vp]),
            "ss_preprocess_backward": (st, [P(SsScene), P(SsCamera), vp, P(SsScene), vp]),
            "ss_l1_loss_grad": (st, [C.c_int64, vp, vp, vp, vp, vp]),
            "ss_adam_init": (st, [P(SsScene), P(SsScene), P(SsScene), P(SsScene), vp]),
            "ss_adam_step": (st, [P(SsScene), P(SsScene), P(SsScene), P(SsScene), P(SsScene), P(SsAdamConfig), vp]),
            "ss_preprocess_backward_assign": (st, [P(SsScene), P(SsCamera), vp, P(SsScene), vp, vp]),
            "ss_adam_step_flagged": (st, [P(SsScene), P(SsScene), P(SsScene), P(SsScene), P(SsScene),
                                          P(SsAdamConfig), vp, vp]),
            "ss_status_string": (C.c_char_p, [st]),
            "ss_last_cuda_error": (C.c_char_p, []),
            "ss_version": (C.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def check(status: int, what: str) -> None:
    if status != SS_OK:
        msg = lib().ss_status_string(status).decode()
        if status == SS_ERR_CUDA:
            msg += " (" + lib().ss_last_cuda_error().decode() + ")"
        raise SsError(f"{what}: {msg}")


def layout(n: int, capacity: int, width: int, height: int) -> SsLayout:
    out = SsLayout()
    check(lib().ss_frame_layout(n, capacity, width, height, C.byref(out)), "ss_frame_layout")
    return out


def workspace_size(n: int, capacity: int, width: int, height: int) -> int:
    return int(lib().ss_frame_workspace_size(n, capacity, width, height))
