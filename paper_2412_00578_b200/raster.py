"""Public Python API over libss (the five C-ABI calls of include/ss.h).

PyTorch is plumbing only: device memory (the scene planes, the frame workspace, outputs)
and the current CUDA stream.  Every computation runs in libss's kernels; there is no CPU
or PyTorch fallback -- constructing a Rasterizer without a CUDA device or without
libss.so raises.

    scene = DeviceScene.from_host(synth_scene)            # SoA planes -> HBM
    rz = Rasterizer(scene, width, height, mode="accutile")
    img = rz.render_frame(camera)                         # [3, H, W] float32 on the device
    rz.prune_score(score)                                 # score[i] += U~_i for that frame
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from ._abi import MODES, SsCamera, SsFrame, SsScene, check, lib


@dataclass
class DeviceScene:
    mean_opac: torch.Tensor   # [N,4] f32 cuda
    scale: torch.Tensor       # [N,4]
    rot: torch.Tensor         # [N,4]
    sh: torch.Tensor          # [N,B,4] per-Gaussian SH blocks
    sh_degree: int

    @property
    def n(self) -> int:
        return int(self.mean_opac.shape[0])

    @staticmethod
    def from_host(scene, device="cuda") -> "DeviceScene":
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(device)
        # SH: host planes [B][N][4] -> the device's per-Gaussian blocks [N][B][4] (include/ss.h)
        return DeviceScene(t(scene.mean_opac), t(scene.scale), t(scene.rot), t(np.transpose(scene.sh, (1, 0, 2))),
                           int(scene.sh_degree))

    def struct(self) -> SsScene:
        return SsScene(self.n, self.sh_degree, self.mean_opac.data_ptr(), self.scale.data_ptr(),
                       self.rot.data_ptr(), self.sh.data_ptr())

    def zeros_like(self) -> "DeviceScene":
        """Gradient arrays with the scene's layout (ss_scene_grad), zero-filled."""
        z = torch.zeros_like
        return DeviceScene(z(self.mean_opac), z(self.scale), z(self.rot), z(self.sh), self.sh_degree)

    def host_sh_planes(self) -> np.ndarray:
        """SH in the host layout [B][N][4] (the inverse of from_host's transpose)."""
        return np.ascontiguousarray(np.transpose(self.sh.cpu().numpy(), (1, 0, 2)))


def camera_struct(cam) -> SsCamera:
    if isinstance(cam, SsCamera):
        return cam
    c = SsCamera()
    c.viewmat[:] = [float(v) for v in np.asarray(cam.viewmat, np.float32).reshape(-1)]
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.campos[:] = [float(v) for v in np.asarray(cam.campos, np.float32)]
    c.width, c.height = int(cam.width), int(cam.height)
    c.z_near, c.clip = float(cam.z_near), float(cam.clip)
    return c


def _stream_handle(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class Rasterizer:
    """One frame workspace (HBM) for a scene and an image size; reusable across views."""

    def __init__(self, scene: DeviceScene, width: int, height: int, mode: str = "accutile",
                 capacity: int | None = None, device=None):
        if not torch.cuda.is_available():
            raise _abi.SsError("libss requires a CUDA device (no CPU fallback)")
        lib()  # fail loudly if libss.so is missing
        self.scene = scene
        self.width, self.height = int(width), int(height)
        self.mode = mode
        self.device = device or scene.mean_opac.device
        self._scene_struct = scene.struct()
        self.capacity = 0
        self._alloc(capacity if capacity is not None else max(1024, 4 * scene.n))

    # ---------------------------------------------------------------- workspace
    def _alloc(self, capacity: int) -> None:
        capacity = int(min(capacity, (1 << 30) - 1))
        nbytes = _abi.workspace_size(self.scene.n, capacity, self.width, self.height)
        # zero-filled once: the sticky overflow counter starts at 0, and the kernels' reads of
        # record words they never use (a 32 B emission record is read whole) see defined bytes
        self.ws = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        self.capacity = capacity
        self.layout = _abi.layout(self.scene.n, capacity, self.width, self.height)
        self.frame = SsFrame(self.ws.data_ptr(), nbytes, self.scene.n, capacity, self.width, self.height)
        self.n_tiles = self.layout.n_tiles

    def _view(self, off: int, count: int, dtype: torch.dtype) -> torch.Tensor:
        itemsize = torch.tensor([], dtype=dtype).element_size()
        return self.ws[off: off + count * itemsize].view(dtype)

    # views of the intermediates (zero-copy)
    def records(self) -> torch.Tensor:
        """[N, 12] float32 render records: (x, y, a, b | c, t, sigma, 0 | f, r, g, b); valid
        only where depth_keys() != 0xFFFFFFFF; the colour only where f = 1 (call
        finalize_colours() first to complete them all)."""
        return self._view(self.layout.rec, 12 * self.scene.n, torch.float32).view(self.scene.n, 12)

    def emit_records(self) -> torch.Tensor:
        """[N, 8] int32 emission records: (count, info, payload 0..5) (include/ss.h)."""
        return self._view(self.layout.erec, 8 * self.scene.n, torch.int32).view(self.scene.n, 8)

    def counts(self) -> torch.Tensor:
        """Per-Gaussian tile count of the current frame (int32, 0 for Gaussians without tiles)."""
        c = self.emit_records()[:, 0]
        return torch.where(self.depth_keys() == -1, torch.zeros_like(c), c)

    def depth_keys(self) -> torch.Tensor:
        return self._view(self.layout.depth_key, self.scene.n, torch.int32)

    def order(self) -> torch.Tensor:
        return self._view(self.layout.order, self.scene.n, torch.int32)

    def sorted_values(self) -> torch.Tensor:
        return self._view(self.layout.sorted_value, self.capacity, torch.int32)

    def ranges(self) -> torch.Tensor:
        return self._view(self.layout.ranges, 2 * self.n_tiles, torch.int32).view(self.n_tiles, 2)

    def tile_counts(self) -> torch.Tensor:
        return self._view(self.layout.tile_count, self.n_tiles, torch.int32)

    def totals(self) -> dict:
        """Device counters (synchronises): visible Gaussians, pairs P, overflow flag."""
        nv = int(self._view(self.layout.n_visible, 1, torch.int32).item())
        P = int(self._view(self.layout.total_pairs, 1, torch.int32).item()) & 0xFFFFFFFF
        ov = int(self._view(self.layout.overflow, 1, torch.int32).item())
        dfr = int(self._view(self.layout.pre_deferred, 1, torch.int32).item())
        return {"n_visible": nv, "pairs": P, "overflow": ov, "deferred": dfr}

    def overflow_count(self) -> int:
        """Frames of this workspace whose pairs exceeded the capacity since the last
        clear_overflow() (sticky device counter; synchronises)."""
        return int(self._view(self.layout.overflow_count, 1, torch.int32).item())

    def clear_overflow(self) -> None:
        self._view(self.layout.overflow_count, 1, torch.int32).zero_()

    # ---------------------------------------------------------------- the five calls
    def preprocess(self, cam, stream=None) -> None:
        self._cam = camera_struct(cam)
        check(lib().ss_preprocess(C.byref(self._scene_struct), C.byref(self._cam), MODES[self.mode],
                                  C.byref(self.frame), C.c_void_p(_stream_handle(stream))), "ss_preprocess")

    def bin(self, cam=None, stream=None) -> None:
        c = camera_struct(cam) if cam is not None else self._cam
        check(lib().ss_bin(C.byref(c), MODES[self.mode], C.byref(self.frame),
                           C.c_void_p(_stream_handle(stream))), "ss_bin")

    def sort(self, stream=None) -> None:
        check(lib().ss_sort(C.byref(self.frame), C.c_void_p(_stream_handle(stream))), "ss_sort")

    def sorted_keys(self, stream=None) -> torch.Tensor:
        keys = torch.zeros(max(1, self.capacity), dtype=torch.int64, device=self.device)
        check(lib().ss_sorted_keys(C.byref(self.frame), C.c_void_p(keys.data_ptr()),
                                   C.c_void_p(_stream_handle(stream))), "ss_sorted_keys")
        return keys

    def render(self, bg=(0.0, 0.0, 0.0), out: torch.Tensor | None = None, want_T=False, want_ncontrib=False,
               stream=None):
        if out is None:
            out = torch.empty((3, self.height, self.width), dtype=torch.float32, device=self.device)
        T = torch.empty((self.height, self.width), dtype=torch.float32, device=self.device) if want_T else None
        nc = torch.empty((self.height, self.width), dtype=torch.int32, device=self.device) if want_ncontrib else None
        bgv = (C.c_float * 3)(*[float(v) for v in bg])
        check(lib().ss_render(C.byref(self.frame), bgv, C.c_void_p(out.data_ptr()),
                              C.c_void_p(T.data_ptr() if T is not None else 0),
                              C.c_void_p(nc.data_ptr() if nc is not None else 0),
                              C.c_void_p(_stream_handle(stream))), "ss_render")
        if want_T or want_ncontrib:
            return out, T, nc
        return out

    def finalize_colours(self, stream=None) -> None:
        """Compute every record colour still pending (inspection; the render path computes the
        colours it needs lazily)."""
        check(lib().ss_finalize_colours(C.byref(self.frame), C.c_void_p(_stream_handle(stream))),
              "ss_finalize_colours")

    def render_stats(self, stream=None) -> dict:
        """Work counts of the render for the current frame (measurement; synchronises)."""
        c = torch.zeros(5, dtype=torch.int64, device=self.device)
        check(lib().ss_render_stats(C.byref(self.frame), C.c_void_p(c.data_ptr()),
                                    C.c_void_p(_stream_handle(stream))), "ss_render_stats")
        v = c.cpu().tolist()
        return {"E_pix": v[0], "E_blend": v[1], "E_cta": v[2], "pixels": v[3], "phantom_pairs": v[4]}

    def prune_score(self, score: torch.Tensor, bg=(0.0, 0.0, 0.0), stream=None) -> torch.Tensor:
        assert score.dtype == torch.float64 and score.numel() == self.scene.n and score.is_cuda
        bgv = (C.c_float * 3)(*[float(v) for v in bg])
        check(lib().ss_prune_score(C.byref(self.frame), bgv, C.c_void_p(score.data_ptr()),
                                   C.c_void_p(_stream_handle(stream))), "ss_prune_score")
        return score

    # ---------------------------------------------------------------- backward (NEXT-2)
    def render_backward(self, dL_dimg: torch.Tensor, T_final: torch.Tensor, n_contrib: torch.Tensor,
                        grad2d: torch.Tensor | None = None, bg=(0.0, 0.0, 0.0), stream=None) -> torch.Tensor:
        """grad2d [N, 12] float32 += dL/d(x2d, y2d, a, b | c, sigma, r, g | b, -, -, -) of the
        current frame, from dL/dC (float32 [3, H, W]) and the T_final / n_contrib of its render."""
        if grad2d is None:
            grad2d = torch.zeros((self.scene.n, 12), dtype=torch.float32, device=self.device)
        for t, shape in ((dL_dimg, (3, self.height, self.width)), (T_final, (self.height, self.width)),
                         (n_contrib, (self.height, self.width))):
            assert tuple(t.shape) == shape and t.is_cuda and t.is_contiguous()
        assert grad2d.dtype == torch.float32 and grad2d.shape == (self.scene.n, 12) and grad2d.is_contiguous()
        bgv = (C.c_float * 3)(*[float(v) for v in bg])
        check(lib().ss_render_backward(C.byref(self.frame), bgv, C.c_void_p(dL_dimg.data_ptr()),
                                       C.c_void_p(T_final.data_ptr()), C.c_void_p(n_contrib.data_ptr()),
                                       C.c_void_p(grad2d.data_ptr()), C.c_void_p(_stream_handle(stream))),
              "ss_render_backward")
        return grad2d

    def preprocess_backward(self, cam, grad2d: torch.Tensor, grads: DeviceScene | None = None,
                            stream=None) -> DeviceScene:
        """Scene-parameter gradients += chain rule of ss_preprocess applied to grad2d."""
        if grads is None:
            grads = self.scene.zeros_like()
        g = grads.struct()
        c = camera_struct(cam)
        check(lib().ss_preprocess_backward(C.byref(self._scene_struct), C.byref(c), C.c_void_p(grad2d.data_ptr()),
                                           C.byref(g), C.c_void_p(_stream_handle(stream))), "ss_preprocess_backward")
        return grads

    def forward_backward(self, cam, dL_dimg_fn, bg=(0.0, 0.0, 0.0), grads: DeviceScene | None = None,
                         stream=None):
        """One training-style step for a view: render, dL/dC = dL_dimg_fn(image), render
        backward, preprocess backward.  Returns (image, grads, grad2d)."""
        img, T, nc = self.render_frame(cam, bg, want_T=True, want_ncontrib=True, stream=stream)
        grad2d = self.render_backward(dL_dimg_fn(img), T, nc, bg=bg, stream=stream)
        grads = self.preprocess_backward(cam, grad2d, grads, stream=stream)
        return img, grads, grad2d

    # ---------------------------------------------------------------- conveniences
    def prepare(self, cam, stream=None) -> None:
        """a1-a5 for one view (preprocess, bin, sort)."""
        self.preprocess(cam, stream)
        self.bin(cam, stream)
        self.sort(stream)

    def ensure_capacity(self, cam, headroom: float = 1.25) -> int:
        """Run a1-a3 once, read P back (synchronises) and grow the pair capacity if needed."""
        self.preprocess(cam)
        self.bin(cam)
        P = self.totals()["pairs"]
        if P > self.capacity:
            self._alloc(int(P * headroom) + 1024)
        return P

    def render_frame(self, cam, bg=(0.0, 0.0, 0.0), out=None, check_overflow=True, stream=None, **kw):
        """Full forward frame.  With check_overflow the pair count is read back and the
        frame re-run once with a larger workspace if the capacity was exceeded."""
        self.prepare(cam, stream)
        if check_overflow and self.totals()["overflow"]:
            self._alloc(int(self.totals()["pairs"] * 1.25) + 1024)
            self.prepare(cam, stream)
        return self.render(bg, out, stream=stream, **kw)


class FramePipeline:
    """N frame workspaces on N CUDA streams (views are independent).

    Views are dealt round-robin to the streams, so one frame's latency-bound kernels (the
    scans, the look-back depth passes, the small level-2 kernels) overlap another frame's
    bandwidth-bound preprocess and render instead of leaving SMs idle between launches
    (measured on B200, MNR360-3M: 1 stream 1263 frames/s, 2 -> 1470, 3 -> 1538, 4 -> 1544).
    Within a stream the frame's kernels keep their programmatic dependent launches."""

    def __init__(self, scene: DeviceScene, width: int, height: int, mode: str = "accutile", n_streams: int = 4,
                 capacity: int | None = None):
        self.n_streams = int(n_streams)
        self.width, self.height = int(width), int(height)
        self.rz = [Rasterizer(scene, width, height, mode=mode, capacity=capacity) for _ in range(self.n_streams)]
        dev = self.rz[0].device
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(self.n_streams)]
        self.outs = [torch.empty((3, height, width), dtype=torch.float32, device=dev) for _ in range(self.n_streams)]
        self._graphs = {}   # (workspace, camera bytes, bg) -> CUDA graph of that frame's a1-a6

    # ---------------------------------------------------------------- CUDA graphs
    def _graph_key(self, k: int, c: SsCamera, bg) -> tuple:
        return (k, bytes(c), tuple(float(v) for v in bg))

    def capture(self, cams, bg=(0.0, 0.0, 0.0)) -> int:
        """Capture, for every camera and every workspace, the frame's whole launch sequence
        (ss_render_frame: 2 memsets + the a1-a6 kernels with their programmatic dependent
        launches) into a CUDA graph, so that render_views(..., graphs=True) enqueues a frame
        with one graph launch instead of ~20 kernel launches (the host enqueue otherwise
        approaches the GPU time per frame).  The graphs bake in the camera, the workspace and
        its output buffer; re-capture after ensure_capacity() reallocates.  Returns the number
        of graphs captured (synchronises)."""
        bgv = (C.c_float * 3)(*[float(v) for v in bg])
        mode = MODES[self.rz[0].mode]
        fn = lib().ss_render_frame
        n = 0
        for cam in cams:
            c = camera_struct(cam)
            for k, (rz, st) in enumerate(zip(self.rz, self.streams)):
                key = self._graph_key(k, c, bg)
                if key in self._graphs:
                    continue
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(st):
                    g.capture_begin()
                    status = fn(C.byref(rz._scene_struct), C.byref(c), mode, C.byref(rz.frame), bgv,
                                C.c_void_p(self.outs[k].data_ptr()), None, None, C.c_void_p(int(st.cuda_stream)))
                    g.capture_end()
                check(status, "ss_render_frame (capture)")
                self._graphs[key] = g
                n += 1
        torch.cuda.synchronize()
        return n

    def drop_graphs(self) -> None:
        self._graphs.clear()

    def ensure_capacity(self, cams, headroom: float = 1.02) -> int:
        """Size every workspace for the largest pair count over `cams` (synchronises)."""
        P = max(self.rz[0].ensure_capacity(c, headroom) for c in cams)
        cap = int(P * headroom) + 4096
        for r in self.rz:
            if r.capacity != cap:
                r._alloc(cap)
                self._graphs.clear()   # the graphs point at the old workspaces
        self.clear_overflow()
        return P

    def overflow_count(self) -> int:
        """Frames (on any workspace) whose pairs exceeded the capacity since the last
        clear_overflow(): one device read per workspace (synchronises).  The render / score
        calls never read it themselves (they only enqueue work); a caller that did not size
        the workspaces with ensure_capacity() checks it after a batch."""
        return sum(r.overflow_count() for r in self.rz)

    def clear_overflow(self) -> None:
        for r in self.rz:
            r.clear_overflow()

    def check_overflow(self) -> None:
        """Raise SsError if a frame since the last clear_overflow() overflowed its workspace
        (its image would be background only, its score contribution zero)."""
        k = self.overflow_count()
        if k:
            raise _abi.SsError(f"{k} frame(s) exceeded the pair capacity {self.rz[0].capacity}; "
                               f"call ensure_capacity() for these cameras and re-run them")

    def render_views(self, cams, bg=(0.0, 0.0, 0.0), on_frame=None, pre_events=None, graphs: bool = False) -> None:
        """Render every camera (a1-a6).  on_frame(j, image, stream) is called right after
        frame j is enqueued, on its stream (e.g. to enqueue a device->host copy); image is
        that stream's output buffer, reused by the stream's next frame.  pre_events[j]
        (optional pair of CUDA events) brackets frame j's ss_preprocess on its stream.  The
        caller's current stream waits for all frames on return (no host synchronisation)."""
        cur = torch.cuda.current_stream()
        for st in self.streams:
            st.wait_stream(cur)
        if graphs:
            # one graph launch per frame on its workspace's stream (capture() must have seen
            # every (camera, workspace) pair); on_frame runs after the frame's launch
            for j, cam in enumerate(cams):
                k = j % self.n_streams
                c = camera_struct(cam)
                g = self._graphs.get(self._graph_key(k, c, bg))
                if g is None:
                    raise _abi.SsError("render_views(graphs=True): frame not captured; call capture(cams) first")
                with torch.cuda.stream(self.streams[k]):
                    g.replay()
                    if on_frame is not None:
                        on_frame(j, self.outs[k], self.streams[k])
            for st in self.streams:
                cur.wait_stream(st)
            return
        if pre_events is None and on_frame is None:
            # the plain path: one C-ABI call per frame (ss_render_frame = a1-a6), no per-frame
            # Python stream contexts -- the host enqueues a frame in a fraction of its GPU time
            bgv = (C.c_float * 3)(*[float(v) for v in bg])
            mode = MODES[self.rz[0].mode]
            handles = [C.c_void_p(int(st.cuda_stream)) for st in self.streams]
            fn = lib().ss_render_frame
            for j, cam in enumerate(cams):
                k = j % self.n_streams
                rz = self.rz[k]
                c = camera_struct(cam)
                status = fn(C.byref(rz._scene_struct), C.byref(c), mode, C.byref(rz.frame), bgv,
                            C.c_void_p(self.outs[k].data_ptr()), None, None, handles[k])
                if status:
                    check(status, "ss_render_frame")
            for st in self.streams:
                cur.wait_stream(st)
            return
        for j, cam in enumerate(cams):
            k = j % self.n_streams
            st, rz = self.streams[k], self.rz[k]
            with torch.cuda.stream(st):
                e = pre_events[j] if pre_events is not None else None
                if e is not None:
                    e[0].record(st)
                rz.preprocess(cam, st)
                if e is not None:
                    e[1].record(st)
                rz.bin(cam, st)
                rz.sort(st)
                rz.render(bg, out=self.outs[k], stream=st)
                if on_frame is not None:
                    on_frame(j, self.outs[k], st)
        for st in self.streams:
            cur.wait_stream(st)


    def score_views(self, cams, score: torch.Tensor, bg=(0.0, 0.0, 0.0)) -> torch.Tensor:
        """a1-a5 + a7 for every camera, the frames in flight on the pipeline's streams, all
        adding into the one float64 score vector (device atomics; no host synchronisation).
        The caller's current stream waits for all frames on return."""
        assert score.dtype == torch.float64 and score.is_cuda
        cur = torch.cuda.current_stream()
        for st in self.streams:
            st.wait_stream(cur)
        for j, cam in enumerate(cams):
            k = j % self.n_streams
            st, rz = self.streams[k], self.rz[k]
            with torch.cuda.stream(st):
                rz.prepare(cam, st)
                rz.prune_score(score, bg, stream=st)
        for st in self.streams:
            cur.wait_stream(st)
        return score


def render_views_to_host(pipe: "FramePipeline", cams, host_out: list, bg=(0.0, 0.0, 0.0), graphs: bool = False) -> None:
    """End-to-end public call: render each camera and land its image in pinned host memory.

    Frames run on the pipeline's streams; frame j's device->host copy is enqueued on its own
    stream right after its render (the copy engine overlaps the other streams' kernels, and the
    stream's next frame waits for the copy before reusing the buffer).  Returns after the last
    copy completes.  host_out[j] must be pinned float32 [3, H, W] tensors."""
    def copy(j, img, st):
        host_out[j].copy_(img, non_blocking=True)
    cs = [camera_struct(c) for c in cams]
    pipe.render_views(cs, bg, on_frame=copy, graphs=graphs)
    torch.cuda.current_stream().synchronize()
    if pipe.overflow_count():   # a view needed more pairs than the workspaces hold: grow, redo
        pipe.clear_overflow()
        pipe.ensure_capacity(cs)
        pipe.render_views(cs, bg, on_frame=copy)
        torch.cuda.current_stream().synchronize()
        pipe.check_overflow()


def prune_select(score: torch.Tensor, ratio: float, stream=None) -> tuple[torch.Tensor, int]:
    """keep mask (uint8, device) removing k = floor(ratio N) Gaussians with the smallest score
    (ties: higher index first), and k."""
    assert score.dtype == torch.float64 and score.is_cuda and score.dim() == 1
    n = score.numel()
    k = int(lib().ss_prune_count(n, float(ratio)))
    ws = torch.empty(int(lib().ss_prune_workspace_size(n)), dtype=torch.uint8, device=score.device)
    keep = torch.empty(n, dtype=torch.uint8, device=score.device)
    check(lib().ss_prune_select(C.c_void_p(score.data_ptr()), n, float(ratio), C.c_void_p(keep.data_ptr()),
                                C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(_stream_handle(stream))),
          "ss_prune_select")
    return keep, k


def compact(scene: DeviceScene, keep: torch.Tensor, n_keep: int, stream=None) -> DeviceScene:
    """Stable stream compaction of every array of a scene-shaped set (scene, or optimiser
    state with the scene's layout) by `keep` (ss_compact_scene)."""
    n, m, dev = scene.n, int(n_keep), scene.mean_opac.device
    out = DeviceScene(torch.empty((max(m, 1), 4), dtype=torch.float32, device=dev)[:m],
                      torch.empty((max(m, 1), 4), dtype=torch.float32, device=dev)[:m],
                      torch.empty((max(m, 1), 4), dtype=torch.float32, device=dev)[:m],
                      torch.empty((m, scene.sh.shape[1], 4), dtype=torch.float32, device=dev), scene.sh_degree)
    ws = torch.empty(int(lib().ss_prune_workspace_size(n)), dtype=torch.uint8, device=dev)
    n_out = torch.zeros(1, dtype=torch.int32, device=dev)
    src, dst = scene.struct(), out.struct()
    check(lib().ss_compact_scene(C.byref(src), C.c_void_p(keep.data_ptr()), C.byref(dst),
                                 C.c_void_p(n_out.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(),
                                 C.c_void_p(_stream_handle(stream))), "ss_compact_scene")
    got = int(n_out.item())   # synchronises: a mismatched mask must not yield a short scene
    if got != m:
        raise _abi.SsError(f"compact: the keep mask keeps {got} Gaussians, the caller allocated {m}")
    return out


def prune(scene: DeviceScene, score: torch.Tensor, ratio: float, stream=None) -> tuple[DeviceScene, torch.Tensor]:
    """The prune step (Sec. 4.2): drop floor(ratio * N) Gaussians with the smallest score (ties:
    higher index first) and return the compacted scene plus the keep mask.  Every rank that
    holds the same all-reduced score gets the same scene (no further exchange)."""
    assert score.numel() == scene.n
    keep, k = prune_select(score, ratio, stream)
    return compact(scene, keep, scene.n - k, stream), keep
