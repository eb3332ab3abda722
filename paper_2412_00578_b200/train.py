"""Pruning-in-the-loop training on synthetic targets.

The paper's training pipeline (Eq. 2, Sec. 4.2): per iteration one view is rendered,
the L1 loss against its target image is differentiated (ss_l1_loss_grad), the gradient flows
through the render backward and the preprocess backward (NEXT-2) into the scene parameters,
and Adam updates them (ss_adam_step).  At the schedule's events the efficient pruning score
Ũ is accumulated over every training view (ss_prune_score, Eqs. 20-21), all-reduced across
ranks, and the lowest ⌊ratio·N⌋ Gaussians are removed together with their optimiser state
(Soft Pruning "immediately before the three opacity resets at 6000, 9000 and 12000", P:424;
Hard Pruning "a constant ratio every 3000 iterations" after densification).  There is
no densification and no opacity reset: the schedule scales the paper's
iterations down (`scaled_schedule`).

Every computation is a libss kernel; this module sequences the calls and owns the buffers.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import torch

from . import dist
from ._abi import SsAdamConfig, check, lib
from .raster import DeviceScene, FramePipeline, Rasterizer, _stream_handle, camera_struct, compact, prune_select


@dataclass
class AdamConfig:
    """3D-GS learning rates (mean scaled by the scene extent)."""
    lr_mean: float = 1.6e-4
    lr_opacity: float = 0.05
    lr_scale: float = 5e-3
    lr_rot: float = 1e-3
    lr_sh_dc: float = 2.5e-3
    lr_sh_rest: float = 2.5e-3 / 20
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15
    extent: float = 1.0

    def struct(self, step: int) -> SsAdamConfig:
        c = SsAdamConfig()
        c.lr_mean, c.lr_opacity, c.lr_scale = self.lr_mean * self.extent, self.lr_opacity, self.lr_scale
        c.lr_rot, c.lr_sh_dc, c.lr_sh_rest = self.lr_rot, self.lr_sh_dc, self.lr_sh_rest
        c.beta1, c.beta2, c.eps, c.step = self.beta1, self.beta2, self.eps, int(step)
        return c


def scaled_schedule(total_iters: int, soft_ratio: float = 0.8, hard_ratio: float = 0.3, paper_iters: int = 30000,
                    soft_at=(6000, 9000, 12000), hard_from: int = 15000, hard_every: int = 3000,
                    soft_events: int = 1) -> dict[int, float]:
    """The paper's schedule (Soft at 6k/9k/12k, Hard every 3k from 15k of 30k)
    scaled to `total_iters`.  Without densification only `soft_events` soft events are kept
    (the first ones)."""
    f = total_iters / paper_iters
    ev = {}
    for it in soft_at[:soft_events]:
        if soft_ratio > 0:
            ev[max(1, int(round(it * f)))] = soft_ratio
    if hard_ratio > 0:
        for it in range(hard_from, paper_iters, hard_every):
            ev[max(1, int(round(it * f)))] = hard_ratio
    return dict(sorted(ev.items()))


class Trainer:
    """Scene + Adam state on the device; one Rasterizer workspace reused across views."""

    def __init__(self, scene: DeviceScene, cams, targets: list[torch.Tensor], bg=(0.0, 0.0, 0.0),
                 mode: str = "accutile", adam: AdamConfig | None = None, seed: int = 0,
                 check_overflow: bool = True, replica: bool = False):
        # Training is single-replica: every step updates this process's scene from one view,
        # with no gradient exchange.  Under a process group of world size > 1 the scenes of the
        # ranks would drift apart (float atomics make each backward's summation order differ),
        # so an all-reduced score would mix different scenes.  replica=True states that this
        # rank trains an independent copy: it then scores all views itself, with no all_reduce.
        _, world, _ = dist.world()
        if world > 1 and not replica:
            raise ValueError("Trainer has no gradient exchange: under world size > 1 pass replica=True "
                             "(independent per-rank copies, no score all_reduce)")
        self.replica = bool(replica) or world == 1
        self.check_overflow = check_overflow   # False: capacity sized up front, no per-step read-back
        self.cams = list(cams)
        self.targets = targets
        self.bg = tuple(float(b) for b in bg)
        self.mode = mode
        self.adam = adam or AdamConfig()
        self.W, self.H = int(self.cams[0].width), int(self.cams[0].height)
        self.cstructs = [camera_struct(c) for c in self.cams]
        self.it = 0
        self.events = None     # optional (start, end) CUDA events around the Adam step (bench)
        self.gen = torch.Generator().manual_seed(seed)
        self._set_scene(scene, init_state=True)
        self.loss_sum = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.dimg = torch.empty((3, self.H, self.W), dtype=torch.float32, device=self.dev)

    # ------------------------------------------------------------------ state
    def _set_scene(self, scene: DeviceScene, init_state: bool, raw=None, m=None, v=None):
        self.scene = scene
        self.dev = scene.mean_opac.device
        cap = max(1024, 8 * scene.n)
        self.rz = Rasterizer(scene, self.W, self.H, mode=self.mode, capacity=cap)
        for c in (self.cams if not getattr(self, "check_overflow", True) else self.cams[: min(4, len(self.cams))]):
            self.rz.ensure_capacity(c, headroom=1.5)
        self.grads = scene.zeros_like()
        self.grad2d = torch.zeros((scene.n, 12), dtype=torch.float32, device=self.dev)
        self.flags = torch.zeros(max(scene.n, 1), dtype=torch.uint8, device=self.dev)
        if init_state:
            self.raw, self.m, self.v = scene.zeros_like(), scene.zeros_like(), scene.zeros_like()
            s = scene.struct()
            check(lib().ss_adam_init(C.byref(s), C.byref(self.raw.struct()), C.byref(self.m.struct()),
                                     C.byref(self.v.struct()), C.c_void_p(_stream_handle(None))), "ss_adam_init")
        else:
            self.raw, self.m, self.v = raw, m, v

    @property
    def n(self) -> int:
        return self.scene.n

    # ------------------------------------------------------------------ one iteration
    def step(self, view: int | None = None) -> None:
        """Render one view, L1 gradient, backward, Adam.  The loss stays on the device
        (self.loss_sum accumulates sum |I - I_gt|; read it with take_loss())."""
        if view is None:
            view = int(torch.randint(len(self.cams), (1,), generator=self.gen))
        self.it += 1
        cam = self.cstructs[view]
        img, T, nc = self.rz.render_frame(cam, self.bg, want_T=True, want_ncontrib=True,
                                          check_overflow=self.check_overflow)
        check(lib().ss_l1_loss_grad(img.numel(), C.c_void_p(img.data_ptr()), C.c_void_p(self.targets[view].data_ptr()),
                                    C.c_void_p(self.dimg.data_ptr()), C.c_void_p(self.loss_sum.data_ptr()),
                                    C.c_void_p(_stream_handle(None))), "ss_l1_loss_grad")
        self.grad2d.zero_()
        self.rz.render_backward(self.dimg, T, nc, grad2d=self.grad2d, bg=self.bg)
        # the gradients of this view's blended Gaussians are written (not accumulated) and
        # flagged; the others count as zero in Adam, so the gradient arrays are never zeroed
        self.flags.zero_()
        check(lib().ss_preprocess_backward_assign(C.byref(self.rz._scene_struct), C.byref(cam),
                                                  C.c_void_p(self.grad2d.data_ptr()), C.byref(self.grads.struct()),
                                                  C.c_void_p(self.flags.data_ptr()),
                                                  C.c_void_p(_stream_handle(None))), "ss_preprocess_backward_assign")
        if self.events is not None:
            self.events[0].record()
        cfg = self.adam.struct(self.it)
        sc = self.scene
        out = DeviceScene(sc.mean_opac, sc.scale, sc.rot, sc.sh, sc.sh_degree)
        check(lib().ss_adam_step_flagged(C.byref(self.grads.struct()), C.byref(self.raw.struct()),
                                         C.byref(self.m.struct()), C.byref(self.v.struct()), C.byref(out.struct()),
                                         C.byref(cfg), C.c_void_p(self.flags.data_ptr()),
                                         C.c_void_p(_stream_handle(None))), "ss_adam_step_flagged")
        if self.events is not None:
            self.events[1].record()
        self.n_loss_values = img.numel()

    def take_loss(self) -> float:
        """Mean L1 of the iterations since the last call (synchronises)."""
        v = float(self.loss_sum.item())
        self.loss_sum.zero_()
        return v

    # ------------------------------------------------------------------ pruning
    def score(self, n_streams: int = 3) -> torch.Tensor:
        """Ũ over every training view: this rank's shard of the views with several frames in
        flight (FramePipeline.score_views), then the float64 all_reduce."""
        rank, world, _ = dist.world()
        mine = list(range(len(self.cams))) if self.replica else dist.views_for_rank(len(self.cams), rank, world)
        score = torch.zeros(self.n, dtype=torch.float64, device=self.dev)
        if mine:
            pipe = FramePipeline(self.scene, self.W, self.H, mode=self.mode, n_streams=n_streams)
            pipe.ensure_capacity([self.cams[v] for v in mine], headroom=1.05)
            pipe.score_views([self.cstructs[v] for v in mine], score, self.bg)
            pipe.check_overflow()
        return score if self.replica else dist.allreduce_scores(score)

    def prune(self, ratio: float, score: torch.Tensor | None = None) -> int:
        """Remove ⌊ratio·N⌋ lowest-Ũ Gaussians with their Adam state; returns the removed count."""
        if score is None:
            score = self.score()
        keep, k = prune_select(score, ratio)
        self.prune_mask(keep, self.n - k)
        return k

    def prune_mask(self, keep: torch.Tensor, n_keep: int) -> None:
        if n_keep <= 0:
            raise ValueError("pruning would empty the scene")
        sc = compact(self.scene, keep, n_keep)
        raw, m, v = (compact(x, keep, n_keep) for x in (self.raw, self.m, self.v))
        self._set_scene(sc, init_state=False, raw=raw, m=m, v=v)

    # ------------------------------------------------------------------ evaluation
    def render_view(self, v: int) -> torch.Tensor:
        return self.rz.render_frame(self.cstructs[v], self.bg).clone()

    def psnr(self, views=None) -> float:
        """Mean PSNR (images in [0, 1] clamped) over `views` against the targets (reporting)."""
        views = range(len(self.cams)) if views is None else views
        ps = []
        for v in views:
            img = self.render_view(v).clamp(0, 1)
            mse = float(((img - self.targets[v].clamp(0, 1)) ** 2).mean())
            ps.append(10 * math.log10(1.0 / max(mse, 1e-12)))
        return sum(ps) / len(ps)

    def fit(self, iters: int, schedule: dict[int, float] | None = None, log_every: int = 0):
        """`iters` iterations; schedule {iteration: prune ratio}.  Returns the history."""
        schedule = schedule or {}
        hist = {"loss": [], "n": [], "events": []}
        acc, cnt = 0.0, 0
        for _ in range(iters):
            self.step()
            if log_every and self.it % log_every == 0:
                hist["loss"].append((self.it, self.take_loss() / (log_every * self.n_loss_values)))
                hist["n"].append((self.it, self.n))
            if self.it in schedule:
                k = self.prune(schedule[self.it])
                hist["events"].append((self.it, schedule[self.it], k, self.n))
        return hist


def render_targets(scene: DeviceScene, cams, bg=(0.0, 0.0, 0.0), mode: str = "accutile") -> list[torch.Tensor]:
    """Synthetic targets: the ground-truth scene rendered by the forward path."""
    rz = Rasterizer(scene, cams[0].width, cams[0].height, mode=mode)
    out = []
    for c in cams:
        rz.ensure_capacity(c)
        out.append(rz.render_frame(c, bg).clone())
    return out
