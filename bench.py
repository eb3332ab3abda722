#!/usr/bin/env python
"""Benchmark of the Speedy-Splat forward hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload mnr360-3m] [--mode accutile] [--views-per-step V]

A STEP is one batch of V camera views per rank, each rendered through the whole forward
path a1-a6 (ss_preprocess -> ss_bin -> ss_sort -> ss_render) with the scene resident in
HBM; `value` = frames rendered by all ranks / max-over-ranks device time (sum of the K
steps' CUDA-event times).  The L2 is flushed between steps, outside the timed regions.  The pruning-score pass (a7 + the NCCL
all_reduce) is timed in the same run and reported in "prune_score".  Under torchrun every
rank renders its round-robin shard of the views (weak scaling: V views per rank per step).

--impl reference runs the CPU oracle (oracle/, plain C, the slow checker) on the host's
cores on the same workload: each step renders one full view per worker process.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP32_LANES_PER_SM = 128  # B200: 4 SMSPs x 32 FP32 lanes (FFMA = 2 flop)


METRIC = ("rendered frames/sec (forward a1-a6) & Gaussian-tile pairs/frame, "
          "3M-Gaussian MipNeRF360-shaped")


def base_config(args, n, W, H, sh_degree, views):
    """The config keys both arms report (the reference arm runs the same workload)."""
    return {"workload": args.workload, "n_gaussians": n, "width": W, "height": H, "views": views,
            "mode": args.mode, "sh_degree": sh_degree}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="mnr360-3m")
    ap.add_argument("--mode", default="accutile", choices=["3sigma", "snugbox", "accutile"])
    ap.add_argument("--views-per-step", type=int, default=64)
    ap.add_argument("--streams", type=int, default=16, help="concurrent frame workspaces (FramePipeline)")
    ap.add_argument("--prune-ratio", type=float, default=0.0,
                    help="pruned-model regime: score all views (a7 + all_reduce), prune this fraction, bench the rest")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="enqueue every frame's kernels instead of one CUDA graph")
    ap.add_argument("--no-pruned", action="store_true", help="skip the pruned-regime (config 5) measurement")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs (truck, garden, playroom)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-score", action="store_true")
    ap.add_argument("--no-backward", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--ncu", action="store_true", help="short run for profilers: no clocks/e2e/cpu legs")
    return ap.parse_args()


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(", ") for r in out.strip().splitlines() if r.count(",") >= 8]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------ oracle (CPU)
_POOL_SCENE = None


def _oracle_frame_worker(args):
    import oracle
    name, view, mode = args
    cams = _POOL_SCENE[1]
    t0 = time.perf_counter()
    f = oracle.frame(_POOL_SCENE[0], cams[view], mode, cap_hint=6 * _POOL_SCENE[0].n)
    return time.perf_counter() - t0, f.P


def oracle_pool(name, mode, workers):
    """Fork a pool of `workers` processes sharing the generated scene (copy-on-write)."""
    global _POOL_SCENE
    import multiprocessing as mp

    from paper_2412_00578_b200 import synth
    if _POOL_SCENE is None:
        _POOL_SCENE = synth.make_workload(name)
    import oracle
    oracle.build()
    ctx = mp.get_context("fork")
    return ctx.Pool(workers)


def run_oracle_steps(name, mode, steps, warmup, workers):
    """Each step: `workers` full oracle frames in parallel (one view per worker process)."""
    pool = oracle_pool(name, mode, workers)
    n_views = len(_POOL_SCENE[1])
    v = 0
    times = []
    pairs = []
    for k in range(warmup + steps):
        jobs = [(name, (v + j) % n_views, mode) for j in range(workers)]
        v += workers
        t0 = time.perf_counter()
        res = pool.map(_oracle_frame_worker, jobs)
        dt = time.perf_counter() - t0
        if k >= warmup:
            times.append(dt)
            pairs += [r[1] for r in res]
    pool.close()
    pool.join()
    total = sum(times)
    sc, cams = _POOL_SCENE
    return {"value": steps * workers / total, "ms_per_step": 1e3 * total / steps, "pairs": pairs,
            "frames": steps * workers, "n": sc.n, "W": cams[0].width, "H": cams[0].height,
            "sh_degree": sc.sh_degree, "views": len(cams)}


def cpu_model() -> str | None:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    workers = max(1, min(8, host_cores()))
    r = run_oracle_steps(args.workload, args.mode, args.steps, args.warmup, workers)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"],
        "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {**base_config(args, r["n"], r["W"], r["H"], r["sh_degree"], r["views"]),
                   "parallelism": "CPU oracle, one view per worker process"},
        "pairs_per_frame": statistics.mean(r["pairs"]) if r["pairs"] else None,
        "cpu_baseline": {"value": r["value"], "unit": "frames/s", "cores": workers, "kind": "oracle",
                         "sample": f"{r['frames']} full views of {args.workload} ({workers} worker processes, "
                                   f"one view each per step; oracle/ss_oracle.c -O2 -ffp-contract=off)"},
        "e2e": {"value": r["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ ours (GPU)
def stage_bytes(stage, N, n_vis, P, n_tiles, W, H, sh_floats, n_col=0):
    """Algorithmic bytes per launch: what the step must move at minimum."""
    if stage == "preprocess":   # mean + depth key of every Gaussian; scale, rot and record of the
        return 16 * N + 32 * n_vis + 48 * n_vis + 4 * N      # visible (colours deferred to the render)
    if stage == "bin":       # depth order (4 passes: key + value read and written), entry scan,
        # level 1 (order + emission record per visible Gaussian, entries written: E <= P / 2), level 2 count
        return 4 * N + 4 * 16 * n_vis + 8 * n_vis + (4 + 32) * n_vis + 8 * (P // 2) + 8 * n_tiles
    if stage == "sort":      # level 2 write: read the entries, one id per pair
        return 8 * (P // 2) + 4 * P
    if stage == "render":    # id + gathered record (36 B used) per pair, image, and the lazy colours:
        return 40 * P + 12 * W * H + n_col * (16 + 4 * sh_floats)   # mean + SH read, q2 written
    raise KeyError(stage)


def run_ours(args):
    import numpy as np
    import torch

    from paper_2412_00578_b200 import dist, synth
    from paper_2412_00578_b200._abi import SsCamera
    from paper_2412_00578_b200.raster import (DeviceScene, FramePipeline, Rasterizer, camera_struct, prune,
                                              render_views_to_host)

    rank, world, local = dist.init()
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; reporting the {world} ranks that ran",
              file=sys.stderr)
    dev_index = dist.local_device(local)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    ranks_per_gpu = -(-world // max(1, torch.cuda.device_count()))
    scene, cams = synth.make_workload(args.workload)
    W, H = cams[0].width, cams[0].height
    my_views = dist.views_for_rank(len(cams), rank, world)
    if args.ncu:
        my_views = my_views[:4]
    ds = DeviceScene.from_host(scene, dev)
    rz = Rasterizer(ds, W, H, mode=args.mode, capacity=max(1024, 4 * scene.n))
    prune_info = None
    if args.prune_ratio > 0:
        # pruned-model regime (BASELINE config 5): U~ over every view (sharded, all_reduce), then
        # the prune step; every rank derives the identical pruned scene
        def score_view(v, score):
            rz.ensure_capacity(cams[v])
            rz.prepare(cams[v])
            rz.prune_score(score)
        score = dist.accumulate_scores(score_view, len(cams), scene.n, dev, rank, world)
        ds, _ = prune(ds, score, args.prune_ratio)
        prune_info = {"ratio": args.prune_ratio, "n_before": scene.n, "n_after": ds.n}
        del rz, score
        rz = Rasterizer(ds, W, H, mode=args.mode, capacity=max(1024, 8 * ds.n))

    # sizing + per-view statistics (untimed): pairs per frame, visible counts, render work
    pairs, nvis, E_pix, E_blend, E_cta, ncol, dfr, phantom = {}, {}, {}, {}, {}, {}, {}, {}
    for v in my_views:
        rz.ensure_capacity(cams[v])
    cap = rz.capacity
    for v in my_views:
        rz.prepare(cams[v])
        rz.render()
        t = rz.totals()
        assert not t["overflow"]
        pairs[v], nvis[v], dfr[v] = t["pairs"], t["n_visible"], t["deferred"]
        ncol[v] = int(((rz.records()[:, 8] == 1.0) & (rz.depth_keys() != -1)).sum().item())
        # work counts (measurement helper, 2 ms per view; skipped under --ncu so that the launch
        # list holds the frame's kernels only)
        st = rz.render_stats() if not args.ncu else {"E_pix": 1, "E_blend": 1, "E_cta": 1, "phantom_pairs": 0}
        E_pix[v], E_blend[v], E_cta[v], phantom[v] = st["E_pix"], st["E_blend"], st["E_cta"], st["phantom_pairs"]
    # shrink capacity to the measured maximum (+2%) so the per-frame memset is tight
    rz._alloc(int(max(pairs.values()) * 1.02) + 4096)

    V = args.views_per_step
    seq = [my_views[j % len(my_views)] for j in range((args.warmup + args.steps) * V)]
    out = torch.empty((3, H, W), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    stages = ["preprocess", "bin", "sort", "render"]
    n_timed = args.steps * V
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(n_timed)]

    cstructs = {v: camera_struct(cams[v]) for v in my_views}   # host-side camera packing, once

    def frame(v, e=None, all_stages=False):
        # timed frames: events only around ss_preprocess (the dominant kernel's launch), so
        # that bin -> sort -> render keep their programmatic dependent launches; the other
        # stages are timed in a separate pass (all_stages) after the timed steps
        cam = cstructs[v]
        if e is not None:
            e[0].record(stream)
        rz.preprocess(cam)
        if e is not None:
            e[1].record(stream)
        rz.bin(cam)
        if e is not None and all_stages:
            e[2].record(stream)
        rz.sort()
        if e is not None and all_stages:
            e[3].record(stream)
        rz.render(out=out)
        if e is not None and all_stages:
            e[4].record(stream)

    pipe = FramePipeline(ds, W, H, mode=args.mode, n_streams=args.streams, capacity=rz.capacity)
    graphs = not args.no_graphs
    graph_info = None
    if graphs:
        # one CUDA graph per (view, workspace): the frame's ~20 launches become one graph launch
        pipe.render_views([cstructs[v] for v in my_views[:args.streams]])   # first-call setup outside capture
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        n_graphs = pipe.capture([cstructs[v] for v in my_views])
        graph_info = {"graphs": n_graphs, "capture_s": time.perf_counter() - g0,
                      "note": "per (view, workspace): ss_render_frame captured once, replayed every step"}
    for j in range(args.warmup):
        pipe.render_views([cstructs[v] for v in seq[j * V:(j + 1) * V]], graphs=graphs)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    if not args.ncu:
        clocks.start()
        time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    # K steps of V views each, timed by events on the caller's stream (the pipeline forks its
    # streams from it and joins them back); every frame's ss_preprocess is bracketed by events
    # on its own stream.  The L2 is flushed (256 MB written) between steps, outside the timed
    # regions, so no step starts with the previous step's data cached.
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    t_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    timed_views = seq[args.warmup * V:]
    h0 = time.perf_counter()
    for k in range(args.steps):
        flush.zero_()
        t_ev[k][0].record(stream)
        pipe.render_views([cstructs[v] for v in timed_views[k * V:(k + 1) * V]], graphs=graphs)
        t_ev[k][1].record(stream)
    host_ms = (time.perf_counter() - h0) * 1e3 / n_timed
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop() if not args.ncu else {}
    ms_total = sum(a.elapsed_time(b) for a, b in t_ev)
    ms_max = dist.max_over_ranks(ms_total)
    value = world * n_timed / (ms_max / 1e3)
    # the workspaces are sized tightly (max P + 2%): no timed frame may have overflowed (an
    # overflowed frame skips its binning and renders background only)
    n_overflow = pipe.overflow_count()
    assert n_overflow == 0, f"{n_overflow} timed frames overflowed the pair capacity"
    # k_preprocess launch durations with frames in flight, from an untimed pipelined pass of V
    # frames with events around every ss_preprocess (the timed steps enqueue each frame with one
    # ss_render_frame call); the per-stage split and the isolated k_preprocess duration come
    # from a separate single-stream pass of V frames
    flush.zero_()
    pipe.render_views([cstructs[v] for v in timed_views[:V]], pre_events=ev[:V])
    torch.cuda.synchronize()
    pre_ms = sum(ev[j][0].elapsed_time(ev[j][1]) for j in range(V)) / V
    ev2 = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(V)]
    flush.zero_()
    for j in range(V):
        frame(timed_views[j], ev2[j], all_stages=True)
    torch.cuda.synchronize()
    stage_ms = {s: sum(ev2[j][i].elapsed_time(ev2[j][i + 1]) for j in range(V)) / V
                for i, s in enumerate(stages)}
    frame_ms = sorted(ev2[j][0].elapsed_time(ev2[j][4]) for j in range(V))   # one frame alone on the GPU
    latency = {"mean_ms": float(np.mean(frame_ms)), "p50_ms": float(np.percentile(frame_ms, 50)),
               "p95_ms": float(np.percentile(frame_ms, 95)),
               "timing": "a1-a6 of one frame, CUDA events, single-stream pass of V frames (no other frame in flight)"}
    pre_iso_ms = stage_ms["preprocess"]

    # ---- per-stage roofline numbers (averages over the timed frames)
    mean = lambda d: float(np.mean([d[v] for v in timed_views]))
    Pm, NVm = mean(pairs), mean(nvis)
    sh_floats = {0: 4, 1: 12, 2: 28, 3: 48}[scene.sh_degree]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    stage_info = {}
    for s in stages:
        if s == "render":
            flops = 18.0 * mean(E_pix)   # ~18 FP32 ops per (pixel, Gaussian) evaluation
            ach = flops / (stage_ms[s] / 1e3) / 1e12
            stage_info[s] = {"ms": stage_ms[s], "bound": "alu", "achieved": ach, "peak": fp32_peak,
                             "unit": "TFLOP/s", "frac": ach / fp32_peak,
                             "gbs_algorithmic": stage_bytes(s, ds.n, NVm, Pm, rz.n_tiles, W, H, sh_floats, mean(ncol))
                             / (stage_ms[s] / 1e3) / 1e9}
        else:
            b = stage_bytes(s, ds.n, NVm, Pm, rz.n_tiles, W, H, sh_floats, mean(ncol))
            ach = b / (stage_ms[s] / 1e3) / 1e9
            stage_info[s] = {"ms": stage_ms[s], "bound": "hbm", "achieved": ach, "peak": hbm_peak,
                             "unit": "GB/s", "frac": ach / hbm_peak, "bytes": b}
    # The dominant KERNEL, by measured launch duration: ss_preprocess and ss_render are one
    # kernel each (k_preprocess after a 4 KB memset; k_render), ss_bin / ss_sort are chains of
    # short kernels.  Both single-kernel stages are reported under roofline["kernels"], timed by
    # CUDA events on the launching stream in the single-stream pass of the same run (a launch
    # has the GPU to itself there, so its share of the frame matches the ncu launch list); the
    # longer one is the line's roofline.  `traffic` = its DRAM bytes per launch from the
    # committed ncu --set full summary (profiles/traffic.json), when present.
    traffic, winst = {}, {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    tsrc = None
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        tsrc = tj.get("source")
        for k, v in tj.get("kernels", {}).items():
            # ss_preprocess = k_preprocess32 (+ k_preprocess64 over its deferred queue): summed
            for kn in ("k_preprocess", "k_render<"):
                if k.startswith(kn):
                    traffic[kn.rstrip("<")] = traffic.get(kn.rstrip("<"), 0.0) + v["dram_bytes"]
                    if v.get("warp_inst"):
                        winst[kn.rstrip("<")] = winst.get(kn.rstrip("<"), 0.0) + v["warp_inst"]
    pre = stage_info["preprocess"]
    kern = {
        "k_preprocess": {"bound": "hbm", "launch_ms": pre_iso_ms,
                         "launches": "k_preprocess32 (float32-certified tile geometry) + k_preprocess64 (the "
                                     "float64 path over the deferred queue, a few hundred Gaussians)", "achieved": pre["achieved"], "peak": hbm_peak,
                         "unit": "GB/s", "frac": pre["frac"], "algorithmic_bytes": pre["bytes"],
                         "traffic": traffic.get("k_preprocess"), "peak_source": hbm_src,
                         "unit_work": "16 B per Gaussian + 4 B depth key + per visible Gaussian 32 B scale/rot "
                                      "+ 48 B record (DESIGN.md §5)",
                         "in_flight": {"launch_ms": pre_ms, "achieved": pre["bytes"] / (pre_ms / 1e3) / 1e9,
                                       "frac": pre["bytes"] / (pre_ms / 1e3) / 1e9 / hbm_peak,
                                       "timing": f"pipelined pass of V frames, {args.streams} frames in flight"}},
    }
    r_ms = stage_ms["render"]
    r_flop = 18.0 * mean(E_pix)
    kern["k_render"] = {"bound": "alu", "launch_ms": r_ms, "achieved": r_flop / (r_ms / 1e3) / 1e12,
                        "peak": fp32_peak, "unit": "TFLOP/s", "frac": r_flop / (r_ms / 1e3) / 1e12 / fp32_peak,
                        "algorithmic_flop": r_flop, "traffic": traffic.get("k_render"),
                        "unit_work": "18 FP32 ops per (pixel, Gaussian) evaluation x E_pix (SURVEY §8(d)); "
                                     "E_pix from ss_render_stats",
                        "peak_source": f"derived: 148 SM x {FP32_LANES_PER_SM} FP32 lanes x 2 flop x {sm_max:.0f} MHz"}
    # The render's instruction-issue view: the FP32 roofline counts only the method's 18 flop
    # per evaluation, while the loop also issues its shared-memory loads, selects, the SFU
    # exponential and the termination test; the issue ceiling (4 warp instructions per SM per
    # cycle) bounds the kernel whatever the mix.  Warp instructions per launch from the same
    # committed capture as `traffic`, over the live launch time.
    if winst.get("k_render"):
        issue_peak = 148 * 4 * sm_max * 1e6
        kern["k_render"]["issue"] = {
            "warp_inst_per_launch": winst["k_render"], "achieved": winst["k_render"] / (r_ms / 1e3),
            "peak": issue_peak, "unit": "warp inst/s", "frac": winst["k_render"] / (r_ms / 1e3) / issue_peak,
            "peak_source": f"148 SM x 4 schedulers x 1 warp instruction per cycle x {sm_max:.0f} MHz",
            "source": tsrc}
    dom = max(kern, key=lambda k: kern[k]["launch_ms"])
    d = kern[dom]
    roof = {"bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"], "unit": d["unit"], "frac": d["frac"],
            "traffic": d["traffic"], "traffic_source": tsrc, "kernel": dom, "launch_ms": d["launch_ms"],
            "timing": "CUDA events on the launching stream, single-stream pass of V frames of the same workload in "
                      "the same run (L2 flushed before it); dominant = the longer single-kernel stage",
            "kernels": kern}

    # ---- pruning-score pass (a1-a5 + a7 over this rank's views, then the NCCL all_reduce)
    score_info = None
    if not args.no_score and not args.ncu:
        score = torch.zeros(ds.n, dtype=torch.float64, device=dev)
        n_sv = min(len(my_views), 2 * V)
        svs = [cstructs[v] if v in cstructs else camera_struct(cams[v]) for v in my_views[:n_sv]]
        pipe.score_views(svs[:4], score)
        score.zero_()
        dist.barrier()
        torch.cuda.synchronize()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        pipe.score_views(svs, score)       # a1-a5 + a7 per view, frames in flight
        b.record(stream)
        dist.allreduce_scores(score)       # no-op at world size 1
        c.record(stream)
        torch.cuda.synchronize()
        pipe.check_overflow()
        ms_s = dist.max_over_ranks(a.elapsed_time(c))
        if world > 1:
            ar = {"ms": dist.max_over_ranks(b.elapsed_time(c)), "bytes": 8 * ds.n, "backend": dist.backend(),
                  "op": "all_reduce(SUM) of the float64 score vector, once per scoring pass",
                  "timing": "CUDA events on the caller's stream around the collective, max over ranks"}
            if dist.backend() == "gloo":
                ar["note"] = f"{world} ranks share {torch.cuda.device_count()} GPU(s): gloo through host memory"
        else:
            ar = "skipped (world 1)"
        score_info = {"views_per_s": world * n_sv / (ms_s / 1e3), "views": world * n_sv,
                      "ms_score_views": dist.max_over_ranks(a.elapsed_time(b)), "allreduce": ar,
                      "dtype": "f64 accumulate, f32 per-pixel", "frames_in_flight": args.streams}

    # ---- backward pass (NEXT-2): forward with T / n_contrib, render backward, preprocess backward
    bw_info = None
    if not args.no_backward:
        n_bw = min(len(my_views), V if not args.ncu else 2)
        grad2d = torch.zeros((ds.n, 12), dtype=torch.float32, device=dev)
        grads = ds.zeros_like()
        dimg = torch.empty((3, H, W), dtype=torch.float32, device=dev).uniform_(-1.0, 1.0)
        bev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(n_bw)]

        def fwd_bwd(v, e=None):
            if e is not None:
                e[0].record(stream)
            rz.prepare(cstructs[v])
            _, T_, nc_ = rz.render(out=out, want_T=True, want_ncontrib=True)
            if e is not None:
                e[1].record(stream)
            grad2d.zero_()
            if e is not None:
                e[2].record(stream)
            rz.render_backward(dimg, T_, nc_, grad2d=grad2d)
            if e is not None:
                e[3].record(stream)
            rz.preprocess_backward(cstructs[v], grad2d, grads)
            if e is not None:
                e[4].record(stream)

        for v in my_views[:4]:
            fwd_bwd(v)
        dist.barrier()
        torch.cuda.synchronize()
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for j, v in enumerate(my_views[:n_bw]):
            fwd_bwd(v, bev[j])
        b.record(stream)
        torch.cuda.synchronize()
        ms_b = dist.max_over_ranks(a.elapsed_time(b))
        n_grad = int((grad2d != 0).any(dim=1).sum().item())   # Gaussians blended in the last view
        rb_ms = sum(e[2].elapsed_time(e[3]) for e in bev) / n_bw
        pb_ms = sum(e[3].elapsed_time(e[4]) for e in bev) / n_bw
        Pb = float(np.mean([pairs[v] for v in my_views[:n_bw]]))
        NVb = float(np.mean([nvis[v] for v in my_views[:n_bw]]))
        # algorithmic bytes: render backward reads id + record per pair, dL/dC + T + n_contrib per
        # pixel, and adds 36 B of gradient per (tile, Gaussian) pair; preprocess backward reads the
        # 48 B grad2d row of every Gaussian, and per Gaussian with a non-zero row (blended somewhere
        # in the view) its parameters (48 B + SH) and a read-modify-write of its gradients (48 B + SH)
        rb_bytes = 40 * Pb + 20 * W * H + 2 * 36 * Pb
        pb_bytes = 48 * ds.n + 3 * n_grad * (48 + 4 * sh_floats)
        bw_info = {"views_per_s": world * n_bw / (ms_b / 1e3), "views": world * n_bw, "blended_gaussians": n_grad,
                   "note": "per view: a1-a6 with T_final / n_contrib, grad2d zeroing, ss_render_backward, "
                           "ss_preprocess_backward (dL/dC uniform random, resident)",
                   "render_backward": {"ms": rb_ms, "bound": "hbm", "bytes": rb_bytes,
                                       "achieved": rb_bytes / (rb_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                                       "frac": rb_bytes / (rb_ms / 1e3) / 1e9 / hbm_peak},
                   "preprocess_backward": {"ms": pb_ms, "bound": "hbm", "bytes": pb_bytes,
                                           "achieved": pb_bytes / (pb_ms / 1e3) / 1e9, "peak": hbm_peak,
                                           "unit": "GB/s", "frac": pb_bytes / (pb_ms / 1e3) / 1e9 / hbm_peak}}
        del grad2d, grads

    # ---- training step (NEXT-3): a1-a6 + L1 + render backward + preprocess backward + Adam
    train_info = None
    if not args.no_train and not args.ncu and prune_info is None:
        from paper_2412_00578_b200.train import AdamConfig, Trainer
        n_tv = min(len(my_views), 8)
        tcams = [cams[v] for v in my_views[:n_tv]]
        targets = [torch.zeros((3, H, W), dtype=torch.float32, device=dev).uniform_(0, 1) for _ in tcams]
        tscene = DeviceScene(ds.mean_opac.clone(), ds.scale.clone(), ds.rot.clone(), ds.sh.clone(), ds.sh_degree)
        tr = Trainer(tscene, tcams, targets, adam=AdamConfig(extent=4.0), check_overflow=False, replica=True)
        for j in range(3):
            tr.step(j % n_tv)
        n_it = max(8, args.steps)
        aev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_it)]
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for j in range(n_it):
            tr.events = aev[j]
            tr.step(j % n_tv)
        b.record(stream)
        torch.cuda.synchronize()
        tr.events = None
        ms_t = dist.max_over_ranks(a.elapsed_time(b))
        adam_ms = sum(x.elapsed_time(y) for x, y in aev) / n_it
        # Adam (flagged): per Gaussian reads raw, m, v and writes raw, m, v, the activated array (7
        # passes over the scene's 240 B: mean_opac, scale, rot, 12 SH float4), plus the gradient of
        # the flagged (blended) Gaussians and one flag byte per Gaussian
        slot_bytes = 16 * (3 + {0: 1, 1: 3, 2: 7, 3: 12}[scene.sh_degree])
        n_flag = int(tr.flags.sum().item())
        adam_bytes = 7 * slot_bytes * ds.n + slot_bytes * n_flag + ds.n
        train_info = {"iters_per_s_per_replica": n_it / (ms_t / 1e3), "iters": n_it, "replicas": world,
                      "flagged": n_flag,
                      "note": "one view per iteration, single replica (ranks train independent copies, no gradient "
                              "exchange; the slowest rank's time): a1-a6 with T/n_contrib, ss_l1_loss_grad, "
                              "ss_render_backward, ss_preprocess_backward_assign (gradients written for the "
                              "blended Gaussians, flagged), ss_adam_step_flagged over all N Gaussians (dense "
                              "Adam, as 3D-GS; unflagged gradients are zero); targets uniform random; capacity "
                              "sized up front",
                      "adam": {"ms": adam_ms, "bound": "hbm", "bytes": adam_bytes,
                               "achieved": adam_bytes / (adam_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                               "frac": adam_bytes / (adam_ms / 1e3) / 1e9 / hbm_peak}}
        del tr, tscene, targets

    # ---- end to end through the public API: camera in, image out to pinned host memory
    e2e = None
    if not args.no_e2e and not args.ncu:
        n_e = min(len(my_views), V)
        host = [torch.empty((3, H, W), dtype=torch.float32).pin_memory() for _ in range(n_e)]
        vs = [cams[v] for v in my_views[:n_e]]
        render_views_to_host(pipe, vs, host, graphs=graphs)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = max(1, args.steps // 4)
        for _ in range(reps):
            render_views_to_host(pipe, vs, host, graphs=graphs)
        dt = dist.max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": world * reps * n_e / dt, "unit": "frames/s",
               "h2d_bytes_per_step": V * ctypes.sizeof(SsCamera), "d2h_bytes_per_step": V * 3 * H * W * 4,
               "note": "scene resident in HBM; per frame the camera (host struct) selects the frame's launch (" +
                       ("its pre-captured CUDA graph" if graphs else "kernel arguments") + ") and the float32 "
                       "image goes device->host into pinned memory, copied on the frame's own stream "
                       f"({args.streams} frames in flight: copies overlap the other streams' kernels)"}

    # ---- pruned-model regime (BASELINE config 5): U~ over every view (this rank's shard, then the
    # all_reduce), the prune step removing 90%, then the same timed loop on the pruned scene
    pruned_info = None
    if not args.no_pruned and not args.ncu and prune_info is None:
        ratio = 0.9
        t0 = time.perf_counter()
        score_all = torch.zeros(ds.n, dtype=torch.float64, device=dev)
        pipe.score_views([cstructs[v] for v in my_views], score_all)
        torch.cuda.synchronize()
        pipe.check_overflow()
        dist.allreduce_scores(score_all)
        pds, _ = prune(ds, score_all, ratio)
        del score_all
        ppipe = FramePipeline(pds, W, H, mode=args.mode, n_streams=args.streams)
        pP = ppipe.ensure_capacity([cstructs[v] for v in my_views], headroom=1.02)
        if graphs:
            ppipe.render_views([cstructs[v] for v in my_views[:args.streams]])
            ppipe.capture([cstructs[v] for v in my_views])
        setup_s = time.perf_counter() - t0
        for j in range(args.warmup):
            ppipe.render_views([cstructs[v] for v in seq[j * V:(j + 1) * V]], graphs=graphs)
        dist.barrier()
        torch.cuda.synchronize()
        pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for k in range(args.steps):
            flush.zero_()
            pev[k][0].record(stream)
            ppipe.render_views([cstructs[v] for v in timed_views[k * V:(k + 1) * V]], graphs=graphs)
            pev[k][1].record(stream)
        torch.cuda.synchronize()
        assert ppipe.overflow_count() == 0
        pms = dist.max_over_ranks(sum(a.elapsed_time(b) for a, b in pev))
        pval = world * n_timed / (pms / 1e3)
        pruned_info = {"value": pval, "unit": "frames/s", "ratio": ratio, "n_gaussians": pds.n,
                       "ms_per_frame": pms / n_timed, "max_pairs_per_frame": pP, "speedup_vs_unpruned": pval / value,
                       "setup_s": setup_s,
                       "note": "BASELINE config 5 on 1 scene: U~ over every view (sharded, all_reduce), prune step "
                               "(lowest 90% removed, ties by index), no fine-tuning; the same timed loop, L2 flushed "
                               "between steps"}
        del ppipe, pds

    # ---- the other BASELINE.json configs, same launch setup (view-sharded over the ranks, graphs,
    # frames in flight, L2 flushed between steps), fewer steps: truck-shaped in the three tile
    # modes (config 2), garden-shaped (config 3), playroom-shaped with the score pass and its
    # all_reduce over every view (config 4), and each scene pruned by 90% (config 5)
    configs_info = None
    if not args.no_configs and not args.ncu and prune_info is None:
        del pipe
        torch.cuda.empty_cache()
        configs_info = run_configs(args, rank, world, dev, stream, flush)

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.ncu:
        workers = max(1, min(8, host_cores()))
        r = run_oracle_steps(args.workload, args.mode, 1, 0, workers)
        r1 = run_oracle_steps(args.workload, args.mode, 1, 0, 1)
        cpu = {"value": r["value"], "unit": "frames/s", "cores": workers, "kind": "oracle",
               "sample": f"{r['frames']} full views of {args.workload} (project, bin, sort, render; one view per "
                         f"worker process)",
               "one_core": {"value": r1["value"], "unit": "frames/s", "cores": 1, "ms_per_frame": r1["ms_per_step"],
                            "sample": f"1 full view of {args.workload}, one process"},
               "cpu_model": cpu_model()}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload + (f"-pruned{args.prune_ratio:g}" if prune_info else ""),
                       "n_gaussians": ds.n, "pruned": prune_info, "width": W, "height": H,
                       "views": len(cams), "views_per_step_per_rank": V, "mode": args.mode,
                       "sh_degree": scene.sh_degree, "parallelism": f"view-parallel x{world}",
                       "process_group": dist.backend() or "none (1 rank)",
                       "gpus_visible": torch.cuda.device_count(), "ranks_per_gpu": ranks_per_gpu,
                       "frames_in_flight": args.streams,
                       "launch": "one CUDA graph per frame (captured per view and workspace)" if graphs
                                 else "one ss_render_frame call per frame",
                       "l2": "flushed between steps (256 MB written outside the timed regions); scene %.0f MB, "
                             "per-frame records %.0f MB" % (ds.n * 240 / 1e6, NVm * 48 / 1e6)},
            "pairs_per_frame": {"mean": Pm, "min": min(pairs.values()), "max": max(pairs.values())},
            "frame_latency": latency,
            "pairs_per_s": value * Pm,
            "visible_per_frame": NVm,
            "preprocess_float64_per_frame": {"mean": mean(dfr), "max": max(dfr[v] for v in timed_views),
                                             "note": "Gaussians whose float32 tile decisions could not be certified "
                                                     "(evaluated on the float64 path, k_preprocess64)"},
            "coloured_per_frame": mean(ncol),
            "stages_ms": {s: stage_ms[s] for s in stages},
            "host_enqueue_ms_per_frame": host_ms,
            "graphs": graph_info,
            "stages": stage_info,
            "render_work": {"E_pix": mean(E_pix), "E_blend": mean(E_blend), "E_cta": mean(E_cta),
                            "pixels": W * H},
            "phantom_tiles": {"per_frame": mean(phantom), "rate": mean(phantom) / Pm,
                              "note": "(tile, Gaussian) pairs whose Gaussian has alpha < 1/255 at every pixel centre "
                                      "of the tile (AccuTile tests the continuous cell, DESIGN.md R23)"},
            "stages_timing": "single-stream pass of V frames after the timed region (every stage bracketed by events)",
            "roofline": roof,
            # ours per frame (profiles/r02/r02_v10_launches.txt): k_preprocess32, k_preprocess64 (the
            # deferred queue), 4 x k_onesweep, k_escan_reduce, k_escan_apply, k_entries, k_big_entries,
            # k_l1_count, k_l1_scan, k_l1_emit, k_l2_count, k_l2_scan, k_l2_write, k_render
            "gpu_launches": n_timed * 17,
            "clocks": clk,
            "e2e": e2e,
            "prune_score": score_info,
            "backward": bw_info,
            "train": train_info,
            "pruned": pruned_info,
            "configs": configs_info,
            "cpu_baseline": cpu,
            "paper_context": {"gpu": "RTX A5000 (PAPER.md P:447)", "accutile_fps_avg_scene": 267,
                              "speedups": {"snugbox": 1.82, "accutile": 1.99, "overall": 6.71}},
        }
        print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(n: int) -> int:
    """`--gpus N` without a torchrun environment: launch N ranks of this command on this node
    (torch.distributed.run, rendezvous on 127.0.0.1), one process per GPU; rank 0 prints the
    line.  NCCL_DEBUG=INFO lets the NCCL communicator report its ranks on stderr."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_configs(args, rank, world, dev, stream, flush, V=64, steps=3, warmup=2):
    """Frames/s of the other BASELINE configs (see the caller)."""
    import torch

    from paper_2412_00578_b200 import dist, synth
    from paper_2412_00578_b200.raster import DeviceScene, FramePipeline, camera_struct, prune

    def fps(ds, cams, mode):
        W, H = cams[0].width, cams[0].height
        mine = dist.views_for_rank(len(cams), rank, world)
        cs = [camera_struct(cams[v]) for v in mine]
        pipe = FramePipeline(ds, W, H, mode=mode, n_streams=args.streams)
        P = pipe.ensure_capacity(cs)
        pipe.render_views(cs[:args.streams])
        pipe.capture(cs)
        seq = [cs[j % len(cs)] for j in range((warmup + steps) * V)]
        for j in range(warmup):
            pipe.render_views(seq[j * V:(j + 1) * V], graphs=True)
        dist.barrier()
        torch.cuda.synchronize()
        ms = 0.0
        for k in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            pipe.render_views(seq[(warmup + k) * V:(warmup + k + 1) * V], graphs=True)
            b.record(stream)
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
        assert pipe.overflow_count() == 0
        ms = dist.max_over_ranks(ms)
        return {"fps": world * steps * V / (ms / 1e3), "max_pairs_per_frame": P}, pipe, cs

    def score_all(ds, cams, pipe, cs, bg=(0.0, 0.0, 0.0)):
        score = torch.zeros(ds.n, dtype=torch.float64, device=dev)
        dist.barrier()
        torch.cuda.synchronize()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        pipe.score_views(cs, score, bg)
        b.record(stream)
        dist.allreduce_scores(score)
        c.record(stream)
        torch.cuda.synchronize()
        pipe.check_overflow()
        info = {"views": len(cams), "views_per_s": len(cams) / (dist.max_over_ranks(a.elapsed_time(b)) / 1e3),
                "allreduce": {"ms": dist.max_over_ranks(b.elapsed_time(c)), "bytes": 8 * ds.n,
                              "backend": dist.backend()} if world > 1 else "skipped (world 1)"}
        return score, info

    out = {}
    for name, modes in (("truck", ("3sigma", "snugbox", "accutile")), ("garden", ("snugbox", "accutile")),
                        ("playroom", ("accutile",))):
        scene, cams = synth.make_workload(name)
        ds = DeviceScene.from_host(scene, dev)
        res = {"n_gaussians": scene.n, "width": cams[0].width, "height": cams[0].height, "views": len(cams)}
        pipe = cs = None
        for mode in modes:
            del pipe
            r, pipe, cs = fps(ds, cams, mode)
            res[mode] = r
        if "3sigma" in res:
            res["speedup_vs_3sigma"] = {m: res[m]["fps"] / res["3sigma"]["fps"] for m in modes}
        # every view's U~ (this rank's shard, then the all_reduce), then the prune step (90%)
        score, sinfo = score_all(ds, cams, pipe, cs)
        if name == "playroom":
            res["score_pass"] = sinfo
        del pipe
        pds, _ = prune(ds, score, 0.9)
        del score
        r, pipe, _ = fps(pds, cams, "accutile")
        res["pruned0.9"] = {**r, "n_gaussians": pds.n, "speedup_vs_accutile": r["fps"] / res["accutile"]["fps"]}
        del pipe, pds, ds, scene
        torch.cuda.empty_cache()
        out[name] = res
    out["note"] = (f"{V} views per step, {steps} timed steps after {warmup}, {args.streams} frames in flight, one CUDA "
                   "graph per frame, L2 flushed between steps; pruned = U~ over every view (sharded, all_reduce), "
                   "then the prune step removing 90%")
    return out


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
