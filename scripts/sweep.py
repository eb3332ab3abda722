"""Frames/s and pairs/frame of every BASELINE.json configuration and tile test (GPU, 1 rank).

    python scripts/sweep.py [--steps 5] [--views 64] [--streams 8] > profiles/r02/r02_sweep.jsonl

One JSON line per (workload, mode): the forward path a1-a6 through the public API, V views
per step with 8 frames in flight (FramePipeline, one CUDA graph per frame as in bench.py), K
timed steps (CUDA events, L2 flushed between steps, 2 warm-up steps), the single-stream per-stage split, plus the
pruned-model regime (BASELINE config 5: U~ over every view, then the prune step removing 90%
of the Gaussians, AccuTile).  The speed-ups of SnugBox and AccuTile over the 3-sigma baseline
are the quantities the paper reports as 1.82x / 1.99x on an RTX A5000.
"""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_00578_b200 import synth  # noqa: E402
from paper_2412_00578_b200.raster import DeviceScene, FramePipeline, Rasterizer, camera_struct, prune  # noqa: E402


def measure(ds, cams, mode, steps, views, streams=8):
    W, H = cams[0].width, cams[0].height
    rz = Rasterizer(ds, W, H, mode=mode, capacity=max(1024, 4 * ds.n))
    vs = list(range(0, len(cams), max(1, len(cams) // views)))[:views]
    pairs = []
    for v in vs:
        rz.ensure_capacity(cams[v])
    for v in vs:
        rz.prepare(cams[v])
        pairs.append(rz.totals()["pairs"])
    rz._alloc(int(max(pairs) * 1.02) + 4096)
    cs = [camera_struct(cams[v]) for v in vs]
    out = torch.empty((3, H, W), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    pipe = FramePipeline(ds, W, H, mode=mode, n_streams=streams, capacity=rz.capacity)
    pipe.render_views(cs[:streams])
    pipe.capture(cs)
    ms = []
    for k in range(steps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        pipe.render_views(cs, graphs=True)
        b.record(st)
        torch.cuda.synchronize()
        if k >= 2:
            ms.append(a.elapsed_time(b))
    # per-stage split, single stream (events around each call)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in cs]
    flush.zero_()
    for c, e in zip(cs, ev):
        e[0].record(st)
        rz.preprocess(c)
        e[1].record(st)
        rz.bin(c)
        e[2].record(st)
        rz.sort()
        e[3].record(st)
        rz.render(out=out)
        e[4].record(st)
    torch.cuda.synchronize()
    stages = {s_: float(np.mean([e[i].elapsed_time(e[i + 1]) for e in ev]))
              for i, s_ in enumerate(["preprocess", "bin", "sort", "render"])}
    del rz, pipe
    return {"fps": len(cs) * len(ms) / (sum(ms) / 1e3), "pairs_per_frame": float(np.mean(pairs)),
            "views": len(cs), "steps": len(ms), "frames_in_flight": streams, "stages_ms_single_stream": stages}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--streams", type=int, default=16)
    args = ap.parse_args()
    for name in ["mnr360-3m", "truck", "garden", "playroom"]:
        scene, cams = synth.make_workload(name)
        ds = DeviceScene.from_host(scene)
        res = {}
        for mode in ["3sigma", "snugbox", "accutile"]:
            res[mode] = measure(ds, cams, mode, args.steps, args.views, args.streams)
            print(json.dumps({"workload": name, "n": scene.n, "mode": mode, **res[mode]}), flush=True)
        base = res["3sigma"]["fps"]
        print(json.dumps({"workload": name, "speedup_vs_3sigma": {m: res[m]["fps"] / base for m in res},
                          "pairs_ratio_3sigma_over": {m: res["3sigma"]["pairs_per_frame"] / res[m]["pairs_per_frame"]
                                                      for m in res}}), flush=True)
        if True:  # pruned-model regime (BASELINE config 5): score all views, drop 90%, AccuTile
            sp = FramePipeline(ds, cams[0].width, cams[0].height, mode="accutile", n_streams=args.streams)
            sp.ensure_capacity(cams)
            score = torch.zeros(scene.n, dtype=torch.float64, device="cuda")
            sp.score_views(cams, score)
            torch.cuda.synchronize()
            sp.check_overflow()
            del sp
            pds, _ = prune(ds, score, 0.9)
            r = measure(pds, cams, "accutile", args.steps, args.views, args.streams)
            print(json.dumps({"workload": name + "-pruned0.9", "n": pds.n, "mode": "accutile", **r,
                              "speedup_vs_unpruned_accutile": r["fps"] / res["accutile"]["fps"]}), flush=True)
        del ds
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
