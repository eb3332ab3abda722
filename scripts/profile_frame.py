"""One frame of the bench workload between cudaProfilerStart/Stop, for ncu captures:

    ncu --profile-from-start off --set full ... python scripts/profile_frame.py [--workload W]
        [--mode M] [--view V] [--score] [--prune-ratio R]

The scene and workspace are set up and one warm-up frame is rendered outside the profiled
range; the profiled range is one frame (a1-a6 through ss_render_frame, as the bench's timed
path enqueues it), plus ss_prune_score with --score."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2412_00578_b200 import synth  # noqa: E402
from paper_2412_00578_b200.raster import DeviceScene, FramePipeline, prune  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="mnr360-3m")
    ap.add_argument("--mode", default="accutile")
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--score", action="store_true")
    ap.add_argument("--prune-ratio", type=float, default=0.0)
    a = ap.parse_args()
    scene, cams = synth.make_workload(a.workload)
    ds = DeviceScene.from_host(scene)
    W, H = cams[0].width, cams[0].height
    if a.prune_ratio > 0:
        pipe = FramePipeline(ds, W, H, mode=a.mode, n_streams=4)
        pipe.ensure_capacity(cams[:8])
        score = torch.zeros(ds.n, dtype=torch.float64, device="cuda")
        pipe.score_views(cams, score)
        ds, _ = prune(ds, score, a.prune_ratio)
        del pipe
    pipe = FramePipeline(ds, W, H, mode=a.mode, n_streams=1)
    cam = cams[a.view]
    pipe.ensure_capacity([cam])
    pipe.render_views([cam])
    s = torch.zeros(ds.n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    pipe.render_views([cam])
    if a.score:
        pipe.rz[0].prune_score(s)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled one frame", pipe.rz[0].totals())


if __name__ == "__main__":
    main()
