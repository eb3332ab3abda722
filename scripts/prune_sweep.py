"""Soft x Hard pruning sweep on a synthetic scene (the structure of the paper's
Fig. 4 sweep, "We sweep pruning percentages in 5% increments"), through
train.Trainer: every cell fits a perturbed copy of a ground-truth scene to its renders with the
scaled schedule (one Soft event at 6k/30k of the run, Hard events every 3k from 15k), then
reports the final count, the reduction factor and the PSNR against the targets.

    python scripts/prune_sweep.py [--iters 600] [--out profiles/r01_prune_sweep.csv]
CSV columns: soft_ratio,hard_ratio,final_count,reduction_factor,psnr_db,wall_ms
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2412_00578_b200 import synth  # noqa: E402
from paper_2412_00578_b200.raster import DeviceScene  # noqa: E402
from paper_2412_00578_b200.train import AdamConfig, Trainer, render_targets, scaled_schedule  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=600)
    ap.add_argument("--n", type=int, default=60000)
    ap.add_argument("--views", type=int, default=16)
    ap.add_argument("--soft", default="0,0.5,0.8,0.9")
    ap.add_argument("--hard", default="0,0.3,0.5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_prune_sweep.csv"))
    args = ap.parse_args()
    gt = synth.orbit_scene(args.n, 5)
    cams = synth.orbit_cameras(args.views, 256, 176)
    targets = render_targets(DeviceScene.from_host(gt), cams)
    init = synth.perturb(gt, seed=1)
    rows = ["soft_ratio,hard_ratio,final_count,reduction_factor,psnr_db,wall_ms"]
    for s in [float(x) for x in args.soft.split(",")]:
        for h in [float(x) for x in args.hard.split(",")]:
            sched = scaled_schedule(args.iters, soft_ratio=s, hard_ratio=h)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tr = Trainer(DeviceScene.from_host(init), cams, targets, adam=AdamConfig(extent=4.0), seed=0)
            tr.fit(args.iters, sched)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3
            ps = tr.psnr()
            rows.append(f"{s},{h},{tr.n},{gt.n / tr.n:.3f},{ps:.3f},{ms:.1f}")
            print(rows[-1], flush=True)
    with open(args.out, "w") as f:
        f.write("\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
