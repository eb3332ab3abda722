"""Two ranks on cuda:0 under a gloo process group, scoring with libss.

The view-parallel score pass as bench.py and Trainer.score run it at world size > 1: each
rank scores its round-robin shard of the views through FramePipeline.score_views (ss_prune_score,
frames in flight), then dist.allreduce_scores sums the float64 vectors.  Both ranks must end with
the identical vector, equal to the single-process score over all views (float64 atomics add in a
different order, so within 1e-9 relative), and the shards' rendered images must equal the
single-process images bitwise (views never communicate).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N, W, H, VIEWS = 30000, 320, 208, 7
BG = (0.2, 0.1, 0.3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_2412_00578_b200 import synth
    from paper_2412_00578_b200.raster import DeviceScene, FramePipeline
    scene, _ = synth.make_workload("mnr360-3m", n=N)
    cams = synth.orbit_cameras(VIEWS, W, H)
    ds = DeviceScene.from_host(scene, "cuda:0")
    pipe = FramePipeline(ds, W, H, n_streams=2)
    pipe.ensure_capacity(cams)
    return ds, cams, pipe


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    from paper_2412_00578_b200 import dist
    dist.init(backend="gloo")
    torch.cuda.set_device(0)
    ds, cams, pipe = _setup()
    mine = dist.views_for_rank(len(cams), rank, world)
    score = torch.zeros(ds.n, dtype=torch.float64, device="cuda:0")
    pipe.score_views([cams[v] for v in mine], score, BG)
    torch.cuda.synchronize()
    pipe.check_overflow()
    dist.allreduce_scores(score)
    imgs = {}
    for v in mine:
        pipe.render_views([cams[v]], BG)
        torch.cuda.synchronize()
        imgs[v] = pipe.outs[0].cpu().numpy()
    np.save(os.path.join(outdir, f"score{rank}.npy"), score.cpu().numpy())
    np.savez(os.path.join(outdir, f"img{rank}.npz"), **{str(k): v for k, v in imgs.items()})
    torch.distributed.destroy_process_group()


def test_two_ranks_one_gpu_gloo(tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    s0, s1 = (np.load(tmp_path / f"score{r}.npy") for r in (0, 1))
    assert np.array_equal(s0, s1), "every rank must hold the identical reduced vector"
    ds, cams, pipe = _setup()
    ref = torch.zeros(ds.n, dtype=torch.float64, device="cuda:0")
    pipe.score_views(cams, ref, BG)
    torch.cuda.synchronize()
    ref = ref.cpu().numpy()
    assert (ref > 0).sum() > 1000
    rel = np.abs(s0 - ref) / np.maximum(ref, 1e-12 * ref.max())
    assert rel.max() <= 1e-9, rel.max()
    for r in (0, 1):
        got = np.load(tmp_path / f"img{r}.npz")
        for k in got.files:
            pipe.render_views([cams[int(k)]], BG)
            torch.cuda.synchronize()
            assert np.array_equal(got[k], pipe.outs[0].cpu().numpy()), f"view {k} differs on rank {r}"


def _nccl_worker(rank, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    import torch.distributed as tdist
    from paper_2412_00578_b200 import dist
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    assert dist.backend() == "nccl"
    ds, cams, pipe = _setup()
    score = torch.zeros(ds.n, dtype=torch.float64, device="cuda:0")
    pipe.score_views(cams, score, BG)
    torch.cuda.synchronize()
    before = score.clone()
    dist.allreduce_scores(score)  # NCCL all_reduce(SUM) over the one rank, on the GPU tensor
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, "before.npy"), before.cpu().numpy())
    np.save(os.path.join(outdir, "after.npy"), score.cpu().numpy())
    tdist.destroy_process_group()


def test_nccl_allreduce_one_rank(tmp_path):
    """The score all_reduce through NCCL (the backend bench.py uses when every rank has its own
    GPU), on the one GPU these boxes have: world size 1, the libss score vector reduced in place
    on cuda:0; a one-rank SUM must return the vector unchanged."""
    import torch.multiprocessing as mp
    mp.start_processes(_nccl_worker, args=(_free_port(), str(tmp_path)), nprocs=1, join=True, start_method="spawn")
    before, after = np.load(tmp_path / "before.npy"), np.load(tmp_path / "after.npy")
    assert (before > 0).sum() > 1000
    assert np.array_equal(before, after)
