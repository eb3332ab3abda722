"""Multi-process (world_size 2, gloo on CPU) coverage of the view-parallel path
(DESIGN.md §6): round-robin view sharding and the single all_reduce of the float64
pruning-score vector.  The per-view score here comes from the CPU oracle so the test
runs without a GPU; on the B200 box the same dist.accumulate_scores drives libss."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from paper_2412_00578_b200 import dist, synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    scene, _ = synth.make_workload("mnr360-3m", n=400)
    cams = synth.orbit_cameras(7, 96, 64)
    return scene, cams


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init(backend="gloo")
    scene, cams = _scene()

    def score_view(v, score):
        s = oracle.score_views(scene, [cams[v]])
        score += torch.from_numpy(s)

    total = dist.accumulate_scores(score_view, len(cams), scene.n, "cpu")
    out[rank] = total.numpy().copy()
    assert dist.max_over_ranks(float(rank)) == world - 1
    torch.distributed.destroy_process_group()


def test_views_partition():
    for n_views in (1, 7, 185, 251):
        for world in (1, 2, 4, 8):
            shards = [dist.views_for_rank(n_views, r, world) for r in range(world)]
            flat = sorted(v for s in shards for v in s)
            assert flat == list(range(n_views))
            assert max(map(len, shards)) - min(map(len, shards)) <= 1


def test_score_allreduce_world2_matches_single_process():
    scene, cams = _scene()
    ref = oracle.score_views(scene, cams)
    assert ref.max() > 0
    with mp.Manager() as m:
        out = m.dict()
        port = _free_port()
        mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="fork")
        r0, r1 = out[0], out[1]
    assert np.array_equal(r0, r1), "every rank must hold the identical reduced vector"
    assert np.allclose(r0, ref, rtol=1e-12, atol=0)


def test_trainer_refuses_unsynchronised_multi_rank(monkeypatch):
    """Training has no gradient exchange: under world size > 1 a Trainer must be an explicit
    independent replica, or its all-reduced scores would mix drifted scenes."""
    from paper_2412_00578_b200.train import Trainer
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    with pytest.raises(ValueError, match="replica"):
        Trainer(None, [], [])
