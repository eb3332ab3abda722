"""Pipelined cost of the stages: V frames on N streams (8 workspaces), timing a1 only, a1-a2
(ss_preprocess + ss_bin), a1-a5 (+ ss_sort) and a1-a6 (+ ss_render); each frame's launches are
captured in one CUDA graph per (view, workspace) for each prefix.  The differences are the
stages' shares of the pipelined frame time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2412_00578_b200 import synth  # noqa: E402
from paper_2412_00578_b200._abi import MODES, check, lib  # noqa: E402
from paper_2412_00578_b200.raster import DeviceScene, FramePipeline, camera_struct  # noqa: E402

scene, cams = synth.make_workload("mnr360-3m")
ds = DeviceScene.from_host(scene)
W, H = cams[0].width, cams[0].height
NS, V = 8, 64
if "--pruned" in sys.argv:  # BASELINE config 5: U~ over every view, 90% removed
    from paper_2412_00578_b200.raster import prune
    sp = FramePipeline(ds, W, H, n_streams=NS)
    sp.ensure_capacity(cams)
    sc = torch.zeros(ds.n, dtype=torch.float64, device="cuda")
    sp.score_views(cams, sc)
    ds, _ = prune(ds, sc, 0.9)
    del sp
pipe = FramePipeline(ds, W, H, n_streams=NS)
views = [camera_struct(cams[v]) for v in range(0, 185, 3)][:V]
pipe.ensure_capacity(views)
bgv = (C.c_float * 3)(0.0, 0.0, 0.0)
mode = MODES["accutile"]
L = lib()


def enqueue(stage, j, cam, st):
    rz = pipe.rz[j % NS]
    s = C.c_void_p(int(st.cuda_stream))
    check(L.ss_preprocess(C.byref(rz._scene_struct), C.byref(cam), mode, C.byref(rz.frame), s), "pre")
    if stage >= 2:
        check(L.ss_bin(C.byref(cam), mode, C.byref(rz.frame), s), "bin")
    if stage >= 3:
        check(L.ss_sort(C.byref(rz.frame), s), "sort")
    if stage >= 4:
        check(L.ss_render(C.byref(rz.frame), bgv, C.c_void_p(pipe.outs[j % NS].data_ptr()), None, None, s), "render")


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
if os.environ.get("SS_L2_PERSIST"):  # experiment: keep the scene's means (read by every frame) in L2
    from cuda.bindings import runtime as rt
    nbytes = int(ds.mean_opac.numel() * 4)
    frac = float(os.environ.get("SS_L2_PERSIST"))
    rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, nbytes)
    for st in pipe.streams:
        v = rt.cudaStreamAttrValue()
        w = v.accessPolicyWindow
        w.base_ptr = ds.mean_opac.data_ptr()
        w.num_bytes = nbytes
        w.hitRatio = frac
        w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
        w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
        v.accessPolicyWindow = w
        err = rt.cudaStreamSetAttribute(st.cuda_stream, rt.cudaStreamAttributeAccessPolicyWindow, v)
        print("policy", err, file=sys.stderr)
res = {}
for stage, name in ((1, "a1"), (2, "a1-a2"), (3, "a1-a5"), (4, "a1-a6")):
    graphs = {}
    for j, cam in enumerate(views):
        st = pipe.streams[j % NS]
        enqueue(stage, j, cam, st)   # first-call setup outside capture
    torch.cuda.synchronize()
    for j, cam in enumerate(views):
        st = pipe.streams[j % NS]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            g.capture_begin()
            enqueue(stage, j, cam, st)
            g.capture_end()
        graphs[j] = g
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    ms = []
    for rep in range(6):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for st in pipe.streams:
            st.wait_stream(cur)
        for j in range(len(views)):
            st = pipe.streams[j % NS]
            with torch.cuda.stream(st):
                graphs[j].replay()
        for st in pipe.streams:
            cur.wait_stream(st)
        b.record(cur)
        torch.cuda.synchronize()
        if rep >= 2:
            ms.append(a.elapsed_time(b))
    res[name] = sum(ms) / len(ms) / len(views)
    print(name, f"{res[name]:.4f} ms/frame pipelined", flush=True)
print({k: round(v, 4) for k, v in res.items()})
