"""C-ABI boundary checks that need no GPU: libss.so loads, exports every symbol that
include/ss.h declares, reports layouts and rejects invalid arguments before any launch."""
import ctypes as C
import os
import re

import pytest

from paper_2412_00578_b200 import _abi
from paper_2412_00578_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _abi.lib()


def test_exports_match_header(lib):
    hdr = open(os.path.join(ROOT, "include", "ss.h")).read()
    declared = set(re.findall(r"^\s*(?:SS_API\s+)?(?:const\s+)?[a-z_0-9]+\s*\*?\s*(ss_[a-z_0-9]+)\s*\(", hdr, re.M))
    assert declared == set(_abi.EXPORTS), declared ^ set(_abi.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.ss_version()


def test_layout_and_workspace(lib):
    L = _abi.layout(1000, 4096, 256, 256)
    assert (L.tiles_x, L.tiles_y, L.n_tiles, L.tile_bits) == (16, 16, 256, 8)
    assert L.total_bytes == _abi.workspace_size(1000, 4096, 256, 256)
    offs = sorted([L.rec, L.erec, L.depth_key, L.order, L.sorted_value,
                   L.ranges, L.tile_count, L.n_visible, L.total_pairs, L.overflow, L.overflow_count])
    assert len(set(offs)) == len(offs) and all(o % 256 == 0 for o in offs)
    L2 = _abi.layout(10, 100, 1297, 840)
    assert (L2.tiles_x, L2.tiles_y, L2.tile_bits) == (82, 53, 13)
    assert _abi.workspace_size(-1, 10, 10, 10) == 0
    # §8(b)'s ss_workspace_size(which, ...): the frame and prune-step workspaces
    b = C.c_size_t(0)
    assert lib.ss_workspace_size(0, 1000, 4096, 256, 256, C.byref(b)) == _abi.SS_OK
    assert b.value == L.total_bytes
    assert lib.ss_workspace_size(1, 1000, 0, 0, 0, C.byref(b)) == _abi.SS_OK
    assert b.value == lib.ss_prune_workspace_size(1000)
    assert lib.ss_workspace_size(2, 1000, 0, 0, 0, C.byref(b)) == _abi.SS_ERR_INVALID_ARG
    assert lib.ss_workspace_size(0, 1000, 0, 0, 16, C.byref(b)) == _abi.SS_ERR_INVALID_ARG
    assert lib.ss_workspace_size(0, -1, 0, 16, 16, C.byref(b)) == _abi.SS_ERR_INVALID_ARG


def test_invalid_arguments_rejected_before_launch(lib):
    st = _abi.SsCamera()
    fr = _abi.SsFrame(None, 0, 10, 100, 64, 64)
    sc = _abi.SsScene(10, 3, None, None, None, None)
    assert lib.ss_preprocess(C.byref(sc), C.byref(st), 2, C.byref(fr), None) == _abi.SS_ERR_INVALID_ARG
    fr.ws = 1234
    fr.ws_bytes = 10  # too small
    assert lib.ss_sort(C.byref(fr), None) == _abi.SS_ERR_INVALID_ARG
    fr.ws_bytes = _abi.workspace_size(10, 100, 64, 64)
    # camera size mismatch / bad sh degree / bad mode / null planes
    st.width, st.height, st.fx, st.fy = 32, 64, 100.0, 100.0
    assert lib.ss_preprocess(C.byref(sc), C.byref(st), 2, C.byref(fr), None) == _abi.SS_ERR_INVALID_ARG
    st.width = 64
    assert lib.ss_preprocess(C.byref(sc), C.byref(st), 2, C.byref(fr), None) == _abi.SS_ERR_INVALID_ARG  # null planes
    sc2 = _abi.SsScene(10, 4, 1, 1, 1, 1)
    assert lib.ss_preprocess(C.byref(sc2), C.byref(st), 2, C.byref(fr), None) == _abi.SS_ERR_INVALID_ARG
    sc3 = _abi.SsScene(10, 3, 1, 1, 1, 1)
    assert lib.ss_preprocess(C.byref(sc3), C.byref(st), 7, C.byref(fr), None) == _abi.SS_ERR_INVALID_ARG
    # camera values: z_near <= 0 or non-finite, negative / non-finite J clamp
    ok = _abi.SsCamera()
    ok.width, ok.height, ok.fx, ok.fy, ok.z_near, ok.clip = 64, 64, 100.0, 100.0, 0.2, 1.3
    for field, bad in (("z_near", 0.0), ("z_near", -0.2), ("z_near", float("nan")), ("clip", -1.0),
                       ("clip", float("inf")), ("fx", float("inf"))):
        c = _abi.SsCamera()
        C.memmove(C.byref(c), C.byref(ok), C.sizeof(c))
        setattr(c, field, bad)
        assert lib.ss_bin(C.byref(c), 2, C.byref(fr), None) == _abi.SS_ERR_INVALID_ARG, (field, bad)
        g = _abi.SsScene(10, 3, 1, 1, 1, 1)  # ss_scene_grad has ss_scene's layout
        assert lib.ss_preprocess_backward(C.byref(sc3), C.byref(c), 1, C.byref(g), None) == _abi.SS_ERR_INVALID_ARG
    big = _abi.SsFrame(1234, 1 << 40, 10, 100, 16 * 65537, 16)
    assert lib.ss_sort(C.byref(big), None) == _abi.SS_ERR_UNSUPPORTED  # > 256 tiles along x
    assert _abi.layout(10, 100, 4096, 4096).n_tiles == 65536  # the largest supported grid (no launch here)
    assert lib.ss_status_string(_abi.SS_ERR_CUDA) == b"SS_ERR_CUDA"


def test_product_package_never_imports_oracle():
    """The product path must not import, link or execute anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2412_00578_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), fn
                assert "liboracle" not in src and "ss_oracle" not in src, fn
