"""CPU: the C ABI library loads and exports its header, struct layouts agree,
host-side logic (filters, sharding, packing, scenes) behaves like the reference."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2604_07980_b200 import _abi, engine, ranger as rg, shard, synth as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ranger_cuda.h")


def header_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:rg_status|void|const char\*)\s+(rg_[a-z0-9_]+)\(", txt, re.M)))


def test_library_loads_and_exports_every_header_symbol():
    lib = rg.lib()  # loads without a GPU
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_abi.SIGNATURES), set(names) ^ set(_abi.SIGNATURES)
    assert lib.rg_build_info().decode().startswith("sm_100a")


def test_sm100a_only_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", rg.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_\d+a?", out.stdout))
    assert archs == {"sm_100a"}, archs


def test_struct_layouts_match_the_c_header():
    src = "#include <stdio.h>\n#include <stddef.h>\n#include \"ranger_cuda.h\"\nint main(){\n"
    structs = {"rg_rect": _abi.Rect, "rg_search_range": _abi.SearchRange, "rg_match_result": _abi.MatchResult,
               "rg_detection": _abi.Detection, "rg_ranger_config": _abi.RangerConfig,
               "rg_object_disparity": _abi.ObjectDisparity, "rg_ranger_stats": _abi.RangerStats,
               "rg_census_cache": _abi.CensusCache, "rg_bm_params": _abi.BmParams,
               "rg_frame_batch": _abi.FrameBatch, "rg_rect_search_config": _abi.RectSearchConfig,
               "rg_rect_state": _abi.RectState, "rg_sgm_params": _abi.SgmParams, "rg_box_stats": _abi.BoxStats, "rg_scene_object": _abi.SceneObject,
               "rg_scene_config": _abi.SceneConfig, "rg_calibration": _abi.Calibration, "rg_vec3": _abi.Vec3,
               "rg_obj_refiner_state": _abi.ObjRefinerState, "rg_class_width": _abi.ClassWidth,
               "rg_record_params": _abi.RecordParams, "rg_depth_record": _abi.DepthRecord,
               "rg_refiner_log": _abi.RefinerLog}
    for cname, py in structs.items():
        for f, _ in py._fields_:
            src += f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));\n'
        src += f'printf("{cname} %zu\\n", sizeof({cname}));\n'
    src += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "l")
        r = subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], capture_output=True)
        if r.returncode != 0:
            pytest.skip("gcc unavailable")
        got = dict(line.rsplit(" ", 1) for line in subprocess.check_output([exe], text=True).splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)


def test_compute_without_gpu_fails_loudly():
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        rg.Context(0)


def test_filter_offset_matches_reference_cases():  # test_autorect.cpp:52-79
    st = rg.RectOffsetState(5, 100)
    rg.filter_offset(st, 1)
    assert [rg.filter_offset(st, v) for v in (5, 9, 2, 8)] == [1.0, 5.0, 2.0, 5.0]
    st = rg.RectOffsetState(5, 1)
    for _ in range(5):
        rg.filter_offset(st, 2)
    assert st.current == 2.0 and rg.filter_offset(st, 9) == 2.0
    st = rg.RectOffsetState(3, 100)
    for v in (1, 2, 3):
        rg.filter_offset(st, v)
    assert rg.filter_offset(st, 4) == 3.0 and rg.filter_offset(st, 5) == 4.0
    st = rg.RectOffsetState(1, 1)
    assert [rg.filter_offset(st, v) for v in (3, 3, 3, 3, -3)] == [1.0, 2.0, 3.0, 3.0, 2.0]
    with pytest.raises(rg.InvalidArgument):
        rg.RectOffsetState(0, 1)


def test_rect_shift_schedule():
    # shift applied to frame t is lround(filter state before frame t)
    assert shard.rect_shift_schedule([3, 3, 3, 3], window=1, rate=1) == [0, 1, 2, 3]
    assert shard.rect_shift_schedule([-2, -2, -2], window=1, rate=1) == [0, -1, -2]


@pytest.mark.parametrize("n,world", [(1, 1), (7, 2), (4096, 8), (5, 8), (256, 3)])
def test_shard_bounds_partition(n, world):
    seen = []
    for r in range(world):
        lo, hi = shard.shard_bounds(n, r, world)
        seen.extend(range(lo, hi))
        assert all(shard.owner_of(f, n, world) == r for f in range(lo, hi))
    assert seen == list(range(n))


@pytest.mark.parametrize("n,world", [(1, 1), (7, 2), (4096, 8), (5, 8), (256, 3), (37, 4), (0, 3)])
def test_c_abi_shard_bounds_equal_python(n, world):
    """rg_shard_bounds (the library's multi-GPU split, csrc/multi.cu) is the
    same contiguous partition as shard.shard_bounds."""
    import ctypes as C
    for r in range(world):
        lo, hi = C.c_int(), C.c_int()
        assert rg.lib().rg_shard_bounds(n, r, world, C.byref(lo), C.byref(hi)) == 0
        assert (lo.value, hi.value) == shard.shard_bounds(n, r, world)
    assert rg.lib().rg_shard_bounds(n, world, world, C.byref(C.c_int()), C.byref(C.c_int())) != 0


def test_pack_detections_roundtrip():
    sc, cfg = S.scene_c1()
    dets = S.ground_truth_detections(sc)
    recs, offs = engine.pack_detections([dets, dets[:3], []])
    assert list(offs) == [0, 8, 11, 11]
    assert recs["id"].tolist() == [d.id for d in dets] + [d.id for d in dets[:3]]
    assert recs.dtype.itemsize == C.sizeof(_abi.Detection)


def test_scene_configs_shapes():
    for fn, n, far in [(S.scene_c1, 8, 5), (S.scene_c2, 64, 48), (S.scene_c3, 256, 192)]:
        sc, cfg = fn()
        dets = S.ground_truth_detections(sc)
        assert len(dets) == n
        kinds = [rg.classify_far_close(d, sc.width, sc.height, cfg.tau_s) for d in dets]
        assert kinds.count(rg.KIND_FAR) == far


def test_vote_state_init_validates_like_the_reference():  # radar_refiner.hpp:37-43
    v = rg.VoteState(4, 0.3, 1.0)
    assert v.to_c().n_bins == 129 and v.smoothed_offset == 0.0 and not v.memory.any()
    for bad in ((0, 0.3, 1.0), (4, 0.0, 1.0), (4, 1.5, 1.0), (33, 0.3, 1.0)):
        with pytest.raises(rg.InvalidArgument):
            rg.VoteState(*bad)


def test_radar_vote_update_host_half():
    """rg_radar_vote_update: one vote at offset +1 px -> the EMA moves toward
    +1 (radar_refiner.hpp:129-155); no votes leave the state untouched."""
    import ctypes as C
    v = rg.VoteState()
    a, off = C.c_double(), C.c_int()
    best = (C.c_double * 1)(1.0)
    found = (C.c_int32 * 1)(1)
    assert rg.lib().rg_radar_vote_update(C.byref(v.to_c()), best, found, 1, C.byref(a), C.byref(off)) == 0
    assert a.value == 0.3 * 1.0 and off.value == round(0.3 * 16)
    before = v.smoothed_offset
    found[0] = 0
    assert rg.lib().rg_radar_vote_update(C.byref(v.to_c()), best, found, 1, C.byref(a), C.byref(off)) == 0
    assert v.smoothed_offset == before
