"""Per-frame records: the sequential tail of
Pipeline::process_frame (pipeline.hpp:180-265 minus the tracker) -- object
refiner (object_refiner.hpp), stereo / ground-point / size cues
(geometry.hpp:198-246), fuse_depth (tracking.hpp:383-394) -> DepthRecord,
RefinerLogRecord.

CPU: rg_frame_records (host code in the library) fed the reference's own raw
per-object disparities against the reference Pipeline with radar, bit-exact.
GPU: Engine.pipeline_frames (device frame loop + rg_frame_records) against
the reference Pipeline end to end, bit-exact.
"""
import ctypes as C

import numpy as np
import pytest

import oracle_lib
from paper_2604_07980_b200 import _abi, ranger as rg, synth as S
from paper_2604_07980_b200.engine import DET_DTYPE, OUT_DTYPE

OFFSETS = [0, 0, 1, 1, 1, 0]


def frames(offsets=OFFSETS, bias=0.6, scene=S.scene_c1):
    Ls, Rs, D, radar = [], [], [], []
    for t, off in enumerate(offsets):
        sc, cfg = scene(seed=90 + t, noise=2.0)
        sc.vertical_offset_px = off
        sc.disparity_bias_px = bias
        for k, o in enumerate(sc.objects):
            o.class_id = k % 3  # 0, 1 have a width prior, 2 has none
        L, R = S.render_stereo_pair(sc)
        Ls.append(L)
        Rs.append(R)
        D.append(S.ground_truth_detections(sc))
        # one return per object at its true position, deterministic jitter
        jit = np.random.default_rng(t).normal(0, 0.05, (len(sc.objects), 3))
        radar.append(np.array([o.position for o in sc.objects], np.float64) + jit)
    return np.stack(Ls), np.stack(Rs), D, radar, cfg, sc


def params(sc, ratio=0.5, refiner=True):
    cx = sc.width / 2.0 if sc.cx < 0 else sc.cx
    cy = sc.height / 2.0 if sc.cy < 0 else sc.cy
    return rg.RecordParams(rg.Calibration(sc.f, sc.b, cx, cy, sc.h_cam), object_refiner=refiner,
                           fuse_sanity_ratio=ratio)


def cdet(d):
    return _abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id)


def ref_pipeline(ref, L, R, D, radar, cfg, rect, p, method=0, bm=None):
    n, h, w = L.shape
    recs, offs = [], [0]
    for d in D:
        recs.extend(cdet(x) for x in d)
        offs.append(len(recs))
    arr = (_abi.Detection * len(recs))(*recs)
    offs = np.asarray(offs, np.int32)
    rxyz = np.ascontiguousarray(np.concatenate(radar), np.float64)
    roffs = np.cumsum([0] + [len(r) for r in radar]).astype(np.int32)
    stride = max(len(d) for d in D)
    out = (_abi.ObjectDisparity * (n * stride))()
    rec = (_abi.DepthRecord * (n * stride))()
    logs = (_abi.RefinerLog * n)()
    cnt = np.zeros(n, np.int32)
    cp, keep = p.to_c()
    st = ref.lib.ref_pipeline_records(
        L.ctypes.data, R.ctypes.data, w, h, n, C.addressof(arr), offs.ctypes.data, rxyz.ctypes.data,
        roffs.ctypes.data, C.byref(cfg.to_c()), C.byref(rect.to_c()), C.byref(cp), method,
        C.byref(bm.to_c()) if bm else None, C.addressof(out), stride, cnt.ctypes.data, C.addressof(rec),
        C.addressof(logs))
    assert st == 0
    objs = [list(out)[t * stride:t * stride + cnt[t]] for t in range(n)]
    recs_t = [list(rec)[t * stride:t * stride + cnt[t]] for t in range(n)]
    return objs, recs_t, list(logs)


def key_obj(o):
    return (int(o["det_id"]) if isinstance(o, np.void) else o.det_id,
            np.float64(o["disparity"] if isinstance(o, np.void) else o.disparity).tobytes(),
            int(o["valid"] if isinstance(o, np.void) else o.valid))


def key_rec(r):
    return (r.frame_id, r.det_id, r.valid, r.source) + tuple(
        np.float64(getattr(r, f)).tobytes() for f in ("disparity", "clp_by_stereo", "clp_by_gpt", "clp_by_size",
                                                      "z_fused"))


def key_log(g):
    return (g.frame_id,) + tuple(np.float64(getattr(g, f)).tobytes() for f in ("rect_delta", "radar_offset",
                                                                              "obj_offset"))


def selection(orc, dets, cfg):
    sel = np.zeros(len(dets), np.int32)
    ns = C.c_int()
    arr = (_abi.Detection * len(dets))(*[cdet(x) for x in dets])
    orc.fn("select_objects")(C.addressof(arr), len(dets), C.byref(cfg.to_c()), sel.ctypes.data, C.byref(ns))
    return np.array(sorted(sel[:ns.value].tolist()), np.int32)


def to_out(objs):
    a = np.zeros(len(objs), OUT_DTYPE)
    for k, o in enumerate(objs):
        a[k] = (o.det_id, o.kind, o.n_blocks_used, o.valid, o.disparity, o.z_cam)
    return a


def to_dets(dets):
    return np.array([(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets], DET_DTYPE)


@pytest.fixture(scope="module")
def ref():
    try:
        return oracle_lib.reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built here")


@pytest.mark.parametrize("ratio", [0.5, 0.02])
def test_frame_records_match_reference_pipeline(ref, orc, ratio):
    L, R, D, radar, cfg, sc = frames()
    rect = rg.RectSearchConfig()
    # the reference's raw per-object disparities (refiner off), then the
    # library's records with the refiner on against the reference's own
    raw, _, raw_logs = ref_pipeline(ref, L, R, D, radar, cfg, rect, params(sc, ratio, refiner=False))
    want_o, want_r, want_l = ref_pipeline(ref, L, R, D, radar, cfg, rect, params(sc, ratio, refiner=True))
    st = rg.ObjRefinerState()
    p = params(sc, ratio, refiner=True)
    offsets, sources = [], set()
    for t in range(len(L)):
        sel = selection(orc, D[t], cfg)
        assert len(sel) == len(raw[t])
        o, r, lg = rg.frame_records(p, t, sc.width, sc.height, to_dets(D[t]), sel, to_out(raw[t]), radar[t], st,
                                    raw_logs[t].rect_delta)
        assert [key_obj(x) for x in o] == [key_obj(x) for x in want_o[t]], t
        assert [key_rec(x) for x in r] == [key_rec(x) for x in want_r[t]], t
        assert key_log(lg) == key_log(want_l[t]), t
        offsets.append(lg.obj_offset)
        sources |= {x.source for x in r}
    assert any(v != 0 for v in offsets)  # the refiner engaged
    if ratio < 0.1:
        assert len(sources) >= 2  # the sanity check sent some objects to a monocular cue


def test_frame_records_dense_match_reference_pipeline(ref, orc):
    L, R, D, radar, cfg, sc = frames(OFFSETS[:3])
    rect = rg.RectSearchConfig(enabled=False)
    bm = rg.BmParams(32, 9, 0, 10, 10, 1)
    p = params(sc)
    want_o, want_r, want_l = ref_pipeline(ref, L, R, D, radar, cfg, rect, p, method=1, bm=bm)
    st = rg.ObjRefinerState()
    for t in range(len(L)):
        sel = selection(orc, D[t], cfg)
        o, r, lg = rg.frame_records(p, t, sc.width, sc.height, to_dets(D[t]), sel, to_out(want_o[t]), radar[t], st,
                                    0.0, dense=True)
        assert [key_rec(x) for x in r] == [key_rec(x) for x in want_r[t]], t
        assert key_log(lg) == key_log(want_l[t]), t


def test_frame_records_errors():
    sc, _ = S.scene_c1()
    p = params(sc)
    d = to_dets(S.ground_truth_detections(sc))
    o = np.zeros(1, OUT_DTYPE)
    with pytest.raises(rg.InvalidArgument):  # selection index out of range
        rg.frame_records(p, 0, sc.width, sc.height, d, np.array([len(d)], np.int32), o, None, rg.ObjRefinerState())
    # a stereo point 1 m ahead paired with a radar return 0.5 m behind the
    # camera: project_radar_to_disparity throws (radar_refiner.hpp:24-25)
    o[0]["valid"], o[0]["disparity"] = 1, sc.f * sc.b
    u, v = d[0]["cx"] * sc.width, d[0]["cy"] * sc.height
    cx, cy = sc.width / 2.0, sc.height / 2.0
    xc, yc = (u - cx) / (1 / sc.b * o[0]["disparity"]), (v - cy) / (1 / sc.b * o[0]["disparity"])
    bad = np.array([[-0.5, -xc, sc.h_cam - yc]])
    with pytest.raises(rg.InvalidArgument):
        rg.frame_records(p, 0, sc.width, sc.height, d, np.array([0], np.int32), o, bad, rg.ObjRefinerState())
    far = np.array([[-50.0, -xc, sc.h_cam - yc]])  # behind the camera but never paired: no error
    rg.frame_records(p, 0, sc.width, sc.height, d, np.array([0], np.int32), o, far, rg.ObjRefinerState())
    with pytest.raises(rg.InvalidArgument):
        rg.Calibration(0.0, 0.3, 320, 240, 1.5)


@pytest.mark.gpu
def test_pipeline_frames_match_reference(ctx, ref):
    import torch

    from paper_2604_07980_b200.engine import FrameEngine

    L, R, D, radar, cfg, sc = frames()
    rect = rg.RectSearchConfig()
    p = params(sc, 0.05)
    want_o, want_r, want_l = ref_pipeline(ref, L, R, D, radar, cfg, rect, p)
    eng = FrameEngine(sc.width, sc.height, cfg, max(len(d) for d in D), ctx=ctx)
    dev = torch.device("cuda", 0)
    objs, recs, logs = eng.pipeline_frames(torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev), D, p,
                                           radar=radar, rect=rect)
    for t in range(len(L)):
        assert [key_obj(x) for x in objs[t]] == [key_obj(x) for x in want_o[t]], t
        assert [key_rec(x) for x in recs[t]] == [key_rec(x) for x in want_r[t]], t
        assert key_log(logs[t]) == key_log(want_l[t]), t
    assert any(lg.obj_offset != 0 for lg in logs) and any(lg.rect_delta != 0 for lg in logs)
