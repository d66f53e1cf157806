"""Sequence orchestration (SURVEY.md 8(e) two-pass schedule, 8(f) row 1):
Pipeline::process_frame's TEMPLATE_MATCHER loop -- offset search on the
uncorrected pair, filter_offset, ranging of shift_vertical(left, lround(cur)).

CPU: the C filter (rg_filter_offset, host code in the library) against the
restatement; the composed oracle schedule against the reference's own
Pipeline (oracle/_ref) when it was built.  GPU: rg_range_sequence against the
composed oracle, frame by frame, bit-exact.
"""
import ctypes as C

import numpy as np
import pytest

import oracle_lib
from paper_2604_07980_b200 import _abi, ranger as rg, synth as S

OFFSETS = [2, 2, 2, 2, -1, -1, 0, 3]


def seq_frames(offsets=OFFSETS, scene=S.scene_c1):
    Ls, Rs, D = [], [], []
    for t, off in enumerate(offsets):
        sc, cfg = scene(seed=70 + t, noise=2.0)
        sc.vertical_offset_px = off
        L, R = S.render_stereo_pair(sc)
        Ls.append(L)
        Rs.append(R)
        D.append(S.ground_truth_detections(sc))
    return np.stack(Ls), np.stack(Rs), D, cfg, sc


def shift_vertical(img, dy):  # image.hpp:145-154
    h = img.shape[0]
    return np.ascontiguousarray(img[np.clip(np.arange(h) - dy, 0, h - 1)])


def rect_roi(w, h, need):  # pipeline.hpp:268-275
    x0, y0, x1, y1 = w // 4, h // 4, w * 3 // 4, h * 3 // 4
    return (x0, y0, max(x1, min(w, x0 + need)), max(y1, min(h, y0 + need)))


def cdet(d):
    return _abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id)


def oracle_sequence(chk, L, R, D, cfg, rect):
    """The schedule restated over the oracle's per-function checkers."""
    st = rg.RectOffsetState(rect.window, rect.rate_limit)
    h, w = L.shape[1:]
    roi = rect_roi(w, h, rect.bm.block_size)
    shifts, deltas, objs = [], [], []
    for t in range(len(L)):
        cur = st.current if rect.enabled else 0.0
        s = int(np.floor(abs(cur) + 0.5)) * (1 if cur >= 0 else -1)  # std::lround
        out, _ = chk.estimate(shift_vertical(L[t], s), R[t], [cdet(d) for d in D[t]], cfg.to_c())
        d = 0
        if rect.enabled:
            _, d, _ = chk.autorect(L[t], R[t], roi, rect.delta_min, rect.delta_max, rect.bm.to_c())
            rg.filter_offset(st, d)
        shifts.append(s)
        deltas.append(d)
        objs.append(out)
    return shifts, deltas, objs


def test_filter_offset_c_matches_restatement():
    lib = rg.lib()
    rng = np.random.default_rng(3)
    for window, rate in [(1, 1.0), (5, 1.0), (4, 0.5), (7, 2.0)]:
        st = rg.RectOffsetState(window, rate)
        cs = _abi.RectState()
        assert lib.rg_rect_state_init(C.byref(cs), window, rate) == 0
        for d in rng.integers(-6, 7, 40):
            want = rg.filter_offset(st, int(d))
            got = C.c_double()
            assert lib.rg_filter_offset(C.byref(cs), int(d), C.byref(got)) == 0
            assert got.value == want
        assert cs.n_hist == len(st.history) and cs.next == st.next
    assert lib.rg_rect_state_init(C.byref(cs), 0, 1.0) != 0  # autorect.hpp:71


def test_oracle_schedule_equals_reference_pipeline(orc):
    try:
        ref = oracle_lib.reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built here")
    L, R, D, cfg, sc = seq_frames()
    rect = rg.RectSearchConfig()
    shifts, deltas, objs = oracle_sequence(orc, L, R, D, cfg, rect)
    n, h, w = L.shape
    recs, offs = [], [0]
    for d in D:
        recs.extend(cdet(x) for x in d)
        offs.append(len(recs))
    arr = (_abi.Detection * len(recs))(*recs)
    offs = np.asarray(offs, np.int32)
    stride = max(len(d) for d in D)
    out = (_abi.ObjectDisparity * (n * stride))()
    cnt = np.zeros(n, np.int32)
    applied = np.zeros(n, np.float64)
    rc = rect.to_c()
    st = ref.lib.ref_pipeline_sequence(L.ctypes.data, R.ctypes.data, w, h, n, C.addressof(arr), offs.ctypes.data,
                                       C.byref(cfg.to_c()), C.byref(rc), sc.f, sc.b, sc.cx, sc.cy, sc.h_cam,
                                       0, None, C.addressof(out), stride, cnt.ctypes.data, applied.ctypes.data)
    assert st == 0
    # shifts actually move, and match the reference's applied rect offset
    assert any(s != 0 for s in shifts)
    assert [int(np.floor(abs(a) + 0.5)) * (1 if a >= 0 else -1) for a in applied] == shifts
    for t in range(n):
        got = [(o.det_id, o.kind, o.n_blocks_used, o.valid, np.float64(o.disparity).tobytes())
               for o in list(out)[t * stride:t * stride + cnt[t]]]
        want = [(o.det_id, o.kind, o.n_blocks_used, o.valid, np.float64(o.disparity).tobytes()) for o in objs[t]]
        assert got == want, t


@pytest.mark.gpu
@pytest.mark.parametrize("enabled", [True, False])
def test_range_sequence_matches_oracle(ctx, orc, enabled):
    import torch
    from paper_2604_07980_b200.engine import FrameEngine, pack_detections

    L, R, D, cfg, sc = seq_frames()
    rect = rg.RectSearchConfig(enabled=enabled)
    shifts, deltas, objs = oracle_sequence(orc, L, R, D, cfg, rect)
    n = len(L)
    eng = FrameEngine(sc.width, sc.height, cfg, max(len(d) for d in D), ctx=ctx)
    recs, offs = pack_detections(D)
    dev = torch.device("cuda", 0)
    out = torch.zeros(n * eng.out_stride * 32, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(n, dtype=torch.int32, device=dev)
    state = rg.RectOffsetState(rect.window, rect.rate_limit)
    # two calls: the filter state carries across batches
    got_s, got_d = [], []
    for a, b in ((0, 5), (5, n)):
        s, d = eng.range_sequence(torch.from_numpy(L[a:b]).to(dev), torch.from_numpy(R[a:b]).to(dev),
                                  torch.from_numpy(pack_detections(D[a:b])[0].view(np.uint8)).to(dev),
                                  torch.from_numpy(pack_detections(D[a:b])[1]).to(dev),
                                  out[a * eng.out_stride * 32:], cnt[a:], rect=rect, state=state)
        got_s += s.tolist()
        got_d += d.tolist()
    torch.cuda.synchronize()
    assert got_s == shifts and got_d == deltas
    o = out.cpu().numpy().reshape(n, eng.out_stride * 32)
    for t in range(n):
        want = b"".join(bytes(x) for x in objs[t])
        assert int(cnt[t]) * 32 == len(want)
        assert o[t, :len(want)].tobytes() == want, t


# ------------------------------------------------------------ dense STEREO_BM branch (8f row 3)
def test_oracle_box_variance_equals_reference(orc):
    if not oracle_lib.have_reference():
        pytest.skip("oracle/_ref not built here")
    ref = oracle_lib.reference()
    rng = np.random.default_rng(4)
    for n in (1, 2, 7, 100):
        raw = rng.integers(-40, 900, (1, n)).astype(np.int16)
        d = _abi.Detection(0.5, 0.5, 1.0, 1.0, 0, 1)
        got = _abi.BoxStats()
        assert orc.lib.orc_box_disparity(raw.ctypes.data, n, 1, C.byref(d), 1, 0.3, 1.0, 0.01, C.byref(got)) == 0
        v = np.sort(raw.ravel() / 16.0)
        near = np.ascontiguousarray(v[(3 * (n - 1)) // 4:])
        want = C.c_double()
        assert ref.lib.ref_dynamic_disparity_variance(near.ctypes.data, len(near), v.ctypes.data, n, 0.3, 1.0, 0.01,
                                                      C.byref(want)) == 0
        assert got.variance == want.value and got.median == v[(n - 1) // 2] and got.count == n


def test_oracle_dense_objects_equal_reference_pipeline(orc):
    """The reference Pipeline with method STEREO_BM (no radar): its objects are
    ObjectDisparity {det id, kind, box median, count} from box_disparity of
    the dense BM map of the rect-corrected pair."""
    if not oracle_lib.have_reference():
        pytest.skip("oracle/_ref not built here")
    ref = oracle_lib.reference()
    L, R, D, cfg, sc = seq_frames([0, 0, 0])
    n, h, w = L.shape
    bm = rg.BmParams(32, 9, 0, 10, 10, 1)  # PipelineConfig::bm defaults (pipeline.hpp:67)
    rect = rg.RectSearchConfig(enabled=False)
    recs, offs = [], [0]
    for d in D:
        recs.extend(cdet(x) for x in d)
        offs.append(len(recs))
    arr = (_abi.Detection * len(recs))(*recs)
    offs = np.asarray(offs, np.int32)
    stride = max(len(d) for d in D)
    out = (_abi.ObjectDisparity * (n * stride))()
    cnt = np.zeros(n, np.int32)
    applied = np.zeros(n)
    assert ref.lib.ref_pipeline_sequence(L.ctypes.data, R.ctypes.data, w, h, n, C.addressof(arr), offs.ctypes.data,
                                         C.byref(cfg.to_c()), C.byref(rect.to_c()), sc.f, sc.b, sc.cx, sc.cy,
                                         sc.h_cam, 1, C.byref(bm.to_c()), C.addressof(out), stride, cnt.ctypes.data,
                                         applied.ctypes.data) == 0
    for t in range(n):
        _, raw = orc.bm(L[t], R[t], bm.to_c())
        sel = np.zeros(len(D[t]), np.int32)
        ns = C.c_int()
        dets = (_abi.Detection * len(D[t]))(*[cdet(x) for x in D[t]])
        orc.fn("select_objects")(C.addressof(dets), len(D[t]), C.byref(cfg.to_c()), sel.ctypes.data, C.byref(ns))
        idx = sorted(sel[:ns.value].tolist())
        boxes = (_abi.Detection * max(len(idx), 1))(*[cdet(D[t][i]) for i in idx])
        st = (_abi.BoxStats * max(len(idx), 1))()
        assert orc.lib.orc_box_disparity(raw.ctypes.data, w, h, C.addressof(boxes), len(idx), 0.3, 1.0, 0.01,
                                         C.addressof(st)) == 0
        got = [(o.det_id, o.kind, o.n_blocks_used, o.valid, o.disparity) for o in list(out)[t * stride:t * stride + cnt[t]]]
        want = []
        for k, i in enumerate(idx):
            d = D[t][i]
            kind = 0 if max(d.w * w, d.h * h) < cfg.tau_s else 1
            want.append((d.id, kind, st[k].count if st[k].valid else 0, int(st[k].valid > 0),
                         st[k].median if st[k].valid else 0.0))
        assert got == want, t


@pytest.mark.gpu
@pytest.mark.parametrize("bs,nd,dmin,ds", [(9, 32, 0, 1), (7, 48, -4, 1), (9, 64, 0, 2)])
def test_dense_objects_match_oracle(ctx, orc, bs, nd, dmin, ds):
    L, R, D, cfg, sc = seq_frames([0, 1])
    bm = rg.BmParams(nd, bs, dmin, 10, 10, ds)
    for t in range(len(L)):
        objs, boxes, raw = rg.dense_objects(L[t], R[t], D[t], cfg, bm, ctx=ctx)
        st, want_raw = orc.bm(L[t], R[t], bm.to_c())
        assert np.array_equal(raw, want_raw)
        sel = np.zeros(len(D[t]), np.int32)
        ns = C.c_int()
        dets = (_abi.Detection * len(D[t]))(*[cdet(x) for x in D[t]])
        orc.fn("select_objects")(C.addressof(dets), len(D[t]), C.byref(cfg.to_c()), sel.ctypes.data, C.byref(ns))
        idx = sorted(sel[:ns.value].tolist())
        bx = (_abi.Detection * max(len(idx), 1))(*[cdet(D[t][i]) for i in idx])
        stt = (_abi.BoxStats * max(len(idx), 1))()
        orc.lib.orc_box_disparity(want_raw.ctypes.data, sc.width, sc.height, C.addressof(bx), len(idx), 0.3, 1.0,
                                  0.01, C.addressof(stt))
        assert len(objs) == len(idx)
        for k, i in enumerate(idx):
            assert objs[k].det_id == D[t][i].id
            assert objs[k].valid == (stt[k].valid > 0)
            if objs[k].valid:
                assert np.float64(objs[k].disparity).tobytes() == np.float64(stt[k].median).tobytes()
                assert np.float64(boxes[k].variance).tobytes() == np.float64(stt[k].variance).tobytes()
                assert boxes[k].count == stt[k].count == objs[k].n_blocks_used


def _radar_frames(n, bias):
    Ls, Rs, D, RA, scs = [], [], [], [], []
    for t in range(n):
        sc, cfg = S.scene_c1(seed=90 + t, noise=2.0)
        sc.disparity_bias_px = bias
        L, R = S.render_stereo_pair(sc)
        Ls.append(L)
        Rs.append(R)
        D.append(S.ground_truth_detections(sc))
        # simulate_radar without noise (synth.hpp:234-249): extent = (depth, width, height)
        RA.append([(o.position, (o.depth_m, o.width_m, o.height_m), o.id) for o in sc.objects])
        scs.append(sc)
    return np.stack(Ls), np.stack(Rs), D, RA, cfg, scs[0]


@pytest.mark.gpu
@pytest.mark.parametrize("bias", [0.0, 1.5, -2.25])
def test_dense_radar_refiner_matches_reference_pipeline(ctx, bias):
    """STEREO_BM with the radar refiner on (PipelineConfig::radar_refiner
    default, pipeline.hpp:69, 182-183): per frame the box medians of the
    refined map and the refiner's radar offset equal the reference Pipeline's,
    the vote state carried across frames (radar_refiner.hpp:111-167)."""
    if not oracle_lib.have_reference():
        pytest.skip("oracle/_ref not built")
    ref = oracle_lib.reference()
    n = 6
    L, R, D, RA, cfg, sc = _radar_frames(n, bias)
    h, w = L.shape[1:]
    bm = rg.BmParams(32, 9, 0, 10, 10, 1)  # PipelineConfig::bm defaults
    calib = rg.Calibration(sc.f, sc.b, w / 2.0, h / 2.0, sc.h_cam)
    vote = rg.VoteState()
    got, got_applied = [], []
    for t in range(n):
        objs, _, _, a = rg.dense_objects_refined(L[t], R[t], D[t], cfg, bm, RA[t], vote, calib, ctx=ctx)
        got.append([(o.det_id, o.kind, o.n_blocks_used, int(o.valid), o.disparity) for o in objs])
        got_applied.append(a)
    recs, offs = [], [0]
    for d in D:
        recs.extend(cdet(x) for x in d)
        offs.append(len(recs))
    arr = (_abi.Detection * len(recs))(*recs)
    offs = np.asarray(offs, np.int32)
    flat = [r for fr in RA for r in fr]
    rarr = rg.radar_array(flat)
    roffs = np.cumsum([0] + [len(fr) for fr in RA]).astype(np.int32)
    stride = max(len(d) for d in D)
    out = (_abi.ObjectDisparity * (n * stride))()
    cnt = np.zeros(n, np.int32)
    applied = np.zeros(n)
    assert ref.lib.ref_pipeline_dense_radar(L.ctypes.data, R.ctypes.data, w, h, n, C.addressof(arr), offs.ctypes.data,
                                            C.addressof(rarr), roffs.ctypes.data, C.byref(cfg.to_c()),
                                            C.byref(calib.to_c()), C.byref(bm.to_c()), 4, 0.3, 1.0, C.addressof(out),
                                            stride, cnt.ctypes.data, applied.ctypes.data) == 0
    for t in range(n):
        want = [(o.det_id, o.kind, o.n_blocks_used, o.valid, o.disparity)
                for o in list(out)[t * stride:t * stride + cnt[t]]]
        assert got[t] == want, t
    assert np.array(got_applied).tobytes() == applied.tobytes()
    if bias != 0.0:
        assert abs(applied[-1]) > 0.1  # the refiner acted
