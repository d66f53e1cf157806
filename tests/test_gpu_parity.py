"""GPU parity: the CUDA path (through the C ABI) against the reference itself
(oracle/_ref, compiled in place; the C restatement where it is absent).

Every comparison is bit-exact: census codes, MatchResult fields (including
the FP64 cost / sub-pixel fields, compared as raw bytes), ObjectDisparity
records, BM raw maps, delta* and per-delta counts.  Seeded inputs at sizes the
oracle finishes in seconds; full-size configs go through bench-style checks in
test_gpu_scale.py.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2604_07980_b200 import _abi, synth as S
from paper_2604_07980_b200 import ranger as rg

pytestmark = pytest.mark.gpu


def rand_img(rng, h, w, vmax=255):
    return rng.integers(0, vmax + 1, (h, w), dtype=np.uint8)


def det_c(d):
    return _abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id)


# ------------------------------------------------------------------ arithmetic
def test_matcher_integer_division_is_ieee(ctx):
    """The matcher's cost / neighbour-cost quotients (integer sum / point
    count) use a table of RN(1/b) and one Markstein correction instead of
    __ddiv_rn; every (a, b) with b <= 4096 and a <= 64 b (a pass's sums are
    <= 63 b) must give the IEEE quotient's bits -- and b beyond the table
    falls back to the division."""
    assert ctx.selftest_division(4096 + 64) == 0


# ------------------------------------------------------------------ census
@pytest.mark.parametrize("w,h,ow,oh", [(9, 9, 9, 9), (20, 15, 20, 15), (41, 33, 20, 16), (64, 48, 64, 48),
                                       (641, 481, 320, 240), (1920, 1080, 960, 540), (133, 77, 66, 38)])
def test_census_transform_matches_oracle(ctx, chk, w, h, ow, oh):
    rng = np.random.default_rng(w * 1000 + h)
    img = rand_img(rng, h, w)
    got = rg.census_transform(img, ow, oh, ctx=ctx).codes
    assert np.array_equal(got, chk.census(img, ow, oh))


def test_census_anchor(ctx):  # test_census.cpp:35-40, acceptance 1
    rows = [[48, 72, 35, 91, 63], [85, 57, 44, 68, 29], [61, 93, 55, 37, 76], [42, 66, 81, 50, 88],
            [73, 38, 59, 94, 46]]
    img = np.zeros((9, 9), np.uint8)
    img[2:7, 2:7] = rows
    assert rg.census_code_at(img, 4, 4, ctx=ctx) == 0x2BD65B6
    assert rg.census_transform(img, ctx=ctx).code(4, 4) == 0x2BD65B6
    assert rg.census_code_at(np.full((9, 9), 77, np.uint8), 4, 4, ctx=ctx) == 1 << 25
    assert rg.census_code_at(img, 1, 4, ctx=ctx) == 0


def test_census_rois_matches_oracle(ctx, chk):
    rng = np.random.default_rng(31)
    img = rand_img(rng, 36, 48)
    rois = [(4, 4, 20, 16), (10, 12, 30, 24), (40, 30, 48, 36), (-3, -2, 5, 4), (30, 1, 20, 9)]
    got = rg.census_transform_rois(img, 48, 36, [rg.CensusRoi(*r) for r in rois], ctx=ctx).codes
    assert np.array_equal(got, chk.census_rois(img, 48, 36, rois))
    got = rg.census_transform_rois(img, 24, 18, [rg.CensusRoi(*r) for r in rois], ctx=ctx).codes
    assert np.array_equal(got, chk.census_rois(img, 24, 18, rois))


def test_census_monotone_invariance(ctx):  # test_census.cpp:63-74
    rng = np.random.default_rng(9)
    img = (rand_img(rng, 30, 40) // 2) * 2
    a = rg.census_transform(img, ctx=ctx).codes
    b = rg.census_transform((40 + img // 2).astype(np.uint8), ctx=ctx).codes
    assert np.array_equal(a, b)


# ------------------------------------------------------------------ matcher
def _gpu_match(ctx, L, R, blocks, mode, tau_v=1.0):
    qb = [rg.QueryBlock(list(p), *r) for p, r in blocks]
    pts, offs, rgs = rg._blocks_csr(qb)
    out = (_abi.MatchResult * len(blocks))()
    L = np.ascontiguousarray(L, np.uint32)
    R = np.ascontiguousarray(R, np.uint32)
    ctx.check(rg.lib().rg_match_blocks(ctx.handle, rg._ptr(L), L.shape[1], L.shape[0], rg._ptr(R), R.shape[1],
                                       R.shape[0], rg._ptr(pts), rg._ptr(offs), rgs, len(blocks), mode, tau_v,
                                       out))
    return list(out)


def _same(a, b):
    fields = ["dx_int", "dy_int", "dx_subpix", "cost", "cost_minus", "cost_plus", "valid_points", "verified",
              "has_value"]
    if a.has_value != b.has_value:
        return False
    if not a.has_value:
        return True
    return all(np.float64(getattr(a, f)).tobytes() == np.float64(getattr(b, f)).tobytes()
               if isinstance(getattr(a, f), float) else getattr(a, f) == getattr(b, f) for f in fields)


@pytest.mark.parametrize("mode", [0, 1])
def test_block_match_random_protocol(ctx, chk, mode):  # test_matching.cpp:78-108
    rng = np.random.default_rng(99 + mode)
    blocks, Ls, Rs = [], [], []
    bad = 0
    for trial in range(120):
        L = chk.census(rand_img(rng, 30, 40))
        R = chk.census(rand_img(rng, 30, 40))
        n = int(rng.integers(1, 13))
        pts = [(int(rng.integers(0, 40)), int(rng.integers(0, 30))) for _ in range(n)]
        dxm = int(rng.integers(-3, 3))
        dym = int(rng.integers(-2, 1))
        blk = [(pts, (dxm, dxm + int(rng.integers(0, 13)), dym, dym + int(rng.integers(0, 4))))]
        st, want = chk.match(L, R, blk, mode)
        got = _gpu_match(ctx, L, R, blk, mode)
        bad += not _same(got[0], want[0])
    assert bad == 0


def test_block_match_big_blocks_and_windows(ctx, chk):
    """Blocks that exercise the global-memory path (window > smem) and the
    zero-code path (points near the border, ROI-masked rasters)."""
    rng = np.random.default_rng(5)
    img_l, img_r = rand_img(rng, 200, 300), rand_img(rng, 200, 300)
    L, R = chk.census(img_l), chk.census(img_r)
    Rm = R.copy()
    Rm[50:120, 100:180] = 0  # holes of undefined codes
    blocks = []
    for k in range(24):
        n = int(rng.integers(1, 80))
        pts = [(int(rng.integers(-5, 305)), int(rng.integers(-5, 205))) for _ in range(n)]
        dx0 = int(rng.integers(-40, 10))
        blocks.append((pts, (dx0, dx0 + int(rng.integers(0, 300)), -2, int(rng.integers(-2, 3)))))
    for Rx in (R, Rm):
        st, want = chk.match(L, Rx, blocks, 1)
        got = _gpu_match(ctx, L, Rx, blocks, 1)
        assert all(_same(g, w) for g, w in zip(got, want))


def test_block_match_empty_range_raises(ctx):
    L = np.zeros((10, 10), np.uint32)
    with pytest.raises(rg.InvalidArgument):
        rg.block_match(rg.QueryBlock([(1, 1)], 3, 2, 0, 0), rg.CensusImage(10, 10, L),
                       rg.CensusImage(10, 10, L), ctx=ctx)
    # an empty block returns nullopt before the range check (census.hpp:181)
    assert rg.block_match(rg.QueryBlock([], 3, 2, 0, 0), rg.CensusImage(10, 10, L),
                          rg.CensusImage(10, 10, L), ctx=ctx) is None


# ------------------------------------------------------------------ object ranger
@pytest.mark.parametrize("name,noise", [("c1", 0.0), ("c1", 2.0), ("c2", 0.0), ("c2", 2.0), ("c3", 2.0),
                                        ("c3s", 2.0)])
def test_estimate_object_disparities_matches_oracle(ctx, chk, name, noise):
    fn = {"c1": S.scene_c1, "c2": S.scene_c2, "c3": S.scene_c3,
          "c3s": lambda seed, noise: S.scene_c3(seed, noise, stress=True)}[name]
    sc, cfg = fn(seed=11, noise=noise)
    L, R = S.render_stereo_pair(sc)
    dets = S.ground_truth_detections(sc)
    stats = rg.RangerStats()
    got = rg.estimate_object_disparities(L, R, dets, cfg, stats=stats, focal_px=2000.0, baseline_m=0.3, ctx=ctx)
    want, wst = chk.estimate(L, R, [det_c(d) for d in dets], cfg.to_c(), 2000.0, 0.3)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert (g.det_id, g.kind, g.n_blocks_used, g.valid) == (w.det_id, w.kind, w.n_blocks_used, bool(w.valid))
        assert np.float64(g.disparity).tobytes() == np.float64(w.disparity).tobytes()
        assert np.float64(g.z_cam).tobytes() == np.float64(w.z_cam).tobytes()
    assert (stats.query_points, stats.n_far, stats.n_close) == (wst.query_points, wst.n_far, wst.n_close)


def test_estimate_cache_fill_and_reuse(ctx, chk):
    sc, cfg = S.scene_c1(seed=4, noise=2.0)
    L, R = S.render_stereo_pair(sc)
    dets = S.ground_truth_detections(sc)
    cache = rg.CensusCache()
    got = rg.estimate_object_disparities(L, R, dets, cfg, cache=cache, ctx=ctx)
    h, w = L.shape
    oc = _abi.CensusCache()
    bufs = [np.zeros((h, w), np.uint32), np.zeros((h, w), np.uint32), np.zeros((h // 2, w // 2), np.uint32),
            np.zeros((h // 2, w // 2), np.uint32)]
    oc.full_left, oc.full_right, oc.scaled_left, oc.scaled_right = [b.ctypes.data for b in bufs]
    want, _ = chk.estimate(L, R, [det_c(d) for d in dets], cfg.to_c(), cache=oc)
    assert cache.has_full == bool(oc.has_full) and cache.has_scaled == bool(oc.has_scaled)
    assert np.array_equal(cache.full_left.codes, bufs[0]) and np.array_equal(cache.full_right.codes, bufs[1])
    assert np.array_equal(cache.scaled_left.codes, bufs[2]) and np.array_equal(cache.scaled_right.codes, bufs[3])
    # a pre-filled full-frame cache gives the same answer (test_template_ranger.cpp:243-274)
    full = rg.CensusCache(rg.census_transform(L, ctx=ctx), rg.census_transform(R, ctx=ctx),
                          rg.census_transform(L, w // 2, h // 2, ctx=ctx),
                          rg.census_transform(R, w // 2, h // 2, ctx=ctx), True, True)
    again = rg.estimate_object_disparities(L, R, dets, cfg, cache=full, ctx=ctx)
    assert [(a.det_id, a.valid, a.disparity, a.n_blocks_used) for a in got] == \
           [(b.det_id, b.valid, b.disparity, b.n_blocks_used) for b in again]


def test_planner_helpers_match_oracle(ctx, chk):
    sc, cfg = S.scene_c3(seed=2, noise=0.0)
    dets = S.ground_truth_detections(sc)
    dc = (_abi.Detection * len(dets))(*[det_c(d) for d in dets])
    for budget in (256, 100, 7, 0):
        cfg.max_objects = budget
        got = rg.select_objects(dets, cfg, ctx=ctx)
        want = np.zeros(len(dets), np.int32)
        n = C.c_int()
        chk.fn("select_objects")(C.addressof(dc), len(dets), C.byref(cfg.to_c()), want.ctypes.data, C.byref(n))
        assert got == list(want[:n.value])
    occ = rg.find_occluders(dets, ctx=ctx)
    off = np.zeros(len(dets) + 1, np.int32)
    idx = np.zeros(len(dets) ** 2, np.int32)
    chk.fn("find_occluders")(C.addressof(dc), len(dets), off.ctypes.data, idx.ctypes.data)
    assert occ == [list(idx[off[i]:off[i + 1]]) for i in range(len(dets))]
    assert sum(1 for o in occ if o) == 96
    rng = np.random.default_rng(3)
    for t in range(40):
        v = np.round(rng.normal(10, 3, int(rng.integers(0, 30))), 1)
        got = rg.aggregate_close_disparities(v, 1.0, 3, ctx=ctx)
        vi, ri = C.c_int32(), C.c_int32()
        dd = C.c_double()
        chk.fn("aggregate_close_disparities")(v.ctypes.data if v.size else None, v.size, 1.0, 3, C.byref(vi),
                                             C.byref(dd), C.byref(ri))
        assert (got.valid, got.disparity, got.run_length) == (bool(vi.value), dd.value, ri.value)


# ------------------------------------------------------------------ BM / autorect
@pytest.mark.parametrize("nd,bs,dmin,ds,tex,uniq", [(12, 5, 0, 1, 10, 10), (12, 5, 3, 1, 10, 10),
                                                    (16, 9, 0, 1, 0, 0), (24, 9, -4, 1, 10, 10),
                                                    (9, 5, 2, 2, 0, 0), (24, 9, 0, 2, 10, 10),
                                                    (40, 7, -5, 1, 0, 15), (64, 9, 0, 1, 10, 10)])
def test_bm_disparity_matches_oracle(ctx, chk, nd, bs, dmin, ds, tex, uniq):
    rng = np.random.default_rng(nd * 31 + bs)
    sc = S.SceneConfig(width=160, height=96, background_contrast=80, seed=3)
    L, _ = S.render_stereo_pair(sc)
    R = np.ascontiguousarray(np.roll(L, -5, axis=1))
    for a, b in ((rand_img(rng, 28, 48), rand_img(rng, 28, 48)), (L, R)):
        p = rg.BmParams(nd, bs, dmin, tex, uniq, ds)
        got = rg.bm_disparity(a, b, p, ctx=ctx)
        st, want = chk.bm(a, b, p.to_c())
        assert st == 0 and np.array_equal(got, want)


@pytest.mark.parametrize("nd,bs,dmin,tex,uniq", [(32, 3, -8, 5, 5), (32, 7, 4, 20, 25), (31, 9, 0, 10, 10),
                                                 (8, 3, 0, 0, 0), (17, 5, -20, 40, 15), (32, 9, -4, 10, 10)])
def test_bm_simd_path_matches_oracle(ctx, chk, nd, bs, dmin, tex, uniq):
    """Wide frames so most bands take the byte-SIMD kernel (nd <= 32, bs <= 9)."""
    rng = np.random.default_rng(nd * 7 + bs + dmin)
    sc = S.SceneConfig(width=320, height=90, background_contrast=90, seed=nd + bs)
    L, _ = S.render_stereo_pair(sc)
    R = np.ascontiguousarray(np.roll(L, -7, axis=1))
    R[::7] = rand_img(rng, R[::7].shape[0], 320)  # some rows unmatched
    for a, b in ((L, R), (rand_img(rng, 70, 300), rand_img(rng, 70, 300))):
        p = rg.BmParams(nd, bs, dmin, tex, uniq, 1)
        got = rg.bm_disparity(a, b, p, ctx=ctx)
        st, want = chk.bm(a, b, p.to_c())
        assert st == 0 and np.array_equal(got, want)


@pytest.mark.parametrize("voff", [-3, 0, 2])
def test_auto_rect_search_matches_oracle(ctx, chk, voff):  # test_autorect.cpp:36-42
    sc = S.SceneConfig(objects=[S.SceneObject(id=1, position=(30.0, 0.0, 1.5), texture_seed=11)],
                       vertical_offset_px=voff)
    L, R = S.render_stereo_pair(sc)
    p = rg.BmParams(24, 9, 0, 10, 10, 1)
    counts = []
    got = rg.auto_rect_search(L, R, rg.ImageRoi(240, 160, 400, 240), -3, 3, p, ctx=ctx, counts_out=counts)
    st, want, wc = chk.autorect(L, R, (240, 160, 400, 240), -3, 3, p.to_c())
    assert got == want == voff
    assert counts == list(wc)


def test_auto_rect_flat_ties(ctx):  # test_autorect.cpp:44-50
    flat = np.zeros((64, 64), np.uint8)
    p = rg.BmParams(24, 9, 0, 10, 10, 1)
    roi = rg.ImageRoi(8, 8, 56, 56)
    assert rg.auto_rect_search(flat, flat, roi, -3, 3, p, ctx=ctx) == 0
    assert rg.auto_rect_search(flat, flat, roi, 1, 3, p, ctx=ctx) == 1
    assert rg.auto_rect_search(flat, flat, roi, -3, -1, p, ctx=ctx) == -1


def test_auto_rect_c4_counts(ctx, chk):
    """C4 scene, central ROI, delta in [-8, 8]: delta* and all 17 counts."""
    sc = S.scene_c4(-5)
    L, R = S.render_stereo_pair(sc)
    p = S.c4_bm()
    counts = []
    got = rg.auto_rect_search(L, R, rg.ImageRoi(*S.C4_ROI), -8, 8, p, ctx=ctx, counts_out=counts)
    assert got == -5
    # oracle on a cheaper sub-ROI for the per-delta counts
    roi = (720, 405, 1200, 675)
    counts = []
    got = rg.auto_rect_search(L, R, rg.ImageRoi(*roi), -8, 8, p, ctx=ctx, counts_out=counts)
    st, want, wc = chk.autorect(L, R, roi, -8, 8, p.to_c())
    assert got == want and counts == list(wc)


@pytest.mark.parametrize("voff", [-8, -5, 0, 3, 8])
def test_auto_rect_c4_full_roi_counts_vs_reference(ctx, chk, voff):
    """C4 at full size: the central 960x540 ROI (480,270)-(1440,810), delta in
    [-8, 8]; delta* and all 17 per-delta counts against the reference's
    auto_rect_search at workers = nproc (autorect.hpp:22-58)."""
    import os
    if getattr(chk, "kind", None) != "reference":
        pytest.skip("oracle/_ref not built")
    sc = S.scene_c4(voff)
    L, R = S.render_stereo_pair(sc)
    p = S.c4_bm()
    counts = []
    got = rg.auto_rect_search(L, R, rg.ImageRoi(*S.C4_ROI), -8, 8, p, ctx=ctx, counts_out=counts)
    st, want, wc = chk.autorect_mt(L, R, S.C4_ROI, -8, 8, p.to_c(), len(os.sched_getaffinity(0)))
    assert st == 0 and got == want == voff
    assert counts == list(wc)


@pytest.mark.parametrize("voff,ds", [(-2, 2), (1, 2), (0, 3)])
def test_auto_rect_search_downscale_on_device(ctx, chk, voff, ds):
    """autorect.hpp:36-44 with BmParams.downscale > 1: the shifted crops, the
    downscaled BM and the counts all on the device; delta* and every count
    equal the reference's."""
    sc = S.SceneConfig(objects=[S.SceneObject(id=1, position=(30.0, 0.0, 1.5), texture_seed=11)],
                       vertical_offset_px=voff)
    L, R = S.render_stereo_pair(sc)
    p = rg.BmParams(24, 9, 0, 10, 10, ds)
    counts = []
    got = rg.auto_rect_search(L, R, rg.ImageRoi(200, 120, 440, 280), -3, 3, p, ctx=ctx, counts_out=counts)
    st, want, wc = chk.autorect(L, R, (200, 120, 440, 280), -3, 3, p.to_c())
    assert st == 0 and got == want
    assert counts == list(wc)


@pytest.mark.parametrize("scale_m", [2.0, 6.0, 12.0])
def test_close_object_with_many_sub_blocks(ctx, chk, scale_m):
    """A large CLOSE box has rows x cols = (h / 24) x (w / 24) sub-blocks
    (template_match.hpp:189-197): 2.0 m at 12 m gives ~8 x 12, 12 m ~ 27 x 40
    (> 64: the aggregation's global-scratch rank sort); objects, kinds, block
    counts and disparities bit-exact against the reference."""
    sc = S.SceneConfig(width=960, height=640, seed=5, noise_sigma=2.0)
    sc.objects = [S.place(sc, 1, 480, 320, 12.0, width_m=scale_m, height_m=scale_m * 0.7),
                  S.place(sc, 2, 200, 150, 150.0)]
    L, R = S.render_stereo_pair(sc)
    dets = S.ground_truth_detections(sc)
    cfg = rg.RangerConfig(max_objects=8, dx_max_far=128, dx_max_close=128)
    got = rg.estimate_object_disparities(L, R, dets, cfg, focal_px=S.F_PX, baseline_m=S.BASELINE_M, ctx=ctx)
    want, _ = chk.estimate(L, R, [det_c(d) for d in dets], cfg.to_c(), S.F_PX, S.BASELINE_M)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert (g.det_id, g.kind, g.n_blocks_used, g.valid) == (w.det_id, w.kind, w.n_blocks_used, bool(w.valid))
        assert np.float64(g.disparity).tobytes() == np.float64(w.disparity).tobytes()
