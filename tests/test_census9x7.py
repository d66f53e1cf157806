"""9x7 / uint64 census extension (BASELINE config 1).

The reference has no 9x7 transform, so parity is UNPINNED against the
reference itself.  What anchors it instead:
  * a numpy restatement written with the same window convention as the 5x5
    numpy restatement below, which is itself pinned to the reference's 5x5
    codes through the C oracle (golden-pinned in test_oracle_cpu.py);
  * known-answer properties: flat image -> sentinel only, undefined border,
    integer image shifts recovered exactly by the 64-bit matcher.
CPU tests check the oracle; `gpu` tests check the CUDA path bit-exactly
against the oracle (codes, MatchResult bytes, ObjectDisparity records).
"""
import numpy as np
import pytest

from paper_2604_07980_b200 import _abi, synth as S
from paper_2604_07980_b200 import ranger as rg


def census_np(img, ry, rx):
    """Window rows -ry..ry, cols -rx..rx, row-major, bit = neighbour > centre,
    sentinel first (census.hpp:43-56 generalised); 0 where the window leaves."""
    h, w = img.shape
    wide = (2 * ry + 1) * (2 * rx + 1) > 31
    out = np.zeros((h, w), np.uint64 if wide else np.uint32)
    if h <= 2 * ry or w <= 2 * rx:
        return out
    a = img.astype(np.int32)
    c = a[ry:h - ry, rx:w - rx]
    code = np.ones(c.shape, np.uint64)
    for dy in range(-ry, ry + 1):
        for dx in range(-rx, rx + 1):
            nb = a[ry + dy:h - ry + dy, rx + dx:w - rx + dx]
            code = (code << np.uint64(1)) | (nb > c).astype(np.uint64)
    out[ry:h - ry, rx:w - rx] = code
    return out


def rand_img(seed, h, w):
    return np.random.default_rng(seed).integers(0, 256, (h, w), dtype=np.uint8)


def shifted_pair(seed, h, w, d):
    """right(x) = left(x + d): left pixel x is right pixel x - d (dx = d)."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 256, (h, w + d), dtype=np.uint8)
    return np.ascontiguousarray(base[:, :w]), np.ascontiguousarray(base[:, d:])


# ----------------------------------------------------------------- CPU: oracle
def test_numpy_5x5_convention_is_the_pinned_one(orc):
    img = rand_img(3, 40, 57)
    assert np.array_equal(census_np(img, 2, 2), orc.census(img))


@pytest.mark.parametrize("h,w", [(7, 9), (8, 10), (31, 45), (64, 97)])
def test_oracle_census64_matches_numpy(orc, h, w):
    img = rand_img(h * 100 + w, h, w)
    assert np.array_equal(orc.census64(img), census_np(img, 3, 4))


def test_oracle_census64_known_answers(orc):
    flat = np.full((20, 30), 99, np.uint8)
    c = orc.census64(flat)
    assert c[3, 4] == np.uint64(1 << 63) and c[16, 25] == np.uint64(1 << 63)
    assert not c[:3].any() and not c[17:].any() and not c[:, :4].any() and not c[:, 26:].any()
    # one brighter neighbour at (-3, -4): the first compare, bit 62
    img = flat.copy()
    img[5, 6] = 200
    assert orc.census64(img)[8, 10] == np.uint64((1 << 63) | (1 << 62))
    # ... and at (+3, +4): the last compare, bit 0
    img = flat.copy()
    img[11, 14] = 200
    assert orc.census64(img)[8, 10] == np.uint64((1 << 63) | 1)
    # downscaled output samples the full-res codes at the nearest source pixel
    img = rand_img(8, 41, 63)
    full = orc.census64(img)
    red = orc.census64(img, 31, 20)
    mx = [int(np.floor(i * 63 / 31 + 0.5)) for i in range(31)]
    my = [int(np.floor(i * 41 / 20 + 0.5)) for i in range(20)]
    assert np.array_equal(red, full[np.ix_(my, mx)])


def test_oracle_match64_recovers_integer_shift(orc):
    L8, R8 = shifted_pair(5, 60, 120, 17)
    L, R = orc.census64(L8), orc.census64(R8)
    pts = [(x, y) for y in range(10, 50, 6) for x in range(40, 100, 7)]
    st, out = orc.match(L, R, [(pts, (0, 40, -1, 1))], 1)
    assert st == 0 and out[0].has_value and out[0].dx_int == 17 and out[0].dy_int == 0
    assert out[0].cost == 0.0 and out[0].verified


def test_oracle_config0_recovers_known_shifts(orc):
    """BASELINE config 0: 640x480, 8 boxes at known integer disparities, 9x7."""
    sc, cfg = S.scene_c1(seed=1, noise=0.0)
    cfg.census_9x7 = True
    L, R = S.render_stereo_pair(sc)
    dets = S.ground_truth_detections(sc)
    out, st = orc.estimate(L, R, [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets],
                           cfg.to_c())
    truth = {k + 1: d for k, d in enumerate([2, 3, 4, 5, 6, 8, 10, 12])}
    assert len(out) == 8 and all(o.valid for o in out)
    for o in out:
        assert abs(o.disparity - truth[o.det_id]) < 0.25, (o.det_id, o.disparity)


def test_estimate_9x7_rejects_cache(orc):
    sc, cfg = S.scene_c1(seed=1, noise=0.0)
    cfg.census_9x7 = True
    L, R = S.render_stereo_pair(sc)
    dets = [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in S.ground_truth_detections(sc)]
    with pytest.raises(AssertionError):
        orc.estimate(L, R, dets, cfg.to_c(), cache=_abi.CensusCache())


# ----------------------------------------------------------------- GPU parity
@pytest.mark.gpu
@pytest.mark.parametrize("w,h,ow,oh", [(9, 7, 9, 7), (20, 15, 20, 15), (41, 33, 20, 16), (641, 481, 320, 240),
                                       (1920, 1080, 960, 540), (133, 77, 66, 38), (8, 6, 8, 6)])
def test_census64_matches_oracle(ctx, orc, w, h, ow, oh):
    img = rand_img(w * 7 + h, h, w)
    got = rg.census_transform64(img, ow, oh, ctx=ctx).codes
    assert got.dtype == np.uint64
    assert np.array_equal(got, orc.census64(img, ow, oh))


def _same(a, b):
    if a.has_value != b.has_value:
        return False
    if not a.has_value:
        return True
    f = ["dx_int", "dy_int", "valid_points", "verified"]
    d = ["dx_subpix", "cost", "cost_minus", "cost_plus"]
    return all(getattr(a, k) == getattr(b, k) for k in f) and \
        all(np.float64(getattr(a, k)).tobytes() == np.float64(getattr(b, k)).tobytes() for k in d)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_match64_random_protocol(ctx, orc, mode):
    rng = np.random.default_rng(77 + mode)
    bad = 0
    for trial in range(80):
        L = orc.census64(rng.integers(0, 256, (30, 40), dtype=np.uint8))
        R = orc.census64(rng.integers(0, 256, (30, 40), dtype=np.uint8))
        n = int(rng.integers(1, 13))
        pts = [(int(rng.integers(0, 40)), int(rng.integers(0, 30))) for _ in range(n)]
        dxm, dym = int(rng.integers(-3, 3)), int(rng.integers(-2, 1))
        blk = [(pts, (dxm, dxm + int(rng.integers(0, 13)), dym, dym + int(rng.integers(0, 4))))]
        _, want = orc.match(L, R, blk, mode)
        qb = [rg.QueryBlock(list(p), *r) for p, r in blk]
        got = rg._match(qb, rg.CensusImage(40, 30, L), rg.CensusImage(40, 30, R), mode, 1.0, ctx)[0]
        if got is None:
            bad += want[0].has_value
        else:
            bad += not (want[0].has_value and got.dx_int == want[0].dx_int and got.dy_int == want[0].dy_int
                        and np.float64(got.dx_subpix).tobytes() == np.float64(want[0].dx_subpix).tobytes()
                        and np.float64(got.cost).tobytes() == np.float64(want[0].cost).tobytes()
                        and got.valid_points == want[0].valid_points and got.verified == bool(want[0].verified))
    assert bad == 0


@pytest.mark.gpu
def test_match64_integer_shift(ctx):
    L8, R8 = shifted_pair(6, 80, 200, 23)
    L, R = rg.census_transform64(L8, ctx=ctx), rg.census_transform64(R8, ctx=ctx)
    pts = [(x, y) for y in range(10, 70, 5) for x in range(60, 180, 9)]
    m = rg.forward_backward_match(rg.QueryBlock(pts, 0, 64, -2, 2), L, R, 1.0, ctx=ctx)
    assert m is not None and (m.dx_int, m.dy_int, m.cost, m.verified) == (23, 0, 0.0, True)


@pytest.mark.gpu
@pytest.mark.parametrize("name,noise", [("c1", 0.0), ("c1", 2.0), ("c2", 2.0), ("c3", 2.0), ("c3s", 2.0)])
def test_estimate_9x7_matches_oracle(ctx, orc, name, noise):
    fn = {"c1": S.scene_c1, "c2": S.scene_c2, "c3": S.scene_c3,
          "c3s": lambda seed, noise: S.scene_c3(seed, noise, stress=True)}[name]
    sc, cfg = fn(seed=13, noise=noise)
    cfg.census_9x7 = True
    L, R = S.render_stereo_pair(sc)
    dets = S.ground_truth_detections(sc)
    stats = rg.RangerStats()
    got = rg.estimate_object_disparities(L, R, dets, cfg, stats=stats, focal_px=2000.0, baseline_m=0.3, ctx=ctx)
    want, wst = orc.estimate(L, R, [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets],
                             cfg.to_c(), 2000.0, 0.3)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert (g.det_id, g.kind, g.n_blocks_used, g.valid) == (w.det_id, w.kind, w.n_blocks_used, bool(w.valid))
        assert np.float64(g.disparity).tobytes() == np.float64(w.disparity).tobytes()
        assert np.float64(g.z_cam).tobytes() == np.float64(w.z_cam).tobytes()
    assert (stats.query_points, stats.n_far, stats.n_close) == (wst.query_points, wst.n_far, wst.n_close)
    # switching back to 5x5 on the same context re-zeroes the margins
    cfg.census_9x7 = False
    got5 = rg.estimate_object_disparities(L, R, dets, cfg, ctx=ctx)
    want5, _ = orc.estimate(L, R, [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets],
                            cfg.to_c())
    assert [(g.det_id, g.valid, np.float64(g.disparity).tobytes()) for g in got5] == \
        [(w.det_id, bool(w.valid), np.float64(w.disparity).tobytes()) for w in want5]


@pytest.mark.gpu
def test_estimate_9x7_cache_raises(ctx):
    sc, cfg = S.scene_c1(seed=1, noise=0.0)
    cfg.census_9x7 = True
    L, R = S.render_stereo_pair(sc)
    with pytest.raises(rg.InvalidArgument):
        rg.estimate_object_disparities(L, R, S.ground_truth_detections(sc), cfg, cache=rg.CensusCache(), ctx=ctx)
