"""CPU: pin the C oracle (test infrastructure) to the reference.

1. against tests/golden/golden.json, generated from the reference itself
   (oracle/_ref, tests/golden/make_golden.py) -- runs everywhere;
2. against oracle/_ref directly on fresh seeded inputs when it was built.
Also pins this repo's renderer (the input generator) to the reference's.
"""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

import oracle_lib
from paper_2604_07980_b200 import _abi, synth as S

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rand_img(seed, h, w):
    return np.random.default_rng(seed).integers(0, 256, (h, w), dtype=np.uint8)


def match_rec(m):
    return [m.has_value, m.dx_int, m.dy_int, m.dx_subpix.hex(), m.cost.hex(), m.cost_minus.hex(),
            m.cost_plus.hex(), m.valid_points, m.verified] if m.has_value else [0]


def od_rec(o):
    return [o.det_id, o.kind, o.n_blocks_used, o.valid, o.disparity.hex(), o.z_cam.hex()]


def scene_of(rec):
    fn = {"c1": S.scene_c1, "c2": S.scene_c2, "c3": S.scene_c3, "c3_stress": S.scene_c3}[rec["scene"]]
    kw = {"stress": True} if rec["stress"] else {}
    return fn(seed=rec["seed"], noise=rec["noise"], **kw)


def test_census_anchor(orc):  # test_census.cpp:35-40
    img = np.zeros((9, 9), np.uint8)
    img[2:7, 2:7] = [[48, 72, 35, 91, 63], [85, 57, 44, 68, 29], [61, 93, 55, 37, 76], [42, 66, 81, 50, 88],
                     [73, 38, 59, 94, 46]]
    assert orc.census(img)[4, 4] == 0x2BD65B6


@pytest.mark.parametrize("rec", GOLDEN["census"], ids=lambda r: f"{r['w']}x{r['h']}->{r['ow']}x{r['oh']}")
def test_oracle_census_golden(orc, rec):
    img = rand_img(rec["seed"], rec["h"], rec["w"])
    assert sha(orc.census(img, rec["ow"], rec["oh"])) == rec["sha"]


def test_oracle_census_rois_golden(orc):
    g = GOLDEN["census_rois"]
    img = rand_img(g["seed"], g["h"], g["w"])
    rois = [tuple(r) for r in g["rois"]]
    assert sha(orc.census_rois(img, 48, 36, rois)) == g["sha_full"]
    assert sha(orc.census_rois(img, 24, 18, rois)) == g["sha_half"]


def test_oracle_match_golden(orc):  # test_matching.cpp:78-108 protocol
    for t in GOLDEN["match"]:
        L, R = orc.census(rand_img(t["s1"], 30, 40)), orc.census(rand_img(t["s2"], 30, 40))
        blk = [([tuple(p) for p in t["pts"]], tuple(t["range"]))]
        for mode, key in ((0, "fwd"), (1, "fb")):
            st, out = orc.match(L, R, blk, mode)
            assert st == 0 and match_rec(out[0]) == t[key]


@pytest.mark.parametrize("key", sorted(GOLDEN["scenes"]))
def test_renderer_and_oracle_scenes_golden(orc, key):
    rec = GOLDEN["scenes"][key]
    sc, cfg = scene_of(rec)
    L, R = S.render_stereo_pair(sc)  # this repo's renderer == the reference renderer
    assert sha(L) == rec["sha_left"] and sha(R) == rec["sha_right"]
    dets = S.ground_truth_detections(sc)
    assert [[d.cx.hex(), d.cy.hex(), d.w.hex(), d.h.hex(), d.class_id, d.id] for d in dets] == rec["dets"]
    out, st = orc.estimate(L, R, [_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets],
                           cfg.to_c(), S.F_PX, S.BASELINE_M)
    assert [od_rec(o) for o in out] == rec["out"]
    assert [st.query_points, st.image_pixels, st.n_far, st.n_close] == rec["stats"]


def test_scene_facts():
    """SURVEY.md 8(d) facts about the configs, recomputed."""
    assert GOLDEN["scenes"]["c2_n0"]["stats"][0] == 14272
    assert GOLDEN["scenes"]["c3_n0"]["stats"][0] == 51614
    assert GOLDEN["scenes"]["c1_n0"]["stats"][0] == 670
    assert all(o[3] == 1 for o in GOLDEN["scenes"]["c2_n0"]["out"])  # 64/64 valid
    assert sum(o[3] for o in GOLDEN["scenes"]["c3_stress_n2"]["out"]) < 256  # stress has invalid boxes


@pytest.mark.parametrize("rec", GOLDEN["bm"], ids=lambda r: str(r["params"]))
def test_oracle_bm_golden(orc, rec):
    a, b = rand_img(rec["seed"], 28, 48), rand_img(rec["seed"] + 1000, 28, 48)
    nd, bs, dmin, ds, tex, uniq = rec["params"]
    st, raw = orc.bm(a, b, _abi.BmParams(nd, bs, dmin, ds, float(tex), float(uniq)))
    assert st == 0 and sha(raw) == rec["sha"]


@pytest.mark.parametrize("rec", GOLDEN["autorect"], ids=lambda r: f"voff{r['voff']}")
def test_oracle_autorect_golden(orc, rec):
    sc = S.SceneConfig(objects=[S.SceneObject(id=1, position=(30.0, 0.0, 1.5), texture_seed=11)],
                       vertical_offset_px=rec["voff"])
    L, R = S.render_stereo_pair(sc)
    assert sha(L) == rec["sha_left"] and sha(R) == rec["sha_right"]
    st, best, counts = orc.autorect(L, R, (240, 160, 400, 240), -3, 3, _abi.BmParams(24, 9, 0, 1, 10.0, 10.0))
    assert best == rec["best"] == rec["voff"] and list(counts) == rec["counts"]


@pytest.mark.skipif(not oracle_lib.have_reference(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_equals_reference_fresh_inputs(orc):
    ref = oracle_lib.reference()
    rng = np.random.default_rng(2024)
    for _ in range(60):
        L = orc.census(rand_img(int(rng.integers(1 << 30)), 30, 40))
        R = orc.census(rand_img(int(rng.integers(1 << 30)), 30, 40))
        n = int(rng.integers(0, 20))
        pts = [(int(rng.integers(-3, 43)), int(rng.integers(-3, 33))) for _ in range(n)]
        dxm, dym = int(rng.integers(-6, 4)), int(rng.integers(-3, 1))
        blk = [(pts, (dxm, dxm + int(rng.integers(0, 20)), dym, dym + int(rng.integers(0, 5))))]
        for mode in (0, 1):
            a, b = orc.match(L, R, blk, mode), ref.match(L, R, blk, mode)
            assert a[0] == b[0] and bytes(a[1][0]) == bytes(b[1][0])
    # object ranger on randomised detection sets (occlusion + selection budget)
    sc, cfg = S.scene_c1(seed=9, noise=2.0)
    L, R = S.render_stereo_pair(sc)
    for t in range(6):
        dets = []
        for k in range(int(rng.integers(1, 20))):
            w, h = float(rng.uniform(0.01, 0.3)), float(rng.uniform(0.01, 0.3))
            dets.append(_abi.Detection(float(rng.uniform(w / 2, 1 - w / 2)), float(rng.uniform(h / 2, 1 - h / 2)),
                                       w, h, 0, int(rng.integers(0, 5))))
        cfg.max_objects = int(rng.integers(0, 20))
        a, sa = orc.estimate(L, R, dets, cfg.to_c())
        b, sb = ref.estimate(L, R, dets, cfg.to_c())
        assert [bytes(x) for x in a] == [bytes(y) for y in b]
        assert bytes(sa) == bytes(sb)


@pytest.mark.parametrize("rec", GOLDEN["sgm"], ids=lambda r: f"sgm{r['params']}")
def test_oracle_sgm_golden(orc, rec):  # sgm.hpp:118-155 pinned to the reference's outputs
    a, b = rand_img(rec["seed"], rec["h"], rec["w"]), rand_img(rec["seed"] + 1000, rec["h"], rec["w"])
    nd, d_lo, p1, p2 = rec["params"]
    raw = orc.sgm(a, b, nd, d_lo, p1, p2)
    assert sha(raw) == rec["sha"] and int((raw != -32768).sum()) == rec["n_valid"]


def test_oracle_sgm_pass_equals_reference_fresh(orc):
    if not oracle_lib.have_reference():
        pytest.skip("oracle/_ref not built here")
    ref = oracle_lib.reference()
    rng = np.random.default_rng(7)
    for (w, h, nd, p1, p2) in [(17, 9, 12, 3, 20), (8, 23, 40, 0, 5), (31, 5, 33, 7, 7)]:
        cost = rng.integers(0, 28, (h, w, nd), dtype=np.uint8)
        for sx, sy in [(1, 0), (0, 1), (1, 1), (-1, 1), (-1, 0), (0, -1), (1, -1), (-1, -1)]:
            acc0 = rng.integers(-5, 5, (h, w, nd)).astype(np.int32)
            a1, a2 = acc0.copy(), acc0.copy()
            assert orc.lib.orc_sgm_direction_pass(cost.ctypes.data, w, h, nd, p1, p2, sx, sy, a1.ctypes.data) == 0
            assert ref.lib.ref_sgm_direction_pass(cost.ctypes.data, w, h, nd, p1, p2, sx, sy, a2.ctypes.data) == 0
            assert np.array_equal(a1, a2), (w, h, nd, sx, sy)


@pytest.mark.skipif(not oracle_lib.have_reference(), reason="oracle/_ref not built (no /root/reference)")
def test_reference_autorect_mt_equals_single_worker(orc):
    """The multi-threaded reference checker of the full-ROI C4 GPU test equals
    the reference at workers = 1 and the restatement (autorect.hpp:22-58)."""
    from paper_2604_07980_b200 import synth as S
    from paper_2604_07980_b200.ranger import BmParams
    sc = S.SceneConfig(objects=[S.SceneObject(id=1, position=(30.0, 0.0, 1.5), texture_seed=11)],
                       vertical_offset_px=2)
    L, R = S.render_stereo_pair(sc)
    p = BmParams(24, 9, 0, 10, 10, 1).to_c()
    roi = (240, 160, 400, 240)
    ref = oracle_lib.checker()
    a = ref.autorect_mt(L, R, roi, -3, 3, p, 4)
    b = ref.ref.autorect(L, R, roi, -3, 3, p)
    c = orc.autorect(L, R, roi, -3, 3, p)
    assert a[0] == b[0] == c[0] == 0 and a[1] == b[1] == c[1] == 2
    assert list(a[2]) == list(b[2]) == list(c[2])
