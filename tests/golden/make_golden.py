#!/usr/bin/env python
"""Generate tests/golden/golden.json from the REFERENCE ITSELF.

Runs the reference's header-only implementation compiled in place
(oracle/_ref/libranger_ref.so, built by oracle/Makefile from
/root/reference/proj/include) on seeded inputs and records its outputs:
census hashes, MatchResults of the test_matching.cpp random protocol,
ObjectDisparity lists of the C1/C2/C3 scenes, BM raw-map hashes and the
auto-rect delta* + per-delta counts.  Inputs are either numpy-seeded random
images or frames rendered by the reference renderer (whose byte hashes are
recorded too, pinning this repo's renderer).  The committed JSON is what the
CPU tests check the C oracle (and the GPU tests check the CUDA path) against
on machines without /root/reference.

    python tests/golden/make_golden.py      # needs oracle/_ref
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_lib  # noqa: E402
from paper_2604_07980_b200 import _abi  # noqa: E402
from paper_2604_07980_b200 import synth as S  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rand_img(seed, h, w):
    return np.random.default_rng(seed).integers(0, 256, (h, w), dtype=np.uint8)


def match_rec(m):
    return [m.has_value, m.dx_int, m.dy_int, m.dx_subpix.hex(), m.cost.hex(), m.cost_minus.hex(),
            m.cost_plus.hex(), m.valid_points, m.verified] if m.has_value else [0]


def od_rec(o):
    return [o.det_id, o.kind, o.n_blocks_used, o.valid, o.disparity.hex(), o.z_cam.hex()]


def ref_render(ref, sc):
    c, objs = sc.to_c()
    L = np.zeros((sc.height, sc.width), np.uint8)
    R = np.zeros_like(L)
    assert ref.lib.ref_render_stereo_pair(C.byref(c), objs, len(sc.objects), L.ctypes.data, R.ctypes.data) == 0
    return L, R


def ref_dets(ref, sc):
    c, objs = sc.to_c()
    out = (_abi.Detection * max(len(sc.objects), 1))()
    n = C.c_int()
    assert ref.lib.ref_ground_truth_detections(C.byref(c), objs, len(sc.objects), out, C.byref(n)) == 0
    return list(out[:n.value])


def main():
    ref = oracle_lib.reference()
    g = {"source": "reference compiled in place (oracle/_ref/libranger_ref.so)"}
    # census
    cen = []
    for (seed, w, h, ow, oh) in [(3, 20, 15, 20, 15), (17, 41, 33, 20, 16), (23, 64, 48, 64, 48),
                                 (5, 641, 481, 320, 240), (8, 133, 77, 66, 38)]:
        img = rand_img(seed, h, w)
        cen.append({"seed": seed, "w": w, "h": h, "ow": ow, "oh": oh, "sha": sha(ref.census(img, ow, oh))})
    rois = [(4, 4, 20, 16), (10, 12, 30, 24), (40, 30, 48, 36), (-3, -2, 5, 4), (30, 1, 20, 9)]
    img = rand_img(31, 36, 48)
    g["census"] = cen
    g["census_rois"] = {"seed": 31, "w": 48, "h": 36, "rois": rois,
                        "sha_full": sha(ref.census_rois(img, 48, 36, rois)),
                        "sha_half": sha(ref.census_rois(img, 24, 18, rois))}
    # matcher: test_matching.cpp:78-108 protocol on numpy-seeded inputs
    rng = np.random.default_rng(99)
    trials = []
    for t in range(120):
        s1, s2 = int(rng.integers(1 << 30)), int(rng.integers(1 << 30))
        n = int(rng.integers(1, 13))
        pts = [(int(rng.integers(0, 40)), int(rng.integers(0, 30))) for _ in range(n)]
        dxm, dym = int(rng.integers(-3, 3)), int(rng.integers(-2, 1))
        r = (dxm, dxm + int(rng.integers(0, 13)), dym, dym + int(rng.integers(0, 4)))
        L, R = ref.census(rand_img(s1, 30, 40)), ref.census(rand_img(s2, 30, 40))
        recs = []
        for mode in (0, 1):
            st, out = ref.match(L, R, [(pts, r)], mode)
            recs.append(match_rec(out[0]))
        trials.append({"s1": s1, "s2": s2, "pts": pts, "range": r, "fwd": recs[0], "fb": recs[1]})
    g["match"] = trials
    # scenes
    scenes = {}
    for name, fn, kw in [("c1", S.scene_c1, {}), ("c2", S.scene_c2, {}), ("c3", S.scene_c3, {}),
                         ("c3_stress", S.scene_c3, {"stress": True})]:
        for noise in (0.0, 2.0):
            sc, cfg = fn(seed=5, noise=noise, **kw)
            L, R = ref_render(ref, sc)
            dets = ref_dets(ref, sc)
            out, st = ref.estimate(L, R, dets, cfg.to_c(), S.F_PX, S.BASELINE_M)
            scenes[f"{name}_n{noise:g}"] = {
                "scene": name, "seed": 5, "noise": noise, "stress": kw.get("stress", False),
                "sha_left": sha(L), "sha_right": sha(R),
                "dets": [[d.cx.hex(), d.cy.hex(), d.w.hex(), d.h.hex(), d.class_id, d.id] for d in dets],
                "out": [od_rec(o) for o in out],
                "stats": [st.query_points, st.image_pixels, st.n_far, st.n_close]}
    g["scenes"] = scenes
    # BM
    bm = []
    for (seed, nd, bs, dmin, ds, tex, uniq) in [(100, 12, 5, 0, 1, 10, 10), (101, 12, 5, 3, 1, 10, 10),
                                                (102, 16, 9, 0, 1, 0, 0), (103, 24, 9, -4, 1, 10, 10),
                                                (104, 9, 5, 2, 2, 0, 0), (105, 40, 7, -5, 1, 0, 15)]:
        a, b = rand_img(seed, 28, 48), rand_img(seed + 1000, 28, 48)
        p = _abi.BmParams(nd, bs, dmin, ds, float(tex), float(uniq))
        st, raw = ref.bm(a, b, p)
        bm.append({"seed": seed, "params": [nd, bs, dmin, ds, tex, uniq], "sha": sha(raw),
                   "n_valid": int((raw != -32768).sum())})
    g["bm"] = bm
    # autorect
    ar = []
    for voff in (-3, 0, 2):
        sc = S.SceneConfig(objects=[S.SceneObject(id=1, position=(30.0, 0.0, 1.5), texture_seed=11)],
                           vertical_offset_px=voff)
        L, R = ref_render(ref, sc)
        st, best, counts = ref.autorect(L, R, (240, 160, 400, 240), -3, 3, _abi.BmParams(24, 9, 0, 1, 10.0, 10.0))
        ar.append({"voff": voff, "sha_left": sha(L), "sha_right": sha(R), "best": best,
                   "counts": [int(c) for c in counts]})
    g["autorect"] = ar
    g["sgm"] = sgm_section(ref)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", os.path.join(HERE, "golden.json"))


SGM_CASES = [(200, 40, 24, 16, 0, 8, 32), (201, 33, 17, 8, -3, 0, 0), (202, 64, 20, 24, 2, 3, 50),
             (203, 16, 12, 40, 0, 10, 10), (204, 90, 7, 32, -8, 8, 32)]


def sgm_section(ref):
    """sgm_disparity of the reference on seeded random pairs: raw-map hashes."""
    out = []
    for (seed, w, h, nd, d_lo, p1, p2) in SGM_CASES:
        a, b = rand_img(seed, h, w), rand_img(seed + 1000, h, w)
        raw = np.zeros((h, w), np.int16)
        assert ref.lib.ref_sgm_disparity(a.ctypes.data, b.ctypes.data, w, h, nd, d_lo, p1, p2, raw.ctypes.data) == 0
        out.append({"seed": seed, "w": w, "h": h, "params": [nd, d_lo, p1, p2], "sha": sha(raw),
                    "n_valid": int((raw != -32768).sum())})
    return out


if __name__ == "__main__":
    if sys.argv[1:] == ["--only", "sgm"]:  # add/refresh just the SGM section
        path = os.path.join(HERE, "golden.json")
        g = json.load(open(path))
        g["sgm"] = sgm_section(oracle_lib.reference())
        with open(path, "w") as f:
            json.dump(g, f, indent=0)
        print("updated sgm in", path)
    else:
        main()
