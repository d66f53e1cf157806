"""CPU: the reference arm's standalone restatements (oracle/ref_arm.py) agree
with the product's ABI structs and scene builders, and the reference's own
renderer driven through them produces the frames the GPU arm ranges."""
import ctypes as C
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import ref_arm  # noqa: E402

from paper_2604_07980_b200 import _abi, synth as S  # noqa: E402
from paper_2604_07980_b200.engine import DET_DTYPE, OUT_DTYPE, pack_detections  # noqa: E402


@pytest.mark.parametrize("name", ["SceneObject", "SceneConfig", "RangerConfig"])
def test_struct_layouts_match_abi(name):
    a, b = getattr(ref_arm, name), getattr(_abi, name)
    assert C.sizeof(a) == C.sizeof(b)
    assert [(f[0], f[1]) for f in a._fields_] == [(f[0], f[1]) for f in b._fields_]


def test_dtypes_match_engine():
    assert ref_arm.DET_DTYPE == DET_DTYPE and ref_arm.OUT_DTYPE == OUT_DTYPE


def test_c2_scene_and_config_match_synth():
    for seed in (1, 17):
        sc, cfg = S.scene_c2(seed=seed, noise=2.0)
        c, objs = sc.to_c()
        rc, robjs = ref_arm.scene_c2(seed, 2.0)
        assert bytes(c) == bytes(rc)
        assert len(robjs) == len(sc.objects)
        assert all(bytes(objs[i]) == bytes(robjs[i]) for i in range(len(robjs)))
        assert bytes(cfg.to_c()) == bytes(ref_arm.ranger_config_c2())


@pytest.mark.skipif(not ref_arm.have_reference(), reason="oracle/_ref not built")
def test_reference_render_equals_product_render_and_detections():
    scenes = [ref_arm.scene_c2(s, 2.0) for s in (1, 2)]
    L, R, dets, offs = ref_arm.render(scenes, threads=2)
    for f, seed in enumerate((1, 2)):
        sc, _ = S.scene_c2(seed=seed, noise=2.0)
        l, r = S.render_stereo_pair(sc)
        assert np.array_equal(L[f], l) and np.array_equal(R[f], r)
        recs, o = pack_detections([S.ground_truth_detections(sc)])
        assert dets[offs[f]:offs[f + 1]].tobytes() == recs.tobytes()
