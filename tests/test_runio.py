"""Run-directory and record formats: io.hpp / pgm.hpp /
pipeline.hpp:346-406 restated in paper_2604_07980_b200/runio.py.

CPU: a run directory written by the reference (make_synthetic_frames +
save_synthetic_run) loads into the same frames / detections / radar, and
re-saving reproduces its files byte for byte; the reference's pipeline
outputs over that run round-trip byte for byte.  GPU: runio.run_directory
(device frame loop + records) writes objects.txt / depth.txt / refiners.txt
identical to the reference CLI path's.
"""
import os

import numpy as np
import pytest

import oracle_lib
from paper_2604_07980_b200 import ranger as rg, runio, synth as S

N_FRAMES = 4


def scene():
    sc, cfg = S.scene_c1(seed=5, noise=2.0)
    sc.disparity_bias_px = 0.6
    for k, o in enumerate(sc.objects):
        o.class_id = k % 3
    return sc, cfg


@pytest.fixture(scope="module")
def ref():
    try:
        return oracle_lib.reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built here")


@pytest.fixture(scope="module")
def run_dir(ref, tmp_path_factory):
    d = str(tmp_path_factory.mktemp("run"))
    sc, _ = scene()
    c, objs = sc.to_c()
    assert ref.lib.ref_save_synthetic_run(C_ref(c), C_ref(objs), len(sc.objects), N_FRAMES, 0.1, d.encode()) == 0
    return d


def C_ref(x):
    import ctypes
    return ctypes.byref(x)


@pytest.fixture(scope="module")
def ref_out(ref, run_dir, tmp_path_factory):
    out = str(tmp_path_factory.mktemp("out"))
    _, cfg = scene()
    rect = rg.RectSearchConfig()
    assert ref.lib.ref_run_directory(run_dir.encode(), out.encode(), C_ref(cfg.to_c()), C_ref(rect.to_c()), 1,
                                     0.5) == 0
    return out


def read(path):
    return open(path, "rb").read()


def test_reference_run_loads_and_resaves_byte_identical(run_dir, tmp_path):
    sc, _ = scene()
    frames = runio.load_run_directory(run_dir)
    assert [f.frame_id for f in frames] == list(range(N_FRAMES))
    for f in frames:  # make_synthetic_frames: scene.seed = base + frame
        s2, _ = scene()
        s2.seed = sc.seed + f.frame_id
        L, R = S.render_stereo_pair(s2)
        assert np.array_equal(f.left, L) and np.array_equal(f.right, R)
        assert len(f.detections) == len(sc.objects) and f.radar.shape == (len(sc.objects), 3)
    dets = runio.load_detections(os.path.join(run_dir, "detections.txt"))
    runio.save_detections(dets, str(tmp_path / "d.txt"))
    assert read(tmp_path / "d.txt") == read(os.path.join(run_dir, "detections.txt"))
    radar = runio.load_radar_records(os.path.join(run_dir, "radar.txt"))
    runio.save_radar_records(radar, str(tmp_path / "r.txt"))
    assert read(tmp_path / "r.txt") == read(os.path.join(run_dir, "radar.txt"))
    runio.save_pgm(frames[1].left, str(tmp_path / "l.pgm"))
    assert read(tmp_path / "l.pgm") == read(os.path.join(run_dir, runio.frame_image_name("left", 1)))
    cal = runio.load_calibration(os.path.join(run_dir, "calib.txt")).to_c()
    assert (cal.f, cal.b, cal.h_cam) == (sc.f, sc.b, sc.h_cam) and list(cal.R) == [0, 0, 1, -1, 0, 0, 0, -1, 0]


def test_reference_outputs_round_trip(ref_out, tmp_path):
    objs = runio.load_object_records(os.path.join(ref_out, "objects.txt"))
    depth = runio.load_depth_records(os.path.join(ref_out, "depth.txt"))
    logs = runio.load_refiner_log(os.path.join(ref_out, "refiners.txt"))
    assert len(objs) == len(depth) > 0 and len(logs) == N_FRAMES
    assert {d.source for d in depth} and any(not np.isnan(d.clp_by_gpt) for d in depth)
    runio.save_pipeline_outputs(objs, depth, logs, str(tmp_path))
    for name in ("objects.txt", "depth.txt", "refiners.txt"):
        assert read(tmp_path / name) == read(os.path.join(ref_out, name)), name


def test_disparity_pgm_and_errors(tmp_path):
    raw = np.array([[-32768, -1, 0], [16, 32767, -16]], np.int16)
    runio.save_disparity_pgm(raw, str(tmp_path / "d.pgm"))
    assert np.array_equal(runio.load_disparity_pgm(str(tmp_path / "d.pgm")), raw)
    assert read(tmp_path / "d.pgm")[:15] == b"P5\n3 2\n65535\n\x00\x00"
    (tmp_path / "c.pgm").write_bytes(b"P5\n# comment\n2 1\n255\n\x07\x09")
    assert runio.load_pgm(str(tmp_path / "c.pgm")).tolist() == [[7, 9]]
    (tmp_path / "t.pgm").write_bytes(b"P5\n2 2\n255\n\x07")
    with pytest.raises(RuntimeError, match="truncated"):
        runio.load_pgm(str(tmp_path / "t.pgm"))
    (tmp_path / "bad.txt").write_text("0 1 FAR 1.0 1\n")
    with pytest.raises(RuntimeError, match="load_object_records: bad line"):
        runio.load_object_records(str(tmp_path / "bad.txt"))
    (tmp_path / "bad2.txt").write_text("# header\n\nx 0.5 1.0 2.0\n")
    with pytest.raises(RuntimeError, match="load_refiner_log: bad integer 'x'"):
        runio.load_refiner_log(str(tmp_path / "bad2.txt"))
    (tmp_path / "bad3.txt").write_text("0 1.5e q 2.0\n")
    with pytest.raises(RuntimeError, match="load_refiner_log: bad number '1.5e'"):
        runio.load_refiner_log(str(tmp_path / "bad3.txt"))
    assert runio.fmt6(float("nan")) == "nan" and runio.fmt6(-0.0) == "-0.000000" and runio.fmt6(2.5e-7) == "0.000000"


@pytest.mark.gpu
def test_run_directory_outputs_match_reference(ctx, run_dir, ref_out, tmp_path):
    from paper_2604_07980_b200.engine import FrameEngine

    sc, cfg = scene()
    frames = runio.load_run_directory(run_dir)
    eng = FrameEngine(sc.width, sc.height, cfg, max(len(f.detections) for f in frames), ctx=ctx)
    params = rg.RecordParams(runio.load_calibration(os.path.join(run_dir, "calib.txt")))
    runio.run_directory(eng, run_dir, str(tmp_path), params, rect=rg.RectSearchConfig())
    for name in ("objects.txt", "depth.txt", "refiners.txt"):
        assert read(tmp_path / name) == read(os.path.join(ref_out, name)), name
