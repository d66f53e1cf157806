"""TEST / BASELINE INFRASTRUCTURE ONLY: the reference arm of bench.py and the
checker of its parity sweep, over oracle/_ref/libranger_ref.so alone.

Nothing here imports paper_2604_07980_b200 or maps libranger_cuda.so: the
reference arm (`bench.py --impl reference`) renders its C2 frames with the
reference's own render_stereo_pair / ground_truth_detections (synth.hpp:142-274)
and ranges them with the reference's estimate_object_disparities
(template_match.hpp:260-363), both compiled in place from /root/reference by
oracle/Makefile.  The ctypes structs restate include/ranger_cuda.h's
rg_scene_config / rg_scene_object / rg_detection / rg_ranger_config /
rg_object_disparity; tests/test_ref_arm.py checks them field for field
against paper_2604_07980_b200/_abi.py and the scenes against synth.scene_c2.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libranger_ref.so")

F_PX, BASELINE_M, H_CAM = 2000.0, 0.30, 1.5
W2, H2 = 1920, 1080


class SceneObject(C.Structure):
    _fields_ = [("id", C.c_int32), ("class_id", C.c_int32), ("px", C.c_double), ("py", C.c_double),
                ("pz", C.c_double), ("width_m", C.c_double), ("height_m", C.c_double),
                ("depth_m", C.c_double), ("contrast", C.c_double), ("disparity_ramp", C.c_double),
                ("texture_seed", C.c_uint64)]


class SceneConfig(C.Structure):
    _fields_ = [
        ("f", C.c_double), ("b", C.c_double), ("cx", C.c_double), ("cy", C.c_double), ("h_cam", C.c_double),
        ("width", C.c_int32), ("height", C.c_int32), ("background_seed", C.c_uint64),
        ("background_contrast", C.c_double), ("vertical_offset_px", C.c_int32), ("texture_quant", C.c_int32),
        ("disparity_bias_px", C.c_double), ("gain", C.c_double), ("rad_bias", C.c_double),
        ("gamma", C.c_double), ("noise_sigma", C.c_double), ("seed", C.c_uint64),
        ("texture_cell_px", C.c_double)]


class RangerConfig(C.Structure):
    _fields_ = [
        ("tau_s", C.c_double), ("close_scale", C.c_int32), ("grid_side_points", C.c_int32),
        ("max_total_points", C.c_int32), ("close_block_side_points", C.c_int32), ("tau_d", C.c_double),
        ("n_min", C.c_int32), ("max_objects", C.c_int32), ("tau_v", C.c_double),
        ("crop_x0", C.c_double), ("crop_y0", C.c_double), ("crop_x1", C.c_double), ("crop_y1", C.c_double),
        ("dx_max_far", C.c_int32), ("dx_max_close", C.c_int32),
        ("census_9x7", C.c_int32), ("reserved", C.c_int32)]


DET_DTYPE = np.dtype([("cx", "<f8"), ("cy", "<f8"), ("w", "<f8"), ("h", "<f8"), ("class_id", "<i4"),
                      ("id", "<i4")])
OUT_DTYPE = np.dtype([("det_id", "<i4"), ("kind", "<i4"), ("n_blocks_used", "<i4"), ("valid", "<i4"),
                      ("disparity", "<f8"), ("z_cam", "<f8")])

_P, _I, _D = C.c_void_p, C.c_int, C.c_double
_lib = None


def have_reference() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(REF_SO)
        _lib.ref_range_frames.restype = _D
        _lib.ref_range_frames.argtypes = [_P, _P, _I, _I, _I, _P, _P, _P, _I, _D, _D, _P, _I, _P]
        _lib.ref_render_frames.restype = _I
        _lib.ref_render_frames.argtypes = [_P, _P, _P, _I, _I, _P, _P, _P, _P]
    return _lib


# ------------------------------------------------------------------ scenes
def _place(w, h, oid, u, v, z, width_m=2.0, height_m=1.6):
    """Object whose box centre projects to (u, v) at depth z (synth.py place)."""
    cx, cy = w / 2.0, h / 2.0
    return SceneObject(oid, 0, z, -(u - cx) * z / F_PX, H_CAM - (v - cy) * z / F_PX, width_m, height_m, 4.0, 60.0,
                       0.0, 100 + oid)


def scene_config(w, h, seed, noise):
    return SceneConfig(F_PX, BASELINE_M, w / 2.0, h / 2.0, H_CAM, w, h, 7, 40.0, 0, 1, 0.0, 1.0, 0.0, 1.0, noise,
                       seed, 6.0)


def scene_c2(seed: int, noise: float = 2.0):
    """C2: 1920x1080, 64 boxes on an 8x8 grid of 240x135 cells; every 4th id
    CLOSE (Z = 40 + 2 (id mod 7), 0.72 of the cell), the rest FAR
    (Z = 100 + 25 (id mod 8), 2.0 x 1.6 m)."""
    objs = []
    for k in range(64):
        oid = k + 1
        u, v = (k % 8 + 0.5) * 240, (k // 8 + 0.5) * 135
        if oid % 4 == 0:
            z = 40.0 + 2.0 * (oid % 7)
            objs.append(_place(W2, H2, oid, u, v, z, 0.72 * 240 * z / F_PX, 0.72 * 135 * z / F_PX))
        else:
            objs.append(_place(W2, H2, oid, u, v, 100.0 + 25.0 * (oid % 8)))
    return scene_config(W2, H2, seed, noise), objs


def ranger_config_c2() -> RangerConfig:
    """RangerConfig defaults (template_match.hpp:33-46) with max_objects 64,
    dx_max_far = dx_max_close = 256, tau_v 1.0."""
    return RangerConfig(48.0, 2, 8, 64, 5, 1.0, 3, 64, 1.0, 0.25, 0.25, 0.75, 0.75, 256, 256, 0, 0)


def render(scenes, threads: int):
    """[(SceneConfig, [SceneObject])] -> (L, R uint8 (n, H, W), dets DET_DTYPE, det offsets int32 (n+1))."""
    n = len(scenes)
    w, h = scenes[0][0].width, scenes[0][0].height
    cfgs = (SceneConfig * n)(*[s[0] for s in scenes])
    flat = [o for s in scenes for o in s[1]]
    objs = (SceneObject * max(len(flat), 1))(*flat)
    offs = np.zeros(n + 1, np.int32)
    offs[1:] = np.cumsum([len(s[1]) for s in scenes])
    L = np.zeros((n, h, w), np.uint8)
    R = np.zeros_like(L)
    dets = np.zeros(max(len(flat), 1), DET_DTYPE)
    nd = np.zeros(n, np.int32)
    st = lib().ref_render_frames(C.addressof(cfgs), C.addressof(objs), offs.ctypes.data, n, threads,
                                 L.ctypes.data, R.ctypes.data, dets.ctypes.data, nd.ctypes.data)
    if st != 0:
        raise RuntimeError(f"ref_render_frames failed ({st})")
    if not np.array_equal(nd, np.diff(offs)):  # ground_truth_detections keeps every in-view object here
        keep = np.concatenate([np.arange(offs[f], offs[f] + nd[f]) for f in range(n)])
        dets = dets[keep]
        offs = np.concatenate([[0], np.cumsum(nd)]).astype(np.int32)
    return L, R, dets[:offs[-1]], offs


def range_frames(L, R, dets, offs, cfg: RangerConfig, threads: int, out_stride: int,
                 focal: float = F_PX, baseline: float = BASELINE_M):
    """Reference estimate_object_disparities, frame-parallel on `threads`
    host threads -> (seconds, records OUT_DTYPE (n, out_stride), counts)."""
    n, h, w = L.shape
    L, R = np.ascontiguousarray(L), np.ascontiguousarray(R)
    out = np.zeros(n * out_stride, OUT_DTYPE)
    cnt = np.zeros(n, np.int32)
    dets = np.ascontiguousarray(dets, DET_DTYPE)
    offs = np.ascontiguousarray(offs, np.int32)
    secs = lib().ref_range_frames(L.ctypes.data, R.ctypes.data, w, h, n, dets.ctypes.data, offs.ctypes.data,
                                  C.byref(cfg), threads, focal, baseline, out.ctypes.data, out_stride,
                                  cnt.ctypes.data)
    return secs, out.reshape(n, out_stride), cnt


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    """lscpu 'Model name', else /proc/cpuinfo."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"
