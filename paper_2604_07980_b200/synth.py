"""Synthetic rectified stereo scenes (input generator for tests and bench).

SceneObject / SceneConfig mirror the reference (synth.hpp:25-52) with the
canonical calibration make_calibration(f, b, cx, cy, h_cam) (geometry.hpp:108-133);
rendering runs the library's bit-exact host port of render_stereo_pair
(synth.hpp:142-230).  The builders below are the BASELINE.json configs as
SURVEY.md 8(d) specifies them (C1..C5).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

from . import _abi
from .ranger import Detection, InvalidArgument, RangerConfig, lib

F_PX, BASELINE_M, H_CAM = 2000.0, 0.30, 1.5


@dataclass
class SceneObject:
    id: int = 0
    position: Tuple[float, float, float] = (0.0, 0.0, 0.0)  # vehicle frame (x fwd, y left, z up), m
    width_m: float = 2.0
    height_m: float = 1.6
    depth_m: float = 4.0
    texture_seed: int = 1
    contrast: float = 60.0
    disparity_ramp: float = 0.0
    class_id: int = 0


@dataclass
class SceneConfig:
    width: int = 640
    height: int = 400
    f: float = F_PX
    b: float = BASELINE_M
    cx: float = -1.0  # < 0: width / 2
    cy: float = -1.0
    h_cam: float = H_CAM
    background_seed: int = 7
    background_contrast: float = 40.0
    vertical_offset_px: int = 0
    disparity_bias_px: float = 0.0
    gain: float = 1.0
    rad_bias: float = 0.0
    gamma: float = 1.0
    noise_sigma: float = 0.0
    seed: int = 1
    texture_quant: int = 1
    texture_cell_px: float = 6.0
    objects: List[SceneObject] = field(default_factory=list)

    def to_c(self):
        cx = self.width / 2.0 if self.cx < 0 else self.cx
        cy = self.height / 2.0 if self.cy < 0 else self.cy
        c = _abi.SceneConfig(self.f, self.b, cx, cy, self.h_cam, self.width, self.height,
                             self.background_seed, self.background_contrast, self.vertical_offset_px,
                             self.texture_quant, self.disparity_bias_px, self.gain, self.rad_bias, self.gamma,
                             self.noise_sigma, self.seed, self.texture_cell_px)
        objs = (_abi.SceneObject * max(len(self.objects), 1))(
            *[_abi.SceneObject(o.id, o.class_id, o.position[0], o.position[1], o.position[2], o.width_m,
                               o.height_m, o.depth_m, o.contrast, o.disparity_ramp, o.texture_seed)
              for o in self.objects])
        return c, objs


def render_stereo_pair(cfg: SceneConfig) -> Tuple[np.ndarray, np.ndarray]:
    """synth.hpp:142-230 -> (left, right) uint8 (H, W)."""
    c, objs = cfg.to_c()
    left = np.zeros((cfg.height, cfg.width), np.uint8)
    right = np.zeros_like(left)
    st = lib().rg_render_stereo_pair(C.byref(c), objs, len(cfg.objects), C.c_void_p(left.ctypes.data),
                                     C.c_void_p(right.ctypes.data), None, None)
    if st != _abi.RG_OK:
        raise InvalidArgument("render_stereo_pair: invalid scene")
    return left, right


def render_frames_device(ctx, cfgs: List[SceneConfig], left, right, frame_stride: int = 0, stream=None) -> None:
    """Device frame source (synth.hpp:142-230 for a batch of scenes, rendered
    in HBM): frame f of `cfgs` lands at byte f * frame_stride of the uint8 CUDA
    tensors `left` / `right` (dense rows; frame_stride defaults to W*H).
    Byte-identical to render_stereo_pair; `stream` is a CUDA stream handle
    (int) or None for the context's stream."""
    if not cfgs:
        raise InvalidArgument("render_frames_device: no scenes")
    w, h = cfgs[0].width, cfgs[0].height
    stride = frame_stride or w * h
    need = (len(cfgs) - 1) * stride + w * h
    for t in (left, right):
        if not t.is_cuda or t.dtype.itemsize != 1 or not t.is_contiguous() or t.numel() < need:
            raise InvalidArgument("render_frames_device: outputs must be contiguous uint8 CUDA tensors "
                                  f"of at least {need} bytes")
    cs, objs, offs = [], [], [0]
    for cfg in cfgs:
        c, o = cfg.to_c()
        cs.append(c)
        objs.extend(o[:len(cfg.objects)])
        offs.append(len(objs))
    carr = (_abi.SceneConfig * len(cs))(*cs)
    oarr = (_abi.SceneObject * max(len(objs), 1))(*objs)
    off = (C.c_int32 * len(offs))(*offs)
    st = lib().rg_render_frames_device(ctx.handle, carr, oarr, off, len(cfgs), C.c_void_p(left.data_ptr()),
                                       C.c_void_p(right.data_ptr()), stride,
                                       C.c_void_p(stream) if stream else None)
    ctx.check(st)


def ground_truth_detections(cfg: SceneConfig) -> List[Detection]:
    """synth.hpp:253-274."""
    c, objs = cfg.to_c()
    out = (_abi.Detection * max(len(cfg.objects), 1))()
    n = C.c_int()
    st = lib().rg_ground_truth_detections(C.byref(c), objs, len(cfg.objects), out, C.byref(n))
    if st != _abi.RG_OK:
        raise InvalidArgument("ground_truth_detections: invalid scene")
    return [Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in out[:n.value]]


def place(cfg: SceneConfig, obj_id: int, u: float, v: float, z: float, **kw) -> SceneObject:
    """Object whose box centre projects to image (u, v) at depth z."""
    cx = cfg.width / 2.0 if cfg.cx < 0 else cfg.cx
    cy = cfg.height / 2.0 if cfg.cy < 0 else cfg.cy
    pos = (z, -(u - cx) * z / cfg.f, cfg.h_cam - (v - cy) * z / cfg.f)
    return SceneObject(id=obj_id, position=pos, texture_seed=100 + obj_id, **kw)


# ---------------------------------------------------------------- BASELINE configs
def scene_c1(seed: int = 1, noise: float = 0.0) -> Tuple[SceneConfig, RangerConfig]:
    """C1: 640x480, 8 boxes at integer disparities on a 4x2 grid (5 FAR + 3 CLOSE)."""
    cfg = SceneConfig(width=640, height=480, seed=seed, noise_sigma=noise)
    for k, d in enumerate([2, 3, 4, 5, 6, 8, 10, 12]):
        z = F_PX * BASELINE_M / d
        cfg.objects.append(place(cfg, k + 1, (k % 4 + 0.5) * 160, (k // 4 + 0.5) * 240, z))
    return cfg, RangerConfig(max_objects=8)


def scene_c2(seed: int = 1, noise: float = 0.0) -> Tuple[SceneConfig, RangerConfig]:
    """C2: 1920x1080, 64 boxes (48 FAR + 16 CLOSE) on an 8x8 grid, dx_max 256."""
    cfg = SceneConfig(width=1920, height=1080, seed=seed, noise_sigma=noise)
    for k in range(64):
        oid = k + 1
        u, v = (k % 8 + 0.5) * 240, (k // 8 + 0.5) * 135
        if oid % 4 == 0:
            z = 40.0 + 2.0 * (oid % 7)
            cfg.objects.append(place(cfg, oid, u, v, z, width_m=0.72 * 240 * z / F_PX,
                                     height_m=0.72 * 135 * z / F_PX))
        else:
            z = 100.0 + 25.0 * (oid % 8)
            cfg.objects.append(place(cfg, oid, u, v, z))
    return cfg, RangerConfig(max_objects=64, dx_max_far=256, dx_max_close=256, tau_v=1.0)


def scene_c3(seed: int = 1, noise: float = 0.0, stress: bool = False) -> Tuple[SceneConfig, RangerConfig]:
    """C3: 2880x1860 on a 16x10 grid of 180x186 px cells: 64 CLOSE boxes and
    96 occluded FAR pairs (256 boxes).  stress=True moves the occluder to
    (+10, +8) so it hides most of each far box."""
    cfg = SceneConfig(width=2880, height=1860, seed=seed, noise_sigma=noise)
    oid = 0
    off = (10.0, 8.0) if stress else (20.0, 16.0)
    for cell in range(160):
        u, v = (cell % 16 + 0.5) * 180, (cell // 16 + 0.5) * 186
        if cell % 5 in (1, 3):
            oid += 1
            z = 40.0 + 2.0 * (oid % 7)
            cfg.objects.append(place(cfg, oid, u, v, z, width_m=0.72 * 180 * z / F_PX,
                                     height_m=0.72 * 186 * z / F_PX))
        else:
            oid += 1
            cfg.objects.append(place(cfg, oid, u, v, 200.0 + 10.0 * (oid % 5)))
            oid += 1
            cfg.objects.append(place(cfg, oid, u + off[0], v + off[1], 120.0))
    return cfg, RangerConfig(max_objects=256, dx_max_far=256, dx_max_close=256)


C4_ROI = (480, 270, 1440, 810)


def c4_bm():
    from .ranger import BmParams
    return BmParams(num_disparities=32, block_size=9, min_disparity=-4, texture_threshold=10,
                    uniqueness_ratio=10, downscale=1)


def scene_c4(offset: int, seed: int = 1) -> SceneConfig:
    """C4: the C2 scene with an injected right-image vertical offset."""
    cfg, _ = scene_c2(seed)
    cfg.vertical_offset_px = offset
    return cfg
