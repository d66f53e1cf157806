"""Run-directory and record-file formats.

The line-delimited record files and 8-bit P5 frames the reference's pipeline
stages exchange (io.hpp, pgm.hpp, pipeline.hpp:346-398), so runs recorded
for (or by) the reference CLI feed this implementation and its outputs diff
byte-for-byte against the reference's.  Floats are written as C's "%.6f"
(io.hpp:25-30; Python's %-formatting rounds the exact binary value the same
way glibc printf does), "nan" for NaN.

Loaders skip blank and '#' lines and reject lines with the wrong token count
with the reference's messages (RuntimeError).
"""
from __future__ import annotations

import math
import os
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .ranger import DEPTH_SOURCES, Detection

KIND_NAMES = {_abi.RG_KIND_FAR: "FAR", _abi.RG_KIND_CLOSE: "CLOSE"}  # io.hpp:91-99


def fmt6(v: float) -> str:  # io.hpp:25-30
    return "nan" if math.isnan(v) else "%.6f" % v


def _tokens(path: str, what: str, n: int):
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"{what}: cannot open {path}") from None
    with f:
        for line in f:
            t = line.split()
            if not t or t[0][0] == "#":
                continue
            if len(t) != n:
                raise RuntimeError(f"{what}: bad line: {line.rstrip(chr(10))}")
            yield t


def _int(tok: str, what: str) -> int:  # io.hpp:51-60 (std::stoi, whole token)
    if not re.fullmatch(r"\s*[+-]?\d+", tok):
        raise RuntimeError(f"{what}: bad integer '{tok}'")
    v = int(tok)
    if not -2**31 <= v < 2**31:
        raise RuntimeError(f"{what}: bad integer '{tok}'")
    return v


def _float(tok: str, what: str) -> float:  # io.hpp:40-49 (std::stod, whole token)
    try:
        return float(tok)
    except ValueError:
        raise RuntimeError(f"{what}: bad number '{tok}'") from None


def _write(path: str, what: str, lines: Sequence[str]) -> None:
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError(f"{what}: cannot open {path}") from None
    with f:
        f.write("".join(lines))


# ---------------------------------------------------------------- detections
def save_detections(recs: Sequence[Tuple[int, Detection]], path: str) -> None:  # io.hpp:109-116
    _write(path, "save_detections", [f"{fid} {d.id} {d.class_id} {fmt6(d.cx)} {fmt6(d.cy)} {fmt6(d.w)} {fmt6(d.h)}\n"
                                     for fid, d in recs])


def load_detections(path: str) -> List[Tuple[int, Detection]]:  # io.hpp:118-138
    w = "load_detections"
    return [(_int(t[0], w), Detection(_float(t[3], w), _float(t[4], w), _float(t[5], w), _float(t[6], w),
                                      _int(t[2], w), _int(t[1], w))) for t in _tokens(path, w, 7)]


# ---------------------------------------------------------------- objects
def save_object_records(recs: Sequence[Tuple[int, object]], path: str) -> None:  # io.hpp:148-155
    """recs: (frame_id, record with det_id / kind / disparity / valid / n_blocks_used)."""
    def g(o, k):
        return o[k] if isinstance(o, np.void) else getattr(o, k)
    _write(path, "save_object_records",
           [f"{fid} {int(g(o, 'det_id'))} {KIND_NAMES[int(g(o, 'kind'))]} {fmt6(float(g(o, 'disparity')))} "
            f"{1 if g(o, 'valid') else 0} {int(g(o, 'n_blocks_used'))}\n" for fid, o in recs])


def load_object_records(path: str) -> List[Tuple[int, _abi.ObjectDisparity]]:  # io.hpp:157-178
    w = "load_object_records"
    kinds = {v: k for k, v in KIND_NAMES.items()}
    out = []
    for t in _tokens(path, w, 6):
        if t[2] not in kinds:
            raise RuntimeError(f"unknown object kind '{t[2]}'")
        o = _abi.ObjectDisparity(_int(t[1], w), kinds[t[2]], _int(t[5], w), int(_int(t[4], w) != 0),
                                 _float(t[3], w), 0.0)
        out.append((_int(t[0], w), o))
    return out


# ---------------------------------------------------------------- radar
def save_radar_records(recs: Sequence[Tuple[int, Sequence[float], Sequence[float]]], path: str) -> None:
    """io.hpp:187-196: (frame_id, position xyz, extent xyz)."""
    _write(path, "save_radar_records", [f"{fid} " + " ".join(fmt6(float(v)) for v in (*p, *e)) + "\n"
                                        for fid, p, e in recs])


def load_radar_records(path: str) -> List[Tuple[int, np.ndarray, np.ndarray]]:  # io.hpp:198-221
    w = "load_radar_records"
    return [(_int(t[0], w), np.array([_float(x, w) for x in t[1:4]]), np.array([_float(x, w) for x in t[4:7]]))
            for t in _tokens(path, w, 7)]


# ---------------------------------------------------------------- refiner log
def save_refiner_log(recs: Sequence[_abi.RefinerLog], path: str) -> None:  # io.hpp:232-238
    _write(path, "save_refiner_log", [f"{r.frame_id} {fmt6(r.rect_delta)} {fmt6(r.radar_offset)} "
                                      f"{fmt6(r.obj_offset)}\n" for r in recs])


def load_refiner_log(path: str) -> List[_abi.RefinerLog]:  # io.hpp:240-258
    w = "load_refiner_log"
    return [_abi.RefinerLog(_int(t[0], w), 0, _float(t[1], w), _float(t[2], w), _float(t[3], w))
            for t in _tokens(path, w, 4)]


# ---------------------------------------------------------------- depth
def save_depth_records(recs: Sequence[_abi.DepthRecord], path: str) -> None:  # io.hpp:276-284
    _write(path, "save_depth_records",
           [f"{r.frame_id} {r.det_id} {fmt6(r.disparity)} {1 if r.valid else 0} {fmt6(r.clp_by_stereo)} "
            f"{fmt6(r.clp_by_gpt)} {fmt6(r.clp_by_size)} {fmt6(r.z_fused)} {DEPTH_SOURCES[r.source]}\n"
            for r in recs])


def load_depth_records(path: str) -> List[_abi.DepthRecord]:  # io.hpp:286-309
    w = "load_depth_records"
    out = []
    for t in _tokens(path, w, 9):
        if t[8] not in DEPTH_SOURCES:
            raise RuntimeError(f"unknown depth source '{t[8]}'")
        out.append(_abi.DepthRecord(_int(t[0], w), _int(t[1], w), _float(t[2], w), int(_int(t[3], w) != 0),
                                    DEPTH_SOURCES.index(t[8]), _float(t[4], w), _float(t[5], w), _float(t[6], w),
                                    _float(t[7], w)))
    return out


# ---------------------------------------------------------------- frames
def save_pgm(img: np.ndarray, path: str) -> None:  # pgm.hpp:34-39
    img = np.ascontiguousarray(img, np.uint8)
    with open(path, "wb") as f:
        f.write(b"P5\n%d %d\n255\n" % (img.shape[1], img.shape[0]))
        f.write(img.tobytes())


def _pnm_header(data: bytes, path: str, maxval: int):
    """pgm.hpp:14-31, 41-56: magic, then w, h, maxval with '#' comments, one
    whitespace byte before the raster."""
    pos = 0
    n = len(data)
    while pos < n and data[pos:pos + 1].isspace():
        pos += 1
    end = pos
    while end < n and not data[end:end + 1].isspace():
        end += 1
    if data[pos:end] != b"P5":
        raise RuntimeError(f"pgm: expected P5 in {path}")
    pos = end
    vals = []
    for _ in range(3):
        while pos < n:
            if data[pos:pos + 1] == b"#":
                nl = data.find(b"\n", pos)
                pos = n if nl < 0 else nl + 1
            elif data[pos:pos + 1].isspace():
                pos += 1
            else:
                break
        m = re.match(rb"[+-]?\d+", data[pos:pos + 16])
        if not m:
            raise RuntimeError("pgm: malformed header")
        vals.append(int(m.group(0)))
        pos += len(m.group(0))
    if vals[2] != maxval:
        raise RuntimeError(f"pgm: expected maxval {maxval} in {path}")
    return vals[0], vals[1], pos + 1


def load_pgm(path: str) -> np.ndarray:  # pgm.hpp:41-57
    try:
        data = open(path, "rb").read()
    except OSError:
        raise RuntimeError(f"pgm: cannot open {path}") from None
    w, h, pos = _pnm_header(data, path, 255)
    if w < 0 or h < 0 or len(data) - pos < w * h:
        raise RuntimeError(f"pgm: truncated raster in {path}")
    return np.frombuffer(data, np.uint8, w * h, pos).reshape(h, w).copy()


def save_disparity_pgm(raw: np.ndarray, path: str) -> None:  # pgm.hpp:60-71
    raw = np.ascontiguousarray(raw, np.int16)
    with open(path, "wb") as f:
        f.write(b"P5\n%d %d\n65535\n" % (raw.shape[1], raw.shape[0]))
        f.write((raw.astype(np.int32) + 32768).astype(">u2").tobytes())


def load_disparity_pgm(path: str) -> np.ndarray:  # pgm.hpp:73-91
    try:
        data = open(path, "rb").read()
    except OSError:
        raise RuntimeError(f"pgm: cannot open {path}") from None
    w, h, pos = _pnm_header(data, path, 65535)
    if w < 0 or h < 0 or len(data) - pos < 2 * w * h:
        raise RuntimeError(f"pgm: truncated raster in {path}")
    enc = np.frombuffer(data, ">u2", w * h, pos).astype(np.int32)
    return (enc - 32768).astype(np.int16).reshape(h, w)


# ---------------------------------------------------------------- calibration
def load_calibration(path: str):
    """load_calibration (geometry.hpp:258-292): `key values` lines (f, b, cx,
    cy, h_cam, R = 9 row-major values, t = 3 values; '#' lines skipped);
    missing R / t default to the canonical rotation / (0, 0, h_cam)."""
    from .ranger import Calibration

    vals = {"f": [0.0], "b": [0.0], "cx": [0.0], "cy": [0.0], "h_cam": [0.0]}
    want = {"f": 1, "b": 1, "cx": 1, "cy": 1, "h_cam": 1, "R": 9, "t": 3}
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"load_calibration: cannot open {path}") from None
    with f:
        for line in f:
            t = line.split()
            if not t or t[0][0] == "#" or t[0] not in want:
                continue
            try:
                v = [float(x) for x in t[1:1 + want[t[0]]]]
            except ValueError:
                v = []
            if len(v) != want[t[0]]:
                raise RuntimeError(f"load_calibration: bad line: {line.rstrip(chr(10))}")
            vals[t[0]] = v
    h = vals["h_cam"][0]
    return Calibration(vals["f"][0], vals["b"][0], vals["cx"][0], vals["cy"][0], h,
                       R=vals.get("R", [0, 0, 1, -1, 0, 0, 0, -1, 0]), t=vals.get("t", [0, 0, h]))


# ---------------------------------------------------------------- run directory
def frame_image_name(side: str, frame_id: int) -> str:  # pipeline.hpp:348-352
    return "%s_%04d.pgm" % (side, frame_id)


@dataclass
class RunFrame:
    """FrameInput minus the ego state (pipeline.hpp:94-100)."""
    frame_id: int
    left: np.ndarray
    right: np.ndarray
    detections: List[Detection] = field(default_factory=list)
    radar: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))


def load_run_directory(d: str) -> List[RunFrame]:  # pipeline.hpp:354-397
    if not os.path.isdir(d):
        raise RuntimeError(f"load_run_directory: no such directory: {d}")
    ids = []
    for name in os.listdir(d):
        m = re.match(r"left_([+-]?\d+)\.pgm", name)  # sscanf("left_%d.pgm")
        if m:
            ids.append(int(m.group(1)))
    ids.sort()
    dets: Dict[int, List[Detection]] = {}
    radar: Dict[int, List[np.ndarray]] = {}
    if os.path.exists(os.path.join(d, "detections.txt")):
        for fid, det in load_detections(os.path.join(d, "detections.txt")):
            dets.setdefault(fid, []).append(det)
    if os.path.exists(os.path.join(d, "radar.txt")):
        for fid, p, _ in load_radar_records(os.path.join(d, "radar.txt")):
            radar.setdefault(fid, []).append(p)
    frames = []
    for i in ids:
        left = load_pgm(os.path.join(d, frame_image_name("left", i)))
        rp = os.path.join(d, frame_image_name("right", i))
        if not os.path.exists(rp):
            raise RuntimeError(f"frame {i}: missing right image {rp}")
        frames.append(RunFrame(i, left, load_pgm(rp), dets.get(i, []),
                               np.array(radar[i]) if i in radar else np.zeros((0, 3))))
    return frames


def save_pipeline_outputs(objects, depth, refiner_log, d: str) -> None:
    """pipeline.hpp:399-406 minus tracks.txt (the tracker is out of scope):
    objects = [(frame_id, record)], depth = [DepthRecord], refiner_log = [RefinerLog]."""
    os.makedirs(d, exist_ok=True)
    save_object_records(objects, os.path.join(d, "objects.txt"))
    save_depth_records(depth, os.path.join(d, "depth.txt"))
    save_refiner_log(refiner_log, os.path.join(d, "refiners.txt"))


def run_directory(engine, run_dir: str, out_dir: str, params, rect=None, cfg=None) -> None:
    """The TEMPLATE_MATCHER method of the reference CLI over a run directory:
    load frames + detections + radar, Engine.pipeline_frames on the device,
    write objects.txt / depth.txt / refiners.txt."""
    import torch

    frames = load_run_directory(run_dir)
    if not frames:
        save_pipeline_outputs([], [], [], out_dir)
        return
    dev = torch.device("cuda", engine.ctx.device)
    L = torch.from_numpy(np.stack([f.left for f in frames])).to(dev)
    R = torch.from_numpy(np.stack([f.right for f in frames])).to(dev)
    objs, recs, logs = engine.pipeline_frames(L, R, [f.detections for f in frames], params,
                                              radar=[f.radar for f in frames],
                                              frame_ids=[f.frame_id for f in frames], rect=rect)
    save_pipeline_outputs([(f.frame_id, o) for f, fo in zip(frames, objs) for o in fo],
                          [r for fr in recs for r in fr], logs, out_dir)
