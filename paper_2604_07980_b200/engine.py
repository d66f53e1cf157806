"""Batched frame ranging engine: the throughput path (one process per GPU).

Frames live on the device (torch uint8 tensors, shape (F, H, W)); detections
are a packed array of rg_detection records with per-frame CSR offsets.  One
call ranges every frame of the batch with four kernel launches (census K1,
planner K3, fused sampler+matcher K2, aggregation+range K4) through
rg_range_frames; rg_range_frames_host is the host-fed variant that streams
pinned host frames through double-buffered device staging.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from .ranger import Context, Detection, RangerConfig, default_context, lib

DET_DTYPE = np.dtype([("cx", "<f8"), ("cy", "<f8"), ("w", "<f8"), ("h", "<f8"), ("class_id", "<i4"),
                      ("id", "<i4")])
OUT_DTYPE = np.dtype([("det_id", "<i4"), ("kind", "<i4"), ("n_blocks_used", "<i4"), ("valid", "<i4"),
                      ("disparity", "<f8"), ("z_cam", "<f8")])
assert DET_DTYPE.itemsize == C.sizeof(_abi.Detection) == 40
assert OUT_DTYPE.itemsize == C.sizeof(_abi.ObjectDisparity) == 32


def pack_detections(frames: Sequence[Sequence[Detection]]):
    """-> (records[DET_DTYPE], offsets[int32, F+1])"""
    offs = np.zeros(len(frames) + 1, np.int32)
    recs = []
    for f, dets in enumerate(frames):
        recs.extend((d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets)
        offs[f + 1] = len(recs)
    arr = np.array(recs, dtype=DET_DTYPE) if recs else np.zeros(0, DET_DTYPE)
    return arr, offs


class FrameEngine:
    """Ranges batches of W x H stereo pairs with a fixed RangerConfig."""

    def __init__(self, width: int, height: int, cfg: RangerConfig, max_dets_per_frame: int,
                 focal_px: float = 0.0, baseline_m: float = 0.0, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.w, self.h = width, height
        self.cfg = cfg
        self._c = cfg.to_c()
        self.max_dets = max_dets_per_frame
        self.out_stride = max(1, min(max_dets_per_frame, cfg.max_objects))
        self.focal, self.baseline = focal_px, baseline_m

    def _batch(self, n_frames, pitch, stride, left, right, dets, offs, out, cnt, shift=None,
               out_index=None) -> _abi.FrameBatch:
        return _abi.FrameBatch(n_frames, self.w, self.h, pitch, stride, left, right, dets, offs, self.max_dets,
                               self.out_stride, out, cnt, self.focal, self.baseline, shift, out_index)

    def range_device(self, left, right, dets, offsets, out, out_count, stream=None, left_shift=None,
                     sync: bool = True) -> None:
        """All arguments are CUDA torch tensors: left/right uint8 (F, H, pitch)
        with unit column stride and the same strides on both sides; dets uint8
        view of DET_DTYPE records; offsets int32 (F+1); out uint8
        (F * out_stride * 32); out_count int32 (F); left_shift int32 (F) or
        None: per-frame shift_vertical of the left image (pipeline.hpp:135-138).
        rg_range_frames is asynchronous: sync=True waits (rg_sync) and
        resubmits the batch once if its block list overflowed; sync=False
        returns at once (call ctx.sync() before reading the results)."""
        F = left.shape[0]
        if left.dim() == 3:
            if left.stride(2) != 1 or tuple(right.stride()) != tuple(left.stride()) or right.shape != left.shape:
                raise ValueError("range_device: left/right must have unit column stride and identical layouts")
            pitch = left.stride(1)
        else:
            pitch = self.w
        b = self._batch(F, pitch, left.stride(0), left.data_ptr(), right.data_ptr(), dets.data_ptr(),
                        offsets.data_ptr(), out.data_ptr(), out_count.data_ptr(),
                        left_shift.data_ptr() if left_shift is not None else None)
        s = C.c_void_p(stream) if stream is not None else None
        for attempt in range(2):
            self.ctx.check(lib().rg_range_frames(self.ctx.handle, C.byref(b), C.byref(self._c), s))
            if not sync or self.ctx.sync() == _abi.RG_OK:
                return
        raise RuntimeError("rg_range_frames: block list overflow persisted after a resubmit")

    def range_host(self, left: np.ndarray, right: np.ndarray, dets: np.ndarray, offsets: np.ndarray,
                   out: np.ndarray, out_count: np.ndarray, chunk: int = 16, stream=None,
                   left_shift: Optional[np.ndarray] = None) -> None:
        """Host (ideally pinned) numpy buffers, C-contiguous (F, H, W) images;
        H2D / compute / D2H inside."""
        F = left.shape[0]
        for a in (left, right):
            if a.shape != (F, self.h, self.w) or not a.flags.c_contiguous or a.dtype != np.uint8:
                raise ValueError("range_host: images must be C-contiguous uint8 (F, H, W)")
        if offsets.dtype != np.int32 or offsets.shape != (F + 1,) or not offsets.flags.c_contiguous:
            raise ValueError("range_host: offsets must be contiguous int32 (F + 1)")
        if left_shift is not None:
            left_shift = np.ascontiguousarray(left_shift, np.int32)
            assert left_shift.shape == (F,)
        b = self._batch(F, self.w, self.w * self.h, left.ctypes.data, right.ctypes.data,
                        dets.ctypes.data if dets.size else 0, offsets.ctypes.data, out.ctypes.data,
                        out_count.ctypes.data, left_shift.ctypes.data if left_shift is not None else None)
        s = C.c_void_p(stream) if stream is not None else None
        self.ctx.check(lib().rg_range_frames_host(self.ctx.handle, C.byref(b), C.byref(self._c), chunk, s))

    def range_sequence(self, left, right, dets, offsets, out, out_count, rect=None, state=None, stream=None,
                       out_index=None, applied=None):
        """Pipeline::process_frame's TEMPLATE_MATCHER loop over consecutive
        device frames (rg_range_sequence): offset search on every uncorrected
        pair, host filter scan, ranging of the rect-corrected pairs.  `state`
        (RectOffsetState) is advanced in place; returns (shifts, delta_stars).
        out_index (device int32, F*out_stride) receives the frame-local
        detection index per output; applied (host float64, F) the rect offset
        in force per frame."""
        from .ranger import RectOffsetState, RectSearchConfig, rect_state_from_c, rect_state_to_c

        rect = rect or RectSearchConfig()
        state = state if state is not None else RectOffsetState(rect.window, rect.rate_limit)
        F = left.shape[0]
        pitch = left.shape[2] if left.dim() == 3 else self.w
        b = self._batch(F, pitch, left.stride(0), left.data_ptr(), right.data_ptr(), dets.data_ptr(),
                        offsets.data_ptr(), out.data_ptr(), out_count.data_ptr(),
                        out_index=out_index.data_ptr() if out_index is not None else None)
        rc, sc = rect.to_c(), rect_state_to_c(state)
        shifts, deltas = np.zeros(F, np.int32), np.zeros(F, np.int32)
        if applied is not None:
            assert applied.dtype == np.float64 and applied.shape == (F,) and applied.flags.c_contiguous
        s = C.c_void_p(stream) if stream is not None else None
        self.ctx.check(lib().rg_range_sequence(self.ctx.handle, C.byref(b), C.byref(self._c), C.byref(rc),
                                               C.byref(sc), shifts.ctypes.data, deltas.ctypes.data,
                                               applied.ctypes.data if applied is not None else None, s))
        rect_state_from_c(sc, state)
        return shifts, deltas

    def pipeline_frames(self, left, right, frames_dets, params, radar=None, frame_ids=None, rect=None,
                        rect_state=None, obj_state=None, stream=None):
        """Pipeline::process_frame, TEMPLATE_MATCHER method, over consecutive
        device frames minus the tracker (pipeline.hpp:124-265): the device
        two-pass frame loop (rg_range_sequence) then, per frame in order on
        the host, the object refiner, the depth cues and fusion
        (rg_frame_records).  frames_dets: per-frame lists of Detection;
        radar: per-frame (n, 3) vehicle-frame positions (or None).
        Returns (objects per frame, DepthRecords per frame, RefinerLog per frame)."""
        import torch

        from .ranger import ObjRefinerState, RectOffsetState, RectSearchConfig, frame_records

        F = left.shape[0]
        dev = left.device
        rect = rect or RectSearchConfig()
        rect_state = rect_state if rect_state is not None else RectOffsetState(rect.window, rect.rate_limit)
        obj_state = obj_state if obj_state is not None else ObjRefinerState()
        recs, offs = pack_detections(frames_dets)
        d_dets = torch.from_numpy(recs.view(np.uint8).copy() if len(recs) else np.zeros(1, np.uint8)).to(dev)
        d_offs = torch.from_numpy(offs).to(dev)
        out = torch.zeros(F * self.out_stride * OUT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        cnt = torch.zeros(F, dtype=torch.int32, device=dev)
        idx = torch.zeros(F * self.out_stride, dtype=torch.int32, device=dev)
        applied = np.zeros(F, np.float64)
        self.range_sequence(left, right, d_dets, d_offs, out, cnt, rect=rect, state=rect_state, stream=stream,
                            out_index=idx, applied=applied)
        if stream is not None:
            torch.cuda.ExternalStream(stream).synchronize()
        else:
            torch.cuda.synchronize(dev)
        objs = unpack_results(out.cpu().numpy(), cnt.cpu().numpy(), self.out_stride)
        sel = idx.cpu().numpy().reshape(F, self.out_stride)
        all_objs, all_recs, logs = [], [], []
        for f in range(F):
            n = len(objs[f])
            fid = int(frame_ids[f]) if frame_ids is not None else f
            o, r, lg = frame_records(params, fid, self.w, self.h, recs[offs[f]:offs[f + 1]], sel[f, :n], objs[f],
                                     radar[f] if radar is not None else None, obj_state, float(applied[f]))
            all_objs.append(o)
            all_recs.append(r)
            logs.append(lg)
        return all_objs, all_recs, logs

    def auto_rect_device(self, left, right, roi, delta_min: int, delta_max: int, bm, best, counts=None,
                         stream=None) -> None:
        """rg_auto_rect_frames over device frames (torch tensors)."""
        F = left.shape[0]
        r = _abi.Rect(*roi)
        p = bm.to_c()
        s = C.c_void_p(stream) if stream is not None else None
        self.ctx.check(lib().rg_auto_rect_frames(
            self.ctx.handle, left.data_ptr(), right.data_ptr(), F, left.stride(0), left.shape[2], self.w, self.h,
            C.byref(r), delta_min, delta_max, C.byref(p), best.data_ptr(),
            counts.data_ptr() if counts is not None else None, s))


def unpack_results(out: np.ndarray, counts: np.ndarray, out_stride: int) -> List[np.ndarray]:
    recs = np.frombuffer(out.tobytes(), dtype=OUT_DTYPE).reshape(-1, out_stride)
    return [recs[f, :int(counts[f])] for f in range(len(counts))]


class MultiRanger:
    """rg_multi_*: host frame batches sharded over several devices (one
    context + host thread each); per-box records gathered in
    frame order to the first device (NCCL send/recv) and/or the host."""

    def __init__(self, devices: Sequence[int], width: int, height: int, cfg: RangerConfig, max_dets_per_frame: int,
                 focal_px: float = 0.0, baseline_m: float = 0.0):
        arr = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        st = lib().rg_multi_create(arr, len(devices), C.byref(h))
        if st != _abi.RG_OK:
            raise RuntimeError(f"rg_multi_create failed ({st}): "
                               f"{(lib().rg_multi_last_error(h) or b'').decode() if h.value else ''}")
        self._h, self.devices = h, list(devices)
        self.w, self.h, self.cfg, self._c = width, height, cfg, cfg.to_c()
        self.max_dets = max_dets_per_frame
        self.out_stride = max(1, min(max_dets_per_frame, cfg.max_objects))
        self.focal, self.baseline = focal_px, baseline_m

    def range_host(self, left: np.ndarray, right: np.ndarray, dets: np.ndarray, offsets: np.ndarray,
                   out: Optional[np.ndarray] = None, out_count: Optional[np.ndarray] = None, d_out0=None,
                   d_count0=None, chunk: int = 64) -> None:
        """left/right C-contiguous uint8 (F, H, W) host arrays (pinned for full
        PCIe rate); out/out_count host arrays and/or d_out0/d_count0 uint8 /
        int32 CUDA tensors on the first device."""
        F = left.shape[0]
        for a in (left, right):
            if a.shape != (F, self.h, self.w) or not a.flags.c_contiguous or a.dtype != np.uint8:
                raise ValueError("MultiRanger.range_host: images must be C-contiguous uint8 (F, H, W)")
        b = _abi.FrameBatch(F, self.w, self.h, self.w, self.w * self.h, left.ctypes.data, right.ctypes.data,
                            dets.ctypes.data if dets.size else 0, offsets.ctypes.data, self.max_dets,
                            self.out_stride, None, None, self.focal, self.baseline, None, None)
        st = lib().rg_multi_range_host(self._h, C.byref(b), C.byref(self._c), chunk,
                                       d_out0.data_ptr() if d_out0 is not None else None,
                                       d_count0.data_ptr() if d_count0 is not None else None,
                                       out.ctypes.data if out is not None else None,
                                       out_count.ctypes.data if out_count is not None else None)
        if st != _abi.RG_OK:
            raise RuntimeError(f"rg_multi_range_host failed ({st}): {lib().rg_multi_last_error(self._h).decode()}")

    def close(self) -> None:
        if self._h:
            lib().rg_multi_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
