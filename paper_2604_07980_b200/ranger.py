"""Python mirror of the reference's object-ranging API, backed by the CUDA library.

Names, argument meaning, defaults and error behaviour follow the reference's
header-only C++ API (proj/include/ranger/{census,template_match,bm,autorect}.hpp);
every call runs on the GPU through the C ABI in include/ranger_cuda.h.  There
is no CPU fallback: importing works without a GPU (the library is loaded, its
symbols bound), but the first compute call raises if no sm_100 device exists.

Reference exceptions map as: std::invalid_argument -> InvalidArgument
(a ValueError), anything else -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi

_PKG = os.path.dirname(os.path.abspath(__file__))
# RG_LIB_PATH: A/B builds of the same library (csrc/Makefile VAR=...)
LIB_PATH = os.environ.get("RG_LIB_PATH") or os.path.join(_PKG, "lib", "libranger_cuda.so")

SUB_LEVELS = 16          # DisparityMap::kSubLevels, image.hpp:53
RAW_INVALID = -32768     # DisparityMap::kInvalid, image.hpp:54
KIND_FAR, KIND_CLOSE = _abi.RG_KIND_FAR, _abi.RG_KIND_CLOSE


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference."""


_lib: Optional[C.CDLL] = None
_lib_lock = threading.Lock()


def lib() -> C.CDLL:
    """The loaded CUDA library (raises loudly if it was not built)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                        "(there is no CPU fallback)")
                _lib = _abi.bind(C.CDLL(LIB_PATH))
    return _lib


class Context:
    """One rg_ctx: a device, its streams and pooled buffers (single-writer)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        st = lib().rg_ctx_create(device, C.byref(self._h))
        if st != _abi.RG_OK:
            msg = lib().rg_create_error().decode()
            raise RuntimeError(f"rg_ctx_create(device={device}) failed: {msg}")
        self.device = device

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def check(self, st: int) -> None:
        if st == _abi.RG_OK:
            return
        msg = lib().rg_last_error(self._h).decode()
        if st == _abi.RG_EINVAL:
            raise InvalidArgument(msg)
        raise RuntimeError(f"ranger CUDA library error {st}: {msg}")

    def close(self) -> None:
        if self._h:
            lib().rg_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    # counters / profiling
    def set_profiling(self, on: bool) -> None:
        self.check(lib().rg_set_profiling(self._h, 1 if on else 0))

    def set_overlap(self, on: bool) -> None:
        """rg_range_frames schedule: chunked census/matcher overlap (opt-in) or one stream (default)."""
        self.check(lib().rg_set_overlap(self._h, 1 if on else 0))

    def set_census_rois(self, on: bool) -> None:
        """rg_set_census_rois: ROI-tile census for big batches (default) or
        the full-frame census always."""
        self.check(lib().rg_set_census_rois(self._h, 1 if on else 0))

    def transfer(self) -> Tuple[int, int]:
        """rg_get_transfer: (host->device, device->host) bytes moved by
        rg_range_frames_host since the last reset_counters()."""
        a, b = C.c_int64(0), C.c_int64(0)
        self.check(lib().rg_get_transfer(self._h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def selftest_division(self, b_max: int = 4096) -> int:
        """rg_selftest_division: mismatches of the matcher's table-driven
        integer division against IEEE division (b <= b_max, a <= 64 b)."""
        n = C.c_int64(0)
        self.check(lib().rg_selftest_division(self._h, int(b_max), C.byref(n)))
        return int(n.value)

    def sync(self) -> int:
        """rg_sync: wait for the asynchronous rg_range_frames batches; returns
        RG_OK or RG_EOVERFLOW (a batch produced no results: resubmit it)."""
        st = lib().rg_sync(self._h)
        if st not in (_abi.RG_OK, _abi.RG_EOVERFLOW):
            self.check(st)
        return st

    def set_sync_mode(self, on: bool) -> None:
        """rg_set_sync_mode: blocking rg_range_frames that re-runs overflowed batches itself."""
        self.check(lib().rg_set_sync_mode(self._h, 1 if on else 0))

    def counters(self) -> Tuple[List[float], List[int], int]:
        t = (C.c_double * 5)()
        n = (C.c_int64 * 5)()
        tot = C.c_int64()
        self.check(lib().rg_get_counters(self._h, t, n, C.byref(tot)))
        return list(t), list(n), tot.value

    def work(self) -> Tuple[int, int]:
        """(Hamming evaluations, planned blocks) of the batched path since the last reset."""
        ev, bl = C.c_int64(), C.c_int64()
        self.check(lib().rg_get_work(self._h, C.byref(ev), C.byref(bl)))
        return ev.value, bl.value

    def reset_counters(self) -> None:
        self.check(lib().rg_reset_counters(self._h))


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("RG_DEVICE") is None
                      else int(os.environ["RG_DEVICE"]))
        _tls.ctx = ctx
    return ctx


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def _gray(img) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.uint8)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise InvalidArgument("GrayImage: dims must be >= 1")  # image.hpp:23
    return a


# ============================================================ census.hpp
@dataclass
class CensusImage:
    """census.hpp:21-39: row-major uint32 codes, 0 = undefined."""
    width: int = 0
    height: int = 0
    codes: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.uint32))
    scale_x: float = 1.0
    scale_y: float = 1.0
    kSpan = 2
    kSentinel = 1 << 25

    def code(self, x: int, y: int) -> int:
        return int(self.codes[y, x])

    def inside(self, x: int, y: int) -> bool:
        return 0 <= x < self.width and 0 <= y < self.height


def census_code_at(img, sx: int, sy: int, ctx: Optional[Context] = None) -> int:
    """census.hpp:43-56."""
    ctx = ctx or default_context()
    a = _gray(img)
    out = C.c_uint32()
    ctx.check(lib().rg_census_code_at(ctx.handle, _ptr(a), a.shape[1], a.shape[0], sx, sy, C.byref(out)))
    return out.value


def census_transform(img, out_w: Optional[int] = None, out_h: Optional[int] = None, workers: int = 1,
                     ctx: Optional[Context] = None) -> CensusImage:
    """census.hpp:69-90 (workers is accepted for API parity; the grid is the parallelism)."""
    ctx = ctx or default_context()
    a = _gray(img)
    h, w = a.shape
    ow = w if out_w is None else int(out_w)
    oh = h if out_h is None else int(out_h)
    codes = np.zeros((max(oh, 0), max(ow, 0)), np.uint32)
    ctx.check(lib().rg_census_transform(ctx.handle, _ptr(a), w, h, ow, oh, _ptr(codes)))
    return CensusImage(ow, oh, codes, ow / w, oh / h)


def census_transform64(img, out_w: Optional[int] = None, out_h: Optional[int] = None,
                       ctx: Optional[Context] = None) -> CensusImage:
    """9x7 extension: 64-bit codes, window rows -3..3 x cols -4..4,
    row-major compare order, sentinel bit 63; same nearest-downscale mapping as
    census_transform.  No reference counterpart (parity unpinned)."""
    ctx = ctx or default_context()
    a = _gray(img)
    h, w = a.shape
    ow = w if out_w is None else int(out_w)
    oh = h if out_h is None else int(out_h)
    codes = np.zeros((max(oh, 0), max(ow, 0)), np.uint64)
    ctx.check(lib().rg_census_transform64(ctx.handle, _ptr(a), w, h, ow, oh, _ptr(codes)))
    return CensusImage(ow, oh, codes, ow / w, oh / h)


@dataclass
class CensusRoi:
    x0: int = 0
    y0: int = 0
    x1: int = 0
    y1: int = 0


def census_transform_rois(img, out_w: int, out_h: int, rois: Sequence[CensusRoi], workers: int = 1,
                          ctx: Optional[Context] = None) -> CensusImage:
    """census.hpp:100-138."""
    ctx = ctx or default_context()
    a = _gray(img)
    h, w = a.shape
    r = (_abi.Rect * max(len(rois), 1))(*[_abi.Rect(q.x0, q.y0, q.x1, q.y1) for q in rois])
    codes = np.zeros((max(out_h, 0), max(out_w, 0)), np.uint32)
    ctx.check(lib().rg_census_transform_rois(ctx.handle, _ptr(a), w, h, out_w, out_h, r, len(rois), _ptr(codes)))
    return CensusImage(out_w, out_h, codes, out_w / w, out_h / h)


def hamming_cost(a: int, b: int) -> int:
    """census.hpp:141."""
    return bin((a ^ b) & 0xFFFFFFFF).count("1")


@dataclass
class QueryBlock:
    """census.hpp:146-152."""
    points: List[Tuple[int, int]] = field(default_factory=list)
    dx_min: int = 0
    dx_max: int = 0
    dy_min: int = 0
    dy_max: int = 0
    owner: int = -1
    kind: int = KIND_FAR


@dataclass
class MatchResult:
    """census.hpp:154-163."""
    dx_int: int = 0
    dy_int: int = 0
    dx_subpix: float = 0.0
    cost: float = 0.0
    cost_minus: float = -1.0
    cost_plus: float = -1.0
    valid_points: int = 0
    verified: bool = False


def subpixel_refine(cost_minus: float, cost_at: float, cost_plus: float) -> float:
    """census.hpp:167-171 (pure arithmetic helper)."""
    denom = cost_minus + cost_plus - 2.0 * cost_at
    if denom <= 0.0:
        return 0.0
    return -(cost_plus - cost_minus) / (2.0 * denom)


def _blocks_csr(blocks: Sequence[QueryBlock]):
    offs = np.zeros(len(blocks) + 1, np.int64)
    pts: List[Tuple[int, int]] = []
    for i, b in enumerate(blocks):
        pts.extend(b.points)
        offs[i + 1] = len(pts)
    p = np.asarray(pts, np.int32).reshape(-1, 2) if pts else np.zeros((0, 2), np.int32)
    rg = (_abi.SearchRange * max(len(blocks), 1))(
        *[_abi.SearchRange(b.dx_min, b.dx_max, b.dy_min, b.dy_max) for b in blocks])
    return np.ascontiguousarray(p), offs, rg


def _match(blocks, left: CensusImage, right: CensusImage, mode: int, tau_v: float, ctx) -> list:
    ctx = ctx or default_context()
    if not blocks:
        return []
    pts, offs, rg = _blocks_csr(blocks)
    wide = left.codes.dtype == np.uint64  # 9x7 extension rasters
    ct = np.uint64 if wide else np.uint32
    L = np.ascontiguousarray(left.codes, ct)
    R = np.ascontiguousarray(right.codes, ct)
    out = (_abi.MatchResult * len(blocks))()
    fn = lib().rg_match_blocks64 if wide else lib().rg_match_blocks
    ctx.check(fn(ctx.handle, _ptr(L), left.width, left.height, _ptr(R), right.width,
                                    right.height, _ptr(pts), _ptr(offs), rg, len(blocks), mode,
                                    float(tau_v), out))
    res = []
    for r in out:
        if not r.has_value:
            res.append(None)
            continue
        res.append(MatchResult(r.dx_int, r.dy_int, r.dx_subpix, r.cost, r.cost_minus, r.cost_plus,
                               r.valid_points, bool(r.verified)))
    return res


def block_match(block: QueryBlock, left: CensusImage, right: CensusImage,
                ctx: Optional[Context] = None) -> Optional[MatchResult]:
    """census.hpp:178-272 (None = std::nullopt)."""
    return _match([block], left, right, _abi.RG_MATCH_FORWARD, 0.0, ctx)[0]


def forward_backward_match(block: QueryBlock, left: CensusImage, right: CensusImage, tau_v: float,
                           ctx: Optional[Context] = None) -> Optional[MatchResult]:
    """census.hpp:281-303."""
    return _match([block], left, right, _abi.RG_MATCH_FWD_BWD, tau_v, ctx)[0]


def batch_match(blocks: Sequence[QueryBlock], left: CensusImage, right: CensusImage, tau_v: float,
                workers: int = 1, ctx: Optional[Context] = None) -> List[Optional[MatchResult]]:
    """census.hpp:307-315: one CTA per block, results by block index."""
    return _match(list(blocks), left, right, _abi.RG_MATCH_FWD_BWD, tau_v, ctx)


# ============================================================ template_match.hpp
@dataclass
class Detection:
    """detection.hpp:8-12 (normalized centre-size box)."""
    cx: float = 0.0
    cy: float = 0.0
    w: float = 0.0
    h: float = 0.0
    class_id: int = 0
    id: int = 0


@dataclass
class PixelBox:
    x0: float = 0.0
    y0: float = 0.0
    x1: float = 0.0
    y1: float = 0.0


@dataclass
class FrontalCrop:
    x0: float = 0.25
    y0: float = 0.25
    x1: float = 0.75
    y1: float = 0.75


@dataclass
class RangerConfig:
    """template_match.hpp:33-46 with the reference's defaults."""
    tau_s: float = 48
    close_scale: int = 2
    grid_side_points: int = 8
    max_total_points: int = 64
    close_block_side_points: int = 5
    tau_d: float = 1.0
    n_min: int = 3
    tau_v: float = 1.0
    max_objects: int = 16
    frontal_crop: FrontalCrop = field(default_factory=FrontalCrop)
    dx_max_far: int = 64
    dx_max_close: int = 192
    census_9x7: bool = False  # extension: 64-bit 9x7 descriptors; no cache

    def to_c(self) -> _abi.RangerConfig:
        c = self.frontal_crop
        return _abi.RangerConfig(float(self.tau_s), self.close_scale, self.grid_side_points,
                                 self.max_total_points, self.close_block_side_points, float(self.tau_d),
                                 self.n_min, self.max_objects, float(self.tau_v), c.x0, c.y0, c.x1, c.y1,
                                 self.dx_max_far, self.dx_max_close, int(bool(self.census_9x7)), 0)


@dataclass
class ObjectDisparity:
    """template_match.hpp:18-24 (+ z_cam when a calibration is given)."""
    det_id: int = -1
    disparity: float = 0.0
    kind: int = KIND_FAR
    n_blocks_used: int = 0
    valid: bool = False
    z_cam: float = 0.0


@dataclass
class RangerStats:
    query_points: int = 0
    image_pixels: int = 0
    n_far: int = 0
    n_close: int = 0


@dataclass
class CensusCache:
    """template_match.hpp:229-234."""
    full_left: CensusImage = field(default_factory=CensusImage)
    full_right: CensusImage = field(default_factory=CensusImage)
    scaled_left: CensusImage = field(default_factory=CensusImage)
    scaled_right: CensusImage = field(default_factory=CensusImage)
    has_full: bool = False
    has_scaled: bool = False


@dataclass
class AggregationResult:
    valid: bool = False
    disparity: float = 0.0
    run_length: int = 0


def dets_array(dets: Sequence[Detection]):
    arr = (_abi.Detection * max(len(dets), 1))(
        *[_abi.Detection(d.cx, d.cy, d.w, d.h, d.class_id, d.id) for d in dets])
    return arr


def validate(cfg: RangerConfig, ctx: Optional[Context] = None) -> None:
    """template_match.hpp:48-61."""
    ctx = ctx or default_context()
    c = cfg.to_c()
    ctx.check(lib().rg_validate_ranger_config(ctx.handle, C.byref(c)))


def to_pixel_box(d: Detection, img_w: int, img_h: int) -> PixelBox:
    """detection.hpp:23-30."""
    return PixelBox((d.cx - d.w / 2) * img_w, (d.cy - d.h / 2) * img_h, (d.cx + d.w / 2) * img_w,
                    (d.cy + d.h / 2) * img_h)


def classify_far_close(d: Detection, img_w: int, img_h: int, tau_s: float) -> int:
    """template_match.hpp:63-67."""
    return KIND_FAR if max(d.w * img_w, d.h * img_h) < tau_s else KIND_CLOSE


def select_objects(dets: Sequence[Detection], cfg: RangerConfig, ctx: Optional[Context] = None) -> List[int]:
    """template_match.hpp:94-114 (runs the device planner's rank kernel)."""
    ctx = ctx or default_context()
    n = len(dets)
    out = np.zeros(max(n, 1), np.int32)
    cnt = C.c_int()
    c = cfg.to_c()
    ctx.check(lib().rg_select_objects(ctx.handle, dets_array(dets), n, C.byref(c), _ptr(out), C.byref(cnt)))
    return [int(i) for i in out[:cnt.value]]


def find_occluders(dets: Sequence[Detection], ctx: Optional[Context] = None) -> List[List[int]]:
    """template_match.hpp:71-89."""
    ctx = ctx or default_context()
    n = len(dets)
    off = np.zeros(n + 1, np.int32)
    idx = np.zeros(max(n * n, 1), np.int32)
    ctx.check(lib().rg_find_occluders(ctx.handle, dets_array(dets), n, _ptr(off), _ptr(idx)))
    return [[int(j) for j in idx[off[i]:off[i + 1]]] for i in range(n)]


def sample_query_points(det: Detection, kind: int, occluder_boxes: Sequence[PixelBox], cfg: RangerConfig,
                        img_w: int, img_h: int, ctx: Optional[Context] = None) -> List[QueryBlock]:
    """template_match.hpp:155-223 (runs the device sampler)."""
    ctx = ctx or default_context()
    occ = np.asarray([[b.x0, b.y0, b.x1, b.y1] for b in occluder_boxes], np.float64).reshape(-1, 4)
    occ = np.ascontiguousarray(occ)
    pb = to_pixel_box(det, img_w, img_h)
    if kind == KIND_FAR:
        cap_blocks = 1
    else:  # template_match.hpp:191-193
        half = cfg.tau_s / 2
        cap_blocks = max(2, int((pb.x1 - pb.x0) / half)) * max(2, int((pb.y1 - pb.y0) / half))
    cap_pts = cap_blocks * max(cfg.max_total_points, 1) + 64
    boff = np.zeros(cap_blocks + 1, np.int64)
    pts = np.zeros((cap_pts, 2), np.int32)
    rg = (_abi.SearchRange * cap_blocks)()
    nb = C.c_int()
    c = cfg.to_c()
    d = dets_array([det])
    ctx.check(lib().rg_sample_query_points(ctx.handle, d, kind, _ptr(occ) if occ.size else None, len(occ),
                                           C.byref(c), img_w, img_h, _ptr(boff), _ptr(pts), rg, cap_blocks,
                                           cap_pts, C.byref(nb)))
    blocks = []
    for b in range(nb.value):
        p = [(int(x), int(y)) for x, y in pts[boff[b]:boff[b + 1]]]
        blocks.append(QueryBlock(p, rg[b].dx_min, rg[b].dx_max, rg[b].dy_min, rg[b].dy_max, -1, kind))
    return blocks


def aggregate_close_disparities(disps: Sequence[float], tau_d: float, n_min: int,
                                ctx: Optional[Context] = None) -> AggregationResult:
    """template_match.hpp:126-148."""
    ctx = ctx or default_context()
    v = np.ascontiguousarray(np.asarray(disps, np.float64).reshape(-1))
    valid, run = C.c_int32(), C.c_int32()
    disp = C.c_double()
    ctx.check(lib().rg_aggregate_close_disparities(ctx.handle, _ptr(v) if v.size else None, v.size,
                                                   float(tau_d), int(n_min), C.byref(valid), C.byref(disp),
                                                   C.byref(run)))
    return AggregationResult(bool(valid.value), disp.value, run.value)


def estimate_object_disparities(left, right, dets: Sequence[Detection], cfg: RangerConfig,
                                cache: Optional[CensusCache] = None, workers: int = 1,
                                stats: Optional[RangerStats] = None, focal_px: float = 0.0,
                                baseline_m: float = 0.0, ctx: Optional[Context] = None
                                ) -> List[ObjectDisparity]:
    """template_match.hpp:260-363: one entry per selected detection, in input order."""
    ctx = ctx or default_context()
    L, R = _gray(left), _gray(right)
    if L.shape != R.shape:
        raise InvalidArgument("estimate_object_disparities: image dims differ")
    h, w = L.shape
    n = len(dets)
    out = (_abi.ObjectDisparity * max(n, 1))()
    n_out = C.c_int()
    st = _abi.RangerStats()
    c = cfg.to_c()
    cc = None
    bufs = []
    if cache is not None:
        s = max(cfg.close_scale, 1)
        cw, ch = w // s, h // s
        fl = np.ascontiguousarray(cache.full_left.codes, np.uint32) if cache.has_full else np.zeros((h, w), np.uint32)
        fr = np.ascontiguousarray(cache.full_right.codes, np.uint32) if cache.has_full else np.zeros((h, w), np.uint32)
        sl = np.ascontiguousarray(cache.scaled_left.codes, np.uint32) if cache.has_scaled else np.zeros((ch, cw), np.uint32)
        sr = np.ascontiguousarray(cache.scaled_right.codes, np.uint32) if cache.has_scaled else np.zeros((ch, cw), np.uint32)
        bufs = [fl, fr, sl, sr]
        cc = _abi.CensusCache(fl.ctypes.data, fr.ctypes.data, sl.ctypes.data, sr.ctypes.data,
                              int(cache.has_full), int(cache.has_scaled))
    ctx.check(lib().rg_estimate_object_disparities(ctx.handle, _ptr(L), _ptr(R), w, h, dets_array(dets), n,
                                                   C.byref(c), C.byref(cc) if cc is not None else None,
                                                   float(focal_px), float(baseline_m), out, C.byref(n_out),
                                                   C.byref(st)))
    if cache is not None:
        s = max(cfg.close_scale, 1)
        cw, ch = w // s, h // s
        if cc.has_full and not cache.has_full:
            cache.full_left = CensusImage(w, h, bufs[0], 1.0, 1.0)
            cache.full_right = CensusImage(w, h, bufs[1], 1.0, 1.0)
            cache.has_full = True
        if cc.has_scaled and not cache.has_scaled:
            cache.scaled_left = CensusImage(cw, ch, bufs[2], cw / w, ch / h)
            cache.scaled_right = CensusImage(cw, ch, bufs[3], cw / w, ch / h)
            cache.has_scaled = True
    if stats is not None:
        stats.query_points, stats.image_pixels = st.query_points, st.image_pixels
        stats.n_far, stats.n_close = st.n_far, st.n_close
    return [ObjectDisparity(o.det_id, o.disparity, o.kind, o.n_blocks_used, bool(o.valid), o.z_cam)
            for o in out[:n_out.value]]


# ============================================================ bm.hpp / autorect.hpp
@dataclass
class BmParams:
    """bm.hpp:15-22 with the reference's defaults."""
    num_disparities: int = 64
    block_size: int = 9
    min_disparity: int = 0
    texture_threshold: float = 10
    uniqueness_ratio: float = 10
    downscale: int = 1

    def to_c(self) -> _abi.BmParams:
        return _abi.BmParams(self.num_disparities, self.block_size, self.min_disparity, self.downscale,
                             float(self.texture_threshold), float(self.uniqueness_ratio))


@dataclass
class ImageRoi:
    x0: int = 0
    y0: int = 0
    x1: int = 0
    y1: int = 0

    def width(self) -> int:
        return self.x1 - self.x0

    def height(self) -> int:
        return self.y1 - self.y0


def validate_bm(p: BmParams, ctx: Optional[Context] = None) -> None:
    ctx = ctx or default_context()
    c = p.to_c()
    ctx.check(lib().rg_validate_bm_params(ctx.handle, C.byref(c)))


def bm_disparity(left, right, p: BmParams, workers: int = 1, ctx: Optional[Context] = None) -> np.ndarray:
    """bm.hpp:113-135: raw int16 map (16 sub-levels, RAW_INVALID = invalid)."""
    ctx = ctx or default_context()
    L, R = _gray(left), _gray(right)
    if L.shape != R.shape:
        c = p.to_c()
        ctx.check(lib().rg_validate_bm_params(ctx.handle, C.byref(c)))
        raise InvalidArgument("bm_disparity: image dims differ")
    h, w = L.shape
    out = np.zeros((h, w), np.int16)
    c = p.to_c()
    ctx.check(lib().rg_bm_disparity(ctx.handle, _ptr(L), _ptr(R), w, h, C.byref(c), _ptr(out)))
    return out


def auto_rect_search(left, right, roi: ImageRoi, delta_min: int, delta_max: int, bm: BmParams,
                     workers: int = 1, ctx: Optional[Context] = None, counts_out: Optional[list] = None) -> int:
    """autorect.hpp:22-58."""
    ctx = ctx or default_context()
    L, R = _gray(left), _gray(right)
    h, w = L.shape
    r = _abi.Rect(roi.x0, roi.y0, roi.x1, roi.y1)
    c = bm.to_c()
    if L.shape != R.shape:
        if roi.width() < bm.block_size or roi.height() < bm.block_size:
            raise InvalidArgument("auto_rect_search: ROI smaller than the match window")
        if roi.x0 < 0 or roi.y0 < 0 or roi.x1 > w or roi.y1 > h:
            raise InvalidArgument("auto_rect_search: ROI leaves the image")
        if delta_min > delta_max:
            raise InvalidArgument("auto_rect_search: empty delta range")
        raise InvalidArgument("auto_rect_search: image dims differ")
    best = C.c_int32()
    nd = max(delta_max - delta_min + 1, 1)
    counts = np.zeros(nd, np.int64)
    ctx.check(lib().rg_auto_rect_search(ctx.handle, _ptr(L), _ptr(R), w, h, C.byref(r), delta_min, delta_max,
                                        C.byref(c), C.byref(best), _ptr(counts)))
    if counts_out is not None:
        counts_out[:] = [int(x) for x in counts]
    return best.value


class RectOffsetState:
    """autorect.hpp:62-75 (host-side sequential consumer of the search)."""

    def __init__(self, k: int = 5, rate: float = 1):
        if k < 1:
            raise InvalidArgument("RectOffsetState: window must be >= 1")
        self.window, self.delta_max, self.current = k, float(rate), 0.0
        self.history: List[int] = []
        self.next = 0


@dataclass
class BoxDisparity:
    """Pipeline::BoxDisparity (pipeline.hpp:298-302)."""
    median: float = 0.0
    variance: float = 0.0
    count: int = 0


@dataclass
class DenseVarianceParams:
    """PipelineConfig sigma_obs2 / var_gamma / sigma_sys2 (pipeline.hpp:78-80 defaults)."""
    sigma_obs2: float = 0.3
    gamma: float = 1.0
    sigma_sys2: float = 0.01


def dense_objects(left, right, dets: Sequence[Detection], cfg: RangerConfig, bm: "BmParams",
                  var: Optional[DenseVarianceParams] = None, ctx: Optional[Context] = None):
    """The STEREO_BM branch of Pipeline::process_frame (pipeline.hpp:140-141,
    207-224): dense BM on the device, select_objects, box_disparity per
    selected box.  Returns ([ObjectDisparity], [Optional[BoxDisparity]], raw map)."""
    ctx = ctx or default_context()
    var = var or DenseVarianceParams()
    L, R = _gray(left), _gray(right)
    h, w = L.shape
    arr = dets_array(dets)
    n = len(dets)
    out = (_abi.ObjectDisparity * max(n, 1))()
    box = (_abi.BoxStats * max(n, 1))()
    n_out = C.c_int()
    raw = np.empty((h, w), np.int16)
    c, b = cfg.to_c(), bm.to_c()
    ctx.check(lib().rg_dense_objects(ctx.handle, _ptr(L), _ptr(R), w, h, arr, n, C.byref(c), C.byref(b),
                                     float(var.sigma_obs2), float(var.gamma), float(var.sigma_sys2), out, box,
                                     C.byref(n_out), _ptr(raw)))
    objs = [ObjectDisparity(o.det_id, o.disparity, o.kind, o.n_blocks_used, bool(o.valid), o.z_cam)
            for o in list(out)[:n_out.value]]
    boxes = [BoxDisparity(x.median, x.variance, x.count) if x.valid > 0 else None for x in list(box)[:n_out.value]]
    return objs, boxes, raw


class VoteState:
    """VoteState (radar_refiner.hpp:30-47): the radar refiner's vote memory,
    carried from frame to frame by the caller (defaults K 4, lambda 0.3,
    sigma 1 px)."""

    def __init__(self, k_px: int = 4, lam: float = 0.3, smooth_sigma_px: float = 1.0):
        self._c = _abi.VoteState()
        if lib().rg_vote_state_init(C.byref(self._c), k_px, lam, smooth_sigma_px) != _abi.RG_OK:
            raise InvalidArgument("VoteState: K must be >= 1 (<= 32 here) and lambda in (0, 1]")

    @property
    def smoothed_offset(self) -> float:
        return self._c.smoothed_offset

    @property
    def memory(self) -> np.ndarray:
        return np.array(self._c.memory[:self._c.n_bins])

    def to_c(self) -> _abi.VoteState:
        return self._c


def radar_array(radar):
    """[(position (x, y, z), extent (x, y, z), id)] -> rg_radar_detection array."""
    return (_abi.RadarDetection * max(len(radar), 1))(
        *[_abi.RadarDetection(_abi.Vec3(*p), _abi.Vec3(*e), int(i), 0) for p, e, i in radar])


def dense_objects_refined(left, right, dets: Sequence[Detection], cfg: RangerConfig, bm: "BmParams", radar,
                          vote: VoteState, calib: "Calibration", var: Optional["DenseVarianceParams"] = None,
                          ctx: Optional[Context] = None):
    """dense_objects with the radar (dense-map) refiner between the BM map and
    the box statistics (pipeline.hpp:182-183; PipelineConfig::radar_refiner
    defaults to true).  radar: [(position, extent, id)] of this frame (vehicle
    frame); vote: the VoteState carried across frames.  Returns ([ObjectDisparity],
    [Optional[BoxDisparity]], refined raw map, radar offset applied)."""
    ctx = ctx or default_context()
    var = var or DenseVarianceParams()
    L, R = _gray(left), _gray(right)
    h, w = L.shape
    arr = dets_array(dets)
    n = len(dets)
    out = (_abi.ObjectDisparity * max(n, 1))()
    box = (_abi.BoxStats * max(n, 1))()
    n_out = C.c_int()
    raw = np.empty((h, w), np.int16)
    applied = C.c_double()
    c, b = cfg.to_c(), bm.to_c()
    ra = radar_array(radar)
    ctx.check(lib().rg_dense_objects_refined(ctx.handle, _ptr(L), _ptr(R), w, h, arr, n, C.byref(c), C.byref(b),
                                             float(var.sigma_obs2), float(var.gamma), float(var.sigma_sys2), ra,
                                             len(radar), C.byref(vote.to_c()), C.byref(calib.to_c()), out, box,
                                             C.byref(n_out), _ptr(raw), C.byref(applied)))
    objs = [ObjectDisparity(o.det_id, o.disparity, o.kind, o.n_blocks_used, bool(o.valid), o.z_cam)
            for o in list(out)[:n_out.value]]
    boxes = [BoxDisparity(x.median, x.variance, x.count) if x.valid > 0 else None for x in list(box)[:n_out.value]]
    return objs, boxes, raw, applied.value


@dataclass
class SgmParams:
    """sgm.hpp:14-19 with the reference's defaults."""
    num_disparities: int = 64
    min_disparity: int = 0
    p1: int = 8
    p2: int = 32

    def to_c(self) -> _abi.SgmParams:
        return _abi.SgmParams(self.num_disparities, self.min_disparity, self.p1, self.p2)


def sgm_disparity(left, right, p: SgmParams, workers: int = 1, ctx: Optional[Context] = None) -> np.ndarray:
    """sgm.hpp:118-155 (census SGM, 4 paths, WTA + sub-pixel): raw int16 map."""
    ctx = ctx or default_context()
    L, R = _gray(left), _gray(right)
    if L.shape != R.shape:
        c = p.to_c()
        ctx.check(lib().rg_validate_sgm_params(ctx.handle, C.byref(c)))
        raise InvalidArgument("sgm_disparity: image dims differ")
    h, w = L.shape
    out = np.empty((h, w), np.int16)
    c = p.to_c()
    ctx.check(lib().rg_sgm_disparity(ctx.handle, _ptr(L), _ptr(R), w, h, C.byref(c), _ptr(out)))
    return out


@dataclass
class RectSearchConfig:
    """pipeline.hpp:52-62 with the reference's defaults."""
    enabled: bool = True
    delta_min: int = -3
    delta_max: int = 3
    window: int = 5
    rate_limit: float = 1.0
    bm: BmParams = field(default_factory=lambda: BmParams(32, 9, -4, 10, 10, 1))

    def to_c(self) -> _abi.RectSearchConfig:
        return _abi.RectSearchConfig(int(bool(self.enabled)), self.delta_min, self.delta_max, self.window,
                                     float(self.rate_limit), self.bm.to_c())


def rect_state_to_c(st: RectOffsetState) -> _abi.RectState:
    if not 1 <= st.window <= _abi.RECT_MAX_WINDOW:
        raise InvalidArgument("RectOffsetState: window must be in [1, 64] for the device path")
    c = _abi.RectState()
    c.window, c.n_hist, c.next, c.delta_max, c.current = st.window, len(st.history), st.next, st.delta_max, st.current
    for i, v in enumerate(st.history):
        c.history[i] = int(v)
    return c


def rect_state_from_c(c: _abi.RectState, st: RectOffsetState) -> None:
    st.window, st.next, st.delta_max, st.current = c.window, c.next, c.delta_max, c.current
    st.history = [int(c.history[i]) for i in range(c.n_hist)]


def filter_offset(st: RectOffsetState, delta_star: int) -> float:
    """autorect.hpp:77-90: lower median of the window, rate-limited."""
    if len(st.history) < st.window:
        st.history.append(delta_star)
    else:
        st.history[st.next] = delta_star
        st.next = (st.next + 1) % len(st.history)
    srt = sorted(st.history)
    cand = float(srt[(len(srt) - 1) // 2])
    step = min(max(cand - st.current, -st.delta_max), st.delta_max)
    st.current += step
    return st.current


class Calibration:
    """StereoCalibration built by make_calibration (geometry.hpp:101-133):
    the canonical camera->vehicle rotation and t = (0, 0, h_cam) unless R
    (row-major, 9 values) / t are given."""

    def __init__(self, f: float, b: float, cx: float, cy: float, h_cam: float, R=None, t=None):
        self._c = _abi.Calibration()
        if lib().rg_make_calibration(f, b, cx, cy, h_cam, C.byref(self._c)) != _abi.RG_OK:
            raise InvalidArgument("make_calibration: f and b must be positive")
        if R is not None:
            r = np.asarray(R, np.float64).reshape(9)
            m = r.reshape(3, 3)  # is_rotation(R, 1e-6), geometry.hpp:65-72, 110-111
            if np.abs(m.T @ m - np.eye(3)).max() > 1e-6 or abs(np.linalg.det(m) - 1.0) > 1e-6:
                raise InvalidArgument("make_calibration: R is not a rotation")
            for i in range(9):
                self._c.R[i] = float(r[i])
        if t is not None:
            for i in range(3):
                self._c.t[i] = float(t[i])

    def to_c(self) -> _abi.Calibration:
        return self._c


@dataclass
class ObjRefinerState:
    """object_refiner.hpp:14-21 (defaults)."""
    prev_offset: float = 0.0
    beta: float = 0.1
    r_max: float = 5.0
    w_p: float = 1.0
    tau: float = 0.5
    rate_limit: float = 0.5

    def to_c(self) -> _abi.ObjRefinerState:
        return _abi.ObjRefinerState(self.prev_offset, self.beta, self.r_max, self.w_p, self.tau, self.rate_limit)

    def update(self, c: _abi.ObjRefinerState) -> None:
        self.prev_offset = c.prev_offset


@dataclass
class RecordParams:
    """The PipelineConfig fields the per-frame records use (pipeline.hpp:64-79,
    tracker.hpp:18): calibration, class widths, object refiner switches and
    the fusion sanity ratio."""
    calib: Calibration
    class_width_m: dict = field(default_factory=lambda: {0: 1.9, 1: 2.5})
    object_refiner: bool = True
    obj_cand_half_px: float = 2.0
    obj_cand_step_px: float = 0.25
    fuse_sanity_ratio: float = 0.5

    def to_c(self):
        cw = (_abi.ClassWidth * max(1, len(self.class_width_m)))()
        for i, (k, v) in enumerate(sorted(self.class_width_m.items())):
            cw[i] = _abi.ClassWidth(int(k), 0, float(v))
        p = _abi.RecordParams(self.calib.to_c(), C.cast(cw, C.c_void_p), len(self.class_width_m),
                              int(self.object_refiner), self.obj_cand_half_px, self.obj_cand_step_px,
                              self.fuse_sanity_ratio)
        return p, cw  # keep cw alive while p is in use


DEPTH_SOURCES = ("STEREO", "GPT", "SIZE")  # DepthSource (geometry.hpp:187), io.hpp:76-82 spelling


def frame_records(params: RecordParams, frame_id: int, img_w: int, img_h: int, dets: np.ndarray,
                  sel: np.ndarray, objects: np.ndarray, radar: Optional[np.ndarray], state: ObjRefinerState,
                  rect_applied: float = 0.0, dense: bool = False):
    """rg_frame_records: pipeline.hpp:180-249 for one frame (host code in the
    library).  dets: the frame's DET_DTYPE records; sel: int32 frame-local
    index per object; objects: OUT_DTYPE records (not modified); radar: (n, 3)
    float64 vehicle-frame positions.  Returns (objects after the object
    refiner offset, list of _abi.DepthRecord, _abi.RefinerLog)."""
    objects = np.array(objects, copy=True)
    dets = np.ascontiguousarray(dets)
    n = len(objects)
    sel = np.ascontiguousarray(sel, np.int32)
    radar = np.ascontiguousarray(radar if radar is not None else np.zeros((0, 3)), np.float64).reshape(-1, 3)
    recs = (_abi.DepthRecord * max(1, n))()
    log = _abi.RefinerLog()
    p, keep = params.to_c()
    st = state.to_c()
    rc = lib().rg_frame_records(C.byref(p), frame_id, img_w, img_h, int(dense), dets.ctypes.data if len(dets) else None,
                                len(dets), sel.ctypes.data, objects.ctypes.data if n else None, n,
                                radar.ctypes.data if len(radar) else None, len(radar), C.byref(st), rect_applied,
                                recs, C.byref(log))
    del keep
    if rc != _abi.RG_OK:
        raise InvalidArgument("frame_records: invalid input (reproject / radar behind camera / indices)")
    state.update(st)
    return objects, list(recs)[:n], log


def range_z(disparity: float, focal_px: float, baseline_m: float) -> float:
    """geometry.hpp:142-146 with the canonical Q (:124-127): z = f / ((1/b) d)."""
    return focal_px / ((1.0 / baseline_m) * disparity)
