"""TEST INFRASTRUCTURE: ctypes access to the CPU checkers under oracle/.

orc_* = oracle/_build/liboracle.so (plain-C restatement, always built)
ref_* = oracle/_ref/libranger_ref.so (the reference compiled in place; only
        present where /root/reference existed at build time)
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2604_07980_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libranger_ref.so")

P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
_SIG = {
    "census_transform": (I, [P, I, I, I, I, P]),
    "census_transform_rois": (I, [P, I, I, I, I, P, I, P]),
    "match_blocks": (I, [P, I, I, P, I, I, P, P, P, I, I, D, P]),
    "select_objects": (I, [P, I, P, P, P]),
    "find_occluders": (I, [P, I, P, P]),
    "sample_query_points": (I, [P, I, P, I, P, I, I, P, P, P, I, I64, P]),
    "aggregate_close_disparities": (I, [P, I, D, I, P, P, P]),
    "estimate_object_disparities": (I, [P, P, I, I, P, I, P, P, D, D, P, P, P]),
    "bm_disparity": (I, [P, P, I, I, P, P]),
    "auto_rect_search": (I, [P, P, I, I, P, I, I, P, P, P]),
}


class Checker:
    """Uniform numpy-facing wrapper over orc_* or ref_*."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.prefix = prefix
        for name, (res, args) in _SIG.items():
            fn = getattr(self.lib, prefix + name)
            fn.restype, fn.argtypes = res, args
        if prefix == "ref_":
            self.lib.ref_render_stereo_pair.restype = I
            self.lib.ref_render_stereo_pair.argtypes = [P, P, I, P, P]
            self.lib.ref_ground_truth_detections.restype = I
            self.lib.ref_ground_truth_detections.argtypes = [P, P, I, P, P]
            self.lib.ref_pipeline_sequence.restype = I
            self.lib.ref_pipeline_sequence.argtypes = [P, P, I, I, I, P, P, P, P, D, D, D, D, D, I, P, P, I, P, P]
            self.lib.ref_pipeline_records.restype = I
            self.lib.ref_pipeline_records.argtypes = [P, P, I, I, I, P, P, P, P, P, P, P, I, P, P, I, P, P, P]
            self.lib.ref_save_synthetic_run.restype = I
            self.lib.ref_save_synthetic_run.argtypes = [P, P, I, I, D, C.c_char_p]
            self.lib.ref_run_directory.restype = I
            self.lib.ref_run_directory.argtypes = [C.c_char_p, C.c_char_p, P, P, I, D]
            self.lib.ref_dynamic_disparity_variance.restype = I
            self.lib.ref_dynamic_disparity_variance.argtypes = [P, I, P, I, D, D, D, P]
            self.lib.ref_pipeline_dense_radar.restype = I
            self.lib.ref_pipeline_dense_radar.argtypes = [P, P, I, I, I, P, P, P, P, P, P, P, I, D, D, P, I, P, P]
            self.lib.ref_bench_estimate.restype = D
            self.lib.ref_bench_estimate.argtypes = [P, P, I, I, I, P, P, P, I, P, I, P]

        for nm, args in (("sgm_direction_pass", [P, I, I, I, I, I, I, I, P]),
                         ("sgm_disparity", [P, P, I, I, I, I, I, I, P])):
            f = getattr(self.lib, prefix + nm)
            f.restype, f.argtypes = I, args
        if prefix == "orc_":  # restatement-only entry points
            self.lib.orc_box_disparity.restype = I
            self.lib.orc_box_disparity.argtypes = [P, I, I, P, I, D, D, D, P]
            self.lib.orc_census_transform64.restype = I
            self.lib.orc_census_transform64.argtypes = [P, I, I, I, I, P]
            self.lib.orc_match_blocks64.restype = I
            self.lib.orc_match_blocks64.argtypes = [P, I, I, P, I, I, P, P, P, I, I, D, P]

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    # ---- census
    def census(self, img: np.ndarray, ow=None, oh=None) -> np.ndarray:
        h, w = img.shape
        ow = w if ow is None else ow
        oh = h if oh is None else oh
        out = np.zeros((oh, ow), np.uint32)
        st = self.fn("census_transform")(img.ctypes.data, w, h, ow, oh, out.ctypes.data)
        assert st == 0, st
        return out

    def census64(self, img: np.ndarray, ow=None, oh=None) -> np.ndarray:
        h, w = img.shape
        ow = w if ow is None else ow
        oh = h if oh is None else oh
        out = np.zeros((oh, ow), np.uint64)
        st = self.lib.orc_census_transform64(img.ctypes.data, w, h, ow, oh, out.ctypes.data)
        assert st == 0, st
        return out

    def sgm(self, left, right, nd, d_lo, p1, p2) -> np.ndarray:
        h, w = left.shape
        out = np.zeros((h, w), np.int16)
        st = self.fn("sgm_disparity")(left.ctypes.data, right.ctypes.data, w, h, nd, d_lo, p1, p2, out.ctypes.data)
        assert st == 0, st
        return out

    def census_rois(self, img, ow, oh, rois) -> np.ndarray:
        h, w = img.shape
        r = (_abi.Rect * max(len(rois), 1))(*[_abi.Rect(*q) for q in rois])
        out = np.zeros((oh, ow), np.uint32)
        st = self.fn("census_transform_rois")(img.ctypes.data, w, h, ow, oh, C.addressof(r), len(rois),
                                              out.ctypes.data)
        assert st == 0, st
        return out

    # ---- matcher: blocks = [(points[(x,y)], (dxmin,dxmax,dymin,dymax))]
    def match(self, L: np.ndarray, R: np.ndarray, blocks, mode=1, tau_v=1.0):
        offs = np.zeros(len(blocks) + 1, np.int64)
        pts = []
        for i, (p, _) in enumerate(blocks):
            pts.extend(p)
            offs[i + 1] = len(pts)
        pa = np.ascontiguousarray(np.asarray(pts, np.int32).reshape(-1, 2))
        rg = (_abi.SearchRange * max(len(blocks), 1))(*[_abi.SearchRange(*r) for _, r in blocks])
        out = (_abi.MatchResult * max(len(blocks), 1))()
        wide = np.asarray(L).dtype == np.uint64
        L = np.ascontiguousarray(L, np.uint64 if wide else np.uint32)
        R = np.ascontiguousarray(R, np.uint64 if wide else np.uint32)
        fn = self.lib.orc_match_blocks64 if wide else self.fn("match_blocks")
        st = fn(L.ctypes.data, L.shape[1], L.shape[0], R.ctypes.data, R.shape[1],
                                     R.shape[0], pa.ctypes.data, offs.ctypes.data, C.addressof(rg),
                                     len(blocks), mode, tau_v, C.addressof(out))
        return st, list(out)[:len(blocks)]

    # ---- object ranger
    def estimate(self, left, right, dets, cfg: _abi.RangerConfig, focal=0.0, baseline=0.0, cache=None):
        h, w = left.shape
        n = len(dets)
        arr = (_abi.Detection * max(n, 1))(*dets)
        out = (_abi.ObjectDisparity * max(n, 1))()
        n_out = C.c_int()
        stats = _abi.RangerStats()
        st = self.fn("estimate_object_disparities")(
            left.ctypes.data, right.ctypes.data, w, h, C.addressof(arr), n, C.byref(cfg),
            C.byref(cache) if cache is not None else None, focal, baseline, C.addressof(out), C.byref(n_out),
            C.byref(stats))
        assert st == 0, st
        return list(out)[:n_out.value], stats

    def bm(self, left, right, p: _abi.BmParams):
        h, w = left.shape
        out = np.zeros((h, w), np.int16)
        st = self.fn("bm_disparity")(left.ctypes.data, right.ctypes.data, w, h, C.byref(p), out.ctypes.data)
        return st, out

    def autorect(self, left, right, roi, dmin, dmax, p: _abi.BmParams):
        h, w = left.shape
        r = _abi.Rect(*roi)
        best = C.c_int32()
        counts = np.zeros(dmax - dmin + 1, np.int64)
        st = self.fn("auto_rect_search")(left.ctypes.data, right.ctypes.data, w, h, C.byref(r), dmin, dmax,
                                         C.byref(p), C.byref(best), counts.ctypes.data)
        return st, best.value, counts


def oracle() -> Checker:
    return Checker(ORACLE_SO, "orc_")


def reference() -> Checker:
    return Checker(REF_SO, "ref_")


def have_reference() -> bool:
    return os.path.exists(REF_SO)


class RefFirst:
    """The GPU parity tests' checker: the reference itself (oracle/_ref) for
    everything it implements, the C restatement for the 9x7 / uint64
    extension (the reference has no 9x7 window) and restatement-only entry
    points."""
    kind = "reference"

    def __init__(self):
        self.ref, self.orc = reference(), oracle()

    def __getattr__(self, name):
        return getattr(self.ref, name)

    def estimate(self, left, right, dets, cfg, *a, **k):
        return (self.orc if cfg.census_9x7 else self.ref).estimate(left, right, dets, cfg, *a, **k)

    def match(self, L, R, blocks, mode=1, tau_v=1.0):
        wide = np.asarray(L).dtype == np.uint64
        return (self.orc if wide else self.ref).match(L, R, blocks, mode, tau_v)

    def census64(self, *a, **k):
        return self.orc.census64(*a, **k)

    def autorect_mt(self, left, right, roi, dmin, dmax, p: _abi.BmParams, workers: int):
        """auto_rect_search + per-delta counts at `workers` host threads."""
        h, w = left.shape
        r = _abi.Rect(*roi)
        best = C.c_int32()
        counts = np.zeros(dmax - dmin + 1, np.int64)
        fn = self.ref.lib.ref_auto_rect_search_mt
        fn.restype, fn.argtypes = I, [P, P, I, I, P, I, I, P, I, P, P]
        st = fn(left.ctypes.data, right.ctypes.data, w, h, C.byref(r), dmin, dmax, C.byref(p), workers,
                C.byref(best), counts.ctypes.data)
        return st, best.value, counts


def checker():
    """oracle/_ref where it was built (the reference compiled in place), else the restatement."""
    return RefFirst() if have_reference() else oracle()
