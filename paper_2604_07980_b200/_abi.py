"""ctypes mirror of include/ranger_cuda.h (the library's C ABI).

Struct layouts here must match the header field for field; tests/test_abi_cpu.py
checks the sizes against the compiled library's expectations and that every
symbol the header declares is exported.
"""
from __future__ import annotations

import ctypes as C

RG_OK, RG_EINVAL, RG_ECUDA, RG_ENOMEM, RG_EOVERFLOW = 0, 1, 2, 3, 4
RG_KIND_FAR, RG_KIND_CLOSE = 0, 1
RG_MATCH_FORWARD, RG_MATCH_FWD_BWD = 0, 1


class Rect(C.Structure):
    _fields_ = [("x0", C.c_int32), ("y0", C.c_int32), ("x1", C.c_int32), ("y1", C.c_int32)]


class SearchRange(C.Structure):
    _fields_ = [("dx_min", C.c_int32), ("dx_max", C.c_int32), ("dy_min", C.c_int32), ("dy_max", C.c_int32)]


class MatchResult(C.Structure):
    _fields_ = [
        ("dx_int", C.c_int32), ("dy_int", C.c_int32), ("dx_subpix", C.c_double), ("cost", C.c_double),
        ("cost_minus", C.c_double), ("cost_plus", C.c_double), ("valid_points", C.c_int32),
        ("verified", C.c_int32), ("has_value", C.c_int32), ("n_points", C.c_int32),
    ]


class Detection(C.Structure):
    _fields_ = [("cx", C.c_double), ("cy", C.c_double), ("w", C.c_double), ("h", C.c_double),
                ("class_id", C.c_int32), ("id", C.c_int32)]


class RangerConfig(C.Structure):
    _fields_ = [
        ("tau_s", C.c_double), ("close_scale", C.c_int32), ("grid_side_points", C.c_int32),
        ("max_total_points", C.c_int32), ("close_block_side_points", C.c_int32), ("tau_d", C.c_double),
        ("n_min", C.c_int32), ("max_objects", C.c_int32), ("tau_v", C.c_double),
        ("crop_x0", C.c_double), ("crop_y0", C.c_double), ("crop_x1", C.c_double), ("crop_y1", C.c_double),
        ("dx_max_far", C.c_int32), ("dx_max_close", C.c_int32),
        ("census_9x7", C.c_int32), ("reserved", C.c_int32),
    ]


class ObjectDisparity(C.Structure):
    _fields_ = [("det_id", C.c_int32), ("kind", C.c_int32), ("n_blocks_used", C.c_int32),
                ("valid", C.c_int32), ("disparity", C.c_double), ("z_cam", C.c_double)]


class RangerStats(C.Structure):
    _fields_ = [("query_points", C.c_int64), ("image_pixels", C.c_int64), ("n_far", C.c_int32),
                ("n_close", C.c_int32)]


class CensusCache(C.Structure):
    _fields_ = [("full_left", C.c_void_p), ("full_right", C.c_void_p), ("scaled_left", C.c_void_p),
                ("scaled_right", C.c_void_p), ("has_full", C.c_int32), ("has_scaled", C.c_int32)]


class BmParams(C.Structure):
    _fields_ = [("num_disparities", C.c_int32), ("block_size", C.c_int32), ("min_disparity", C.c_int32),
                ("downscale", C.c_int32), ("texture_threshold", C.c_double), ("uniqueness_ratio", C.c_double)]


class BoxStats(C.Structure):
    _fields_ = [("valid", C.c_int32), ("count", C.c_int32), ("median", C.c_double), ("variance", C.c_double)]


class SgmParams(C.Structure):
    _fields_ = [("num_disparities", C.c_int32), ("min_disparity", C.c_int32), ("p1", C.c_int32), ("p2", C.c_int32)]


class RectSearchConfig(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("delta_min", C.c_int32), ("delta_max", C.c_int32), ("window", C.c_int32),
                ("rate_limit", C.c_double), ("bm", BmParams)]


RECT_MAX_WINDOW = 64


class RectState(C.Structure):
    _fields_ = [("window", C.c_int32), ("n_hist", C.c_int32), ("next", C.c_int32), ("pad", C.c_int32),
                ("delta_max", C.c_double), ("current", C.c_double), ("history", C.c_int32 * RECT_MAX_WINDOW)]


class FrameBatch(C.Structure):
    _fields_ = [
        ("n_frames", C.c_int32), ("width", C.c_int32), ("height", C.c_int32), ("pitch", C.c_int32),
        ("frame_stride", C.c_int64), ("d_left", C.c_void_p), ("d_right", C.c_void_p),
        ("d_dets", C.c_void_p), ("d_det_offsets", C.c_void_p), ("max_dets_per_frame", C.c_int32),
        ("out_stride", C.c_int32), ("d_out", C.c_void_p), ("d_out_count", C.c_void_p),
        ("focal_px", C.c_double), ("baseline_m", C.c_double), ("d_left_shift", C.c_void_p),
        ("d_out_index", C.c_void_p),
    ]


class Calibration(C.Structure):
    _fields_ = [("f", C.c_double), ("b", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("h_cam", C.c_double), ("R", C.c_double * 9), ("t", C.c_double * 3)]


class Vec3(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("z", C.c_double)]


class RadarDetection(C.Structure):
    _fields_ = [("position", Vec3), ("extent", Vec3), ("id", C.c_int32), ("pad", C.c_int32)]


RG_VOTE_MAX_BINS = 1025


class VoteState(C.Structure):
    _fields_ = [("k_px", C.c_int32), ("n_bins", C.c_int32), ("lambda_", C.c_double),
                ("smooth_sigma_px", C.c_double), ("smoothed_offset", C.c_double),
                ("memory", C.c_double * RG_VOTE_MAX_BINS)]


class ObjRefinerState(C.Structure):
    _fields_ = [("prev_offset", C.c_double), ("beta", C.c_double), ("r_max", C.c_double), ("w_p", C.c_double),
                ("tau", C.c_double), ("rate_limit", C.c_double)]


class ClassWidth(C.Structure):
    _fields_ = [("class_id", C.c_int32), ("pad", C.c_int32), ("width_m", C.c_double)]


class RecordParams(C.Structure):
    _fields_ = [("calib", Calibration), ("class_widths", C.c_void_p), ("n_class_widths", C.c_int32),
                ("object_refiner", C.c_int32), ("obj_cand_half_px", C.c_double), ("obj_cand_step_px", C.c_double),
                ("fuse_sanity_ratio", C.c_double)]


class DepthRecord(C.Structure):
    _fields_ = [("frame_id", C.c_int32), ("det_id", C.c_int32), ("disparity", C.c_double), ("valid", C.c_int32),
                ("source", C.c_int32), ("clp_by_stereo", C.c_double), ("clp_by_gpt", C.c_double),
                ("clp_by_size", C.c_double), ("z_fused", C.c_double)]


class RefinerLog(C.Structure):
    _fields_ = [("frame_id", C.c_int32), ("pad", C.c_int32), ("rect_delta", C.c_double),
                ("radar_offset", C.c_double), ("obj_offset", C.c_double)]


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
        ("texture_cell_px", C.c_double),
    ]


P = C.c_void_p
I = C.c_int
I64 = C.c_int64
D = C.c_double

# name -> (restype, argtypes); every symbol of include/ranger_cuda.h
SIGNATURES = {
    "rg_ctx_create": (I, [I, C.POINTER(P)]),
    "rg_ctx_destroy": (None, [P]),
    "rg_last_error": (C.c_char_p, [P]),
    "rg_create_error": (C.c_char_p, []),
    "rg_build_info": (C.c_char_p, []),
    "rg_selftest_division": (I, [P, I, C.POINTER(C.c_int64)]),
    "rg_get_transfer": (I, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "rg_set_profiling": (I, [P, I]),
    "rg_set_overlap": (I, [P, I]),
    "rg_set_census_rois": (I, [P, I]),
    "rg_sync": (I, [P]),
    "rg_set_sync_mode": (I, [P, I]),
    "rg_get_counters": (I, [P, P, P, P]),
    "rg_reset_counters": (I, [P]),
    "rg_get_work": (I, [P, P, P]),
    "rg_census_code_at": (I, [P, P, I, I, I, I, P]),
    "rg_census_transform": (I, [P, P, I, I, I, I, P]),
    "rg_census_transform_rois": (I, [P, P, I, I, I, I, P, I, P]),
    "rg_match_blocks": (I, [P, P, I, I, P, I, I, P, P, P, I, I, D, P]),
    "rg_census_transform64": (I, [P, P, I, I, I, I, P]),
    "rg_match_blocks64": (I, [P, P, I, I, P, I, I, P, P, P, I, I, D, P]),
    "rg_validate_ranger_config": (I, [P, P]),
    "rg_select_objects": (I, [P, P, I, P, P, P]),
    "rg_find_occluders": (I, [P, P, I, P, P]),
    "rg_sample_query_points": (I, [P, P, I, P, I, P, I, I, P, P, P, I, I64, P]),
    "rg_aggregate_close_disparities": (I, [P, P, I, D, I, P, P, P]),
    "rg_estimate_object_disparities": (I, [P, P, P, I, I, P, I, P, P, D, D, P, P, P]),
    "rg_range_frames": (I, [P, P, P, P]),
    "rg_range_frames_host": (I, [P, P, P, I, P]),
    "rg_shard_bounds": (I, [I, I, I, P, P]),
    "rg_vote_state_init": (I, [P, I, D, D]),
    "rg_radar_refine_step": (I, [P, P, I, I, P, I, P, P, P]),
    "rg_radar_refine_step_host": (I, [P, P, I, I, P, I, P, P, P]),
    "rg_radar_boxes": (I, [P, I, P, I, I, P, P, P]),
    "rg_radar_vote_update": (I, [P, P, P, I, P, P]),
    "rg_dense_objects_refined": (I, [P, P, P, I, I, P, I, P, P, D, D, D, P, I, P, P, P, P, P, P, P]),
    "rg_multi_create": (I, [P, I, P]),
    "rg_multi_destroy": (None, [P]),
    "rg_multi_last_error": (C.c_char_p, [P]),
    "rg_multi_range_host": (I, [P, P, P, I, P, P, P, P]),
    "rg_rect_state_init": (I, [P, I, D]),
    "rg_filter_offset": (I, [P, I, P]),
    "rg_range_sequence": (I, [P, P, P, P, P, P, P, P, P]),
    "rg_obj_refiner_state_init": (I, [P]),
    "rg_make_calibration": (I, [D, D, D, D, D, P]),
    "rg_frame_records": (I, [P, I, I, I, I, P, I, P, P, I, P, I, P, D, P, P]),
    "rg_validate_bm_params": (I, [P, P]),
    "rg_bm_disparity": (I, [P, P, P, I, I, P, P]),
    "rg_auto_rect_search": (I, [P, P, P, I, I, P, I, I, P, P, P]),
    "rg_auto_rect_frames": (I, [P, P, P, I, I64, I, I, I, P, I, I, P, P, P, P]),
    "rg_box_disparity": (I, [P, P, I, I, P, I, I, I, D, D, D, P]),
    "rg_dense_objects": (I, [P, P, P, I, I, P, I, P, P, D, D, D, P, P, P, P]),
    "rg_validate_sgm_params": (I, [P, P]),
    "rg_sgm_disparity": (I, [P, P, P, I, I, P, P]),
    "rg_sgm_frames": (I, [P, P, P, I, I64, I, I, I, P, P, P]),
    "rg_sgm_cost_volume": (I, [P, P, P, I, I, P, P]),
    "rg_sgm_direction_pass": (I, [P, P, I, I, I, I, I, I, I, P]),
    "rg_render_stereo_pair": (I, [P, P, I, P, P, P, P]),
    "rg_ground_truth_detections": (I, [P, P, I, P, P]),
    "rg_render_frames_device": (I, [P, P, P, P, I, P, P, I64, P]),
}


def bind(lib: C.CDLL) -> C.CDLL:
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
