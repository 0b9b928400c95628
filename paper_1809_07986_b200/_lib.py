"""ctypes binding of the product library ``lib/libtsgm_b200.so`` (C-ABI in
``include/tsgm_b200.h``). Fails loudly when the library is missing: there is
no CPU fallback anywhere in this package."""
from __future__ import annotations

import ctypes as C
import os

from ._build import lib_path

TSGM_OK, TSGM_INVALID_ARGUMENT, TSGM_RUNTIME_ERROR = 0, 1, 2

OUT = dict(
    state_d=0, state_p=1, state_valid=2, export_d=3, export_valid=4, diff=5, mask=6,
    pred_d=7, pred_p=8, pred_valid=9, lo=10, hi=11, meas_d=12, meas_valid=13, offsets=14,
    cost=15, agg=16, subpixel=17,
)
TSGM_KEEP_VOLUMES = 1
TSGM_FORCE_SCANLINE_AGG = 2
TSGM_SUBPIXEL = 4
TSGM_STAGE_TIMINGS = 8


class StageTimingsC(C.Structure):
    """tsgm_stage_timings (StepTimings + SgmStageTimings, temporal_filter.hpp:57-62,
    sgm.hpp:59-64), seconds of device time."""
    _fields_ = [("predict_s", C.c_double), ("ranges_s", C.c_double), ("census_s", C.c_double),
                ("cost_s", C.c_double), ("aggregate_s", C.c_double), ("wta_s", C.c_double),
                ("correct_s", C.c_double)]


class SgmParamsC(C.Structure):
    _fields_ = [("p1", C.c_int32), ("p2", C.c_int32), ("paths", C.c_int32),
                ("path_set", C.c_int32), ("d_max", C.c_int32)]


class FilterConfigC(C.Structure):
    _fields_ = [("q", C.c_double), ("r", C.c_double), ("p_init", C.c_double),
                ("disc_thresh", C.c_double), ("min_range_halfwidth", C.c_int32),
                ("range_use_stddev", C.c_int32), ("range_stddev_gain", C.c_double)]


class StereoCalibC(C.Structure):
    _fields_ = [("focal_px", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("baseline_m", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("d_max", C.c_int32)]


class ConfigC(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("max_slots", C.c_int32),
                ("device", C.c_int32), ("calib", StereoCalibC), ("sgm", SgmParamsC),
                ("filter", FilterConfigC), ("mask_tau", C.c_double), ("flags", C.c_uint32),
                ("vol_slots", C.c_int32)]


_lib = None

# Every exported symbol of include/tsgm_b200.h (checked by the CPU tests).
EXPORTS = [
    "tsgm_last_error", "tsgm_create", "tsgm_destroy", "tsgm_reset", "tsgm_set_state",
    "tsgm_step", "tsgm_step_device", "tsgm_fetch", "tsgm_fetch_batch", "tsgm_cells", "tsgm_sync",
    "tsgm_timer_begin", "tsgm_timer_end", "tsgm_bench_aggregate", "tsgm_volume_slots", "tsgm_launch_count",
    "tsgm_census_transform", "tsgm_build_cost_volume", "tsgm_aggregate_paths",
    "tsgm_winner_takes_all", "tsgm_median_refine", "tsgm_sgm_match", "tsgm_relative_motion",
    "tsgm_disparity_homography", "tsgm_warp_state_ex", "tsgm_predict",
    "tsgm_reject_discontinuities", "tsgm_fill_zoom_holes", "tsgm_derive_search_ranges",
    "tsgm_correct", "tsgm_step_once", "tsgm_step_once_t", "tsgm_sgm_match_t",
    "tsgm_step_device_after", "tsgm_inputs_consumed", "tsgm_last_stage_timings",
    "tsgm_last_kernels", "tsgm_last_chunks",
    "tsgm_integral_image", "tsgm_detect_candidate_windows", "tsgm_greedy_merge",
    "tsgm_detect_moving_objects", "tsgm_detect", "tsgm_count_outliers",
    "tsgm_count_outliers_batch", "tsgm_calib_bins", "tsgm_estimate_process_noise",
    "tsgm_estimate_measurement_noise", "tsgm_accumulate_error_map", "tsgm_calib_release",
    "tsgm_quantize_disparity", "tsgm_quantize_disparity_map", "tsgm_write_disparity_png",
    "tsgm_write_disparity_png_map", "tsgm_write_export_png", "tsgm_write_export_pngs",
    "tsgm_write_boxes", "tsgm_read_disparity_png",
]


class CalibOptionsC(C.Structure):
    """tsgm_calib_options (CalibOptions, noise_calib.hpp:43-49)."""
    _fields_ = [("outlier_gate_px", C.c_double), ("bin_width", C.c_double),
                ("q_floor", C.c_double)]


class NoiseEstimateC(C.Structure):
    """tsgm_noise_estimate (NoiseEstimate + ErrorHistogram, noise_calib.hpp:14-55)."""
    _fields_ = [("variance", C.c_double), ("samples_used", C.c_int64), ("lo", C.c_double),
                ("hi", C.c_double), ("bin_width", C.c_double), ("underflow", C.c_int64),
                ("overflow", C.c_int64), ("within_1px", C.c_int64), ("total", C.c_int64),
                ("sum", C.c_double), ("sum_sq", C.c_double), ("n_bins", C.c_int32),
                ("counts", C.c_void_p)]


class OutlierOptionsC(C.Structure):
    """tsgm_outlier_options (OutlierOptions, eval.hpp:13-19)."""
    _fields_ = [("abs_thresh_px", C.c_double), ("rel_thresh", C.c_double),
                ("strict_density", C.c_int32)]


class BoxC(C.Structure):
    """tsgm_box (DetectionBox, motion_detect.hpp:24-34)."""
    _fields_ = [("x0", C.c_int32), ("y0", C.c_int32), ("x1", C.c_int32), ("y1", C.c_int32),
                ("score", C.c_double)]


class DetectConfigC(C.Structure):
    """tsgm_detect_config (DetectConfig, motion_detect.hpp:36-44)."""
    _fields_ = [("window_wh", C.c_void_p), ("n_windows", C.c_int32),
                ("score_thresh", C.c_double), ("merge_stop_iou", C.c_double),
                ("min_box_area", C.c_int64)]


def load():
    """The product library; raises if it is not built (no fallback)."""
    global _lib
    if _lib is None:
        # TSGM_LIB_VARIANT=<suffix> loads libtsgm_b200<suffix>.so (kernel-tuning builds)
        path = lib_path(f"libtsgm_b200{os.environ.get('TSGM_LIB_VARIANT', '')}.so")
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: the CUDA path is required (run __graft_entry__.build())")
        lib = C.CDLL(path)
        lib.tsgm_last_error.restype = C.c_char_p
        lib.tsgm_launch_count.restype = C.c_uint64
        lib.tsgm_launch_count.argtypes = [C.c_void_p]
        lib.tsgm_create.argtypes = [C.POINTER(ConfigC), C.POINTER(C.c_void_p)]
        lib.tsgm_destroy.argtypes = [C.c_void_p]
        for name in ("tsgm_reset",):
            getattr(lib, name).argtypes = [C.c_void_p, C.c_int32]
        lib.tsgm_set_state.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        for name in ("tsgm_step", "tsgm_step_device"):
            getattr(lib, name).argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p]
        lib.tsgm_step_device_after.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                               C.c_void_p, C.c_void_p, C.c_void_p]
        lib.tsgm_inputs_consumed.argtypes = [C.c_void_p, C.c_void_p]
        lib.tsgm_last_kernels.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
        lib.tsgm_last_chunks.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        lib.tsgm_last_stage_timings.argtypes = [C.c_void_p, C.POINTER(StageTimingsC)]
        lib.tsgm_fetch.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t]
        lib.tsgm_fetch_batch.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                         C.c_size_t]
        lib.tsgm_cells.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64)]
        lib.tsgm_sync.argtypes = [C.c_void_p]
        lib.tsgm_volume_slots.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        lib.tsgm_timer_begin.argtypes = [C.c_void_p]
        lib.tsgm_timer_end.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
        lib.tsgm_bench_aggregate.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                             C.POINTER(C.c_float), C.POINTER(C.c_uint64)]
        dc = C.POINTER(DetectConfigC)
        lib.tsgm_integral_image.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        for name in ("tsgm_detect_candidate_windows", "tsgm_detect_moving_objects"):
            getattr(lib, name).argtypes = [C.c_void_p, C.c_int32, C.c_int32, dc, C.c_void_p,
                                           C.c_int64, C.POINTER(C.c_int64)]
        lib.tsgm_greedy_merge.argtypes = [C.c_void_p, C.c_int64, dc, C.POINTER(C.c_int64)]
        lib.tsgm_detect.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, dc, C.c_void_p, C.c_int64,
                                    C.c_void_p]
        oc = C.POINTER(OutlierOptionsC)
        lib.tsgm_count_outliers.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                            C.c_int32, oc, C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int64)]
        lib.tsgm_count_outliers_batch.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                                  C.c_void_p, oc, C.c_void_p, C.c_void_p]
        co, ne = C.POINTER(CalibOptionsC), C.POINTER(NoiseEstimateC)
        lib.tsgm_calib_bins.argtypes = [co, C.POINTER(C.c_int32)]
        lib.tsgm_estimate_process_noise.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                                    C.c_void_p, C.POINTER(StereoCalibC), co, ne]
        lib.tsgm_estimate_measurement_noise.argtypes = [
            C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
            C.POINTER(SgmParamsC), co, ne]
        lib.tsgm_calib_release.argtypes = []
        lib.tsgm_quantize_disparity.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        lib.tsgm_quantize_disparity_map.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                                    C.c_void_p]
        lib.tsgm_write_disparity_png.argtypes = [C.c_char_p, C.c_void_p, C.c_int32, C.c_int32]
        lib.tsgm_write_disparity_png_map.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_int32,
                                                     C.c_int32]
        lib.tsgm_write_export_png.argtypes = [C.c_void_p, C.c_int32, C.c_char_p]
        lib.tsgm_write_export_pngs.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        lib.tsgm_write_boxes.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_int32]
        lib.tsgm_read_disparity_png.argtypes = [C.c_char_p, C.POINTER(C.c_int32),
                                                C.POINTER(C.c_int32), C.c_void_p, C.c_size_t]
        lib.tsgm_accumulate_error_map.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                                  C.c_void_p, C.POINTER(StereoCalibC), C.c_void_p]
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == TSGM_OK:
        return
    msg = load().tsgm_last_error().decode()
    if rc == TSGM_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise RuntimeError(msg)


def ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None
