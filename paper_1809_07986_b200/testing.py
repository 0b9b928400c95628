"""Uniform numpy-level adapter over the GPU path, with the same method names
as the CPU checkers in oracle/ (so one parity test body runs against both).
Every method calls the CUDA library; nothing falls back to the CPU."""
from __future__ import annotations

import numpy as np

from . import tsgm


class GpuBackend:
    kind = "gpu"
    _shared = None

    @classmethod
    def shared(cls):
        if cls._shared is None:
            cls._shared = cls()
        return cls._shared

    def census(self, img):
        return tsgm.census_transform(img)

    def cost_volume(self, left, right, lo, hi, threads=1):
        return tsgm.build_cost_volume(left, right, lo, hi)

    def aggregate(self, cost, lo, hi, params):
        return tsgm.aggregate_paths(cost, lo, hi, params)

    def wta(self, agg, lo, hi):
        return tsgm.winner_takes_all(agg, lo, hi)

    def median(self, d, valid):
        return tsgm.median_refine(d, valid)

    def sgm_match(self, left, right, lo, hi, params, threads=1):
        return tsgm.sgm_match(left, right, lo, hi, params)

    def relative_motion(self, prev12, cur12):
        return tsgm.relative_motion(prev12, cur12)

    def homography(self, R, t, calib):
        return tsgm.disparity_homography(R, t, calib)

    def warp(self, d, p, valid, H, d_max):
        return tsgm.warp_state_ex(d, p, valid, H, d_max)

    def predict(self, d, p, valid, R, t, calib, filt):
        return tsgm.predict(d, p, valid, R, t, calib, filt)

    def reject(self, d, p, valid, filt):
        return tsgm.reject_discontinuities(d, p, valid, filt)

    def fill(self, d, p, valid):
        return tsgm.fill_zoom_holes(d, p, valid)

    def ranges(self, d, p, valid, calib, filt):
        return tsgm.derive_search_ranges(d, p, valid, calib, filt)

    def correct(self, d, p, valid, md, mv, filt):
        return tsgm.correct(d, p, valid, md, mv, filt)

    def step(self, state, left, right, R, t, calib, params, filt, threads=1, debug=False,
             mask_tau=3.0):
        if not debug:
            return tsgm.step(state, left, right, R, t, calib, params, filt)
        # debug: run through an Engine so the intermediates can be fetched
        h, w = np.asarray(left).shape
        cal = tsgm._as(calib, tsgm.StereoCalib)
        cal = tsgm.StereoCalib(cal.focal_px, cal.cx, cal.cy, cal.baseline_m, w, h, cal.d_max)
        eng = tsgm.Engine(tsgm.EngineConfig(cal, tsgm._as(params, tsgm.SgmParams),
                                            tsgm._as(filt, tsgm.FilterConfig), 1,
                                            mask_tau=mask_tau))
        try:
            if state is not None:
                eng.set_state(0, *state)
            eng.step([0], [left], [right], [(R, t)])
            out = dict(d=eng.fetch(0, "state_d"), p=eng.fetch(0, "state_p"),
                       valid=eng.fetch(0, "state_valid"), export_d=eng.fetch(0, "export_d"),
                       export_valid=eng.fetch(0, "export_valid"), diff=eng.fetch(0, "diff"),
                       pred_d=eng.fetch(0, "pred_d"), pred_p=eng.fetch(0, "pred_p"),
                       pred_valid=eng.fetch(0, "pred_valid"), lo=eng.fetch(0, "lo"),
                       hi=eng.fetch(0, "hi"), meas_d=eng.fetch(0, "meas_d"),
                       meas_valid=eng.fetch(0, "meas_valid"), mask=eng.fetch(0, "mask"))
        finally:
            eng.close()
        return out

    # ---- box detector (motion_detect.cpp) ----
    def integral_image(self, m):
        return tsgm.integral_image(m)

    def candidates(self, diff, cfg, threads=1):
        return tsgm.detect_candidate_windows(diff, cfg)

    def greedy_merge(self, boxes, cfg):
        return tsgm.greedy_merge(boxes, cfg)

    def detect(self, diff, cfg, threads=1):
        return tsgm.detect_moving_objects(diff, cfg)

    # ---- outlier metric (eval.cpp) ----
    def count_outliers(self, d, valid, gt, abs_thresh=3.0, rel_thresh=0.05, strict=False):
        return tsgm.count_outliers(d, valid, gt, tsgm.OutlierOptions(abs_thresh, rel_thresh, strict))

    # noise calibration, in the oracle's dict format
    @staticmethod
    def _frames(gt, poses=None, left=None, right=None):
        out = []
        for k in range(len(gt)):
            out.append(tsgm.SequenceFrame(
                k, None if left is None else left[k], None if right is None else right[k],
                None if poses is None else np.asarray(poses[k]).reshape(3, 4), gt[k]))
        return out

    @staticmethod
    def _est(e):
        h = e.hist
        return dict(variance=e.variance, mean=h.mean(), within_1px=h.fraction_within_1px(),
                    samples_used=e.samples_used, total=h.total(), underflow=h.underflow,
                    overflow=h.overflow, counts=h.counts, sum=h.sum, sum_sq=h.sum_sq)

    def process_noise(self, gt, poses, calib, opts):
        return self._est(tsgm.estimate_process_noise(self._frames(gt, poses), calib, opts))

    def measurement_noise(self, left, right, gt, params, opts):
        return self._est(tsgm.estimate_measurement_noise(
            self._frames(gt, None, left, right), params, 1, opts))

    def error_map(self, gt, poses, calib):
        return tsgm.accumulate_error_map(self._frames(gt, poses), calib)
