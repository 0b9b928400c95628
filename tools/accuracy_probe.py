"""Accuracy sanity check of the config-2 workload, on CPU.

Runs the reference algorithm (the C oracle, oracle/ — test infrastructure) on
config-2 sequences for 30 frames and reports, per checked frame:

* the outlier rate (eval.cpp:59-85: |e| > 3 px and |e|/gt > 5%) of the
  temporal path's WTA measurement and of full-range SGM on the same frame;
* for the temporal outliers, whether the pixel had a full-range window, the
  ground truth OUTSIDE its reduced window (the filter lost track), or inside
  (SGM chose wrong within the window);
* the prediction error of valid predictions;

and checks the scene's geometry: the ground truth of frame k warped by the
filter's own forward warp (warp_state_ex with the frame's relative motion)
against the ground truth of frame k+1.

    python tools/accuracy_probe.py [seeds...]  -> JSON on stdout
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as o  # noqa: E402
from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402

W, H, D = 1242, 375, 128


def outliers(d, valid, g):
    ev = g > 0
    e = np.abs(d - g)
    return (e > 3) & (e / np.maximum(g, 1e-9) > 0.05) & ev & (valid > 0), ev


def probe(seed, frames=30, check=(0, 4, 9, 14, 19, 24, 29)):
    cfg = SceneConfig.baseline_config(2, seed=seed, n_movers=seed % 5, frames=frames)
    L, R, poses, gt = render(cfg, 0, frames, gt=True)
    calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, W, H, D)
    sgm = tsgm.SgmParams(10, 120, 8, 0, D)
    filt = tsgm.FilterConfig(q=0.5, r=1.0, p_init=4096.0, disc_thresh=2.0, min_range_halfwidth=2,
                             range_use_stddev=True, range_stddev_gain=3.0)
    port = o.port()
    st = None
    rows = []
    for k in range(frames):
        Rm, t = (np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(poses[k - 1], poses[k])
        r = port.step(st, L[k], R[k], Rm, t, calib, sgm, filt, debug=True)
        st = (r["d"], r["p"], r["valid"])
        if k not in check:
            continue
        g = gt[k].astype(np.float64)
        out, ev = outliers(r["meas_d"], r["meas_valid"], g)
        lo, hi = r["lo"].astype(int), r["hi"].astype(int)
        full = (hi - lo + 1) == D
        inwin = (g >= lo - 0.5) & (g <= hi + 0.5)
        lo0 = np.zeros((H, W), np.uint16)
        hi0 = np.full((H, W), D - 1, np.uint16)
        fd, fv = port.sgm_match(L[k], R[k], lo0, hi0, sgm)
        fout, _ = outliers(fd, fv, g)
        pv = r["pred_valid"] > 0
        n_out = max(int(out.sum()), 1)
        rows.append({
            "frame": k,
            "temporal_outlier_pct": round(100 * out.sum() / ev.sum(), 2),
            "full_range_outlier_pct": round(100 * fout.sum() / ev.sum(), 2),
            "temporal_outliers_full_window_pct": round(100 * np.sum(out & full) / n_out, 1),
            "temporal_outliers_gt_outside_window_pct": round(100 * np.sum(out & ~full & ~inwin) / n_out, 1),
            "temporal_outliers_gt_inside_window_pct": round(100 * np.sum(out & ~full & inwin) / n_out, 1),
            "pred_err_gt3px_pct": round(100 * np.sum(pv & (g > 0) & (np.abs(r["pred_d"] - g) > 3)) /
                                        max(np.sum(pv & (g > 0)), 1), 2),
            "full_window_px_pct": round(100 * full.mean(), 1),
        })
    geo = []
    for k in (0, 10, 20, frames - 2):
        g0, g1 = gt[k].astype(np.float64), gt[k + 1].astype(np.float64)
        Rm, t = tsgm.relative_motion(poses[k], poses[k + 1])
        wd, _, wv, _ = port.warp(g0, np.zeros_like(g0), (g0 > 0).astype(np.uint8),
                                 port.homography(Rm, t, calib), D)
        m = (wv > 0) & (g1 > 0)
        e = wd[m] - g1[m]
        geo.append({"frame": k, "median_err_px": float(np.median(e)),
                    "p90_abs_err_px": round(float(np.percentile(np.abs(e), 90)), 3),
                    "frac_abs_err_gt1": round(float((np.abs(e) > 1).mean()), 4)})
    return {"seed": seed, "movers": seed % 5, "frames": rows, "gt_warp_consistency": geo}


def main():
    seeds = [int(a) for a in sys.argv[1:]] or [0, 4]
    print(json.dumps({"workload": "BASELINE configs[2] scenes, reference algorithm (C oracle)",
                      "sequences": [probe(s) for s in seeds]}, indent=1))


if __name__ == "__main__":
    main()
