"""Single-sequence configs (BASELINE configs 0, 1, 3): per-frame
latency on the B200 against the reference CPU build at threads=1 and
threads=nproc, frame 0 and the mean/median of frames >= 1 (as eval.hpp:73 /
eval.cpp:177-179 report them).

GPU: one sequence, all frames, through the host-image API (tsgm_step; H2D of
both images inside each frame's CUDA-event bracket). Reference: the in-place
build (oracle/_ref/libtsgm_ref.so, tsgm::step) on a bounded prefix of the
same frames. Config 3's full-range rows reset the state every frame (the
full-range step; the reference's benchmark full mode is sgm_match + median,
eval.cpp:125-137, which the step from an empty state contains).

    python tools/config_report.py [ref_frames] > profiles/r01_config_report.json
"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def summarize(ms):
    rest = ms[1:]
    return {"frame0_ms": round(ms[0], 3),
            "mean_ms_frames_ge1": round(statistics.mean(rest), 3) if rest else None,
            "median_ms_frames_ge1": round(statistics.median(rest), 3) if rest else None}


def gpu_run(L, R, mots, calib, params, filt, reset_each):
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=1, keep_volumes=False))
    out = []
    for rep in range(2):  # warm-up pass, then the timed pass
        eng.reset(0)
        ms = []
        for k in range(len(L)):
            if reset_each:
                eng.reset(0)
            eng.sync()
            eng.timer_begin()
            eng.step([0], [L[k]], [R[k]], [mots[k]])
            ms.append(eng.timer_end())
        out = ms
    cells = eng.cells(0)
    # the standalone C->S aggregation on the last frame's volume
    agg_ms, agg_cells = eng.bench_aggregate([0], reps=5)
    eng.close()
    return out, cells, (agg_ms, agg_cells)


def ref_run(ref, L, R, mots, calib, params, filt, reset_each, frames, threads):
    state, ms = None, []
    for k in range(frames):
        if reset_each:
            state = None
        t0 = time.perf_counter()
        r = ref.step(state, L[k], R[k], mots[k][0], mots[k][1], calib, params, filt,
                     threads=threads)
        ms.append((time.perf_counter() - t0) * 1e3)
        state = (r["d"], r["p"], r["valid"])
    return ms


def main():
    ref_frames = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    from oracle import Reference
    ref = Reference()
    nproc = os.cpu_count() or 1
    rows = []
    cases = [("config 0", 0, {}, 128, None, 8), ("config 1", 1, {}, 128, None, 30)]
    cases += [("config 3 full D=128", 3, {}, 128, "full", 30),
              ("config 3 full D=256", 3, {"d_max": 256}, 256, "full", 30)]
    cases += [(f"config 3 reduced h={h}", 3, {}, 128, h, 30) for h in (2, 4, 8, 16)]
    for name, cfg_id, over, d_max, mode, frames in cases:
        cfg = SceneConfig.baseline_config(cfg_id, frames=frames, **over)
        L, R, P, _ = render(cfg)
        mots = [(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
                for k in range(frames)]
        calib = tsgm.StereoCalib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, cfg.width,
                                 cfg.height, d_max)
        params = tsgm.SgmParams(10, 120, 8, 0, d_max)
        if mode is None or mode == "full":
            filt = tsgm.FilterConfig(p_init=max(4096.0, d_max * d_max / 4.0),
                                     range_use_stddev=True, range_stddev_gain=3.0)
        else:
            filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=1e-9,
                                     min_range_halfwidth=mode)
        reset_each = mode == "full"
        gms, cells, (agg_ms, agg_cells) = gpu_run(L, R, mots, calib, params, filt, reset_each)
        agg_frac = (3.0 * agg_cells + 4.0 * cfg.width * cfg.height) / (agg_ms * 1e-3) / (peak() * 1e9)
        nf = min(ref_frames, frames)
        r1 = ref_run(ref, L, R, mots, calib, params, filt, reset_each, nf, 1)
        rn = ref_run(ref, L, R, mots, calib, params, filt, reset_each, nf, nproc)
        g = summarize(gms)
        c1, cn = summarize(r1), summarize(rn)
        key = "mean_ms_frames_ge1" if frames > 1 else "frame0_ms"
        rows.append({"config": name, "frames": frames, "width": cfg.width, "height": cfg.height,
                     "d_max": d_max, "last_frame_cells": cells,
                     "gpu": g, "gpu_frames_per_s": round(1e3 * frames / sum(gms), 1),
                     "gpu_gdisp_evals_per_s_last_frame": round(cells / (gms[-1] * 1e-3) / 1e9, 2),
                     "aggregation_ms": round(agg_ms, 4), "aggregation_hbm_frac": round(agg_frac, 4),
                     "reference_threads_1": dict(c1, frames_timed=nf),
                     f"reference_threads_{nproc}": dict(cn, frames_timed=nf),
                     "speedup_vs_ref_nproc_frames_ge1": round(cn[key] / g[key], 1)
                     if cn[key] and g[key] else None})
        print(json.dumps(rows[-1]), file=sys.stderr)
    print(json.dumps({"note": "single sequence per config; GPU through tsgm_step (host images, "
                              "H2D inside each frame's event bracket); reference = in-place "
                              "build of the reference sources, tsgm::step",
                      "nproc": nproc, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
