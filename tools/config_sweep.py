"""BASELINE config 3 — window-size sweep on the B200.

For full-range SGM at D=128 and D=256 (every frame full range: the state is
reset each frame, as the reference's benchmark full mode, eval.cpp:125-137)
and reduced windows of half-width h in {2, 4, 8, 16} (stddev ranges with a
vanishing gain and min_range_halfwidth = h, so windows are exactly 2h+1 levels
before edge clamping), run S sequences x F frames of the config-3 scene and
report frames/s, Gdisparity-evals/s (cells/s) and the standalone C->S
aggregation's fraction of the HBM roofline (B_agg = 3N + 4P per frame).

    python tools/config_sweep.py [S] [F] > profiles/r01_config3_sweep.json
"""
import json
import os
import sys

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


def run(name, d_max, half, S, F, frames):
    calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, 1242, 375, d_max)
    sgm = tsgm.SgmParams(10, 120, 8, 0, d_max)
    full = half is None
    filt = tsgm.FilterConfig(p_init=max(4096.0, d_max * d_max / 4.0), range_use_stddev=True,
                             range_stddev_gain=1e-9 if not full else 3.0,
                             min_range_halfwidth=half if not full else 2)
    eng = tsgm.Engine(tsgm.EngineConfig(calib, sgm, filt, max_slots=S, keep_volumes=False))
    slots = list(range(S))
    L, R, M = frames
    ms_total, cells = 0.0, 0
    for rep in range(2):  # warm-up pass, then the timed pass
        for s in slots:
            eng.reset(s)
        eng.sync()
        eng.timer_begin()
        for k in range(F):
            if full:
                for s in slots:
                    eng.reset(s)
            eng.step(slots, [L[i][k] for i in range(S)], [R[i][k] for i in range(S)],
                     [M[i][k] for i in range(S)])
        ms = eng.timer_end()
        if rep == 1:
            ms_total = ms
    # cells of the last frame, and the standalone aggregation on its volumes
    agg_ms, agg_cells = eng.bench_aggregate(slots, reps=5)
    b_agg = 3.0 * agg_cells + 4.0 * 1242 * 375 * S
    eng.close()
    return {"setting": name, "d_max": d_max, "half_width": half, "sequences": S, "frames": F,
            "ms_per_pass_incl_h2d": round(ms_total, 3),
            "frames_per_s": round(S * F / (ms_total * 1e-3), 1),
            "last_frame_cells": int(agg_cells),
            "aggregation_ms": round(agg_ms, 4),
            "aggregation_gcells_per_s": round(agg_cells / (agg_ms * 1e-3) / 1e9, 2),
            "aggregation_hbm_frac": round(b_agg / (agg_ms * 1e-3) / 1e9 / peak(), 4)}


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    L, R, M = [], [], []
    for s in range(S):
        cfg = SceneConfig.baseline_config(3, seed=s, frames=F)
        l, r, P, _ = render(cfg)
        L.append(l)
        R.append(r)
        M.append([(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
                  for k in range(F)])
    rows = [run("full D=128", 128, None, S, F, (L, R, M)),
            run("full D=256", 256, None, S, F, (L, R, M))]
    for h in (2, 4, 8, 16):
        rows.append(run(f"reduced h={h}", 128, h, S, F, (L, R, M)))
    print(json.dumps({"config": "BASELINE configs[3] window sweep, 1242x375, 8 paths, P1=10 P2=120",
                      "note": "full range: state reset every frame; reduced: 2h+1-level windows",
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
