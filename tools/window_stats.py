"""Window statistics of the config-2 workload (CPU, the reference algorithm
through the C oracle — test infrastructure): for reduced frames, the share of
full-range windows (pixels and cells), the narrow windows' level and quad
counts, and the utilisation of the scan's 4-window full-range passes (G = 8
lanes x 4 quads) over 32-pixel warp steps. The aggregation's design (DESIGN.md
section 4) is tuned to these numbers.

    python tools/window_stats.py [seed] [frames] > profiles/r02_window_stats.json
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Port  # noqa: E402
from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402


def main():
    seed = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    port = Port()
    calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, 1242, 375, 128)
    params = tsgm.SgmParams(10, 120, 8, 0, 128)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    cfg = SceneConfig.baseline_config(2, seed=seed, n_movers=seed % 5, frames=F)
    L, R, P, _ = render(cfg)
    state, rows = None, []
    for k in range(F):
        Rm, t = (np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
        ref = port.step(state, L[k], R[k], Rm, t, calib, params, filt, debug=True)
        state = (ref["d"], ref["p"], ref["valid"])
        if k == 0:
            continue
        lo, hi = ref["lo"].astype(int), ref["hi"].astype(int)
        n = hi - lo + 1
        nq = (hi >> 2) - (lo >> 2) + 1
        full = n == 128
        c = np.pad(full, ((0, 0), (0, 1248 - 1242))).reshape(375, -1, 32).sum(2)
        passes = np.ceil(c / 4)
        rows.append({
            "frame": k, "cells_per_px": round(float(n.mean()), 2),
            "full_px_pct": round(100 * float(full.mean()), 2),
            "full_cells_pct": round(100 * float(n[full].sum() / n.sum()), 2),
            "narrow_levels_hist": {int(v): int(x) for v, x in enumerate(np.bincount(n[~full])) if x},
            "narrow_quads_hist": {int(v): int(x) for v, x in enumerate(np.bincount(nq[~full])) if x},
            "full_pass_utilisation_vertical": round(float(c.sum() / max(1.0, 4 * passes.sum())), 3),
            "warp_steps_without_full_window_pct": round(100 * float((c == 0).mean()), 1)})
    print(json.dumps({"workload": f"config 2 sequence seed {seed} ({seed % 5} movers), reduced frames",
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
