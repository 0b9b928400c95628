"""Profiling probe: the standalone aggregation of 64 config-2 sequences' 4th
frame with only some directions (TSGM_SCAN_DIRS bitmask: 3 = horizontal,
12 = vertical, 240 = diagonal, 255 = all), to see where the scan's time goes
per direction class. Run under ncu's launch list for per-kernel times.

    python tools/scan_dirs_probe.py [S]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    F = 4
    calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, 1242, 375, 128)
    sgm = tsgm.SgmParams(10, 120, 8, 0, 128)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    eng = tsgm.Engine(tsgm.EngineConfig(calib, sgm, filt, max_slots=S, keep_volumes=False))
    seqs = [render(SceneConfig.baseline_config(2, seed=s, n_movers=s % 5, frames=F)) for s in range(S)]
    for k in range(F):
        mots = [(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
                for (_, _, P, _) in seqs]
        eng.step(list(range(S)), [L[k] for (L, _, _, _) in seqs], [R[k] for (_, R, _, _) in seqs],
                 mots)
    eng.sync()
    for mask in (255, 3, 12, 240, 252):
        os.environ["TSGM_SCAN_DIRS"] = str(mask)
        ms, cells = eng.bench_aggregate(list(range(S)), reps=2)
        print(f"dirs {mask:3d}: {ms:.3f} ms (scan + combine) for {cells / 1e6:.1f} M cells", flush=True)
    os.environ.pop("TSGM_SCAN_DIRS")


if __name__ == "__main__":
    main()
