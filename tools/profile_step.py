"""Small driver for ncu captures: a few batched frames of the BASELINE config-2
workload (S sequences x F frames), then the standalone C->S aggregation on the
last frame's volumes. Usage: python tools/profile_step.py [S] [F] [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, 1242, 375, 128)
    sgm = tsgm.SgmParams(10, 120, 8, 0, 128)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    eng = tsgm.Engine(tsgm.EngineConfig(calib, sgm, filt, max_slots=S))
    seqs = [render(SceneConfig.baseline_config(2, seed=s, n_movers=s % 5, frames=F)) for s in range(S)]
    for k in range(F):
        mots = [(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
                for (_, _, P, _) in seqs]
        eng.step(list(range(S)), [L[k] for (L, _, _, _) in seqs], [R[k] for (_, R, _, _) in seqs],
                 mots)
    eng.sync()
    ms, cells = eng.bench_aggregate(list(range(S)), reps=reps)
    b = 3.0 * cells + 4.0 * 1242 * 375 * S
    print(f"aggregation: {ms:.3f} ms for {cells/1e6:.1f} M cells -> {b/ms/1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
