"""Profiling probe: standalone aggregation of S config-2 sequences' 4th frame
per direction class (TSGM_SCAN_DIRS) and per environment setting.

    python tools/scan_dirs_probe2.py S "K1=V1,K2=V2" "K1=V3" ...
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402


def main():
    S = int(sys.argv[1])
    settings = sys.argv[2:] or [""]
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
    for st in settings:
        kv = dict(x.split("=") for x in st.split(",") if x)
        os.environ.update(kv)
        row = []
        for mask in [int(m) for m in os.environ.get("PROBE_MASKS", "255,3,12,240").split(",")]:
            os.environ["TSGM_SCAN_DIRS"] = str(mask)
            ms, cells = eng.bench_aggregate(list(range(S)), reps=3)
            row.append(f"{mask}:{ms:.3f}")
        os.environ.pop("TSGM_SCAN_DIRS")
        print(f"S={S} [{st}] {eng.last_kernels()} ms(scan+combine) " + " ".join(row), flush=True)
        for k_ in kv:
            os.environ.pop(k_)


if __name__ == "__main__":
    main()
