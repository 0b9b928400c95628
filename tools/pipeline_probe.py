"""Probe: does splitting a small per-GPU batch over several contexts (each
with its own stream) overlap one group's latency-bound scan tail with the
other groups' work? S sequences x F frames (config-2 scenes), device-resident
images; frames/s for 1, 2 and 4 contexts, optionally staggered by one frame.

    python tools/pipeline_probe.py [S] [F]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, 1242, 375, 128)
    sgm = tsgm.SgmParams(10, 120, 8, 0, 128)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    L = torch.empty((S, F, 375, 1242), dtype=torch.uint8)
    R = torch.empty_like(L)
    mot = np.zeros((S, F, 12))
    for i in range(S):
        _, _, P, _ = render(SceneConfig.baseline_config(2, seed=i, n_movers=i % 5, frames=F),
                            out_left=L[i].numpy(), out_right=R[i].numpy())
        for k in range(1, F):
            Rm, t = tsgm.relative_motion(P[k - 1], P[k])
            mot[i, k, :9], mot[i, k, 9:] = Rm.ravel(), t
        mot[i, 0, :9] = np.eye(3).ravel()
    dL, dR = L.cuda(), R.cuda()
    torch.cuda.synchronize()

    def run(groups, stagger):
        size = S // groups
        engs = [tsgm.Engine(tsgm.EngineConfig(calib, sgm, filt, max_slots=size, keep_volumes=False))
                for _ in range(groups)]
        idx = [list(range(g * size, (g + 1) * size)) for g in range(groups)]

        def one_pass():
            for e in engs:
                for s in range(size):
                    e.reset(s)
            for k in range(F + (groups - 1 if stagger else 0)):
                for g, e in enumerate(engs):
                    kk = k - (g if stagger else 0)
                    if 0 <= kk < F:
                        e.step_device(list(range(size)), [dL[i, kk].data_ptr() for i in idx[g]],
                                      [dR[i, kk].data_ptr() for i in idx[g]], mot[idx[g], kk, :])
            for e in engs:
                e.sync()
        one_pass()
        t0 = time.perf_counter()
        reps = 2
        for _ in range(reps):
            one_pass()
        dt = (time.perf_counter() - t0) / reps
        for e in engs:
            e.close()
        return S * F / dt

    for groups, stagger in ((1, False), (2, False), (2, True), (4, False), (4, True)):
        if S % groups:
            continue
        print(f"S={S} groups={groups} stagger={stagger}: {run(groups, stagger):.0f} frames/s",
              flush=True)


if __name__ == "__main__":
    main()
