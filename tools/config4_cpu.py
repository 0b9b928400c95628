"""BASELINE config 4 on the host CPU: the reference's own step() (compiled in
place, oracle/_ref/libtsgm_ref.so) on S config-4 sequences (2048x1024, D=256,
gain +-10%, occluding movers), one sequence per host thread, the first F
frames of each (frame 0 full range, then reduced frames), compute only
(eval.cpp:123-158). A bounded sample: the full 256 x 20 workload would take
hours on 16 cores.

    python tools/config4_cpu.py [S] [F] > profiles/r02_config4_cpu.json
"""
import concurrent.futures as cf
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as o  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 1)
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    threads = os.cpu_count() or 1
    try:
        impl, kind = o.reference(), "reference"
    except Exception:
        impl, kind = o.port(), "port"
    cfgs = [SceneConfig.baseline_config(4, seed=s, frames=F) for s in range(S)]
    c0 = cfgs[0]
    calib = o.Calib(c0.focal, c0.cx, c0.cy, c0.baseline, c0.width, c0.height, c0.d_max)
    sgm = o.SgmParams(10, 120, 8, 0, c0.d_max)
    filt = o.FilterConfig(q=0.5, r=1.0, p_init=16384.0, disc_thresh=2.0, min_range_halfwidth=2,
                          range_use_stddev=True, range_stddev_gain=3.0)
    seqs = [render(c, 0, F, threads=threads) for c in cfgs]
    prepared = []
    for (L, R, P, _) in seqs:
        mot = [(np.eye(3), np.zeros(3))] + [impl.relative_motion(P[k - 1], P[k]) for k in range(1, F)]
        prepared.append((L, R, mot))

    def run_seq(i):
        L, R, mot = prepared[i]
        st, times = None, []
        for k in range(F):
            t0 = time.perf_counter()
            res = impl.step(st, L[k], R[k], mot[k][0], mot[k][1], calib, sgm, filt)
            times.append(time.perf_counter() - t0)
            st = (res["d"], res["p"], res["valid"])
        return times

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        times = list(ex.map(run_seq, range(S)))
    wall = time.perf_counter() - t0
    print(json.dumps({
        "config": f"BASELINE configs[4] on the host: {S} sequences x first {F} frames, "
                  f"{c0.width}x{c0.height}, D={c0.d_max}",
        "kind": kind, "threads": threads,
        "frames_per_s": round(S * F / wall, 3), "wall_s": round(wall, 1),
        "frame0_s_mean": round(float(np.mean([t[0] for t in times])), 3),
        "frames_ge1_s_mean": round(float(np.mean([x for t in times for x in t[1:]])), 3) if F > 1 else None,
        "note": "per-frame times under full concurrency (one sequence per thread)"}, indent=1))


if __name__ == "__main__":
    main()
