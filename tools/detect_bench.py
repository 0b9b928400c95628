"""Box detector throughput on the config-2 workload:
after F frames of S sequences, detect_moving_objects on every sequence's diff
map, batched (GPU SAT + scoring, host merges on worker threads), against the
reference's detect_moving_objects on the same diff maps (CPU, one call per map
with threads=nproc, as eval/cmd_detect call it).

    python tools/detect_bench.py [S] [F] > profiles/r01_detect_bench.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, 1242, 375, 128)
    params = tsgm.SgmParams(10, 120, 8, 0, 128)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=S, keep_volumes=False))
    seqs = [render(SceneConfig.baseline_config(2, seed=s, n_movers=s % 5, frames=F))
            for s in range(S)]
    slots = list(range(S))
    for k in range(F):
        mots = [(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
                for (_, _, P, _) in seqs]
        eng.step(slots, [s[0][k] for s in seqs], [s[1][k] for s in seqs], mots)
    eng.sync()
    cfg = tsgm.DetectConfig()
    eng.detect(slots, cfg)  # warm
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        boxes = eng.detect(slots, cfg)
    gpu_s = (time.perf_counter() - t0) / reps
    diffs = [eng.fetch(s, "diff") for s in slots]
    eng.close()
    from oracle import Reference
    from oracle.oracle import DetectConfig
    ref = Reference()
    nproc = os.cpu_count() or 1
    sample = min(S, 8)
    t0 = time.perf_counter()
    ok = True
    for i in range(sample):
        want = ref.detect(diffs[i], DetectConfig(), threads=nproc)
        ok &= bool(np.array_equal(want, boxes[i]))
    ref_s = (time.perf_counter() - t0) / sample
    print(json.dumps({
        "workload": f"config-2 diff maps after {F} frames, {S} sequences, 1242x375, default DetectConfig",
        "gpu_batched_ms_per_frame_batch": round(gpu_s * 1e3, 3),
        "gpu_maps_per_s": round(S / gpu_s, 1),
        "reference_ms_per_map": round(ref_s * 1e3, 3),
        "reference_threads": nproc,
        "reference_maps_timed": sample,
        "speedup_maps_per_s": round((S / gpu_s) / (1.0 / ref_s), 1),
        "boxes_per_map_mean": round(float(np.mean([len(b) for b in boxes])), 2),
        "bit_exact_vs_reference": ok}, indent=1))
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
