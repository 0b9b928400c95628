"""Noise calibration throughput on a config-1 sequence
(1242x375, D=128, 30 frames with movers): the GPU's batched
estimate_process_noise / estimate_measurement_noise / accumulate_error_map
(host arrays in, estimates out: copies included) against the reference's
noise_calib.cpp on the same frames (CPU; sgm_match with threads=nproc, as
tsgm_main's calibrate command runs it). The reference's measurement noise is
timed on a bounded sample of frames; every timed reference result is checked
against the GPU's on the same frames (counts and map exact, variance 1e-9
relative: FP64 reassociation of the sums, amplified by the variance formula).

    python tools/noise_bench.py [F] [ref_meas_frames] > profiles/r01_noise_bench.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402
from paper_1809_07986_b200.testing import GpuBackend  # noqa: E402


def timed(fn, reps=1):
    fn()  # warm
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    return out, (time.perf_counter() - t0) / reps


def same(a, b):
    return (all(a[k] == b[k] for k in ("samples_used", "total", "underflow", "overflow"))
            and np.array_equal(a["counts"], b["counts"])
            and abs(a["variance"] - b["variance"]) <= 1e-9 * max(abs(b["variance"]), 1e-300))


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    FM = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    cfg = SceneConfig.baseline_config(1, frames=F)
    left, right, poses, gt = render(cfg, gt=True)
    gt = gt.astype(np.float64)
    p12 = poses.reshape(-1, 12)
    calib = O.Calib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, cfg.width, cfg.height, cfg.d_max)
    sgm = O.SgmParams(10, 120, 8, 0, cfg.d_max)
    opts = O.CalibOpts()
    gpu = GpuBackend.shared()
    g_proc, t_proc = timed(lambda: gpu.process_noise(gt, p12, calib, opts), 3)
    g_meas, t_meas = timed(lambda: gpu.measurement_noise(left, right, gt, sgm, opts), 2)
    g_map, t_map = timed(lambda: gpu.error_map(gt, p12, calib), 3)
    g_meas_s = gpu.measurement_noise(left[:FM], right[:FM], gt[:FM], sgm, opts)

    ref = O.reference()
    nproc = os.cpu_count() or 1
    t0 = time.perf_counter()
    r_proc = ref.process_noise(gt, p12, calib, opts)
    rt_proc = time.perf_counter() - t0
    t0 = time.perf_counter()
    r_meas = ref.measurement_noise(left[:FM], right[:FM], gt[:FM], sgm, opts, threads=nproc)
    rt_meas = time.perf_counter() - t0
    t0 = time.perf_counter()
    r_map = ref.error_map(gt, p12, calib)
    rt_map = time.perf_counter() - t0
    ok = same(g_proc, r_proc) and same(g_meas_s, r_meas) and np.array_equal(g_map, r_map)
    pairs = F - 1
    print(json.dumps({
        "workload": f"config-1 sequence, {F} frames, 1242x375, D=128, P1=10, P2=120, 8 paths, "
                    "CalibOptions defaults (gate 10 px, bin 0.25)",
        "gpu": {"process_noise_ms": round(t_proc * 1e3, 2),
                "process_pairs_per_s": round(pairs / t_proc, 1),
                "measurement_noise_ms": round(t_meas * 1e3, 2),
                "measurement_frames_per_s": round(F / t_meas, 1),
                "error_map_ms": round(t_map * 1e3, 2),
                "note": "host arrays in, estimate out (pageable H2D copies included); warm calls: the device working set is cached between calls (tsgm_calib_release frees it)"},
        "reference": {"threads": nproc, "process_noise_ms": round(rt_proc * 1e3, 2),
                      "process_pairs_per_s": round(pairs / rt_proc, 1),
                      "measurement_frames_timed": FM,
                      "measurement_frames_per_s": round(FM / rt_meas, 2),
                      "error_map_ms": round(rt_map * 1e3, 2)},
        "speedup": {"process": round(rt_proc / t_proc, 1),
                    "measurement": round((F / t_meas) / (FM / rt_meas), 1),
                    "error_map": round(rt_map / t_map, 1)},
        "process_variance": g_proc["variance"], "measurement_variance": g_meas["variance"],
        "exact_vs_reference": bool(ok)}, indent=1))
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
