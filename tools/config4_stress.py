"""BASELINE config 4 on one B200: the per-GPU share of the high-res stress test
(256 sequences x 20 frames at 2048x1024, D=256, 8 paths, gain +-10%, movers up
to 30% of the image, 32 sequences per GPU on 8 GPUs).

32 sequences' Kalman state stays resident; the per-frame volumes (~6 GB per
sequence at frame 0) run through the context's volume working set (vol_slots,
auto-sized to free memory), so the matching stages execute in chunks. Reports
frames/s through the host-image API, the working set and device memory, and
spot-checks sequence 0's first frames bit-exact against the oracle.

    python tools/config4_stress.py [sequences] [frames] [check_frames] [vol_slots]

vol_slots = the volume pool in worst-case (full-range) sequences (0 = auto).
Volumes are packed by their actual cells, so frame 0 (full range) needs
ceil(S / vol_slots) chunks and the reduced frames usually one.
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
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    check = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    vs = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    import torch
    cfgs = [SceneConfig.baseline_config(4, seed=s, frames=F) for s in range(S)]
    c0 = cfgs[0]
    calib = tsgm.StereoCalib(c0.focal, c0.cx, c0.cy, c0.baseline, c0.width, c0.height, c0.d_max)
    params = tsgm.SgmParams(10, 120, 8, 0, c0.d_max)
    filt = tsgm.FilterConfig(p_init=16384.0, range_use_stddev=True, range_stddev_gain=3.0)
    t0 = time.time()
    seqs = [render(c) for c in cfgs]
    t_render = time.time() - t0
    free0, total = torch.cuda.mem_get_info()
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=S, keep_volumes=False,
                                        vol_slots=vs))
    free1, _ = torch.cuda.mem_get_info()
    slots = list(range(S))
    mots = [[(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
             for k in range(F)] for (_, _, P, _) in seqs]
    ed0 = []
    chunks = []
    eng.sync()
    eng.timer_begin()
    for k in range(F):
        eng.step(slots, [s[0][k] for s in seqs], [s[1][k] for s in seqs], [m[k] for m in mots])
        chunks.append(eng.last_chunks())
        if k < check:
            ed0.append((eng.fetch(0, "export_d"), eng.fetch(0, "state_p"), eng.fetch(0, "mask")))
    ms = eng.timer_end()
    vol_slots = eng.vol_slots
    # the standalone C->S aggregation on the last frame's volumes (one chunk)
    agg_ms, agg_cells = eng.bench_aggregate(slots, reps=3)
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    agg_frac = (3.0 * agg_cells + 4.0 * c0.width * c0.height * S) / (agg_ms * 1e-3) / (peak * 1e9)
    eng.close()
    from oracle import Port
    port = Port()
    state, ok = None, True
    L, R, _, _ = seqs[0]
    for k in range(check):
        ref = port.step(state, L[k], R[k], mots[0][k][0], mots[0][k][1], calib, params, filt,
                        debug=True)
        ok &= bool(np.array_equal(ed0[k][0], ref["export_d"]) and
                   np.array_equal(ed0[k][1], ref["p"]) and np.array_equal(ed0[k][2], ref["mask"]))
        state = (ref["d"], ref["p"], ref["valid"])
    print(json.dumps({
        "config": "BASELINE configs[4], per-GPU share: %d sequences x %d frames, %dx%d, D=%d" %
                  (S, F, c0.width, c0.height, c0.d_max),
        "frames_per_s_host_api": round(S * F / (ms * 1e-3), 2),
        "ms_total": round(ms, 1),
        "vol_slots": vol_slots,
        "aggregation_ms": round(agg_ms, 3), "aggregation_cells": agg_cells,
        "aggregation_hbm_frac": round(agg_frac, 4),
        "volume_chunks_per_frame": chunks,
        "device_mem_gb": {"total": round(total / 2**30, 1),
                          "context": round((free0 - free1) / 2**30, 1)},
        "render_s": round(t_render, 1),
        "parity_seq0_frames": check, "parity_bit_exact": ok}, indent=1))
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
