"""Export throughput: after F frames of S config-2
sequences, every slot's export map written as a KITTI 16-bit PNG through
Engine.write_export_png (device quantisation, 2 B/px over PCIe, host zlib
PNG) vs fetching the map (i32 + u8, 5 B/px) and quantising + encoding on the
host (numpy restatement + the same zlib container). The reference's own
writer needs libpng (absent), so it is not timed.

    python tools/export_bench.py [S] [F] > profiles/r01_export_bench.json
"""
import json
import os
import struct
import sys
import tempfile
import time
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1809_07986_b200 import tsgm  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402


def host_png(raw):
    h, w = raw.shape
    rows = np.zeros((h, 1 + 2 * w), np.uint8)
    rows[:, 1::2], rows[:, 2::2] = raw >> 8, raw & 0xff

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xffffffff)
    return (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 16, 0, 0, 0, 0)) +
            chunk(b"IDAT", zlib.compress(rows.tobytes(), 6)) + chunk(b"IEND", b""))


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, 1242, 375, 128)
    eng = tsgm.Engine(tsgm.EngineConfig(calib, tsgm.SgmParams(10, 120, 8, 0, 128),
                                        tsgm.FilterConfig(range_use_stddev=True,
                                                          range_stddev_gain=3.0),
                                        max_slots=S))
    seqs = [render(SceneConfig.baseline_config(2, seed=s, n_movers=s % 5, frames=F))
            for s in range(S)]
    for k in range(F):
        mots = [(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
                for (_, _, P, _) in seqs]
        eng.step(list(range(S)), [L[k] for (L, _, _, _) in seqs], [R[k] for (_, R, _, _) in seqs],
                 mots)
    eng.sync()
    with tempfile.TemporaryDirectory() as tmp:
        eng.write_export_png(0, os.path.join(tmp, "w.png"))  # warm
        t0 = time.perf_counter()
        for s in range(S):
            eng.write_export_png(s, os.path.join(tmp, f"{s}.png"))
        gpu_s = (time.perf_counter() - t0) / S
        t0 = time.perf_counter()
        eng.write_export_pngs(list(range(S)), [os.path.join(tmp, f"b{s}.png") for s in range(S)])
        batch_s = (time.perf_counter() - t0) / S
        same = True
        t0 = time.perf_counter()
        for s in range(S):
            raw = O.quantize_disparity_map(eng.fetch(s, "export_d"), eng.fetch(s, "export_valid"))
            with open(os.path.join(tmp, f"h{s}.png"), "wb") as f:
                f.write(host_png(raw))
        host_s = (time.perf_counter() - t0) / S
        for s in range(S):
            want = tsgm.read_png16(os.path.join(tmp, f"h{s}.png"))
            same &= bool(np.array_equal(tsgm.read_png16(os.path.join(tmp, f"{s}.png")), want))
            same &= bool(np.array_equal(tsgm.read_png16(os.path.join(tmp, f"b{s}.png")), want))
    eng.close()
    print(json.dumps({
        "workload": f"export maps of {S} config-2 sequences after {F} frames, 1242x375",
        "gpu_quantise_ms_per_map": round(gpu_s * 1e3, 3),
        "gpu_maps_per_s": round(1.0 / gpu_s, 1),
        "gpu_batched_maps_per_s": round(1.0 / batch_s, 1),
        "host_threads": os.cpu_count(),
        "host_fetch_quantise_ms_per_map": round(host_s * 1e3, 3),
        "pcie_bytes_per_map": {"device_quantised": 2 * 1242 * 375,
                               "fetch_then_quantise": 5 * 1242 * 375},
        "note": "all include the PNG encode and file write: the library's zlib level 1 (GPU rows), "
                "Python zlib level 6 (host row)",
        "same_samples": same}, indent=1))


if __name__ == "__main__":
    main()
