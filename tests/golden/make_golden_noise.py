"""Regenerate tests/golden/noise_calib.npz from the
reference itself (run HERE only: needs /root/reference for oracle/_ref).

Inputs are this repo's own synthetic scenes (paper_1809_07986_b200.scene,
BASELINE config-1 style with movers, reduced size); outputs are the
UNMODIFIED reference's estimate_process_noise / estimate_measurement_noise /
accumulate_error_map / write_calib_report (noise_calib.cpp, compiled in place
by oracle/Makefile and bound by oracle/ref_runner.cpp).

    python tests/golden/make_golden_noise.py
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1809_07986_b200.scene import SceneConfig, render  # noqa: E402

# (name, scene overrides, calib opts (gate, bin width, q floor), sgm (p1, p2, paths, set))
CASES = [
    ("a", dict(width=128, height=80, focal=90.0, cx=63.5, cy=39.5, d_max=64, seed=5,
               n_movers=2, frames=4), (10.0, 0.25, 0.1), (10, 120, 8, 0)),
    ("b", dict(width=96, height=72, focal=80.0, cx=47.5, cy=35.5, d_max=48, seed=8,
               n_movers=1, frames=3, noise_sigma=6.0), (4.0, 0.5, 0.05), (6, 65, 4, 1)),
]


def main() -> None:
    O.build()
    ref = O.reference()
    out = {}
    for name, kw, (gate, bw, qf), (p1, p2, paths, pset) in CASES:
        cfg = SceneConfig.baseline_config(1, **kw)
        left, right, poses, gt = render(cfg, gt=True)
        gt = gt.astype(np.float64)
        calib = O.Calib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, cfg.width, cfg.height, cfg.d_max)
        opts = O.CalibOpts(gate, bw, qf)
        sgm = O.SgmParams(p1, p2, paths, pset, cfg.d_max)
        p12 = poses.reshape(-1, 12)
        out[f"{name}_left"], out[f"{name}_right"] = left, right
        out[f"{name}_gt"], out[f"{name}_poses"] = gt, p12
        out[f"{name}_calib"] = np.array([cfg.focal, cfg.cx, cfg.cy, cfg.baseline, cfg.width,
                                         cfg.height, cfg.d_max])
        out[f"{name}_opts"] = np.array([gate, bw, qf])
        out[f"{name}_sgm"] = np.array([p1, p2, paths, pset, cfg.d_max], np.int32)
        for kind, r in (("process", ref.process_noise(gt, p12, calib, opts)),
                        ("meas", ref.measurement_noise(left, right, gt, sgm, opts))):
            out[f"{name}_{kind}_moments"] = np.array([r["variance"], r["mean"], r["within_1px"]])
            out[f"{name}_{kind}_ints"] = np.array([r["samples_used"], r["total"], r["underflow"],
                                                   r["overflow"]], np.int64)
            out[f"{name}_{kind}_counts"] = r["counts"]
        out[f"{name}_error_map"] = ref.error_map(gt, p12, calib)
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "report.txt")
            ref.calib_report(path, left, right, gt, p12, calib, sgm, opts)
            out[f"{name}_report"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "noise_calib.npz"), **out)
    print("wrote", os.path.join(HERE, "noise_calib.npz"))


if __name__ == "__main__":
    main()
