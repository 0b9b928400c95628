"""Regenerate tests/golden/export.npz from the reference
itself (run HERE only): builds tests/golden/make_golden_export.cpp against the
UNMODIFIED dataset.cpp / geometry.cpp (compiled in place from
/root/reference/proj/src) with the Eigen stand-in and oracle/io_shim.cpp
(records the 16-bit image write_disparity_png hands to libpng), runs it, and
packs its record stream.

    python tests/golden/make_golden_export.py
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
from make_golden import parse  # noqa: E402

REF = "/root/reference/proj"


def main() -> None:
    with tempfile.TemporaryDirectory() as tmp:
        exe = os.path.join(tmp, "mk")
        subprocess.run(["g++", "-std=gnu++20", "-O2", "-ffp-contract=off", f"-I{REF}/include",
                        f"-I{ROOT}/oracle/eigen_shim", os.path.join(HERE, "make_golden_export.cpp"),
                        os.path.join(ROOT, "oracle", "io_shim.cpp"), f"{REF}/src/dataset.cpp",
                        f"{REF}/src/geometry.cpp", "-o", exe], check=True)
        out = os.path.join(tmp, "export.bin")
        subprocess.run([exe, out, tmp], check=True)
        recs = parse(out)
    np.savez_compressed(os.path.join(HERE, "export.npz"), **recs)
    print("wrote", os.path.join(HERE, "export.npz"), sorted(recs))


if __name__ == "__main__":
    main()
