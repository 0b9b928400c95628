"""Regenerate tests/golden/*.npz from the reference itself (run HERE only).

Builds tests/golden/make_golden.cpp against the unmodified reference sources in
/root/reference/proj/src, the reference's own test oracles
(/root/reference/proj/tests/oracles.hpp, included in place, not copied) and the
Eigen stand-in in oracle/eigen_shim, runs it, and converts its record stream
into compressed .npz fixtures. The GPU box never runs this: the .npz files are
committed.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/proj"
SRCS = ["matching_cost.cpp", "sgm.cpp", "geometry.cpp", "temporal_filter.cpp",
        "motion_detect.cpp", "eval.cpp"]


def build_and_run(tmp: str) -> str:
    exe = os.path.join(tmp, "make_golden")
    cmd = ["g++", "-std=gnu++20", "-O2", "-ffp-contract=off", "-pthread",
           f"-I{REF}/include", f"-I{REF}/tests", f"-I{ROOT}/oracle/eigen_shim",
           os.path.join(HERE, "make_golden.cpp"), *[f"{REF}/src/{s}" for s in SRCS], "-o", exe]
    subprocess.run(cmd, check=True)
    out = os.path.join(tmp, "golden.bin")
    subprocess.run([exe, out], check=True)
    return out


def parse(path: str) -> dict:
    recs = {}
    with open(path, "rb") as f:
        buf = f.read()
    i = 0
    while i < len(buf):
        j = buf.index(b"\0", i)
        name = buf[i:j].decode()
        i = j + 1
        j = buf.index(b"\0", i)
        dtype = buf[i:j].decode()
        i = j + 1
        (nd,) = struct.unpack_from("<i", buf, i)
        i += 4
        shape = struct.unpack_from("<" + "q" * nd, buf, i)
        i += 8 * nd
        (nb,) = struct.unpack_from("<Q", buf, i)
        i += 8
        arr = np.frombuffer(buf[i:i + nb], dtype=np.dtype("<" + dtype)).reshape(shape)
        i += nb
        recs[name] = arr.copy()
    return recs


def main() -> None:
    if not os.path.isdir(REF):
        sys.exit("reference sources not present; golden fixtures are committed")
    with tempfile.TemporaryDirectory() as tmp:
        recs = parse(build_and_run(tmp))
    groups: dict[str, dict] = {}
    for name, arr in recs.items():
        g, rest = name.split("/", 1)
        groups.setdefault(g, {})[rest.replace("/", "__")] = arr
    for g, arrs in groups.items():
        np.savez_compressed(os.path.join(HERE, f"{g}.npz"), **arrs)
        print(f"{g}.npz: {len(arrs)} arrays")


if __name__ == "__main__":
    main()
