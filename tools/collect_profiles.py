"""Turn one measurement directory (tools/measure_all.sh under gpurun) into the
committed profiles/r02_* files. Reads only files; no GPU needed.

    python tools/collect_profiles.py gpurun_out/final2 "<what tree this is>"
"""
import contextlib
import io
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import summarize_ncu  # noqa: E402

PROF = os.path.join(ROOT, "profiles")


def quiet(fn, *a):
    with contextlib.redirect_stdout(io.StringIO()):
        fn(*a)


def last_json(path):
    lines = [ln for ln in open(path).read().strip().splitlines() if ln.strip().startswith("{")]
    return json.loads(lines[-1]) if len(lines) >= 1 and not open(path).read().lstrip().startswith("{\n") \
        else json.load(open(path))


def num(v):
    return float(str(v).split()[0].replace(",", ""))


def main():
    src, tree = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "round-2 tree")
    j = lambda n: os.path.join(src, n)  # noqa: E731
    for name, dst in (("bench.json", "r02_bench.json"), ("bench_reference.json", "r02_bench_reference.json"),
                      ("batch_sweep.json", "r02_batch_sweep.json"), ("config3_sweep.json", "r02_config3_sweep.json"),
                      ("config4_stress.json", "r02_config4_stress.json"), ("config4_cpu.json", "r02_config4_cpu.json"),
                      ("config_report.json", "r02_config_report.json")):
        if os.path.exists(j(name)):
            json.dump(last_json(j(name)), open(os.path.join(PROF, dst), "w"), indent=1)
    for name, dst in (("pytest_gpu.log", "r02_pytest_gpu.log"), ("smoke.log", "r02_smoke.log"),
                      ("gpu.txt", "r02_gpu_box.txt"), ("bench_launches.csv", "r02_step_launches_bench.csv")):
        if os.path.exists(j(name)):
            shutil.copy(j(name), os.path.join(PROF, dst))
    if os.path.exists(j("bench_launches.csv")):
        quiet(summarize_ncu.launch_list, j("bench_launches.csv"), os.path.join(PROF, "r02_step_launches_bench.json"))
    # standalone aggregation: scan + combine full captures, DRAM bytes per cell
    if os.path.exists(j("agg_details.csv")):
        tmp = os.path.join(src, "_agg.json")
        quiet(summarize_ncu.full, j("agg_details.csv"), tmp, j("agg_raw.csv"))
        agg = json.load(open(tmp))
        cells = None
        for ln in open(j("ncu_agg.log")):
            if ln.startswith("aggregation:"):
                cells = float(ln.split(" for ")[1].split(" M")[0]) * 1e6
        cap = ("ncu --set full --clock-control none, tools/profile_step.py 64 4 1: 64 config-2 sequences, "
               "standalone C->S aggregation (tsgm_bench_aggregate, S written) on frame 3's volumes, "
               f"{cells / 1e6:.1f} M cells; {tree}")
        scan = next(v for k, v in agg.items() if "scan_kernel" in k)
        comb = next(v for k, v in agg.items() if "combine_wta" in k)
        sname = next(k for k in agg if "scan_kernel" in k).split(" ", 1)[1]
        cname = next(k for k in agg if "combine_wta" in k).split(" ", 1)[1]
        json.dump({sname: scan, "_capture": cap, "_cells": cells},
                  open(os.path.join(PROF, "r02_scan_kernel_ncu_full.json"), "w"), indent=1)
        json.dump({cname: comb, "_capture": cap, "_cells": cells},
                  open(os.path.join(PROF, "r02_combine_ncu_full.json"), "w"), indent=1)

        def dram(k):
            u = 1e9 if "Gbyte" in k["dram__bytes_read.sum"] else 1e6 if "Mbyte" in k["dram__bytes_read.sum"] else 1.0
            return (num(k["dram__bytes_read.sum"]) + num(k["dram__bytes_write.sum"])) * u
        json.dump({"source": "profiles/r02_scan_kernel_ncu_full.json + profiles/r02_combine_ncu_full.json "
                             "(ncu --set full, 64 config-2 sequences, standalone C->S aggregation on frame 3's volumes)",
                   "scan_dram_bytes": dram(scan), "combine_dram_bytes": dram(comb), "cells": cells,
                   "bytes_per_cell": (dram(scan) + dram(comb)) / cells, "algorithmic_bytes_per_cell": 3.0,
                   "note": "roofline.traffic = bytes_per_cell x cells of the timed launch; the excess over 3 B/cell "
                           "is the per-direction u8 path costs (8 written by the scan, 8 read by the combine, windows "
                           "allocated in multiples of 4 quads), the 8 direction passes over the quad-layout C and "
                           "the 8-byte scan records"},
                  open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
        os.remove(tmp)
    # every step kernel (one reduced frame of 64 sequences)
    if os.path.exists(j("step_details.csv")):
        tmp = os.path.join(src, "_step.json")
        quiet(summarize_ncu.full, j("step_details.csv"), tmp, j("step_raw.csv"))
        st = json.load(open(tmp))
        kern, total = {}, 0.0
        for k, v in st.items():
            name = k.split(" ", 1)[1]
            if name in kern:
                continue  # first launch of each kernel
            kern[name] = v
            d = v.get("duration", "0 us")
            total += num(d) * (1e-3 if "us" in d else 1.0 if "ms" in d else 1e-6)
        json.dump({"_capture": "ncu --set full --clock-control none --launch-skip 12 -c 16, tools/profile_step.py 64 3 1: "
                               "config 2, 64 sequences, reduced frames (cold cache, serialised replays; durations are "
                               f"per launch); {tree}",
                   "kernels": kern, "frame_ms_serialised": round(total, 3)},
                  open(os.path.join(PROF, "r02_step_kernels_ncu_full.json"), "w"), indent=1)
        os.remove(tmp)
    print("profiles written from", src)


if __name__ == "__main__":
    main()
