"""Summarise ncu captures for profiles/ (read here, no GPU needed).

    python tools/summarize_ncu.py full  <report.ncu-rep> <out.json>   # --set full capture
    python tools/summarize_ncu.py list  <launches.csv>   <out.json>   # gpu__time_duration list
    python tools/summarize_ncu.py csv   <details.csv>,<raw.csv> <out.json>  # exported pages

`full` extracts duration, DRAM bytes (read+write), executed instructions,
issue/occupancy figures and pipe utilisation per profiled kernel; `list` sums
the launch list per kernel (share of the step).
"""
import collections
import csv
import io
import json
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"

FULL_METRICS = {
    "Duration": "duration",
    "DRAM Throughput": "dram_throughput_pct",
    "Memory Throughput": "memory_throughput",
    "Executed Instructions": "executed_instructions",
    "Issue Slots Busy": "issue_slots_busy_pct",
    "Eligible Warps Per Scheduler": "eligible_warps_per_scheduler",
    "Achieved Occupancy": "achieved_occupancy_pct",
    "Theoretical Occupancy": "theoretical_occupancy_pct",
    "Registers Per Thread": "registers_per_thread",
    "Compute (SM) Throughput": "sm_throughput_pct",
    "L1/TEX Hit Rate": "l1_hit_pct",
    "L2 Hit Rate": "l2_hit_pct",
    "Grid Size": "grid_size",
    "Block Size": "block_size",
}


def _page(rep, page):
    if rep.endswith(".csv"):  # an exported page (--page details|raw --csv) from the GPU box
        return open(rep).read()
    return subprocess.run([NCU, "-i", rep, "--page", page, "--csv"], capture_output=True,
                          text=True).stdout


def full(rep, out, raw_rep=None):
    """One entry per profiled launch ("<ID> <kernel>"), details + raw pipe metrics."""
    rows = list(csv.reader(io.StringIO(_page(rep, "details"))))
    hdr = rows[0]
    ki, si, ni, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Section Name", "Metric Name",
                                                  "Metric Unit", "Metric Value"))
    kern = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        k = f'{r[hdr.index("ID")]} {r[ki].split("(")[0]}'
        d = kern.setdefault(k, {})
        if r[ni] in FULL_METRICS:
            d[FULL_METRICS[r[ni]]] = f"{r[vi]} {r[ui]}".strip()
    rr = list(csv.reader(io.StringIO(_page(raw_rep or rep, "raw"))))
    if len(rr) > 2:
        h = rr[0]
        want = ["dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "gpu__time_duration.sum"]
        units = rr[1]
        for row in rr[2:]:
            k = f'{row[h.index("ID")]} {row[h.index("Kernel Name")].split("(")[0]}'
            d = kern.setdefault(k, {})
            for w in want:
                if w in h:
                    d[w] = f"{row[h.index(w)]} {units[h.index(w)]}".strip()
    json.dump(kern, open(out, "w"), indent=1)
    print(json.dumps(kern, indent=1))


def launch_list(path, out):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = [r for r in rows if r[0] == "ID"][0]
    data = rows[rows.index(hdr) + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    for r in data:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    res = {"total_ms": T, "kernels": [
        {"kernel": k, "ms": round(v, 4), "share": round(v / T, 4), "launches": cnt[k]}
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1])]}
    json.dump(res, open(out, "w"), indent=1)
    for e in res["kernels"]:
        print(f"{e['ms']:10.3f} ms {e['share']*100:5.1f}%  x{e['launches']:3d}  {e['kernel']}")


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    if mode == "csv":
        det, raw = src.split(",")
        full(det, dst, raw)
    else:
        (full if mode == "full" else launch_list)(src, dst)
