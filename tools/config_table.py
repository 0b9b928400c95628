"""Per-config results table: for every
BASELINE config, the reference CPU path (cores stated), one B200, and the
standalone aggregation's fraction of the HBM roofline, with frame 0 (full
range) and frames >= 1 (reduced) split as eval.cpp:177-179 reports them.
Reads the JSON files the measurement tools wrote; no GPU needed.

    python tools/config_table.py <dir> > profiles/r02_config_table.json

<dir> holds: bench.json, bench_reference.json (config 2), config_report.json
(configs 0, 1, 3 single sequence), config3_sweep.json (config 3 batched),
config4_stress.json + config4_cpu.json (config 4), batch_sweep.json.
"""
import json
import os
import sys


def load(d, name):
    p = os.path.join(d, name)
    return json.load(open(p)) if os.path.exists(p) else None


def main():
    d = sys.argv[1]
    rows = []
    bench, ref = load(d, "bench.json"), load(d, "bench_reference.json")
    rep, sweep = load(d, "config_report.json"), load(d, "config3_sweep.json")
    c4, c4cpu, bs = load(d, "config4_stress.json"), load(d, "config4_cpu.json"), load(d, "batch_sweep.json")
    if rep:
        n = rep["nproc"]
        for r in rep["rows"]:
            cpu = r[f"reference_threads_{n}"]
            g = r["gpu"]
            rows.append({
                "config": r["config"] + " (1 sequence)", "size": f"{r['width']}x{r['height']} D={r['d_max']}",
                "cpu_frame0_ms": cpu["frame0_ms"], "cpu_frames_ge1_ms": cpu["mean_ms_frames_ge1"],
                "cpu_cores": n, "cpu_kind": "reference (in-place build, tsgm::step, threads=%d)" % n,
                "gpu_frame0_ms": g["frame0_ms"], "gpu_frames_ge1_ms": g["mean_ms_frames_ge1"],
                "gpu_frames_per_s": r["gpu_frames_per_s"],
                "speedup_frames_ge1": r["speedup_vs_ref_nproc_frames_ge1"],
                "aggregation_hbm_frac": r.get("aggregation_hbm_frac"),
                "note": "latency: one sequence leaves the GPU mostly idle"})
    if bench and ref:
        rows.append({
            "config": "config 2 (64 x 30, 1 GPU)", "size": "1242x375 D=128",
            "cpu_frames_per_s": ref["value"], "cpu_cores": ref["cpu_baseline"]["cores"],
            "cpu_kind": "reference, one sequence per thread, full workload",
            "cpu_sample": ref["cpu_baseline"]["sample"],
            "gpu_frames_per_s": bench["value"], "gpu_e2e_frames_per_s": bench["e2e"]["value"],
            "speedup_e2e": round(bench["e2e"]["value"] / ref["value"], 1),
            "aggregation_hbm_frac": bench["roofline"]["frac"],
            "aggregation_ms": bench["roofline"]["ms"]})
    if bs:
        for r in bs["rows"]:
            rows.append({"config": f"config 2 share: {r['sequences']} sequences per GPU",
                         "gpu_frames_per_s": r["value"], "gpu_e2e_frames_per_s": r["e2e"],
                         "share_of_64_sequence_rate": r.get("share")})
    if sweep:
        for r in sweep["rows"]:
            rows.append({"config": f"config 3 {r['setting']} ({r['sequences']} sequences batched)",
                         "gpu_frames_per_s": r["frames_per_s"],
                         "aggregation_gcells_per_s": r["aggregation_gcells_per_s"],
                         "aggregation_hbm_frac": r["aggregation_hbm_frac"]})
    if c4:
        row = {"config": "config 4 per-GPU share (32 x 20, 1 GPU)", "size": "2048x1024 D=256",
               "gpu_frames_per_s": c4["frames_per_s_host_api"],
               "gpu_context_gb": c4["device_mem_gb"]["context"],
               "volume_chunks_per_frame": c4["volume_chunks_per_frame"],
               "aggregation_hbm_frac": c4.get("aggregation_hbm_frac"),
               "parity_bit_exact_spot_check": c4["parity_bit_exact"]}
        if c4cpu:
            F = 20
            per_seq_s = c4cpu["frame0_s_mean"] + (F - 1) * c4cpu["frames_ge1_s_mean"]
            row.update({"cpu_cores": c4cpu["threads"], "cpu_kind": c4cpu["kind"],
                        "cpu_frame0_s": c4cpu["frame0_s_mean"],
                        "cpu_frames_ge1_s": c4cpu["frames_ge1_s_mean"],
                        "cpu_frames_per_s_20_frame_mix": round(c4cpu["threads"] * F / per_seq_s, 3),
                        "cpu_sample": c4cpu["config"]})
            row["speedup_vs_cpu_20_frame_mix"] = round(c4["frames_per_s_host_api"] /
                                                       row["cpu_frames_per_s_20_frame_mix"], 1)
        rows.append(row)
    print(json.dumps({"rows": rows}, indent=1))


if __name__ == "__main__":
    main()
