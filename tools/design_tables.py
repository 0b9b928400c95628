"""Regenerate the measured tables of DESIGN.md (section 4 per-kernel ncu table,
section 7a per-config table) from the committed profiles/r02_* files.

    python tools/design_tables.py        # rewrites DESIGN.md in place
"""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = lambda n: os.path.join(ROOT, "profiles", n)  # noqa: E731


def num(v):
    return float(str(v).split()[0].replace(",", ""))


def ms(d):
    return num(d) * (1e-3 if "us" in d else 1.0)


def kernel_table():
    d = json.load(open(P("r02_step_kernels_ncu_full.json")))["kernels"]
    rows = sorted(d.items(), key=lambda kv: -ms(kv[1]["duration"]))
    out = ["| kernel | ms | DRAM % | issue slots % | ALU pipe % | achieved occupancy |", "|---|---|---|---|---|---|"]
    for k, v in rows:
        alu = v.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "0")
        out.append(f"| `{k.replace('void ', '')}` | {ms(v['duration']):.3f} | {num(v['dram_throughput_pct']):.1f} | "
                   f"{num(v['issue_slots_busy_pct']):.1f} | {num(alu):.0f} | {num(v['achieved_occupancy_pct']):.1f} % |")
    return "\n".join(out)


def config_table():
    t = json.load(open(P("r02_config_table.json")))
    rows = {r["config"]: r for r in (t["rows"] if isinstance(t, dict) else t)}
    g = lambda name: rows[name]  # noqa: E731
    c0, c1 = g("config 0 (1 sequence)"), g("config 1 (1 sequence)")
    c2 = g("config 2 (64 x 30, 1 GPU)")
    sh = [g(f"config 2 share: {n} sequences per GPU") for n in (32, 16, 8)]
    f128, f256 = g("config 3 full D=128 (1 sequence)"), g("config 3 full D=256 (1 sequence)")
    b128, b256 = g("config 3 full D=128 (32 sequences batched)"), g("config 3 full D=256 (32 sequences batched)")
    red = [g(f"config 3 reduced h={h} (1 sequence)") for h in (2, 4, 8, 16)]
    redb = [g(f"config 3 reduced h={h} (32 sequences batched)") for h in (2, 4, 8, 16)]
    c4 = g("config 4 per-GPU share (32 x 20, 1 GPU)")
    L = ["| config | CPU reference (16 cores) | B200 ×1 | speed-up | agg. frac |", "|---|---|---|---|---|"]
    for name, c in (("0: 1 seq × 8, 1242×375 D=128", c0), ("1: 1 seq × 30 with movers", c1)):
        L.append(f"| {name} | frame 0 {c['cpu_frame0_ms']:.0f} ms, frames ≥ 1 {c['cpu_frames_ge1_ms']:.0f} ms | "
                 f"frame 0 {c['gpu_frame0_ms']:.2f} ms, frames ≥ 1 {c['gpu_frames_ge1_ms']:.2f} ms "
                 f"({c['gpu_frames_per_s']:.0f} frames/s) | {c['speedup_frames_ge1']:.0f}× (frames ≥ 1) | "
                 f"{c['aggregation_hbm_frac']:.3f} (latency-bound) |")
    L.append(f"| 2: 64 × 30 (the metric) | {c2['cpu_frames_per_s']:.1f} frames/s (full workload, one sequence per core) | "
             f"{c2['gpu_frames_per_s']:.0f} frames/s device-resident, **{c2['gpu_e2e_frames_per_s']:.0f} frames/s e2e** "
             f"(host frames in, maps out) | **{c2['speedup_e2e']:.1f}× e2e** | **{c2['aggregation_hbm_frac']:.3f}** |")
    L.append("| 2 at 32 / 16 / 8 sequences per GPU (2/4/8-GPU shares) | — | "
             + " / ".join(f"{r['gpu_frames_per_s']:.0f}" for r in sh) + " frames/s ("
             + " / ".join(f"{r['share_of_64_sequence_rate']:.2f}" for r in sh) + " of the 64-sequence rate) | — | — |")
    L.append(f"| 3: full range D=128 / D=256, 1 seq | {f128['cpu_frames_ge1_ms']:.0f} / {f256['cpu_frames_ge1_ms']:.0f} ms per frame | "
             f"{f128['gpu_frames_ge1_ms']:.2f} / {f256['gpu_frames_ge1_ms']:.2f} ms | {f128['speedup_frames_ge1']:.0f}× / "
             f"{f256['speedup_frames_ge1']:.0f}× | {f128['aggregation_hbm_frac']:.3f} / {f256['aggregation_hbm_frac']:.3f} |")
    L.append(f"| 3: full range D=128 / D=256, 32 seqs batched | — | {b128['gpu_frames_per_s']:.0f} / {b256['gpu_frames_per_s']:.0f} "
             f"frames/s | — | {b128['aggregation_hbm_frac']:.3f} / {b256['aggregation_hbm_frac']:.3f} |")
    L.append("| 3: reduced h = 2 / 4 / 8 / 16, 1 seq | " + " / ".join(f"{r['cpu_frames_ge1_ms']:.0f}" for r in red)
             + " ms (frames ≥ 1) | " + " / ".join(f"{r['gpu_frames_ge1_ms']:.2f}" for r in red) + " ms | "
             + f"{min(r['speedup_frames_ge1'] for r in red):.0f}× – {max(r['speedup_frames_ge1'] for r in red):.0f}× | "
             + f"{min(r['aggregation_hbm_frac'] for r in red):.3f} – {max(r['aggregation_hbm_frac'] for r in red):.3f} |")
    L.append("| 3: reduced h = 2 / 4 / 8 / 16, 32 seqs batched | — | " + " / ".join(f"{r['gpu_frames_per_s']:.0f}" for r in redb)
             + " frames/s | — | " + " / ".join(f"{r['aggregation_hbm_frac']:.3f}" for r in redb) + " |")
    L.append(f"| 4: 32 × 20 per-GPU share, 2048×1024 D=256 | {c4['cpu_frames_per_s_20_frame_mix']:.1f} frames/s for the 20-frame mix "
             f"(16 sequences' first 3 frames: frame 0 {c4['cpu_frame0_s']:.1f} s, frames ≥ 1 {c4['cpu_frames_ge1_s']:.2f} s per core) | "
             f"{c4['gpu_frames_per_s']:.0f} frames/s in a {c4['gpu_context_gb']:.0f} GB context, 1 volume chunk per reduced frame, "
             f"bit-exact spot check | {c4['speedup_vs_cpu_20_frame_mix']:.0f}× | {c4['aggregation_hbm_frac']:.3f} |")
    return "\n".join(L)


def replace_table(text, header_prefix, new):
    lines = text.split("\n")
    i = next(k for k, ln in enumerate(lines) if ln.startswith(header_prefix))
    j = i
    while j < len(lines) and lines[j].startswith("|"):
        j += 1
    return "\n".join(lines[:i] + new.split("\n") + lines[j:])


def main():
    path = os.path.join(ROOT, "DESIGN.md")
    s = open(path).read()
    s = replace_table(s, "| kernel | ms | DRAM %", kernel_table())
    s = replace_table(s, "| config | CPU reference", config_table())
    open(path, "w").write(s)
    print(kernel_table())
    print(config_table())


if __name__ == "__main__":
    main()
