#!/usr/bin/env python
"""Benchmark of the tsgm per-frame hot path on B200 (driver contract).

Workload (BASELINE.json configs[2], the metric's 1/2/4/8-GPU configuration):
64 independent synthetic stereo sequences x 30 frames at 1242x375, D=128,
8 paths, P1=10, P2=120, +-3 sigma reduced windows, seeds 0..63 with
(seed % 5) movers. A "step" is one pass of the hot path over the whole batch:
every slot reset to the empty state, then 30 batched frames (frame 0 full
range, 29 reduced). Sequences are sharded contiguously over ranks with no
data-path collective (one process per GPU); `value` = all frames all ranks
processed / max-over-ranks device time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: under torchrun (RANK/WORLD_SIZE/LOCAL_RANK in the environment) each
process is one rank; without them, ``--gpus N`` (N > 1) launches the N ranks
itself (one process per GPU, same environment contract as torchrun) and
forwards rank 0's JSON line. Ranks use NCCL only for the final stats gather
and the max-over-ranks timing (``--backend gloo --dry-run`` exercises this
launcher on CPU without the engine: tests/test_bench_launcher.py).

--impl reference times the reference's own CPU implementation (the
unmodified reference sources compiled in place into oracle/_ref, else the C
restatement) on ALL host cores over the FULL workload (64 sequences x 30
frames, one sequence per core at a time, compute only as eval.cpp:123-158
times it). Its frames come pre-rendered from tools/bin/render_frames (a
separate C process) and its motions from the reference's relative_motion, so
that process maps no library of the product package.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_, H_, D_ = 1242, 375, 128
N_SEQ, N_FRAMES = 64, 30
P1, P2 = 10, 120
HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback


def rank_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(n: int) -> int:
    """torchrun's contract without torchrun: N processes of this script with
    RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT set, one per GPU
    (rank r -> cuda:r). Rank 0 prints the JSON line (inherited stdout). Returns
    the worst exit code; a failing rank terminates the others."""
    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]],
                                      env=env))
    rc = 0
    alive = list(procs)
    while alive:
        for p in list(alive):
            code = p.poll()
            if code is None:
                continue
            alive.remove(p)
            rc = max(rc, abs(code))
            if code != 0:
                for q in alive:
                    q.terminate()
        time.sleep(0.05)
    return rc


def init_dist(args, world: int, local: int):
    """The process group of this rank (None at world size 1)."""
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist
    if args.backend == "nccl":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    return dist


def reduce_over_ranks(dist, x: float, op: str, device) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def scene_cfg(seed: int, frames: int = N_FRAMES):
    from paper_1809_07986_b200.scene import SceneConfig
    return SceneConfig.baseline_config(2, seed=seed, n_movers=seed % 5, frames=frames)


def params():
    from paper_1809_07986_b200 import tsgm
    calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, W_, H_, D_)
    sgm = tsgm.SgmParams(P1, P2, 8, 0, D_)
    filt = tsgm.FilterConfig(q=0.5, r=1.0, p_init=4096.0, disc_thresh=2.0,
                             min_range_halfwidth=2, range_use_stddev=True, range_stddev_gain=3.0)
    return calib, sgm, filt


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------- ours
def run_dry(args):
    """--dry-run: the multi-rank plumbing without the engine (CPU, gloo): each
    rank takes its contiguous shard, "steps" it (a checksum of its sequence
    ids), and the job line is built from the gathered stats and the
    max-over-ranks time exactly as for the GPU run. For the launcher tests."""
    from paper_1809_07986_b200.sharding import RankStats, gather_stats, job_throughput, shard
    rank, world, local = rank_info()
    dist = init_dist(args, world, local)
    my = list(shard(args.seqs, world, rank))
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    chk = 0
    for _ in range(args.steps):
        for s in my:
            chk = (chk * 31 + s) % 1000003
    ms = (time.perf_counter() - t0) * 1e3 / max(1, args.steps) + 1.0 + rank  # rank-dependent
    ms = reduce_over_ranks(dist, ms, "max", "cpu")
    stats = gather_stats(RankStats(rank, len(my), len(my) * args.frames, 0.0, ms))
    job = job_throughput(stats)
    if rank == 0:
        print(json.dumps({"metric": "dry-run (launcher plumbing only, no engine)", "dry_run": True,
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": ms, "value": job["frames_per_s"], "unit": "frames/s",
                          "frames": job["frames"], "max_device_ms": job["max_device_ms"],
                          "ranks": [[s.rank, s.sequences, s.frames] for s in stats],
                          "checksum": chk}), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_ours(args):
    import torch

    from paper_1809_07986_b200 import tsgm
    from paper_1809_07986_b200.scene import render
    from paper_1809_07986_b200.sharding import RankStats, gather_stats, job_throughput, shard

    rank, world, local = rank_info()
    torch.cuda.set_device(local)
    dist = init_dist(args, world, local)
    dev = f"cuda:{local}"
    my = list(shard(args.seqs, world, rank))
    n = len(my)
    calib, sgm, filt = params()

    # inputs: render this rank's sequences (host, pinned) and make them resident
    nthreads = os.cpu_count() or 8
    P = W_ * H_
    host_l = torch.empty((n, args.frames, H_, W_), dtype=torch.uint8).pin_memory()
    host_r = torch.empty((n, args.frames, H_, W_), dtype=torch.uint8).pin_memory()
    motions = np.zeros((n, args.frames, 12))
    for i, s in enumerate(my):
        cfg = scene_cfg(s, args.frames)
        L, R, poses, _ = render(cfg, 0, args.frames, threads=nthreads,
                                out_left=host_l[i].numpy(), out_right=host_r[i].numpy())
        for k in range(args.frames):
            if k == 0:
                Rm, t = np.eye(3), np.zeros(3)
            else:
                Rm, t = tsgm.relative_motion(poses[k - 1], poses[k])
            motions[i, k, :9] = Rm.ravel()
            motions[i, k, 9:] = t
    dev_l = host_l.to(dev)
    dev_r = host_r.to(dev)
    torch.cuda.synchronize()

    # contexts per GPU: the batch split over independent contexts (own
    # streams) so one group's issue-bound scan overlaps the others' DRAM-bound
    # kernels (tsgm.PipelinedEngine); auto = 2 for 16..63 sequences per GPU
    groups = args.groups if args.groups > 0 else (2 if 16 <= n < 64 else 1)
    ecfg = tsgm.EngineConfig(calib, sgm, filt, max_slots=n, device=local, keep_volumes=False)
    eng = tsgm.PipelinedEngine(ecfg, groups) if groups > 1 else tsgm.Engine(ecfg)
    slots = list(range(n))
    lptr = [[dev_l[i, k].data_ptr() for i in range(n)] for k in range(args.frames)]
    rptr = [[dev_r[i, k].data_ptr() for i in range(n)] for k in range(args.frames)]

    def one_step_device():
        for s in slots:
            eng.reset(s)
        for k in range(args.frames):
            eng.step_device(slots, lptr[k], rptr[k], motions[:, k, :])

    # pinned output buffers for the e2e leg (export map + posterior variance + mask)
    out_ed = torch.empty((n, H_, W_), dtype=torch.int32).pin_memory().numpy()
    out_ev = torch.empty((n, H_, W_), dtype=torch.uint8).pin_memory().numpy()
    out_p = torch.empty((n, H_, W_), dtype=torch.float64).pin_memory().numpy()
    out_mask = torch.empty((n, H_, W_), dtype=torch.uint8).pin_memory().numpy()
    host_l_np = host_l.numpy()
    host_r_np = host_r.numpy()

    def one_step_e2e():
        for s in slots:
            eng.reset(s)
        for k in range(args.frames):
            eng.step(slots, [host_l_np[i, k] for i in range(n)],
                     [host_r_np[i, k] for i in range(n)],
                     [(motions[i, k, :9].reshape(3, 3), motions[i, k, 9:]) for i in range(n)])
            eng.fetch_batch(slots, "export_d", [out_ed[i] for i in range(n)])
            eng.fetch_batch(slots, "export_valid", [out_ev[i] for i in range(n)])
            eng.fetch_batch(slots, "state_p", [out_p[i] for i in range(n)])
            eng.fetch_batch(slots, "mask", [out_mask[i] for i in range(n)])
        eng.sync()
    e2e_h2d = n * args.frames * 2 * P
    e2e_d2h = n * args.frames * P * (4 + 1 + 8 + 1)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up
    for _ in range(args.warmup):
        one_step_device()
    eng.sync()

    # timed region: device-resident inputs
    barrier()
    l0 = eng.launches
    with ClockSampler(local) as clk:
        eng.timer_begin()
        for _ in range(args.steps):
            one_step_device()
        ms = eng.timer_end()
    launches = (eng.launches - l0) // max(1, args.steps)
    barrier()
    ms = reduce_over_ranks(dist, ms, "max", dev)
    ms_per_step = ms / args.steps

    # cells per step (all frames) and accuracy — outside the timed region.
    # Accuracy: KITTI-style outliers (eval.cpp:59-85, 3 px and 5%) of the
    # export maps against the synthetic ground truth, pooled over sequences,
    # at frame 0 (full-range SGM) and at the last frame (the temporal path).
    gts = {}
    for k in (0, args.frames - 1):
        gts[k] = []
        for s in my:
            _, _, _, g = render(scene_cfg(s, args.frames), k, k + 1, threads=nthreads, gt=True)
            gts[k].append(g[0].astype(np.float64))
    acc = {}
    cells_step = 0.0
    for s in slots:
        eng.reset(s)
    for k in range(args.frames):
        eng.step_device(slots, lptr[k], rptr[k], motions[:, k, :])
        cells_step += sum(eng.cells(s) for s in slots)
        if k in gts:
            ev, out = eng.count_outliers(slots, gts[k], "export_d")
            n_valid = float(sum(int(eng.fetch(s, "export_valid").sum()) for s in slots))
            acc[k] = (reduce_over_ranks(dist, float(ev.sum()), "sum", dev),
                      reduce_over_ranks(dist, float(out.sum()), "sum", dev),
                      reduce_over_ranks(dist, n_valid, "sum", dev))
    stats = gather_stats(RankStats(rank, n, n * args.frames, cells_step, ms_per_step), device=dev)
    job = job_throughput(stats)
    cells_step = job["cells"]
    frames_total = job["frames"]

    # roofline of the dominant kernel (8-path C -> S aggregation), standalone,
    # on the last (reduced) frame's volumes of all slots
    # (with several contexts: one full-batch context, stepped through the
    # frames once more, so the launch is the same as with a single context)
    if groups > 1:
        eng.close()
        eng = tsgm.Engine(ecfg)
        for k in range(args.frames):
            eng.step_device(slots, lptr[k], rptr[k], motions[:, k, :])
        eng.sync()
    agg_ms, agg_cells = eng.bench_aggregate(slots, reps=10)
    if groups > 1:
        eng.close()
        eng = tsgm.PipelinedEngine(ecfg, groups)
    b_agg = 3.0 * agg_cells + 4.0 * P * n
    peak, peak_kind = peaks()
    achieved = b_agg / (agg_ms * 1e-3) / 1e9

    # e2e: public API with host buffers, H2D + D2H inside the timed region
    one_step_e2e()
    barrier()
    t0 = time.perf_counter()
    for _ in range(max(1, args.steps)):
        one_step_e2e()
    eng.sync()
    e2e_s = (time.perf_counter() - t0) / max(1, args.steps)
    e2e_s = reduce_over_ranks(dist, e2e_s, "max", dev)
    eng.close()
    barrier()

    result = None
    if rank == 0:
        value = frames_total / (ms_per_step * 1e-3)
        # the reference CPU path beside every GPU count (rank 0, after all
        # ranks have finished their GPU work)
        cpu = None if args.no_cpu_baseline else cpu_reference_sample(args)
        traffic = load_traffic(agg_cells)

        def acc_of(k):
            ev, out, nv = acc[k]
            return {"frame": k, "pooled_outlier_pct": round(100.0 * out / max(ev, 1.0), 3),
                    "evaluated_px": int(ev),
                    "density_pct": round(100.0 * nv / (args.seqs * W_ * H_), 2)}
        result = {
            "metric": "frames/sec (batched tsgm step, 1242x375, D=128, 8 paths)",
            "value": round(value, 2),
            "unit": "frames/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 3),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "u8/u16 cost+aggregation, f64 Kalman state",
            "data": "synthetic (seeded KITTI-like scenes, BASELINE configs[2]; no KITTI in image)",
            "config": {"workload": "configs[2]: 64 sequences x 30 frames, 1242x375",
                       "sequences": args.seqs, "frames": args.frames, "width": W_,
                       "height": H_, "d_max": D_, "paths": 8, "p1": P1, "p2": P2,
                       "window": "+-3 sigma (range_use_stddev, gain 3), min half-width 2",
                       "parallelism": f"sequence shards over {world} GPU(s), no collective",
                       "ranks": [[st.rank, st.sequences] for st in stats],
                       "contexts_per_gpu": groups,
                       "l2": "inputs larger than L2 (1.8 GB of frames + volumes per step)"},
            "gdisp_evals_per_s": round(cells_step / (ms_per_step * 1e-3) / 1e9, 3),
            "cells_per_step": int(cells_step),
            "e2e": {"value": round(frames_total / e2e_s, 2), "unit": "frames/s",
                    "h2d_bytes_per_step": int(e2e_h2d * world),
                    "d2h_bytes_per_step": int(e2e_d2h * world),
                    "outputs": "export map (i32 d + u8 valid), posterior p (f64), mask (u8)"},
            "roofline": {"bound": "hbm", "kernel": "8-path aggregation C->S (standalone)",
                         "achieved": round(achieved, 1), "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "algorithmic_bytes": int(b_agg), "ms": round(agg_ms, 4),
                         "cells": int(agg_cells), "limiter": load_limiter(achieved / peak)},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "accuracy": {"outlier_rule": "|e| > 3 px and |e|/gt > 5%",
                         "frame0_full_range": acc_of(0),
                         "last_frame_temporal": acc_of(args.frames - 1),
                         "counted_on": "GPU (tsgm_count_outliers_batch)"},
        }
        if cpu is not None:
            result["cpu_baseline"] = cpu
        print(json.dumps(result), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return result


def _num(v):
    try:
        return float(str(v).split()[0].replace(",", ""))
    except (TypeError, ValueError):
        return None


def load_limiter(frac=None):
    """What actually bounds the aggregation, from the committed ncu captures of
    the same standalone C->S launch (profiles/r0*_*_ncu_full.json): issue
    slots and DRAM per kernel, the measured DRAM bytes per cell, the scan's
    lane-instructions per cell-direction, and the two ceilings they imply for
    roofline.frac (all DRAM bytes at peak; the scan at 100% issue)."""
    out, caps = {}, {}
    for name, fns in (("scan", ("r02_scan_kernel_ncu_full.json", "r01_scan_kernel_ncu_full.json")),
                      ("combine", ("r02_combine_ncu_full.json", "r01_combine_ncu_full.json"))):
        for fn in fns:
            try:
                with open(os.path.join(ROOT, "profiles", fn)) as f:
                    d = json.load(f)
                k = next(v for k, v in d.items() if not k.startswith("_"))
                out[name] = {key: k.get(key) for key in ("issue_slots_busy_pct", "dram_throughput_pct",
                                                          "eligible_warps_per_scheduler",
                                                          "achieved_occupancy_pct")}
                out[name]["capture"] = fn
                caps[name] = (k, d.get("_cells"))
                break
            except (OSError, ValueError, StopIteration):
                continue
    if "scan" in caps and "combine" in caps and caps["scan"][1]:
        (ks, cells), (kc, _) = caps["scan"], caps["combine"]
        dram = sum(_num(k.get(m)) or 0.0 for k in (ks, kc)
                   for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        unit = 1e9 if "Gbyte" in str(ks.get("dram__bytes_read.sum")) else 1.0
        bpc = dram * unit / cells
        lipcd = (_num(ks.get("executed_instructions")) or 0.0) * 32.0 / (8.0 * cells)
        out["capture_cells"] = int(cells)
        out["dram_bytes_per_cell"] = round(bpc, 2)
        out["scan_lane_instr_per_cell_direction"] = round(lipcd, 2)
        out["ceiling_frac_all_bytes_at_peak"] = round(3.17 / bpc, 4)
        issue = _num(ks.get("issue_slots_busy_pct"))
        if frac is not None and issue:
            out["ceiling_frac_scan_at_full_issue"] = round(frac * 100.0 / issue, 4)
    if out:
        out["reading"] = ("the scan is integer-issue bound (exact u16x2 min-plus recursions); "
                          "see DESIGN.md section 4")
    return out or None


def load_traffic(cells: float):
    """DRAM bytes of the aggregation launch, from the committed ncu capture
    (profiles/traffic.json: measured bytes per cell x this launch's cells)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return int(t["bytes_per_cell"] * cells)
    except Exception:
        return None


# ---------------------------------------------------------------------- reference (CPU)
def cpu_model() -> str:
    """The host CPU (report the CPU model with the core count)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def render_tool() -> str:
    path = os.path.join(ROOT, "tools", "bin", "render_frames")
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
    return path


def load_sequences(seeds, frames: int):
    """Frames + poses of config-2 sequences from tools/bin/render_frames (a
    separate C process: this process maps no product library)."""
    import tempfile
    P = W_ * H_
    per = 2 * P * frames + 96 * frames
    d = "/dev/shm" if os.path.isdir("/dev/shm") else None
    with tempfile.NamedTemporaryFile(dir=d, suffix=".bin") as tf:
        subprocess.run([render_tool(), "2", str(seeds[0]), str(seeds[-1] + 1), str(frames), tf.name],
                       check=True)
        raw = np.fromfile(tf.name, np.uint8)
    if raw.size != per * len(seeds):
        raise RuntimeError("render_frames: unexpected output size")
    out = []
    for i in range(len(seeds)):
        b = raw[i * per:(i + 1) * per]
        L = b[:P * frames].reshape(frames, H_, W_)
        R = b[P * frames:2 * P * frames].reshape(frames, H_, W_)
        poses = b[2 * P * frames:].view(np.float64).reshape(frames, 12)
        out.append((L, R, poses))
    return out


def reference_impl():
    """The reference compiled in place (oracle/_ref/libtsgm_ref.so), else the
    C restatement; with the reference's own relative_motion."""
    from oracle import oracle as o
    try:
        return o.reference(), "reference"
    except Exception:
        return o.port(), "port"


def run_cpu_sequences(seqs, threads: int):
    """One sequence per host thread (step() is re-entrant), every frame of
    each; returns (wall seconds, per-frame seconds). Compute only: the frames
    and motions are prepared before the clock starts (eval.cpp:123-158)."""
    from oracle import oracle as o
    impl, kind = reference_impl()
    calib = o.Calib(720.0, 621.0, 187.5, 0.54, W_, H_, D_)
    sgm = o.SgmParams(P1, P2, 8, 0, D_)
    filt = o.FilterConfig(q=0.5, r=1.0, p_init=4096.0, disc_thresh=2.0, min_range_halfwidth=2,
                          range_use_stddev=True, range_stddev_gain=3.0)
    prepared = []
    for (L, R, poses) in seqs:
        mot = [(np.eye(3), np.zeros(3))]
        for k in range(1, len(L)):
            mot.append(impl.relative_motion(poses[k - 1], poses[k]))
        prepared.append((L, R, mot))

    def run_seq(i):
        L, R, mot = prepared[i]
        st = None
        times = []
        for k in range(len(L)):
            t0 = time.perf_counter()
            res = impl.step(st, L[k], R[k], mot[k][0], mot[k][1], calib, sgm, filt)
            times.append(time.perf_counter() - t0)
            st = (res["d"], res["p"], res["valid"])
        return times

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        all_times = list(ex.map(run_seq, range(len(prepared))))
    return time.perf_counter() - t0, all_times, kind


def cpu_reference_sample(args):
    """cpu_baseline of our arm: the reference on the host cores, one config-2
    sequence per core for all 30 frames (no extrapolation), ~10 s."""
    threads = os.cpu_count() or 1
    seqs = load_sequences(list(range(threads)), N_FRAMES)
    wall, times, kind = run_cpu_sequences(seqs, threads)
    frames = sum(len(t) for t in times)
    t_first = float(np.mean([t[0] for t in times]))
    t_rest = float(np.mean([x for t in times for x in t[1:]]))
    return {"value": round(frames / wall, 3), "unit": "frames/s", "cores": threads, "kind": kind,
            "cpu_model": cpu_model(),
            "sample": (f"{threads} config-2 sequences (seeds 0..{threads - 1}, one per core) x "
                       f"{N_FRAMES} frames, all frames timed, {wall:.1f}s wall; per frame under "
                       f"full concurrency: frame 0 {t_first:.3f}s, frames>=1 {t_rest:.3f}s")}


def run_reference(args):
    """The reference arm: the reference's CPU implementation on all host cores
    over the FULL config-2 workload (64 sequences x 30 frames) once."""
    rank, world, _ = rank_info()
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    seeds = list(range(args.seqs))
    seqs = load_sequences(seeds, args.frames)
    wall, times, kind = run_cpu_sequences(seqs, threads)
    frames = sum(len(t) for t in times)
    value = frames / wall
    t_first = float(np.mean([t[0] for t in times]))
    t_rest = float(np.mean([x for t in times for x in t[1:]]))
    cpu = {"value": round(value, 3), "unit": "frames/s", "cores": threads, "kind": kind,
           "cpu_model": cpu_model(),
           "sample": (f"full workload: {args.seqs} sequences x {args.frames} frames on {threads} "
                      f"threads (one sequence per thread at a time), {wall:.1f}s wall, compute "
                      f"only; per frame: frame 0 {t_first:.3f}s, frames>=1 {t_rest:.3f}s")}
    result = {
        "metric": "frames/sec (batched tsgm step, 1242x375, D=128, 8 paths)",
        "value": round(value, 3), "unit": "frames/s", "n_gpus": world,
        "steps": 1, "steps_requested": args.steps, "warmup": 0,
        "ms_per_step": round(wall * 1e3, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "u8/u16 cost+aggregation, f64 Kalman state",
        "data": "synthetic (seeded KITTI-like scenes, BASELINE configs[2])",
        "config": {"workload": "configs[2]: 64 sequences x 30 frames, 1242x375",
                   "sequences": args.seqs, "frames": args.frames, "d_max": D_, "paths": 8,
                   "p1": P1, "p2": P2, "same_config": True,
                   "inputs": "tools/bin/render_frames (separate C process), relative_motion of "
                             "the reference"},
        "impl": "reference",
        "cpu_baseline": cpu,
        "e2e": {"value": round(value, 3), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(result), flush=True)
    return result


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seqs", type=int, default=N_SEQ)
    ap.add_argument("--frames", type=int, default=N_FRAMES)
    ap.add_argument("--groups", type=int, default=0,
                    help="contexts per GPU (0 = auto: 2 for 16..63 sequences per GPU)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher/rank plumbing only, no engine (CPU tests)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)  # rank 0 of any launch; the CPU needs no ranks
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args.gpus))
    if args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
