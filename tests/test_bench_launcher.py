"""bench.py's multi-rank launcher and its reference arm, on CPU.

* ``--gpus N`` without torchrun spawns N ranks with torchrun's environment
  contract; ``--backend gloo --dry-run`` runs the rank plumbing (contiguous
  shards, barrier, max-over-ranks time, stats gather, rank-0 JSON line)
  without the engine.
* ``--impl reference`` runs the reference's CPU step over every frame of
  every sequence, with frames from the separate render tool; its process maps
  no library of the product package.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=300, env=None):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout, env=e)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("world,sizes", [(2, [32, 32]), (3, [22, 21, 21])])
def test_launcher_spawns_ranks(world, sizes):
    j = _bench("--gpus", str(world), "--backend", "gloo", "--dry-run", "--steps", "2",
               "--warmup", "0")
    assert j["dry_run"] and j["n_gpus"] == world
    assert [r[1] for r in j["ranks"]] == sizes
    assert [r[0] for r in j["ranks"]] == list(range(world))
    assert j["frames"] == 64 * 30
    # every rank adds 1 + rank ms to its time: the job time is the slowest rank's
    assert j["max_device_ms"] >= 1.0 + (world - 1)
    assert j["ms_per_step"] == j["max_device_ms"]


def test_launcher_under_torchrun_env_is_one_rank():
    """With WORLD_SIZE=1 in the environment the script is a single rank (the
    torchrun path) and does not spawn."""
    j = _bench("--gpus", "4", "--backend", "gloo", "--dry-run", "--steps", "1",
               env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert j["n_gpus"] == 1 and j["ranks"] == [[0, 64, 1920]]


def test_reference_arm_maps_no_product_library():
    from oracle import oracle as o
    if not os.path.exists(o.REF_SO) and not os.path.exists(o.PORT_SO):
        pytest.skip("oracle not built")
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--seqs','2',"
            "'--frames','2']; import bench; bench.main(); "
            "maps=open('/proc/self/maps').read(); "
            "print('PRODUCT_MAPPED', 'paper_1809_07986_b200/lib' in maps)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    j = json.loads(next(ln for ln in r.stdout.splitlines() if ln.startswith("{")))
    assert j["impl"] == "reference" and j["config"]["same_config"]
    assert j["cpu_baseline"]["kind"] in ("reference", "port")
    assert j["e2e"]["h2d_bytes_per_step"] == 0
    assert "PRODUCT_MAPPED False" in r.stdout
