"""Config 2's strong-scaling shares on one B200: bench.py at
64/G sequences per GPU for G = 1, 2, 4, 8 (64, 32, 16, 8 sequences), each
share's frames/s as a fraction of the 64-sequence rate.

    python tools/batch_sweep.py > profiles/r02_batch_sweep.json
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rows = []
    for n in (64, 32, 16, 8):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--seqs", str(n),
                              "--no-cpu-baseline"], capture_output=True, text=True, check=True)
        d = json.loads(out.stdout.strip().splitlines()[-1])
        rows.append({"sequences": n, "gpus_equivalent": 64 // n, "value": d["value"],
                     "e2e": d["e2e"]["value"]})
    for r in rows:
        r["share"] = round(r["value"] / rows[0]["value"], 3)
        r["job_frames_per_s_if_linear_over_gpus"] = round(r["value"] * r["gpus_equivalent"], 1)
    print(json.dumps({"workload": "configs[2] at 64/G sequences per GPU, 30 frames, 1242x375",
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
