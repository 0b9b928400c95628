"""Summarise an ncu source-page export (`ncu -i rep --page source --csv`) of one
kernel: total warp-instructions and stall samples, the L1 request totals, the
SASS split into regions of equal execution count (loop bodies and branches
show up as runs of instructions executed equally often), and the
instructions holding the most stall samples.

    python tools/source_regions.py <source.csv> <out.json> [min_share_pct]
"""
import csv
import json
import sys


def main():
    src, out = sys.argv[1:3]
    min_share = float(sys.argv[3]) if len(sys.argv) > 3 else 0.4
    rows = list(csv.reader(open(src)))
    kernel = rows[0][1] if rows and len(rows[0]) > 1 else ""
    hdr, data = rows[1], rows[2:]
    ci, si = hdr.index("Instructions Executed"), hdr.index("# Samples")
    num = lambda r, i: int(r[i] or 0)  # noqa: E731
    tot, ts = sum(num(r, ci) for r in data), sum(num(r, si) for r in data)
    res = {"kernel": kernel, "warp_instructions": tot, "stall_samples": ts, "sass_lines": len(data)}
    for c in ("L1 Tag Requests Global", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
              "L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Ideal"):
        if c in hdr:
            res[c.lower().replace(" ", "_")] = sum(num(r, hdr.index(c)) for r in data)
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    res["stall_reasons_pct"] = {hdr[i]: round(100.0 * sum(num(r, i) for r in data) / max(ts, 1), 1)
                                for i in stall_cols if sum(num(r, i) for r in data) > 0.005 * ts}
    segs, cur = [], None
    for i, r in enumerate(data):
        c = num(r, ci)
        if cur is None or abs(c - cur["executions"]) > 0.02 * max(c, cur["executions"], 1):
            cur = {"first_sass_line": i, "last_sass_line": i, "executions": c, "instr": 0, "samples": 0,
                   "starts_with": r[1].strip()[:60]}
            segs.append(cur)
        cur["last_sass_line"] = i
        cur["instr"] += c
        cur["samples"] += num(r, si)
    res["regions"] = [
        {"sass_lines": [s["first_sass_line"], s["last_sass_line"]],
         "instructions_in_region": s["last_sass_line"] - s["first_sass_line"] + 1,
         "executions": s["executions"], "share_of_instructions_pct": round(100.0 * s["instr"] / tot, 2),
         "share_of_stall_samples_pct": round(100.0 * s["samples"] / max(ts, 1), 2),
         "starts_with": s["starts_with"]}
        for s in segs if s["instr"] > min_share / 100.0 * tot]
    top = sorted(range(len(data)), key=lambda i: -num(data[i], si))[:12]
    res["top_stall_instructions"] = [
        {"sass_line": i, "sass": data[i][1].strip()[:70], "executions": num(data[i], ci),
         "stall_samples_pct": round(100.0 * num(data[i], si) / max(ts, 1), 2),
         "top_reason": max(((hdr[j], num(data[i], j)) for j in stall_cols), key=lambda x: x[1])[0]}
        for i in top]
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k not in ("regions", "top_stall_instructions")},
                     indent=1))


if __name__ == "__main__":
    main()
