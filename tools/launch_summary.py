"""Summarise an ncu ``--metrics gpu__time_duration.sum --csv`` launch list into
per-kernel launch counts, mean durations and share of the captured time
(development tool).

    python tools/launch_summary.py gpurun_out/launches.csv profiles/launches_bench_r01_summary.json
"""
import csv
import json
import re
import sys


def main(src, out):
    lines = [ln for ln in open(src) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    acc = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*$", "", r["Kernel Name"]).strip()
        t = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        a = acc.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in acc.values())
    res = {k: {"launches": n, "mean_us": s / n, "share": s / tot} for k, (n, s) in acc.items()}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
