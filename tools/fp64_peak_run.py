"""Run tools/fp64_peak (DFMA / DMMA / mixed microbenchmarks) with nvidia-smi
clock sampling during the run; print one JSON line with the peaks and the
clock record (median SM clock under load, max clock, throttle reasons).

  python tools/fp64_peak_run.py > profiles/fp64_peak_r02.json
"""

import json
import os
import statistics
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    exe = os.path.join(HERE, "fp64_peak")
    if not os.path.exists(exe):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                               os.path.join(HERE, "fp64_peak.cu")])
    log = "/tmp/fp64_peak_clocks.csv"
    smi = subprocess.Popen(["nvidia-smi", "--id=0",
                            "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                            "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                            "clocks_event_reasons.sw_power_cap,utilization.gpu",
                            "--format=csv,noheader,nounits", "-lms", "20"],
                           stdout=open(log, "w"), stderr=subprocess.DEVNULL)
    try:
        out = subprocess.check_output([exe], text=True)
    finally:
        smi.terminate()
        smi.wait()
    d = json.loads(out)
    rows = [[x.strip() for x in ln.split(",")] for ln in open(log) if ln.count(",") >= 6]
    busy = [r for r in rows if r[6].isdigit() and int(r[6]) > 50]
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    d["clocks"] = {
        "samples": len(rows), "samples_under_load": len(busy),
        "sm_mhz_median_under_load": statistics.median(float(r[0]) for r in busy) if busy else None,
        "sm_max_mhz": float(rows[0][1]) if rows else None,
        "reasons": sorted({n for r in rows for n, v in zip(names, r[2:6]) if v.lower() == "active"}),
    }
    print(json.dumps(d))


if __name__ == "__main__":
    sys.exit(main())
