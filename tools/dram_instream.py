"""In-stream DRAM traffic of the substep kernel: summarise a single-pass ncu
capture (``--metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control
none``: one pass per kernel, so no replay and no cache flush between the
launches of a batch -- the L2 state each launch sees is the one the previous
launch left, as in a real substep batch) into the median per-launch bytes of
the SUBSTEP launches (development tool).

    python tools/dram_instream.py gpurun_out/dram_instream_k4.csv conv2d_sf_kernel<4, 1> profiles/dram_instream_k4_r02.json
"""
import csv
import json
import statistics
import sys


def main(src, pattern, out):
    lines = [ln for ln in open(src) if ln.startswith('"')]
    per = {}
    for r in csv.DictReader(lines):
        if pattern not in r["Kernel Name"]:
            continue
        per.setdefault(r["ID"], {})[r["Metric Name"]] = float(r["Metric Value"])
    rd = [v["dram__bytes_read.sum"] for v in per.values()]
    wr = [v["dram__bytes_write.sum"] for v in per.values()]
    res = {"kernel": pattern, "launches": len(rd), "dram_read_bytes_median": statistics.median(rd),
           "dram_write_bytes_median": statistics.median(wr), "dram_read_bytes": rd, "dram_write_bytes": wr,
           "capture": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none "
                      "--clock-control none (single pass, L2 state carried from launch to launch)",
           "source": src}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps({k: v for k, v in res.items() if "median" in k or k == "launches"}))


if __name__ == "__main__":
    main(*sys.argv[1:4])
