"""Per-source-line warp-stall profile from an ncu report (development tool).

    python tools/ncu_lines.py <report.ncu-rep> <object.o> [top]

Reads the SASS source page of the (first) kernel in the report, maps each
instruction offset to its CUDA source line with ``nvdisasm -g`` on the same
build's cubin (extracted from the object file), and prints the lines with the
most stall samples and their dominant stall reasons.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, obj, top=30):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    kname = rows[0][1]
    h = rows[1]
    data = []
    for r in rows[2:]:          # first launch only (a report may hold several)
        if len(r) != len(h) or r[0] == h[0]:
            if data:
                break
            continue
        data.append(r)
    iS = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    base = int(data[0][0], 16)
    mangled = None
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
        cub = [os.path.join(td, f) for f in os.listdir(td) if f.endswith(".cubin")][0]
        sass = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    # pick the function whose SASS matches the report's first instructions
    funcs = re.split(r"\n\s*\.text\.", sass)
    targs = "".join(f"Li{v}E" for v in re.findall(r"\(int\)(-?\d+)", kname))
    funcs = [f for f in funcs if targs in f.split(":", 1)[0]] or funcs
    want = [re.sub(r"\s+", " ", r[1].strip().rstrip(";")) for r in data[:12]]
    line_of = {}
    for f in funcs:
        name = f.split(":", 1)[0]
        ins = {}
        cur = None
        for ln in f.splitlines():
            m = re.search(r'line (\d+)', ln)
            if "//##" in ln and m:
                fm = re.search(r'File "([^"]+)"', ln)
                cur = (os.path.basename(fm.group(1)) if fm else "?", int(m.group(1)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", ln)
            if m:
                ins[int(m.group(1), 16)] = (cur, re.sub(r"\s+", " ", m.group(2).strip()))
        seq = [v[1] for _, v in sorted(ins.items())][:12]
        if len(seq) == 12 and all(a.split(" ")[0] == b.split(" ")[0] for a, b in zip(seq, want)):
            mangled = name
            line_of = {o: v[0] for o, v in ins.items()}
            break
    if mangled is None:
        sys.exit("could not match the report's kernel to a function in the object")
    agg = collections.defaultdict(lambda: collections.Counter())
    tot = 0.0
    for r in data:
        off = int(r[0], 16) - base
        key = line_of.get(off)
        s = float(r[iS] or 0)
        tot += s
        agg[key]["_all"] += s
        for i in stall_cols:
            agg[key][h[i]] += float(r[i] or 0)
    print(f"{kname}  ({mangled}), {tot:.0f} samples")
    for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["_all"])[:top]:
        reasons = ", ".join(f"{n[6:]} {v / c['_all'] * 100:.0f}%" for n, v in c.most_common(5) if n != "_all" and v)
        print(f"{c['_all'] / tot * 100:5.1f}%  {key}  [{reasons}]")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
