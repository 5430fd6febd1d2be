"""Per-kernel SASS instruction summary of the built objects (cuobjdump -sass):
counts of the instructions that prove the B200 paths (DMMA tensor-core FP64,
UBLKCP / UTMA* bulk copies, SYNCS mbarrier ops, LDGSTS cp.async) and the ones
that flag spills (LDL / STL), plus DFMA / LDS / LDC.  Static counts (one per
instruction in the binary), not executed counts.

  python tools/sass_summary.py > profiles/sass_r02.json
"""
import glob
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["DMMA", "DFMA", "DMUL", "DADD", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "LDGSTS", "LDL", "STL", "LDS",
       "STS", "LDC", "LDG", "STG", "SHFL", "BAR"]
INTERESTING = re.compile(r"conv2d_sf_kernel|conv2d_sfm_kernel|conv2d_thread_kernel|conv2d_thread_split_kernel|prep_thread2d|conv3d_kernel|prep_tile2d|"
                         r"prep_modal2d|prep_tile3d|prep_fused2d|richardson|modal_rows")


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    res = {}
    for obj in sorted(glob.glob(os.path.join(ROOT, "paper_1508_04245_b200", "_obj", "*.o"))):
        txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        funcs = re.split(r"\n\s*Function : ", txt)
        names = []
        bodies = {}
        for f in funcs[1:]:
            name = f.split("\n", 1)[0].strip()
            names.append(name)
            bodies[name] = f
        dm = demangle(names)
        for name in names:
            pretty = dm.get(name, name)
            if not INTERESTING.search(pretty):
                continue
            body = bodies[name]
            ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", body)
            counts = {op: sum(1 for i in ins if i.split(".")[0] == op) for op in OPS}
            counts["total"] = len(ins)
            res[pretty] = {"object": os.path.basename(obj), **counts}
    json.dump(res, sys.stdout, indent=1, sort_keys=True)
    print()


if __name__ == "__main__":
    main()
