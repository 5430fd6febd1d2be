"""Build a variant of libhdgconv.so in which only order_k<K>.cu (or
order3d_k<K>.cu with dim=3) is recompiled with extra nvcc flags; every other
object comes from the default in-tree build (development A/B tool).

    python tools/build_order_variant.py <name> <K> [3d] [flags...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1508_04245_b200 import build as B  # noqa: E402


def main(name, k, *flags):
    three = bool(flags) and flags[0] == "3d"
    if three:
        flags = flags[1:]
    B.build()
    unit = f"order3d_k{k}" if three else f"order_k{k}"
    out = os.path.join(ROOT, "tools", "variants", name)
    os.makedirs(out, exist_ok=True)
    obj = os.path.join(out, unit + ".o")
    r = subprocess.run([B.nvcc(), *B.ARCH, *B.FLAGS, *flags, "-c", "-o", obj, os.path.join(B.CSRC, unit + ".cu")],
                       capture_output=True, text=True, timeout=1800)
    open(obj[:-2] + ".log", "w").write(r.stderr)
    if r.returncode:
        raise RuntimeError(r.stderr)
    objs = [os.path.join(B.OBJ, os.path.basename(s)[:-3] + ".o") for s in B.units()
            if os.path.basename(s)[:-3] != unit] + [obj, B._tables_object()]
    lib = os.path.join(out, "libhdgconv.so")
    subprocess.check_call([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs])
    for line in r.stderr.splitlines():
        if "spill" in line or "Used" in line:
            pass
    print(lib)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *sys.argv[3:])
