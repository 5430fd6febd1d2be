"""Build an experimental variant of libhdgconv.so with extra nvcc flags into
tools/variants/<name>/ (load it with HDGC_LIB=...)."""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1508_04245_b200", "csrc")


def main(name, *flags):
    out = os.path.join(ROOT, "tools", "variants", name)
    os.makedirs(out, exist_ok=True)
    base = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
            "-Xcompiler", "-fPIC", "-Xptxas", "-v", *flags]

    def comp(src):
        obj = os.path.join(out, os.path.basename(src)[:-3] + ".o")
        r = subprocess.run(base + ["-c", "-o", obj, src], capture_output=True, text=True, timeout=1800)
        open(obj[:-2] + ".log", "w").write(r.stderr)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, sorted(glob.glob(os.path.join(CSRC, "*.cu")))))
    sys.path.insert(0, ROOT)
    from paper_1508_04245_b200 import build as B
    os.makedirs(B.OBJ, exist_ok=True)
    objs.append(B._tables_object())   # built-in tables of hdgc_create_k
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                           os.path.join(out, "libhdgconv.so"), *objs,
                           ])
    print(os.path.join(out, "libhdgconv.so"))


if __name__ == "__main__":
    main(sys.argv[1], *sys.argv[2:])
