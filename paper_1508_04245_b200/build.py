"""In-tree build of the CUDA library (sm_100a) — ``python -m paper_1508_04245_b200.build``.

Produces ``paper_1508_04245_b200/libhdgconv.so``.  Every translation unit
(hdgconv.cu: C ABI + setup kernels; order_k<K>.cu: the kernels of order K)
is compiled in parallel with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -Xptxas -v -c``
and linked with ``nvcc -shared``.  Objects are cached by source mtime.  The
.so is git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
OUT = os.path.join(HERE, "libhdgconv.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# no library dependencies beyond the CUDA runtime (every kernel is in csrc/)
LIBS = []
FLAGS = ["-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "hdgconv.h")])


def units():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src):
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    if not _stale(obj, [src] + headers()):
        return obj, None
    cmd = [nvcc(), *ARCH, *FLAGS, "-c", "-o", obj + ".tmp", src]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{res.stdout}{res.stderr}")
    os.replace(obj + ".tmp", obj)
    with open(obj[:-2] + ".ptxas.log", "w") as fh:
        fh.write(res.stderr)
    return obj, res.stderr


def _tables_object() -> str:
    """The built-in reference tables of hdgc_create_k: tables_blob.py writes
    them (same code path as forms.device_tables), an .incbin assembly stub
    puts them into .rodata of the library."""
    blob = os.path.join(OBJ, "tables_blob.bin")
    asm = os.path.join(OBJ, "tables_blob.S")
    obj = os.path.join(OBJ, "tables_blob.o")
    deps = [os.path.join(HERE, f) for f in ("tables_blob.py", "basis.py", "basis3d.py", "forms.py")]
    if _stale(blob, deps):
        sys.path.insert(0, ROOT)
        from paper_1508_04245_b200 import tables_blob
        tables_blob.write_blob(blob + ".tmp")
        os.replace(blob + ".tmp", blob)
    if _stale(obj, [blob]):
        with open(asm, "w") as fh:
            fh.write("  .section .rodata\n  .balign 16\n  .globl hdgc_tables_blob\n"
                     "  .type hdgc_tables_blob, @object\nhdgc_tables_blob:\n"
                     f'  .incbin "{blob}"\n  .globl hdgc_tables_blob_end\nhdgc_tables_blob_end:\n'
                     '  .section .note.GNU-stack,"",@progbits\n')
        subprocess.check_call(["gcc", "-c", "-fPIC", "-o", obj, asm])
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in glob.glob(os.path.join(OBJ, "*.o")) + glob.glob(os.path.join(OBJ, "tables_blob.*")):
            os.remove(f)
    srcs = units()
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, srcs))
    objs = [o for o, _ in results] + [_tables_object()]
    if _stale(OUT, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", OUT + ".tmp", *objs, *LIBS]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}{res.stderr}")
        os.replace(OUT + ".tmp", OUT)
    if verbose:
        for _, log in results:
            if log:
                print(log)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
