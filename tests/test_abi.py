"""C-ABI library: loads, exports every symbol include/hdgconv.h declares, and
rejects bad arguments with status codes + last-error text — no GPU needed."""

import ctypes as C
import os
import re

import pytest

from paper_1508_04245_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "hdgconv.h")).read()
    return sorted(set(re.findall(r"\b(hdgc_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header_symbols():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SYMBOLS)


def test_version_and_error_paths():
    lib = _lib.load()
    assert b"sm_100a" in lib.hdgc_version()
    h = C.c_void_p()
    rc = lib.hdgc_create(None, None, C.byref(h))
    assert rc == -1 and b"null" in lib.hdgc_last_error()
    md = _lib.MeshDesc(dim=5)
    td = _lib.TablesDesc(k=4)
    assert lib.hdgc_create(C.byref(md), C.byref(td), C.byref(h)) == -4    # unsupported dim
    md.dim = 2
    td.k = 12
    assert lib.hdgc_create(C.byref(md), C.byref(td), C.byref(h)) == -4    # unsupported order
    td.k, td.nqv, td.nf = 4, 35, 7
    assert lib.hdgc_create(C.byref(md), C.byref(td), C.byref(h)) == -1    # wrong rule size
    assert b"nqv" in lib.hdgc_last_error()
    assert lib.hdgc_apply_v(None, None, None, None, None, None) == -1
    assert lib.hdgc_destroy(None) == 0


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load(str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_LIB", None)
    _lib.load()


def test_operator_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1508_04245_b200 import mesh as M
    from paper_1508_04245_b200.forms import ConvectionOperator
    with pytest.raises(RuntimeError, match="CUDA"):
        ConvectionOperator(M.generate_structured((0, 0, 1, 1), 2, 2), 2)


def test_library_has_no_cublas_dependency():
    """Every kernel is in csrc/: the library links no BLAS (only the CUDA runtime)."""
    import subprocess
    out = subprocess.run(["readelf", "-d", _lib.LIB_PATH], capture_output=True, text=True).stdout
    needed = [l for l in out.splitlines() if "NEEDED" in l]
    assert needed and not any("blas" in l.lower() for l in needed), needed


def test_builtin_table_blob_matches_python_tables():
    """hdgc_create_k's tables (build-time blob in the library) are exactly the
    arrays ConvectionOperator passes to hdgc_create (same basis modules)."""
    import struct
    import numpy as np
    from paper_1508_04245_b200 import build as Bd
    from paper_1508_04245_b200 import tables_blob as TB
    raw = open(os.path.join(Bd.OBJ, "tables_blob.bin"), "rb").read()
    magic, n = struct.unpack_from("<2q", raw, 0)
    assert magic == TB.MAGIC and n == len(TB.ORDERS)
    per = 5 + 2 * len(TB.FIELDS)
    hdr = struct.unpack_from(f"<{n * per}q", raw, 16)
    data = np.frombuffer(raw, dtype="<f8", offset=16 + 8 * n * per)
    for e in range(n):
        dim, k, nqv, nf, col_n = hdr[e * per:e * per + 5]
        if (dim, k) not in ((2, 2), (2, 4), (3, 3)):
            continue
        ref = TB.entry_tables(dim, k)
        assert (nqv, nf, col_n) == (ref["nqv"], ref["nf"], ref["col_n"])
        for i, f in enumerate(TB.FIELDS):
            off, cnt = hdr[e * per + 5 + 2 * i:e * per + 7 + 2 * i]
            a = ref["arrays"].get(f)
            assert (cnt == 0) == (a is None), (dim, k, f)
            if a is not None:
                assert np.array_equal(data[off:off + cnt], a), (dim, k, f)
