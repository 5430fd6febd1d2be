"""Build-time table blob for ``hdgc_create_k`` (include/hdgconv.h).

``hdgc_create`` takes the reference-element tables from the caller; a caller
without this package (C, Go, Rust ... over the C ABI) would have to
re-implement the BDM / Dubiner / quadrature construction.  ``build.py``
therefore runs :func:`write_blob` once per build: it evaluates exactly the
tables ``forms.device_tables`` / ``device_tables3`` upload (basis.py and
basis3d.py, pinned bit-identical to the reference's ``hdgflow.polybasis``)
for every supported (dim, k) — 2D k = 1..8, 3D k = 1..4 — and writes them as
one binary blob that is assembled into ``libhdgconv.so`` (``.incbin``), where
``hdgc_create_k(mesh, k)`` looks them up.

Blob layout (little-endian): int64 magic ``MAGIC``, int64 entry count, then
per entry 5 int64 (dim, k, nqv, nf, col_n) and ``len(FIELDS)`` (offset,
count) int64 pairs (offsets in doubles from the start of the data section,
count 0 = field absent), then the float64 data section.
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = 0x314C4254_43474448          # "HDGCTBL1"
FIELDS = ("coef", "div_modal", "vol_w", "vol_D", "vol_G", "fac_w", "fac_L", "fac_D", "fac_len",
          "col_A", "col_Ad", "col_B", "col_Bd", "col_xi", "col_wa", "col_wy", "col_inv1my",
          "col_C", "col_Cd", "col_pf")
ORDERS = [(2, k) for k in range(1, 9)] + [(3, k) for k in range(1, 5)]


def entry_tables(dim: int, k: int) -> dict:
    """The table arrays of one (dim, k), as ConvectionOperator passes them."""
    from . import basis as B
    from .forms import device_tables, device_tables3
    if dim == 2:
        tab = device_tables(k)
        out = {f: tab[f] for f in FIELDS[:9]}
        col_n = 0
        if k >= 3:
            ct = B.collapsed_tables(k)
            col_n = ct["n"]
            for name in ("A", "Ad", "B", "Bd", "xi", "wa", "wy", "inv1my"):
                out["col_" + name] = ct[name]
    else:
        tab = device_tables3(k)
        out = {f: tab[f] for f in FIELDS[:9]}
        ct = tab["col3"]
        col_n = ct["n"]
        for name in ("A", "Ad", "B", "Bd", "C", "Cd", "pf"):
            out["col_" + name] = ct[name]
    return {"nqv": int(tab["nqv"]), "nf": int(tab["nf"]), "col_n": int(col_n),
            "arrays": {f: np.ascontiguousarray(v, dtype=np.float64).ravel() for f, v in out.items()}}


def write_blob(path: str) -> None:
    entries = [(dim, k, entry_tables(dim, k)) for dim, k in ORDERS]
    header = [MAGIC, len(entries)]
    data = []
    off = 0
    for dim, k, e in entries:
        header += [dim, k, e["nqv"], e["nf"], e["col_n"]]
        for f in FIELDS:
            a = e["arrays"].get(f)
            if a is None:
                header += [0, 0]
            else:
                header += [off, a.size]
                data.append(a)
                off += a.size
    with open(path, "wb") as fh:
        fh.write(struct.pack(f"<{len(header)}q", *header))
        fh.write(np.concatenate(data).astype("<f8").tobytes())
