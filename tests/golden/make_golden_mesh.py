"""Golden fixtures for the text mesh loader (mesh.load_mesh) FROM THE
REFERENCE loader (hdgflow.mesh2d.load_mesh, MESH:298-334):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_mesh.py

Parses every tests/golden/meshes/*.txt with the reference and stores the
resulting Mesh arrays in tests/golden/mesh_load.npz (keys <name>__<attr>),
plus the reference's error message for each malformed case.
"""
from __future__ import annotations

import glob
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
from hdgflow import mesh2d as rmesh  # noqa: E402  (reference)

ATTRS = ("vertices", "triangles", "facet_vertices", "facet_elems", "facet_local", "facet_flip")

BAD = {
    "bad_header": "3 1\n0 0\n1 0\n0 1\n0 1 2\n",
    "bad_count": "3 1 0\n0 0\n1 0\n0 1\n",
    "bad_float": "3 1 0\n0 0\n1 x\n0 1\n0 1 2\n",
    "bad_index": "3 1 0\n0 0\n1 0\n0 1\n0 1 3\n",
    "bad_marker": "3 1 1\n0 0\n1 0\n0 1\n0 1 2\n0 1\n",
    "empty": "# nothing\n\n",
}


def main():
    out = {}
    for path in sorted(glob.glob(os.path.join(HERE, "meshes", "*.txt"))):
        name = os.path.basename(path)[:-4]
        m = rmesh.load_mesh(path)
        for a in ATTRS:
            out[f"{name}__{a}"] = np.asarray(getattr(m, a))
        labels = getattr(m, "facet_labels", None)
        if labels is not None:
            f = np.array(sorted(labels), dtype=np.int64)
            out[f"{name}__label_facets"] = f
            out[f"{name}__label_names"] = np.array([labels[i] for i in f])
    for name, text in BAD.items():
        p = os.path.join("/tmp", f"golden_mesh_{name}.txt")
        with open(p, "w") as fh:
            fh.write(text)
        try:
            rmesh.load_mesh(p)
            out[f"err__{name}"] = np.array("")
        except rmesh.MeshError as e:
            out[f"err__{name}"] = np.array(str(e).replace(p, "<path>"))
    np.savez(os.path.join(HERE, "mesh_load.npz"), **out)
    print(sorted(out))


if __name__ == "__main__":
    main()
