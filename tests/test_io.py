"""Text mesh loader/saver (mesh.load_mesh / save_mesh vs the reference loader's
golden output, tests/golden/make_golden_mesh.py), field dumps and step logs
(dumps.py)."""

import io
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from paper_1508_04245_b200 import dumps as D
from paper_1508_04245_b200 import fields as F
from paper_1508_04245_b200 import mesh as M

ATTRS = ("vertices", "triangles", "facet_vertices", "facet_elems", "facet_local", "facet_flip")


def test_load_mesh_matches_reference():
    g = load_golden("mesh_load.npz")
    m = M.load_mesh(os.path.join(GOLDEN, "meshes", "jitter3.txt"))
    for a in ATTRS:
        assert np.array_equal(np.asarray(getattr(m, a)), g[f"jitter3__{a}"]), a
    f = g["jitter3__label_facets"]
    assert sorted(m.facet_labels) == list(f)
    assert [m.facet_labels[i] for i in f] == list(g["jitter3__label_names"])


@pytest.mark.parametrize("name,text", [
    ("bad_header", "3 1\n0 0\n1 0\n0 1\n0 1 2\n"),
    ("bad_count", "3 1 0\n0 0\n1 0\n0 1\n"),
    ("bad_float", "3 1 0\n0 0\n1 x\n0 1\n0 1 2\n"),
    ("bad_index", "3 1 0\n0 0\n1 0\n0 1\n0 1 3\n"),
    ("bad_marker", "3 1 1\n0 0\n1 0\n0 1\n0 1 2\n0 1\n"),
    ("empty", "# nothing\n\n"),
])
def test_load_mesh_errors_match_reference(tmp_path, name, text):
    p = tmp_path / f"{name}.txt"
    p.write_text(text)
    with pytest.raises(M.MeshError) as ei:
        M.load_mesh(str(p))
    assert str(ei.value).replace(str(p), "<path>") == str(load_golden("mesh_load.npz")[f"err__{name}"])


def test_save_load_round_trip(tmp_path):
    m = M.generate_jittered(5, 0.2, seed=3)
    p = str(tmp_path / "m.txt")
    M.save_mesh(m, p)
    m2 = M.load_mesh(p)
    for a in ATTRS:
        assert np.array_equal(np.asarray(getattr(m, a)), np.asarray(getattr(m2, a))), a
    assert m.facet_labels == m2.facet_labels


def test_field_dump_piola_and_vdg_agree():
    # I is the exact embedding W_h -> V_h on affine elements, so the two dumps coincide
    m = M.generate_jittered(6, 0.2, seed=1)
    k = 3
    sf = F.StreamFunction(2, 2)
    u = F.interpolate_curl(m, k, sf)
    a, b = io.StringIO(), io.StringIO()
    D.dump_field(a, m, k, u, "Hdiv", n=4)
    D.dump_field(b, m, k, F.transfer_I_host(m, k, u), "VectorDG", n=4)
    ta = np.loadtxt(io.StringIO(a.getvalue()), delimiter=",", skiprows=1)
    tb = np.loadtxt(io.StringIO(b.getvalue()), delimiter=",", skiprows=1)
    assert a.getvalue().splitlines()[0] == "element,xi,eta,x,y,v0,v1"
    assert ta.shape == (m.n_elements * 15, 7)
    assert np.array_equal(ta[:, :5], tb[:, :5])
    assert np.abs(ta[:, 5:] - tb[:, 5:]).max() < 1e-12 * np.abs(ta[:, 5:]).max()
    # and approximate the exact velocity at the physical points
    ex = sf.velocity(ta[:, 3], ta[:, 4])
    assert np.abs(ta[:, 5:] - ex).max() < 0.05 * np.abs(ex).max()


def test_max_divergence_and_step_log(tmp_path):
    m = M.generate_structured((0, 0, 1, 1), 4, 4)
    u = F.interpolate_curl(m, 4, F.StreamFunction(4, 1))
    assert D.max_divergence(m, 4, u) < 1e-10 * np.abs(u).max() * 16
    log = D.StepLog(str(tmp_path / "steps.csv"))
    log.log(0.1, "oifs_euler", [1.5, 2.25], 0, 1e-14)
    log.log(0.2, "frac_theta", [1.0], 17, 2e-14)
    text = open(tmp_path / "steps.csv").read()
    assert text.replace("\r\n", "\n") == log.to_csv().replace("\r\n", "\n")
    assert text.splitlines()[0] == "t,scheme,stage_ms,richardson_iterations,max_divergence"
    assert "frac_theta,1,17" in text
