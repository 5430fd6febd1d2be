"""Curved elements (MESH:381-443, 555-615),
host side and oracle, CPU only.

Pins: the ring mesh, its isoparametric maps and geometry_map against the
reference's own output (tests/golden/curved.npz, make_golden_curved.py), the
curved-mesh oracle against the affine oracle and against the operator's known
answers, and the device tables (block mass inverse, L2
projection) against the oracle."""
import os

import numpy as np
import pytest

from oracle import convection as O
from oracle import curved as OC
from paper_1508_04245_b200 import basis as B
from paper_1508_04245_b200 import fields as F
from paper_1508_04245_b200 import mesh as M
from paper_1508_04245_b200.curved import curved_tables

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "curved.npz"))
CIRCLE = M.Circle((0.5, 0.5), 0.15)


def ring(g, n_theta=16, n_layers=3):
    m = M.generate_ring(CIRCLE, (0.0, 0.0, 1.0, 1.0), n_theta, n_layers)
    return M.curve_boundary(m, "obstacle", CIRCLE, g)


@pytest.mark.parametrize("g", [2, 3])
def test_ring_and_curved_maps_match_reference(g):
    m = ring(g)
    for a in ("vertices", "triangles", "facet_vertices", "facet_elems", "facet_local", "facet_flip"):
        np.testing.assert_array_equal(getattr(m, a), GOLD[f"g{g}_{a}"], err_msg=a)
    np.testing.assert_array_equal(m.curved_elements(), GOLD[f"g{g}_curved_elems"])
    cm = np.stack([m.curved_maps[int(e)] for e in m.curved_elements()])
    np.testing.assert_allclose(cm, GOLD[f"g{g}_curved_coeffs"], rtol=0, atol=1e-13)
    x, J, det = m.geometry_batch(m.curved_elements(), GOLD["pts"])
    np.testing.assert_allclose(x, GOLD[f"g{g}_geo_x"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(J, GOLD[f"g{g}_geo_J"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(det, GOLD[f"g{g}_geo_det"], rtol=0, atol=1e-12)
    assert abs(m.total_area() - float(GOLD[f"g{g}_total_area"])) < 1e-13
    lab = {int(f): str(n) for f, n in zip(GOLD[f"g{g}_labels_f"], GOLD[f"g{g}_labels_n"])}
    assert m.facet_labels == lab


def test_curved_area_converges_to_annulus():
    exact = 1.0 - np.pi * 0.15 ** 2
    errs = [abs(ring(g, 32, 4).total_area() - exact) for g in (1, 2, 3)]
    assert errs[1] < errs[0] / 50 and errs[2] < errs[1]


def test_curve_boundary_errors():
    m = M.generate_ring(CIRCLE, (0.0, 0.0, 1.0, 1.0), 16, 3)
    with pytest.raises(M.MeshError):
        M.curve_boundary(m, "obstacle", CIRCLE, 0)
    with pytest.raises(M.MeshError):
        M.curve_boundary(m, "nothing", CIRCLE, 2)
    with pytest.raises(M.MeshError):
        M.curve_boundary(m, "obstacle", M.Circle((0.5, 0.5), 0.2), 2)
    with pytest.raises(M.MeshError):
        M.generate_ring(CIRCLE, (0.0, 0.0, 1.0, 1.0), 6, 2)       # outer segment spans a corner
    assert not M.curve_boundary(m, "obstacle", CIRCLE, 1).curved_maps


def test_interior_edges_of_curved_elements_are_affine():
    """the neighbour correspondence t' = 1 - t (MESH:201) still holds"""
    m = ring(3)
    t = np.linspace(0.0, 1.0, 7)
    for e in m.curved_elements():
        for loc in range(3):
            f = m.elem_facets[e, loc]
            if m.facet_elems[f, 1] < 0:
                continue
            x = m.geometry_batch([e], B.ref_edge_points(loc, t))[0][0]
            a, b = (m.vertices[m.triangles[e, v]] for v in B.REF_EDGES[loc])
            np.testing.assert_allclose(x, a + t[:, None] * (b - a), rtol=0, atol=1e-14)


def test_oracle_matches_affine_oracle_on_straight_ring():
    m = M.generate_ring(CIRCLE, (0.0, 0.0, 1.0, 1.0), 16, 3)
    sf = F.StreamFunction(4, 1, (1.0, 0.3))
    for k in (2, 4):
        u = F.interpolate_curl(m, k, sf)
        w = F.transfer_I_host(m, k, u)
        inf = F.inflow_values(m, k, sf)
        r0 = O.apply_convection(m, k, u, w, inf)
        r1 = OC.apply_convection(m, k, u, w, inf)
        assert np.linalg.norm(r1 - r0) / np.linalg.norm(r0) < 1e-13


@pytest.mark.parametrize("k", [2, 3])
def test_oracle_known_answers_on_curved_ring(k):
    """constants transported exactly and zero velocity
     on the curved mesh"""
    m = ring(3)
    sf = F.StreamFunction(4, 2, (1.0, 0.3))
    u = F.interpolate_curl(m, k, sf)
    nbs = B.nbs_of(k)
    d0 = B.dubiner_values(k, np.array([[0.2, 0.2]]))[0, 0]
    wc = np.zeros((m.n_elements, 2 * nbs))
    wc[:, 0], wc[:, nbs] = 1.0 / d0, -2.0 / d0
    inf = np.zeros((m.boundary_facets.size, B.facet_rule(k).points.size, 2))
    inf[..., 0], inf[..., 1] = 1.0, -2.0
    assert np.abs(OC.apply_convection(m, k, u, wc, inf)).max() < 1e-12
    w = np.random.default_rng(0).standard_normal(wc.shape)
    assert np.abs(OC.apply_convection(m, k, np.zeros_like(u), w)).max() == 0.0


def test_mass_blocks_and_tables():
    m = ring(3)
    k = 3
    Mb = OC.mass_blocks(m, k)
    ce = m.curved_elements()
    aff = np.setdiff1d(np.arange(m.n_elements), ce)
    nbs = B.nbs_of(k)
    np.testing.assert_allclose(Mb[aff], 0.5 * m.affine_det[aff, None, None] * np.eye(nbs), rtol=1e-13,
                               atol=1e-15)
    off = Mb[ce] - np.einsum("nii->ni", Mb[ce])[..., None] * np.eye(nbs)
    assert np.abs(off).max() > 1e-8                                  # genuinely non-diagonal blocks
    assert np.all(np.linalg.eigvalsh(Mb[ce]) > 0)
    tab = curved_tables(m, k)
    np.testing.assert_array_equal(tab["elems"], ce)
    np.testing.assert_allclose(tab["minv"], np.linalg.inv(Mb[ce]), rtol=1e-11, atol=1e-9)
    # I_T columns vs the oracle's projection of unit BDM vectors
    nb = 2 * nbs
    for j in range(0, nb, 5):
        e = np.zeros((m.n_elements, nb))
        e[:, j] = 1.0
        ref = OC.transfer_I(m, k, e)[ce]
        np.testing.assert_allclose(tab["itrans"][:, :, j], ref, rtol=0, atol=1e-11 * np.abs(ref).max())
    # area through the blocks: int detJ = M[0,0] / D0^2
    d0 = B.dubiner_values(k, np.array([[0.2, 0.2]]))[0, 0]
    assert abs(Mb[:, 0, 0].sum() / d0 ** 2 - m.total_area()) < 1e-12


def test_host_inputs_on_curved_mesh():
    m = ring(3)
    k = 4
    sf = F.StreamFunction(4, 3)
    u = F.interpolate_curl(m, k, sf)
    np.testing.assert_allclose(F.transfer_I_host(m, k, u), OC.transfer_I(m, k, u), rtol=0, atol=1e-12)
    # max speed: per-point Piola on curved elements vs a direct evaluation
    q = B.volume_rule(k)
    phi = B.build_bdm_basis(k).values(q.points)
    _, J, det = m.geometry_batch(np.arange(m.n_elements), q.points)
    uu = np.einsum("npcd,pjd,nj->npc", J, phi, u) / det[..., None]
    assert abs(F.max_speed_host(m, k, u) - np.sqrt((uu ** 2).sum(-1)).max()) < 1e-12


def test_oracle_reproduces_reference_fixture():
    """the committed curved goldens (oracle on the reference's mesh + polybasis)
    are reproduced with this package's mesh and basis"""
    m = ring(3)
    k = int(GOLD["k"])
    u, w, inf = GOLD["u"], GOLD["w"], GOLD["inflow"]
    r = OC.apply_convection(m, k, u, w, inf)
    assert np.linalg.norm(r - GOLD["r"]) / np.linalg.norm(GOLD["r"]) < 1e-13
    np.testing.assert_allclose(OC.transfer_I(m, k, u), w, rtol=0, atol=1e-12)
