"""Host mesh + synthetic field construction vs the reference (CPU)."""

import numpy as np
import pytest

from conftest import load_golden
from paper_1508_04245_b200 import basis as B
from paper_1508_04245_b200 import fields as F
from paper_1508_04245_b200 import mesh as M

GM = load_golden("meshes.npz")
ARRAYS = ("vertices", "triangles", "facet_vertices", "facet_elems", "facet_local", "facet_flip",
          "elem_facets", "affine_det")


def test_structured_matches_reference_mesh2d():
    m = M.generate_structured((0.0, 0.0, 2.0, 1.0), 6, 5)
    for a in ARRAYS:
        assert np.array_equal(getattr(m, a), GM[f"rect_{a}"]), a


def test_build_matches_reference_on_jittered():
    m = M.build_mesh(GM["jit_vertices"], GM["jit_triangles"])
    for a in ARRAYS:
        assert np.array_equal(getattr(m, a), GM[f"jit_{a}"]), a


def test_orientation_fixed_and_interior_facets_reversed():
    # clockwise input triangles are reoriented (MESH:168-176); interior facets
    # are always traversed backwards by the neighbour (MESH:201)
    verts, tris = M._structured_arrays(4, 3)
    tris = tris[:, [0, 2, 1]]
    m = M.build_mesh(verts, tris)
    assert (m.affine_det > 0).all()
    assert m.facet_flip[m.interior_facets, 1].all()


def test_mesh_errors():
    with pytest.raises(M.MeshError):
        M.build_mesh(np.array([[0, 0], [1, 0], [2, 0]], float), np.array([[0, 1, 2]]))
    with pytest.raises(M.MeshError):
        M.generate_structured((0, 0, 1, 1), 0, 3)
    # an edge shared by three triangles
    v = np.array([[0, 0], [1, 0], [0, 1], [0, -1], [1, 1]], float)
    with pytest.raises(M.MeshError):
        M.build_mesh(v, np.array([[0, 1, 2], [0, 3, 1], [0, 1, 4]]))


def test_neighbour_tables():
    m = M.generate_structured((0, 0, 1, 1), 5, 4)
    nbr, ne, bs = m.element_neighbours()
    T, e = np.nonzero(nbr >= 0)
    assert np.array_equal(nbr[nbr[T, e], ne[T, e]], T)
    assert np.array_equal(ne[nbr[T, e], ne[T, e]], e)
    assert sorted(bs[bs >= 0].tolist()) == list(range(m.boundary_facets.size))


def test_jittered_mesh_valid_and_covers_square():
    m = M.generate_jittered(32, 0.2, seed=3)
    assert (m.affine_det > 0).all()
    assert abs(m.total_area() - 1.0) < 1e-12


@pytest.mark.parametrize("k", [1, 2, 4, 6, 8])
def test_interpolant_divergence_free_and_conforming(k):
    m = M.generate_jittered(8, 0.2, seed=1)
    u = F.interpolate_curl(m, k, F.StreamFunction(4, 7, (1.0, 0.3)))
    b = B.build_bdm_basis(k)
    q = B.quad_triangle(2 * k)
    div = np.einsum("pj,nj->np", b.divergence(q.points), u) / m.affine_det[:, None]
    scale = np.abs(u).max() / m.h_min()
    assert np.abs(div).max() < 1e-13 * scale * k * k       # exact recipe
    # element-local H(div) conformity
    nbr, ne, _ = m.element_neighbours()
    ce = u[:, :3 * (k + 1)].reshape(-1, 3, k + 1) * B.REF_EDGE_LENGTHS[None, :, None]
    T, e = np.nonzero(nbr >= 0)
    sgn = (-1.0) ** (np.arange(k + 1) + 1)
    assert np.abs(ce[T, e] - sgn * ce[nbr[T, e], ne[T, e]]).max() < 1e-13 * np.abs(ce).max()


def test_interpolant_reproduces_field():
    m = M.generate_structured((0, 0, 1, 1), 16, 16)
    k = 4
    sf = F.StreamFunction(3, 2)
    u = F.interpolate_curl(m, k, sf)
    w = F.transfer_I_host(m, k, u)
    q = B.quad_triangle(2 * k)
    D = B.dubiner_values(k, q.points)
    x = m.affine_origin[:, None, :] + np.einsum("ncd,pd->npc", m.affine_jac, q.points)
    exact = sf.velocity(x[..., 0], x[..., 1])
    approx = np.einsum("pm,ncm->npc", D, w.reshape(-1, 2, B.nbs_of(k)))
    assert np.abs(approx - exact).max() < 1e-3 * np.abs(exact).max()


def test_inflow_layout_and_cfl():
    m = M.generate_structured((0, 0, 1, 1), 4, 4)
    sf = F.StreamFunction(2, 0, (1.0, 0.3))
    inf = F.inflow_values(m, 3, sf)
    assert inf.shape == (m.boundary_facets.size, B.facet_rule(3).weights.size, 2)
    assert F.cfl_dt(0.1, 2, 1.0) == pytest.approx(0.0025)
    assert F.cfl_dt(0.1, 2, 0.0) == float("inf")
