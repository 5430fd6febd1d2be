"""Global H(div) dof map (paper_1508_04245_b200/fespace.py) against the oracle
restatement of the SPEC numbering and the physical flux-moment definition."""

import numpy as np
import pytest

from oracle import fespace as OF
from paper_1508_04245_b200 import fespace as FS
from paper_1508_04245_b200 import fields as F
from paper_1508_04245_b200 import mesh as M


def test_spec_examples():
    # 2-triangle square, Hdiv(1) -> 5 facets x 2 = 10
    m = M.generate_structured((0, 0, 1, 1), 1, 1)
    assert FS.build_hdiv_dofmap(m, 1).ndof == 10
    for k in (1, 2, 4):
        m = M.generate_structured((0, 0, 1, 1), 4, 3)
        dm = FS.build_hdiv_dofmap(m, k)
        assert dm.ndof == m.n_facets * (k + 1) + m.n_elements * (k + 1) * (k - 1)


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_numbering_matches_oracle(k):
    m = M.generate_jittered(5, 0.2, seed=1)
    dm = FS.build_hdiv_dofmap(m, k)
    dofs, ndof = OF.numbering(m, k)
    assert ndof == dm.ndof and np.array_equal(dofs, dm.element_dofs)
    # every facet dof appears once (boundary) or twice (interior); interiors once
    cnt = np.bincount(dm.element_dofs.ravel(), minlength=dm.ndof)
    ne = k + 1
    assert np.array_equal(cnt[:m.n_facets * ne].reshape(-1, ne)[:, 0], np.where(m.facet_elems[:, 1] >= 0, 2, 1))
    assert np.all(cnt[m.n_facets * ne:] == 1)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_factors_reproduce_physical_flux_moments(k):
    # the global dof of the interpolated field equals int_F u.n_f L_m ds of the exact field
    m = M.generate_jittered(6, 0.2, seed=2)
    sf = F.StreamFunction(3, 4, wind=(0.7, -0.2))
    u = F.interpolate_curl(m, k, sf)
    dm = FS.build_hdiv_dofmap(m, k)
    g = FS.global_from_local(dm, u)
    mom = OF.flux_moments(m, k, sf.velocity, nq=24)
    gf = g[:dm.n_facet_dofs].reshape(-1, k + 1)
    # mode 0 is the exact flux psi(b) - psi(a) in the interpolant: tight; higher modes carry the
    # interpolant's quad_interval(2k+2) error on the sine field, far below an orientation/scale error
    assert np.abs(gf[:, 0] - mom[:, 0]).max() < 1e-12 * np.abs(mom).max()
    assert np.abs(gf - mom).max() < 2e-3 * np.abs(mom).max()
    # gather of the global vector reproduces the (conforming) element-local field
    assert np.abs(OF.gather(dm.element_dofs, dm.factors, g) - u).max() < 1e-12 * np.abs(u).max()


def test_scatter_is_the_adjoint_of_gather():
    k = 3
    m = M.generate_structured((0, 0, 1, 1), 5, 4)
    dm = FS.build_hdiv_dofmap(m, k)
    rng = np.random.default_rng(0)
    g, r = rng.standard_normal(dm.ndof), rng.standard_normal(dm.element_dofs.shape)
    lhs = np.sum(OF.scatter(dm.element_dofs, dm.factors, r, dm.ndof) * g)
    rhs = np.sum(r * OF.gather(dm.element_dofs, dm.factors, g))
    assert abs(lhs - rhs) < 1e-12 * np.abs(r).sum()
