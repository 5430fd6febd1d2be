"""GPU parity of the global H(div) gather / scatter / C^U assembly
(hdgc_set_dofmap, hdgc_gather, hdgc_scatter, hdgc_apply_u) against the oracle
(oracle/fespace.py + the oracle transfer/apply chain)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import convection as O  # noqa: E402
from oracle import fespace as OF  # noqa: E402
from paper_1508_04245_b200 import basis as B  # noqa: E402
from paper_1508_04245_b200 import fespace as FS  # noqa: E402
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200 import mesh3d as M3  # noqa: E402
from paper_1508_04245_b200.forms import (ConvectionData, ConvectionOperator, FESpace,  # noqa: E402
                                         apply_convection_U)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_gather_scatter_bit_exact(k):
    m = M.generate_jittered(9, 0.2, seed=k)
    dm = FS.build_hdiv_dofmap(m, k)
    op = ConvectionOperator(m, k)
    op.set_dofmap(dm)
    rng = np.random.default_rng(k)
    g = rng.standard_normal(dm.ndof)
    r = rng.standard_normal(dm.element_dofs.shape)
    assert np.array_equal(op.gather(dev(g)).cpu().numpy(), OF.gather(dm.element_dofs, dm.factors, g))
    assert np.array_equal(op.scatter(dev(r)).cpu().numpy(), OF.scatter(dm.element_dofs, dm.factors, r, dm.ndof))


@pytest.mark.parametrize("k", [2, 4])
def test_apply_u_vs_oracle_chain(k):
    m = M.generate_jittered(8, 0.2, seed=3)
    sf = F.StreamFunction(4, 2, wind=(1.0, 0.3))
    u_loc = F.interpolate_curl(m, k, sf)
    inflow = F.inflow_values(m, k, sf)
    sp = FESpace(m, "Hdiv", k)
    dm = sp.dofmap()
    u_glob = FS.global_from_local(dm, u_loc)
    r = apply_convection_U(dev(u_glob), sp, ConvectionData(dev(inflow))).cpu().numpy()
    assert r.shape == (sp.ndof,)
    op = ConvectionOperator(m, k)
    # composition: exactly scatter(apply_w(gather(u)))
    ul = OF.gather(dm.element_dofs, dm.factors, u_glob)
    rw = op.apply_w(dev(ul), dev(inflow)).cpu().numpy()
    assert np.array_equal(r, OF.scatter(dm.element_dofs, dm.factors, rw, dm.ndof))
    # oracle chain: I -> extended-precision flux-form C^V -> I^T -> scatter
    w = O.transfer_I(m, k, ul)
    rv = O.apply_convection_flux_form(m, k, ul, w, inflow).astype(float)
    ref = OF.scatter(dm.element_dofs, dm.factors, O.transfer_IT(m, k, rv), dm.ndof)
    cond = B.build_bdm_basis(k).cond
    assert np.linalg.norm(r - ref) / np.linalg.norm(ref) < 1e-12 * cond


def test_dofmap_errors():
    m = M.generate_structured((0, 0, 1, 1), 3, 3)
    op = ConvectionOperator(m, 2)
    dm = FS.build_hdiv_dofmap(m, 2)
    bad = dm.element_dofs.copy()
    bad[0, :3] = 0                                   # dof 0 used by more than two local dofs
    with pytest.raises(RuntimeError, match="more than two"):
        op.set_dofmap(FS.HdivDofMap(2, dm.ndof, dm.n_facet_dofs, bad, dm.factors))
    import ctypes as C
    from paper_1508_04245_b200 import _lib
    fresh = ConvectionOperator(m, 2)
    z = dev(np.zeros(dm.element_dofs.shape))
    rc = _lib.load().hdgc_scatter(fresh.handle, C.c_void_p(z.data_ptr()), C.c_void_p(z.data_ptr()), None)
    assert rc == -1 and b"no dof map" in _lib.load().hdgc_last_error()
    m3 = M3.generate_cube(2)
    op3 = ConvectionOperator(m3, 1)
    with pytest.raises(RuntimeError, match="2D"):
        op3.set_dofmap(FS.HdivDofMap(1, 4, 0, np.zeros((m3.n_elements, 12), dtype=np.int64),
                                     np.ones((m3.n_elements, 12))))
