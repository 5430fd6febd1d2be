"""GPU: the library's guards — norm-blowup flag, 16-byte pointer
alignment, and on-device mesh validation at hdgc_create (all through the C ABI)."""

import ctypes as C
import types

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1508_04245_b200 import _lib  # noqa: E402
from paper_1508_04245_b200 import basis as B  # noqa: E402
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import fields3d as F3  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200 import mesh3d as M3  # noqa: E402
from paper_1508_04245_b200 import timeloop as TL  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionData, ConvectionOperator, FEField, FESpace  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _field(n, k):
    m = M.generate_structured((0, 0, 1, 1), n, n)
    u = F.interpolate_curl(m, k, F.StreamFunction(4, 1))
    return m, u, F.transfer_I_host(m, k, u)


@pytest.mark.parametrize("k", [2, 4])
def test_blowup_flag_substeps_and_propagate(k):
    m, u, w = _field(8, k)
    op = ConvectionOperator(m, k)
    dt = F.cfl_dt(m.h_min(), k, F.max_speed_host(m, k, u))
    ud = dev(u)
    good = op.substeps(ud, dev(w), dt, 20)
    op.check_finite()                                     # stable: no flag
    assert torch.isfinite(good).all()
    bad = op.substeps(ud, dev(w), 1e4 * dt, 400)          # far beyond the CFL limit
    assert not torch.isfinite(bad).all()
    with pytest.raises(_lib.NormBlowupError, match="blow-up"):
        op.check_finite()
    op.check_finite()                                     # the check cleared the flag
    with pytest.raises(_lib.NormBlowupError):             # numpy path checks by itself
        op.substeps(u, w, 1e4 * dt, 400)
    sp = FESpace(m, "Hdiv", k)
    with pytest.raises(_lib.NormBlowupError):             # propagate_convection's guard
        TL.propagate_convection(dev(w), 0.0, 400 * 1e4 * dt, FEField(sp, ud), dt=1e4 * dt, scheme="ssprk2")
    v, nsub, _ = TL.propagate_convection(dev(w), 0.0, 10 * dt, FEField(sp, ud), dt=dt)
    assert nsub == 10 and torch.isfinite(v).all()
    # host end-to-end variant returns HDGC_EBLOWUP
    with pytest.raises(_lib.NormBlowupError):
        op.substeps_host(u, w, 1e4 * dt, 400)


def test_blowup_flag_3d_and_richardson():
    m = M3.generate_cube(3)
    k = 2
    u = F3.interpolate_curl3(m, k, F3.VectorPotential(2, 1))
    op = ConvectionOperator(m, k)
    w = op.transfer(dev(u))
    dt = 0.1 * m.h_min() / (k * k * op.max_speed(dev(u)))
    bad = op.substeps(dev(u), w.clone(), 1e4 * dt, 300)
    assert not torch.isfinite(bad).all()
    with pytest.raises(_lib.NormBlowupError):
        op.check_finite()
    g = w.clone()
    g[0, 0] = float("nan")
    with pytest.raises(_lib.NormBlowupError, match="non-finite residual"):
        op.richardson(dev(u), g, torch.zeros_like(g), 1e-3, 0.5)
    op.check_finite()


def test_misaligned_pointers():
    m, u, w = _field(4, 4)
    op = ConvectionOperator(m, 4)
    ref = op.apply(dev(u), dev(w))
    n = u.size
    buf = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    wv = buf[1:].view(u.shape)                 # contiguous, 8-byte aligned only
    wv.copy_(dev(w))
    assert wv.data_ptr() % 16 == 8
    assert torch.equal(op.apply(dev(u), wv), ref)          # forms clones it to an aligned copy
    lib = _lib.load()
    r = torch.empty_like(ref)
    rc = lib.hdgc_apply_v(op.handle, C.c_void_p(dev(u).data_ptr()), C.c_void_p(wv.data_ptr()), None,
                          C.c_void_p(r.data_ptr()), None)
    assert rc == -1 and b"16-byte" in lib.hdgc_last_error()
    rc = lib.hdgc_substeps(op.handle, C.c_void_p(dev(u).data_ptr()), C.c_void_p(wv.data_ptr()), None,
                           C.c_double(1e-6), 3, None)
    assert rc == -1
    with pytest.raises(ValueError, match="aligned"):
        op.substeps(dev(u), wv, 1e-6, 2)


def _copy2d(m, **kw):
    d = dict(vertices=m.vertices.copy(), triangles=m.triangles.copy(), facet_elems=m.facet_elems.copy(),
             facet_local=m.facet_local.copy(), n_elements=m.n_elements, n_facets=m.n_facets)
    d.update(kw)
    d["n_facets"] = len(d["facet_elems"])
    return types.SimpleNamespace(**d)


def _create_error(mesh, k=2):
    with pytest.raises(RuntimeError) as ei:
        ConvectionOperator(mesh, k)
    assert "status -1" in str(ei.value)
    return str(ei.value)


def test_mesh_validation_2d():
    m = M.generate_structured((0, 0, 1, 1), 3, 3)
    ConvectionOperator(_copy2d(m), 2)                                    # the copy itself is fine
    fe = m.facet_elems.copy()
    i = int(np.nonzero(fe[:, 1] >= 0)[0][0])
    fe[i, 1] = m.n_elements + 5
    assert "out of range" in _create_error(_copy2d(m, facet_elems=fe))
    fe = np.concatenate([m.facet_elems, m.facet_elems[:1]])
    fl = np.concatenate([m.facet_local, m.facet_local[:1]])
    assert "more than one" in _create_error(_copy2d(m, facet_elems=fe, facet_local=fl))
    assert "missing" in _create_error(_copy2d(m, facet_elems=m.facet_elems[1:], facet_local=m.facet_local[1:]))
    tri = m.triangles.copy()
    tri[3, 1] = len(m.vertices) + 2
    assert "vertex id" in _create_error(_copy2d(m, triangles=tri))
    tri = m.triangles.copy()
    tri[0] = tri[0, ::-1]                                                # clockwise
    assert "detJ" in _create_error(_copy2d(m, triangles=tri))


def test_mesh_validation_3d():
    m = M3.generate_cube(2)
    tets = m.tets.copy()
    tets[0, [1, 2]] = tets[0, [2, 1]]                                     # unsorted vertex ids
    bad = types.SimpleNamespace(vertices=m.vertices, tets=tets, triangles=tets, facet_elems=m.facet_elems,
                                facet_local=m.facet_local, n_elements=m.n_elements, n_facets=m.n_facets)
    assert "ascending" in _create_error(bad)


@pytest.mark.parametrize("dim,k", [(2, 2), (2, 4), (2, 7), (3, 3)])
def test_create_k_builtin_tables_bitwise(dim, k):
    """hdgc_create_k(mesh, k) — the library's build-time tables, what a
    non-Python caller uses — gives bitwise the results of hdgc_create with the
    tables passed from Python."""
    if dim == 2:
        m, u, w = _field(8, k)
        inf = None
    else:
        m = M3.generate_cube(3)
        vp = F3.VectorPotential(3, 5, (0.3, 0.2, -0.5))
        u = F3.interpolate_curl3(m, k, vp)
        w = F3.transfer_I3_host(m, k, u)
        inf = dev(F3.inflow_values3(m, k, vp))
    a = ConvectionOperator(m, k)
    b = ConvectionOperator(m, k, builtin_tables=True)
    assert torch.equal(a.apply(dev(u), dev(w), inf), b.apply(dev(u), dev(w), inf))
    assert torch.equal(a.substeps(dev(u), dev(w), 1e-4, 5, inf), b.substeps(dev(u), dev(w), 1e-4, 5, inf))


def test_create_k_unsupported_order():
    m = M.generate_structured((0, 0, 1, 1), 2, 2)
    with pytest.raises(RuntimeError, match="status -4"):
        ConvectionOperator(m, 9, builtin_tables=True)
