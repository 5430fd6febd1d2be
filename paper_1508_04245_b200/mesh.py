"""Affine triangle meshes for the convection path (host side).

A from-scratch, vectorised restatement of the parts of the reference module
``hdgflow.mesh2d`` (``/root/reference/pkg/src/hdgflow/mesh2d.py``) that the
convection apply consumes, with the reference's attribute names and
conventions so a reference ``Mesh`` and a ``TriMesh`` are interchangeable
for every consumer in this package:

* triangles counter-clockwise (orientation fixed on build)   (MESH:168-176)
* facets keyed by the sorted vertex pair, numbered in sorted key order; the
  lowest element index owns the facet; the facet is stored in the owner's
  traversal direction; ``facet_flip[f, 1]`` marks a neighbour that traverses
  it the other way                                            (MESH:178-207)
* facet normal = tangent rotated by -90 degrees (outward for the owner)
                                                              (MESH:111-120)
* ``elem_facets``/``elem_flip``, affine ``J`` (columns = edges), ``detJ``,
  ``J^-1`` and origin                                          (MESH:122-150)
* ``generate_structured``: 2 nx ny triangles, diagonals lower-left to
  upper-right, ``(a, b, c), (a, c, d)`` per cell              (MESH:341-378)

The reference builds facets with Python dictionaries (21.5 s at 524k
triangles); this module sorts packed int64 edge keys instead
(well under a second), producing identical arrays.
"""

from __future__ import annotations

import numpy as np

from dataclasses import dataclass

from .basis import REF_EDGES, REF_VERTICES, quad_triangle

__all__ = ["MeshError", "TriMesh", "Circle", "build_mesh", "generate_structured", "generate_jittered",
           "generate_ring", "curve_boundary", "geometry_map", "load_mesh", "save_mesh"]


class MeshError(Exception):
    """Invalid mesh topology or geometry (MESH:18-19)."""


@dataclass(frozen=True)
class Circle:
    """Circular boundary geometry for curved facets (MESH:23-27)."""

    center: tuple
    radius: float


def lattice(g: int):
    """Principal lattice exponents/nodes of a degree-g triangle, (i, j) with
    j outer, i inner — the ordering of the curved-map monomial fit (MESH:48-50)."""
    return [(i, j) for j in range(g + 1) for i in range(g + 1 - j)]


def _monomials(exps, pts, deriv=False):
    """x^i y^j at pts (n, 2) -> (n, nm); with deriv also d/dx, d/dy -> (n, nm, 2)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    e = np.asarray(exps, dtype=np.int64).reshape(-1, 2)
    x, y = pts[:, :1], pts[:, 1:2]
    ei, ej = e[None, :, 0], e[None, :, 1]
    val = x ** ei * y ** ej
    if not deriv:
        return val
    gx = np.where(ei > 0, ei * x ** np.maximum(ei - 1, 0) * y ** ej, 0.0)
    gy = np.where(ej > 0, ej * x ** ei * y ** np.maximum(ej - 1, 0), 0.0)
    return val, np.stack([gx, gy], axis=-1)


class TriMesh:
    """Immutable triangulation with oriented facets: affine elements, plus
    optional degree-g isoparametric maps on the elements along curved
    boundary labels (``curved_maps``, MESH:94-150, 555-615)."""

    def __init__(self, vertices, triangles, facet_vertices, facet_elems, facet_local,
                 facet_flip, facet_labels=None, geometry_order=1, curved_maps=None, curved_geometry=None):
        self.vertices = np.ascontiguousarray(vertices, dtype=float)
        self.triangles = np.ascontiguousarray(triangles, dtype=np.int64)
        self.facet_vertices = np.ascontiguousarray(facet_vertices, dtype=np.int64)
        self.facet_elems = np.ascontiguousarray(facet_elems, dtype=np.int64)
        self.facet_local = np.ascontiguousarray(facet_local, dtype=np.int64)
        self.facet_flip = np.ascontiguousarray(facet_flip, dtype=bool)
        self.facet_labels = dict(facet_labels or {})
        self.geometry_order = int(geometry_order)
        self.curved_maps = dict(curved_maps or {})            # elem -> (2, n_mono) monomial coefficients
        self.curved_geometry = dict(curved_geometry or {})    # label -> Circle
        self.n_elements = len(self.triangles)
        self.n_facets = len(self.facet_vertices)

        a = self.vertices[self.facet_vertices[:, 0]]
        b = self.vertices[self.facet_vertices[:, 1]]
        tang = b - a
        self.facet_h = np.hypot(tang[:, 0], tang[:, 1])
        if np.any(self.facet_h <= 0):
            raise MeshError("degenerate facet")
        self.facet_tangent = tang / self.facet_h[:, None]
        self.facet_normal = np.stack([self.facet_tangent[:, 1], -self.facet_tangent[:, 0]], axis=1)

        self.elem_facets = np.full((self.n_elements, 3), -1, dtype=np.int64)
        self.elem_flip = np.zeros((self.n_elements, 3), dtype=bool)
        for side in range(2):
            sel = self.facet_elems[:, side] >= 0
            e = self.facet_elems[sel, side]
            loc = self.facet_local[sel, side]
            self.elem_facets[e, loc] = np.nonzero(sel)[0]
            self.elem_flip[e, loc] = self.facet_flip[sel, side]
        if (self.elem_facets < 0).any():
            raise MeshError("element with unmatched facet")

        v0, v1, v2 = (self.vertices[self.triangles[:, i]] for i in range(3))
        J = np.stack([v1 - v0, v2 - v0], axis=2)
        self.affine_jac = J
        self.affine_det = J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0]
        if np.any(self.affine_det <= 0):
            raise MeshError("inverted or degenerate element")
        self.affine_origin = v0
        inv = np.empty_like(J)
        inv[:, 0, 0] = J[:, 1, 1]
        inv[:, 0, 1] = -J[:, 0, 1]
        inv[:, 1, 0] = -J[:, 1, 0]
        inv[:, 1, 1] = J[:, 0, 0]
        self.affine_inv = inv / self.affine_det[:, None, None]

    # -- queries (reference names) -------------------------------------------

    @property
    def interior_facets(self):
        return np.nonzero(self.facet_elems[:, 1] >= 0)[0]

    @property
    def boundary_facets(self):
        return np.nonzero(self.facet_elems[:, 1] < 0)[0]

    def h_min(self) -> float:
        """Smallest facet length (MESH:290-291)."""
        return float(self.facet_h.min())

    def total_area(self) -> float:
        area = float(0.5 * self.affine_det.sum())
        if self.curved_maps:
            ce = self.curved_elements()
            q = quad_triangle(max(2 * self.geometry_order, 2))
            _, _, det = self.geometry_batch(ce, q.points)
            area += float((det @ q.weights).sum() - 0.5 * self.affine_det[ce].sum())
        return area

    def is_curved(self, elem) -> bool:
        return int(elem) in self.curved_maps

    def curved_elements(self) -> np.ndarray:
        """Sorted ids of the elements carrying a curved map."""
        return np.array(sorted(self.curved_maps), dtype=np.int64)

    def curved_facets(self) -> np.ndarray:
        """Facets on a curved boundary label (MESH:246-252)."""
        return np.array(sorted(f for f, lab in self.facet_labels.items() if lab in self.curved_geometry),
                        dtype=np.int64)

    def facets_with_label(self, label) -> np.ndarray:
        return np.array(sorted(f for f, lab in self.facet_labels.items() if lab == label), dtype=np.int64)

    def geometry_batch(self, elems, ref_pts):
        """x (n, p, 2), J (n, p, 2, 2) and detJ (n, p) of the elements ``elems``
        at the reference points: the curved map where one is attached, the
        affine map otherwise (vectorised MESH:254-278)."""
        elems = np.asarray(elems, dtype=np.int64).reshape(-1)
        pts = np.atleast_2d(np.asarray(ref_pts, dtype=float))
        n, p = elems.size, pts.shape[0]
        J = np.broadcast_to(self.affine_jac[elems][:, None], (n, p, 2, 2)).copy()
        x = self.affine_origin[elems][:, None, :] + np.einsum("ncd,pd->npc", self.affine_jac[elems], pts)
        cur = np.array([int(e) in self.curved_maps for e in elems], dtype=bool)
        if cur.any():
            val, grad = _monomials(lattice(self.geometry_order), pts, deriv=True)
            cm = np.stack([self.curved_maps[int(e)] for e in elems[cur]])      # (nc, 2, nm)
            x[cur] = np.einsum("ncm,pm->npc", cm, val)
            J[cur] = np.einsum("ncm,pmd->npcd", cm, grad)
        det = J[..., 0, 0] * J[..., 1, 1] - J[..., 0, 1] * J[..., 1, 0]
        return x, J, det

    def geometry_map(self, elem, ref_pts):
        """(x, J, detJ) of one element at reference points, shapes (n,2),
        (n,2,2), (n,) — the reference's ``Mesh.geometry_map`` (MESH:254-278)."""
        x, J, det = self.geometry_batch([elem], ref_pts)
        return x[0], J[0], det[0]

    # -- adjacency views used by the device context --------------------------

    def element_neighbours(self):
        """(nbr, nbr_edge, bnd_slot), each (NT, 3) int64.

        nbr[T, e] is the element across local edge e (-1 on the boundary),
        nbr_edge[T, e] its local edge index, bnd_slot[T, e] the position of
        the facet in ``boundary_facets`` order (-1 for interior facets) —
        the row of the inflow array ``(NBF, nf, 2)``.
        """
        NT = self.n_elements
        nbr = np.full((NT, 3), -1, dtype=np.int64)
        nbr_edge = np.full((NT, 3), -1, dtype=np.int64)
        bnd = np.full((NT, 3), -1, dtype=np.int64)
        fe, fl = self.facet_elems, self.facet_local
        inner = fe[:, 1] >= 0
        for s, o in ((0, 1), (1, 0)):
            nbr[fe[inner, s], fl[inner, s]] = fe[inner, o]
            nbr_edge[fe[inner, s], fl[inner, s]] = fl[inner, o]
        bf = np.nonzero(~inner)[0]
        bnd[fe[bf, 0], fl[bf, 0]] = np.arange(bf.size)
        return nbr, nbr_edge, bnd


def build_mesh(vertices, triangles, boundary_markers=None) -> TriMesh:
    """Assemble a TriMesh from raw arrays (restates Mesh.build, MESH:155-216)."""
    vertices = np.asarray(vertices, dtype=float)
    tri = np.array(triangles, dtype=np.int64, copy=True)
    NT = len(tri)
    # counter-clockwise orientation
    p0, p1, p2 = (vertices[tri[:, i]] for i in range(3))
    det = (p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1]) - (p1[:, 1] - p0[:, 1]) * (p2[:, 0] - p0[:, 0])
    if np.any(det == 0):
        raise MeshError(f"triangle {int(np.nonzero(det == 0)[0][0])} is degenerate")
    flip = det < 0
    tri[flip, 1], tri[flip, 2] = tri[flip, 2].copy(), tri[flip, 1].copy()

    # element edges in (element, local edge) order
    la = np.array([e[0] for e in REF_EDGES])
    lb = np.array([e[1] for e in REF_EDGES])
    ea = tri[:, la].ravel()               # start vertex, index = 3*t + loc
    eb = tri[:, lb].ravel()
    lo = np.minimum(ea, eb)
    hi = np.maximum(ea, eb)
    nv = max(int(vertices.shape[0]), 1)
    key = lo * nv + hi
    order = np.argsort(key, kind="stable")   # ties keep (element, local) order
    ks = key[order]
    start = np.ones(ks.size, dtype=bool)
    start[1:] = ks[1:] != ks[:-1]
    gid = np.cumsum(start) - 1
    counts = np.bincount(gid)
    if counts.max() > 2:
        bad = int(np.nonzero(counts > 2)[0][0])
        k0 = ks[np.nonzero(gid == bad)[0][0]]
        raise MeshError(f"facet {(int(k0 // nv), int(k0 % nv))} shared by {counts[bad]} elements")
    NF = counts.size
    first = np.nonzero(start)[0]
    o0 = order[first]                    # owner: lowest element (stable sort)
    t0, l0 = o0 // 3, o0 % 3
    facet_vertices = np.stack([ea[o0], eb[o0]], axis=1)
    facet_elems = np.full((NF, 2), -1, dtype=np.int64)
    facet_local = np.full((NF, 2), -1, dtype=np.int64)
    facet_flip = np.zeros((NF, 2), dtype=bool)
    facet_elems[:, 0] = t0
    facet_local[:, 0] = l0
    two = counts == 2
    o1 = order[first[two] + 1]
    facet_elems[two, 1] = o1 // 3
    facet_local[two, 1] = o1 % 3
    facet_flip[two, 1] = ea[o1] != ea[o0[two]]

    labels = {}
    if boundary_markers:
        fkey = {int(k): f for f, k in zip(np.nonzero(~two)[0], ks[first[~two]])}
        for pair, lab in boundary_markers.items():
            a, b = sorted(pair)
            f = fkey.get(int(a) * nv + int(b))
            if f is None:
                raise MeshError(f"boundary markers on non-boundary edges: {[(a, b)]}")
            labels[f] = lab
    return TriMesh(vertices, tri, facet_vertices, facet_elems, facet_local, facet_flip, labels)


def _structured_arrays(nx, ny, rect=(0.0, 0.0, 1.0, 1.0)):
    x0, y0, x1, y1 = rect
    xs = np.linspace(x0, x1, nx + 1)
    ys = np.linspace(y0, y1, ny + 1)
    X, Y = np.meshgrid(xs, ys)            # vertex id = j*(nx+1) + i
    verts = np.stack([X.ravel(), Y.ravel()], axis=1)
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    a = (j * (nx + 1) + i).ravel()
    b = a + 1
    c = a + nx + 2
    d = a + nx + 1
    tris = np.empty((2 * nx * ny, 3), dtype=np.int64)
    tris[0::2] = np.stack([a, b, c], axis=1)
    tris[1::2] = np.stack([a, c, d], axis=1)
    return verts, tris


def _structured_markers(nx, ny, labels):
    left, right, bottom, top = labels
    vid = lambda i, j: j * (nx + 1) + i
    m = {}
    for j in range(ny):
        m[(vid(0, j), vid(0, j + 1))] = left
        m[(vid(nx, j), vid(nx, j + 1))] = right
    for i in range(nx):
        m[(vid(i, 0), vid(i + 1, 0))] = bottom
        m[(vid(i, ny), vid(i + 1, ny))] = top
    return m


def generate_structured(rect, nx, ny, labels=("left", "right", "bottom", "top")) -> TriMesh:
    """Structured triangulation of a rectangle (MESH:341-378)."""
    x0, y0, x1, y1 = rect
    if nx < 1 or ny < 1 or x1 <= x0 or y1 <= y0:
        raise MeshError("degenerate rectangle or nonpositive subdivision")
    verts, tris = _structured_arrays(nx, ny, rect)
    return build_mesh(verts, tris, _structured_markers(nx, ny, labels))


def generate_jittered(n, amplitude=0.2, seed=0, labels=("left", "right", "bottom", "top")) -> TriMesh:
    """Unit square, n x n cells, interior vertices moved by U(-a h, a h) per
    coordinate with h = 1/n (BASELINE cfg3), built through ``build_mesh``."""
    verts, tris = _structured_arrays(n, n)
    h = 1.0 / n
    rng = np.random.default_rng(seed)
    jit = rng.uniform(-amplitude * h, amplitude * h, size=verts.shape)
    ii = np.arange(verts.shape[0])
    vi, vj = ii % (n + 1), ii // (n + 1)
    interior = (vi > 0) & (vi < n) & (vj > 0) & (vj < n)
    verts = verts.copy()
    verts[interior] += jit[interior]
    return build_mesh(verts, tris, _structured_markers(n, n, labels))


def geometry_map(mesh, elem, ref_pts):
    """Module-level alias of ``TriMesh.geometry_map`` (MESH:638-640)."""
    return mesh.geometry_map(elem, ref_pts)


def generate_ring(circle: Circle, rect, n_theta, n_layers, theta_offset=0.0, radial_fractions=None,
                  inner_label="obstacle", outer_labels=("left", "right", "bottom", "top")) -> TriMesh:
    """O-grid between a circle and an enclosing rectangle, 2 n_theta n_layers
    triangles (restates MESH:381-443): ray i at angle theta_offset + 2 pi i /
    n_theta runs from the circle to the rectangle, layer s at radial fraction
    s; cell (i, j) -> triangles (a, b, c), (a, c, d).  Inner chords carry
    ``inner_label`` (curve them with ``curve_boundary``); each outer segment
    must lie on one rectangle side."""
    (cx, cy), r = circle.center, circle.radius
    x0, y0, x1, y1 = rect
    th = theta_offset + 2.0 * np.pi * np.arange(n_theta) / n_theta
    d = np.stack([np.cos(th), np.sin(th)], axis=1)
    # distance along each ray to the rectangle: smallest positive hit
    with np.errstate(divide="ignore", invalid="ignore"):
        tx = np.where(d[:, 0] > 1e-14, (x1 - cx) / d[:, 0], np.where(d[:, 0] < -1e-14, (x0 - cx) / d[:, 0], np.inf))
        ty = np.where(d[:, 1] > 1e-14, (y1 - cy) / d[:, 1], np.where(d[:, 1] < -1e-14, (y0 - cy) / d[:, 1], np.inf))
    hit = np.minimum(np.where(tx > 0, tx, np.inf), np.where(ty > 0, ty, np.inf))
    c = np.array([cx, cy])
    inner = c + r * d
    outer = c + hit[:, None] * d
    fr = np.linspace(0.0, 1.0, n_layers + 1) if radial_fractions is None else np.asarray(radial_fractions, float)
    verts = np.concatenate([inner * (1.0 - s) + outer * s for s in fr], axis=0)
    vid = lambda i, j: j * n_theta + (i % n_theta)
    tris = []
    for j in range(n_layers):
        for i in range(n_theta):
            a, b, cc, dd = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            tris += [(a, b, cc), (a, cc, dd)]
    markers = {tuple(sorted((vid(i, 0), vid(i + 1, 0)))): inner_label for i in range(n_theta)}
    left, right, bottom, top = outer_labels
    tol = 1e-10 * max(x1 - x0, y1 - y0)
    for i in range(n_theta):
        a, b = vid(i, n_layers), vid(i + 1, n_layers)
        pa, pb = verts[a], verts[b]
        for lab, ax, val in ((left, 0, x0), (right, 0, x1), (bottom, 1, y0), (top, 1, y1)):
            if abs(pa[ax] - val) < tol and abs(pb[ax] - val) < tol:
                markers[tuple(sorted((a, b)))] = lab
                break
        else:
            raise MeshError("outer ring segment spans a rectangle corner; "
                            "choose theta_offset/n_theta so rays hit corners")
    return build_mesh(verts, np.array(tris, dtype=np.int64), markers)


def _on_edge(ea, eb, pt, tol=1e-12):
    """Parameter s in [0, 1] of pt on the segment ea -> eb, or None."""
    d, w = eb - ea, pt - ea
    if abs(d[0] * w[1] - d[1] * w[0]) > tol:
        return None
    s = float(np.dot(w, d) / np.dot(d, d))
    return min(max(s, 0.0), 1.0) if -tol <= s <= 1.0 + tol else None


def curve_boundary(mesh: TriMesh, label, geometry: Circle, g: int) -> TriMesh:
    """Attach degree-g isoparametric maps to the owners of the ``label``
    facets (restates MESH:555-615): the degree-g lattice of each owner is
    placed at its affine position, the nodes on the labelled edge are moved
    onto the circle at equal angle steps between the edge's end points, and
    the map x(x_hat) = sum_m c_m x_hat^i y_hat^j interpolates the nodes.
    Interior edges keep their affine lattice nodes, so they stay straight
    and are parametrised exactly as in the neighbour's affine map."""
    if g < 1:
        raise MeshError("geometry order must be >= 1")
    if not isinstance(geometry, Circle):
        raise MeshError("only circular boundary geometry is supported")
    facets = mesh.facets_with_label(label)
    if facets.size == 0:
        raise MeshError(f"no facets labeled {label!r}")
    c = np.asarray(geometry.center, dtype=float)
    r = float(geometry.radius)
    for f in facets:
        for v in mesh.facet_vertices[f]:
            if abs(np.linalg.norm(mesh.vertices[v] - c) - r) > 1e-8 * r:
                raise MeshError(f"facet {f} endpoint not on the circle")
    geom = dict(mesh.curved_geometry)
    geom[label] = geometry

    def rebuild(order, maps):
        return TriMesh(mesh.vertices, mesh.triangles, mesh.facet_vertices, mesh.facet_elems, mesh.facet_local,
                       mesh.facet_flip, mesh.facet_labels, geometry_order=order, curved_maps=maps,
                       curved_geometry=geom)

    if g == 1:
        return rebuild(1, {})
    exps = lattice(g)
    nodes = np.array([(i / g, j / g) for i, j in exps])
    V = _monomials(exps, nodes)
    owned = {}
    for f in facets:
        owned.setdefault(int(mesh.facet_elems[f, 0]), []).append(int(f))
    maps = dict(mesh.curved_maps)
    for e, fl in owned.items():
        corners = mesh.vertices[mesh.triangles[e]]
        phys = corners[0] + nodes @ np.stack([corners[1] - corners[0], corners[2] - corners[0]])
        for f in fl:
            loc = int(np.nonzero(mesh.elem_facets[e] == f)[0][0])
            la, lb = REF_EDGES[loc]
            ta = np.arctan2(*(corners[la] - c)[::-1])
            tb = np.arctan2(*(corners[lb] - c)[::-1])
            dth = (tb - ta + np.pi) % (2.0 * np.pi) - np.pi      # short arc
            for m, pt in enumerate(nodes):
                s = _on_edge(REF_VERTICES[la], REF_VERTICES[lb], pt)
                if s is not None:
                    phys[m] = c + r * np.array([np.cos(ta + s * dth), np.sin(ta + s * dth)])
        maps[e] = np.linalg.solve(V, phys).T.copy()               # (2, n_mono)
    out = rebuild(g, maps)
    q = quad_triangle(max(4, 2 * g + 2))
    _, _, det = out.geometry_batch(out.curved_elements(), q.points)
    if np.any(det <= 0):
        raise MeshError(f"curved element {int(out.curved_elements()[np.nonzero((det <= 0).any(1))[0][0]])} "
                        "has nonpositive Jacobian")
    return out


# ---------------------------------------------------------------------------
# text mesh format (mesh2d.load_mesh, MESH:298-334): header "NV NT NBF", then NV
# "x y" lines, NT "v0 v1 v2" lines, NBF "v0 v1 label" lines; '#' starts a comment.


def load_mesh(path) -> TriMesh:
    """Read the reference's text mesh format; MeshError("<path>:<line>: ...")
    on malformed input, as the reference loader reports it."""
    data = []
    with open(path) as fh:
        for no, raw in enumerate(fh, 1):
            body = raw.partition("#")[0].split()
            if body:
                data.append((no, body))
    if not data:
        raise MeshError(f"{path}: empty mesh file")

    def fields(entry, conv, expect):
        no, tok = entry
        if len(tok) != len(conv):
            raise MeshError(f"{path}:{no}: expected {expect}")
        try:
            return [c(t) for c, t in zip(conv, tok)]
        except ValueError as err:
            raise MeshError(f"{path}:{no}: {err}") from None

    nv, nt, nbf = fields(data[0], (int, int, int), "NV NT NBF header")
    if len(data) != 1 + nv + nt + nbf:
        raise MeshError(f"{path}: expected {1 + nv + nt + nbf} data lines, got {len(data)}")
    vsec, tsec, bsec = data[1:1 + nv], data[1 + nv:1 + nv + nt], data[1 + nv + nt:]
    verts = np.array([fields(e, (float, float), "x y") for e in vsec], dtype=float).reshape(nv, 2)
    tris = np.array([fields(e, (int, int, int), "v0 v1 v2") for e in tsec], dtype=np.int64).reshape(nt, 3)
    markers = {}
    for no, tok in bsec:
        if len(tok) != 3:
            raise MeshError(f"{path}:{no}: expected 'v0 v1 label'")
        try:
            a, b = int(tok[0]), int(tok[1])
        except ValueError as err:
            raise MeshError(f"{path}:{no}: {err}") from None
        markers[(min(a, b), max(a, b))] = tok[2]
    for (no, _), t in zip(tsec, tris):
        if t.min() < 0 or t.max() >= nv:
            raise MeshError(f"{path}:{no}: vertex index out of range")
    return build_mesh(verts, tris, markers)


def save_mesh(mesh: TriMesh, path) -> None:
    """Write ``mesh`` in the text format read by load_mesh (labelled boundary
    facets only; vertex coordinates with 17 significant digits, so a save/load
    round trip reproduces the mesh bit for bit)."""
    lab = getattr(mesh, "facet_labels", None) or {}
    with open(path, "w") as fh:
        fh.write(f"{mesh.vertices.shape[0]} {mesh.n_elements} {len(lab)}\n")
        for x, y in mesh.vertices:
            fh.write(f"{x:.17g} {y:.17g}\n")
        for a, b, c in mesh.triangles:
            fh.write(f"{a} {b} {c}\n")
        for f in sorted(lab):
            a, b = mesh.facet_vertices[f]
            fh.write(f"{a} {b} {lab[f]}\n")
