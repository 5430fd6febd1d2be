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

from .basis import REF_EDGES

__all__ = ["MeshError", "TriMesh", "build_mesh", "generate_structured", "generate_jittered", "load_mesh",
           "save_mesh"]


class MeshError(Exception):
    """Invalid mesh topology or geometry (MESH:18-19)."""


class TriMesh:
    """Immutable affine triangulation with oriented facets."""

    def __init__(self, vertices, triangles, facet_vertices, facet_elems, facet_local,
                 facet_flip, facet_labels=None):
        self.vertices = np.ascontiguousarray(vertices, dtype=float)
        self.triangles = np.ascontiguousarray(triangles, dtype=np.int64)
        self.facet_vertices = np.ascontiguousarray(facet_vertices, dtype=np.int64)
        self.facet_elems = np.ascontiguousarray(facet_elems, dtype=np.int64)
        self.facet_local = np.ascontiguousarray(facet_local, dtype=np.int64)
        self.facet_flip = np.ascontiguousarray(facet_flip, dtype=bool)
        self.facet_labels = dict(facet_labels or {})
        self.curved_maps = {}
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
        return float(0.5 * self.affine_det.sum())

    def is_curved(self, elem) -> bool:
        return False

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
