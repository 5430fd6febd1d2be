"""Affine tetrahedral meshes for the 3D convection path (BASELINE cfg5).

No reference code exists for 3D.  Conventions mirror the 2D
``mesh2d.Mesh`` (MESH:86-216) where they carry over:

* faces keyed by the sorted vertex triple, numbered in sorted key order; the
  lowest element index owns the face; ``facet_elems``/``facet_local`` as in 2D,
  local face f opposite local vertex f;
* every tetrahedron's vertices are stored in increasing global id (SURVEY §7,
  "ordering each tet's vertices by global id, so that shared faces agree"):
  the two elements sharing a face then parametrise it identically (same
  vertex order), so facet quadrature points coincide pointwise and no face
  permutation is needed.  The price is detJ < 0 on about half the elements,
  handled by sign(detJ) in the operator;
* ``generate_cube``: n^3 cubes, each split into the 6 Kuhn tetrahedra
  (paths 000 -> 111 through the axis permutations), conforming across cubes.
"""

from __future__ import annotations

from itertools import permutations

import numpy as np

from .mesh import MeshError

__all__ = ["TetMesh", "build_tet_mesh", "generate_cube"]


class TetMesh:
    def __init__(self, vertices, tets, facet_vertices, facet_elems, facet_local):
        self.vertices = np.ascontiguousarray(vertices, dtype=float)
        self.tets = np.ascontiguousarray(tets, dtype=np.int64)
        self.triangles = self.tets            # element array under the 2D attribute name
        self.facet_vertices = facet_vertices
        self.facet_elems = facet_elems
        self.facet_local = facet_local
        self.n_elements = len(self.tets)
        self.n_facets = len(facet_vertices)
        v = [self.vertices[self.tets[:, i]] for i in range(4)]
        J = np.stack([v[1] - v[0], v[2] - v[0], v[3] - v[0]], axis=2)     # columns = edges
        self.affine_jac = J
        self.affine_det = np.linalg.det(J)
        if np.any(np.abs(self.affine_det) <= 1e-300):
            raise MeshError("degenerate tetrahedron")
        self.affine_inv = np.linalg.inv(J)
        self.affine_origin = v[0]
        a = self.vertices[facet_vertices[:, 0]]
        b = self.vertices[facet_vertices[:, 1]]
        c = self.vertices[facet_vertices[:, 2]]
        cr = np.cross(b - a, c - a)
        self.facet_area = 0.5 * np.linalg.norm(cr, axis=1)

    @property
    def boundary_facets(self):
        return np.nonzero(self.facet_elems[:, 1] < 0)[0]

    @property
    def interior_facets(self):
        return np.nonzero(self.facet_elems[:, 1] >= 0)[0]

    def h_min(self) -> float:
        """Shortest edge length."""
        e = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
        return float(min(np.linalg.norm(self.vertices[self.tets[:, a]] - self.vertices[self.tets[:, b]],
                                        axis=1).min() for a, b in e))

    def total_volume(self) -> float:
        return float(np.abs(self.affine_det).sum() / 6.0)

    def element_neighbours(self):
        NT = self.n_elements
        nbr = np.full((NT, 4), -1, dtype=np.int64)
        nbf = np.full((NT, 4), -1, dtype=np.int64)
        bnd = np.full((NT, 4), -1, dtype=np.int64)
        fe, fl = self.facet_elems, self.facet_local
        inner = fe[:, 1] >= 0
        for s, o in ((0, 1), (1, 0)):
            nbr[fe[inner, s], fl[inner, s]] = fe[inner, o]
            nbf[fe[inner, s], fl[inner, s]] = fl[inner, o]
        bf = np.nonzero(~inner)[0]
        bnd[fe[bf, 0], fl[bf, 0]] = np.arange(bf.size)
        return nbr, nbf, bnd


def build_tet_mesh(vertices, tets) -> TetMesh:
    """Sort each tet's vertices by global id and match faces by sorted key."""
    vertices = np.asarray(vertices, dtype=float)
    tets = np.sort(np.asarray(tets, dtype=np.int64), axis=1)
    NT = len(tets)
    loc = [tuple(v for v in range(4) if v != f) for f in range(4)]
    fv = np.stack([tets[:, list(l)] for l in loc], axis=1).reshape(-1, 3)   # sorted triples
    nv = max(int(vertices.shape[0]), 1)
    key = (fv[:, 0] * nv + fv[:, 1]) * nv + fv[:, 2]
    order = np.argsort(key, kind="stable")
    ks = key[order]
    start = np.ones(ks.size, dtype=bool)
    start[1:] = ks[1:] != ks[:-1]
    counts = np.bincount(np.cumsum(start) - 1)
    if counts.max() > 2:
        raise MeshError("face shared by more than two tetrahedra")
    NF = counts.size
    first = np.nonzero(start)[0]
    o0 = order[first]
    facet_vertices = fv[o0]
    fe = np.full((NF, 2), -1, dtype=np.int64)
    fl = np.full((NF, 2), -1, dtype=np.int64)
    fe[:, 0], fl[:, 0] = o0 // 4, o0 % 4
    two = counts == 2
    o1 = order[first[two] + 1]
    fe[two, 1], fl[two, 1] = o1 // 4, o1 % 4
    return TetMesh(vertices, tets, facet_vertices, fe, fl)


def generate_cube(n: int) -> TetMesh:
    """Unit cube, n^3 cells x 6 Kuhn tetrahedra (BASELINE cfg5: n = 32)."""
    if n < 1:
        raise MeshError("nonpositive subdivision")
    g = np.linspace(0.0, 1.0, n + 1)
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    verts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    vid = lambda i, j, k: (k * (n + 1) + j) * (n + 1) + i
    kk, jj, ii = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
    tets = []
    for perm in permutations(range(3)):
        p = [np.zeros(3, dtype=int)]
        for ax in perm:
            q = p[-1].copy()
            q[ax] += 1
            p.append(q)
        tets.append(np.stack([vid(ii + d[0], jj + d[1], kk + d[2]) for d in p], axis=1))
    # cell-major order: the 6 tets of a cell are adjacent in memory
    tets = np.stack(tets, axis=1).reshape(-1, 4)
    return build_tet_mesh(verts, tets)
