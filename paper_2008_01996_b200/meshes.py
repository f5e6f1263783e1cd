"""Structured triangulations used to build the benchmark inputs (host side).

Input generators only: they produce the spatial meshes the solver is fed,
following the reference conventions so that the assembled operators are the
ones the reference would build.

* L-shape: lattice spacing 0.5*2**-level on (-1,1)^2 minus [0,1]x[-1,0],
  squares split along the bottom-left/top-right diagonal
  (reference `pkg/src/kronheat/lshape.py:122-158`).
* Unit square: the same lattice/diagonal/ordering rules on (0,1)^2
  (the reference has no square mesher).
"""

from dataclasses import dataclass

import numpy as np

from .errors import DegenerateElement


@dataclass(frozen=True)
class TriangleMesh:
    """Conforming triangulation with per-vertex boundary flags
    (same fields as reference `lshape.py:52-119`)."""

    vertices: np.ndarray
    triangles: np.ndarray
    boundary_flags: np.ndarray
    level: int = 0

    def __post_init__(self):
        object.__setattr__(self, "vertices", np.asarray(self.vertices, dtype=float))
        object.__setattr__(self, "triangles", np.asarray(self.triangles, dtype=np.int64))
        object.__setattr__(self, "boundary_flags", np.asarray(self.boundary_flags, dtype=bool))
        if self.vertices.ndim != 2 or self.vertices.shape[1] != 2:
            raise ValueError("vertices must have shape (n, 2)")
        if self.triangles.ndim != 2 or self.triangles.shape[1] != 3:
            raise ValueError("triangles must have shape (m, 3)")
        if self.boundary_flags.shape != (len(self.vertices),):
            raise ValueError("one boundary flag per vertex required")

    @property
    def n_vertices(self):
        return len(self.vertices)

    @property
    def n_triangles(self):
        return len(self.triangles)

    @property
    def interior(self):
        return np.flatnonzero(~self.boundary_flags)

    @property
    def boundary(self):
        return np.flatnonzero(self.boundary_flags)

    @property
    def n_interior(self):
        return int(np.count_nonzero(~self.boundary_flags))

    def areas(self):
        p = self.vertices[self.triangles]
        e1 = p[:, 1] - p[:, 0]
        e2 = p[:, 2] - p[:, 0]
        a = 0.5 * (e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
        if np.any(a <= 0.0):
            raise DegenerateElement("triangle with non-positive area")
        return a


def _lattice_mesh(keep_vertex, keep_square, lo, hi, scale, on_boundary, level):
    """Generic lattice triangulation.

    Lattice points (i, j) for i, j in [lo, hi] are numbered with j as the
    outer loop and i inner (reference `lshape.py:133-141`); each kept square
    emits (bl, br, tr) then (bl, tr, tl) (`lshape.py:143-154`).
    """
    span = hi - lo + 1
    ii, jj = np.meshgrid(np.arange(lo, hi + 1), np.arange(lo, hi + 1), indexing="xy")
    ii = ii.ravel()
    jj = jj.ravel()  # j outer, i inner
    keep = keep_vertex(ii, jj)
    index = -np.ones(span * span, dtype=np.int64)
    index[keep] = np.arange(int(keep.sum()))
    verts = np.column_stack([ii[keep] / scale, jj[keep] / scale])

    si, sj = np.meshgrid(np.arange(lo, hi), np.arange(lo, hi), indexing="xy")
    si = si.ravel()
    sj = sj.ravel()
    ks = keep_square(si, sj)
    si, sj = si[ks], sj[ks]

    def idx(i, j):
        return index[(j - lo) * span + (i - lo)]

    bl, br, tr, tl = idx(si, sj), idx(si + 1, sj), idx(si + 1, sj + 1), idx(si, sj + 1)
    tris = np.empty((2 * len(si), 3), dtype=np.int64)
    tris[0::2] = np.column_stack([bl, br, tr])
    tris[1::2] = np.column_stack([bl, tr, tl])
    return TriangleMesh(verts, tris, on_boundary(verts), level=level)


def on_lshape_boundary(points, tol=1e-12):
    """Boundary predicate of the L-shape (reference `lshape.py:24-49`)."""
    p = np.asarray(points, dtype=float)
    x, y = p[:, 0], p[:, 1]
    outer = (np.abs(np.abs(x) - 1.0) <= tol) | (np.abs(np.abs(y) - 1.0) <= tol)
    reentrant = ((np.abs(x) <= tol) & (y <= tol)) | ((np.abs(y) <= tol) & (x >= -tol))
    return outer | reentrant


def build_lshape_mesh(level):
    """L-shape lattice mesh; level 0 has 24 triangles and 5 interior vertices."""
    if level < 0:
        raise ValueError("level must be >= 0")
    m = 2 ** (level + 1)
    return _lattice_mesh(
        keep_vertex=lambda i, j: ~((i > 0) & (j < 0)),
        keep_square=lambda i, j: ~((i >= 0) & (j <= -1)),
        lo=-m, hi=m, scale=float(m), on_boundary=on_lshape_boundary, level=level)


def on_square_boundary(points, tol=1e-12):
    p = np.asarray(points, dtype=float)
    x, y = p[:, 0], p[:, 1]
    return (np.abs(x) <= tol) | (np.abs(x - 1.0) <= tol) | (np.abs(y) <= tol) | (np.abs(y - 1.0) <= tol)


def build_square_mesh(n):
    """Unit square with n x n lattice squares; (n-1)^2 interior vertices.

    Vertex (i/n, j/n) gets index j*(n+1)+i.
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    return _lattice_mesh(
        keep_vertex=lambda i, j: np.ones(i.shape, dtype=bool),
        keep_square=lambda i, j: np.ones(i.shape, dtype=bool),
        lo=0, hi=n, scale=float(n), on_boundary=on_square_boundary, level=0)
