"""P1 spatial operators and space-time load vectors (host input generators).

Restates the reference assembly (`pkg/src/kronheat/fem.py`) so the benchmark
inputs are built the way the reference builds them:

* `assemble_p1`          -> fem.py:205-256 (M, A, interior/boundary blocks, M10)
* `triangle_rule`        -> fem.py:49-123 (Strang-Fix / Dunavant rules)
* `project_rhs`          -> fem.py:267-297 (cell averages, graded panels on cell 0)
* `assemble_global_rhs`  -> fem.py:312-346
* `dirichlet_lift`       -> fem.py:300-309

These run once per problem, outside every timed region.
"""

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .errors import DegenerateElement, DimensionMismatch


@dataclass(frozen=True)
class SpatialOperators:
    """P1 matrices split by boundary flags (reference fem.py:140-176)."""

    M_full: sp.csr_matrix
    A_full: sp.csr_matrix
    interior: np.ndarray
    boundary: np.ndarray
    interior_index: np.ndarray
    M_II: sp.csr_matrix
    A_II: sp.csr_matrix
    M_IB: sp.csr_matrix
    A_IB: sp.csr_matrix
    M10: sp.csr_matrix

    @property
    def n_interior(self):
        return len(self.interior)


def _rule_s3(a):
    b = 1.0 - 2.0 * a
    return [(a, a), (a, b), (b, a)]


def _rule_s6(a, b):
    c = 1.0 - a - b
    return [(a, b), (b, a), (a, c), (c, a), (b, c), (c, b)]


_R15 = math.sqrt(15.0)
# (points, weights normalised to one) on the reference triangle; published
# symmetric rules of degree 1, 2, 3, 5 and 6.
_RULES = {
    1: ([(1 / 3, 1 / 3)], [1.0]),
    2: (_rule_s3(1 / 6), [1 / 3] * 3),
    3: ([(1 / 3, 1 / 3)] + _rule_s3(1 / 5), [-27 / 48] + [25 / 48] * 3),
    5: ([(1 / 3, 1 / 3)] + _rule_s3((6 - _R15) / 21) + _rule_s3((6 + _R15) / 21),
        [9 / 40] + [(155 - _R15) / 1200] * 3 + [(155 + _R15) / 1200] * 3),
    6: (_rule_s3(0.063089014491502) + _rule_s3(0.249286745170910)
        + _rule_s6(0.310352451033785, 0.053145049844816),
        [0.050844906370207] * 3 + [0.116786275726379] * 3 + [0.082851075618374] * 6),
}


def triangle_rule(order):
    """Smallest catalogued rule of degree >= order; weights sum to 1/2."""
    if order < 1:
        raise ValueError("quadrature order must be >= 1")
    for deg in sorted(_RULES):
        if deg >= order:
            pts, wts = _RULES[deg]
            return np.array(pts, dtype=float), 0.5 * np.array(wts, dtype=float)
    raise ValueError("quadrature order above 6 is not needed by the benchmarks")


def gauss_rule_01(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


_GRADED_SPLITS = 12


def _time_panels(ell, tq, tw):
    """Quadrature on temporal cell ``ell`` in unit coordinates; cell 0 is
    split into dyadic panels toward t=0 (reference fem.py:108-137)."""
    if ell == 0:
        edges = np.concatenate([[0.0], 2.0 ** -np.arange(_GRADED_SPLITS - 1, -1, -1.0)])
    else:
        edges = np.array([0.0, 1.0])
    width = np.diff(edges)
    return ((edges[:-1, None] + width[:, None] * tq[None, :]).ravel(),
            (width[:, None] * tw[None, :]).ravel())


def _geometry(mesh):
    p = mesh.vertices[mesh.triangles]
    y = p[:, :, 1]
    x = p[:, :, 0]
    b = np.stack([y[:, 1] - y[:, 2], y[:, 2] - y[:, 0], y[:, 0] - y[:, 1]], axis=1)
    c = np.stack([x[:, 2] - x[:, 1], x[:, 0] - x[:, 2], x[:, 1] - x[:, 0]], axis=1)
    two_area = b[:, 0] * c[:, 1] - b[:, 1] * c[:, 0]
    if np.any(two_area <= 0.0):
        raise DegenerateElement("triangle with non-positive area")
    grads = np.stack([b, c], axis=2) / two_area[:, None, None]
    return 0.5 * two_area, grads


def assemble_p1(mesh):
    """Assemble P1 mass/stiffness and the interior/boundary blocks."""
    area, grads = _geometry(mesh)
    tris = mesh.triangles
    n = mesh.n_vertices
    ke = np.einsum("tid,tjd,t->tij", grads, grads, area)
    me = (area[:, None, None] / 12.0) * (np.ones((3, 3)) + np.eye(3))
    rows = np.repeat(tris, 3, axis=1).ravel()
    cols = np.tile(tris, (1, 3)).ravel()
    A_full = sp.coo_matrix((ke.ravel(), (rows, cols)), shape=(n, n)).tocsr()
    M_full = sp.coo_matrix((me.ravel(), (rows, cols)), shape=(n, n)).tocsr()

    interior, boundary = mesh.interior, mesh.boundary
    iidx = -np.ones(n, dtype=np.int64)
    iidx[interior] = np.arange(len(interior))
    flat = tris.ravel()
    keep = iidx[flat] >= 0
    m10 = sp.coo_matrix(
        (np.repeat(area / 3.0, 3)[keep],
         (iidx[flat][keep], np.repeat(np.arange(len(tris)), 3)[keep])),
        shape=(len(interior), len(tris))).tocsr()
    return SpatialOperators(
        M_full=M_full, A_full=A_full, interior=interior, boundary=boundary,
        interior_index=iidx,
        M_II=M_full[interior][:, interior].tocsr(),
        A_II=A_full[interior][:, interior].tocsr(),
        M_IB=M_full[interior][:, boundary].tocsr(),
        A_IB=A_full[interior][:, boundary].tocsr(),
        M10=m10)


def _space_points(mesh, pts):
    p = mesh.vertices[mesh.triangles]
    bary = np.column_stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]])
    phys = np.einsum("qi,tid->tqd", bary, p)
    return phys[..., 0], phys[..., 1]


def project_rhs(mesh_x, mesh_t, f, quad_order=6):
    """Cell averages of f(x1, x2, t) over triangle x interval cells,
    shape (n_triangles, n_cells) (reference fem.py:267-297)."""
    pts, wts = triangle_rule(quad_order)
    tq, tw = gauss_rule_01((quad_order + 4) // 2)
    x1, x2 = _space_points(mesh_x, pts)
    nodes = np.asarray(mesh_t.nodes)
    out = np.empty((mesh_x.n_triangles, len(nodes) - 1))
    for ell in range(len(nodes) - 1):
        h = nodes[ell + 1] - nodes[ell]
        acc = 0.0
        for q, wq in zip(*_time_panels(ell, tq, tw)):
            acc = acc + wq * (f(x1, x2, nodes[ell] + h * q) @ wts)
        out[:, ell] = 2.0 * acc
    return out


def project_rhs_separable(mesh_x, mesh_t, space_fn, time_fn, quad_order=6):
    """`project_rhs` for f = space_fn(x1, x2) * time_fn(t).

    Same quadrature as `project_rhs`; the tensor structure turns the
    n_triangles x n_cells x n_points evaluation into an outer product, which
    is what makes the 512^2 x 1024 configuration assemblable on a host.
    """
    pts, wts = triangle_rule(quad_order)
    tq, tw = gauss_rule_01((quad_order + 4) // 2)
    x1, x2 = _space_points(mesh_x, pts)
    s = space_fn(x1, x2) @ wts
    nodes = np.asarray(mesh_t.nodes)
    g = np.empty(len(nodes) - 1)
    for ell in range(len(nodes) - 1):
        h = nodes[ell + 1] - nodes[ell]
        q, w = _time_panels(ell, tq, tw)
        g[ell] = float(np.sum(w * time_fn(nodes[ell] + h * q)))
    return 2.0 * np.outer(s, g)


def dirichlet_lift(mesh_x, mesh_t, g):
    bv = mesh_x.vertices[mesh_x.boundary]
    t = np.asarray(mesh_t.nodes)[1:]
    return g(bv[:, :1], bv[:, 1:2], t[None, :])


def assemble_global_rhs(F, ops, temp, lift=None):
    """vec(M10 F C^T - M_IB G A^T - A_IB G M^T), spatial index fastest
    (reference fem.py:312-346)."""
    n_t = temp.A.shape[0]
    if F.shape != (ops.M10.shape[1], n_t):
        raise DimensionMismatch(f"F has shape {F.shape}, expected {(ops.M10.shape[1], n_t)}")
    rhs = ops.M10 @ F @ temp.C.T
    if lift is not None:
        if lift.shape != (ops.M_IB.shape[1], n_t):
            raise DimensionMismatch(f"lift has shape {lift.shape}")
        rhs = rhs - ops.M_IB @ lift @ temp.A.T - ops.A_IB @ lift @ temp.M.T
    return np.asarray(rhs).ravel(order="F")
