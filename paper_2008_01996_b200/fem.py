"""P1 spatial operators and space-time load vectors (host input generators).

Restates the reference assembly (`pkg/src/kronheat/fem.py`) so the benchmark
inputs are built the way the reference builds them:

* `assemble_p1`          -> fem.py:205-256 (M, A, interior/boundary blocks, M10)
* `triangle_rule`        -> fem.py:49-123 (Strang-Fix / Dunavant rules)
* `project_rhs`          -> fem.py:267-297 (cell averages, graded panels on cell 0)
* `assemble_global_rhs`  -> fem.py:312-346
* `dirichlet_lift`       -> fem.py:300-309
* `error_norms`          -> fem.py:358-418 (collapsed rules beyond degree 6: fem.py:67-81)
* GPU versions of `project_rhs` / `error_norms`: quadrature_gpu.py

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


def _collapsed_rule(order):
    """Collapsed (Duffy) tensor rule exact to total degree `order`
    (reference fem.py:67-81): x = u (1 - v), y = v, Gauss-Legendre in u and
    Gauss-Jacobi(1, 0) in v (the Jacobian 1 - v is the Jacobi weight), both
    mapped to [0, 1]; weights sum to 1/2."""
    from scipy.special import roots_jacobi

    n = (order + 2) // 2
    u, wu = np.polynomial.legendre.leggauss(n)
    u, wu = 0.5 * (u + 1.0), 0.5 * wu
    xj, wj = roots_jacobi(n, 1.0, 0.0)
    v, wv = 0.5 * (xj + 1.0), 0.25 * wj
    uu, vv = np.meshgrid(u, v, indexing="ij")
    return np.column_stack([(uu * (1.0 - vv)).ravel(), vv.ravel()]), np.outer(wu, wv).ravel()


def triangle_rule(order):
    """Smallest catalogued rule of degree >= order, else the collapsed rule
    (reference fem.py:84-104); weights sum to 1/2."""
    if order < 1:
        raise ValueError("quadrature order must be >= 1")
    for deg in sorted(_RULES):
        if deg >= order:
            pts, wts = _RULES[deg]
            return np.array(pts, dtype=float), 0.5 * np.array(wts, dtype=float)
    return _collapsed_rule(order)


def error_quadrature(quad_order=None):
    """(triangle rule, time rule) of the error norms (reference
    fem.py:349-355): degree 12 / 8 Gauss points by default."""
    if quad_order is None:
        return triangle_rule(12), gauss_rule_01(8)
    return triangle_rule(quad_order), gauss_rule_01((quad_order + 2) // 2)


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


def error_norms(coeffs, mesh_x, mesh_t, u, grad, dt, quad_order=None):
    """Space-time L2 and H1-seminorm errors of the P1 x P1 function with
    nodal coefficients `coeffs` (n_vertices x N_t, boundary values included,
    zero at t = 0) against exact callables u, grad = (u_x, u_y), dt = u_t
    (reference fem.py:358-418, same quadrature and summation structure).
    Host restatement; `quadrature_gpu.error_norms_gpu` is the device path."""
    if coeffs.shape != (mesh_x.n_vertices, mesh_t.n_cells):
        raise DimensionMismatch(f"coeffs shape {coeffs.shape} does not match "
                                f"{(mesh_x.n_vertices, mesh_t.n_cells)}")
    (pts, wts), (tq, tw) = error_quadrature(quad_order)
    area, grads = _geometry(mesh_x)
    tris = mesh_x.triangles
    x1, x2 = _space_points(mesh_x, pts)
    lam = np.column_stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]])
    w_sp = 2.0 * area[:, None] * wts[None, :]
    full = np.hstack([np.zeros((mesh_x.n_vertices, 1)), coeffs])
    nodes = np.asarray(mesh_t.nodes)
    acc_l2 = acc_h1 = 0.0
    for ell in range(mesh_t.n_cells):
        h = nodes[ell + 1] - nodes[ell]
        c_lo, c_hi = full[:, ell][tris], full[:, ell + 1][tris]
        c_dt = (c_hi - c_lo) / h
        for q, wq in zip(*_time_panels(ell, tq, tw)):
            t = nodes[ell] + h * q
            c = (1.0 - q) * c_lo + q * c_hi
            uh = np.einsum("ti,qi->tq", c, lam)
            duh = np.einsum("ti,qi->tq", c_dt, lam)
            gh = np.einsum("ti,tid->td", c, grads)
            wt = wq * h
            e = u(x1, x2, t) - uh
            acc_l2 += wt * np.sum(w_sp * e * e)
            ed = dt(x1, x2, t) - duh
            g1, g2 = grad(x1, x2, t)
            e1, e2 = g1 - gh[:, None, 0], g2 - gh[:, None, 1]
            acc_h1 += wt * np.sum(w_sp * (ed * ed + e1 * e1 + e2 * e2))
    return math.sqrt(acc_l2), math.sqrt(acc_h1)


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
