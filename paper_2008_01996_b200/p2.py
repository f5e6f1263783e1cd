"""P2 discretisations for configuration c5 (host input generators).

BASELINE.json config 5 asks for quadratic elements in space AND time. The
reference implements only P1 (reference SPEC.md:12), so nothing here has a
reference counterpart; it is pinned instead through the exact embedding
P1 subset P2 on the same mesh: with E the nodal interpolation of P1 functions
into P2 (vertex dofs copy, midpoint dofs average their two endpoints),

    M^P1 = E^T M^P2 E,   A^P1 = E^T A^P2 E          (space, any mesh)
    A_t^P1 = E_t^T A_t^P2 E_t, M_t^P1 = E_t^T M_t^P2 E_t   (time, same j_max)

holds exactly (up to rounding) for the reference's own P1 assembly
(tests/test_p2.py), and the P2 FD solution is checked against the
reference's dense Kronecker oracle / BS solvers run on these operators.

Space: 6-node triangles, local dofs [v0, v1, v2, e01, e12, e20], basis
lambda_i (2 lambda_i - 1) and 4 lambda_i lambda_j, element matrices by exact
quadrature; an edge dof is on the boundary when its edge belongs to one
triangle only.

Time: on each cell [t_{c-1}, t_c] the Lagrange basis L0, L1 (midpoint), L2;
global dofs in time order (m_1, t_1, m_2, t_2, ..., m_N, t_N), the t_0 vertex
dropped like the P1 hat at node 0 (reference temporal.py:18-20). The sine
coefficients a_j = (2/T) int q sin(w t), w = theta_j / T, and
b_j = int q cos(w t) of a piecewise quadratic q with q(0) = 0, cos(theta_j) = 0
have the closed forms (two integrations by parts, q''' = 0 on each cell)

    int q sin(w t) = (1/w) sum_c ( [q' sin(w t)]_c / w + q''_c [cos(w t)]_c / w^2 )
    int q cos(w t) = q(T) sin(theta_j) / w
                     + (1/w) sum_c ( [q' cos(w t)]_c / w - q''_c [sin(w t)]_c / w^2 )

([.]_c = value at the cell's right end minus left end, one-sided q'), which
reduce to the reference's P1 formulas (temporal.py:98-151) for q'' = 0. The
matrices are then the same truncated series as for P1:
A = 1/2 sum theta_j a a^T, M = sum a b^T, C = sum a d^T.
"""

import numpy as np
import scipy.sparse as sp

from .errors import DegenerateElement
from .fem import SpatialOperators, triangle_rule
from .temporal import _CHUNK, DEFAULT_J_MAX, TemporalOperators, _is_cuda, assemble_native

# ---------------------------------------------------------------------------
# space


def p2_dofs(mesh):
    """(element dof table (n_tri, 6), dof coordinates, dof boundary flags,
    edge list (n_edges, 2)) for the P2 space on `mesh`; vertex dofs keep the
    vertex numbers, edge dofs follow as n_vertices + edge index."""
    tris = mesh.triangles
    nv = mesh.n_vertices
    loc = np.array([[0, 1], [1, 2], [2, 0]])
    e = tris[:, loc]                                   # (n_tri, 3, 2)
    key = np.sort(e, axis=2).reshape(-1, 2)
    edges, inv, count = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    inv = inv.reshape(-1)
    dof = np.concatenate([tris, nv + inv.reshape(-1, 3)], axis=1)
    coords = np.concatenate([mesh.vertices, 0.5 * (mesh.vertices[edges[:, 0]] + mesh.vertices[edges[:, 1]])])
    edge_boundary = count == 1
    if np.any(edge_boundary & ~(mesh.boundary_flags[edges[:, 0]] & mesh.boundary_flags[edges[:, 1]])):
        raise DegenerateElement("boundary edge with an interior endpoint")
    flags = np.concatenate([mesh.boundary_flags, edge_boundary])
    return dof, coords, flags, edges


def _p2_basis(pts):
    """Values (q, 6) and barycentric-gradient coefficients of the P2 basis at
    reference points; grads returned as (q, 6, 3): d phi / d lambda_k."""
    l = np.column_stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]])
    pairs = [(0, 1), (1, 2), (2, 0)]
    val = np.empty((len(pts), 6))
    dl = np.zeros((len(pts), 6, 3))
    for i in range(3):
        val[:, i] = l[:, i] * (2.0 * l[:, i] - 1.0)
        dl[:, i, i] = 4.0 * l[:, i] - 1.0
    for k, (i, j) in enumerate(pairs):
        val[:, 3 + k] = 4.0 * l[:, i] * l[:, j]
        dl[:, 3 + k, i] = 4.0 * l[:, j]
        dl[:, 3 + k, j] = 4.0 * l[:, i]
    return val, dl


def assemble_p2(mesh):
    """P2 mass/stiffness with the same block structure as `fem.assemble_p1`."""
    from .fem import _geometry

    area, grads = _geometry(mesh)                      # grads: (t, 3 lambda, 2)
    dof, coords, flags, _ = p2_dofs(mesh)
    n = len(coords)
    pts5, w5 = triangle_rule(5)                        # exact for degree 4 (mass)
    val, _ = _p2_basis(pts5)
    mref = 2.0 * np.einsum("q,qi,qj->ij", w5, val, val)          # for unit area
    mref = 0.5 * (mref + mref.T)                       # exactly symmetric
    me = area[:, None, None] * mref[None]
    pts2, w2 = triangle_rule(2)                        # gradients are linear: degree 2
    _, dl = _p2_basis(pts2)
    g = np.einsum("qik,tkd->tqid", dl, grads)          # physical gradients
    ke = 2.0 * area[:, None, None] * np.einsum("q,tqid,tqjd->tij", w2, g, g)
    ke = 0.5 * (ke + ke.transpose(0, 2, 1))
    rows = np.repeat(dof, 6, axis=1).ravel()
    cols = np.tile(dof, (1, 6)).ravel()
    A_full = sp.coo_matrix((ke.ravel(), (rows, cols)), shape=(n, n)).tocsr()
    M_full = sp.coo_matrix((me.ravel(), (rows, cols)), shape=(n, n)).tocsr()
    interior = np.flatnonzero(~flags)
    boundary = np.flatnonzero(flags)
    iidx = -np.ones(n, dtype=np.int64)
    iidx[interior] = np.arange(len(interior))
    # M10[i, cell] = int_cell phi_i: 0 for vertex dofs, |T|/3 for edge dofs
    flat = dof[:, 3:].ravel()
    keep = iidx[flat] >= 0
    m10 = sp.coo_matrix(
        (np.repeat(area / 3.0, 3)[keep], (iidx[flat][keep], np.repeat(np.arange(len(dof)), 3)[keep])),
        shape=(len(interior), len(dof))).tocsr()
    return SpatialOperators(
        M_full=M_full, A_full=A_full, interior=interior, boundary=boundary, interior_index=iidx,
        M_II=M_full[interior][:, interior].tocsr(), A_II=A_full[interior][:, interior].tocsr(),
        M_IB=M_full[interior][:, boundary].tocsr(), A_IB=A_full[interior][:, boundary].tocsr(),
        M10=m10)


def p1_in_p2(mesh):
    """Interpolation E (n_P2 x n_P1) of P1 vertex functions into P2."""
    _, coords, _, edges = p2_dofs(mesh)
    nv = mesh.n_vertices
    ne = len(edges)
    rows = np.concatenate([np.arange(nv), nv + np.arange(ne), nv + np.arange(ne)])
    cols = np.concatenate([np.arange(nv), edges[:, 0], edges[:, 1]])
    vals = np.concatenate([np.ones(nv), np.full(2 * ne, 0.5)])
    return sp.csr_matrix((vals, (rows, cols)), shape=(len(coords), nv))


# ---------------------------------------------------------------------------
# time

# one-sided derivatives (times h) at the left/right cell end and q'' (times
# h^2) of the local Lagrange basis L0 (left vertex), L1 (midpoint), L2 (right)
_DQ_LEFT = np.array([-3.0, 4.0, -1.0])
_DQ_RIGHT = np.array([1.0, -4.0, 3.0])
_D2Q = np.array([4.0, -8.0, 4.0])


def temporal_p2_dof_map(n_cells):
    """(n_cells, 3) global dof of (L0, L1, L2) per cell, -1 for the dropped
    t_0 vertex; dof order (m_1, t_1, m_2, t_2, ...)."""
    c = np.arange(n_cells)
    return np.stack([2 * c - 1, 2 * c, 2 * c + 1], axis=1)


def _p2_coeffs(xp, nd, theta, T, sign):
    """Sine coefficients a (2N x J) and cosine integrals b (2N x J) of the P2
    temporal basis for frequencies theta (J,), nodes nd (N+1,)."""
    n = nd.shape[0] - 1
    h = nd[1:] - nd[:-1]
    w = theta / T
    arg = xp.outer(nd, w) if xp is np else xp.outer(nd, w)
    s, c = xp.sin(arg), xp.cos(arg)
    ds = s[1:] - s[:-1]                                # [sin]_c  (N, J)
    dc = c[1:] - c[:-1]                                # [cos]_c
    inv_h = (1.0 / h)[:, None]
    inv_h2 = inv_h * inv_h
    sin_int = []
    cos_int = []
    for k in range(3):
        # [q' sin]_c and [q' cos]_c with one-sided q' of basis k
        qs = (_DQ_RIGHT[k] * s[1:] - _DQ_LEFT[k] * s[:-1]) * inv_h
        qc = (_DQ_RIGHT[k] * c[1:] - _DQ_LEFT[k] * c[:-1]) * inv_h
        d2 = _D2Q[k] * inv_h2
        sin_int.append((qs / w + d2 * dc / (w * w)) / w)
        cos_int.append((qc / w - d2 * ds / (w * w)) / w)
    # assemble per global dof: midpoint m_c <- L1 of cell c; vertex t_c <- L2
    # of cell c + L0 of cell c+1
    zeros = xp.zeros_like(sin_int[0][:1])
    def glue(parts):
        mid = parts[1]
        vert = parts[2] + xp.cat([parts[0][1:], zeros]) if xp is not np else \
            parts[2] + np.concatenate([parts[0][1:], zeros])
        out = xp.stack([mid, vert], 1) if xp is not np else np.stack([mid, vert], axis=1)
        return out.reshape(2 * n, -1)
    a = glue(sin_int) * (2.0 / T)
    b = glue(cos_int)
    # q(T) sin(theta_j) / w only for the last vertex (q(T) = 1)
    b[2 * n - 1] += sign * (T / theta)
    d = ds * (T / theta)                               # int_cell cos(w t), (N, J)
    return a, b, d


def assemble_temporal_operators_p2(mesh, j_max=DEFAULT_J_MAX, device=None):
    """A_t, M_t (2N x 2N) and C_t (2N x N) of the P2 temporal space, same
    truncated series and chunk order as the P1 assembly (temporal.py); on a
    CUDA device through the hand-written kernels (csrc/temporal.cu)."""
    if j_max < 0:
        raise ValueError("j_max must be >= 0")
    if _is_cuda(device):
        A, M, C = assemble_native(mesh.nodes, 2, j_max, device)
        return TemporalOperators(A=A, M=M, C=C, j_max=int(j_max))
    nodes = np.asarray(mesh.nodes, dtype=float)
    T = float(nodes[-1])
    n = len(nodes) - 1
    starts = range((j_max // _CHUNK) * _CHUNK, -1, -_CHUNK)
    if device is None:
        xp = np
        nd = nodes
        triA = np.zeros((2 * n, 2 * n))
        M = np.zeros((2 * n, 2 * n))
        C = np.zeros((2 * n, n))
    else:
        import torch
        xp = torch
        nd = torch.tensor(nodes, dtype=torch.float64, device=device)
        triA = torch.zeros((2 * n, 2 * n), dtype=torch.float64, device=device)
        M = torch.zeros_like(triA)
        C = torch.zeros((2 * n, n), dtype=torch.float64, device=device)
    for j0 in starts:
        j1 = min(j0 + _CHUNK, j_max + 1)
        if xp is np:
            j = np.arange(j0, j1)
            sign = np.where(j % 2 == 0, 1.0, -1.0)
        else:
            j = torch.arange(j0, j1, device=device, dtype=torch.float64)
            sign = 1.0 - 2.0 * torch.remainder(j, 2.0)
        theta = np.pi * (j + 0.5)
        a, b, d = _p2_coeffs(xp, nd, theta, T, sign)
        wa = a * xp.sqrt(theta)
        triA += 0.5 * (wa @ wa.T)
        M += a @ b.T
        C += a @ d.T
    if xp is not np:
        triA, M, C = (x.cpu().numpy() for x in (triA, M, C))
    low = np.tril(triA)
    A = low + np.tril(low, -1).T
    return TemporalOperators(A=A, M=M, C=C, j_max=int(j_max))


def temporal_p1_in_p2(n_cells):
    """E_t (2N x N): P1 hat at t_i -> P2 vertex dof t_i + 1/2 of the two
    adjacent midpoint dofs (only m_N on the right of t_N: none)."""
    rows, cols, vals = [], [], []
    for i in range(1, n_cells + 1):
        col = i - 1
        rows += [2 * i - 1, 2 * i - 2]
        cols += [col, col]
        vals += [1.0, 0.5]
        if i < n_cells:
            rows.append(2 * i)
            cols.append(col)
            vals.append(0.5)
    return sp.csr_matrix((vals, (rows, cols)), shape=(2 * n_cells, n_cells))
