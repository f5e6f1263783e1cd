"""Host symbolic analysis (nested dissection, fronts, maps) checked on CPU:
every front's row list must contain the exact Cholesky fill of its pivot
columns, the tree must be a postorder, and fill must grow like n log n
(reference contracts: pkg/tests/test_sparse_direct.py:21-56)."""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2008_01996_b200 import fem, meshes
from paper_2008_01996_b200 import sparse_direct as sd
from paper_2008_01996_b200.errors import DimensionMismatch


def laplacian_1d(n):
    return sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(n, n), format="csr")


def grid_5pt(k):
    I = sp.identity(k, format="csr")
    T = laplacian_1d(k)
    return (sp.kron(I, T) + sp.kron(T, I)).tocsr()


def spd_cases():
    sq = fem.assemble_p1(meshes.build_square_mesh(18))
    ls = fem.assemble_p1(meshes.build_lshape_mesh(3))
    rng = np.random.default_rng(0)
    R = sp.random(120, 120, density=0.03, random_state=1)
    R = R + R.T
    R = R + sp.identity(120) * (abs(R).sum(axis=1).max() + 1)
    blocks = sp.block_diag([grid_5pt(5), laplacian_1d(7) + sp.identity(7), sp.identity(3)]).tocsr()
    return {
        "square18": (sq.M_II + sq.A_II).tocsr(),
        "lshape3": (ls.M_II + ls.A_II).tocsr(),
        "lap1d": (laplacian_1d(300) + sp.identity(300)).tocsr(),
        "grid5pt": (grid_5pt(16) + sp.identity(256)).tocsr(),
        "random": sp.csr_matrix(R),
        "disconnected": blocks,
        "identity": sp.identity(10, format="csr"),
        "scalar": sp.csr_matrix([[2.0]]),
    }


@pytest.mark.parametrize("name", list(spd_cases()))
@pytest.mark.parametrize("leaf", [1, 8, 24])
def test_front_rows_cover_cholesky_fill(name, leaf):
    K = spd_cases()[name]
    sym = sd.analyze(K, leaf_size=leaf)
    n = K.shape[0]
    perm = sym.perm
    assert np.array_equal(np.sort(perm), np.arange(n))
    first, p, q, par, dep, rows = sym.fronts()
    assert p.sum() == n and np.all(p >= 1)
    # contiguous pivot ranges in postorder, parents after children
    assert np.array_equal(np.sort(first), np.concatenate([[0], np.cumsum(p)[:-1]]))
    assert np.all((par == -1) | (par > np.arange(len(p))))
    assert np.all(dep[par >= 0] == dep[par[par >= 0]] + 1)
    L = np.linalg.cholesky(K[perm][:, perm].toarray())
    off = np.concatenate([[0], np.cumsum(q)])
    for f in range(len(p)):
        allowed = np.zeros(n, bool)
        allowed[first[f]:first[f] + p[f]] = True
        allowed[rows[off[f]:off[f + 1]]] = True
        assert np.all(rows[off[f]:off[f + 1]] >= first[f] + p[f])
        for j in range(first[f], first[f] + p[f]):
            nz = np.nonzero(np.abs(L[j:, j]) > 1e-14 * np.abs(L[j, j]))[0] + j
            assert allowed[nz].all(), (f, j)
    # update rows of a child are a subset of the parent's rows
    for f in range(len(p)):
        if par[f] >= 0:
            P = par[f]
            prow = set(range(first[P], first[P] + p[P])) | set(rows[off[P]:off[P + 1]])
            assert set(rows[off[f]:off[f + 1]]) <= prow


def test_identity_has_no_fill():
    sym = sd.analyze(sp.identity(10, format="csr"))
    assert sym.factor_nnz == 10


def test_tridiagonal_low_fill():
    # with scalar leaves the dissection of a path has no fill beyond 3n;
    # the default dense leaves trade a little storage for fewer, larger fronts
    assert sd.analyze(laplacian_1d(50), leaf_size=1).factor_nnz <= 4 * 50
    assert sd.analyze(laplacian_1d(50)).factor_nnz <= 12 * 50


def test_grid_fill_growth_subquadratic():
    # reference test_sparse_direct.py:43-47 (n quadruples, dense ratio 16)
    a = sd.analyze(grid_5pt(32)).factor_nnz
    b = sd.analyze(grid_5pt(64)).factor_nnz
    assert b / a < 6.5


def test_p1_grid_flops_scale_like_nested_dissection():
    s = [sd.analyze((o.M_II + o.A_II).tocsr()).stats
         for o in (fem.assemble_p1(meshes.build_square_mesh(64)), fem.assemble_p1(meshes.build_square_mesh(128)))]
    # ND on a 2D grid: flops ~ n^1.5 (x8 per refinement), fill ~ n log n
    assert s[1]["flops"] / s[0]["flops"] < 10.0
    assert s[1]["factor_nnz"] / s[0]["factor_nnz"] < 5.5


def test_counter_increments():
    before = sd.analyze_call_count()
    sd.analyze(sp.identity(3, format="csr"))
    assert sd.analyze_call_count() == before + 1


def test_rejects_rectangular():
    with pytest.raises(DimensionMismatch):
        sd.analyze(sp.csr_matrix(np.ones((2, 3))))


def test_align_values_rejects_entries_outside_pattern():
    sym = sd.analyze(laplacian_1d(5))
    bad = laplacian_1d(5).tolil()
    bad[0, 4] = 1.0
    with pytest.raises(DimensionMismatch):
        sym.align_values(bad.tocsr())


def test_analysis_is_deterministic():
    K = spd_cases()["square18"]
    a, b = sd.analyze(K), sd.analyze(K)
    assert np.array_equal(a.perm, b.perm)
    assert a.stats == b.stats


def test_native_pattern_is_the_symmetrized_union():
    """kh_symbolic_pattern returns A | A^T with the full diagonal, sorted and
    without duplicates -- the same CSR as the host symmetrization."""
    import scipy.sparse as sp

    from paper_2008_01996_b200 import sparse_direct as sd

    rng = np.random.default_rng(3)
    n = 300
    A = sp.random(n, n, density=0.02, random_state=rng, format="csr")
    A = (A + sp.eye(n, format="csr") * 0).tocsr()
    dup = sp.csr_matrix((np.ones(5), ([0, 0, 1, 7, 7], [3, 3, 2, 9, 9])), shape=(n, n))
    P = (A + dup).tocsr()
    s = sd.analyze(P, 8)
    ip, ix = sd.symmetrized_pattern(P + sp.eye(n, format="csr"))
    assert np.array_equal(s.indptr, ip) and np.array_equal(s.indices, ix)
    assert s.stats["nnz"] == len(ix)
