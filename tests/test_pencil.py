"""Host pencil: the Cholesky-reduced eigensolver (dgeev on L^-1 M_t L^-T, one
real SVD) against the reference's QZ route (dggev + complex SVD) and against
the reference's own pencil statistics in the golden fixtures
(reference solvers.py:166-206, dense.py:178-234)."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2008_01996_b200 import dense, solvers
from paper_2008_01996_b200.temporal import TemporalMesh, assemble_temporal_operators


def _match(a, b):
    """Index arrays (i, j) pairing every a[i] with its nearest b[j]."""
    from scipy.optimize import linear_sum_assignment

    return linear_sum_assignment(np.abs(a[:, None] - b[None, :]))


def _eig_gap(a, b):
    i, j = _match(a, b)
    return np.abs(a[i] - b[j]).max()


def _pencils(temporal):
    return solvers.build_pencil(temporal, "fd", eig="reduced"), solvers.build_pencil(temporal, "fd", eig="qz")


@pytest.mark.parametrize("name", ["lshape0", "odd", "random_11", "random_12", "random_13", "c1"])
def test_reduced_matches_reference_statistics(name):
    system, ref = load_golden(name)
    p, q = _pencils(system.temporal)
    assert p.min_re_lambda == pytest.approx(float(ref["fd_min_re_lambda"]), rel=1e-10)
    # the QZ route reproduces the reference's statistics exactly
    assert q.min_re_lambda == float(ref["fd_min_re_lambda"])
    assert q.form.sigma_min == pytest.approx(float(ref["fd_sigma_min"]), rel=1e-12)
    assert q.form.sigma_max == pytest.approx(float(ref["fd_sigma_max"]), rel=1e-12)
    assert q.form.kappa2 == pytest.approx(float(ref["fd_kappa2"]), rel=1e-12)
    # the reduced route's X differs from dggev's by a column scaling within
    # [1/sqrt(2), sqrt(2)] (phase-dependent max |Re|+|Im| normalisation)
    assert p.form.kappa2 == pytest.approx(float(ref["fd_kappa2"]), rel=1.0)
    # eigenvalue condition numbers are O(kappa_2(X)): agreement to eps * kappa_2
    tol = max(1e-12, 1e-15 * q.form.kappa2)
    assert _eig_gap(p.eigenvalues, q.eigenvalues) < tol * np.abs(q.eigenvalues).max()


@pytest.mark.parametrize("nodes", [np.linspace(0, 1, 33), (np.arange(41) / 40.0) ** 2, np.linspace(0, 2, 97)])
def test_reduced_matches_qz(nodes):
    tops = assemble_temporal_operators(TemporalMesh(nodes), j_max=100_000)
    p, q = _pencils(tops)
    fp, fq = p.form, q.form
    lam = np.abs(p.eigenvalues).max()
    assert _eig_gap(p.eigenvalues, q.eigenvalues) < max(1e-12, 1e-15 * fq.kappa2) * lam
    # same vectors up to a complex column factor c with |c| in [1/sqrt2, sqrt2]
    order_p, order_q = _match(fp.D, fq.D)
    Xp, Xq = fp.X[:, order_p], fq.X[:, order_q]
    c = np.einsum("ij,ij->j", Xq.conj(), Xp) / np.einsum("ij,ij->j", Xq.conj(), Xq)
    assert np.all(np.abs(c) > 0.7071) and np.all(np.abs(c) < 1.4143)
    assert np.linalg.norm(Xp - Xq * c[None, :]) < 1e-9 * fq.kappa2 * np.linalg.norm(Xq)
    # same conventions: pairs adjacent with +Im first, exact conjugate vectors,
    # columns scaled to max |Re|+|Im| = 1
    n = len(fp.D)
    j = 0
    while j < n:
        if fp.D[j].imag != 0.0:
            assert fp.D[j].imag > 0 and fp.D[j + 1] == np.conj(fp.D[j])
            assert np.array_equal(fp.X[:, j + 1], np.conj(fp.X[:, j]))
            j += 2
        else:
            j += 1
    assert np.allclose(np.max(np.abs(fp.X.real) + np.abs(fp.X.imag), axis=0), 1.0, rtol=1e-15, atol=0)
    # the SVD is an SVD of X
    assert np.linalg.norm(fp.U @ np.diag(fp.sigma) @ fp.Vh - fp.X) < 1e-13 * fp.sigma[0] * n
    assert np.allclose(fp.U.conj().T @ fp.U, np.eye(n), atol=1e-13)
    assert np.allclose(fp.Vh @ fp.Vh.conj().T, np.eye(n), atol=1e-13)
    # eigen-residual P X - X D
    P = dense.spd_solve(p.chol_A, tops.M)
    res = np.linalg.norm(P @ fp.X - fp.X * fp.D[None, :])
    assert dense.pencil_residual(P, fp.X, fp.D) == pytest.approx(res, rel=1e-6, abs=1e-14)
    assert res < 1e-12 * max(np.linalg.norm(P), 1.0)


def test_unknown_eigensolver_rejected():
    system, _ = load_golden("c1")
    with pytest.raises(ValueError):
        solvers.build_pencil(system.temporal, "fd", eig="nope")


@pytest.mark.parametrize("name", ["lshape0", "c1"])
def test_reduced_pencil_reports_reference_statistics(name):
    from paper_2008_01996_b200.solvers import SolveReport

    system, ref = load_golden(name)
    p = solvers.build_pencil(system.temporal, "fd", eig="reduced")
    rep = SolveReport(variant="fd", dof=1, n_t=1, m_x=1)
    rep.spectral_source = solvers.spectral_source(p)
    assert rep.sigma_min == pytest.approx(float(ref["fd_sigma_min"]), rel=1e-12)
    assert rep.sigma_max == pytest.approx(float(ref["fd_sigma_max"]), rel=1e-12)
    assert rep.kappa2 == pytest.approx(float(ref["fd_kappa2"]), rel=1e-12)


def test_report_spectral_fields_assignable():
    """sigma_min / sigma_max / kappa2 are plain fields as in the reference
    (solvers.py:136-139): constructor arguments, assignable, 0.0 when unset."""
    from paper_2008_01996_b200.solvers import SolveReport

    rep = SolveReport(variant="fd", dof=4, n_t=2, m_x=2, sigma_min=0.5, kappa2=3.0)
    assert rep.sigma_min == 0.5 and rep.kappa2 == 3.0 and rep.sigma_max == 0.0
    rep.sigma_max = 2.0
    rep.kappa2 = 4.0
    assert (rep.sigma_max, rep.kappa2) == (2.0, 4.0)
    blank = SolveReport(variant="fd", dof=1, n_t=1, m_x=1)
    assert (blank.sigma_min, blank.sigma_max, blank.kappa2) == (0.0, 0.0, 0.0)
    # an assigned value wins over the lazy source
    blank.spectral_source = lambda: (1.0, 8.0)
    assert blank.kappa2 == 8.0
    blank.kappa2 = 7.0
    assert blank.kappa2 == 7.0 and blank.sigma_min == 1.0
    assert "sigma_min=1.0" in repr(blank)


def test_report_t_total_reference_convention():
    """t_total = decompose + transform_in + spatial + transform_out
    (solvers.py:146-149); refinement is reported separately."""
    from paper_2008_01996_b200.solvers import SolveReport

    rep = SolveReport(variant="fd", dof=1, n_t=1, m_x=1, t_decompose=1.0, t_transform_in=2.0, t_spatial=3.0,
                      t_transform_out=4.0, t_refine=5.0)
    assert rep.t_total == 10.0
    assert rep.t_solve == 15.0
    assert rep.csv_row().split(",")[4:8] == ["1.000000", "2.000000", "3.000000", "4.000000"]


def test_spectral_source_of_reference_style_pencil():
    """A pencil without spectral_stats (the reference's own
    PencilFactorization) reports its form's singular values."""
    import types

    form = types.SimpleNamespace(sigma_min=0.25, sigma_max=4.0)
    pencil = types.SimpleNamespace(variant="fd", chol_A=None, form=form)
    assert solvers.spectral_source(pencil)() == (0.25, 4.0)
