"""GPU FD solve vs the reference (golden fixtures) and the CPU oracle.

Bars: against the backward-stable reference BS-complex solution <= 1e-10
relative l2 with space-time residual <= 1e-11 (after refinement); against the
reference FD <= max(1e-10, the reference FD's own distance to BS) -- the
reference FD is itself only kappa_2(X_t)*eps accurate (SURVEY.md finding 3).
"""

import dataclasses

import numpy as np
import pytest

from conftest import load_golden, rel_diff
from paper_2008_01996_b200 import solvers
from paper_2008_01996_b200.errors import DefectivePencil

pytestmark = pytest.mark.gpu

NAMES = ["lshape0", "odd", "random_11", "random_12", "random_13", "c1"]


@pytest.mark.parametrize("name", NAMES)
def test_fd_matches_reference(cuda_ok, name):
    system, ref = load_golden(name)
    sol, rep = solvers.solve_fd(system)
    u = sol.coefficients
    assert rel_diff(u, ref["bs"]) < 1e-10
    gap = rel_diff(ref["fd"], ref["bs"])
    assert rel_diff(u, ref["fd"]) < max(1e-10, 2.0 * gap)
    assert rep.residual < 1e-11
    assert rep.analyze_calls == 1
    assert rep.kappa2 == pytest.approx(float(ref["fd_kappa2"]), rel=1e-10)
    assert rep.min_re_lambda == pytest.approx(float(ref["fd_min_re_lambda"]), rel=1e-10)
    if "dense" in ref:
        assert rel_diff(u, ref["dense"]) < 1e-10


@pytest.mark.parametrize("name", NAMES)
def test_plain_fd_without_refinement(cuda_ok, name):
    """refine=0 is the reference's plain FD: same accuracy class as the CPU FD."""
    system, ref = load_golden(name)
    sol, rep = solvers.solve_fd(system, refine=0)
    ref_gap = rel_diff(ref["fd"], ref["bs"])
    assert rel_diff(sol.coefficients, ref["bs"]) < max(1e-10, 10.0 * ref_gap)
    assert rep.refine_steps == 0
    assert rep.fd_residual == pytest.approx(rep.residual)


@pytest.mark.parametrize("name", ["lshape0", "c1"])
def test_residual_matches_oracle(cuda_ok, name):
    from oracle import fd_oracle as orc

    system, ref = load_golden(name)
    for key in ("fd", "bs"):
        got = solvers.residual(system, ref[key])
        want = orc.residual(*orc.system_arrays(system), ref[key])
        assert got == pytest.approx(want, rel=1e-6, abs=1e-16)


def test_reported_residual_is_reproducible(cuda_ok):
    system, _ = load_golden("lshape0")
    sol, rep = solvers.solve_fd(system)
    assert solvers.residual(system, sol.coefficients) == pytest.approx(rep.residual, rel=1e-6, abs=1e-16)


def test_fd_reports_spectral_stats(cuda_ok):
    system, _ = load_golden("lshape0")
    _, rep = solvers.solve_fd(system)
    assert rep.kappa2 == pytest.approx(9.576, rel=1e-3)   # reference test_solvers.py:204-208
    assert rep.sigma_min > 0.0 and rep.min_re_lambda > 0.0


def test_fd_threads_agree(cuda_ok):
    system, _ = load_golden("lshape0")
    a, _ = solvers.solve_fd(system, threads=1)
    b, r = solvers.solve_fd(system, threads=3)
    assert rel_diff(a.coefficients, b.coefficients) < 1e-13
    assert r.threads == 3


def test_fd_is_deterministic(cuda_ok):
    system, _ = load_golden("c1")
    a, _ = solvers.solve_fd(system)
    b, _ = solvers.solve_fd(system)
    assert np.array_equal(a.coefficients, b.coefficients)


def test_batching_and_refactoring_agree(cuda_ok):
    system, _ = load_golden("c1")
    a, _ = solvers.solve_fd(system)
    b, _ = solvers.solve_fd(system, max_batch=5, keep_factors=False)
    assert rel_diff(a.coefficients, b.coefficients) < 1e-13


def test_scalar_reduction(cuda_ok):
    system, _ = load_golden("lshape0")
    m, a = 0.7, 2.3
    temp = system.temporal
    rng = np.random.default_rng(8)
    rhs = rng.standard_normal(temp.A.shape[0])
    from conftest import _Spatial
    import scipy.sparse as sp

    one = solvers.SpaceTimeSystem(temporal=temp, spatial=_Spatial(sp.csr_matrix([[m]]), sp.csr_matrix([[a]])),
                                  rhs=rhs)
    expect = np.linalg.solve(m * temp.A + a * temp.M, rhs)
    sol, _ = solvers.solve_fd(one)
    assert rel_diff(sol.coefficients, expect) < 1e-10


def test_fd_falls_back_to_bs_complex(cuda_ok, monkeypatch):
    system, ref = load_golden("lshape0")

    def broken(system, pencil=None, threads=1):
        raise DefectivePencil("forced")

    monkeypatch.setattr(solvers, "solve_fd", broken)
    sol, report = solvers.solve(system, "fd")
    assert report.variant == "bs-complex"
    assert "DefectivePencil" in report.fallback
    assert rel_diff(sol.coefficients, ref["dense"]) < 1e-10


def test_no_fallback_propagates(cuda_ok, monkeypatch):
    system, _ = load_golden("lshape0")

    def broken(system, pencil=None, threads=1):
        raise DefectivePencil("forced")

    monkeypatch.setattr(solvers, "solve_fd", broken)
    with pytest.raises(DefectivePencil):
        solvers.solve(system, "fd", fallback=False)


@pytest.mark.parametrize("name", ["lshape0", "odd", "random_11", "c1"])
def test_bs_complex_matches_reference(cuda_ok, name):
    system, ref = load_golden(name)
    sol, rep = solvers.solve_bs_complex(system)
    assert rel_diff(sol.coefficients, ref["bs"]) < 1e-11
    assert rep.residual < 1e-12
    assert rep.analyze_calls == 1


@pytest.mark.parametrize("name", ["c1", "lshape0"])
def test_fused_forward_sweep_agrees(cuda_ok, name):
    """The first application with the forward sweep fused into the
    factorization (kh_plan_factor_fwd) and the separate factor + sweeps give
    the same solution (different rounding order only)."""
    import torch

    from paper_2008_01996_b200.engine import FDEngine, modal_plan

    system, ref = load_golden(name)
    modal = modal_plan(system.temporal, solvers.build_pencil(system.temporal, "fd"))
    F = torch.from_numpy(np.ascontiguousarray(system.rhs)).cuda().view(system.n_t, system.m_x)
    out = []
    for fuse in (True, False):
        eng = FDEngine(system.spatial.M_II, system.spatial.A_II, modal, fuse_forward=fuse)
        U, info = eng.solve(F)   # refined: the plain FD amplifies rounding by kappa_2(X_t)
        out.append(U.cpu().numpy().ravel())
        assert eng.factored and info["residual"] < 1e-12
    assert rel_diff(out[0], out[1]) < 1e-12
    assert rel_diff(out[1], ref["bs"]) < 1e-10


# ---- drop-in: a pencil built by the reference itself ---------------------------
@dataclasses.dataclass(frozen=True)
class _RefEigenSvdForm:
    """The attribute set of the reference's kronheat.dense.EigenSvdForm (dense.py:81-106)."""

    X: np.ndarray
    D: np.ndarray
    U: np.ndarray
    sigma: np.ndarray
    Vh: np.ndarray

    @property
    def sigma_min(self):
        return float(self.sigma[-1])

    @property
    def sigma_max(self):
        return float(self.sigma[0])

    @property
    def kappa2(self):
        return float(self.sigma[0] / self.sigma[-1])


@dataclasses.dataclass(frozen=True)
class _RefPencil:
    """The attribute set of kronheat.solvers.PencilFactorization (solvers.py:85-101):
    no spectral_stats, no temporal operators."""

    variant: str
    chol_A: np.ndarray
    form: object

    @property
    def eigenvalues(self):
        return self.form.D

    @property
    def min_re_lambda(self):
        return float(np.min(self.eigenvalues.real))


def _reference_pencil(name):
    import os

    from conftest import GOLDEN

    z = np.load(os.path.join(GOLDEN, "ref_pencil.npz"))
    form = _RefEigenSvdForm(*(z[f"{name}_{f}"] for f in ("X", "D", "U", "sigma", "Vh")))
    return _RefPencil(variant=str(z[f"{name}_variant"]), chol_A=z[f"{name}_chol_A"], form=form)


@pytest.mark.parametrize("name", ["lshape0", "c1"])
def test_fd_accepts_reference_pencil(cuda_ok, name):
    """The reference's own pencil (tests/golden/make_ref_pencil.py) goes straight
    into the drop-in solve_fd; the report carries the reference's statistics."""
    system, ref = load_golden(name)
    pencil = _reference_pencil(name)
    sol, rep = solvers.solve_fd(system, pencil=pencil)
    assert rel_diff(sol.coefficients, ref["bs"]) < 1e-10
    assert rep.residual < 1e-11
    assert rep.kappa2 == pytest.approx(float(ref["fd_kappa2"]), rel=1e-12)
    assert rep.sigma_min == pytest.approx(float(ref["fd_sigma_min"]), rel=1e-12)
    assert rep.min_re_lambda == pytest.approx(float(ref["fd_min_re_lambda"]), rel=1e-12)
    assert rep.t_total == pytest.approx(rep.t_decompose + rep.t_transform_in + rep.t_spatial + rep.t_transform_out)


@pytest.mark.parametrize("name", ["lshape0", "odd", "random_11", "random_12", "random_13", "c1"])
def test_bs_real_matches_reference(cuda_ok, name):
    # bsreal.npz: the reference's own solve_bs_real on the same systems (tests/golden/make_golden_bsreal.py)
    import os

    from conftest import GOLDEN

    system, ref = load_golden(name)
    z = np.load(os.path.join(GOLDEN, "bsreal.npz"))
    sol, rep = solvers.solve(system, "bs-real")
    assert rep.variant == "bs-real"
    assert rel_diff(sol.coefficients, z[f"{name}_bsr"]) < 1e-11
    assert rel_diff(sol.coefficients, ref["bs"]) < 1e-11
    assert rep.residual < 1e-12
    assert rep.analyze_calls == 1   # one union analysis serves the real and the paired blocks
    assert rep.min_re_lambda == pytest.approx(float(z[f"{name}_bsr_min_re_lambda"]), rel=1e-10)


def test_bs_real_matches_oracle_on_graded_mesh(cuda_ok):
    # odd N_t on a graded mesh: a real eigenvalue among the 2 x 2 blocks, c2-like spatial pattern
    from oracle import fd_oracle as orc
    from paper_2008_01996_b200 import problems

    system, _ = problems.build_system(mesh=("square", 24), n_t=13, rhs="seeded", j_max=50_000, grading=2.0)
    sol, rep = solvers.solve_bs_real(system)
    ref = orc.solve_bs_real(*orc.system_arrays(system))
    assert rel_diff(sol.coefficients, ref) < 1e-10
    assert orc.residual(*orc.system_arrays(system), sol.coefficients) < 1e-12
