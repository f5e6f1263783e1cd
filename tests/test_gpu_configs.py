"""Full-size BASELINE.json configurations on the GPU, checked through
size-independent properties (residual, linearity, determinism) and, where
the CPU oracle finishes in seconds, against the backward-stable
Bartels-Stewart oracle."""

import numpy as np
import pytest

from conftest import rel_diff

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2_system(cuda_ok):
    import torch

    from paper_2008_01996_b200 import problems

    system, info = problems.build_system("c2", temporal_device=torch.device("cuda", 0))
    assert info["m_x"] == 12033 and info["n_t"] == 128
    return system


@pytest.fixture(scope="module")
def c3_system(cuda_ok):
    import torch

    from paper_2008_01996_b200 import problems

    system, info = problems.build_system("c3", temporal_device=torch.device("cuda", 0))
    assert info["m_x"] == 65025 and info["n_t"] == 256
    return system


def test_c2_matches_bs_oracle(c2_system):
    from oracle import fd_oracle as orc
    from paper_2008_01996_b200 import solvers

    sol, rep = solvers.solve_fd(c2_system)
    assert rep.residual < 1e-11
    ref = orc.solve_bs_complex(*orc.system_arrays(c2_system))
    assert rel_diff(sol.coefficients, ref) < 1e-10
    # the residual reported by the GPU agrees with the oracle's own residual
    assert orc.residual(*orc.system_arrays(c2_system), sol.coefficients) < 1e-11


def test_c2_plain_fd_is_kappa_limited(c2_system):
    from paper_2008_01996_b200 import solvers

    _, rep = solvers.solve_fd(c2_system, refine=0)
    # kappa_2(X_t) ~ 7.5e7 at N_t=128: the unrefined FD sits near kappa*eps
    assert 1e-12 < rep.fd_residual < 1e-6


def test_c3_residual_linearity_determinism(c3_system):
    import dataclasses

    from paper_2008_01996_b200 import solvers

    pencil = solvers.build_pencil(c3_system.temporal, "fd")
    a, rep = solvers.solve_fd(c3_system, pencil=pencil)
    assert rep.residual < 1e-11
    assert rep.refine_steps >= 1
    b, _ = solvers.solve_fd(c3_system, pencil=pencil)
    assert np.array_equal(a.coefficients, b.coefficients)
    # scaling the rhs by 2 is exact in binary floating point
    two = dataclasses.replace(c3_system, rhs=2.0 * c3_system.rhs)
    c, _ = solvers.solve_fd(two, pencil=pencil)
    assert np.array_equal(c.coefficients, 2.0 * a.coefficients)
    # the GPU residual of the solution agrees with a fresh residual evaluation
    assert solvers.residual(c3_system, a.coefficients) == pytest.approx(rep.residual, rel=1e-3, abs=1e-16)


def test_c3_superposition(c3_system):
    import dataclasses

    from paper_2008_01996_b200 import solvers

    pencil = solvers.build_pencil(c3_system.temporal, "fd")
    rng = np.random.default_rng(7)
    f2 = rng.standard_normal(c3_system.rhs.shape)
    s1, _ = solvers.solve_fd(c3_system, pencil=pencil)
    s2, _ = solvers.solve_fd(dataclasses.replace(c3_system, rhs=f2), pencil=pencil)
    s12, _ = solvers.solve_fd(dataclasses.replace(c3_system, rhs=c3_system.rhs + f2), pencil=pencil)
    assert rel_diff(s1.coefficients + s2.coefficients, s12.coefficients) < 1e-12
