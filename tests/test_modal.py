"""Host-side modal plan (pair halving in the real eigenbasis), checked on the
CPU with SuperLU solves standing in for the GPU kernels: the halved FD must
reproduce the reference FD to kappa_2(X_t)*eps and be real by construction."""

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from conftest import load_golden, rel_diff
from paper_2008_01996_b200 import solvers
from paper_2008_01996_b200.engine import conjugate_pairs, modal_plan


def halved_fd(system):
    p = solvers.build_pencil(system.temporal, "fd")
    mp = modal_plan(system.temporal, p)
    n, nt = system.m_x, system.n_t
    F = np.asarray(system.rhs).reshape(n, nt, order="F")
    G = F @ mp.w_in
    nk = mp.n_k
    M, A = system.spatial.M_II.tocsc(), system.spatial.A_II.tocsc()
    Z = np.zeros((n, nk), complex)
    for k in range(nk):
        Z[:, k] = spla.spsolve((M + mp.lam[k] * A).astype(complex), G[:, k] + 1j * G[:, nk + k])
    U = np.hstack([Z.real, Z.imag]) @ mp.w_out
    return U.ravel(order="F"), mp, p


@pytest.mark.parametrize("name", ["lshape0", "odd", "random_11", "random_12", "random_13", "c1"])
def test_halved_fd_matches_reference_fd(name):
    system, ref = load_golden(name)
    u, mp, p = halved_fd(system)
    gap = rel_diff(ref["fd"], ref["bs"])
    assert rel_diff(u, ref["bs"]) < max(1e-11, 10 * gap)
    assert mp.n_k == mp.n_pairs + mp.n_single
    assert 2 * mp.n_pairs + mp.n_single == system.n_t


def test_odd_system_has_real_mode():
    system, _ = load_golden("odd")
    p = solvers.build_pencil(system.temporal, "fd")
    reps, singles = conjugate_pairs(p.form.D, p.form.X)
    assert len(singles) == 1 and len(reps) == 1
    assert p.form.D[singles[0]].imag == 0.0


def test_pairs_found_even_when_eigenvalues_are_not_bitwise_conjugate():
    from paper_2008_01996_b200 import problems

    system, _ = problems.build_system(mesh=("square", 4), n_t=64, rhs="seeded", j_max=50_000)
    p = solvers.build_pencil(system.temporal, "fd")
    reps, singles = conjugate_pairs(p.form.D, p.form.X)
    assert len(singles) == 0 and len(reps) == 32
