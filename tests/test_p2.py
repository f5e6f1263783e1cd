"""P2 in space and time (configuration c5). The reference has no P2
discretisation, so the assembly is pinned to the reference's P1 assembly
through the exact embedding P1 subset P2 (M^P1 = E^T M^P2 E, likewise A, and
the temporal H_T matrices), including the reference-generated temporal
fixture; the P2 system is then solved by the CPU oracle (reference BS
restatement) and by the halved FD with SuperLU standing in for the GPU."""

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from conftest import GOLDEN, rel_diff
from oracle import fd_oracle as orc
from paper_2008_01996_b200 import fem, meshes, p2, problems, solvers, temporal
from paper_2008_01996_b200.engine import conjugate_pairs, modal_plan


def _maxabs(a):
    a = a.toarray() if hasattr(a, "toarray") else np.asarray(a)
    return float(np.abs(a).max())


@pytest.mark.parametrize("mesh", [meshes.build_square_mesh(4), meshes.build_square_mesh(7),
                                  meshes.build_lshape_mesh(1)])
def test_space_embedding_reproduces_p1(mesh):
    o1, o2 = fem.assemble_p1(mesh), p2.assemble_p2(mesh)
    E = p2.p1_in_p2(mesh)
    for big, small in ((o2.M_full, o1.M_full), (o2.A_full, o1.A_full)):
        assert _maxabs(E.T @ big @ E - small) < 1e-13 * _maxabs(small)
    # interior P2 dofs restrict to interior P1 vertices
    bflags = np.zeros(o2.M_full.shape[0], bool)
    bflags[o2.boundary] = True
    assert np.array_equal(bflags[: mesh.n_vertices], mesh.boundary_flags)


def test_space_invariants():
    mesh = meshes.build_square_mesh(6)
    o2 = p2.assemble_p2(mesh)
    n = o2.M_full.shape[0]
    assert o2.M_full.sum() == pytest.approx(1.0, rel=1e-14)              # int 1 = |Omega|
    assert np.abs(o2.A_full @ np.ones(n)).max() < 1e-13                  # constants in the kernel
    x = p2.p2_dofs(mesh)[1][:, 0]
    assert x @ (o2.A_full @ x) == pytest.approx(1.0, rel=1e-13)         # |grad x|^2 over the square
    q = x * x                                                            # P2 interpolates x^2 exactly
    assert q @ (o2.M_full @ np.ones(n)) == pytest.approx(1.0 / 3.0, rel=1e-13)
    assert q @ (o2.A_full @ q) == pytest.approx(4.0 / 3.0, rel=1e-13)   # int |2x|^2
    assert abs(o2.M_full - o2.M_full.T).max() == 0.0
    assert (2 * 6 - 1) ** 2 == o2.n_interior


@pytest.mark.parametrize("nodes", [np.linspace(0, 1, 9), (np.arange(9) / 8.0) ** 2, np.linspace(0, 3, 6)])
def test_time_embedding_reproduces_p1(nodes):
    tm = temporal.TemporalMesh(nodes)
    t1 = temporal.assemble_temporal_operators(tm, j_max=100_000)
    t2 = p2.assemble_temporal_operators_p2(tm, j_max=100_000)
    Et = p2.temporal_p1_in_p2(tm.n_cells)
    assert _maxabs(Et.T @ t2.A @ Et - t1.A) < 1e-13 * _maxabs(t1.A)
    assert _maxabs(Et.T @ t2.M @ Et - t1.M) < 1e-13 * _maxabs(t1.M)
    assert _maxabs(Et.T @ t2.C - t1.C) < 1e-13 * _maxabs(t1.C)
    assert np.array_equal(t2.A, t2.A.T)
    assert np.linalg.eigvalsh(t2.A).min() > 0.0
    lam = np.linalg.eigvals(np.linalg.solve(t2.A, t2.M))
    assert lam.real.min() > 0.0


def test_time_embedding_matches_reference_fixture():
    """E_t^T A^P2 E_t against the reference's own P1 matrices (graded N_t=8)."""
    z = np.load(f"{GOLDEN}/temporal.npz")
    tm = temporal.TemporalMesh(z["graded8_nodes"])
    t2 = p2.assemble_temporal_operators_p2(tm, j_max=100_000)
    Et = p2.temporal_p1_in_p2(tm.n_cells)
    for mat, key in ((t2.A, "graded8_A"), (t2.M, "graded8_M")):
        ref = z[key]
        assert _maxabs(Et.T @ mat @ Et - ref) < 1e-12 * _maxabs(ref)


def test_temporal_p2_device_path_matches_host():
    torch = pytest.importorskip("torch")
    tm = temporal.TemporalMesh((np.arange(7) / 6.0) ** 2)
    host = p2.assemble_temporal_operators_p2(tm, j_max=70_000)
    dev = p2.assemble_temporal_operators_p2(tm, j_max=70_000, device=torch.device("cpu"))
    for a, b in ((host.A, dev.A), (host.M, dev.M), (host.C, dev.C)):
        assert _maxabs(a - b) < 1e-13 * _maxabs(a)


def _small_p2(cells=6, n=5):
    return problems.build_system(mesh=("square", n), n_t=cells, rhs="seeded", degree=2, grading=2.0,
                                 j_max=100_000)[0]


def test_p2_system_oracle_bs_matches_dense():
    system = _small_p2()
    arrs = orc.system_arrays(system)
    u_bs = orc.solve_bs_complex(*arrs)
    u_dense = orc.solve_dense(*arrs)
    assert rel_diff(u_bs, u_dense) < 1e-11
    assert orc.residual(*arrs, u_bs) < 1e-13


def test_p2_halved_fd_matches_oracle():
    """The modal plan (pair halving; a graded P2 pencil may carry real
    eigenvalues) reproduces the oracle BS solution with SuperLU solves."""
    system = _small_p2()
    p = solvers.build_pencil(system.temporal, "fd", eig="reduced")
    mp = modal_plan(system.temporal, p)
    reps, singles = conjugate_pairs(p.form.D, p.form.X)
    assert 2 * len(reps) + len(singles) == system.n_t
    n, nt = system.m_x, system.n_t
    F = np.asarray(system.rhs).reshape(n, nt, order="F")
    G = F @ mp.w_in
    nk = mp.n_k
    M, A = system.spatial.M_II.tocsc(), system.spatial.A_II.tocsc()
    Z = np.zeros((n, nk), complex)
    for k in range(nk):
        Z[:, k] = spla.spsolve((M + mp.lam[k] * A).astype(complex), G[:, k] + 1j * G[:, nk + k])
    u = (np.hstack([Z.real, Z.imag]) @ mp.w_out).ravel(order="F")
    ref = orc.solve_bs_complex(*orc.system_arrays(system))
    u_fd, _ = orc.solve_fd(*orc.system_arrays(system))
    gap = rel_diff(u_fd, ref)
    assert rel_diff(u, ref) < max(1e-11, 10 * gap)


def test_c5_config_shapes():
    cfg = problems.CONFIGS["c5"]
    assert cfg["degree"] == 2 and cfg["n_t"] == 512
    # P2 on the 128 grid has the c3 interior size
    assert (2 * 128 - 1) ** 2 == 65_025
