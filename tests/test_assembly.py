"""Host input generators vs the reference's own assembly (golden fixtures)."""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import GOLDEN
from paper_2008_01996_b200 import fem, meshes, temporal


def _csr(z, p):
    return sp.csr_matrix((z[f"{p}_data"], z[f"{p}_indices"], z[f"{p}_indptr"]), shape=tuple(z[f"{p}_shape"]))


def test_temporal_graded_matches_reference():
    z = np.load(os.path.join(GOLDEN, "temporal.npz"))
    t = temporal.assemble_temporal_operators(temporal.TemporalMesh(z["graded8_nodes"]), j_max=100_000)
    for k in "AMC":
        ref = z[f"graded8_{k}"]
        assert np.max(np.abs(getattr(t, k) - ref)) <= 1e-13 * np.max(np.abs(ref))
    assert np.array_equal(t.A, t.A.T)


def test_temporal_uniform_default_jmax_matches_reference():
    z = np.load(os.path.join(GOLDEN, "temporal.npz"))
    t = temporal.assemble_temporal_operators(temporal.TemporalMesh(np.linspace(0.0, 1.0, 33)))
    for k in "AMC":
        ref = z[f"uniform32_{k}"]
        assert np.max(np.abs(getattr(t, k) - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("name,make", [("lshape2", lambda: meshes.build_lshape_mesh(2)),
                                       ("square8", lambda: meshes.build_square_mesh(8))])
def test_p1_matches_reference(name, make):
    z = np.load(os.path.join(GOLDEN, "p1.npz"))
    ops = fem.assemble_p1(make())
    assert np.array_equal(ops.interior, z[f"{name}_interior"])
    for mine, key in ((ops.M_II, "M"), (ops.A_II, "A"), (ops.M10, "M10")):
        ref = _csr(z, f"{name}_{key}")
        d = (sp.csr_matrix(mine) - ref)
        assert (abs(d).max() if d.nnz else 0.0) <= 1e-14 * abs(ref).max()


def test_lshape_interior_counts():
    # reference test_lshape.py:16
    assert [meshes.build_lshape_mesh(l).n_interior for l in range(4)] == [5, 33, 161, 705]


def test_square_sizes():
    assert meshes.build_square_mesh(32).n_interior == 961
    assert meshes.build_square_mesh(256).n_interior == 65025


def test_separable_projection_matches_generic():
    mx = meshes.build_lshape_mesh(1)
    mt = temporal.TemporalMesh(np.linspace(0.0, 1.0, 6))
    s = lambda x, y: np.sin(np.pi * x) * np.sin(np.pi * y)
    g = lambda t: 2.0 * t + 2.0 * np.pi**2 * t**2
    a = fem.project_rhs(mx, mt, lambda x, y, t: s(x, y) * g(t), quad_order=6)
    b = fem.project_rhs_separable(mx, mt, s, g, quad_order=6)
    assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(a))


def test_c1_inputs_match_reference_fixture():
    # BASELINE config 1 built by the restated generators equals the inputs the
    # reference assembled for the golden fixture (same mesh, series, seed)
    from conftest import load_golden
    from paper_2008_01996_b200 import problems

    system, _ = problems.build_system("c1")
    ref, _ = load_golden("c1")
    assert np.array_equal(system.rhs, ref.rhs)
    for mine, theirs in ((system.temporal.A, ref.temporal.A), (system.temporal.M, ref.temporal.M)):
        assert np.max(np.abs(mine - theirs)) <= 1e-13 * np.max(np.abs(theirs))
    for mine, theirs in ((system.spatial.M_II, ref.spatial.M_II), (system.spatial.A_II, ref.spatial.A_II)):
        d = sp.csr_matrix(mine) - theirs
        assert (abs(d).max() if d.nnz else 0.0) <= 1e-14 * abs(theirs).max()
