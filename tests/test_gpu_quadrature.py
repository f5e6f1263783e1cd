"""GPU space-time quadrature (csrc/quadrature.cu via NVRTC) against the
reference's own RHS projection and error norms (tests/golden/quadrature.npz)."""

import numpy as np
import pytest

from test_quadrature import F, U, UT, UX, UY, fixture

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("order,key", [(6, "project6"), (3, "project3")])
def test_project_rhs_gpu_matches_reference(cuda_ok, order, key):
    from paper_2008_01996_b200 import quadrature_gpu as q

    z, mesh, tm = fixture()
    out = q.project_rhs_gpu(mesh, tm, F, quad_order=order)
    assert np.abs(out - z[key]).max() < 1e-13 * np.abs(z[key]).max()


@pytest.mark.parametrize("order,keys", [(None, ("l2", "h1")), (6, ("l2_q6", "h1_q6"))])
def test_error_norms_gpu_match_reference(cuda_ok, order, keys):
    from paper_2008_01996_b200 import quadrature_gpu as q

    z, mesh, tm = fixture()
    l2, h1 = q.error_norms_gpu(z["coeffs"], mesh, tm, U, UX, UY, UT, quad_order=order)
    assert l2 == pytest.approx(float(z[keys[0]]), rel=1e-12)
    assert h1 == pytest.approx(float(z[keys[1]]), rel=1e-12)


def test_project_rhs_gpu_c2_matches_separable_host(cuda_ok):
    """c2's load (L-shape level 5 x 128 cells) on the GPU against the host's
    separable projection used by problems.build_system."""
    from paper_2008_01996_b200 import fem, meshes, quadrature_gpu as q, temporal

    mesh = meshes.build_lshape_mesh(5)
    tm = temporal.TemporalMesh(np.linspace(0.0, 1.0, 129))
    host = fem.project_rhs_separable(mesh, tm, lambda x, y: np.sin(np.pi * x) * np.sin(np.pi * y),
                                     lambda t: 2.0 * t + 2.0 * np.pi**2 * t**2, quad_order=6)
    dev = q.project_rhs_gpu(mesh, tm, F, quad_order=6)
    assert np.abs(dev - host).max() < 1e-12 * np.abs(host).max()
