"""Space-time quadrature: RHS projection and error norms against the
reference's own outputs (tests/golden/quadrature.npz, made by
tests/golden/make_quadrature_golden.py), host restatement and the NVRTC
build of the GPU kernels (csrc/quadrature.cu)."""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2008_01996_b200 import fem, meshes, temporal

PI = np.pi
U = "sin(pi*x)*sin(pi*y)*t*t"
UX = "pi*cos(pi*x)*sin(pi*y)*t*t"
UY = "pi*sin(pi*x)*cos(pi*y)*t*t"
UT = "2.0*t*sin(pi*x)*sin(pi*y)"
F = "(2.0*t + 2.0*pi*pi*t*t)*sin(pi*x)*sin(pi*y)"


def fixture():
    z = np.load(f"{GOLDEN}/quadrature.npz")
    mesh = meshes.TriangleMesh(z["vertices"], z["triangles"], z["boundary_flags"])
    return z, mesh, temporal.TemporalMesh(z["nodes"])


def u(x, y, t):
    return np.sin(PI * x) * np.sin(PI * y) * t * t


def grad(x, y, t):
    return (PI * np.cos(PI * x) * np.sin(PI * y) * t * t, PI * np.sin(PI * x) * np.cos(PI * y) * t * t)


def dt(x, y, t):
    return 2.0 * t * np.sin(PI * x) * np.sin(PI * y)


def f(x, y, t):
    return (2.0 * t + 2.0 * PI * PI * t * t) * np.sin(PI * x) * np.sin(PI * y)


@pytest.mark.parametrize("order,key", [(6, "project6"), (3, "project3")])
def test_project_rhs_matches_reference(order, key):
    z, mesh, tm = fixture()
    out = fem.project_rhs(mesh, tm, f, quad_order=order)
    assert np.abs(out - z[key]).max() < 1e-13 * np.abs(z[key]).max()


@pytest.mark.parametrize("order,keys", [(None, ("l2", "h1")), (6, ("l2_q6", "h1_q6"))])
def test_error_norms_match_reference(order, keys):
    z, mesh, tm = fixture()
    l2, h1 = fem.error_norms(z["coeffs"], mesh, tm, u, grad, dt, quad_order=order)
    assert l2 == pytest.approx(float(z[keys[0]]), rel=1e-12)
    assert h1 == pytest.approx(float(z[keys[1]]), rel=1e-12)


def test_collapsed_rule_is_exact():
    pts, wts = fem.triangle_rule(12)
    assert wts.sum() == pytest.approx(0.5, rel=1e-15)
    # int_T x^a y^b = a! b! / (a + b + 2)!
    from math import factorial

    for a, b in ((0, 0), (3, 4), (12, 0), (5, 7), (6, 6)):
        exact = factorial(a) * factorial(b) / factorial(a + b + 2)
        assert np.sum(wts * pts[:, 0] ** a * pts[:, 1] ** b) == pytest.approx(exact, rel=1e-13)


def test_gpu_kernels_compile_for_sm100a():
    pytest.importorskip("cuda.bindings")
    from paper_2008_01996_b200 import quadrature_gpu as q

    assert q.cubin(q.rhs_defines(F))[:4] == b"\x7fELF"
    assert q.cubin(q.error_defines(U, UX, UY, UT))[:4] == b"\x7fELF"
