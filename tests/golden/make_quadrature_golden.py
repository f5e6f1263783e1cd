"""Golden fixture for the space-time quadrature (RHS projection and error
norms), generated with the reference package in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_quadrature_golden.py

quadrature.npz stores the inputs (L-shape level-1 mesh, graded temporal mesh
of 8 cells, nodal coefficients) and the reference's project_rhs
(fem.py:267-297) and error_norms (fem.py:358-418) outputs for
u = sin(pi x) sin(pi y) t^2, f = u_t - lap u.
"""

import os

import numpy as np

import kronheat as kh  # the reference

HERE = os.path.dirname(os.path.abspath(__file__))
PI = np.pi


def u(x, y, t):
    return np.sin(PI * x) * np.sin(PI * y) * t * t


def grad(x, y, t):
    return (PI * np.cos(PI * x) * np.sin(PI * y) * t * t, PI * np.sin(PI * x) * np.cos(PI * y) * t * t)


def dt(x, y, t):
    return 2.0 * t * np.sin(PI * x) * np.sin(PI * y)


def f(x, y, t):
    return (2.0 * t + 2.0 * PI * PI * t * t) * np.sin(PI * x) * np.sin(PI * y)


def main():
    mesh = kh.build_lshape_mesh(1)
    g = kh.refine_bisect(kh.TemporalMesh(np.array((0.0, 1.0 / 32.0, 1.0 / 16.0, 1.0 / 8.0, 1.0 / 2.0))))
    F6 = kh.project_rhs(mesh, g, f, quad_order=6)
    F3 = kh.project_rhs(mesh, g, f, quad_order=3)
    v = mesh.vertices
    t = g.nodes[1:]
    coeffs = u(v[:, :1], v[:, 1:2], t[None, :])
    coeffs = coeffs + 1e-2 * np.random.default_rng(5).standard_normal(coeffs.shape)
    l2, h1 = kh.error_norms(coeffs, mesh, g, u, grad, dt)
    l2_6, h1_6 = kh.error_norms(coeffs, mesh, g, u, grad, dt, quad_order=6)
    np.savez_compressed(os.path.join(HERE, "quadrature.npz"), vertices=mesh.vertices, triangles=mesh.triangles,
                        boundary_flags=mesh.boundary_flags, nodes=g.nodes, project6=F6, project3=F3,
                        coeffs=coeffs, l2=l2, h1=h1, l2_q6=l2_6, h1_q6=h1_6)
    print("quadrature.npz", F6.shape, l2, h1, l2_6, h1_6)


if __name__ == "__main__":
    main()
