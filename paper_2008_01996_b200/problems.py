"""The BASELINE.json configurations as seeded synthetic inputs (host side).

There is no external dataset: every configuration is a mesh + temporal
partition + right-hand side built here:

* c1: unit square 32x32 (M_x=961), uniform N_t=32, T=1, rhs ~ N(0,1) seed 0
* c2: L-shape level 5 (M_x=12,033), N_t=128, u = sin(pi x) sin(pi y) t^2
* c3: unit square 256x256 (M_x=65,025), N_t=256, rhs ~ N(0,1) seed 0
* c4: unit square 512x512 (M_x=261,121), N_t=1024, u = sin(pi x) sin(2 pi y) sin(pi t)

Seeded load vectors use numpy default_rng(0).standard_normal(N_t*M_x) in
reference order (reference idiom, tests/test_solvers.py:97-98). j_max is the
reference default 2e6 (temporal.py:40) unless overridden (tests use less).
* c5: unit square 128x128 with P2 in space (M_x=65,025), P2 in time on 512
  cells graded toward t=0 (t_i = (i/512)^2, 1024 temporal dofs), rhs ~ N(0,1)
  seed 0. The reference has no P2 discretization: `p2.py` builds it and pins
  it to the reference's P1 assembly through the exact P1-in-P2 embedding.
"""

import numpy as np

from . import fem, meshes, temporal
from .solvers import SpaceTimeSystem

CONFIGS = {
    "c1": dict(mesh=("square", 32), n_t=32, rhs="seeded"),
    "c2": dict(mesh=("lshape", 5), n_t=128, rhs="sin_sin_t2"),
    "c3": dict(mesh=("square", 256), n_t=256, rhs="seeded"),
    "c4": dict(mesh=("square", 512), n_t=1024, rhs="sin_sin2_sint"),
    "c5": dict(mesh=("square", 128), n_t=512, rhs="seeded", degree=2, grading=2.0),
}


def spatial_mesh(kind, size):
    if kind == "square":
        return meshes.build_square_mesh(size)
    if kind == "lshape":
        return meshes.build_lshape_mesh(size)
    raise ValueError(kind)


def build_system(name=None, *, mesh=None, n_t=None, rhs="seeded", j_max=temporal.DEFAULT_J_MAX,
                 temporal_device=None, seed=0, nodes=None, degree=1, grading=1.0):
    """Returns (SpaceTimeSystem, info dict).

    ``n_t`` is the number of temporal cells; with ``degree=2`` (P2 in space
    and time, `p2.py`) the system has 2 n_t temporal dofs. ``grading`` g
    places the nodes at t_i = (i / n_t)^g unless ``nodes`` is given.
    """
    if name is not None:
        cfg = CONFIGS[name]
        mesh, n_t, rhs = cfg["mesh"], cfg["n_t"], cfg["rhs"]
        degree, grading = cfg.get("degree", 1), cfg.get("grading", 1.0)
    mesh_x = spatial_mesh(*mesh)
    if nodes is None:
        nodes = (np.arange(n_t + 1) / n_t) ** grading if grading != 1.0 else np.linspace(0.0, 1.0, n_t + 1)
    mesh_t = temporal.TemporalMesh(nodes)
    if degree == 1:
        ops = fem.assemble_p1(mesh_x)
        temp = temporal.assemble_temporal_operators(mesh_t, j_max=j_max, device=temporal_device)
    elif degree == 2:
        from . import p2

        if rhs != "seeded":
            raise ValueError("P2 systems take a seeded load vector")
        ops = p2.assemble_p2(mesh_x)
        temp = p2.assemble_temporal_operators_p2(mesh_t, j_max=j_max, device=temporal_device)
    else:
        raise ValueError(f"degree must be 1 or 2, got {degree}")
    n_t = temp.A.shape[0]
    m_x = ops.n_interior
    if rhs == "seeded":
        f = np.random.default_rng(seed).standard_normal(n_t * m_x)
    elif rhs == "sin_sin_t2":
        # u = sin(pi x) sin(pi y) t^2 -> f = u_t - lap u = (2t + 2 pi^2 t^2) S
        F = fem.project_rhs_separable(
            mesh_x, mesh_t, lambda x, y: np.sin(np.pi * x) * np.sin(np.pi * y),
            lambda t: 2.0 * t + 2.0 * np.pi**2 * t**2, quad_order=6)
        f = fem.assemble_global_rhs(F, ops, temp)
    elif rhs == "sin_sin2_sint":
        # u = sin(pi x) sin(2 pi y) sin(pi t) -> f = (pi cos(pi t) + 5 pi^2 sin(pi t)) S
        F = fem.project_rhs_separable(
            mesh_x, mesh_t, lambda x, y: np.sin(np.pi * x) * np.sin(2.0 * np.pi * y),
            lambda t: np.pi * np.cos(np.pi * t) + 5.0 * np.pi**2 * np.sin(np.pi * t), quad_order=6)
        f = fem.assemble_global_rhs(F, ops, temp)
    else:
        raise ValueError(f"unknown rhs kind {rhs!r}")
    system = SpaceTimeSystem(temporal=temp, spatial=ops, rhs=np.ascontiguousarray(f))
    info = {"m_x": m_x, "n_t": n_t, "dof": m_x * n_t, "mesh": f"{mesh[0]}-{mesh[1]}", "rhs": rhs,
            "j_max": j_max, "degree": degree, "grading": grading}
    return system, info
