"""Generate golden fixtures from the reference package (run in the build
container, where /root/reference exists; the fixtures travel, the reference
does not).

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tests/golden/make_golden.py

Every fixture stores the reference's INPUTS next to its OUTPUTS, so the GPU
tests feed byte-identical operators to both implementations:

* lshape0.npz  -- reference test problem make_problem(level=0) (test_solvers.py:41-51):
                  solve_fd, solve_bs_complex, solve_dense_oracle, report stats
* odd.npz      -- three uniform cells (one real eigenvalue; test_solvers.py:217-229)
* random_<s>.npz -- random_system(n_t=6, m_x=7, seed=s) for s in 11, 12, 13 (test_solvers.py:288-298)
* c1.npz       -- BASELINE config 1 (32x32 unit square, N_t=32, seeded rhs), reference
                  solve_fd (+ report) and solve_bs_complex
* temporal.npz -- assemble_temporal_operators on a graded N_t=8 mesh (j_max=1e5) and a
                  uniform N_t=32 mesh (j_max=2e6)
* p1.npz       -- assemble_p1 on the L-shape level 2 and the 8x8 unit square
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import kronheat as kh  # noqa: E402  (the reference)
from kronheat import solvers as ks  # noqa: E402
from paper_2008_01996_b200 import meshes as my_meshes  # noqa: E402  (square lattice arrays only)

BASE_NODES = (0.0, 1.0 / 32.0, 1.0 / 16.0, 1.0 / 8.0, 1.0 / 2.0)


def csr_fields(prefix, M):
    M = sp.csr_matrix(M)
    return {f"{prefix}_data": M.data, f"{prefix}_indices": M.indices, f"{prefix}_indptr": M.indptr,
            f"{prefix}_shape": np.array(M.shape)}


def system_fields(system):
    d = {"A_t": system.temporal.A, "M_t": system.temporal.M, "C_t": system.temporal.C, "rhs": system.rhs}
    d.update(csr_fields("M_x", system.spatial.M_II))
    d.update(csr_fields("A_x", system.spatial.A_II))
    return d


def report_fields(prefix, rep):
    return {f"{prefix}_{k}": np.array(getattr(rep, k)) for k in
            ("residual", "min_re_lambda", "sigma_min", "sigma_max", "kappa2", "analyze_calls")}


def solve_all(system, dense=False):
    out = {}
    sol, rep = ks.solve_fd(system)
    out["fd"] = sol.coefficients
    out.update(report_fields("fd", rep))
    sol, rep = ks.solve_bs_complex(system)
    out["bs"] = sol.coefficients
    out.update(report_fields("bs", rep))
    if dense:
        out["dense"] = ks.solve_dense_oracle(system).coefficients
    return out


def make_problem(level=0, j_max=100_000):
    mesh_x = kh.build_lshape_mesh(level)
    mesh_t = kh.TemporalMesh(np.array(BASE_NODES))
    ops = kh.assemble_p1(mesh_x)
    temp = kh.assemble_temporal_operators(mesh_t, j_max=j_max)
    F = kh.project_rhs(mesh_x, mesh_t, kh.manufactured.source_f, quad_order=4)
    lift = kh.dirichlet_lift(mesh_x, mesh_t, kh.manufactured.exact_u)
    rhs = kh.assemble_global_rhs(F, ops, temp, lift=lift)
    return ks.SpaceTimeSystem(temporal=temp, spatial=ops, rhs=rhs)


def square_ops(n):
    m = my_meshes.build_square_mesh(n)
    return kh.assemble_p1(kh.TriangleMesh(m.vertices, m.triangles, m.boundary_flags))


def main():
    # reference test problem, level 0
    s = make_problem(0)
    np.savez_compressed(os.path.join(HERE, "lshape0.npz"), **system_fields(s), **solve_all(s, dense=True))

    # odd number of cells: one real eigenvalue
    mesh_x = kh.build_lshape_mesh(0)
    mesh_t = kh.TemporalMesh(np.linspace(0.0, 0.5, 4))
    ops = kh.assemble_p1(mesh_x)
    temp = kh.assemble_temporal_operators(mesh_t, j_max=100_000)
    F = kh.project_rhs(mesh_x, mesh_t, kh.manufactured.source_f, quad_order=4)
    lift = kh.dirichlet_lift(mesh_x, mesh_t, kh.manufactured.exact_u)
    s = ks.SpaceTimeSystem(temporal=temp, spatial=ops, rhs=kh.assemble_global_rhs(F, ops, temp, lift=lift))
    np.savez_compressed(os.path.join(HERE, "odd.npz"), **system_fields(s), **solve_all(s, dense=True))

    # random systems of the reference suite
    import test_solvers as ts  # reference tests (helpers only)

    for seed in (11, 12, 13):
        s = ts.random_system(n_t=6, m_x=7, seed=seed)
        np.savez_compressed(os.path.join(HERE, f"random_{seed}.npz"), **system_fields(s),
                            **solve_all(s, dense=True))

    # BASELINE config 1
    ops = square_ops(32)
    temp = kh.assemble_temporal_operators(kh.TemporalMesh(np.linspace(0.0, 1.0, 33)))
    rhs = np.random.default_rng(0).standard_normal(32 * ops.n_interior)
    s = ks.SpaceTimeSystem(temporal=temp, spatial=ops, rhs=rhs)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **system_fields(s), **solve_all(s))

    # temporal assembly
    g = kh.TemporalMesh(np.array(BASE_NODES))
    g = kh.refine_bisect(g)
    t8 = kh.assemble_temporal_operators(g, j_max=100_000)
    t32 = kh.assemble_temporal_operators(kh.TemporalMesh(np.linspace(0.0, 1.0, 33)))
    np.savez_compressed(os.path.join(HERE, "temporal.npz"), graded8_nodes=g.nodes, graded8_A=t8.A,
                        graded8_M=t8.M, graded8_C=t8.C, uniform32_A=t32.A, uniform32_M=t32.M, uniform32_C=t32.C)

    # P1 assembly
    lo = kh.assemble_p1(kh.build_lshape_mesh(2))
    sq = square_ops(8)
    d = {}
    for name, o in (("lshape2", lo), ("square8", sq)):
        d.update(csr_fields(f"{name}_M", o.M_II))
        d.update(csr_fields(f"{name}_A", o.A_II))
        d.update(csr_fields(f"{name}_M10", o.M10))
        d[f"{name}_interior"] = o.interior
    np.savez_compressed(os.path.join(HERE, "p1.npz"), **d)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
