"""Host pencil cost at c3 (N_t=256): where build_pencil's time goes."""
import sys, time, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
import scipy.linalg as sla
from paper_2008_01996_b200 import problems, solvers, dense
from paper_2008_01996_b200.temporal import TemporalMesh, assemble_temporal_operators
from paper_2008_01996_b200.engine import modal_plan
tops = assemble_temporal_operators(TemporalMesh(np.linspace(0, 1, 257)))
for rep in range(2):
    t0 = time.perf_counter(); L = dense.cholesky_lower(tops.A); P = dense.spd_solve(L, tops.M); t1 = time.perf_counter()
    vals, vecs = dense.eig_pencil(tops.M, tops.A); t2 = time.perf_counter()
    res = np.linalg.norm(P @ vecs - vecs * vals[None, :], "fro"); t3 = time.perf_counter()
    form = dense.svd_of_eigenvectors(vecs, vals); t4 = time.perf_counter()
    w, v = sla.eig(P); t5 = time.perf_counter()
    C = sla.solve_triangular(L, sla.solve_triangular(L, tops.M, lower=True).T, lower=True)
    t6 = time.perf_counter(); w2, v2 = sla.eig(C); t7 = time.perf_counter()
    pen = solvers.build_pencil(tops, "fd"); t8 = time.perf_counter()
    mp = modal_plan(tops, pen); t9 = time.perf_counter()
    print(f"chol+P {1e3*(t1-t0):.1f} dggev {1e3*(t2-t1):.1f} resid {1e3*(t3-t2):.1f} svd(X) {1e3*(t4-t3):.1f} "
          f"dgeev(P) {1e3*(t5-t4):.1f} dgeev(C) {1e3*(t7-t6):.1f} build_pencil {1e3*(t8-t7):.1f} modal {1e3*(t9-t8):.1f} ms")
