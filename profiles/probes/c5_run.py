"""c5 (P2 space x P2 graded time) on one GPU: assembly time, FD solve phases,
refinement history, GPU Bartels-Stewart cross-check."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np, torch
from paper_2008_01996_b200 import problems, solvers, bartels_stewart
dev = torch.device("cuda", 0)
t0 = time.perf_counter()
system, info = problems.build_system("c5", temporal_device=dev)
print("assembly %.1f s" % (time.perf_counter() - t0), info, flush=True)
print("nnz/row", system.spatial.M_II.nnz / system.m_x, flush=True)
for it in range(2):
    t0 = time.perf_counter()
    sol, rep = solvers.solve_fd(system)
    t1 = time.perf_counter()
    print(f"FD total {t1-t0:.3f} s dof/s {system.dof/(t1-t0):.3e} residual {rep.residual:.2e} fd_residual {rep.fd_residual:.2e} "
          f"steps {rep.refine_steps} minRe {rep.min_re_lambda:.3e} decompose {rep.t_decompose:.3f} spatial {rep.t_spatial:.3f} refine {rep.t_refine:.3f} | "
          + " ".join(f"{k} {v:.3f}" for k, v in rep.phases.items()), flush=True)
print("kappa2 %.3e" % rep.kappa2, flush=True)
t0 = time.perf_counter()
bs, rbs = bartels_stewart.solve_bs_complex(system)
t1 = time.perf_counter()
d = np.linalg.norm(bs.coefficients - sol.coefficients) / np.linalg.norm(bs.coefficients)
print(f"BS total {t1-t0:.2f} s residual {rbs.residual:.2e} rel diff FD vs BS {d:.2e}", flush=True)
