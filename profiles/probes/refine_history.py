"""Residual history of the refined FD solve for a config (default c4)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np, torch
from paper_2008_01996_b200 import problems, solvers
from paper_2008_01996_b200.engine import FDEngine, modal_plan
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
refine = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda", 0)
system, info = problems.build_system(cfg, temporal_device=dev)
pencil = solvers.build_pencil(system.temporal, "fd")
print(cfg, "kappa2", pencil.form.sigma[0] / pencil.form.sigma[-1])
modal = modal_plan(system.temporal, pencil)
eng = FDEngine(system.spatial.M_II, system.spatial.A_II, modal, device=dev)
print("keep_factors", eng.keep_factors, "batch", eng.batch)
F = torch.from_numpy(np.ascontiguousarray(system.rhs)).to(dev).view(system.n_t, system.m_x)
U, inf = eng.solve(F, refine=refine, tol=1e-15)
print("residuals", ["%.3e" % r for r in inf["residuals"]])
if len(sys.argv) > 3 and sys.argv[3] == "host":
    # the same solution's residual evaluated on the host (numpy/scipy, other rounding)
    import time
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "oracle"))
    u = U.reshape(-1).cpu().numpy()
    t0 = time.time()
    n, nt = system.m_x, system.n_t
    Um = u.reshape(n, nt, order="F")
    KU = system.spatial.M_II @ (Um @ system.temporal.A.T) + system.spatial.A_II @ (Um @ system.temporal.M.T)
    r = np.linalg.norm(system.rhs.reshape(n, nt, order="F") - KU) / np.linalg.norm(system.rhs)
    print("host residual (numpy/scipy) %.3e  (%.1f s)" % (r, time.time() - t0))
    print("gpu residual of the same u %.3e" % solvers.residual(system, u))
