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
