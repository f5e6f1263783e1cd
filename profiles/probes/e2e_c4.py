"""Where the end-to-end time of solve_fd goes at c4 (267M dofs): phases."""
import sys, os, time, dataclasses
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np, torch
from paper_2008_01996_b200 import problems, solvers
dev = torch.device("cuda", 0)
t0 = time.perf_counter()
system, info = problems.build_system(sys.argv[1] if len(sys.argv) > 1 else "c4", temporal_device=dev)
print("build %.1f s" % (time.perf_counter() - t0), flush=True)
pinned = torch.empty(system.rhs.shape, dtype=torch.float64, pin_memory=True)
pinned.copy_(torch.from_numpy(system.rhs))
system = dataclasses.replace(system, rhs=pinned.numpy())
for it in range(2):
    t0 = time.perf_counter()
    sol, rep = solvers.solve_fd(system)
    t1 = time.perf_counter()
    print(f"total {t1-t0:.2f} s: decompose {rep.t_decompose:.2f} tin {rep.t_transform_in:.2f} spatial {rep.t_spatial:.2f} "
          f"tout {rep.t_transform_out:.2f} refine {rep.t_refine:.2f} steps {rep.refine_steps} res {rep.residual:.2e} | "
          + " ".join(f"{k} {v:.2f}" for k, v in rep.phases.items()), flush=True)
