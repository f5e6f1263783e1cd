"""solve_fd(system) (pencil built inside) phase times at c3, steady state."""
import sys, os, time, dataclasses
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np, torch
from paper_2008_01996_b200 import problems, solvers
dev = torch.device("cuda", 0)
system, info = problems.build_system(sys.argv[1] if len(sys.argv) > 1 else "c3", temporal_device=dev)
pinned = torch.empty(system.rhs.shape, dtype=torch.float64, pin_memory=True)
pinned.copy_(torch.from_numpy(system.rhs))
system = dataclasses.replace(system, rhs=pinned.numpy())
for it in range(5):
    t0 = time.perf_counter()
    sol, rep = solvers.solve_fd(system)
    t1 = time.perf_counter()
    print(f"total {1e3*(t1-t0):.1f} ms: decompose {1e3*rep.t_decompose:.1f} spatial {1e3*rep.t_spatial:.1f} "
          f"tin {1e3*rep.t_transform_in:.1f} tout {1e3*rep.t_transform_out:.1f} refine {1e3*rep.t_refine:.1f} | "
          + " ".join(f"{k} {1e3*v:.1f}" for k, v in rep.phases.items()))
for eig in ("reduced", "qz"):
    t0 = time.perf_counter(); pen = solvers.build_pencil(system.temporal, "fd", eig=eig)
    print("build_pencil(%s) alone %.1f ms" % (eig, 1e3 * (time.perf_counter() - t0)))
