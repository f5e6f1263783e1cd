"""Where the end-to-end solve_fd(system) time goes at a config (default c3):
host milestones from SolveReport.phases, per-stage times, three runs.

    python profiles/probes/e2e_phases.py [c3]
"""
import dataclasses
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2008_01996_b200 import problems, solvers  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
dev = torch.device("cuda", 0)
system, info = problems.build_system(cfg, temporal_device=dev)
pinned = torch.empty(system.rhs.shape, dtype=torch.float64, pin_memory=True)
pinned.copy_(torch.from_numpy(system.rhs))
system = dataclasses.replace(system, rhs=pinned.numpy())
import os  # noqa: E402

runs = int(os.environ.get("E2E_RUNS", 4))
toggle = os.environ.get("E2E_TOGGLE")  # name of an env switch flipped 1/0 on alternate runs (A/B on one box)
for it in range(runs):
    if toggle:
        os.environ[toggle] = str(it % 2)
    t0 = time.perf_counter()
    sol, rep = solvers.solve_fd(system)
    t1 = time.perf_counter()
    print(json.dumps({"run": it, **({toggle: os.environ[toggle]} if toggle else {}), "total_ms": round(1e3 * (t1 - t0), 2),
                      "stages_ms": {k: round(1e3 * getattr(rep, k), 2) for k in
                                    ("t_decompose", "t_transform_in", "t_spatial", "t_transform_out", "t_refine")},
                      "milestones_ms": {k: round(1e3 * v, 2) for k, v in rep.phases.items()},
                      "residual": rep.residual}), flush=True)
