import time, dataclasses, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2008_01996_b200 import problems, solvers, sparse_direct
from paper_2008_01996_b200.engine import FDEngine, modal_plan
dev = torch.device('cuda', 0)
system, info = problems.build_system('c3', temporal_device=dev)
pencil = solvers.build_pencil(system.temporal, 'fd')
pinned = torch.empty(system.rhs.shape, dtype=torch.float64, pin_memory=True); pinned.copy_(torch.from_numpy(system.rhs))
system = dataclasses.replace(system, rhs=pinned.numpy())
for it in range(3):
    t0 = time.perf_counter()
    sol, rep = solvers.solve_fd(system, pencil=pencil)
    t1 = time.perf_counter()
    print(f"total {1e3*(t1-t0):.1f} ms: decompose {1e3*rep.t_decompose:.1f} spatial(setup+solve) {1e3*rep.t_spatial:.1f} tin {1e3*rep.t_transform_in:.1f} tout {1e3*rep.t_transform_out:.1f} refine {1e3*rep.t_refine:.1f}")
# breakdown of setup
t0=time.perf_counter(); sym = sparse_direct.analyze(system.spatial.A_II + system.spatial.M_II); t1=time.perf_counter()
print(f"analyze {1e3*(t1-t0):.1f} ms")
modal = modal_plan(system.temporal, pencil)
t0=time.perf_counter(); eng = FDEngine(system.spatial.M_II, system.spatial.A_II, modal, device=dev, symbolic=sym); torch.cuda.synchronize(); t1=time.perf_counter()
print(f"engine(plan) {1e3*(t1-t0):.1f} ms")
t0=time.perf_counter(); eng.factor(); torch.cuda.synchronize(); t1=time.perf_counter()
print(f"factor {1e3*(t1-t0):.1f} ms")
