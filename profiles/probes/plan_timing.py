"""Where the FDEngine (plan) creation time goes at c3 (host side of e2e)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, scipy.sparse as sp, torch
from paper_2008_01996_b200 import problems, solvers, sparse_direct as sd
from paper_2008_01996_b200.engine import FDEngine, modal_plan

system, _ = problems.build_system("c3", temporal_device=torch.device("cuda", 0))
pen = solvers.build_pencil(system.temporal, "fd", eig="reduced")
modal = modal_plan(system.temporal, pen)
M, A = system.spatial.M_II, system.spatial.A_II
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sym = sd.analyze((sp.csr_matrix(M) + sp.csr_matrix(A)).tocsr())
    t1 = time.perf_counter()
    al = (sym.align_values(M), sym.align_values(A))
    t2 = time.perf_counter()
    nb = sd.plan_bytes(sym, 128, 128)
    t3 = time.perf_counter()
    plan = sd._Plan(sym, al[0], al[1], 128, 128, 0)
    t4 = time.perf_counter()
    del plan
    eng = FDEngine(M, A, modal, device=torch.device("cuda", 0), symbolic=sym, aligned=al)
    t5 = time.perf_counter()
    del eng
    print(f"analyze {1e3*(t1-t0):.1f} align {1e3*(t2-t1):.1f} plan_bytes {1e3*(t3-t2):.1f} "
          f"_Plan {1e3*(t4-t3):.1f} FDEngine {1e3*(t5-t4):.1f} ms", flush=True)
import cProfile, pstats
cProfile.run("eng = FDEngine(M, A, modal, device=torch.device('cuda', 0), symbolic=sym, aligned=al)", "/tmp/fdprof")
pstats.Stats("/tmp/fdprof").sort_stats("tottime").print_stats(12)
