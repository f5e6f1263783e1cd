import numpy as np, sys, time, os
sys.path.insert(0,'/root/repo')
os.environ["KH_ANALYZE_TIMING"]="1"
from paper_2008_01996_b200 import problems, sparse_direct as sd
system,_ = problems.build_system(mesh=("square",256), n_t=8, rhs="seeded", j_max=1000)
for _ in range(3):
    t=time.perf_counter()
    sym = sd.analyze(system.spatial.M_II, 24, union_with=system.spatial.A_II)
    t1=time.perf_counter()
    al = (sym.align_values(system.spatial.M_II), sym.align_values(system.spatial.A_II))
    t2=time.perf_counter()
    sd.plan_bytes(sym,1,1)
    t3=time.perf_counter()
    print("analyze %.1f align %.1f sched %.1f ms"%((t1-t)*1e3,(t2-t1)*1e3,(t3-t2)*1e3))
