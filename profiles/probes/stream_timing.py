"""Where a CTA of fwd_stream_kernel spends its cycles (clock64 of thread 0,
debug build with -DKH_STREAM_TIMING), per tree level of one c3 solve.

    python profiles/probes/stream_timing.py build   # here
    python profiles/probes/stream_timing.py run     # GPU box
"""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libkh_stream_timing.so")

if sys.argv[1] == "build":
    from paper_2008_01996_b200 import build as b

    b.build(out=LIB, defines=["KH_STREAM_TIMING"])
    print("built", LIB)
else:
    import numpy as np
    import torch

    os.environ.setdefault("KH_SOLVE_LANES", "1")
    from paper_2008_01996_b200 import _native, problems, solvers
    from paper_2008_01996_b200.engine import FDEngine, modal_plan

    _native.LIB_PATH = LIB
    lib = _native.load()
    fn = lib.kh_debug_stream_cycles
    fn.argtypes = [ctypes.c_void_p]
    dev = torch.device("cuda", 0)
    system, _ = problems.build_system("c3", temporal_device=dev)
    modal = modal_plan(system.temporal, solvers.build_pencil(system.temporal, "fd"))
    eng = FDEngine(system.spatial.M_II, system.spatial.A_II, modal, device=dev)
    F = torch.from_numpy(np.asarray(system.rhs)).to(dev).view(system.n_t, system.m_x)
    U, info = eng.solve(F, refine=1)
    torch.cuda.synchronize()
    buf = np.zeros(8, dtype=np.uint64)
    fn(buf.ctypes.data)  # reset
    eng.fd_apply(eng.R, U, accumulate=False)  # one solve with retained factors
    torch.cuda.synchronize()
    fn(buf.ctypes.data)
    names = ["prologue", "mbar wait", "block solve", "rows", "barrier+issue"]
    ctas, stages = int(buf[6]), int(buf[5])
    print(f"CTAs {ctas}, stages {stages} ({stages / max(ctas, 1):.1f} per CTA)")
    print("prologue cycles per CTA:", int(buf[0]) // max(ctas, 1))
    for i in range(1, 5):
        print(f"{names[i]:14s} cycles per stage: {int(buf[i]) / max(stages, 1):.0f}")
