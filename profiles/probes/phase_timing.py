"""Per-phase cycle counts of factor_front_kernel (clock64, debug builds).

    python profiles/probes/phase_timing.py build [v..]    # here: compile variants
    python profiles/probes/phase_timing.py run <variant>  # GPU box: c3 factor

Variants differ only in compile-time switches; each prints, per front class,
the average cycles per CTA of: index staging, assembly (originals +
children), blocked LDL^T, write-out, and the factorization time per step.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

VARIANTS = {
    "default": [],
    "nola": ["KH_LOOKAHEAD_MIN_NW=99"],
    "allla": ["KH_LOOKAHEAD_MIN_NW=1"],
    "f32b10": ["KH_F32_MINB=10"],
    "f32b12": ["KH_F32_MINB=12"],
}


def lib_path(v):
    return os.path.join(HERE, f"libkh_phase_{v}.so")


def build(only=()):
    from paper_2008_01996_b200 import build as b

    for v, d in VARIANTS.items():
        if only and v not in only:
            continue
        b.build(out=lib_path(v), defines=["KH_PHASE_TIMING", *d])
        print("built", lib_path(v))


def run(v):
    import ctypes

    import numpy as np
    import torch

    from paper_2008_01996_b200 import _native, problems, solvers
    from paper_2008_01996_b200.engine import FDEngine, modal_plan

    _native.LIB_PATH = lib_path(v)
    lib = _native.load()
    fn = lib.kh_debug_phase_cycles
    fn.argtypes = [ctypes.c_void_p]
    dev = torch.device("cuda", 0)
    system, _ = problems.build_system("c3", temporal_device=dev)
    modal = modal_plan(system.temporal, solvers.build_pencil(system.temporal, "fd"))
    eng = FDEngine(system.spatial.M_II, system.spatial.A_II, modal, device=dev)
    buf = np.zeros(72, dtype=np.uint64)
    wbuf = np.zeros(64, dtype=np.uint64)
    wfn = lib.kh_debug_wphase_cycles
    wfn.argtypes = [ctypes.c_void_p]
    times = []
    for it in range(4):
        eng.factored = False
        ev = []
        eng.factor(events=ev)
        torch.cuda.synchronize()
        times.append(ev[0][0].elapsed_time(ev[0][1]))
        if it == 0:
            fn(buf.ctypes.data)  # discard warm-up counts
            wfn(wbuf.ctypes.data)
    fn(buf.ctypes.data)
    wfn(wbuf.ctypes.data)
    print(f"variant {v}: factor ms/step {np.mean(times[1:]):.2f}")
    names = ["staging", "assembly", "ldlt", "write", "(a)", "(b)", "(c)"]
    for ms in (2, 3, 4, 6, 8):
        row = buf[ms * 8: ms * 8 + 8].astype(float)
        n = row[7]
        if n == 0:
            continue
        parts = " ".join(f"{nm}={row[i] / n:6.0f}" for i, nm in enumerate(names))
        print(f"  MS={ms * 16:3d} CTAs={int(n):7d} cycles/CTA: {parts} total={row[:4].sum() / n:8.0f}")
    wnames = ["setup", "originals", "children", "ldlt", "write"]
    for mt in (4, 5, 6):
        row = wbuf[mt * 8: mt * 8 + 8].astype(float)
        n = row[7]
        if n == 0:
            continue
        parts = " ".join(f"{nm}={row[i] / n:6.0f}" for i, nm in enumerate(wnames))
        print(f"  warp MT={mt} warps={int(n):7d} cycles/warp: {parts} total={row[:5].sum() / n:8.0f}")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2])
