"""Temporal H_T assembly on the GPU: hand-written kernels (kh_ht_assemble)
vs the same series in torch ops, at the c3/c4 (P1) and c5 (P2) sizes."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np, torch
from paper_2008_01996_b200 import temporal, p2
dev = torch.device("cuda", 0)
def torch_p1(tm, j):
    # the torch-op route (device other than cuda string match): call internals directly
    return temporal.assemble_temporal_operators.__wrapped__(tm, j) if hasattr(temporal.assemble_temporal_operators, "__wrapped__") else None
for name, nodes, deg in (("c3 P1 N=256", np.linspace(0, 1, 257), 1), ("c4 P1 N=1024", np.linspace(0, 1, 1025), 1),
                         ("c5 P2 N=512 graded", (np.arange(513) / 512.0) ** 2, 2)):
    tm = temporal.TemporalMesh(nodes)
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        A, M, C = temporal.assemble_native(nodes, deg, 2_000_000, dev)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    nr = deg * (len(nodes) - 1)
    flops = 2.0 * 2_000_001 * (2 * nr * nr + nr * (len(nodes) - 1))
    print(f"{name}: native {1e3*(t1-t0):.1f} ms ({flops/(t1-t0)/1e12:.1f} TF/s incl. coefficient kernels)", flush=True)
