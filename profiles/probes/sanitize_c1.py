"""Small workload for compute-sanitizer runs (one tool per gpurun call):

    compute-sanitizer --tool memcheck  python profiles/probes/sanitize_c1.py
    compute-sanitizer --tool racecheck python profiles/probes/sanitize_c1.py

Covers the fused-front factorization (bulk smem->global writes after
fence.proxy.async), the large-front chain (square 48: fronts with m > 128),
the bulk-copy staged solves, the compensated residual and the fused GEMM +
row scatter (kh_dgemm_rowscatter into local slots) + slot sum.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2008_01996_b200 import _native, problems, solvers  # noqa: E402

torch.cuda.set_device(0)
for mesh, nt in ((("square", 32), 32), (("square", 48), 8)):
    system, _ = problems.build_system(mesh=mesh, n_t=nt, rhs="seeded", j_max=20_000)
    sol, rep = solvers.solve_fd(system)
    res_dd = solvers.residual(system, sol.coefficients, compensated=True)
    print(f"{mesh} N_t={nt}: residual {rep.residual:.2e} (compensated {res_dd:.2e}), steps {rep.refine_steps}")
    assert rep.residual < 1e-11

# fused GEMM + row scatter into two local "peer" slots, then the ordered slot sum
m, n, k, parts = 300, 40, 64, 2
rp = (m + parts - 1) // parts
A = torch.randn(k, m, dtype=torch.float64, device="cuda")   # column-major m x k
B = torch.randn(n, k, dtype=torch.float64, device="cuda")   # column-major k x n
slots = torch.zeros(parts, n, rp, dtype=torch.float64, device="cuda")
dst = torch.tensor([slots[c].data_ptr() for c in range(parts)], dtype=torch.int64, device="cuda")
st = _native.stream_handle()
_native.call("kh_dgemm_rowscatter", m, n, k, A.data_ptr(), m, B.data_ptr(), k, dst.data_ptr(), parts, rp, rp, st)
out = torch.zeros(n * rp, dtype=torch.float64, device="cuda")
_native.call("kh_sum_parts", parts, slots.data_ptr(), n * rp, out.data_ptr(), st)
torch.cuda.synchronize()
C = (A.T.cpu().numpy() @ B.T.cpu().numpy())
got = np.concatenate([slots[c].cpu().numpy().T[: min(rp, m - c * rp)] for c in range(parts)])
assert np.allclose(got, C, rtol=1e-12, atol=1e-12)
print("rowscatter ok")
