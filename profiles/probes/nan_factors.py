"""Which factor panels hold non-finite lower-part entries after a factorization
on a NaN-poisoned workspace (KH_POISON=1)? Debug probe for uninitialized reads."""
import ctypes
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch  # noqa: E402

from paper_2008_01996_b200 import _native, fem, problems  # noqa: E402
from paper_2008_01996_b200 import sparse_direct as sd  # noqa: E402

mesh = ("square", int(sys.argv[1]) if len(sys.argv) > 1 else 64)
ops = fem.assemble_p1(problems.spatial_mesh(*mesh))
M, A = ops.M_II.tocsr(), ops.A_II.tocsr()
rng = np.random.default_rng(3)
lam = rng.uniform(0.01, 3.0, 9) + 1j * rng.uniform(-40.0, 40.0, 9)
sym = sd.analyze((M + A).tocsr())
plan = sd._Plan(sym, sym.align_values(M), sym.align_values(A), 4, 9, torch.cuda.current_device())
st = _native.stream_handle()
for s0 in range(0, 9, 4):
    plan.factor(s0, lam[s0:s0 + 4], st)
torch.cuda.synchronize()
ptr = ctypes.c_void_p()
tot = ctypes.c_int64()
_native.call("kh_plan_factor_storage", plan.raw, ctypes.byref(ptr), ctypes.byref(tot))
first, p, q, par, dep, rows = sym.fronts()
m = p + q
nel = 9 * tot.value * 2
buf = torch.empty(nel, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
ctypes.CDLL(None)  # noqa
cudart = torch.cuda.cudart()
# copy raw device memory into buf
import cuda.bindings.runtime as rt  # noqa: E402
rt.cudaMemcpy(buf.data_ptr(), ptr.value, nel * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
h = buf.cpu().numpy().view(np.complex128).reshape(9, tot.value)
off = np.concatenate([[0], np.cumsum(m.astype(np.int64) * p)])
bad = {}
for s in range(9):
    for f in range(len(p)):
        P = h[s, off[f]:off[f + 1]].reshape(p[f], m[f]).T  # column-major m x p
        low = np.tril(P[:, :]) if True else P
        mask = np.tril(np.ones((m[f], p[f]), bool))
        if not np.all(np.isfinite(P[mask])):
            bad.setdefault(s, []).append((f, int(dep[f]), int(m[f]), int(p[f])))
for s in sorted(bad):
    print("slot", s, "bad fronts", len(bad[s]), bad[s][:8])
print("max depth", dep.max(), "checked", len(p), "fronts")
n = M.shape[0]
B = rng.standard_normal((n, 9)) + 1j * rng.standard_normal((n, 9))
bre = torch.tensor(np.ascontiguousarray(B.real.T), device="cuda")
bim = torch.tensor(np.ascontiguousarray(B.imag.T), device="cuda")
for order in ([0, 4, 8], [4, 0, 8], [4, 4, 0]):
    xre, xim = torch.full_like(bre, 7.0), torch.full_like(bim, 7.0)
    for s0 in order:
        c = min(4, 9 - s0)
        plan.solve(s0, c, bre.data_ptr() + 8 * s0 * n, bim.data_ptr() + 8 * s0 * n, n,
                   xre.data_ptr() + 8 * s0 * n, xim.data_ptr() + 8 * s0 * n, n, st)
        torch.cuda.synchronize()
        X = xre.cpu().numpy().T
        print("order", order, "after s0", s0, "nan shifts", [k for k in range(9) if not np.all(np.isfinite(X[:, k]))])
