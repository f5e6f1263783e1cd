"""Golden bs-real outputs: the reference's own `solve_bs_real` (solvers.py:226-301)
run on the systems already stored in the golden fixtures (run in the build
container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_bsreal.py

The inputs are read back from lshape0/odd/random_*/c1.npz (byte-identical
operators), wrapped in the reference's SpaceTimeSystem and solved by the
reference; bsreal.npz stores `<fixture>_bsr` (coefficients) and
`<fixture>_bsr_residual` / `_min_re_lambda` / `_analyze_calls` (report).
"""

import os

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))

from kronheat import solvers as ks  # noqa: E402  (the reference)

FIXTURES = ("lshape0", "odd", "random_11", "random_12", "random_13", "c1")


class _Temporal:
    def __init__(self, A, M, C):
        self.A, self.M, self.C = A, M, C

    @property
    def n(self):
        return self.A.shape[0]


class _Spatial:
    def __init__(self, M, A):
        self.M_II, self.A_II = M, A

    @property
    def n_interior(self):
        return self.M_II.shape[0]


def _csr(z, p):
    return sp.csr_matrix((z[f"{p}_data"], z[f"{p}_indices"], z[f"{p}_indptr"]), shape=tuple(z[f"{p}_shape"]))


def main():
    out = {}
    for name in FIXTURES:
        z = np.load(os.path.join(HERE, f"{name}.npz"))
        s = ks.SpaceTimeSystem(temporal=_Temporal(z["A_t"], z["M_t"], z["C_t"]),
                               spatial=_Spatial(_csr(z, "M_x"), _csr(z, "A_x")), rhs=z["rhs"])
        sol, rep = ks.solve_bs_real(s)
        out[f"{name}_bsr"] = sol.coefficients
        for k in ("residual", "min_re_lambda", "analyze_calls"):
            out[f"{name}_bsr_{k}"] = np.array(getattr(rep, k))
        print(name, rep.residual, rep.analyze_calls)
    np.savez_compressed(os.path.join(HERE, "bsreal.npz"), **out)


if __name__ == "__main__":
    main()
