"""Reference-built FD pencils for the drop-in test (run where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ref_pencil.py

For the fixtures lshape0 and c1, `kronheat.solvers.build_pencil(temporal, "fd")`
(reference solvers.py:166-206) is applied to the fixture's own temporal
operators and every array of the resulting PencilFactorization / EigenSvdForm
is stored in ref_pencil.npz as <name>_<field>. tests/test_gpu_fd.py rebuilds
objects with exactly the reference's attributes from them and passes the
pencil straight into the drop-in solve_fd.
"""

import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from kronheat import solvers as ks  # noqa: E402  (the reference)

out = {}
for name in ("lshape0", "c1"):
    z = np.load(os.path.join(HERE, f"{name}.npz"))
    temporal = types.SimpleNamespace(A=z["A_t"], M=z["M_t"], C=z["C_t"])
    pencil = ks.build_pencil(temporal, "fd")
    assert type(pencil).__name__ == "PencilFactorization" and type(pencil.form).__name__ == "EigenSvdForm"
    out[f"{name}_variant"] = np.array(pencil.variant)
    out[f"{name}_chol_A"] = pencil.chol_A
    for f in ("X", "D", "U", "sigma", "Vh"):
        out[f"{name}_{f}"] = getattr(pencil.form, f)
np.savez_compressed(os.path.join(HERE, "ref_pencil.npz"), **out)
print("wrote", sorted(out))
