import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libkhb200.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


def _csr(z, prefix):
    return sp.csr_matrix((z[f"{prefix}_data"], z[f"{prefix}_indices"], z[f"{prefix}_indptr"]),
                         shape=tuple(z[f"{prefix}_shape"]))


class _Temporal:
    def __init__(self, A, M, C):
        self.A, self.M, self.C = A, M, C

    @property
    def n(self):
        return self.A.shape[0]


class _Spatial:
    def __init__(self, M, A):
        self.M_II, self.A_II = M, A
        n = M.shape[0]
        self.interior = np.arange(n)
        self.boundary = np.empty(0, dtype=np.int64)

    @property
    def n_interior(self):
        return self.M_II.shape[0]


def load_golden(name):
    """(system, outputs dict) from a reference-generated fixture."""
    from paper_2008_01996_b200.solvers import SpaceTimeSystem

    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    system = SpaceTimeSystem(temporal=_Temporal(z["A_t"], z["M_t"], z["C_t"]),
                             spatial=_Spatial(_csr(z, "M_x"), _csr(z, "A_x")), rhs=z["rhs"])
    return system, {k: z[k] for k in z.files}


def rel_diff(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    # GPU tests never skip: a missing device or library must fail loudly
    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    from paper_2008_01996_b200 import _native

    _native.load()
    return True
