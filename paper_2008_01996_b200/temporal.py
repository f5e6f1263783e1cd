"""Temporal H_T matrices A_t, M_t, C_t (host input generator).

Restates reference `pkg/src/kronheat/temporal.py:98-151, 300-329`: the hat
functions are expanded in the sine basis sin(theta_j t/T), theta_j = pi/2+j*pi,
and the three matrices are truncated series

    A[l,k] = 1/2 sum_j theta_j a[k][j] a[l][j]      (SPD, assembled as a SYRK)
    M[l,k] =     sum_j a[l][j] b[k][j]              (nonsymmetric)
    C[k,l] =     sum_j a[k][j] d[l][j]

accumulated over frequency chunks of 32768 in descending j (temporal.py:236-238).

`device` selects where the chunk products run: None = numpy/BLAS on the host
(the reference's own route), or a torch CUDA device for large N_t, where the
host route costs minutes. Either way this runs once
per problem, outside the timed solve.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

DEFAULT_J_MAX = 2_000_000
_CHUNK = 1 << 15


@dataclass(frozen=True)
class TemporalMesh:
    """Partition 0 = t_0 < ... < t_N = T (reference temporal.py:47-89)."""

    nodes: np.ndarray

    def __post_init__(self):
        nodes = np.asarray(self.nodes, dtype=float)
        if nodes.ndim != 1 or nodes.size < 2:
            raise ValueError("need at least two nodes")
        if nodes[0] != 0.0:
            raise ValueError("mesh must start at t = 0")
        if not np.all(np.diff(nodes) > 0):
            raise ValueError("nodes must be strictly increasing")
        nodes = nodes.copy()
        nodes.flags.writeable = False
        object.__setattr__(self, "nodes", nodes)

    @property
    def T(self):
        return float(self.nodes[-1])

    @property
    def n_cells(self):
        return len(self.nodes) - 1

    @property
    def h(self):
        return np.diff(self.nodes)


def refine_bisect(mesh):
    mids = 0.5 * (mesh.nodes[:-1] + mesh.nodes[1:])
    return TemporalMesh(np.sort(np.concatenate([mesh.nodes, mids])))


@dataclass(frozen=True)
class TemporalOperators:
    """Dense temporal matrices (reference temporal.py:196-207)."""

    A: np.ndarray
    M: np.ndarray
    C: np.ndarray
    j_max: int

    @property
    def n(self):
        return self.A.shape[0]


def _slope_bracket(xp, vals, h):
    """(v_l - v_{l-1})/h_l - (v_{l+1} - v_l)/h_{l+1}; last row keeps only the
    first slope (reference temporal.py:118-126)."""
    d = (vals[1:] - vals[:-1]) / h[:, None]
    out = d.clone() if xp is not np else d.copy()
    out[:-1] -= d[1:]
    return out


def _is_cuda(device):
    return device is not None and str(device).startswith("cuda")


def assemble_native(nodes, degree, j_max, device):
    """A, M, C from the hand-written CUDA assembly (csrc/temporal.cu,
    kh_ht_assemble) on a CUDA `device`; returned as host arrays with A's lower
    triangle mirrored like the reference's dsyrk (temporal.py:325-328)."""
    import torch

    from . import _native

    _native.load()
    dev = torch.device(device)
    nodes = np.array(nodes, dtype=np.float64)  # writable copy for torch
    n_cells = len(nodes) - 1
    nr = degree * n_cells
    need = ctypes.c_int64()
    _native.call("kh_ht_workspace_bytes", int(degree), int(n_cells), ctypes.byref(need))
    with torch.cuda.device(dev):
        d_nodes = torch.from_numpy(nodes).to(dev)
        A = torch.empty((nr, nr), dtype=torch.float64, device=dev)      # column-major storage
        M = torch.empty_like(A)
        C = torch.empty((n_cells, nr), dtype=torch.float64, device=dev)
        ws = torch.empty(int(need.value), dtype=torch.uint8, device=dev)
        _native.call("kh_ht_assemble", int(degree), int(n_cells), d_nodes.data_ptr(), int(j_max), A.data_ptr(),
                     M.data_ptr(), C.data_ptr(), ws.data_ptr(), int(need.value), _native.stream_handle())
        A, M, C = (x.T.cpu().numpy() for x in (A, M, C))
    low = np.tril(A)
    return np.ascontiguousarray(low + np.tril(low, -1).T), np.ascontiguousarray(M), np.ascontiguousarray(C)


def assemble_temporal_operators(mesh, j_max=DEFAULT_J_MAX, device=None):
    """P1 temporal H_T matrices. ``device`` None: numpy/BLAS on the host (the
    reference's route); a CUDA device: the hand-written kernels of
    csrc/temporal.cu; another torch device (e.g. "cpu"): the same series in
    torch ops (kept to cross-check the chunk arithmetic)."""
    if j_max < 0:
        raise ValueError("j_max must be >= 0")
    if _is_cuda(device):
        A, M, C = assemble_native(mesh.nodes, 1, j_max, device)
        return TemporalOperators(A=A, M=M, C=C, j_max=int(j_max))
    nodes = np.asarray(mesh.nodes, dtype=float)
    T = float(nodes[-1])
    n = len(nodes) - 1
    starts = range((j_max // _CHUNK) * _CHUNK, -1, -_CHUNK)
    if device is None:
        xp = np
        nd = nodes
        h = np.diff(nodes)
        triA = np.zeros((n, n))
        M = np.zeros((n, n))
        C = np.zeros((n, n))
    else:
        import torch
        xp = torch
        nd = torch.tensor(nodes, dtype=torch.float64, device=device)
        h = nd[1:] - nd[:-1]
        triA = torch.zeros((n, n), dtype=torch.float64, device=device)
        M = torch.zeros_like(triA)
        C = torch.zeros_like(triA)
    for j0 in starts:
        j1 = min(j0 + _CHUNK, j_max + 1)
        if xp is np:
            j = np.arange(j0, j1)
            theta = np.pi * (j + 0.5)
            arg = np.outer(nd, theta / T)
            s, c = np.sin(arg), np.cos(arg)
            sign = np.where(j % 2 == 0, 1.0, -1.0)
        else:
            j = torch.arange(j0, j1, device=device, dtype=torch.float64)
            theta = np.pi * (j + 0.5)
            arg = torch.outer(nd, theta / T)
            s, c = torch.sin(arg), torch.cos(arg)
            sign = 1.0 - 2.0 * torch.remainder(j, 2.0)
        a = _slope_bracket(xp, s, h) * (2.0 * T / theta**2)
        b = _slope_bracket(xp, c, h) * (T**2 / theta**2)
        b[n - 1] += sign * T / theta
        d = (s[1:] - s[:-1]) * (T / theta)
        w = a * xp.sqrt(theta)
        triA += 0.5 * (w @ w.T)
        M += a @ b.T
        C += a @ d.T
    if xp is not np:
        triA, M, C = (x.cpu().numpy() for x in (triA, M, C))
    # the reference accumulates only the lower triangle (dsyrk) and mirrors it,
    # so A is exactly symmetric
    low = np.tril(triA)
    A = low + np.tril(low, -1).T
    return TemporalOperators(A=A, M=M, C=C, j_max=int(j_max))
