"""Drop-in for the reference's `kronheat.sparse_direct` on the GPU.

Reference: pkg/src/kronheat/sparse_direct.py. Same entry points and error
behaviour:

* `analyze(pattern)`            -> sparse_direct.py:112-152 (one symbolic analysis,
                                   global call counter `analyze_call_count`, :21-26)
* `factorize(symbolic, matrix)` -> :155-188 (pivot guard 1e-13 * max|a| -> SingularMatrix)
* `solve(numeric, rhs, refine)` -> :191-209 (multi-column rhs, optional refinement)
* `factor_solve(matrix, rhs)`   -> :212-215

Differences by design: the symbolic phase is a host C++ nested dissection
(`csrc/symbolic.cpp`) instead of SuperLU's MMD, and the numeric phase is the
batched pivot-free complex-symmetric LDL^T on the GPU (`csrc/frontal.cu`)
instead of SuperLU LU. The matrices must therefore be (complex) symmetric --
every matrix the FD path produces is (M_x + lambda A_x with symmetric M_x, A_x).
There is no CPU fallback.
"""

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _native
from .errors import DimensionMismatch, UsageError

PIVOT_THRESHOLD = 1e-13
DEFAULT_LEAF_SIZE = 24

_analyze_calls = 0


def analyze_call_count():
    """Total number of symbolic analyses performed in this process."""
    return _analyze_calls


def symmetrized_pattern(matrix):
    """Canonical CSR (sorted, no duplicates) of the union pattern A | A^T."""
    A = sp.csr_matrix(matrix)
    if A.shape[0] != A.shape[1]:
        raise DimensionMismatch("pattern must be square")
    S = sp.csr_matrix((np.ones(A.nnz), A.indices, A.indptr), shape=A.shape)
    S = (S + S.T).tocsr()
    S.sum_duplicates()
    S.sort_indices()
    return S.indptr.astype(np.int64), S.indices.astype(np.int64)


class _Handle:
    """Owns a kh_symbolic*."""

    def __init__(self, raw):
        self.raw = raw

    def __del__(self, _native=_native):  # module globals may be gone at interpreter exit
        if self.raw and _native is not None and _native._lib is not None:
            _native._lib.kh_symbolic_free(self.raw)
            self.raw = None


@dataclass(frozen=True)
class SymbolicFactorization:
    """Nested-dissection ordering and front structure (immutable, shareable).

    ``perm`` is the symmetric permutation (perm[k] = original index eliminated
    k-th); ``factor_nnz`` counts the entries of L including the diagonal.
    """

    n: int
    perm: np.ndarray
    factor_nnz: int
    indptr: np.ndarray = field(repr=False)
    indices: np.ndarray = field(repr=False)
    stats: dict = field(repr=False, default_factory=dict)
    handle: object = field(repr=False, default=None, compare=False)

    @property
    def pattern_key(self):
        return (self.n, self.indptr.tobytes(), self.indices.tobytes())

    def fronts(self):
        """Per-front (first, npiv, nupd, parent, depth) arrays."""
        nf = int(self.stats["n_fronts"])
        first = np.zeros(nf, np.int64)
        p, q, par, dep = (np.zeros(nf, np.int32) for _ in range(4))
        _native.call("kh_symbolic_fronts", self.handle.raw, _native.ptr(first), _native.ptr(p),
                     _native.ptr(q), _native.ptr(par), _native.ptr(dep))
        rows = np.zeros(int(q.sum()), np.int64)
        _native.call("kh_symbolic_rows", self.handle.raw, _native.ptr(rows))
        return first, p, q, par, dep, rows

    def align_values(self, matrix, dtype=float):
        """Values of `matrix` on the analyzed pattern (missing entries -> 0).

        Raises DimensionMismatch if the matrix has an entry outside it.
        """
        A = sp.csr_matrix(matrix)
        if A.shape != (self.n, self.n):
            raise DimensionMismatch(f"matrix shape {A.shape} does not match analysis ({self.n})")
        if not A.has_canonical_format:
            A = A.copy()
            A.sum_duplicates()
        ip = np.ascontiguousarray(A.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(A.indices, dtype=np.int64)
        parts = [np.real(A.data)] + ([np.imag(A.data)] if np.iscomplexobj(A.data) else [])
        outs = []
        for part in parts:
            v = np.ascontiguousarray(part, dtype=np.float64)
            o = np.empty(len(self.indices), dtype=np.float64)
            _native.call("kh_align_values", self.n, _native.ptr(self.indptr), _native.ptr(self.indices),
                         _native.ptr(ip), _native.ptr(ix), _native.ptr(v), _native.ptr(o))
            outs.append(o)
        if np.dtype(dtype).kind == "c":
            return outs[0] + 1j * (outs[1] if len(outs) > 1 else 0.0)
        return outs[0]


def analyze(pattern, leaf_size=DEFAULT_LEAF_SIZE, union_with=None):
    """Symbolic analysis of a sparsity pattern (symmetrized by union first).

    ``union_with``: a second pattern of the same shape; the analysis is then of
    the union of both (the FD path's M_x + A_x, solvers.py:216-223), merged
    natively instead of summed on the host."""
    global _analyze_calls
    # the native analysis symmetrizes the pattern itself (A | A^T, diagonal
    # added, duplicates merged) and returns that canonical CSR
    A = sp.csr_matrix(pattern)
    if A.shape[0] != A.shape[1]:
        raise DimensionMismatch("pattern must be square")
    n = A.shape[0]
    in_ptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    in_idx = np.ascontiguousarray(A.indices, dtype=np.int64)
    lib = _native.load()
    raw = ctypes.c_void_p()
    if union_with is None:
        _native.check(lib.kh_analyze(n, _native.ptr(in_ptr), _native.ptr(in_idx), int(leaf_size),
                                     ctypes.byref(raw)))
    else:
        B = sp.csr_matrix(union_with)
        if B.shape != A.shape:
            raise DimensionMismatch("patterns differ in shape")
        b_ptr = np.ascontiguousarray(B.indptr, dtype=np.int64)
        b_idx = np.ascontiguousarray(B.indices, dtype=np.int64)
        _native.check(lib.kh_analyze_union(n, _native.ptr(in_ptr), _native.ptr(in_idx), _native.ptr(b_ptr),
                                           _native.ptr(b_idx), int(leaf_size), ctypes.byref(raw)))
    handle = _Handle(raw.value)
    st = _native.SymbolicStats()
    _native.check(lib.kh_symbolic_stats_get(handle.raw, ctypes.byref(st)))
    stats = {name: getattr(st, name) for name, _ in st._fields_}
    indptr = np.zeros(n + 1, np.int64)
    indices = np.zeros(int(st.nnz), np.int64)
    _native.check(lib.kh_symbolic_pattern(handle.raw, _native.ptr(indptr), _native.ptr(indices)))
    perm = np.zeros(n, np.int64)
    if n:
        _native.check(lib.kh_symbolic_perm(handle.raw, _native.ptr(perm)))
    _analyze_calls += 1
    return SymbolicFactorization(n=n, perm=perm, factor_nnz=int(st.factor_nnz), indptr=indptr,
                                 indices=indices, stats=stats, handle=handle)


class _Plan:
    """Owns a kh_plan* (device factor storage + work space)."""

    def __init__(self, symbolic, m_vals, a_vals, max_batch, slots, device):
        import torch

        self.raw = ctypes.c_void_p()
        self.symbolic = symbolic
        self.device = device
        self.max_batch = int(max_batch)
        self.slots = int(slots)
        mv = np.ascontiguousarray(m_vals, dtype=np.float64)
        av = np.ascontiguousarray(a_vals, dtype=np.float64)
        # one workspace from torch's caching allocator: repeated solves reuse
        # it without cudaMalloc/cudaFree (which would synchronize the device)
        nbytes = plan_bytes(symbolic, self.max_batch, self.slots)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", int(device)))
        if os.environ.get("KH_POISON"):  # debugging: NaN-fill the workspace (uninitialized reads show up)
            self.workspace.fill_(255)
        _native.call("kh_plan_create", symbolic.handle.raw, int(device), _native.ptr(symbolic.indptr),
                     _native.ptr(symbolic.indices), _native.ptr(mv), _native.ptr(av), self.max_batch,
                     self.slots, self.workspace.data_ptr(), nbytes, ctypes.byref(self.raw))

    def factor(self, slot0, lambdas, stream):
        lam = np.ascontiguousarray(np.asarray(lambdas, dtype=np.complex128))
        _native.call("kh_plan_factor", self.raw, int(slot0), len(lam), _native.ptr(lam), stream)

    def factor_solve(self, slot0, lambdas, b_re, b_im, ldb, x_re, x_im, ldx, stream):
        """factor + solve of one batch, forward sweep fused into the factorization."""
        lam = np.ascontiguousarray(np.asarray(lambdas, dtype=np.complex128))
        _native.call("kh_plan_factor_solve", self.raw, int(slot0), len(lam), _native.ptr(lam), b_re, b_im, int(ldb),
                     x_re, x_im, int(ldx), stream)

    def set_level_timing(self, on):
        _native.call("kh_plan_set_level_timing", self.raw, int(bool(on)))

    def level_times(self):
        """Milliseconds per tree level (index = depth, 0 = root) of the most
        recent factorization (after set_level_timing(True))."""
        nl = int(self.symbolic.stats["depth"]) + 1
        out = np.zeros(nl, dtype=np.float32)
        _native.call("kh_plan_level_times", self.raw, out.ctypes.data, nl)
        return out.astype(np.float64)

    def factor_fwd(self, slot0, lambdas, b_re, b_im, ldb, stream):
        lam = np.ascontiguousarray(np.asarray(lambdas, dtype=np.complex128))
        _native.call("kh_plan_factor_fwd", self.raw, int(slot0), len(lam), _native.ptr(lam), b_re, b_im, int(ldb),
                     stream)

    def solve_bwd(self, slot0, nshift, x_re, x_im, ldx, stream):
        _native.call("kh_plan_solve_bwd", self.raw, int(slot0), int(nshift), x_re, x_im, int(ldx), stream)

    def pivot_check(self, slot0, nshift, stream, threshold=PIVOT_THRESHOLD):
        _native.call("kh_plan_pivot_check", self.raw, int(slot0), int(nshift), float(threshold), stream,
                     None, None)

    def solve(self, slot0, nshift, b_re, b_im, ldb, x_re, x_im, ldx, stream):
        _native.call("kh_plan_solve", self.raw, int(slot0), int(nshift), b_re, b_im, int(ldb), x_re, x_im,
                     int(ldx), stream)

    def residual(self, nt, Y, ldy, F, ldf, R, ldr, norms2, stream):
        _native.call("kh_plan_residual", self.raw, int(nt), Y, int(ldy), F, int(ldf), R, int(ldr), norms2,
                     stream)

    def residual_scale(self, nt, Y, ldy, F, ldf, norms2, stream):
        _native.call("kh_plan_residual_scale", self.raw, int(nt), Y, int(ldy), F, int(ldf), norms2, stream)

    def residual_dd(self, nt, Y1, ldy1, Y2hi, Y2lo, ldy2, F, ldf, R, ldr, norms2, stream):
        _native.call("kh_plan_residual_dd", self.raw, int(nt), Y1, int(ldy1), Y2hi, Y2lo, int(ldy2), F, int(ldf),
                     R, int(ldr), norms2, stream)

    def __del__(self, _native=_native):
        if getattr(self, "raw", None) and self.raw.value and _native is not None and _native._lib is not None:
            _native._lib.kh_plan_free(self.raw)
            self.raw = ctypes.c_void_p()


def plan_bytes(symbolic, max_batch, slots):
    out = ctypes.c_int64()
    _native.call("kh_plan_bytes", symbolic.handle.raw, int(max_batch), int(slots), ctypes.byref(out))
    return int(out.value)


def _check_symmetric(A):
    A = sp.csr_matrix(A)
    d = A - A.T
    if d.nnz and np.max(np.abs(d.data)) > 1e-14 * max(np.max(np.abs(A.data)), 1e-300):
        raise UsageError("pivot-free LDL^T needs a (complex) symmetric matrix")


class NumericFactorization:
    """LDL^T factors of one matrix on the GPU, bound to a SymbolicFactorization.

    The matrix K is stored as the shifted pair Re(K) + i * Im(K), so real and
    complex symmetric matrices go through the same batched kernels.
    """

    def __init__(self, symbolic, plan, is_complex, matrix):
        self.symbolic = symbolic
        self._plan = plan
        self.is_complex = is_complex
        self._matrix = matrix

    def solve(self, rhs, refine=False):
        return solve(self, rhs, refine=refine)


def factorize(symbolic, matrix):
    """Numeric factorization on the GPU reusing a symbolic analysis.

    Raises SingularMatrix if a pivot magnitude falls below 1e-13 times the
    largest entry (reference sparse_direct.py:182-187).
    """
    import torch

    _native.require_cuda()
    A = sp.csr_matrix(matrix)
    if A.shape != (symbolic.n, symbolic.n):
        raise DimensionMismatch(f"matrix shape {A.shape} does not match analysis ({symbolic.n})")
    _check_symmetric(A)
    is_complex = np.iscomplexobj(A.data)
    vals = symbolic.align_values(A, dtype=complex if is_complex else float)
    m_vals = np.real(vals).astype(np.float64)
    a_vals = np.imag(vals).astype(np.float64) if is_complex else np.zeros_like(m_vals)
    device = torch.cuda.current_device()
    plan = _Plan(symbolic, m_vals, a_vals, 1, 1, device)
    stream = _native.stream_handle()
    plan.factor(0, [1j if is_complex else 0.0], stream)
    plan.pivot_check(0, 1, stream)
    return NumericFactorization(symbolic, plan, is_complex, A)


def _solve_cols(numeric, B):
    import torch

    n = numeric.symbolic.n
    dev = torch.device("cuda", numeric._plan.device)
    out = np.empty(B.shape, dtype=complex if (numeric.is_complex or np.iscomplexobj(B)) else float)
    stream = _native.stream_handle()
    for j in range(B.shape[1]):
        b = B[:, j]
        b_re = torch.tensor(np.real(b), dtype=torch.float64, device=dev)
        b_im = torch.tensor(np.imag(b), dtype=torch.float64, device=dev) if np.iscomplexobj(b) else None
        x_re = torch.empty(n, dtype=torch.float64, device=dev)
        x_im = torch.empty(n, dtype=torch.float64, device=dev)
        numeric._plan.solve(0, 1, _native.ptr(b_re), _native.ptr(b_im), n, _native.ptr(x_re),
                            _native.ptr(x_im), n, stream)
        xr, xi = x_re.cpu().numpy(), x_im.cpu().numpy()
        out[:, j] = xr + 1j * xi if np.iscomplexobj(out) else xr
    return out


def solve(numeric, rhs, refine=False):
    """Solve with GPU factors; accepts multi-column rhs (reference :191-209)."""
    rhs = np.asarray(rhs)
    n = numeric.symbolic.n
    if rhs.shape[0] != n:
        raise DimensionMismatch(f"rhs has {rhs.shape[0]} rows, expected {n}")
    B = rhs.reshape(n, -1)
    X = _solve_cols(numeric, B)
    if refine:
        R = B - numeric._matrix @ X
        X = X + _solve_cols(numeric, R)
    return X.reshape(rhs.shape)


def factor_solve(matrix, rhs):
    sym = analyze(matrix)
    return factorize(sym, matrix).solve(rhs)
