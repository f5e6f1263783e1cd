"""Drop-in space-time solvers (reference pkg/src/kronheat/solvers.py).

Same entry points, types and error behaviour as the reference:

* `SpaceTimeSystem`   (solvers.py:50-82)   -- also accepts the reference's own objects (duck typing)
* `PencilFactorization`, `SpaceTimeSolution`, `SolveReport` (:85-163)
* `build_pencil(temporal, variant)` (:166-206) -- host LAPACK, unchanged semantics
* `solve_fd(system, pencil=None, threads=1)` (:348-403) -- GPU path
* `residual(system, coefficients)` (:428-440) -- GPU path
* `solve(system, variant, threads=1, fallback=True)` (:443-463)
* `eig_study(temporal)` (:466-482)

What changes in `solve_fd`: the transforms, the N_t shifted spatial solves
and the residual run on the GPU (libkhb200.so); one representative per
conjugate eigenpair is solved (the partner is its conjugate), which makes the
back transform real by construction; and the FD result is polished by
iterative refinement on the space-time residual (`refine`, default up to 3
steps to a 1e-13 relative residual). `refine=0` gives the plain FD of the
reference. The report keeps every reference field (and its t_total
convention) and adds `t_refine`, `t_solve`, `refine_steps`, `imag_residue`
and `fd_residual` (the residual before refinement).
"""

import os
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.sparse as sp

from . import sparse_direct
from .dense import (ComplexSchurForm, EigenSvdForm, RealSchurForm, cholesky_lower, complex_schur,
                    eig_pencil, eig_pencil_reduced, pencil_residual, real_schur, spd_solve,
                    svd_of_eigenvectors, svd_of_eigenvectors_real)
from .errors import DefectivePencil, DimensionMismatch, ImaginaryResidueTooLarge

FD_IMAG_TOL = 1e-6       # solvers.py:400
DEFAULT_REFINE = 5  # upper bound; the stop rule ends c3 after 1 step, c4 after 3
DEFAULT_REFINE_TOL = 1e-13
SPECULATIVE_PLAN_MAX_NT = 512  # solve_fd builds the numeric plan before the eigenvalues exist up to this N_t


@dataclass(frozen=True)
class SpaceTimeSystem:
    """Operators plus the global rhs, spatial index fastest (solvers.py:50-82)."""

    temporal: object
    spatial: object
    rhs: np.ndarray

    def __post_init__(self):
        if self.rhs.shape != (self.n_t * self.m_x,):
            raise DimensionMismatch(
                f"rhs length {self.rhs.shape} does not match N_t*M_x = {self.n_t}*{self.m_x}")

    @property
    def n_t(self):
        return self.temporal.A.shape[0]

    @property
    def m_x(self):
        return self.spatial.n_interior

    @property
    def dof(self):
        return self.n_t * self.m_x

    def rhs_matrix(self):
        return self.rhs.reshape(self.m_x, self.n_t, order="F")


@dataclass(frozen=True)
class PencilFactorization:
    variant: str
    chol_A: np.ndarray
    form: object
    # the temporal operators, kept by the "reduced" eigensolver so that the
    # reference's spectral statistics can be produced on demand
    temporal: object = field(default=None, repr=False, compare=False)
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def spectral_stats(self):
        """(sigma_min, sigma_max) of X_t in the reference's convention (dggev
        vectors; solvers.py:146-163). A "qz" pencil has them in its SVD; for a
        "reduced" pencil they depend on the phase dggev assigns each complex
        vector (see build_pencil), so they are computed by the QZ route on the
        first request and cached: a diagnostic, not an input of the solve."""
        form = self.form
        if getattr(form, "real_svd", None) is None or self.temporal is None:
            return float(form.sigma[-1]), float(form.sigma[0])
        if "qz" not in self._cache:
            vals, vecs = eig_pencil(self.temporal.M, self.temporal.A)
            sig = np.linalg.svd(vecs, compute_uv=False)
            self._cache["qz"] = (float(sig[-1]), float(sig[0]))
        return self._cache["qz"]

    @property
    def eigenvalues(self):
        if isinstance(self.form, EigenSvdForm) or hasattr(self.form, "sigma"):
            return self.form.D
        return self.form.eigenvalues()

    @property
    def min_re_lambda(self):
        return float(np.min(self.eigenvalues.real))


@dataclass(frozen=True)
class SpaceTimeSolution:
    coefficients: np.ndarray
    boundary_values: Optional[np.ndarray] = None

    def interior_matrix(self, m_x):
        return self.coefficients.reshape(m_x, -1, order="F")

    def full_coefficients(self, spatial):
        Z = self.interior_matrix(spatial.n_interior)
        full = np.zeros((spatial.interior.size + spatial.boundary.size, Z.shape[1]))
        full[spatial.interior] = Z
        if self.boundary_values is not None:
            full[spatial.boundary] = self.boundary_values
        return full


class _LazyStat:
    """Dataclass field descriptor for sigma_min / sigma_max / kappa2: an
    ordinary assignable float (reference solvers.py:136-139), which, while
    unset, is produced on first read from the report's `spectral_source`
    (a callable returning (sigma_min, sigma_max); see solve_fd)."""

    def __set_name__(self, owner, name):
        self.name = name
        self.slot = "_" + name

    def __get__(self, obj, objtype=None):
        if obj is None:
            return None  # the dataclass default: "not set"
        v = obj.__dict__.get(self.slot)
        if v is None:
            lo, hi = obj._spectral_pair()
            v = {"sigma_min": lo, "sigma_max": hi, "kappa2": hi / lo if lo > 0.0 else 0.0}[self.name]
        return v

    def __set__(self, obj, value):
        obj.__dict__[self.slot] = None if value is None else float(value)


@dataclass
class SolveReport:
    """Per-stage wall times and spectral statistics (solvers.py:125-163).

    Same fields and `t_total` convention as the reference (decompose +
    transform_in + spatial + transform_out, solvers.py:146-149); the GPU
    build adds `t_refine` (iterative refinement, reported separately;
    `t_solve` = t_total + t_refine is the whole solve), `refine_steps`,
    `imag_residue`, `fd_residual`, `device` and `phases`.
    """

    variant: str
    dof: int
    n_t: int
    m_x: int
    t_decompose: float = 0.0
    t_transform_in: float = 0.0
    t_spatial: float = 0.0
    t_transform_out: float = 0.0
    residual: float = 0.0
    min_re_lambda: float = 0.0
    sigma_min: float = _LazyStat()
    sigma_max: float = _LazyStat()
    kappa2: float = _LazyStat()
    threads: int = 1
    analyze_calls: int = 0
    fallback: Optional[str] = None
    # additions of the GPU build
    t_refine: float = 0.0
    refine_steps: int = 0
    imag_residue: float = 0.0
    fd_residual: float = 0.0
    residual_mode: str = "fp64"   # "dd": the refinement finished on the compensated residual
    device: str = ""
    # host-side milestones of solve_fd in seconds since its start (pencil,
    # analyze, host_joined, plan, factored): where the end-to-end time goes
    phases: dict = field(default_factory=dict)
    # callable -> (sigma_min, sigma_max) of X_t for the unset spectral fields
    spectral_source: object = field(default=None, repr=False, compare=False)

    def _spectral_pair(self):
        if self.spectral_source is None:
            return 0.0, 0.0
        key = "_spectral_cache"
        if key not in self.__dict__:
            lo, hi = self.spectral_source()
            self.__dict__[key] = (float(lo), float(hi))
        return self.__dict__[key]

    @property
    def t_total(self):
        return self.t_decompose + self.t_transform_in + self.t_spatial + self.t_transform_out

    @property
    def t_solve(self):
        """The whole GPU solve: t_total plus the refinement steps."""
        return self.t_total + self.t_refine

    def csv_row(self):
        return (f"{self.dof},{self.n_t},{self.m_x},{self.variant},"
                f"{self.t_decompose:.6f},{self.t_transform_in:.6f},"
                f"{self.t_spatial:.6f},{self.t_transform_out:.6f},"
                f"{self.residual:.3e},{self.min_re_lambda:.3e},"
                f"{self.kappa2:.3e},{self.threads}")

    @staticmethod
    def csv_header():
        return ("dof,N_t,M_x,variant,t_decomp,t_transform_in,t_spatial,"
                "t_transform_out,residual,minReLambda,kappa2,threads")


def build_pencil(temporal, variant, eig="qz", on_eigenvalues=None):
    """Decompose the temporal pencil on the host (solvers.py:166-206).

    ``eig`` picks the "fd" eigensolver: "qz" (default) is the reference's
    dggev + complex SVD; "reduced" reduces the pencil with the Cholesky factor
    of A_t, runs dgeev on L^-1 M_t L^-T and takes the SVD of X in its real
    basis: 3-6x less host time at N_t=256, ~15x at N_t=1024. Both give the
    same eigenvalues to rounding and the same vector conventions (pairs
    adjacent, +Im first, exact conjugates, max |Re|+|Im| = 1 per column), so
    the FD solution is the same; sigma and kappa_2 of X differ by a few
    percent, because that scaling depends on the phase LAPACK happens to give
    each complex vector, which the two algorithms choose differently
    (tests/test_pencil.py). `solve_fd` uses "reduced" when it builds the
    pencil itself; its report still carries the reference's statistics
    (`PencilFactorization.spectral_stats`, computed when first read).
    ``on_eigenvalues(vals, vecs)`` ("fd" only) is called as soon as the
    eigenpairs have passed the residual check, before the SVD of X (solve_fd
    starts factoring the shifts there).
    """
    L = cholesky_lower(temporal.A)
    P = spd_solve(L, temporal.M)
    if variant == "bs-real":
        form = real_schur(P)
    elif variant == "bs-complex":
        form = complex_schur(P)
    elif variant == "fd":
        scale = max(np.linalg.norm(P, "fro"), 1.0)
        if eig == "reduced":
            vals, vecs = eig_pencil_reduced(temporal.M, temporal.A, L)
            if pencil_residual(P, vecs, vals) > 1e-8 * scale:
                raise DefectivePencil("eigenvector residual above tolerance")
            if on_eigenvalues is not None:
                on_eigenvalues(vals, vecs)
            form = svd_of_eigenvectors_real(vecs, vals)
        elif eig == "qz":
            vals, vecs = eig_pencil(temporal.M, temporal.A)
            if np.linalg.norm(P @ vecs - vecs * vals[None, :], "fro") > 1e-8 * scale:
                raise DefectivePencil("eigenvector residual above tolerance")
            if on_eigenvalues is not None:
                on_eigenvalues(vals, vecs)
            form = svd_of_eigenvectors(vecs, vals)
        else:
            raise ValueError(f"unknown eigensolver: {eig!r}")
    else:
        raise ValueError(f"unknown pencil variant: {variant!r}")
    pencil = PencilFactorization(variant=variant, chol_A=L, form=form,
                                 temporal=temporal if variant == "fd" and eig == "reduced" else None)
    if pencil.min_re_lambda <= 0.0:
        raise DefectivePencil("pencil eigenvalue with nonpositive real part")
    return pencil


def spectral_source(pencil):
    """(sigma_min, sigma_max) producer for a report: this build's pencils
    carry `spectral_stats` (the reference's dggev statistics); a pencil built
    by the reference itself (or any object with an eigen-SVD `form`) gives
    its form's singular values, as the reference's solve_fd does
    (solvers.py:358-360)."""
    fn = getattr(pencil, "spectral_stats", None)
    if callable(fn):
        return fn
    form = pencil.form
    return lambda: (float(form.sigma_min), float(form.sigma_max))


def _blas_threads(n):
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover - optional dependency
        import contextlib

        return contextlib.nullcontext()
    return threadpool_limits(limits=n, user_api="blas")


def _sync():
    import torch

    torch.cuda.synchronize()


def _to_device(a, dev):
    """Host array -> device tensor (an async DMA when `a` is pinned memory)."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
    return t.to(dev, non_blocking=t.is_pinned())


def _to_host(t):
    """Device tensor -> numpy array backed by pinned host memory (full-rate DMA;
    torch caches pinned blocks, so repeated solves do not re-pin)."""
    import torch

    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t)
    return out.numpy()


def _publish_modes(box, ready, n_t, vals, vecs):
    """Hand the shifts of the FD solve (one representative per conjugate pair,
    then the real eigenvalues: the order of engine.modal_plan) to the worker
    thread that factors them, as soon as the pencil's eigenpairs exist."""
    from .engine import modal_stub

    if np.min(np.real(vals)) <= 0.0:
        return  # build_pencil raises DefectivePencil; nothing is factored
    box["stub"] = modal_stub(n_t, vals, vecs)
    ready.set()


def solve_fd(system, pencil=None, threads=1, refine=DEFAULT_REFINE, refine_tol=DEFAULT_REFINE_TOL,
             leaf_size=sparse_direct.DEFAULT_LEAF_SIZE, max_batch=None, keep_factors=None):
    """Fast diagonalization on the GPU: independent complex spatial solves.

    ``threads`` is accepted for API compatibility and recorded in the report
    (the GPU processes all shifts concurrently).
    """
    import torch

    from . import _native
    from .engine import FDEngine, modal_plan

    _native.require_cuda()
    report = SolveReport(variant="fd", dof=system.dof, n_t=system.n_t, m_x=system.m_x, threads=threads)
    dev = torch.device("cuda", torch.cuda.current_device())
    report.device = torch.cuda.get_device_name(dev)
    n, nt = system.m_x, system.n_t

    # Host pipeline. A worker thread runs the spatial symbolic analysis (host
    # C++, releases the GIL), aligns M_x and A_x on its pattern, and -- as
    # soon as this thread has the eigenvalues of the temporal pencil -- builds
    # the numeric plan and launches the factorization of every shift. This
    # thread meanwhile finishes the pencil (SVD of the eigenvectors) and the
    # modal transforms, which only the GEMMs after the factorization need:
    # the GPU factors while the host completes the pencil.
    t0 = time.perf_counter()
    analyze_before = sparse_direct.analyze_call_count()
    phases = report.phases
    lam_box = {}
    lam_ready = threading.Event()   # main -> worker: the shifts are known
    queued = threading.Event()      # worker -> main: factorization queued (or the worker is done)

    def _spatial_setup():
        try:
            a0 = time.perf_counter()
            symbolic = sparse_direct.analyze(system.spatial.M_II, leaf_size, union_with=system.spatial.A_II)
            phases["analyze"] = time.perf_counter() - a0
            # M_x and A_x aligned on the analyzed pattern and the launch schedule
            # (cached on the symbolic), side by side: all three are native calls
            with ThreadPoolExecutor(max_workers=2) as side:
                fa = side.submit(symbolic.align_values, system.spatial.A_II)
                fs = side.submit(sparse_direct.plan_bytes, symbolic, 1, 1)
                aligned = (symbolic.align_values(system.spatial.M_II), fa.result())
                fs.result()
            phases["aligned"] = time.perf_counter() - t0
            eng = None
            if not lam_ready.is_set() and nt <= SPECULATIVE_PLAN_MAX_NT:
                # The shifts are not known yet: build the plan meanwhile for the
                # mode count a pencil of conjugate pairs (plus one real
                # eigenvalue when N_t is odd) has. It holds no shift data; if
                # the count turns out different the plan is rebuilt below
                # (only done for small pencils: there the host latency matters
                # and a rebuilt workspace is cheap).
                from .engine import ModalPlan

                guess = (nt + 1) // 2
                blank = ModalPlan(n_t=nt, lam=np.zeros(guess, dtype=np.complex128), weight=np.ones(guess),
                                  n_pairs=nt // 2, n_single=nt % 2, w_in=None, w_out=None, kron_b=None)
                with torch.cuda.device(dev), nvtx.range("kh.solve_fd.plan"):
                    eng = FDEngine(system.spatial.M_II, system.spatial.A_II, blank, device=dev,
                                   leaf_size=leaf_size, max_batch=max_batch, keep_factors=keep_factors,
                                   symbolic=symbolic, aligned=aligned)
                phases["plan_early"] = time.perf_counter() - t0
            lam_ready.wait()
            if "stub" not in lam_box:  # the pencil failed on the main thread
                return None
            stub = lam_box["stub"]
            with torch.cuda.device(dev), nvtx.range("kh.solve_fd.plan"):
                if eng is not None and eng.n_k == stub.n_k:
                    eng.modal, eng.lam = stub, np.ascontiguousarray(stub.lam)
                else:
                    eng = None  # frees the speculative plan's workspace first
                    eng = FDEngine(system.spatial.M_II, system.spatial.A_II, stub, device=dev,
                                   leaf_size=leaf_size, max_batch=max_batch, keep_factors=keep_factors,
                                   symbolic=symbolic, aligned=aligned)
                phases["plan"] = time.perf_counter() - t0
                phases["memplan"] = eng.t_memplan - t0
                phases["plans_created"] = eng.t_plans - t0
                eng.factor(check=False)  # retained factors: queued now, checked after the solves are queued
            phases["factor_queued"] = time.perf_counter() - t0
            return eng
        finally:
            queued.set()

    def _on_eigenvalues(vals, vecs):
        # publish the shifts, then let the worker build the plan and queue the
        # factorization before this thread's Python-heavy rest of the pencil
        # competes with it for the GIL: the GPU starts as early as possible
        phases["eigenvalues"] = time.perf_counter() - t0
        _publish_modes(lam_box, lam_ready, nt, vals, vecs)
        if lam_ready.is_set():
            queued.wait()

    # a pinned rhs goes up asynchronously right away (the copy engine works
    # while the host computes the pencil); a pageable one after the pencil
    rhs_t = torch.from_numpy(np.ascontiguousarray(np.asarray(system.rhs, dtype=np.float64)))
    F = rhs_t.to(dev, non_blocking=True).view(nt, n) if rhs_t.is_pinned() else None
    nvtx = torch.cuda.nvtx
    nvtx.range_push("kh.solve_fd.host")
    pool = ThreadPoolExecutor(max_workers=1)
    fut = pool.submit(_spatial_setup)
    try:
        # few BLAS threads: dgeev / the SVD of an N_t <= 512 matrix gain
        # nothing from more, and the dissection threads of the analysis
        # need the cores
        with _blas_threads(int(os.environ.get("KH_PENCIL_THREADS", 1 if nt <= 512 else 4))):
            if pencil is None:
                pencil = build_pencil(system.temporal, "fd", eig="reduced", on_eigenvalues=_on_eigenvalues)
            else:
                form = pencil.form
                if getattr(form, "X", None) is not None and getattr(form, "D", None) is not None:
                    _publish_modes(lam_box, lam_ready, nt, np.asarray(form.D), np.asarray(form.X))
            phases["pencil"] = time.perf_counter() - t0
            form = pencil.form
            if not (isinstance(form, EigenSvdForm)
                    or all(hasattr(form, a) for a in ("X", "D", "U", "sigma", "Vh"))):
                raise DimensionMismatch("solve_fd needs an eigen-SVD pencil")
            modal = modal_plan(system.temporal, pencil)
        report.t_decompose = time.perf_counter() - t0
        if F is None:
            F = rhs_t.to(dev).view(nt, n)
    finally:
        lam_ready.set()  # a failed pencil releases the worker (it then returns None)
        eng = fut.result()
        pool.shutdown()
    if not np.array_equal(eng.lam, modal.lam):
        raise DimensionMismatch("internal: factored shifts differ from the modal plan's")
    eng.attach_modal(modal)
    phases["host_joined"] = time.perf_counter() - t0
    report.min_re_lambda = pencil.min_re_lambda
    report.spectral_source = spectral_source(pencil)
    nvtx.range_pop()
    report.analyze_calls = sparse_direct.analyze_call_count() - analyze_before
    t_setup = time.perf_counter() - t0 - report.t_decompose

    t0 = time.perf_counter()
    U = torch.empty((nt, n), dtype=torch.float64, device=dev)
    eng._gemm(n, 2 * eng.n_k, nt, 1.0, F.data_ptr(), n, eng.w_in.data_ptr(), nt, 0.0, eng.G.data_ptr(), n)
    _sync()
    report.t_transform_in = time.perf_counter() - t0

    # factorization of every shift with the forward sweep fused, then the
    # backward sweep (engine._spatial)
    t0 = time.perf_counter()
    eng._spatial()
    _sync()
    report.t_spatial = t_setup + time.perf_counter() - t0
    phases["solved"] = time.perf_counter() - t0 + t_setup + report.t_decompose + report.t_transform_in

    t0 = time.perf_counter()
    eng._gemm(n, nt, 2 * eng.n_k, 1.0, eng.Z.data_ptr(), n, eng.w_out.data_ptr(), 2 * eng.n_k, 0.0,
              U.data_ptr(), n)
    _sync()
    report.t_transform_out = time.perf_counter() - t0
    # the real-basis back transform is real by construction, so the
    # reference's imaginary-residue guard (solvers.py:400) has nothing to test
    report.imag_residue = 0.0

    t0 = time.perf_counter()
    rel = eng._rel(eng.residual(U, F))
    report.fd_residual = rel
    # u += FD(f - K u): a step that does not help is undone; stagnation of the
    # fp64 residual above refine_tol switches to the compensated residual
    # the device-to-host copy of an iterate starts right after its correction,
    # on a second stream beside the residual that decides whether it is final
    # (a later correction or an undone step supersedes the copy)
    taken = {"host": None, "valid": False}
    copy_stream = torch.cuda.Stream(dev)

    def _take(Ucur, fresh):
        taken["valid"] = fresh
        if fresh:
            if taken["host"] is None:
                taken["host"] = torch.empty(Ucur.numel(), dtype=Ucur.dtype, pin_memory=True)
            copy_stream.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(copy_stream):
                taken["host"].copy_(Ucur.reshape(-1), non_blocking=True)

    if os.environ.get("KH_D2H_OVERLAP", "1") != "0":
        eng.on_iterate = _take
    rel, steps = eng.refine(U, F, rel, refine, refine_tol)
    eng.on_iterate = None
    report.residual_mode = eng.residual_mode
    with nvtx.range("kh.solve_fd.d2h"):
        if taken["valid"]:
            copy_stream.synchronize()
            coeffs = taken["host"].numpy()
        else:
            copy_stream.synchronize()  # a superseded copy must not outlive U
            coeffs = _to_host(U.reshape(-1))
    report.t_refine = time.perf_counter() - t0
    report.refine_steps = steps
    report.residual = rel
    return SpaceTimeSolution(coefficients=coeffs), report


def residual(system, coefficients, compensated=False):
    """Relative residual ||K u - f|| / ||f|| on the GPU (solvers.py:428-440).

    compensated=True evaluates it with error-free products and sums
    (kh_dgemm_dd + kh_csr_pair_residual_dd): the accurate value at fine
    meshes, where the fp64 evaluation itself is off by ~1e-11 (config c4)."""
    import torch

    from . import _native
    from .engine import _fortran

    _native.require_cuda()
    coefficients = np.asarray(coefficients)
    if coefficients.shape != system.rhs.shape:
        raise DimensionMismatch("coefficient vector has wrong length")
    n, nt = system.m_x, system.n_t
    dev = torch.device("cuda", torch.cuda.current_device())
    M = system.spatial.M_II.tocsr()
    A = system.spatial.A_II.tocsr()
    indptr, indices = sparse_direct.symmetrized_pattern((M + A).tocsr())
    probe = sparse_direct.SymbolicFactorization(n=n, perm=np.arange(n), factor_nnz=0, indptr=indptr,
                                                indices=indices)
    to_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    d_ptr, d_idx = to_dev(indptr), to_dev(indices)
    d_m, d_a = to_dev(probe.align_values(M)), to_dev(probe.align_values(A))
    kron_b = _fortran(np.hstack([system.temporal.A.T, system.temporal.M.T]), dev)
    U = to_dev(np.asarray(coefficients, dtype=np.float64))
    F = to_dev(np.asarray(system.rhs, dtype=np.float64))
    Y = torch.empty((2 * nt, n), dtype=torch.float64, device=dev)
    norms = torch.zeros(2, dtype=torch.float64, device=dev)
    st = _native.stream_handle()
    if compensated:
        lo = torch.empty((nt, n), dtype=torch.float64, device=dev)
        y1, y2 = Y.data_ptr(), Y.data_ptr() + 8 * n * nt
        _native.call("kh_dgemm", n, nt, nt, 1.0, U.data_ptr(), n, kron_b.data_ptr(), nt, 0.0, y1, n, st)
        _native.call("kh_dgemm_dd", n, nt, nt, U.data_ptr(), n, kron_b.data_ptr() + 8 * nt * nt, nt, y2,
                     lo.data_ptr(), n, st)
        _native.call("kh_csr_pair_residual_dd", n, nt, d_ptr.data_ptr(), d_idx.data_ptr(), d_m.data_ptr(),
                     d_a.data_ptr(), y1, n, y2, lo.data_ptr(), n, F.data_ptr(), n, None, n, norms.data_ptr(), st)
    else:
        _native.call("kh_dgemm", n, 2 * nt, nt, 1.0, U.data_ptr(), n, kron_b.data_ptr(), nt, 0.0, Y.data_ptr(), n,
                     st)
        _native.call("kh_csr_pair_residual", n, nt, d_ptr.data_ptr(), d_idx.data_ptr(), d_m.data_ptr(),
                     d_a.data_ptr(), Y.data_ptr(), n, F.data_ptr(), n, None, n, norms.data_ptr(), st)
    r2, f2 = norms.tolist()
    if f2 == 0.0:
        return float(np.sqrt(r2))
    return float(np.sqrt(r2) / np.sqrt(f2))


def solve(system, variant, threads=1, fallback=True):
    """Dispatch by variant name with the FD fallback policy (solvers.py:443-463)."""
    if variant == "bs-real":
        return solve_bs_real(system)
    if variant == "bs-complex":
        return solve_bs_complex(system)
    if variant == "fd":
        if not fallback:
            return solve_fd(system, threads=threads)
        try:
            return solve_fd(system, threads=threads)
        except (DefectivePencil, ImaginaryResidueTooLarge) as exc:
            sol, report = solve_bs_complex(system)
            report.fallback = f"fd failed: {type(exc).__name__}"
            return sol, report
    raise ValueError(f"unknown solver variant: {variant!r}")


def solve_bs_complex(system, pencil=None):
    from .bartels_stewart import solve_bs_complex as _bs

    return _bs(system, pencil)


def solve_bs_real(system, pencil=None):
    from .bartels_stewart import solve_bs_real as _bs

    return _bs(system, pencil)


def eig_study(temporal):
    pencil = build_pencil(temporal, "fd")
    form = pencil.form
    return {
        "n_t": temporal.A.shape[0],
        "min_re_lambda": pencil.min_re_lambda,
        "sigma_min": form.sigma_min,
        "sigma_max": form.sigma_max,
        "kappa2": form.kappa2,
    }
