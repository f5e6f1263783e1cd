"""GPU orchestration of the Fast-Diagonalization solve (host control, device data).

One `FDEngine` owns everything a solve needs on the device:

1. the host-side modal plan (`modal_plan`): the reference's
   G = F A_t^-1 conj(U) S^-1 conj(Vh) (solvers.py:368-372) and
   U = Z Vh^T S U^T (solvers.py:397-400) folded into one real N_t x 2N_k
   matrix per direction, restricted to one representative per conjugate
   eigenpair (the partner's solve is the complex conjugate, so the back
   transform 2 Re(z x^T) is real by construction);
2. the symbolic analysis of M_x + A_x (one per engine, solvers.py:379) and a
   numeric plan holding the LDL^T factors of every shift M_x + lambda_k A_x;
3. device buffers for F, G, Z, U and the residual.

`solve(F)` runs transform-in GEMM -> batched factor/solve -> transform-out
GEMM, then iterative refinement on the space-time residual (not in the
reference; needed because FD's accuracy is limited by kappa_2(X_t), see
DESIGN.md). All kernels are in libkhb200.so; torch only allocates memory.
"""

import os
import time
from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import _native, sparse_direct
from .dense import real_basis, spd_solve
from .errors import DefectivePencil, DimensionMismatch



@dataclass
class ModalPlan:
    n_t: int
    lam: np.ndarray        # (N_k,) complex; conjugate-pair representatives first, then singles
    weight: np.ndarray     # 2.0 for pair representatives, 1.0 for singles
    n_pairs: int
    n_single: int
    w_in: np.ndarray       # (N_t, 2 N_k): [Re W_in[:, modes] | Im W_in[:, modes]]
    w_out: np.ndarray      # (2 N_k, N_t): [w Re W_out[modes, :] ; -w Im W_out[modes, :]]
    kron_b: np.ndarray     # (N_t, 2 N_t): [A_t^T | M_t^T] for K u = vec(M_x U A_t^T + A_x U M_t^T)

    @property
    def n_k(self):
        return len(self.lam)


# iterative refinement stops once a step fails to halve the residual (the
# classic rule: further steps only shuffle rounding errors at the floor of
# evaluating f - K u); a step that does not lower it at all is undone
# (FDEngine.refine_step), so the best iterate is returned
REFINE_MIN_GAIN = 0.5
# refinement on the compensated residual (fp64 evaluation floor above the
# tolerance: fine meshes, config c4) stops at this relative residual, one
# decade under the 1e-11 bar of BASELINE.json
DD_TOL = 1e-12
# ... entered once the fp64 residual is within this factor of its estimated
# rounding floor (c4: after two steps; c3, c5: never)
FLOOR_MARGIN = 10.0


def conjugate_pairs(D, X):
    """Split eigen-indices into (+Im representative of conjugate pairs, singles).

    dggev returns a complex pair adjacent with +Im first, and eig_pencil builds
    the two eigenvectors as exact conjugates (reference dense.py:210-220);
    the eigenvalues themselves may differ from exact conjugates in the last
    bit (alpha/beta rounding), so pairs are identified by the vectors.
    """
    reps, singles = [], []
    n = len(D)
    j = 0
    while j < n:
        if (D[j].imag > 0.0 and j + 1 < n and D[j + 1].imag < 0.0
                and np.array_equal(X[:, j + 1], np.conj(X[:, j]))):
            reps.append(j)
            j += 2
        else:
            singles.append(j)
            j += 1
    return np.array(reps, dtype=np.int64), np.array(singles, dtype=np.int64)


def modal_stub(n_t, D, X):
    """The shifts of a modal plan (same order as `modal_plan`: conjugate-pair
    representatives, then the real eigenvalues) without its transforms: what
    an FDEngine needs to factor before the SVD of X is done
    (FDEngine.attach_modal supplies the rest)."""
    reps, singles = conjugate_pairs(D, X)
    lam = np.concatenate([np.asarray(D)[reps], np.asarray(D)[singles].real.astype(np.complex128)])
    weight = np.concatenate([np.full(len(reps), 2.0), np.ones(len(singles))])
    return ModalPlan(n_t=n_t, lam=np.ascontiguousarray(lam, dtype=np.complex128), weight=weight,
                     n_pairs=len(reps), n_single=len(singles), w_in=None, w_out=None, kron_b=None)


def modal_plan(temporal, pencil):
    """Real-basis FD transforms with one solve per conjugate pair.

    The reference applies X^-1 = V S^-1 U^* from the complex SVD of X
    (solvers.py:368-372). Here X is first mapped to the
    real basis X_r = [.., Re x_j, Im x_j, .., x_real, ..] (X_r = X T with T
    block-diagonal), and the SVD damping is applied to X_r. The computed
    inverse columns of a pair are then exact conjugates,
        (X^-T)[:, j] = (r1 - i r2) / 2,   r1, r2 = columns of X_r^-T,
    so solving only the representative and taking 2 Re(z_j x_j^T) is
    consistent with the inverse to working precision. (Using the complex
    inverse's column j alone is not: its deviation from conjugate symmetry
    is kappa_2(X) eps, amplified again by kappa_2 in the back transform.)
    """
    form = pencil.form
    n_t = temporal.A.shape[0]
    X = form.X
    reps, singles = conjugate_pairs(form.D, X)
    if any(abs(form.D[j].imag) > 0.0 for j in singles):
        # only reachable for complex pencils that dggev never produces for real (M_t, A_t)
        raise DefectivePencil("unpaired complex eigenvalue in a real pencil")
    # real basis in eigenvalue order: pair j -> columns (Re x_j, Im x_j);
    # real eigenvalue -> x_j; Y = X_r diag(s) has the singular values of X
    Xr, s = real_basis(X, form.D)
    where = {j: j for j in list(reps) + list(singles)}
    if getattr(form, "real_svd", None) is not None:
        Ur, sr, Vrh, s = form.real_svd
    else:
        Ur, sr, Vrh = sla.svd(Xr * s[None, :])
    if sr[-1] <= 0.0:
        raise DefectivePencil("eigenvector matrix is numerically singular")
    # W_r = A_t^-1 X_r^-T = A_t^-1 Y^-T diag(s) = A_t^-1 U S^-1 V^T diag(s)
    # (damped through the SVD like the reference's X^-1)
    Wr = (spd_solve(pencil.chol_A, Ur / sr[None, :]) @ Vrh) * s[None, :]
    nk = len(reps) + len(singles)
    w_in = np.zeros((n_t, 2 * nk))
    w_out = np.zeros((2 * nk, n_t))
    lam = np.empty(nk, dtype=np.complex128)
    for k, j in enumerate(reps):
        c = where[j]
        w_in[:, k] = 0.5 * Wr[:, c]            # Re of (r1 - i r2) / 2
        w_in[:, nk + k] = -0.5 * Wr[:, c + 1]  # Im
        w_out[k, :] = 2.0 * Xr[:, c]           # 2 Re(z x^T) = 2 (z_r x_r^T - z_i x_i^T)
        w_out[nk + k, :] = -2.0 * Xr[:, c + 1]
        lam[k] = form.D[j]
    for s, j in enumerate(singles):
        k = len(reps) + s
        c = where[j]
        w_in[:, k] = Wr[:, c]
        w_out[k, :] = Xr[:, c]
        lam[k] = form.D[j].real
    kron_b = np.ascontiguousarray(np.hstack([temporal.A.T, temporal.M.T]))
    weight = np.concatenate([np.full(len(reps), 2.0), np.ones(len(singles))])
    return ModalPlan(n_t=n_t, lam=lam, weight=weight, n_pairs=len(reps), n_single=len(singles),
                     w_in=np.ascontiguousarray(w_in), w_out=np.ascontiguousarray(w_out), kron_b=kron_b)


def _on_device(fn):
    """Run an FDEngine method with the engine's device current (streams,
    kh_dgemm and the torch allocations then all refer to that device; the
    caller's current device is restored afterwards), inside an NVTX range
    "kh.<method>" (engine phases in ncu --nvtx / Nsight timelines)."""
    import functools

    name = "kh." + fn.__name__.lstrip("_")

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        import torch

        with torch.cuda.device(self.device), torch.cuda.nvtx.range(name):
            return fn(self, *args, **kwargs)

    return wrapper


def _fortran(t_np, device, async_copy=False):
    """Host (rows x cols) array -> device column-major buffer (as a torch tensor
    of shape (cols, rows), i.e. the transpose view, contiguous).
    async_copy: stage through pinned memory and copy without blocking the host
    (the copy is queued behind the stream's work, e.g. a factorization)."""
    import torch

    a = np.asarray(t_np, dtype=np.float64)
    t = torch.from_numpy(np.ascontiguousarray(a.T))
    if async_copy:
        return t.pin_memory().to(device, non_blocking=True)
    return t.to(device)


class FDEngine:
    """Device-resident FD solver for one (M_x, A_x, temporal pencil) triple."""

    def __init__(self, M_x, A_x, modal, device=None, keep_factors=None, max_batch=None,
                 leaf_size=sparse_direct.DEFAULT_LEAF_SIZE, mem_fraction=0.85, symbolic=None, pipes=1,
                 fuse_forward=None, aligned=None):
        import torch

        _native.require_cuda()
        if device is None:
            device = torch.cuda.current_device()
        self.device = device if isinstance(device, torch.device) else torch.device("cuda", int(device))
        M = sp.csr_matrix(M_x)
        A = sp.csr_matrix(A_x)
        if M.shape != A.shape or M.shape[0] != M.shape[1]:
            raise DimensionMismatch("spatial matrices must be square and of equal shape")
        self.n = M.shape[0]
        self.modal = modal
        # optional hook on_iterate(U, fresh) of the refinement: called right after U
        # received a correction (fresh=True) or lost it again (an undone step)
        self.on_iterate = None
        self.n_t = modal.n_t
        self.n_k = modal.n_k
        self.sym = symbolic if symbolic is not None else sparse_direct.analyze((M + A).tocsr(), leaf_size)
        # values of M and A on the analyzed pattern (`aligned` = precomputed pair)
        mv, av = aligned if aligned is not None else (self.sym.align_values(M), self.sym.align_values(A))

        # shift pipelines: the shifts are split into `pipes` contiguous ranges,
        # each with its own plan (factor storage, work space, side streams) and
        # stream, so that one range's narrow top-of-tree launches could overlap
        # the other's wide ones (KH_PIPES overrides). Measured at c3: 1 pipe
        # 43.96, 2 pipes 44.22, 4 pipes 46.76 ms/step -- the top-level kernels
        # already fill the GPU -- so the default is a single plan.
        nk = max(self.n_k, 1)
        npipe = max(1, min(nk, int(os.environ.get("KH_PIPES", pipes))))
        bounds = [round(i * self.n_k / npipe) for i in range(npipe + 1)]
        sizes = [max(bounds[i + 1] - bounds[i], 1) for i in range(npipe)]

        sized = {}

        def total_bytes(b, keep):
            # each plan_bytes builds the launch schedule on the host: memoise
            if (b, keep) not in sized:
                sized[(b, keep)] = sum(sparse_direct.plan_bytes(self.sym, min(b, sz), sz if keep else min(b, sz))
                                       for sz in sizes)
            return sized[(b, keep)]

        # memory plan: keep every shift's factors when they fit
        with torch.cuda.device(self.device):
            free, _ = torch.cuda.mem_get_info()
            # blocks torch has cached but not handed out are free for us too
            free += torch.cuda.memory_reserved(self.device) - torch.cuda.memory_allocated(self.device)
        work = 8 * self.n * (2 * self.n_k * 2 + 2 * self.n_t * 3) + 8 * self.n_t * 8 * self.n_t
        budget = mem_fraction * free - work
        batch = min(max(sizes), max_batch or nk)
        if keep_factors is None:
            # keep every shift's factors if they fit with a working batch of
            # at least 16 shifts in flight (update buffers scale with it)
            b = batch
            floor = max(1, 16 // npipe)
            while b > floor and total_bytes(b, True) > budget:
                b = (b + 1) // 2
            keep_factors = total_bytes(b, True) <= budget
            if keep_factors:
                batch = b
        if not keep_factors:
            while batch > 1 and total_bytes(batch, False) > budget:
                batch = (batch + 1) // 2
        self.keep_factors = bool(keep_factors)
        self.batch = int(batch)
        self.t_memplan = time.perf_counter()
        self.pipes = []
        for i in range(npipe):
            k0, k1 = bounds[i], bounds[i + 1]
            b = min(self.batch, max(k1 - k0, 1))
            plan = sparse_direct._Plan(self.sym, mv, av, b, (k1 - k0 if self.keep_factors else b) or 1,
                                       self.device.index)
            self.pipes.append((plan, k0, k1, b, torch.cuda.Stream(device=self.device)))
        self.t_plans = time.perf_counter()
        self.plan = self.pipes[0][0]   # residual kernels (CSR of M, A) and single-pipe callers
        self.factored = False
        self.unchecked = []  # (plan, slot, count) factored without their pivot check yet
        # first application with retained factors: factor with the forward
        # sweep fused (kh_plan_factor_fwd) or factor, then sweep. Measured
        # equal at c3 (42.02 ms/step either way: the in-kernel sweep costs
        # what the standalone pass does), so the default keeps the two
        # apart and the factorization's roofline clean; without retained
        # factors every application is fused (no extra pass over factors
        # that are discarded anyway). KH_FUSED_FWD=1 flips the default.
        if fuse_forward is None:
            fuse_forward = os.environ.get("KH_FUSED_FWD", "0") == "1"
        self.fuse_forward = bool(fuse_forward)
        # compensated residual once the fp64 one stagnates above the tolerance
        # ("auto"), always (True) or never (False); KH_COMPENSATED overrides
        env = os.environ.get("KH_COMPENSATED")
        self.compensated = {"1": True, "0": False}.get(env, "auto")
        self.residual_mode = "fp64"

        dev = self.device
        f64 = torch.float64
        self.w_in = self.w_out = self.kron_b = None
        if modal.w_in is not None:
            self.attach_modal(modal)
        n, nt, nk2 = self.n, self.n_t, 2 * self.n_k
        self.G = torch.empty((nk2, n), dtype=f64, device=dev)   # column-major n x 2N_k
        self.Z = torch.empty((nk2, n), dtype=f64, device=dev)
        self.Y = torch.empty((2 * nt, n), dtype=f64, device=dev)
        self.R = torch.empty((nt, n), dtype=f64, device=dev)
        self.norms = torch.zeros(4, dtype=f64, device=dev)
        self.lam = np.ascontiguousarray(modal.lam)
        self.gpu_launches = 0
        # optional list of (start, end) CUDA events around every factorization
        # launch sequence (bench.py's roofline; also covers refactoring when
        # the factors are not kept)
        self.event_log = None
        # optional per-phase CUDA-event timers (bench.py's per-kernel rooflines)
        self.timers = None

    def attach_modal(self, modal):
        """Upload the modal transforms (W_in, W_out, [A_t^T | M_t^T]) of `modal`,
        whose shifts must be the ones the engine was built for (an engine built
        from `modal_stub` factors before the transforms exist)."""
        if not np.array_equal(np.asarray(modal.lam), self.lam if hasattr(self, "lam") else modal.lam):
            raise DimensionMismatch("modal plan shifts differ from the engine's")
        dev = self.device
        self.modal = modal
        # pinned, non-blocking: the host does not wait for work already queued
        self.w_in = _fortran(modal.w_in, dev, True)        # (2N_k, N_t) storage of N_t x 2N_k
        self.w_out = _fortran(modal.w_out, dev, True)      # (N_t, 2N_k) storage of 2N_k x N_t
        self.kron_b = _fortran(modal.kron_b, dev, True)    # (2N_t, N_t) storage of N_t x 2N_t

    # ---- primitives -----------------------------------------------------------
    def _stream(self):
        import torch

        return _native.stream_handle(torch.cuda.current_stream(self.device))

    def _timed(self, name, fn, *args):
        """fn(*args), bracketed by CUDA events on the current stream when
        self.timers (dict name -> [(start, end, info)]) is set (bench.py)."""
        if self.timers is None:
            return fn(*args)
        import torch

        st = torch.cuda.current_stream(self.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        out = fn(*args)
        e1.record(st)
        self.timers.setdefault(name, []).append((e0, e1))
        return out

    def _gemm(self, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc):
        _native.call("kh_dgemm", m, n, k, float(alpha), A, lda, B, ldb, float(beta), C, ldc, self._stream())
        self.gpu_launches += 1

    def _run_pipes(self, body, join=True):
        """Run body(plan, k0, k1, batch, stream) for every pipe, each on its own
        stream forked from the current one; join=True joins them back."""
        import torch

        main = torch.cuda.current_stream(self.device)
        fork = torch.cuda.Event()
        fork.record(main)
        for plan, k0, k1, b, st in self.pipes:
            st.wait_event(fork)
            body(plan, k0, k1, b, st)
        if join:
            self._join_pipes()

    def _join_pipes(self):
        import torch

        main = torch.cuda.current_stream(self.device)
        for *_, st in self.pipes:
            main.wait_stream(st)

    @_on_device
    def factor(self, events=None, check=True):
        """Factor M_x + lambda_k A_x for every retained shift (no-op otherwise).

        `events`: optional list that receives a (start, end) CUDA-event pair
        bracketing the factorization launches (for the roofline). The pivot
        guard synchronizes with the host; check=False defers it to the next
        application (`_spatial`), so that its solves are queued first."""
        if not self.keep_factors:
            return
        import torch

        main = torch.cuda.current_stream(self.device)
        if events is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)

        def body(plan, k0, k1, b, ts):
            st = _native.stream_handle(ts)
            for s0 in range(k0, k1, b):
                s1 = min(k1, s0 + b)
                plan.factor(s0 - k0, self.lam[s0:s1], st)
                self.gpu_launches += self.sym.stats["depth"] + 4

        self._run_pipes(body)
        if events is not None:
            e1.record(main)
            events.append((e0, e1))
        if check:
            for plan, k0, k1, b, st in self.pipes:
                plan.pivot_check(0, k1 - k0, self._stream())
        else:
            self.unchecked = [(plan, 0, k1 - k0) for plan, k0, k1, b, st in self.pipes]
        self.factored = True

    @_on_device
    def _spatial(self):
        """Z[:, k] = (M_x + lambda_k A_x)^-1 G[:, k] for all modes.

        Without retained factors (first application, or factors not kept) each
        batch is factored with the forward sweep fused into the factorization
        (kh_plan_factor_fwd) and then swept backward: the factors are read
        back once instead of twice. The shift pipelines run concurrently; the
        pivot checks (host synchronizations) come after everything is queued.
        """
        import torch

        n, nk = self.n, self.n_k
        g, z = self.G.data_ptr(), self.Z.data_ptr()
        depth = self.sym.stats["depth"] + 1
        fuse = not (self.keep_factors and self.factored)
        if fuse and self.keep_factors and not self.fuse_forward:
            # separate factorization, then the standalone sweeps
            self.factor(events=self.event_log)
            fuse = False
        log = self.event_log if fuse else None
        main = torch.cuda.current_stream(self.device)
        if log is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
        fac_done = []
        checks = []

        def body(plan, k0, k1, b, ts):
            st = _native.stream_handle(ts)
            for s0 in range(k0, k1, b):
                s1 = min(k1, s0 + b)
                slot = s0 - k0 if self.keep_factors else 0
                xr, xi = z + 8 * s0 * n, z + 8 * (nk + s0) * n
                if fuse:
                    plan.factor_fwd(slot, self.lam[s0:s1], g + 8 * s0 * n, g + 8 * (nk + s0) * n, n, st)
                    if log is not None:
                        ev = torch.cuda.Event()
                        ev.record(ts)
                        fac_done.append(ev)
                    plan.solve_bwd(slot, s1 - s0, xr, xi, n, st)
                    self.gpu_launches += 3 * depth + 5
                    if self.keep_factors:
                        checks.append((plan, slot, s1 - s0))
                    else:  # the slots are reused by the next batch: check now
                        plan.pivot_check(slot, s1 - s0, st)
                else:
                    plan.solve(slot, s1 - s0, g + 8 * s0 * n, g + 8 * (nk + s0) * n, n, xr, xi, n, st)
                    self.gpu_launches += 2 * depth + 2

        self._run_pipes(body, join=False)
        if log is not None:
            # end of the factorization: the last pipe's factor launches
            for ev in fac_done:
                main.wait_event(ev)
            e1.record(main)
            log.append((e0, e1))
        self._join_pipes()
        checks += self.unchecked
        self.unchecked = []
        for plan, slot, cnt in checks:
            plan.pivot_check(slot, cnt, self._stream())
        if fuse and self.keep_factors:
            self.factored = True

    @_on_device
    def refine_step(self, U, F, rel, dd=False):
        """One Richardson step u += FD(f - K u) on the residual held in R.
        The correction goes to the (then free) G buffer and is added with a
        daxpy, so a step that fails to lower the residual is undone: returns
        (new relative residual, residual of the returned U, keep_going).
        dd: the new residual is evaluated in compensated arithmetic."""
        import torch

        n, nt = self.n, self.n_t
        corr = self.G.view(-1)[: n * nt].view(nt, n)  # G is consumed by the first GEMM of fd_apply
        self.fd_apply(self.R, corr, accumulate=False)
        st = self._stream()
        _native.call("kh_daxpy", U.numel(), 1.0, corr.data_ptr(), U.data_ptr(), st)
        if self.on_iterate is not None:
            self.on_iterate(U, True)  # e.g. solve_fd starts the device-to-host copy beside the residual
        new = self._rel(self.residual(U, F, dd=dd))
        if not new < rel:
            # rounding floor reached: undo the step, keep the best iterate
            _native.call("kh_daxpy", U.numel(), -1.0, corr.data_ptr(), U.data_ptr(), st)
            if self.on_iterate is not None:
                self.on_iterate(U, False)  # U changed again: what was taken above is stale
            self.gpu_launches += 2
            return new, rel, False
        self.gpu_launches += 1
        return new, new, new < REFINE_MIN_GAIN * rel

    @_on_device
    def fd_apply(self, F, U, accumulate=False):
        """U (+)= FD(F): F and U are device column-major n x N_t buffers (torch
        tensors of shape (N_t, n))."""
        n, nt, nk2 = self.n, self.n_t, 2 * self.n_k
        self._timed("gemm", self._gemm, n, nk2, nt, 1.0, F.data_ptr(), n, self.w_in.data_ptr(), nt, 0.0,
                    self.G.data_ptr(), n)
        fused = not (self.keep_factors and self.factored)
        self._timed("factor_solve" if fused else "solve", self._spatial)
        self._timed("gemm", self._gemm, n, nt, nk2, 1.0, self.Z.data_ptr(), n, self.w_out.data_ptr(), nk2,
                    1.0 if accumulate else 0.0, U.data_ptr(), n)

    @_on_device
    def residual(self, U, F, keep_r=True, dd=False):
        """Device: R = F - K U; returns (||R||^2, ||F||^2) as a device tensor slice.

        dd=True evaluates it in compensated arithmetic (kh_dgemm_dd for
        U M_t^T, kh_plan_residual_dd): the low parts of U M_t^T go to the
        Z buffer, which is free between FD applications."""
        n, nt = self.n, self.n_t
        if not dd:
            self._timed("gemm_kron", self._gemm, n, 2 * nt, nt, 1.0, U.data_ptr(), n, self.kron_b.data_ptr(), nt,
                        0.0, self.Y.data_ptr(), n)
            self._timed("residual", self.plan.residual, nt, self.Y.data_ptr(), n, F.data_ptr(), n,
                        self.R.data_ptr() if keep_r else None, n, self.norms.data_ptr(), self._stream())
            self.gpu_launches += 2
            return self.norms[:2]
        st = self._stream()
        y1, y2 = self.Y.data_ptr(), self.Y.data_ptr() + 8 * n * nt
        self._timed("gemm_kron", self._gemm, n, nt, nt, 1.0, U.data_ptr(), n, self.kron_b.data_ptr(), nt, 0.0, y1, n)
        self._timed("gemm_dd", _native.call, "kh_dgemm_dd", n, nt, nt, U.data_ptr(), n,
                    self.kron_b.data_ptr() + 8 * nt * nt, nt, y2, self.Z.data_ptr(), n, st)
        self._timed("residual_dd", self.plan.residual_dd, nt, y1, n, y2, self.Z.data_ptr(), n, F.data_ptr(), n,
                    self.R.data_ptr() if keep_r else None, n, self.norms.data_ptr(), st)
        self.gpu_launches += 4
        return self.norms[:2]

    @_on_device
    def solve(self, F, U=None, refine=5, tol=1e-13):
        """Full FD solve of K u = f on the device with iterative refinement.

        Returns (U, info); U is a device tensor (N_t, n) = column-major n x N_t.
        """
        import torch

        if U is None:
            U = torch.empty((self.n_t, self.n), dtype=torch.float64, device=self.device)
        # not yet factored: the first application factors (forward sweep fused)
        self.fd_apply(F, U, accumulate=False)
        info = {"imag_residue": 0.0, "residuals": [], "refine_steps": 0}
        norms = self.residual(U, F).tolist()
        rel = float(np.sqrt(norms[0]) / np.sqrt(norms[1])) if norms[1] > 0 else float(np.sqrt(norms[0]))
        info["residuals"].append(rel)
        rel, steps = self.refine(U, F, rel, refine, tol, info["residuals"])
        info["refine_steps"] = steps
        info["residual"] = rel
        info["residual_mode"] = self.residual_mode
        return U, info

    @_on_device
    def eval_floor(self):
        """Relative rounding floor of the fp64 residual of the U whose K U the
        last residual() left in Y: eps || |f| + |M_x| |Y1| + |A_x| |Y2| || / ||f||,
        times a small safety factor."""
        self.plan.residual_scale(self.n_t, self.Y.data_ptr(), self.n, self._F.data_ptr(), self.n,
                                 self.norms[2:].data_ptr(), self._stream())
        self.gpu_launches += 2
        s2, f2 = self.norms[2:4].tolist()
        return 4.0 * 2.0 ** -52 * float(np.sqrt(s2) / np.sqrt(f2)) if f2 > 0 else 0.0

    def refine(self, U, F, rel, max_steps, tol, history=None):
        """Iterative refinement u += FD(f - K u) from the residual held in R
        (relative value `rel`, evaluated for this U: K U is still in Y) until
        `tol`, `max_steps`, or stagnation. Compensated residual
        (self.compensated): True -- always; False -- never; "auto" -- once the
        fp64 residual is within FLOOR_MARGIN of its own rounding floor
        (eval_floor, estimated after the first step) while still above `tol`,
        or stagnates above `tol`; refinement on the compensated residual stops
        at max(tol, DD_TOL). Returns (relative residual of U, steps taken)."""
        steps, dd = 0, self.compensated is True
        self.residual_mode = "fp64"
        floor = None  # estimated after the first step, if refinement goes on
        self._F = F
        if dd and rel > tol:
            rel = self._rel(self.residual(U, F, dd=True))
            self.residual_mode = "dd"
        while rel > (max(tol, DD_TOL) if dd else tol) and steps < max_steps:
            new, rel, go = self.refine_step(U, F, rel, dd=dd)
            steps += 1
            if history is not None:
                history.append(new)
            if floor is None and not dd and self.compensated == "auto" and go and rel > tol:
                floor = self.eval_floor()  # Y holds K U of the new iterate
            switch = not dd and self.compensated == "auto" and (not go or rel < FLOOR_MARGIN * (floor or 0.0))
            if not go and not switch:  # stagnation at the evaluation floor (a worse step was undone)
                break
            if switch and rel > tol:
                dd = True
                self.residual_mode = "dd"
                rel = self._rel(self.residual(U, F, dd=True))
                if history is not None:
                    history.append(rel)
            elif not go:
                break
        return rel, steps

    @staticmethod
    def _rel(norms):
        r2, f2 = norms.tolist()
        return float(np.sqrt(r2) / np.sqrt(f2)) if f2 > 0 else float(np.sqrt(r2))
