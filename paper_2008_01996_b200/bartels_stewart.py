"""Bartels-Stewart with a complex Schur form on the GPU (reference
solvers.py:304-345) -- the FD fallback target of `solve` (solvers.py:457-462)
and the backward-stable cross-check.

All N_t shifted matrices M_x + S_kk A_x are factored in one batched call
(they are independent); only the triangular back-substitution over k is
sequential: rhs_k = G_k - A_x (Z[:, k+1:] S[k, k+1:]^T), a DMMA GEMV plus the
fused CSR residual kernel, then one solve with the retained factors.
`solve_bs_real` (solvers.py:226-301) follows the reference's real-Schur block
recursion; each 2 x 2 block's 2 M_x indefinite system is solved as the
equivalent complex-symmetric M_x system (see its docstring).
"""

import time

import numpy as np

from . import _native, sparse_direct
from .errors import DimensionMismatch, ImaginaryResidueTooLarge, UsageError

BS_IMAG_TOL = 1e-9  # solvers.py:342


def solve_bs_complex(system, pencil=None, leaf_size=sparse_direct.DEFAULT_LEAF_SIZE):
    import torch

    from .dense import ComplexSchurForm, spd_solve
    from .engine import _fortran
    from .solvers import SolveReport, SpaceTimeSolution, build_pencil, residual

    _native.require_cuda()
    report = SolveReport(variant="bs-complex", dof=system.dof, n_t=system.n_t, m_x=system.m_x)
    t0 = time.perf_counter()
    if pencil is None:
        pencil = build_pencil(system.temporal, "bs-complex")
    if not isinstance(pencil.form, ComplexSchurForm) and not hasattr(pencil.form, "S"):
        raise DimensionMismatch("solve_bs_complex needs a complex Schur pencil")
    W, S = pencil.form.W, pencil.form.S
    n, nt = system.m_x, system.n_t
    w_in_c = spd_solve(pencil.chol_A, np.conj(W))             # G = F A^-1 conj(W)
    w_in = np.hstack([w_in_c.real, w_in_c.imag])              # N_t x 2N_t
    wt = W.T
    w_out = np.vstack([wt.real, -wt.imag])                    # 2N_t x N_t: Re(Z W^T)
    w_out_im = np.vstack([wt.imag, wt.real])                  # Im(Z W^T)
    # per-row GEMV operands: B1_k = [Re S[k,:], Im S[k,:]], B2_k = [-Im S[k,:], Re S[k,:]]
    b1 = np.stack([np.stack([S.real[k], S.imag[k]]) for k in range(nt)])   # (N_t, 2, N_t)
    b2 = np.stack([np.stack([-S.imag[k], S.real[k]]) for k in range(nt)])
    lam = np.ascontiguousarray(np.diag(S).astype(np.complex128))
    report.t_decompose = time.perf_counter() - t0
    report.min_re_lambda = pencil.min_re_lambda

    dev = torch.device("cuda", torch.cuda.current_device())
    f64 = torch.float64
    st = _native.stream_handle()
    t0 = time.perf_counter()
    F = torch.from_numpy(np.ascontiguousarray(system.rhs, dtype=np.float64)).to(dev)
    d_win = _fortran(w_in, dev)
    G = torch.empty((2 * nt, n), dtype=f64, device=dev)
    _native.call("kh_dgemm", n, 2 * nt, nt, 1.0, F.data_ptr(), n, d_win.data_ptr(), nt, 0.0, G.data_ptr(), n, st)
    torch.cuda.synchronize()
    report.t_transform_in = time.perf_counter() - t0

    t0 = time.perf_counter()
    before = sparse_direct.analyze_call_count()
    M = system.spatial.M_II.tocsr()
    A = system.spatial.A_II.tocsr()
    sym = sparse_direct.analyze((M + A).tocsr(), leaf_size)
    mv, av = sym.align_values(M), sym.align_values(A)
    free, _ = torch.cuda.mem_get_info(dev)
    # blocks torch has cached but not handed out are free for the plan too
    free += torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
    batch = nt
    while batch > 1 and sparse_direct.plan_bytes(sym, batch, nt) > 0.7 * free:
        batch = (batch + 1) // 2
    if sparse_direct.plan_bytes(sym, batch, nt) > 0.7 * free:
        raise UsageError("bs-complex needs every shift's factors resident; not enough device memory")
    plan = sparse_direct._Plan(sym, mv, av, batch, nt, dev.index)
    for s0 in range(0, nt, batch):
        plan.factor(s0, lam[s0:s0 + batch], st)
    plan.pivot_check(0, nt, st)
    d_ptr = torch.from_numpy(sym.indptr).to(dev)
    d_idx = torch.from_numpy(sym.indices).to(dev)
    d_mv = torch.from_numpy(mv).to(dev)
    d_av = torch.from_numpy(av).to(dev)
    d_b1 = torch.from_numpy(np.ascontiguousarray(b1)).to(dev)
    d_b2 = torch.from_numpy(np.ascontiguousarray(b2)).to(dev)
    Z = torch.zeros((2 * nt, n), dtype=f64, device=dev)
    Y = torch.zeros((4, n), dtype=f64, device=dev)   # [0 | 0 | c_re | c_im]
    R = torch.empty((2, n), dtype=f64, device=dev)
    norms = torch.zeros(2, dtype=f64, device=dev)
    zp, gp, yp, rp = Z.data_ptr(), G.data_ptr(), Y.data_ptr(), R.data_ptr()
    for k in range(nt - 1, -1, -1):
        m = nt - k - 1
        if m > 0:
            # c = Z[:, k+1:] S[k, k+1:]^T  (complex, as two real GEMMs into Y[:, 2:4])
            off = 8 * (k * 2 * nt + k + 1)
            _native.call("kh_dgemm", n, 2, m, 1.0, zp + 8 * (k + 1) * n, n, d_b1.data_ptr() + off, nt, 0.0,
                         yp + 16 * n, n, st)
            _native.call("kh_dgemm", n, 2, m, 1.0, zp + 8 * (nt + k + 1) * n, n, d_b2.data_ptr() + off, nt, 1.0,
                         yp + 16 * n, n, st)
        # rhs = G[:, k] - A_x c  (F columns: G_re[:, k] and G_im[:, k], ldf = N_t * n)
        _native.call("kh_csr_pair_residual", n, 2, d_ptr.data_ptr(), d_idx.data_ptr(), d_mv.data_ptr(),
                     d_av.data_ptr(), yp, n, gp + 8 * k * n, nt * n, rp, n, norms.data_ptr(), st)
        plan.solve(k, 1, rp, rp + 8 * n, n, zp + 8 * k * n, zp + 8 * (nt + k) * n, n, st)
    torch.cuda.synchronize()
    report.analyze_calls = sparse_direct.analyze_call_count() - before
    report.t_spatial = time.perf_counter() - t0

    t0 = time.perf_counter()
    U = torch.empty((nt, n), dtype=f64, device=dev)
    d_wout = _fortran(w_out, dev)
    d_wim = _fortran(w_out_im, dev)
    _native.call("kh_dgemm", n, nt, 2 * nt, 1.0, zp, n, d_wout.data_ptr(), 2 * nt, 0.0, U.data_ptr(), n, st)
    Ui = torch.empty((nt, n), dtype=f64, device=dev)
    _native.call("kh_dgemm", n, nt, 2 * nt, 1.0, zp, n, d_wim.data_ptr(), 2 * nt, 0.0, Ui.data_ptr(), n, st)
    nrm = torch.zeros(2, dtype=f64, device=dev)
    _native.call("kh_sumsq", U.data_ptr(), n * nt, nrm.data_ptr(), st)
    _native.call("kh_sumsq", Ui.data_ptr(), n * nt, nrm.data_ptr() + 8, st)
    u2, i2 = nrm.tolist()
    tot = np.sqrt(u2 + i2)
    if tot > 0 and np.sqrt(i2) > BS_IMAG_TOL * tot:
        raise ImaginaryResidueTooLarge(f"imaginary residue {np.sqrt(i2) / tot:.3e} above {BS_IMAG_TOL:.1e}")
    coeffs = U.reshape(-1).cpu().numpy()
    report.t_transform_out = time.perf_counter() - t0
    report.imag_residue = float(np.sqrt(i2) / tot) if tot > 0 else 0.0
    report.residual = residual(system, coeffs)
    return SpaceTimeSolution(coefficients=coeffs), report


def _real_schur_blocks(R):
    """Diagonal blocks of a standardized real Schur form (LAPACK dgees):
    (k, k) for a real eigenvalue, (k-1, k) for a 2 x 2 block [[a, b1], [b2, a]]
    with b1 b2 < 0, scanned from the bottom as the reference does
    (solvers.py:256-257)."""
    blocks, k = [], R.shape[0] - 1
    while k >= 0:
        if k == 0 or R[k, k - 1] == 0.0:
            blocks.append((k, k))
            k -= 1
        else:
            blocks.append((k - 1, k))
            k -= 2
    return blocks


def solve_bs_real(system, pencil=None, leaf_size=sparse_direct.DEFAULT_LEAF_SIZE):
    """Bartels-Stewart with a real Schur form (reference solvers.py:226-301).

    Same block back-substitution over the quasi-triangular R as the
    reference, the spatial systems on the GPU. A real eigenvalue R_kk is one
    shifted system M_x + R_kk A_x (solvers.py:258-268). A standardized 2 x 2
    block [[a, b1], [b2, a]] couples z_{k-1}, z_k through
        D z_{k-1} + b1 A z_k = r1,   b2 A z_{k-1} + D z_k = r2   (D = M + a A),
    which the reference solves as one scaled 2 M_x symmetric-indefinite system
    (solvers.py:269-289). Here the same pair is ONE complex-symmetric M_x
    system: with beta = sqrt(-b1 b2) and c = beta / b2,
        (M + (a + i beta) A) w = r1 + i c r2,   z_{k-1} = Re w,  z_k = Im w / c,
    (expand and use beta^2 = -b1 b2), so it goes through the batched pivot-free
    LDL^T with the shifted matrices of bs-complex/FD (M_x + lambda A_x with
    Re lambda > 0 is complex symmetric with an SPD real part; the indefinite
    real 2 M_x form would need pivoting). The solution is the same up to
    rounding; one symbolic analysis serves every block (the reference runs a
    second one for the 2 M_x pattern: `analyze_calls` is 1 here).
    """
    import torch

    from .dense import RealSchurForm, spd_solve
    from .engine import _fortran
    from .solvers import SolveReport, SpaceTimeSolution, build_pencil, residual

    _native.require_cuda()
    report = SolveReport(variant="bs-real", dof=system.dof, n_t=system.n_t, m_x=system.m_x)
    t0 = time.perf_counter()
    if pencil is None:
        pencil = build_pencil(system.temporal, "bs-real")
    if not isinstance(pencil.form, RealSchurForm) and not hasattr(pencil.form, "R"):
        raise DimensionMismatch("solve_bs_real needs a real Schur pencil")
    Q, Rs = np.asarray(pencil.form.Q, dtype=np.float64), np.asarray(pencil.form.R, dtype=np.float64)
    n, nt = system.m_x, system.n_t
    blocks = _real_schur_blocks(Rs)
    lam = np.empty(len(blocks), dtype=np.complex128)
    scale = np.ones(len(blocks))
    for s, (i, k) in enumerate(blocks):
        if i == k:
            lam[s] = Rs[k, k]
        else:
            a, b1, b2 = Rs[i, i], Rs[i, k], Rs[k, i]
            if b1 * b2 >= 0.0:
                raise DimensionMismatch("real Schur 2 x 2 block is not standardized (b1 b2 >= 0)")
            beta = np.sqrt(-b1 * b2)
            lam[s] = complex(a, beta)
            scale[s] = beta / b2
    w_in = spd_solve(pencil.chol_A, Q)                         # G = F A_t^-1 Q
    report.t_decompose = time.perf_counter() - t0
    report.min_re_lambda = pencil.min_re_lambda

    dev = torch.device("cuda", torch.cuda.current_device())
    f64 = torch.float64
    st = _native.stream_handle()
    t0 = time.perf_counter()
    F = torch.from_numpy(np.ascontiguousarray(system.rhs, dtype=np.float64)).to(dev)
    d_win = _fortran(w_in, dev)
    G = torch.empty((nt, n), dtype=f64, device=dev)
    _native.call("kh_dgemm", n, nt, nt, 1.0, F.data_ptr(), n, d_win.data_ptr(), nt, 0.0, G.data_ptr(), n, st)
    torch.cuda.synchronize()
    report.t_transform_in = time.perf_counter() - t0

    t0 = time.perf_counter()
    before = sparse_direct.analyze_call_count()
    M = system.spatial.M_II.tocsr()
    A = system.spatial.A_II.tocsr()
    sym = sparse_direct.analyze((M + A).tocsr(), leaf_size)
    mv, av = sym.align_values(M), sym.align_values(A)
    ns = len(blocks)
    free, _ = torch.cuda.mem_get_info(dev)
    free += torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
    batch = ns
    while batch > 1 and sparse_direct.plan_bytes(sym, batch, ns) > 0.7 * free:
        batch = (batch + 1) // 2
    if sparse_direct.plan_bytes(sym, batch, ns) > 0.7 * free:
        raise UsageError("bs-real needs every block's factors resident; not enough device memory")
    plan = sparse_direct._Plan(sym, mv, av, batch, ns, dev.index)
    for s0 in range(0, ns, batch):
        plan.factor(s0, lam[s0:s0 + batch], st)
    plan.pivot_check(0, ns, st)
    d_ptr = torch.from_numpy(sym.indptr).to(dev)
    d_idx = torch.from_numpy(sym.indices).to(dev)
    d_mv = torch.from_numpy(mv).to(dev)
    d_av = torch.from_numpy(av).to(dev)
    d_rt = _fortran(np.ascontiguousarray(Rs.T), dev)            # column j of R^T = row j of R
    Z = torch.zeros((nt, n), dtype=f64, device=dev)
    # residual operands [Y1 | Y2] = [0 | C]: one buffer per block width, Y1 never written
    Ys = {1: torch.zeros((2, n), dtype=f64, device=dev), 2: torch.zeros((4, n), dtype=f64, device=dev)}
    Rr = torch.empty((2, n), dtype=f64, device=dev)
    Wi = torch.empty((1, n), dtype=f64, device=dev)
    zero = torch.zeros((1, n), dtype=f64, device=dev)
    norms = torch.zeros(2, dtype=f64, device=dev)
    zp, gp, rp, rtp = Z.data_ptr(), G.data_ptr(), Rr.data_ptr(), d_rt.data_ptr()
    for s, (i, k) in enumerate(blocks):
        w = k - i + 1                                           # 1 or 2 coupled columns
        m = nt - k - 1
        yp = Ys[w].data_ptr()
        if m > 0:   # (the first block has C = 0: its buffer is still zero)
            # C = Z[:, k+1:] R[i:k+1, k+1:]^T  (acc of solvers.py:265-267, :284-288)
            _native.call("kh_dgemm", n, w, m, 1.0, zp + 8 * (k + 1) * n, n, rtp + 8 * ((k + 1) + i * nt), nt,
                         0.0, yp + 8 * w * n, n, st)
        # rhs = G[:, i:k+1] - A_x C
        _native.call("kh_csr_pair_residual", n, w, d_ptr.data_ptr(), d_idx.data_ptr(), d_mv.data_ptr(),
                     d_av.data_ptr(), yp, n, gp + 8 * i * n, n, rp, n, norms.data_ptr(), st)
        if w == 1:
            plan.solve(s, 1, rp, zero.data_ptr(), n, zp + 8 * k * n, Wi.data_ptr(), n, st)
            continue
        c = scale[s]
        _native.call("kh_daxpy", n, c - 1.0, rp + 8 * n, rp + 8 * n, st)          # r2 <- c r2
        plan.solve(s, 1, rp, rp + 8 * n, n, zp + 8 * i * n, zp + 8 * k * n, n, st)
        _native.call("kh_daxpy", n, 1.0 / c - 1.0, zp + 8 * k * n, zp + 8 * k * n, st)  # z_k = Im w / c
    torch.cuda.synchronize()
    report.analyze_calls = sparse_direct.analyze_call_count() - before
    report.t_spatial = time.perf_counter() - t0

    t0 = time.perf_counter()
    U = torch.empty((nt, n), dtype=f64, device=dev)
    d_qt = _fortran(np.ascontiguousarray(Q.T), dev)
    _native.call("kh_dgemm", n, nt, nt, 1.0, zp, n, d_qt.data_ptr(), nt, 0.0, U.data_ptr(), n, st)
    coeffs = U.reshape(-1).cpu().numpy()
    report.t_transform_out = time.perf_counter() - t0
    report.residual = residual(system, coeffs)
    return SpaceTimeSolution(coefficients=coeffs), report
