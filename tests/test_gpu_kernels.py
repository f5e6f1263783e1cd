"""GPU parity of the native kernels through the C-ABI: DMMA GEMM and the
batched multifrontal LDL^T (ports of the reference's sparse_direct contracts,
pkg/tests/test_sparse_direct.py)."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import load_golden, rel_diff
from paper_2008_01996_b200 import _native
from paper_2008_01996_b200 import sparse_direct as sd
from paper_2008_01996_b200.errors import DimensionMismatch, SingularMatrix

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (7, 5, 3), (129, 65, 17), (1000, 256, 256), (4097, 130, 33)])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_dgemm_matches_numpy(cuda_ok, m, n, k, beta):
    import torch

    rng = np.random.default_rng(m + n + k)
    A = rng.standard_normal((m, k))
    B = rng.standard_normal((k, n))
    C0 = rng.standard_normal((m, n))
    dA, dB, dC = _dev(A.T), _dev(B.T), _dev(C0.T)  # column-major storage
    _native.call("kh_dgemm", m, n, k, 1.5, dA.data_ptr(), m, dB.data_ptr(), k, beta, dC.data_ptr(), m,
                 _native.stream_handle())
    got = dC.cpu().numpy().T
    want = 1.5 * A @ B + beta * C0
    assert np.max(np.abs(got - want)) <= 1e-13 * max(1.0, np.max(np.abs(want))) * np.sqrt(k)
    torch.cuda.synchronize()


def test_dgemm_strided_lda(cuda_ok):
    rng = np.random.default_rng(5)
    m, n, k, lda = 301, 40, 57, 333
    A = rng.standard_normal((lda, k))
    B = rng.standard_normal((k, n))
    dA, dB = _dev(A.T), _dev(B.T)
    import torch

    dC = torch.zeros((n, m), dtype=torch.float64, device="cuda")
    _native.call("kh_dgemm", m, n, k, 1.0, dA.data_ptr(), lda, dB.data_ptr(), k, 0.0, dC.data_ptr(), m,
                 _native.stream_handle())
    assert np.allclose(dC.cpu().numpy().T, A[:m] @ B, rtol=1e-13, atol=1e-12)


def laplacian_1d(n):
    return sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(n, n), format="csr")


def grid_5pt(k):
    I = sp.identity(k, format="csr")
    T = laplacian_1d(k)
    return (sp.kron(I, T) + sp.kron(T, I)).tocsr()


def test_identity(cuda_ok):
    sym = sd.analyze(sp.identity(4, format="csr"))
    num = sd.factorize(sym, sp.identity(4, format="csr"))
    assert np.allclose(num.solve(np.arange(4.0)), np.arange(4.0))


def test_laplacian_eigenfunction(cuda_ok):
    n = 1023
    h = 1.0 / (n + 1)
    x = np.linspace(h, 1.0 - h, n)
    sol = sd.factor_solve(laplacian_1d(n) / h**2, np.sin(np.pi * x))
    assert np.max(np.abs(sol - np.sin(np.pi * x) / np.pi**2)) < 5 * h**2


def test_multi_rhs_matches_columns(cuda_ok):
    rng = np.random.default_rng(4)
    A = grid_5pt(8) + sp.identity(64)
    B = rng.standard_normal((64, 5))
    num = sd.factorize(sd.analyze(A), A)
    X = num.solve(B)
    for j in range(5):
        assert np.allclose(X[:, j], num.solve(B[:, j]), atol=1e-14)


def test_pattern_reuse_across_shifts(cuda_ok):
    rng = np.random.default_rng(9)
    M = grid_5pt(6)
    A = sp.identity(36, format="csr")
    sym = sd.analyze((M + A).tocsr())
    for alpha in (0.5, 2.0, 17.0):
        K = (M + alpha * A).tocsr()
        b = rng.standard_normal(36)
        x = sd.factorize(sym, K).solve(b)
        assert np.linalg.norm(K @ x - b) / np.linalg.norm(b) < 1e-12


def test_complex_symmetric_matches_real_block_oracle(cuda_ok):
    rng = np.random.default_rng(12)
    n = 30
    M = (laplacian_1d(n) + sp.identity(n)).tocsr()
    A = laplacian_1d(n)
    lam = 0.7 + 1.9j
    K = (M + lam * A).astype(complex).tocsr()
    f = rng.standard_normal(n)
    z = sd.factor_solve(K, f.astype(complex))
    Mr = (M + lam.real * A).toarray()
    Ai = (lam.imag * A).toarray()
    xy = np.linalg.solve(np.block([[Mr, -Ai], [-Ai, -Mr]]), np.concatenate([f, np.zeros(n)]))
    oracle = xy[:n] + 1j * xy[n:]
    assert np.linalg.norm(z - oracle) / np.linalg.norm(oracle) < 1e-10


def test_singular_matrix_detected(cuda_ok):
    bad = sp.csr_matrix(np.array([[1.0, 1.0], [1.0, 1.0]]))
    with pytest.raises(SingularMatrix):
        sd.factorize(sd.analyze(bad), bad)


def test_deterministic_factorization(cuda_ok):
    A = grid_5pt(10) + sp.identity(100)
    sym = sd.analyze(A)
    b = np.random.default_rng(1).standard_normal(100)
    x1 = sd.factorize(sym, A).solve(b)
    x2 = sd.factorize(sym, A).solve(b)
    assert np.array_equal(x1, x2)


def test_refinement_keeps_residual_small(cuda_ok):
    rng = np.random.default_rng(30)
    A = grid_5pt(12) * 1e6 + sp.identity(144)
    b = rng.standard_normal(144)
    x = sd.factorize(sd.analyze(A), A).solve(b, refine=True)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12


def test_rhs_dimension_check(cuda_ok):
    num = sd.factorize(sd.analyze(sp.identity(4, format="csr")), sp.identity(4, format="csr"))
    with pytest.raises(DimensionMismatch):
        num.solve(np.ones(5))


@pytest.mark.parametrize("mesh,small_max,leaf,warp", [
    (("square", 40), None, None, None), (("lshape", 4), None, None, None), (("square", 128), None, None, None),
    # every front through the level-synchronous large-front kernels
    (("square", 64), "0", None, None), (("lshape", 4), "0", None, None),
    # fused classes capped at m <= 64 / leaves large enough for the 96 and 128 classes
    (("square", 64), "64", None, None), (("square", 96), None, 80, None), (("square", 64), None, 8, None),
    # the fused m <= 128 class (off by default: those fronts take the large-front path)
    (("square", 96), "128", 80, None),
    # m <= 48 through the shared-memory fused kernel instead of the register-resident warp kernel
    (("square", 64), None, None, "0"), (("lshape", 4), None, 16, "0"),
    # warp kernels with small leaves (partial 8-pivot blocks, p < 8)
    (("square", 64), None, 5, None), (("lshape", 4), None, 11, None)])
def test_batched_shifts_match_superlu(cuda_ok, monkeypatch, mesh, small_max, leaf, warp):
    """Many complex shifts M + lam_k A in one batched factorization vs SuperLU,
    through every front-class code path (KH_SMALL_MAX caps the fused classes,
    KH_WARP_CLASSES selects the register-resident warp kernels)."""
    import torch

    from paper_2008_01996_b200 import fem, problems

    if small_max is not None:
        monkeypatch.setenv("KH_SMALL_MAX", small_max)
    if warp is not None:
        monkeypatch.setenv("KH_WARP_CLASSES", warp)
    ops = fem.assemble_p1(problems.spatial_mesh(*mesh))
    M, A = ops.M_II.tocsr(), ops.A_II.tocsr()
    n = M.shape[0]
    rng = np.random.default_rng(3)
    lam = rng.uniform(0.01, 3.0, 9) + 1j * rng.uniform(-40.0, 40.0, 9)
    sym = sd.analyze((M + A).tocsr(), **({} if leaf is None else {"leaf_size": leaf}))
    plan = sd._Plan(sym, sym.align_values(M), sym.align_values(A), 4, 9, torch.cuda.current_device())
    st = _native.stream_handle()
    for s0 in range(0, 9, 4):
        plan.factor(s0, lam[s0:s0 + 4], st)
    plan.pivot_check(0, 9, st)
    B = rng.standard_normal((n, 9)) + 1j * rng.standard_normal((n, 9))
    bre, bim = _dev(B.real.T), _dev(B.imag.T)
    xre = torch.empty_like(bre)
    xim = torch.empty_like(bim)
    for s0 in range(0, 9, 4):
        c = min(4, 9 - s0)
        plan.solve(s0, c, bre.data_ptr() + 8 * s0 * n, bim.data_ptr() + 8 * s0 * n, n,
                   xre.data_ptr() + 8 * s0 * n, xim.data_ptr() + 8 * s0 * n, n, st)
    X = xre.cpu().numpy().T + 1j * xim.cpu().numpy().T
    for k in range(9):
        K = (M + lam[k] * A).astype(complex).tocsc()
        ref = spla.spsolve(K, B[:, k])
        assert np.linalg.norm(X[:, k] - ref) / np.linalg.norm(ref) < 1e-11, k
        assert np.linalg.norm(K @ X[:, k] - B[:, k]) / np.linalg.norm(B[:, k]) < 1e-12


@pytest.mark.parametrize("ns", [1, 5, 9, 22])
def test_shift_lanes_do_not_change_the_bits(cuda_ok, monkeypatch, ns):
    """A batch walks the tree in 1..4 lanes of shifts on separate stream sets
    (KH_LANES / KH_SOLVE_LANES, read at plan creation): ragged splits (lanes
    of 4k shifts, a short last lane, fewer shifts than lanes) and every lane
    count give bitwise the same solution, which matches SuperLU."""
    import torch

    from paper_2008_01996_b200 import fem, problems

    ops = fem.assemble_p1(problems.spatial_mesh("square", 64))
    M, A = ops.M_II.tocsr(), ops.A_II.tocsr()
    n = M.shape[0]
    rng = np.random.default_rng(11)
    lam = rng.uniform(0.01, 3.0, ns) + 1j * rng.uniform(-40.0, 40.0, ns)
    B = rng.standard_normal((n, ns)) + 1j * rng.standard_normal((n, ns))
    sym = sd.analyze((M + A).tocsr())
    mv, av = sym.align_values(M), sym.align_values(A)
    st = _native.stream_handle()
    out = {}
    monkeypatch.setenv("KH_LANES_MIN_WORK", "0")  # small batches run in one lane by default
    for fl, sl in [(1, 1), (2, 2), (3, 2), (4, 4), (2, 1)]:
        monkeypatch.setenv("KH_LANES", str(fl))
        monkeypatch.setenv("KH_SOLVE_LANES", str(sl))
        plan = sd._Plan(sym, mv, av, ns, ns, torch.cuda.current_device())
        plan.factor(0, lam, st)
        plan.pivot_check(0, ns, st)
        bre, bim = _dev(B.real.T), _dev(B.imag.T)
        xre, xim = torch.empty_like(bre), torch.empty_like(bim)
        plan.solve(0, ns, bre.data_ptr(), bim.data_ptr(), n, xre.data_ptr(), xim.data_ptr(), n, st)
        out[(fl, sl)] = xre.cpu().numpy().T + 1j * xim.cpu().numpy().T
        del plan
    base = out[(1, 1)]
    for key, X in out.items():
        assert np.array_equal(X, base), key
    for k in (0, ns - 1):
        K = (M + lam[k] * A).astype(complex).tocsc()
        assert np.linalg.norm(K @ base[:, k] - B[:, k]) / np.linalg.norm(B[:, k]) < 1e-12, k


def test_many_shifts_wide_level_kernels(cuda_ok):
    """160 shifts in one batch: the large-front levels exceed the narrow-level
    CTA threshold, so the wide-level solve kernels run (the 9-shift cases above
    use the narrow ones)."""
    import torch

    from paper_2008_01996_b200 import fem, problems

    ops = fem.assemble_p1(problems.spatial_mesh("square", 96))
    M, A = ops.M_II.tocsr(), ops.A_II.tocsr()
    n, ns = M.shape[0], 160
    rng = np.random.default_rng(8)
    lam = rng.uniform(0.01, 3.0, ns) + 1j * rng.uniform(-40.0, 40.0, ns)
    sym = sd.analyze((M + A).tocsr())
    plan = sd._Plan(sym, sym.align_values(M), sym.align_values(A), ns, ns, torch.cuda.current_device())
    st = _native.stream_handle()
    plan.factor(0, lam, st)
    plan.pivot_check(0, ns, st)
    B = rng.standard_normal((n, ns)) + 1j * rng.standard_normal((n, ns))
    bre, bim = _dev(B.real.T), _dev(B.imag.T)
    xre, xim = torch.empty_like(bre), torch.empty_like(bim)
    plan.solve(0, ns, bre.data_ptr(), bim.data_ptr(), n, xre.data_ptr(), xim.data_ptr(), n, st)
    X = xre.cpu().numpy().T + 1j * xim.cpu().numpy().T
    for k in (0, 57, 159):
        K = (M + lam[k] * A).astype(complex).tocsc()
        assert np.linalg.norm(K @ X[:, k] - B[:, k]) / np.linalg.norm(B[:, k]) < 1e-12, k


@pytest.mark.gpu
@pytest.mark.parametrize("key,j_max", [("graded8", 100_000), ("uniform32", 2_000_000)])
def test_native_temporal_assembly_matches_reference_fixture(cuda_ok, key, j_max):
    """kh_ht_assemble (csrc/temporal.cu) against the reference's own
    assemble_temporal_operators output (tests/golden/temporal.npz)."""
    import torch

    from conftest import GOLDEN
    from paper_2008_01996_b200 import temporal

    z = np.load(f"{GOLDEN}/temporal.npz")
    nodes = z["graded8_nodes"] if key == "graded8" else np.linspace(0.0, 1.0, 33)
    t = temporal.assemble_temporal_operators(temporal.TemporalMesh(nodes), j_max=j_max,
                                             device=torch.device("cuda", 0))
    for mat, name in ((t.A, "A"), (t.M, "M"), (t.C, "C")):
        ref = z[f"{key}_{name}"]
        assert np.abs(mat - ref).max() < 1e-13 * np.abs(ref).max(), name
    assert np.array_equal(t.A, t.A.T)


@pytest.mark.gpu
@pytest.mark.parametrize("nodes", [(np.arange(17) / 16.0) ** 2, np.linspace(0.0, 2.0, 41)])
def test_native_temporal_p2_matches_host(cuda_ok, nodes):
    import torch

    from paper_2008_01996_b200 import p2, temporal

    tm = temporal.TemporalMesh(nodes)
    host = p2.assemble_temporal_operators_p2(tm, j_max=300_000)
    dev = p2.assemble_temporal_operators_p2(tm, j_max=300_000, device=torch.device("cuda", 0))
    # low frequencies on the small graded cells cancel in the closed forms
    # (q'' [cos] / w^2 against q' [sin] / w): host (np.sin of the rounded
    # product) and device (sincospi) agree to ~1e-13 of the largest entry
    for a, b in ((host.A, dev.A), (host.M, dev.M), (host.C, dev.C)):
        assert np.abs(a - b).max() < 1e-11 * np.abs(a).max()


# ---- compensated residual pieces (residual.cu) ---------------------------------
def test_dgemm_dd_matches_extended_precision(cuda_ok):
    """kh_dgemm_dd: hi + lo within a few ulps of extended precision relative
    to |A| |B| even where the fp64 product cancels."""
    import torch

    from paper_2008_01996_b200 import _native

    rng = np.random.default_rng(0)
    m, n, k = 300, 70, 513
    A = rng.standard_normal((m, k))
    B = rng.standard_normal((k, n))
    B[:, :35] -= B[:, :35].mean(axis=0)
    Ad = torch.from_numpy(A.ravel(order="F")).cuda()
    Bd = torch.from_numpy(B.ravel(order="F")).cuda()
    hi = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    lo = torch.zeros_like(hi)
    _native.call("kh_dgemm_dd", m, n, k, Ad.data_ptr(), m, Bd.data_ptr(), k, hi.data_ptr(), lo.data_ptr(), m,
                 _native.stream_handle())
    got = (hi.cpu().numpy().reshape(m, n, order="F").astype(np.longdouble)
           + lo.cpu().numpy().reshape(m, n, order="F").astype(np.longdouble))
    want = A.astype(np.longdouble) @ B.astype(np.longdouble)
    scale = (np.abs(A) @ np.abs(B)).astype(np.longdouble)
    err = float(np.max(np.abs(got - want) / scale))
    err64 = float(np.max(np.abs((A @ B) - want) / scale))
    assert err < 1e-18 and err < 1e-2 * err64, (err, err64)


def test_compensated_residual_matches_oracle_on_c1(cuda_ok):
    """solvers.residual(compensated=True) == the fp64 one (and the oracle's)
    where fp64 is accurate (c1), for both reference solutions."""
    from oracle import fd_oracle as orc
    from paper_2008_01996_b200 import solvers

    system, ref = load_golden("c1")
    for key in ("fd", "bs"):
        want = orc.residual(*orc.system_arrays(system), ref[key])
        got = solvers.residual(system, ref[key], compensated=True)
        assert got == pytest.approx(want, rel=1e-4, abs=1e-16)
    rows = np.arange(0, system.m_x, 97)
    _, rel_ld = orc.residual_rows_longdouble(*orc.system_arrays(system), ref["fd"], rows)
    _, rel_ld_bs = orc.residual_rows_longdouble(*orc.system_arrays(system), ref["bs"], rows)
    assert rel_ld > 0 and rel_ld_bs > 0


def test_engine_compensated_refinement_c1(cuda_ok):
    """FDEngine with compensated=True refines on the compensated residual and
    reaches the reference BS solution."""
    import torch

    from paper_2008_01996_b200 import solvers
    from paper_2008_01996_b200.engine import FDEngine, modal_plan

    system, ref = load_golden("c1")
    modal = modal_plan(system.temporal, solvers.build_pencil(system.temporal, "fd"))
    F = torch.from_numpy(np.ascontiguousarray(system.rhs)).cuda().view(system.n_t, system.m_x)
    eng = FDEngine(system.spatial.M_II, system.spatial.A_II, modal)
    eng.compensated = True
    U, info = eng.solve(F)
    assert info["residual_mode"] == "dd" and info["residual"] < 1e-13
    assert rel_diff(U.cpu().numpy().ravel(), ref["bs"]) < 1e-10
