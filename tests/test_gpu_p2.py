"""P2 in space and time (configuration c5) on the GPU: the FD solve against
the CPU oracle's Bartels-Stewart solution at sizes the oracle finishes in
seconds, and at full c5 size through the space-time residual and the GPU
Bartels-Stewart cross-check BASELINE.json asks for."""

import numpy as np
import pytest

from conftest import rel_diff

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,cells", [(8, 8), (16, 16), (24, 40)])
def test_p2_fd_matches_oracle(cuda_ok, n, cells):
    from oracle import fd_oracle as orc
    from paper_2008_01996_b200 import problems, solvers

    system, info = problems.build_system(mesh=("square", n), n_t=cells, degree=2, grading=2.0,
                                         j_max=200_000)
    sol, rep = solvers.solve_fd(system)
    arrs = orc.system_arrays(system)
    ref = orc.solve_bs_complex(*arrs)
    assert rel_diff(sol.coefficients, ref) < 1e-10
    assert rep.residual < 1e-11
    assert orc.residual(*arrs, sol.coefficients) < 1e-11


def test_p2_fd_matches_gpu_bs(cuda_ok):
    from paper_2008_01996_b200 import bartels_stewart, problems, solvers

    system, _ = problems.build_system(mesh=("square", 16), n_t=24, degree=2, grading=2.0, j_max=200_000)
    a, _ = solvers.solve_fd(system)
    b, rb = bartels_stewart.solve_bs_complex(system)
    assert rel_diff(a.coefficients, b.coefficients) < 1e-10
    assert rb.residual < 1e-11


@pytest.mark.slow
def test_c5_full_size(cuda_ok):
    """c5: M_x = 65,025 (P2 on the 128 grid), 1024 P2 temporal dofs on the
    graded mesh; FD with refinement against the GPU Bartels-Stewart solve."""
    import torch

    from paper_2008_01996_b200 import bartels_stewart, problems, solvers

    system, info = problems.build_system("c5", temporal_device=torch.device("cuda", 0))
    assert info["m_x"] == 65025 and info["n_t"] == 1024
    sol, rep = solvers.solve_fd(system)
    assert rep.min_re_lambda > 0.0
    assert rep.residual < 1e-11
    bs, rbs = bartels_stewart.solve_bs_complex(system)
    assert rbs.residual < 1e-11
    assert rel_diff(sol.coefficients, bs.coefficients) < 1e-10
