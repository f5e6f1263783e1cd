"""The CPU oracle (oracle/fd_oracle.py) pinned against outputs of the
reference package itself (tests/golden/*.npz, made by make_golden.py)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel_diff
from oracle import fd_oracle as orc

SMALL = ["lshape0", "odd", "random_11", "random_12", "random_13"]


@pytest.mark.parametrize("name", SMALL + ["c1"])
def test_oracle_fd_matches_reference(name):
    system, ref = load_golden(name)
    u, p = orc.solve_fd(*orc.system_arrays(system))
    assert rel_diff(u, ref["fd"]) < 1e-12
    assert orc.residual(*orc.system_arrays(system), u) == pytest.approx(float(ref["fd_residual"]), rel=1e-6, abs=1e-15)
    assert p["sigma"][0] / p["sigma"][-1] == pytest.approx(float(ref["fd_kappa2"]), rel=1e-10)
    assert np.min(p["D"].real) == pytest.approx(float(ref["fd_min_re_lambda"]), rel=1e-10)


@pytest.mark.parametrize("name", SMALL + ["c1"])
def test_oracle_bs_complex_matches_reference(name):
    system, ref = load_golden(name)
    u = orc.solve_bs_complex(*orc.system_arrays(system))
    assert rel_diff(u, ref["bs"]) < 1e-12
    assert orc.residual(*orc.system_arrays(system), u) < 1e-12


@pytest.mark.parametrize("name", SMALL + ["c1"])
def test_oracle_bs_real_matches_reference(name):
    # bsreal.npz: the reference's solve_bs_real on the same stored systems (make_golden_bsreal.py)
    system, _ = load_golden(name)
    ref = np.load(os.path.join(GOLDEN, "bsreal.npz"))
    u = orc.solve_bs_real(*orc.system_arrays(system))
    assert rel_diff(u, ref[f"{name}_bsr"]) < 1e-12
    assert orc.residual(*orc.system_arrays(system), u) == pytest.approx(float(ref[f"{name}_bsr_residual"]),
                                                                        rel=1e-3, abs=1e-15)


@pytest.mark.parametrize("name", SMALL)
def test_oracle_dense_matches_reference(name):
    system, ref = load_golden(name)
    u = orc.solve_dense(*orc.system_arrays(system))
    assert rel_diff(u, ref["dense"]) < 1e-12


def test_c1_reference_fd_gap_is_documented():
    # the reference FD at config 1 sits ~1e-10 from the backward-stable BS
    # solution (kappa_2(X_t) ~ 8.8e5); this is the floor any faithful FD has
    system, ref = load_golden("c1")
    gap = rel_diff(ref["fd"], ref["bs"])
    assert 1e-12 < gap < 1e-9
    assert float(ref["bs_residual"]) < 1e-13
