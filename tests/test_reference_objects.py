"""The drop-in's host path with objects built by the reference itself
(skipped where /root/reference is absent, e.g. on the GPU box; the GPU side
of the same check is tests/test_gpu_fd.py::test_fd_accepts_reference_pencil)."""

import os
import sys

import numpy as np
import pytest

from conftest import load_golden

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def ks():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from kronheat import solvers

    return solvers


def test_modal_plan_and_report_with_reference_pencil(ks):
    from paper_2008_01996_b200 import solvers
    from paper_2008_01996_b200.engine import modal_plan

    system, ref = load_golden("c1")
    pencil = ks.build_pencil(system.temporal, "fd")
    assert not hasattr(pencil, "spectral_stats")
    plan = modal_plan(system.temporal, pencil)
    assert plan.n_k == system.n_t // 2
    rep = solvers.SolveReport(variant="fd", dof=system.dof, n_t=system.n_t, m_x=system.m_x)
    rep.spectral_source = solvers.spectral_source(pencil)
    assert rep.kappa2 == pytest.approx(float(ref["fd_kappa2"]), rel=1e-12)
    # W_in / W_out invert each other on the retained modes (FD identity on the temporal factor)
    recon = plan.w_in @ plan.w_out
    At_inv = np.linalg.inv(system.temporal.A)
    assert np.linalg.norm(recon - At_inv) / np.linalg.norm(At_inv) < 1e-8


def test_reference_report_fields_match_dropin(ks):
    from paper_2008_01996_b200 import solvers

    ref_fields = [f.name for f in ks.SolveReport.__dataclass_fields__.values()]
    ours = solvers.SolveReport.__dataclass_fields__
    for name in ref_fields:
        assert name in ours, name
    rep = solvers.SolveReport("fd", 1, 1, 1, 0.1, 0.2, 0.3, 0.4, 1e-12, 0.5, 1.0, 2.0, 2.0, 3, 1, None)
    assert (rep.sigma_min, rep.sigma_max, rep.kappa2, rep.threads) == (1.0, 2.0, 2.0, 3)
