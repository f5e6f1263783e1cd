"""The multi-GPU driver (distributed.py) on the real kernels with an NCCL
process group of one rank (the pool gives one GPU; world>1 host logic is
covered by tests/test_multirank.py on gloo)."""

import os
import socket

import numpy as np
import pytest

from conftest import load_golden, rel_diff

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_fd_world1_nccl(cuda_ok):
    import torch
    import torch.distributed as dist

    from paper_2008_01996_b200 import solvers
    from paper_2008_01996_b200.distributed import ShardedFD
    from paper_2008_01996_b200.engine import modal_plan

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        system, ref = load_golden("c1")
        modal = modal_plan(system.temporal, solvers.build_pencil(system.temporal, "fd"))
        run = ShardedFD(system.spatial.M_II, system.spatial.A_II, modal, 0, 1, device=torch.device("cuda", 0))
        F = torch.from_numpy(np.ascontiguousarray(system.rhs)).cuda().view(system.n_t, system.m_x)
        _, info = run.solve(F)
        u = run.gather().reshape(-1).cpu().numpy()
        assert rel_diff(u, ref["bs"]) < 1e-10
        assert info["residual"] < 1e-11

        # public multi-GPU entry point: same rows as solve_fd, host output
        from paper_2008_01996_b200.distributed import solve_fd_sharded

        (r0, r1), U_rows, rep = solve_fd_sharded(system)
        assert (r0, r1) == (0, system.m_x)
        assert U_rows.shape == (system.n_t, system.m_x)
        assert rel_diff(U_rows.reshape(-1), ref["bs"]) < 1e-10
        assert rep.residual < 1e-11
    finally:
        dist.destroy_process_group()
