"""World-size-2 gloo test of the multi-GPU host logic (distributed.py): mode
sharding, the row-chunk layout of the partial back transform, the
reduce-scatter / all-gather plumbing and the shared refinement loop. The
device kernels are emulated with numpy/SuperLU (`_CpuOps`), so this runs on
CPU; the result must equal the single-process solve."""

import os
import socket

import numpy as np
import pytest
import scipy.sparse.linalg as spla
import torch
import torch.multiprocessing as mp

from paper_2008_01996_b200.distributed import restrict_modal, row_chunk, shard_range


class _CpuOps:
    device = torch.device("cpu")

    def __init__(self, M, A, modal):
        self.M, self.A, self.modal = M.tocsc(), A.tocsc(), modal
        self.nk = modal.n_k

    def factor(self, events=None):
        self.lu = [spla.splu((self.M + l * self.A).astype(complex).tocsc()) for l in self.modal.lam]

    def apply_local(self, F):
        Fm = F.numpy().T  # n x N_t
        G = Fm @ self.modal.w_in
        Z = np.zeros((Fm.shape[0], self.nk), complex)
        for k in range(self.nk):
            Z[:, k] = self.lu[k].solve(G[:, k] + 1j * G[:, self.nk + k])
        self.Z = np.hstack([Z.real, Z.imag])

    def out_chunk(self, r0, rows, dst, ldd):
        dst[:, :rows] = torch.from_numpy((self.Z[r0:r0 + rows] @ self.modal.w_out).T)

    def z_rows(self, send, row_blocks):
        for c, (r0, rows) in enumerate(row_blocks):
            if rows:
                send[c, :self.Z.shape[1], :rows] = torch.from_numpy(np.ascontiguousarray(self.Z[r0:r0 + rows].T))

    def gemm_rows(self, recv, wperm, out):
        Zcat = recv.numpy().reshape(-1, recv.shape[2]).T       # rp x K
        out[:] = torch.from_numpy(np.ascontiguousarray((Zcat @ wperm.numpy()).T))

    def y_shard(self, U, rows, ld, dst):
        dst[:, :rows] = torch.from_numpy((U[:, :rows].numpy().T @ self.modal.kron_b).T)

    def residual_full(self, Y, F):
        nt = self.modal.n_t
        Yn = Y.numpy().T
        R = F.numpy().T - (self.M @ Yn[:, :nt] + self.A @ Yn[:, nt:])
        self.R = torch.from_numpy(np.ascontiguousarray(R.T))
        return self.R, float(np.linalg.norm(R) / np.linalg.norm(F.numpy()))

    def axpy_(self, y, x, alpha=1.0):
        y.add_(x, alpha=alpha)


def _worker(rank, world, port, name, out_dir, collective="nccl"):
    import torch.distributed as dist

    from conftest import load_golden
    from paper_2008_01996_b200 import solvers
    from paper_2008_01996_b200.distributed import ShardedFD
    from paper_2008_01996_b200.engine import modal_plan

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    system, _ = load_golden(name)
    modal = modal_plan(system.temporal, solvers.build_pencil(system.temporal, "fd"))
    k0, k1 = shard_range(modal.n_k, world, rank)
    ops = _CpuOps(system.spatial.M_II, system.spatial.A_II, restrict_modal(modal, k0, k1))
    run = ShardedFD(system.spatial.M_II, system.spatial.A_II, modal, rank, world, ops=ops, collective=collective)
    F = torch.from_numpy(np.ascontiguousarray(system.rhs)).view(system.n_t, system.m_x)
    _, info = run.solve(F, refine=3, tol=1e-13)
    U = run.gather()
    np.save(os.path.join(out_dir, f"u{rank}.npy"), U.numpy().ravel())
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(info["residuals"]))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,collective", [("lshape0", "nccl"), ("c1", "nccl"), ("c1", "alltoall"),
                                             ("odd", "alltoall")])
def test_two_ranks_match_reference(tmp_path, name, collective):
    """reduce-scatter of the partial back transforms ("nccl" path) or
    all-to-all of Z by rows + local GEMM ("alltoall")."""
    from conftest import load_golden, rel_diff

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path), collective), nprocs=world, join=True)
    u0, u1 = np.load(tmp_path / "u0.npy"), np.load(tmp_path / "u1.npy")
    assert np.array_equal(u0, u1)  # every rank gathers the same solution
    r0, r1 = np.load(tmp_path / "r0.npy"), np.load(tmp_path / "r1.npy")
    assert np.array_equal(r0, r1)  # identical residual history -> identical control flow
    _, ref = load_golden(name)
    assert rel_diff(u0, ref["bs"]) < 1e-10
    assert r0[-1] < 1e-11


def test_shard_range_covers_all_modes():
    for n in (0, 1, 5, 64, 129):
        for world in (1, 2, 3, 8):
            blocks = [shard_range(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_row_chunks_cover_rows():
    for n, world in ((10, 3), (65025, 8), (1, 4)):
        rp = row_chunk(n, world)
        assert rp * world >= n and rp * (world - 1) < n or n < world
