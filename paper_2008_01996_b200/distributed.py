"""Multi-GPU FD: shifts sharded over ranks, back transform finished by a
reduce-scatter by spatial rows (BASELINE.json north star).

One process per GPU (torchrun). Rank r owns a contiguous block of the N_k
modal shifts (conjugate-pair representatives first). Per FD application:

1. G_r = F W_in[:, modes_r]              local DMMA GEMM (F is resident on every rank)
2. Z_r = (M_x + lambda_k A_x)^-1 G_r      local batched LDL^T solves
3. P_r[c] = Z_r[rows_c, :] W_out[modes_r, :]   partial back transform, written
                                          directly in row-chunk layout (chunk c =
                                          spatial rows of rank c, column-major)
4. U_shard = sum_r P_r[rank]              NCCL reduce-scatter (the cross-mode sum)

Refinement needs K u: Y_shard = U_shard [A_t^T | M_t^T] is row-local; the
Y shards are all-gathered and every rank forms the full residual
R = F - (M_x Y1 + A_x Y2) (a cheap SpMM) so that step 1 of the next
application again has all spatial rows. Norms are then identical on every
rank, so the refinement loop takes the same branch everywhere.

The device work is behind `ops` (default: the FDEngine kernels); the
collectives are plain torch.distributed calls, so the same driver runs on
NCCL/GPU and, in tests, on gloo/CPU with an emulated `ops`.

Steps 3-4 have two implementations (`collective=`):
  "nccl": per destination chunk a local GEMM into P_r[c], then
          `reduce_scatter_tensor` (the baseline);
  "p2p":  ONE GEMM kernel (`kh_dgemm_rowscatter`) writes each finished tile of
          P_r[c] straight into rank c's receive slot r through CUDA-IPC peer
          mappings over NVLink, so the transfer overlaps the math tile by tile;
          after a barrier each rank sums its g slots in rank order
          (`kh_sum_parts`: deterministic, identical to the NCCL result up to
          the summation order).
"""

import math

import numpy as np

from .engine import REFINE_MIN_GAIN, ModalPlan


def shard_range(n_items, world, rank):
    """Balanced contiguous block [k0, k1) of n_items for `rank`."""
    base, extra = divmod(n_items, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def row_chunk(n, world):
    """Rows per chunk of the reduce-scatter (last chunk padded)."""
    return max(1, math.ceil(n / world))


def restrict_modal(modal, k0, k1):
    nk = modal.n_k
    cols = np.r_[k0:k1, nk + k0:nk + k1]
    n_pairs = int(np.clip(modal.n_pairs - k0, 0, k1 - k0))
    return ModalPlan(n_t=modal.n_t, lam=modal.lam[k0:k1].copy(), weight=modal.weight[k0:k1].copy(),
                     n_pairs=n_pairs, n_single=(k1 - k0) - n_pairs,
                     w_in=np.ascontiguousarray(modal.w_in[:, cols]),
                     w_out=np.ascontiguousarray(modal.w_out[cols, :]), kron_b=modal.kron_b)


class EngineOps:
    """Device primitives of one rank on top of FDEngine (libkhb200 kernels)."""

    def __init__(self, engine):
        self.e = engine

    def factor(self, events=None):
        """Refactor on the next application (fused with its forward sweep)."""
        self.e.factored = False
        self.e.event_log = events

    def apply_local(self, F):
        """G = F W_in_local; Z = solves (stays in the engine)."""
        e = self.e
        n, nt, nk2 = e.n, e.n_t, 2 * e.n_k
        if nk2:
            e._gemm(n, nk2, nt, 1.0, F.data_ptr(), n, e.w_in.data_ptr(), nt, 0.0, e.G.data_ptr(), n)
            e._spatial()

    def out_chunk(self, r0, rows, dst, ldd):
        """dst (rows x N_t, ld ldd) = Z[r0:r0+rows, :] W_out_local."""
        e = self.e
        nk2 = 2 * e.n_k
        if nk2 == 0:
            dst.zero_()
            return
        e._gemm(rows, e.n_t, nk2, 1.0, e.Z.data_ptr() + 8 * r0, e.n, e.w_out.data_ptr(), nk2, 0.0,
                dst.data_ptr(), ldd)

    def out_scatter(self, dst_table, parts, rp):
        """Z W_out_local with row block c written to dst_table[c] (fused scatter)."""
        from . import _native

        e = self.e
        nk2 = 2 * e.n_k
        _native.call("kh_dgemm_rowscatter", e.n, e.n_t, nk2, e.Z.data_ptr(), e.n, e.w_out.data_ptr(), max(nk2, 1),
                     dst_table.data_ptr(), parts, rp, rp, e._stream())
        e.gpu_launches += 1

    def z_rows(self, send, row_blocks):
        """send[c, :2 nk_local, :rows_c] = Z_local[rows of block c, :]^T (the
        all-to-all's outgoing blocks: this rank's modes for rank c's rows)."""
        e = self.e
        Zt = e.Z.view(2 * e.n_k, e.n)
        for c, (r0, rows) in enumerate(row_blocks):
            if rows and e.n_k:
                send[c, :2 * e.n_k, :rows].copy_(Zt[:, r0:r0 + rows])

    def gemm_rows(self, recv, wperm, out):
        """out (rp x N_t, col-major) = [received modes] (rp x K) W_perm (K x N_t)."""
        e = self.e
        K = recv.shape[0] * recv.shape[1]
        rp = recv.shape[2]
        e._gemm(rp, e.n_t, K, 1.0, recv.data_ptr(), rp, wperm.data_ptr(), K, 0.0, out.data_ptr(), rp)

    def y_shard(self, U_shard, rows, ld, dst):
        """dst (rows x 2N_t, ld) = U_shard [A_t^T | M_t^T]."""
        e = self.e
        e._gemm(rows, 2 * e.n_t, e.n_t, 1.0, U_shard.data_ptr(), ld, e.kron_b.data_ptr(), e.n_t, 0.0,
                dst.data_ptr(), ld)

    def residual_full(self, Y, F):
        """R (engine buffer) = F - (M Y1 + A Y2); returns (R, rel residual)."""
        e = self.e
        e.plan.residual(e.n_t, Y.data_ptr(), e.n, F.data_ptr(), e.n, e.R.data_ptr(), e.n, e.norms.data_ptr(),
                        e._stream())
        return e.R, e._rel(e.norms[:2])

    def axpy_(self, y, x, alpha=1.0):
        from . import _native

        _native.call("kh_daxpy", y.numel(), float(alpha), x.data_ptr(), y.data_ptr(), self.e._stream())


class PeerSlots:
    """Receive slots for the fused GEMM + reduce-scatter over peer memory.

    recv[s] (column-major rp x N_t) receives the partial back transform that
    rank s computed for this rank's rows. Every rank maps the other ranks'
    receive buffers with CUDA IPC and keeps a device table dst[c] = (rank c's
    recv) + slot `rank`, the target of kh_dgemm_rowscatter.
    """

    def __init__(self, world, rank, nt, rp, device, group=None):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _native

        self.world, self.rank, self.group = world, rank, group
        self.slot = nt * rp
        self.recv = torch.zeros((world, nt, rp), dtype=torch.float64, device=device)
        self.mapped = []
        # every step is local and its outcome is exchanged before anyone acts
        # on it, so a failing rank cannot leave the others blocked in a
        # collective; `ok` tells the caller whether to fall back to NCCL
        mine = None
        try:
            handle = ctypes.create_string_buffer(64)
            offset = ctypes.c_int64()
            _native.call("kh_ipc_handle", self.recv.data_ptr(), handle, ctypes.byref(offset))
            mine = (handle.raw, int(offset.value))
        except Exception as exc:  # noqa: BLE001 -- reported through the flag
            self.error = f"kh_ipc_handle: {exc}"
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        opened = all(h is not None for h in handles)
        bases = []
        if opened:
            try:
                for c in range(world):
                    if c == rank:
                        bases.append(self.recv.data_ptr())
                    else:
                        ptr = ctypes.c_void_p()
                        raw, off = handles[c]
                        _native.call("kh_ipc_open", ctypes.create_string_buffer(raw, 64), ctypes.byref(ptr))
                        self.mapped.append(ptr.value)
                        bases.append(ptr.value + off)   # the peer's recv inside its allocation
            except Exception as exc:  # noqa: BLE001
                self.error = f"kh_ipc_open: {exc}"
                opened = False
        flags = [None] * world
        dist.all_gather_object(flags, opened, group=group)
        self.ok = all(flags)
        if not self.ok:
            self.close()
            return
        self.dst = torch.tensor([b + 8 * rank * self.slot for b in bases], dtype=torch.int64, device=device)

    def close(self):
        from . import _native

        for ptr in self.mapped:
            _native.call("kh_ipc_close", ptr)
        self.mapped = []


class ShardedFD:
    """FD over `world` ranks of torch.distributed (row-sharded result)."""

    def __init__(self, M_x, A_x, modal, rank, world, device=None, leaf_size=None, ops=None, group=None,
                 engine_kwargs=None, collective="nccl"):
        import torch

        if collective not in ("nccl", "p2p", "alltoall"):
            raise ValueError(f"unknown collective {collective!r}")
        self.rank, self.world, self.group = rank, world, group
        self.k0, self.k1 = shard_range(modal.n_k, world, rank)
        self.local = restrict_modal(modal, self.k0, self.k1)
        self.n = M_x.shape[0]
        self.n_t = modal.n_t
        self.rp = row_chunk(self.n, world)
        if ops is None:
            from . import sparse_direct
            from .engine import FDEngine

            kw = dict(engine_kwargs or {})
            if leaf_size is not None:
                kw["leaf_size"] = leaf_size
            else:
                kw.setdefault("leaf_size", sparse_direct.DEFAULT_LEAF_SIZE)
            self.engine = FDEngine(M_x, A_x, self.local, device=device, **kw)
            ops = EngineOps(self.engine)
            dev = self.engine.device
        else:
            self.engine = getattr(ops, "engine", None)
            dev = getattr(ops, "device", torch.device("cpu"))
        self.ops = ops
        f64 = torch.float64
        g, rp, nt = world, self.rp, self.n_t
        self.P = torch.zeros((g, nt, rp), dtype=f64, device=dev)     # partial chunks, col-major rp x N_t each
        self.U = torch.zeros((nt, rp), dtype=f64, device=dev)        # this rank's rows of u
        self.D = torch.zeros((nt, rp), dtype=f64, device=dev)        # correction shard
        self.Ys = torch.zeros((2 * nt, rp), dtype=f64, device=dev)
        self.Yall = torch.zeros((g, 2 * nt, rp), dtype=f64, device=dev)
        self.Y = torch.zeros((2 * nt, self.n), dtype=f64, device=dev)  # col-major n x 2N_t
        self.gpu_launches = 0
        self.collective = collective
        self.peers = PeerSlots(world, rank, nt, rp, dev, group) if collective == "p2p" else None
        if self.peers is not None and not self.peers.ok:
            # peer mapping failed on some rank: every rank takes the NCCL path
            import warnings

            warnings.warn("peer-memory slots unavailable (%s); using NCCL reduce-scatter"
                          % getattr(self.peers, "error", "another rank failed"))
            self.peers = None
            self.collective = collective = "nccl"
        if collective == "alltoall":
            # all-to-all of Z by spatial rows, then one local GEMM per rank:
            # sends 2 N_k n / g values per rank instead of n N_t
            blocks = [shard_range(modal.n_k, world, c) for c in range(world)]
            self.kmax = max(1, max(b - a for a, b in blocks))
            K = world * 2 * self.kmax
            wperm = np.zeros((K, nt))
            for c, (a, b) in enumerate(blocks):
                wperm[c * 2 * self.kmax:c * 2 * self.kmax + 2 * (b - a)] = restrict_modal(modal, a, b).w_out
            self.send = torch.zeros((world, 2 * self.kmax, rp), dtype=f64, device=dev)
            self.recv = torch.zeros_like(self.send)
            self.wperm = (torch.from_numpy(np.ascontiguousarray(wperm.T)).to(dev) if dev.type == "cuda"
                          else torch.from_numpy(wperm))

    def close(self):
        """Teardown of the peer-memory path: unmap the other ranks' receive
        buffers, then wait until every rank has done so, so no receive
        buffer is freed while a peer still maps it. Collective over the group
        (call it on every rank; idempotent)."""
        if self.peers is None:
            return
        import torch.distributed as dist

        self.peers.close()
        self.peers = None
        if dist.is_initialized():
            dist.barrier(group=self.group)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def rows(self, c):
        r0 = c * self.rp
        return r0, max(0, min(self.n, r0 + self.rp) - r0)

    def _apply(self, F, out):
        """out (this rank's rows) = FD(F), F full (col-major n x N_t)."""
        import torch.distributed as dist

        self.ops.apply_local(F)
        if self.peers is not None:
            self._apply_p2p(out)
            return
        if self.collective == "alltoall":
            self.ops.z_rows(self.send, [self.rows(c) for c in range(self.world)])
            dist.all_to_all_single(self.recv.view(-1), self.send.view(-1), group=self.group)
            self.ops.gemm_rows(self.recv, self.wperm, out)
            return
        for c in range(self.world):
            r0, rows = self.rows(c)
            if rows < self.rp:
                self.P[c].zero_()
            if rows:
                self.ops.out_chunk(r0, rows, self.P[c], self.rp)
        dist.reduce_scatter_tensor(out.view(-1), self.P.view(-1), group=self.group)

    def _apply_p2p(self, out):
        """Fused back transform + reduce-scatter over peer memory."""
        import torch
        import torch.distributed as dist

        from . import _native

        pe = self.peers
        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # every rank has consumed its slots of the previous exchange
        self.ops.out_scatter(pe.dst, self.world, self.rp)
        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # all tiles destined to this rank have landed
        _native.call("kh_sum_parts", self.world, pe.recv.data_ptr(), pe.slot, out.data_ptr(),
                     _native.stream_handle())

    def _residual(self):
        import torch.distributed as dist

        r0, rows = self.rows(self.rank)
        if rows:
            self.ops.y_shard(self.U, rows, self.rp, self.Ys)
        dist.all_gather_into_tensor(self.Yall.view(-1), self.Ys.view(-1), group=self.group)
        # chunked (g, 2N_t, rp) -> column-major n x 2N_t
        self.Y.copy_(self.Yall.permute(1, 0, 2).reshape(2 * self.n_t, self.world * self.rp)[:, :self.n])
        return self.ops.residual_full(self.Y, self._F)

    def solve(self, F, refine=5, tol=1e-13, factor_events=None):
        """Returns (U_shard, info): U_shard is (N_t, rp) = column-major rows
        [rank*rp, rank*rp + rows) of u."""
        self._F = F
        self.ops.factor(factor_events)
        self._apply(F, self.U)
        R, rel = self._residual()
        info = {"residuals": [rel], "refine_steps": 0, "imag_residue": 0.0}
        steps = 0
        while rel > tol and steps < refine:
            self._apply(R, self.D)
            self.ops.axpy_(self.U, self.D)
            steps += 1
            R, new = self._residual()
            info["residuals"].append(new)
            if not new < rel:
                # the step did not help (rounding floor): undo it, keep the best iterate
                self.ops.axpy_(self.U, self.D, -1.0)
                break
            stalled = not new < REFINE_MIN_GAIN * rel  # stagnation: classic IR stop rule
            rel = new
            if stalled:
                break
        info["refine_steps"] = steps
        info["residual"] = rel
        return self.U, info

    def gather(self):
        """Full u (column-major n x N_t as an (N_t, n) tensor) on every rank."""
        import torch
        import torch.distributed as dist

        allU = torch.zeros((self.world, self.n_t, self.rp), dtype=self.U.dtype, device=self.U.device)
        dist.all_gather_into_tensor(allU.view(-1), self.U.view(-1), group=self.group)
        return allU.permute(1, 0, 2).reshape(self.n_t, self.world * self.rp)[:, :self.n].contiguous()


def solve_fd_sharded(system, pencil=None, refine=5, refine_tol=1e-13, leaf_size=None, group=None,
                     collective="p2p"):
    """Multi-GPU counterpart of solvers.solve_fd (reference solvers.py:348-403)
    for one process per GPU under an initialized torch.distributed group.

    Every rank passes the same `system`; rank r returns its row block of u:
    (rows, U_rows, report) where `rows` = (r0, r1) are interior spatial rows
    and U_rows is the host (N_t, r1 - r0) array of u[r0:r1, :] (column-major
    layout of the reference's coefficient vector restricted to those rows).
    The report is the same on every rank except the timings.
    """
    import time

    import torch
    import torch.distributed as dist

    from . import _native, solvers
    from .engine import modal_plan

    from concurrent.futures import ThreadPoolExecutor

    import numpy as np
    import scipy.sparse as sp

    from . import sparse_direct

    _native.require_cuda()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    report = solvers.SolveReport(variant="fd", dof=system.dof, n_t=system.n_t, m_x=system.m_x)
    dev = torch.device("cuda", torch.cuda.current_device())
    report.device = torch.cuda.get_device_name(dev)
    n, nt = system.m_x, system.n_t
    leaf = leaf_size or sparse_direct.DEFAULT_LEAF_SIZE
    t0 = time.perf_counter()
    # as in solvers.solve_fd: pinned rhs up at once, the symbolic analysis on
    # a worker thread beside the host pencil (few BLAS threads)
    rhs_t = torch.from_numpy(np.ascontiguousarray(np.asarray(system.rhs, dtype=np.float64)))
    F = rhs_t.to(dev, non_blocking=True).view(nt, n) if rhs_t.is_pinned() else None
    pattern = (sp.csr_matrix(system.spatial.M_II) + sp.csr_matrix(system.spatial.A_II)).tocsr()
    with ThreadPoolExecutor(max_workers=1) as pool:
        fut = pool.submit(sparse_direct.analyze, pattern, leaf)
        with solvers._blas_threads(1 if nt <= 512 else 4):
            if pencil is None:
                pencil = solvers.build_pencil(system.temporal, "fd", eig="reduced")
            modal = modal_plan(system.temporal, pencil)
        report.t_decompose = time.perf_counter() - t0
        if F is None:
            F = rhs_t.to(dev).view(nt, n)
        symbolic = fut.result()
    report.min_re_lambda = pencil.min_re_lambda
    report.spectral_source = solvers.spectral_source(pencil)
    t0 = time.perf_counter()
    with ShardedFD(system.spatial.M_II, system.spatial.A_II, modal, rank, world, device=dev,
                   leaf_size=leaf, group=group, collective=collective,
                   engine_kwargs={"symbolic": symbolic}) as runner:
        U, info = runner.solve(F, refine=refine, tol=refine_tol)
        r0, rows = runner.rows(rank)
        out = solvers._to_host(U[:, :rows])
    report.t_spatial = time.perf_counter() - t0
    report.fd_residual = info["residuals"][0]
    report.refine_steps = info["refine_steps"]
    report.residual = info["residual"]
    return (r0, r0 + rows), out, report
