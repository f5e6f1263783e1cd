"""Predicted 1 -> 8 GPU curve of the shift-sharded FD step, measured on ONE GPU.

    python profiles/probes/scaling_predict.py [c3 c4]

For N = 1, 2, 4, 8 the per-rank device work of ShardedFD.solve (distributed.py)
is run for rank 0's block of shifts, restrict_modal(modal, 0, n_k / N): the
local transform-in GEMM, the factorization + sweeps of its shifts, the
partial back transform over ALL spatial rows, the full residual (every rank
forms it) and one refinement step (c3 and c4 take one / three, as measured
on one GPU; the same count is used for every N). What one GPU cannot show is
the exchange: per FD application a reduce-scatter of the partial back
transform (each rank sends (N-1)/N x 8 n N_t bytes) and, per residual, an
all-gather of Y (2 N_t x n x 8 bytes in total); they are estimated at the
NVLink 5 rate (900 GB/s per direction) and
listed separately. Prints one JSON line per (config, N).
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

NVLINK_GBS = 900.0
REFINE_STEPS = {"c3": 1, "c4": 3}


def main(cfgs):
    import gc

    import torch

    from paper_2008_01996_b200 import problems, solvers
    from paper_2008_01996_b200.distributed import restrict_modal
    from paper_2008_01996_b200.engine import FDEngine, modal_plan

    dev = torch.device("cuda", 0)
    for cfg in cfgs:
        system, info = problems.build_system(cfg, temporal_device=dev)
        modal = modal_plan(system.temporal, solvers.build_pencil(system.temporal, "fd", eig="reduced"))
        n, nt = system.m_x, system.n_t
        F = torch.from_numpy(system.rhs).to(dev).view(nt, n)
        base = None
        for N in (1, 2, 4, 8):
            k1 = -(-modal.n_k // N)
            eng = FDEngine(system.spatial.M_II, system.spatial.A_II, restrict_modal(modal, 0, k1), device=dev)
            U = torch.empty((nt, n), dtype=torch.float64, device=dev)

            def step():
                eng.factored = False
                eng.fd_apply(F, U)
                eng.residual(U, F)
                for _ in range(REFINE_STEPS[cfg]):
                    eng.fd_apply(eng.R, U, accumulate=True)
                    eng.residual(U, F)

            step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3 if cfg == "c3" else 1
            e0.record()
            for _ in range(reps):
                step()
            e1.record()
            torch.cuda.synchronize()
            t_dev = e0.elapsed_time(e1) / reps
            apps = 1 + REFINE_STEPS[cfg]
            rs = (N - 1) / N * 8 * n * nt / (NVLINK_GBS * 1e9) * 1e3 * apps
            ag = (N - 1) / N * 8 * 2 * nt * n / (NVLINK_GBS * 1e9) * 1e3 * apps
            t = t_dev + rs + ag
            base = base or t
            print(json.dumps({"config": cfg, "n_gpus": N, "shifts_per_rank": k1, "rank_device_ms": round(t_dev, 2),
                              "reduce_scatter_ms_est": round(rs, 3), "allgather_y_ms_est": round(ag, 3),
                              "step_ms_pred": round(t, 2), "dof_per_s_pred": system.dof / (t / 1e3),
                              "speedup_pred": round(base / t, 2), "keep_factors": eng.keep_factors}), flush=True)
            del eng, U
            gc.collect()
            torch.cuda.empty_cache()
        del F
        gc.collect()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3", "c4"])
