"""Benchmark: space-time DoFs solved per second by the FD solver (fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

One step = one full FD solve of the configuration on device-resident inputs:
batched LDL^T factorization of every shift, transform-in GEMM, batched
solves, transform-out GEMM, and iterative refinement to a 1e-13 relative
space-time residual. Setup (host pencil decomposition, symbolic analysis,
plan creation, uploads) is outside the timed region, as the reference's own
`solve_fd(system, pencil=...)` allows; `e2e` times the public API call
`solve_fd(system, pencil)` with host buffers instead (analysis, uploads and
the download of the solution included).

Multi-GPU (torchrun): the shifts are sharded over ranks, each rank does a
partial back-transform and the cross-mode sum is an NCCL reduce-scatter by
spatial rows (paper_2008_01996_b200/distributed.py).
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "space-time DoFs solved/sec (FD, fp64)"
UNIT = "dof/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--refine", type=int, default=5)
    ap.add_argument("--leaf-size", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--j-max", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-levels", action="store_true",
                    help="skip the extra per-level-timed factorization (launch-list captures)")
    ap.add_argument("--collective", choices=["p2p", "nccl", "alltoall"], default="p2p",
                    help="N>1 back-transform reduce-scatter: fused GEMM + peer-memory scatter, or NCCL")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the multi-GPU driver even with one rank (testing the N>1 path on one GPU)")
    ap.add_argument("--spawn-check", action="store_true",
                    help="(tests) each rank prints its rank and world size and exits before touching a GPU")
    ap.add_argument("--ref-budget", type=float, default=240.0,
                    help="reference arm: seconds of full solves after the first (steps are capped to fit)")
    ap.add_argument("--ref-processes", action="store_true",
                    help="reference arm: time the shift solves over a process pool instead of threads")
    ap.add_argument("--ref-quick", action="store_true",
                    help="reference arm: skip the process-pool and sampled cross-checks")
    return ap.parse_args()


def spawn_ranks(args):
    """`--gpus N` (N > 1) without a torchrun environment: run this script
    again under torch.distributed.run with N ranks on this node (one process
    per GPU, rendezvous on 127.0.0.1); rank 0 prints the JSON line. Returns
    the launcher's exit code, or None when no spawn is needed."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ---- clocks ---------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- peaks ------------------------------------------------------------------------
def measured_peaks(device):
    import torch

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mp = json.load(fh)
        peaks["hbm_gbs"] = mp.get("hbm_gbs")
        peaks["fp64_tflops"] = mp.get("fp64_tflops")
        peaks["source"] = "MEASURED_PEAKS.json"
    except OSError:
        peaks["hbm_gbs"] = 6650.0
        peaks["source"] = "fallback (B200_PROFILING.md)"
    if not peaks.get("fp64_tflops"):
        # MEASURED_PEAKS.json carries no fp64 figure: measure cuBLAS DGEMM here
        # with the driver's protocol (8192^3, best of 10, CUDA events)
        n = 8192
        a = torch.randn(n, n, dtype=torch.float64, device=device)
        b = torch.randn(n, n, dtype=torch.float64, device=device)
        for _ in range(2):
            torch.matmul(a, b)
        best = 1e30
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        peaks["fp64_tflops"] = 2.0 * n**3 / best / 1e12
        peaks["fp64_source"] = "cuBLAS DGEMM 8192^3 best of 10, measured in this run"
        del a, b
        torch.cuda.empty_cache()
    else:
        peaks["fp64_source"] = "MEASURED_PEAKS.json"
    return peaks


# ---- CPU baseline (oracle port, bounded sample) -------------------------------------
def cpu_fd_sample(system, n_shift_sample, threads=1):
    """Time the reference algorithm (oracle/fd_oracle.py restatement of
    solvers.py:348-403) on a bounded sample: full pencil, transforms and
    analysis, `n_shift_sample` of the N_t spatial factor+solves; the solve
    time is extrapolated linearly to all N_t shifts."""
    from concurrent.futures import ThreadPoolExecutor

    import scipy.sparse as sp

    from oracle import fd_oracle as orc

    A_t, M_t, M_x, A_x, rhs = orc.system_arrays(system)
    n_t, m_x = A_t.shape[0], M_x.shape[0]
    t0 = time.perf_counter()
    p = orc.fd_pencil(A_t, M_t)
    t_pencil = time.perf_counter() - t0
    t0 = time.perf_counter()
    F = rhs.reshape(m_x, n_t, order="F")
    G = (orc._transform_in(p["L"], F, np.conj(p["U"])) / p["sigma"][None, :]) @ np.conj(p["Vh"])
    t_in = time.perf_counter() - t0
    t0 = time.perf_counter()
    M, A = sp.csr_matrix(M_x), sp.csr_matrix(A_x)
    perm = orc.mmd_analyze((M + A).tocsr())
    t_an = time.perf_counter() - t0
    Mc, Ac = M.astype(complex), A.astype(complex)
    ks = np.linspace(0, n_t - 1, n_shift_sample).astype(int)
    Z = np.zeros((m_x, n_t), complex)

    def one(k):
        K = (Mc + p["D"][k] * Ac).tocsr()
        return k, orc.superlu_solve(perm, orc.superlu_factor(perm, K), G[:, k])

    t0 = time.perf_counter()
    if threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            for k, z in pool.map(one, ks):
                Z[:, k] = z
    else:
        for k in ks:
            Z[:, k] = one(k)[1]
    t_sp = (time.perf_counter() - t0) * n_t / len(ks)
    t0 = time.perf_counter()
    U = ((Z @ p["Vh"].T) * p["sigma"][None, :]) @ p["U"].T
    _ = np.ascontiguousarray(U.real)
    t_out = time.perf_counter() - t0
    total = t_pencil + t_in + t_an + t_sp + t_out
    return {"t_total": total, "t_pencil": t_pencil, "t_spatial_extrap": t_sp, "t_transform": t_in + t_out,
            "t_analyze": t_an, "sample_shifts": int(len(ks)), "n_t": n_t}


def cpu_fd_full(system, workers, mode):
    """One unsampled reference FD solve: the oracle port of solve_fd
    (solvers.py:348-403; oracle.fd_oracle.solve_fd_parallel) with all N_t
    SuperLU factor + solves over `workers` threads (mode "threads": the
    reference's own thread pool) or processes (the pool is created inside
    the timed region)."""
    from oracle import fd_oracle as orc

    tm = {}
    u, _ = orc.solve_fd_parallel(*orc.system_arrays(system), workers, timings=tm, mode=mode)
    return dict(tm, u=u, workers=workers, n_t=system.n_t)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def shift_sample_size(cfg):
    return {"c1": 32, "c2": 32, "c3": 12, "c4": 3}.get(cfg, 8)


# ---- main -------------------------------------------------------------------------
def workload_config(args, info, system, world):
    """The `config` dict, identical in both arms (--impl ours / reference)."""
    return {"workload": f"{args.config}: {info['mesh']} M_x={system.m_x} N_t={system.n_t} dof={system.dof} "
                        f"rhs={info['rhs']}",
            "j_max": info["j_max"],
            "parallelism": "single GPU" if world == 1 else f"shift-sharded x{world}"}


def main():
    args = parse()
    rc = spawn_ranks(args)
    if rc is not None:
        sys.exit(rc)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.spawn_check:
        print(json.dumps({"rank": rank, "world": world, "local_rank": local}), flush=True)
        return
    if args.impl == "reference":
        return run_reference(args, world, rank)
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.force_sharded
    if sharded:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    from paper_2008_01996_b200 import problems, solvers, sparse_direct
    from paper_2008_01996_b200.engine import FDEngine, modal_plan

    kw = {} if args.j_max is None else {"j_max": args.j_max}
    system, info = problems.build_system(args.config, temporal_device=dev, **kw)
    pencil = solvers.build_pencil(system.temporal, "fd")
    modal = modal_plan(system.temporal, pencil)
    n, nt = system.m_x, system.n_t
    dof = system.dof
    leaf = args.leaf_size or sparse_direct.DEFAULT_LEAF_SIZE

    if sharded:
        from paper_2008_01996_b200.distributed import ShardedFD

        runner = ShardedFD(system.spatial.M_II, system.spatial.A_II, modal, rank, world, device=dev,
                           leaf_size=leaf, collective=args.collective)
        eng = runner.engine
    else:
        runner = None
        eng = FDEngine(system.spatial.M_II, system.spatial.A_II, modal, device=dev, leaf_size=leaf)
    F = torch.from_numpy(np.ascontiguousarray(system.rhs)).to(dev).view(nt, n)
    U = torch.empty((nt, n), dtype=torch.float64, device=dev)
    stats = eng.sym.stats

    fac_events = []
    phase_timers = {}

    def step(record=False):
        eng.factored = False
        eng.event_log = fac_events if record else None  # refactoring when the factors are not kept
        eng.timers = phase_timers if record else None
        if record:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        if runner is not None:
            out = runner.solve(F, refine=args.refine, factor_events=fac_events if record else None)
        else:
            # refactor inside the step: the first application factors every
            # shift with the forward sweep fused (engine._spatial)
            out = eng.solve(F, U, refine=args.refine)
        if record:
            e1.record()
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if sharded:
        torch.distributed.barrier()
    from paper_2008_01996_b200 import _native

    launches0 = _native.launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    fac_events.clear()
    torch.cuda.synchronize()
    t_start.record()
    infos = []
    for _ in range(args.steps):
        _, inf = step(record=True)
        infos.append(inf)
    t_end.record()
    torch.cuda.synchronize()
    ck = clocks.stop()
    elapsed = t_start.elapsed_time(t_end) / 1e3
    if sharded:
        tt = torch.tensor([elapsed], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        elapsed = float(tt.item())
    launches = (_native.launch_count() - launches0) // max(args.steps, 1)
    ms = elapsed / args.steps * 1e3
    value = dof * args.steps / elapsed

    # roofline of the dominant kernel: the batched LDL^T factorization (DMMA fp64)
    fac_s = sum(a.elapsed_time(b) for a, b in fac_events) / 1e3 / max(args.steps, 1)
    n_shift_local = eng.n_k
    fac_flops = stats["flops"] * n_shift_local
    peaks = measured_peaks(dev) if rank == 0 else {}

    # per-level roofline of the factorization ("report the
    # fraction against whichever bound is binding, per tree level"): one more
    # factorization outside the timed region with CUDA events at the level
    # boundaries; algorithmic flops and bytes per level from the fronts
    levels = None
    if not sharded and len(eng.pipes) == 1 and eng.keep_factors and not args.no_levels:
        levels = factor_levels(eng, peaks)

    # per-phase rooflines from the CUDA events around each phase (engine.timers)
    kernels = {}
    if not sharded:
        def ms_of(name):
            return sum(a.elapsed_time(b) for a, b in phase_timers.get(name, [])) / max(args.steps, 1)

        calls = {k: len(v) / max(args.steps, 1) for k, v in phase_timers.items()}
        st_ = eng.sym.stats
        nk_ = eng.n_k
        hbm = peaks.get("hbm_gbs")
        fp64 = peaks.get("fp64_tflops")
        gemm_flops = calls.get("gemm", 0) * 2.0 * n * nt * 2 * nk_ + calls.get("gemm_kron", 0) * 2.0 * n * 2 * nt * nt
        gemm_ms = ms_of("gemm") + ms_of("gemm_kron")
        if gemm_ms > 0:
            a_ = gemm_flops / (gemm_ms / 1e3) / 1e12
            kernels["transform_gemms"] = {"bound": "tensor", "achieved": a_, "peak": fp64, "unit": "TFLOP/s",
                                          "frac": a_ / fp64 if fp64 else None, "ms_per_step": gemm_ms,
                                          "work": "modal transforms F W_in, Z W_out and the residual's "
                                                  "U [A_t^T | M_t^T]: 2 m n k flops per call (dgemm_kernel)"}
        if ms_of("solve") > 0:
            b_ = calls["solve"] * 2 * st_["panel_entries"] * 16.0 * nk_   # forward + backward read every factor
            a_ = b_ / (ms_of("solve") / 1e3) / 1e9
            kernels["refinement_solves"] = {"bound": "hbm", "achieved": a_, "peak": hbm, "unit": "GB/s",
                                            "frac": a_ / hbm if hbm else None, "ms_per_step": ms_of("solve"),
                                            "work": "forward + backward sweeps over the retained factors "
                                                    "(16 B per complex factor entry, each read once per sweep)"}
        if ms_of("residual") > 0:
            b_ = calls["residual"] * (8.0 * n * nt * 4 + 24.0 * st_["nnz"])
            a_ = b_ / (ms_of("residual") / 1e3) / 1e9
            kernels["residual_spmm"] = {"bound": "hbm", "achieved": a_, "peak": hbm, "unit": "GB/s",
                                        "frac": a_ / hbm if hbm else None, "ms_per_step": ms_of("residual"),
                                        "work": "R = F - (M_x Y1 + A_x Y2): Y (2 N_t), F, R columns + CSR once"}
        if ms_of("factor_solve") > 0:
            kernels["factor_plus_solve_ms_per_step"] = ms_of("factor_solve")
        if ms_of("gemm_dd") > 0:
            # compensated U M_t^T: one TwoProd + TwoSum (~9 fp64 ops) per multiply-add
            madd = calls.get("gemm_dd", 0) * float(n) * nt * nt
            kernels["compensated_residual"] = {
                "ms_per_step": ms_of("gemm_dd") + ms_of("residual_dd"), "calls_per_step": calls.get("gemm_dd", 0),
                "gemm_dd_ms": ms_of("gemm_dd"),
                "gemm_dd_gmadd_per_s": madd / (ms_of("gemm_dd") / 1e3) / 1e9,
                "work": "kh_dgemm_dd (U M_t^T as hi + lo, Dot2) + kh_plan_residual_dd; used once the fp64 "
                        "residual nears its rounding floor"}

    # the e2e runs build their own plans: release this one's device memory
    # first (at c4 its retained factors take 136 GB of the 180)
    coll = runner.collective if runner is not None else args.collective
    fused_fwd = bool(getattr(eng, "fuse_forward", False))
    eng = runner = U = F = None
    import gc

    gc.collect()
    torch.cuda.empty_cache()
    e2e = None
    if not sharded and rank == 0 and not args.no_e2e:
        e2e = measure_e2e(system, pencil, args, leaf)
    elif sharded and not args.no_e2e:
        e2e = measure_e2e_sharded(system, pencil, args, leaf)

    if rank == 0:
        achieved = fac_flops / fac_s / 1e12 if fac_s > 0 else None
        traffic = load_traffic(args.config)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, info, system, world),
            "knobs": {"refine": args.refine, "leaf_size": leaf,
                      "shifts_solved": int(modal.n_k), "conjugate_pairs": int(modal.n_pairs),
                      "l2": "inputs larger than L2 (factors %.1f GB, F %.0f MB)" % (
                          stats["panel_entries"] * 16 * n_shift_local / 1e9, 8 * dof / 1e6),
                      "collective": ({"p2p": "fused GEMM->peer-memory scatter",
                                      "nccl": "GEMM + NCCL reduce_scatter",
                                      "alltoall": "NCCL all-to-all of Z by rows + local GEMM"}[coll]
                                     if sharded else None)},
            "residual": infos[-1]["residual"], "refine_steps": infos[-1]["refine_steps"],
            "residual_mode": infos[-1].get("residual_mode", "fp64"),
            "residual_history": infos[-1]["residuals"],
            "fd_residual": infos[-1]["residuals"][0],
            "gpu_launches": int(launches),
            "clocks": ck,
            "roofline": {"kernel": "batched multifrontal complex LDL^T: all launches of one factorization "
                                   "(factor_front_kernel, big_*, schur_update_kernel"
                                   + ("; the first solve's forward sweep runs fused inside, its flops are "
                                      "not counted)" if fused_fwd else ")"),
                         "bound": "tensor", "achieved": achieved, "peak": peaks.get("fp64_tflops"),
                         "unit": "TFLOP/s", "frac": (achieved / peaks["fp64_tflops"]) if achieved else None,
                         "peak_source": peaks.get("fp64_source"),
                         "flops_per_shift": stats["flops"], "shifts": int(n_shift_local),
                         "ms_per_step": fac_s * 1e3, "share_of_step": fac_s * 1e3 / ms,
                         "traffic": traffic, "levels": levels},
            "e2e": e2e,
            "kernels": kernels,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_subprocess(args)
        print(json.dumps(line), flush=True)
    if sharded:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def load_traffic(cfg):
    """DRAM bytes per step of the factorization launches, from the committed
    ncu launch list (profiles/traffic.json, written by profiles/summarize.py)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            ent = json.load(fh).get(cfg)
        return None if ent is None else ent["factor_dram_bytes_per_step"]
    except (OSError, ValueError, KeyError):
        return None


def factor_levels(eng, peaks):
    """Per tree level: fronts, ms, algorithmic TF/s and GB/s and their
    fractions of the FP64 / HBM peaks, for one factorization of all shifts
    (forward sweep fused, as in the step). Bytes: each front's panel (m p)
    and update block (q(q+1)/2) written once and its children's update
    blocks read once, 16 B per complex entry."""
    import torch

    plan = eng.pipes[0][0]
    first, p, q, par, dep, _ = eng.sym.fronts()
    m = (p + q).astype(np.float64)
    flops = np.zeros(len(p))
    for f in range(len(p)):
        r = m[f] - np.arange(p[f]) - 1.0
        flops[f] = float(np.sum(8.0 * r * (r + 1.0) / 2.0 + 8.0 * r))
    upd = q.astype(np.float64) * (q + 1) / 2.0
    child_upd = np.zeros(len(p))
    for f in range(len(p)):
        if par[f] >= 0:
            child_upd[par[f]] += upd[f]
    nbytes = 16.0 * (m * p + upd + child_upd)
    plan.set_level_timing(True)
    eng.factored = False
    eng.event_log = eng.timers = None
    eng._spatial()
    torch.cuda.synchronize()
    ms = plan.level_times()
    plan.set_level_timing(False)
    nk = eng.n_k
    out = []
    for d in range(len(ms)):
        sel = dep == d
        fl, by = flops[sel].sum() * nk, nbytes[sel].sum() * nk
        t = ms[d] / 1e3
        tf, gb = (fl / t / 1e12, by / t / 1e9) if t > 0 else (0.0, 0.0)
        out.append({"depth": d, "fronts": int(sel.sum()), "max_m": int(m[sel].max()), "ms": float(ms[d]),
                    "tflops": tf, "frac_fp64": tf / peaks["fp64_tflops"] if peaks.get("fp64_tflops") else None,
                    "gbs": gb, "frac_hbm": gb / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None})
    return out


def measure_e2e(system, pencil, args, leaf):
    """Public API with host buffers, the reference's t_total convention:
    solve_fd(system) per step (temporal pencil dgeev + SVD on the host,
    overlapped with the spatial analysis; plan; factor; solve; refinement;
    D2H of u). `pencil_reused` is the same call with a prebuilt pencil."""
    import torch

    import dataclasses

    from paper_2008_01996_b200 import solvers

    # the step's input lives in pinned host memory (the contract's e2e setup)
    pinned = torch.empty(system.rhs.shape, dtype=torch.float64, pin_memory=True)
    pinned.copy_(torch.from_numpy(system.rhs))
    system = dataclasses.replace(system, rhs=pinned.numpy())

    def timed(pen):
        for _ in range(2):  # warm-up (steady state: the pinned result buffers are cached)
            solvers.solve_fd(system, pencil=pen, refine=args.refine, leaf_size=leaf)
        torch.cuda.synchronize()
        times = []
        for _ in range(max(1, args.e2e_steps)):
            t0 = time.perf_counter()
            _, rep = solvers.solve_fd(system, pencil=pen, refine=args.refine, leaf_size=leaf)
            times.append(time.perf_counter() - t0)
        return float(np.mean(times)), rep

    t_full, rep = timed(None)
    t_reuse, _ = timed(pencil)
    n, nt = system.m_x, system.n_t
    nnz = system.spatial.M_II.nnz
    h2d = 8 * n * nt + 8 * nt * (2 * nt) * 3 + 8 * (n + 1) + 8 * 3 * 2 * nnz
    return {"value": system.dof / t_full, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(8 * n * nt), "steps": max(1, args.e2e_steps),
            "includes": "solve_fd(system): host pencil (Cholesky-reduced dgeev + real SVD), symbolic analysis, plan upload, H2D of f, "
                        "factorization, solve, refinement, D2H of u",
            "pencil_reused": {"value": system.dof / t_reuse, "unit": UNIT,
                              "includes": "solve_fd(system, pencil) with the pencil built once outside"},
            "residual": rep.residual}


def measure_e2e_sharded(system, pencil, args, leaf):
    """N GPUs through the public multi-GPU API: distributed.solve_fd_sharded
    per step (host rhs in pinned memory -> every rank, analysis, plan,
    factor, solve, NCCL reduce-scatter, refinement, D2H of each rank's rows);
    max time over ranks."""
    import dataclasses

    import torch
    import torch.distributed as dist

    from paper_2008_01996_b200.distributed import solve_fd_sharded

    n, nt = system.m_x, system.n_t
    pinned = torch.empty(system.rhs.shape, dtype=torch.float64, pin_memory=True)
    pinned.copy_(torch.from_numpy(system.rhs))
    system = dataclasses.replace(system, rhs=pinned.numpy())
    solve_fd_sharded(system, pencil=None, refine=args.refine, leaf_size=leaf, collective=args.collective)
    torch.cuda.synchronize()
    dist.barrier()
    steps = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(steps):
        (r0, r1), _, rep = solve_fd_sharded(system, pencil=None, refine=args.refine, leaf_size=leaf,
                                            collective=args.collective)
    el = torch.tensor([(time.perf_counter() - t0) / steps], device=torch.device("cuda", torch.cuda.current_device()))
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    nnz = system.spatial.M_II.nnz
    h2d = 8 * n * nt + 8 * nt * (2 * nt) * 3 + 8 * (n + 1) + 8 * 3 * 2 * nnz
    return {"value": system.dof / float(el.item()), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(8 * (r1 - r0) * nt), "steps": steps,
            "includes": "per rank: host pencil, symbolic analysis, plan upload, H2D of f, sharded factor/solve/refinement, "
                        "NCCL reduce-scatter + all-gather, D2H of the rank's rows of u (rank-0 bytes shown)",
            "residual": rep.residual}


def cpu_baseline_subprocess(args):
    """cpu_baseline of our arm: one unsampled reference solve with its shifts
    over a process pool (~10 s at c3 on 16 cores), timed in a fresh process
    (no CUDA context in the forking process) by the reference arm's own code
    (`--impl reference --steps 1 --warmup 0 --ref-processes`)."""
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--steps", "1", "--warmup", "0",
           "--config", args.config, "--ref-processes", "--ref-quick"]
    if args.j_max is not None:
        cmd += ["--j-max", str(args.j_max)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800).stdout.strip().splitlines()
        ref = json.loads(out[-1])
    except (subprocess.SubprocessError, ValueError, IndexError) as exc:
        return {"value": None, "unavailable": f"reference timing failed: {exc}"}
    return dict(ref["cpu_baseline"])


def run_reference(args, world, rank):
    """The reference's CPU algorithm on this host: the oracle port of
    solve_fd (same LAPACK / SuperLU calls as the reference). Every timed step
    is one full, unsampled solve with the reference's own parallelism, a
    thread pool of all host cores over the shifts (solvers.py:387-390);
    steps after the first stop once --ref-budget seconds are spent (the line
    reports the steps actually timed). Reported beside it: the same solve
    with the shifts over a process pool (what the host cores give the
    algorithm without the GIL) and a 12-shift single-thread extrapolation
    (cross-check). --ref-processes makes the process pool the timed steps
    (our arm's cpu_baseline)."""
    if rank != 0:
        return
    from paper_2008_01996_b200 import problems

    kw = {} if args.j_max is None else {"j_max": args.j_max}
    system, info = problems.build_system(args.config, **kw)
    workers = os.cpu_count() or 1
    mode = "processes" if args.ref_processes else "threads"
    for _ in range(args.warmup):
        cpu_fd_sample(system, 2, 1)
    totals, spent = [], 0.0
    for i in range(max(1, args.steps)):
        if i > 0 and spent + totals[-1] > args.ref_budget:
            break
        r = cpu_fd_full(system, workers, mode)
        totals.append(r["t_total"])
        spent += r["t_total"]
    from oracle import fd_oracle as orc

    res = orc.residual(*orc.system_arrays(system), r["u"])
    t = float(np.mean(totals))
    value = system.dof / t
    what = "processes" if mode == "processes" else "threads (the reference's ThreadPoolExecutor)"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": len(totals),
            "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": workload_config(args, info, system, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                             "cpu_model": cpu_model(),
                             "sample": (f"full solve: oracle port of the reference solve_fd, all {system.n_t} "
                                        f"SuperLU shift factor+solves over {workers} {what}, pencil, "
                                        f"transforms and MMD analysis included; {len(totals)} solve(s), "
                                        f"t_total={t:.2f}s")},
            "residual": res,
            "phases_s": {k: r[k] for k in ("t_pencil", "t_transform", "t_analyze", "t_spatial")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if mode == "threads" and not args.ref_quick:
        rp = cpu_fd_full(system, workers, "processes")
        line["process_pool"] = {"value": system.dof / rp["t_total"], "cores": workers,
                                "sample": f"the same full solve, shifts over {workers} processes (no GIL), "
                                          f"t_total={rp['t_total']:.2f}s"}
        cross = cpu_fd_sample(system, shift_sample_size(args.config), 1)
        line["extrapolated_sample"] = {"value": system.dof / cross["t_total"], "cores": 1,
                                       "sample": f"{cross['sample_shifts']} of {cross['n_t']} shifts, 1 thread, "
                                                 "extrapolated linearly (cross-check only)"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
