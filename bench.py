"""bench.py — usFFT detection-step throughput on B200 (BASELINE.json metric).

One *step* = one whole Step-2 detection round of Alg. 1 (plan,
lattice nodes + index maps, one batched PCG FE solve per lattice node, exchange, lattice FFT,
keys, threshold, per-node selection, votes, union, resolve) at a fixed dimension t of the
workload named by --config (default: BASELINE configs[4] = config 5, the scale workload whose
samples BASELINE shards over 1/2/4/8 GPUs; --config 2 is the d_y = 10 periodic workload).
The I^(1..t-1) and I^(t) sets the round works on come from running the real algorithm (Step 1
and Step 2 up to t-1) during setup.  value = PDE samples solved per second over all ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

--gpus N > 1 outside torchrun re-launches itself under torch.distributed.run with N ranks (one
GPU each, NCCL); under torchrun WORLD_SIZE must equal N.  The samples of each round are sharded
across ranks (strong scaling: the round's work is fixed); rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "usFFT step: PDE samples solved/s + lattice-FFT GB/s vs HBM peak, at 1/2/4/8 B200"
UNIT = "samples/s"
FLOPS_PER_NODE_ITER = 22      # Jacobi PCG, 5-point stencil: DESIGN.md §5 (algorithmic count)


def mg_flops_per_iter(n: int) -> int:
    """Algorithmic flops of one multigrid-preconditioned CG iteration on an n x n mesh (DESIGN.md
    §5): 51 per fine node (smoothing, residual, restriction share, prolongation, A u, 3 dots,
    4 vector updates), 38 per node of the smoothed level 1, and the level-2/3 part of the cycle
    as applied: the 9-point restriction to level 2 (10 per node) and the dense level-2 map
    K (2 U2^2).  The per-sample setup (coefficients, operators, K) is not counted."""
    u0, u1, u2 = (n - 1) ** 2, (n // 2 - 1) ** 2, (n // 4 - 1) ** 2
    return 51 * u0 + 38 * u1 + 10 * u2 + 2 * u2 * u2


def cl_flops_per_iter(n: int, split: bool = False):
    """Algorithmic flops of one CG iteration of the cluster multigrid kernel (k_pcg_cl, n = 64,
    128), phase by phase: per fine node 47, of them 22 in fp64 (the CG: p update 2,
    w = A u + (w,u) 11, x / r / s updates + (r,r) 7, (r,u) 2) and 25 in fp32 (the fine part of the
    V-cycle: z0 and the residual 10, prolongation 3, post-smoothing 12); per node of every
    smoothed coarse level down to 16 cells per side 37 (residual 10, restriction 12,
    prolongation 3, post-smoothing 12); the restriction to the 8-cell level (12 per node) and the
    dense map K of the 8- and 4-cell levels (2 x 49^2), all fp32 (Z32).  Redundant work (the
    coarse levels are replicated in every CTA of a cluster) and the per-sample setup are not
    counted.  split=True returns (fp64 flops, fp32 flops)."""
    u = []
    m = n
    while m >= 8:
        u.append((m - 1) ** 2)
        m //= 2
    f64 = 22 * u[0]
    f32 = 25 * u[0] + sum(37 * v for v in u[1:-1]) + 12 * u[-1] + 2 * u[-1] * u[-1]
    return (f64, f32) if split else f64 + f32


SURVEY_FLOPS_PER_NODE_ITER = 20   # on-chip PCG unit, ~20 fp64 flops per node-iteration


def mgg_flops_per_iter(n: int) -> int:
    """Algorithmic flops of one CG iteration of the scratch-slab multigrid kernel (k_pcg_mgg, n =
    64, 128), phase by phase: per fine node 47 (p update 2, A p + p.q 11, x / r /
    z0 updates + r.r 7, residual 10, prolongation 3, post-smoothing 12, r.u 2); per node of a
    smoothed coarse level 37 (residual 10, restriction 12, prolongation 3, post-smoothing 12);
    restriction to the 3 x 3 exact level 12 per node and its dense solve 2 * 81."""
    L = 0
    while (n >> L) > 4:
        L += 1
    u = [((n >> l) - 1) ** 2 for l in range(L + 1)]
    return 47 * u[0] + sum(37 * u[l] for l in range(1, L)) + 12 * u[L] + 2 * 81


FP64_FMA_PER_CLK_PER_SM = 64  # B200 fp64 datapath: 37 TF at 1.965 GHz x 148 SMs
FP32_FMA_PER_CLK_PER_SM = 128  # B200 fp32 datapath: 74 TF at 1.965 GHz x 148 SMs


def ncu_traffic(kernel_prefix: str):
    """dram read+write bytes per launch of a kernel from the newest committed ncu --set full
    summary (profiles/*_ncu.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu.json")),
                   key=lambda p: ("final" in os.path.basename(p), p))   # the round's final capture first
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in reversed(files):
        for d in json.load(open(path)).get("full", []):
            if kernel_prefix in d.get("kernel", ""):
                tot = 0.0
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    val, unit = d[m].split()
                    tot += float(val) * scale.get(unit, 1.0)
                return {"bytes": tot, "source": os.path.relpath(path, ROOT)}
    return None


def peaks():
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        m = json.load(open(path))
        p.update({k: m[k] for k in ("hbm_gbs", "sm_max_mhz") if k in m})
        p["source"] = "measured (MEASURED_PEAKS.json)"
    return p


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def setup_detector(cfg, device, group, t_bench):
    """Run Step 1 and Step 2 up to t_bench-1 to obtain the round's real I^(1..t-1) and I^(t)."""
    import torch
    from paper_2109_04131_b200.driver import Detector
    det = Detector(cfg, device=device, group=group, timing=True)
    I1d = det.step1()
    I_prev, _ = det.step2(I1d, t_stop=t_bench - 1)
    torch.cuda.synchronize()
    return det, I_prev.contiguous(), I1d[t_bench - 1].contiguous()


def run_ours(args):
    import torch
    import torch.distributed as dist
    from usfft_inputs import config

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # one GPU per rank; with fewer visible GPUs than ranks (the --backend gloo check of the
    # multi-rank flow on one GPU) ranks share devices round-robin
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.backend)
    cfg = config(args.config)
    if args.precond:
        cfg["precond"] = args.precond
    t_b = args.t if args.t else min(5, cfg["d"])
    det, I_prev, kt = setup_detector(cfg, local, group, t_b)
    s_t = cfg["s_local"] if t_b < cfg["d"] else cfg["s"]
    n_prev = I_prev.shape[0]
    nJ = n_prev * kt.numel()
    stream = det.ctx.stream
    flush = torch.empty(int(256 * 2 ** 20) // 4, dtype=torch.float32, device="cuda")   # 256 MB > L2

    def one(i, want_coef=True):
        flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
        return det.round(2, t_b, i, I_prev, n_prev, kt, s_t, flags, want_coef=want_coef,
                         keep_iters=True)

    for w in range(args.warmup):
        one(1000 + w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.cudart().cudaProfilerStart()          # ncu --profile-from-start off: timed steps only
    launches0 = det.ctx.launches()
    step_ms, phase_runs, iters_sum, samples = [], {}, 0, 0
    det.timing = False                               # no per-phase events / syncs inside timed steps
    for k in range(args.steps):
        flush.fill_(float(k))                         # evict L2 between timed iterations
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = one(k + 1)
        e1.record(stream)
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        if args.verbose:
            print(f"step {k}: {step_ms[-1]:.3f} ms", file=sys.stderr, flush=True)
        iters_sum += int(res.iters.sum().item()) if res.iters is not None and res.iters.numel() else 0
        samples += res.plan.L * res.plan.M
    launches = det.ctx.launches() - launches0
    torch.cuda.cudart().cudaProfilerStop()
    clk = clocks.stop()
    # per-phase breakdown from the same rounds re-run untimed with per-phase CUDA events; the
    # events bracket host-side enqueue gaps too, so one slow re-run (allocator growth, a host
    # hiccup) would skew a mean: each phase reports its median over the K re-runs
    det.timing = True
    for k in range(args.steps):
        flush.fill_(float(k))
        res_p = one(k + 1)
        if args.verbose:
            print(f"phases {k}: " + " ".join(f"{a}={b:.3f}" for a, b in res_p.times.items()),
                  file=sys.stderr, flush=True)
        for name, ms in res_p.times.items():
            phase_runs.setdefault(name, []).append(ms)
    phase = {name: float(np.median(v)) for name, v in phase_runs.items()}      # ms per step
    total_ms = float(np.sum(step_ms))
    t_tensor = torch.tensor([total_ms, phase.get("pde", 0.0) * args.steps], dtype=torch.float64,
                            device="cuda")
    it_tensor = torch.tensor([iters_sum], dtype=torch.int64, device="cuda")
    if world > 1:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
        dist.all_reduce(it_tensor, op=dist.ReduceOp.SUM)
    total_ms, pde_ms = t_tensor.tolist()
    iters_all = int(it_tensor.item())

    # ---- e2e: host buffers in, host result out, through the public API ------------------------
    # the user's view: inputs in pinned host memory, results copied back into pinned host
    # buffers, no per-phase event timing inside the round
    Ih = I_prev.cpu().pin_memory()
    kh = kt.cpu().pin_memory()
    det.timing = False
    # output buffers sized by an untimed pass over the same rounds (|D| differs per round; a
    # G_loc x |J| worst case does not fit pinned host memory at configs 4-5)
    nd_max = 1
    for k in range(args.steps):
        flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
        nd_max = max(nd_max, det.round(2, t_b, 5000 + k, I_prev, n_prev, kt, s_t, flags, want_coef=True).n_det)
    out_idx_h = torch.empty(nd_max, dtype=torch.int32).pin_memory()
    out_coef_h = torch.empty(det.G_loc * nd_max * 2, dtype=torch.float64).pin_memory()
    e2e_ms, h2d, d2h = [], 0, 0
    for k in range(args.steps):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        Id = Ih.to("cuda", non_blocking=True)
        kd = kh.to("cuda", non_blocking=True)
        flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
        res = det.round(2, t_b, 5000 + k, Id, n_prev, kd, s_t, flags, want_coef=True)
        nd = res.n_det
        out_idx_h[:nd].copy_(res.det_idx, non_blocking=True)
        nc = res.coef.numel() if res.coef is not None else 0
        if nc:
            out_coef_h[:nc].copy_(res.coef.reshape(-1), non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        h2d = Ih.numel() * 2 + kh.numel() * 2
        d2h = nd * 4 + nc * 8
    det.timing = True
    e2e_t = torch.tensor([float(np.sum(e2e_ms))], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)

    if rank == 0:
        pk = peaks()
        G = det.G
        P = res.plan
        value = samples / (total_ms / 1e3)
        # dominant kernel: the batched PCG -> fp64 ALU roofline
        from paper_2109_04131_b200.binding import effective_precond
        mg = effective_precond(cfg) == "mg"
        n_mesh = cfg["n"]
        if mg and n_mesh in (16, 32):
            kname, kdesc = "k_pcg_mg", "k_pcg_mg (batched multigrid-preconditioned CG, on-chip, 1 CTA/sample)"
            fpi = mg_flops_per_iter(n_mesh)
        elif mg and n_mesh in (64, 128):
            kname, kdesc = "k_pcg_cl", ("k_pcg_cl (batched multigrid-preconditioned CG, on-chip, one "
                                        "thread-block cluster of %d CTAs per sample)" % (8 if n_mesh == 128 else 4))
            fpi = cl_flops_per_iter(n_mesh)
        elif mg:
            kname, kdesc = "k_pcg_mgg", "k_pcg_mgg (batched multigrid-preconditioned CG, scratch slab, 1 CTA/sample)"
            fpi = mgg_flops_per_iter(n_mesh)
        else:
            kname, kdesc = "k_pcg_reg", "k_pcg_reg (batched Jacobi PCG, register-resident, 1 CTA/sample)"
            fpi = FLOPS_PER_NODE_ITER * G
        flops = fpi * iters_all
        fp64_peak = 148 * FP64_FMA_PER_CLK_PER_SM * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
        fp32_peak = 148 * FP32_FMA_PER_CLK_PER_SM * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
        # k_pcg_cl runs its V-cycle in fp32 (Z32): fp64-equivalent flops = F64 + F32 x (P64 / P32),
        # so achieved / fp64 peak is the share of the kernel time the ALU roofline needs
        f64, f32 = cl_flops_per_iter(n_mesh, split=True) if kname == "k_pcg_cl" else (fpi, 0)
        flops_eq = (f64 + f32 * fp64_peak / fp32_peak) * iters_all
        ach = flops_eq / (pde_ms / 1e3) / 1e12 / world if pde_ms > 0 else 0.0
        fft_ms = phase.get("fft", 0.0)
        Mh = P.M // 2 + 1
        fft_bytes = G * P.L * P.M * 8 + G * P.L * Mh * 16
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config{args.config}:{cfg['name']} Step-2 round t={t_b}",
                       "G": G, "d": cfg["d"], "M": P.M, "L": P.L, "samples_per_step": P.L * P.M,
                       "nJ": nJ, "s_tilde": s_t, "cg_iters_mean": iters_all / max(samples, 1),
                       "l2": "flushed between timed steps (256 MB write)",
                       "parallelism": f"samples sharded over {world} GPU(s)"},
            "roofline": {"kernel": kdesc, "bound": "alu",
                         "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": ach / fp64_peak if fp64_peak else None,
                         "traffic": (ncu_traffic(kname) or {}).get("bytes"),
                         "traffic_source": (ncu_traffic(kname) or {}).get("source"),
                         "peak_source": "derived: 148 SM x 64 fp64 FMA/clk x 2 x sm_max_mhz",
                         "flops_per_sample_iter": fpi, "precond": "mg" if mg else "jacobi",
                         "fp64_flops_per_sample_iter": f64, "fp32_flops_per_sample_iter": f32,
                         "fp32_peak": fp32_peak,
                         "achieved_def": "(F64 + F32 x P64/P32) / PDE time; frac = achieved / P64",
                         "frac_survey_unit": (SURVEY_FLOPS_PER_NODE_ITER * G * iters_all / (pde_ms / 1e3) / 1e12
                                              / world / fp64_peak) if pde_ms > 0 and fp64_peak else None,
                         "survey_unit": "20 fp64 flops per fine node and CG iteration (SURVEY §8(d))"},
            "fft": {"kernel": ("k_fft_rader_r (Rader on row pairs, register-radix in-place passes)"
                               if P.M in (401, 4001) else "k_fft_rader_t (Rader/Stockham)"),
                    "bytes_def": "8 G L M read + 16 G L (M/2+1) written (the FFT's algorithmic bytes) / fft phase time",
                    "ms_per_step": fft_ms, "keys_ms_per_step": phase.get("keys"),
                    "achieved_gbs": fft_bytes / (fft_ms / 1e3) / 1e9 if fft_ms else None,
                    "hbm_peak_gbs": pk["hbm_gbs"],
                    "frac": (fft_bytes / (fft_ms / 1e3) / 1e9) / pk["hbm_gbs"] if fft_ms else None},
            "phase_ms_per_step": phase,
            "phase_stat": "median over the K untimed re-runs with per-phase events",
            "e2e": {"value": samples / (e2e_t.item() / 1e3) if e2e_t.item() else None, "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk,
            "peaks": pk,
        }
        if args.cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, P, G, s_t, nJ)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _oracle_solves(job):
    """Worker: the oracle's banded-Cholesky FE solves of a block of sample columns."""
    cfg, Y = job
    from threadpoolctl import threadpool_limits
    from oracle import fe as ofe
    with threadpool_limits(1):
        return ofe.sample_pde(cfg, Y)


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(cfg, P, G, s_t, nJ, n_solve=None, pool=None):
    """The oracle as it stands, on a bounded sample of one round, on all host cores: n_solve
    banded-Cholesky FE solves spread over a process pool (one solve per core at a time; samples
    are independent), and the oracle's lattice DFT + detection (numpy, multi-threaded
    BLAS) of the round's L lattices of M samples for a subset of G_sub nodes and the round's |J|.
    The round time is modelled from the two measured parts: B solves at the measured rate plus
    the detection part scaled by G / G_sub."""
    import multiprocessing as mp
    from oracle import detect as odet
    from oracle import dft as odft
    cores = cpu_cores()
    Btot = P.L * P.M
    rng = np.random.default_rng(0)
    if n_solve is None:
        per = 1e-6 * G * 15 + 1e-3                          # ~ s per solve on one core
        n_solve = max(cores, min(64 * cores, int(8.0 * cores / per)))
    Y = rng.random((cfg["d"], n_solve))
    blocks = [(cfg, Y[:, k::cores]) for k in range(cores) if Y[:, k::cores].shape[1]]
    own = pool is None
    if own:
        pool = mp.get_context("fork").Pool(cores)
    t0 = time.perf_counter()
    pool.map(_oracle_solves, blocks)
    t_solve = (time.perf_counter() - t0) / n_solve
    if own:
        pool.close()
    nJ_s = min(nJ, 20000)
    # ~2e9 complex multiply-adds of direct DFT (L lattices x M samples x <= min(|J|, M) bins)
    G_sub = max(1, min(G, int(2e9 / (P.L * P.M * min(nJ_s, P.M)))))
    U = rng.standard_normal((G_sub, Btot))
    bins = rng.integers(0, P.M, size=(P.L, nJ_s))
    t0 = time.perf_counter()
    V = odft.round_values(U, P.M, P.L, bins)
    odet.detect_round(V, bins, s_t, cfg["theta_rel"])
    t_rest = (time.perf_counter() - t0) * (G / G_sub) * (nJ / nJ_s)
    t_round = Btot * t_solve + t_rest
    return {"value": Btot / t_round, "unit": UNIT, "cores": cores, "kind": "oracle",
            "modelled": True, "t_round_s": t_round,
            "sample": f"{n_solve} FE solves on {cores} processes (scaled to B={Btot}), plus the oracle's "
                      f"DFT+detect of a full round for {G_sub} of {G} nodes and {nJ_s} of {nJ} candidates "
                      f"(scaled to G and |J|); modelled round time {t_round:.1f} s"}


# |J_t| of the Step-2 round the GPU arm times (t = 5; t = 3 for config 4), measured by the GPU
# arm's own setup (profiles/r1_bench_configs.jsonl, BENCH_r01.json): the reference arm cannot run
# the GPU setup, so it takes the round size from these measurements
ROUND_NJ = {1: 205, 2: 1000, 3: 1755, 4: 2031105, 5: 1105}


def run_reference(args):
    """Reference arm = the oracle (CPU, all host cores), rank 0 only; each step a bounded sample
    of the round the GPU arm times, its round time modelled from the measured parts."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    from usfft_inputs import config
    from oracle import plan as oplan
    cfg = config(args.config)
    t_b = args.t if args.t else min(5, cfg["d"])
    s_t = cfg["s_local"] if t_b < cfg["d"] else cfg["s"]
    nJ = ROUND_NJ.get(args.config, 1000)
    M = oplan.lattice_size(s_t, cfg["N"])
    L = oplan.num_lattices(nJ)

    class _P:
        pass
    P = _P()
    P.M, P.L = M, L
    G = (cfg["n"] - 1) ** 2
    cores = cpu_cores()
    pool = mp.get_context("fork").Pool(cores)
    n_step = cores * (2 if G > 4000 else 8)
    for _ in range(args.warmup):
        cpu_baseline(cfg, P, G, s_t, nJ, n_solve=cores, pool=pool)
    t0 = time.perf_counter()
    vals, rounds = [], []
    for _ in range(args.steps):
        cb = cpu_baseline(cfg, P, G, s_t, nJ, n_solve=n_step, pool=pool)
        vals.append(cb["value"])
        rounds.append(cb["t_round_s"])
    wall = time.perf_counter() - t0
    pool.close()
    v = float(np.mean(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(rounds)),
            "ms_per_step_kind": "modelled from the measured bounded sample (see cpu_baseline.sample)",
            "wall_ms_per_step": 1e3 * wall / max(args.steps, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config{args.config}:{cfg['name']} Step-2 round t={t_b}",
                       "G": G, "M": M, "L": L, "nJ": nJ},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "modelled": True,
                             "sample": f"per step: {n_step} FE solves on {cores} processes scaled to B = {L * M}, "
                                       "plus the DFT+detect of a node subset of the round scaled to G"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


def relaunch_distributed(args):
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run, N ranks."""
    import socket
    import torch
    n_vis = torch.cuda.device_count()
    if args.gpus > n_vis and args.backend == "nccl":
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only {n_vis} GPU(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")             # rank count and transport visible in stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execvpe(sys.executable, cmd, env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--t", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: functional check with ranks sharing a GPU)")
    ap.add_argument("--precond", default="", choices=["", "jacobi", "mg"])
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        relaunch_distributed(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
