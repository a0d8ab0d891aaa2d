#!/usr/bin/env python
"""Benchmark: Crank-Nicolson steps/s at N = 2^20 (BASELINE.json configs[2], the
tempered-stable CGMY case), with assembly + H-LU time and the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One "step" is one CN step u <- A+^{-1} A- u on the resident vector, applied as one
H-matvec of the propagator Z = (A+)^{-1} built from the H-LU factors
(u <- 2 Z u - u; ``--method inverse`` uses A- and the two
triangular-inverse factors instead).  Under torchrun (N > 1) every rank runs an
independent replica (single-RHS stepping does not shard); ``value``
is the sum over ranks, timing is the max over ranks.

``--workload cfg4`` runs BASELINE.json configs[3] instead: N = 2^18 - 1, 256
right-hand sides stepped together on the FP64 tensor cores (DMMA), columns sharded
256/G across ranks (strong scaling), roofline against the measured DMMA peak.

``--impl reference`` times the reference algorithm (the oracle restatement of
levyh hops.matvec + hops.solve, oracle/levyh_oracle.py) on the host cores, on the
same N = 2^20 operator (factors built on the GPU and exported, because the
reference cannot assemble or compress at this size: SURVEY G7).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Crank-Nicolson steps/s at N=2^20 (cfg3 CGMY); assembly+H-LU time; % of HBM roofline"

# configs[2] of BASELINE.json
CFG3 = dict(workload="cfg3: CGMY C=1 G=5 M=10 Y=0.5 on [-4,4], N=2^20-1, a=0.05 b=0.1 c=-0.05, "
                     "dt=2^-13, leaf 64, eta 1, ACA tol 1e-9, fp64, u0=max(e^x-1,0)",
            n=2 ** 19, L=4.0, L_W=8.0, a=0.05, b=0.1, c=-0.05, dt=8.0 / 2 ** 20 * 16, leaf=64,
            eps1=1e-9, eps2=1e-10)


CFG4 = dict(workload="cfg4: fractional Laplacian s=0.5 on [-1,1], N=2^18-1, a=b=c=0, dt=h, 256 RHS "
                     "(seed 0, 8 Gaussian bumps each: centres U(-0.8,0.8), widths U(0.02,0.2), "
                     "amplitudes N(0,1)), leaf 64, eta 1, ACA tol 1e-10, fp64",
            n=2 ** 17, K=256, leaf=64, eps1=1e-10, eps2=1e-10)
METRIC4 = "Crank-Nicolson steps/s of the 256-RHS batch at N=2^18 (cfg4); FP64 tensor (DMMA) roofline"
CFG5 = dict(workload="cfg5: fractional Laplacian s=0.8 on [-1,1], N=2^22-1, a=0.1 b=c=0, dt=h, leaf 128, "
                     "eta 1, ACA tol 1e-10, fp64, u0=(1-x^2)_+^3; phases: assembly (sharded across ranks), "
                     "H-LU, 50 CN steps",
            n=2 ** 21, leaf=128, eps1=1e-10, eps2=1e-10, steps=50)
METRIC5 = "cfg5 (N=2^22): assembly + H-LU time, CN steps/s"


def cfg3_config(args, N, world):
    """The `config` of a cfg3 line: identical in the b200 and the reference arm (the algorithm
    each arm runs is the top-level `algorithm` key)."""
    return {"workload": CFG3["workload"] if args.n is None else f"cfg3 operator at n={args.n}",
            "N": N, "leaf": CFG3["leaf"], "eps1": CFG3["eps1"], "eps2": CFG3["eps2"],
            "parallelism": (f"stepping: replicas x{world}; assembly (ACA): admissible blocks sharded over "
                            f"{world} ranks + NCCL all-gather of the factors" if world > 1 else "replicas x1"),
            "l2": "inputs larger than L2 (the operator streamed every step is >= 0.8 GB vs 126 MB L2)"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) > 8:
                for k, nm in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def max_over_ranks(value, world, device):
    """Timing contract: the job's time is the slowest rank's (all_reduce MAX)."""
    if world <= 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


SOLVE_DESC = {
    "propagator": "u <- 2 Z u - u with Z = (A+)^-1 = (LU)^-1 precomputed as an H-matrix from the H-LU "
                  "(one H-matvec per step, DESIGN.md)",
    "inverse": "A- matvec + triangular-inverse H-factors L^-1, U^-1 of the H-LU (DESIGN.md)",
}


def build_system(P, cfg=CFG3, n=None, method="propagator", world=1):
    """Operator assembly (GPU symbol + ACA compression) and factorisation, timed."""
    import torch

    n = n or cfg["n"]
    t0 = time.perf_counter()
    nu = P.cgmy_measure(1.0, 5.0, 10.0, 0.5)
    s = P.FracCNSystem(nu, cfg["a"], cfg["b"], cfg["c"], n, cfg["dt"], L=cfg["L"], L_W=cfg["L_W"],
                       drift_compensation=True, distributed=world > 1)
    torch.cuda.synchronize()
    t_symbol = time.perf_counter() - t0
    hc = P.HConfig(n_min=cfg["leaf"], eps1=cfg["eps1"])
    t1 = time.perf_counter()
    Hp, Hm = s.build_pair(hc)
    torch.cuda.synchronize()
    t_aca = time.perf_counter() - t1
    s.h_minus = Hm
    mem_p = P.memory_report(Hp)
    t2 = time.perf_counter()
    F = P.hlu(Hp, cfg["eps2"])
    torch.cuda.synchronize()
    t_lu = time.perf_counter() - t2
    st = np.zeros(8)
    P._lib.lib().lh_hlu_stats(F.h.handle, P._lib.host_ptr(st))
    t3 = time.perf_counter()
    if method == "propagator":
        F.prepare_propagator()
    elif method == "inverse":
        F.prepare_inverse()
    torch.cuda.synchronize()
    t_prep = time.perf_counter() - t3
    s.factor = F
    s.method = method
    times = dict(symbol_s=t_symbol, aca_s=t_aca, assembly_s=t_symbol + t_aca, hlu_s=t_lu,
                 assembly_sharding=(dict((k, round(v, 4) if isinstance(v, float) else v)
                                         for k, v in Hp.shard_stats.items())
                                    if getattr(Hp, "shard_stats", None) else "unsharded (1 rank)"),
                 hlu_plan_s=float(st[1]), hlu_exec_s=float(st[3]), hlu_tasks=int(st[0]),
                 hlu_plan_chunks=int(st[4]),
                 # the factorisation's algorithmic FP64 work (task list at the factor's
                 # final ranks) and the rates over the executor's seconds
                 hlu_gflop=round(float(st[5]) / 1e9, 1), hlu_gbytes=round(float(st[6]) / 1e9, 1),
                 hlu_tflops=round(float(st[5]) / max(float(st[3]), 1e-9) / 1e12, 3),
                 hlu_GBps=round(float(st[6]) / max(float(st[3]), 1e-9) / 1e9, 1))
    if method == "propagator":
        ps = F.propagator_stats()
        times.update(propagator_s=t_prep, propagator_plan_s=float(ps[1]),
                     propagator_exec_s=float(ps[3]), propagator_tasks=int(ps[0]),
                     propagator_nearfield_lowrank_leaves=int(ps[4]),
                     propagator_coarsening_merges=int(ps[5]),
                     propagator_single_rhs_form=["H-matrix", "shared leaf bases", "nested H2 bases"][int(ps[6])],
                     propagator_form_probe_rel_err=f"{float(ps[7]):.2e}", propagator_leaf_basis_mean=float(ps[8]),
                     propagator_basis_transfer_coupling_scalars=int(ps[9]))
    elif method == "inverse":
        times.update(inverse_factors_s=t_prep)
    free_b, total_b = torch.cuda.mem_get_info()
    times.update(stored_scalars_plus=mem_p["stored_scalars"], setup_total_s=time.perf_counter() - t0,
                 device_mem_used_gb=round((total_b - free_b) / 1e9, 2),
                 note="*_plan_s is host planning on background threads started at the end of "
                      "assembly (overlaps ACA/LU execution); setup_total_s = symbol + ACA + H-LU + "
                      f"{method} preparation, wall clock")
    return s, F, Hm, times


def cpu_reference_steps(P, s, F, Hm, u0, n_steps, max_seconds=None):
    """The reference algorithm on host cores, on the GPU-built factors exported to host:
    levyh.hops.solve(F, levyh.hops.matvec(H-, u)) of the unmodified reference (baseline/_ref)
    when it is installed (kind "reference"), else the oracle restatement (kind "port")."""
    from oracle import levyh_bridge as LB

    leaf = CFG3["leaf"]
    t0 = time.perf_counter()
    levyh = LB.import_levyh()
    if levyh is not None:
        hops = levyh.hops
        Fr = hops.HFactorization(LB.hmatrix_from_export(levyh, s.x, leaf, *P.hmatrix.export_layout(F.h)),
                                 CFG3["eps2"])
        Hr = LB.hmatrix_from_export(levyh, s.x, leaf, *P.hmatrix.export_layout(Hm))
        step, kind = (lambda u: hops.solve(Fr, hops.matvec(Hr, u))), "reference"
    else:
        from oracle import export_bridge as EB
        from oracle import levyh_oracle as O

        Fr = EB.tree_from_export(s.x, leaf, *P.hmatrix.export_layout(F.h))
        Hr = EB.tree_from_export(s.x, leaf, *P.hmatrix.export_layout(Hm))
        step, kind = (lambda u: O.lu_solve(Fr, O.hmatvec(Hr, u))), "port"
    t_export = time.perf_counter() - t0
    u = np.asarray(u0, dtype=float).copy()
    times = []
    for k in range(n_steps):
        t = time.perf_counter()
        u = step(u)
        times.append(time.perf_counter() - t)
        if max_seconds and sum(times) > max_seconds:
            break
    return u, times, t_export, kind


def cpu_info():
    info = {"cores": os.cpu_count()}
    try:
        from threadpoolctl import threadpool_info

        info["blas_threads"] = max((d.get("num_threads", 0) for d in threadpool_info()), default=None)
    except Exception:
        info["blas_threads"] = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return info


def step_roofline(P, ctx, Hm, F, u0, method, ms_per_step, N, traffic_file=True):
    """Per-kernel roofline of one CN step (lh_step_profile: CUDA events on the library stream
    around each launch, 5 steps, algorithmic bytes per launch) against the measured HBM peak."""
    import torch

    L = P._lib.lib()
    mcode = P.SOLVE_METHODS[method]
    prof = np.zeros(16)
    uprof = torch.from_numpy(np.asarray(u0, dtype=float).copy()).cuda()
    P._lib.check(L.lh_step_profile(ctx.h, Hm.handle, F.h.handle, uprof.data_ptr(), 5, mcode,
                                   P._lib.host_ptr(prof)), ctx.h)
    zform = int(F.propagator_stats()[6]) if method == "propagator" else 0
    if method == "propagator" and prof[11] == 1.0:
        # two-kernel H2 step (h2step.cu): x staging copy, K1 (column walk + the
        # dense diagonal leaves), K2 (couplings, row walk, row bases Q_t, epilogue)
        names = ["xpad", "h2s_up(K1)", "h2s_down(K2)"]  # xpad: once per call (0 per step)
        stored = {"A-": int(prof[12]), "Z=(A+)^-1": int(prof[13]), "LU factor": int(prof[15])}
    elif method == "propagator":
        # nested (H2) form: the walk is four short latency-bound launches (leaf / up / couple /
        # down); the segment kernel is the dominant single kernel
        names = ["walk(Z)" if zform == 2 else "vtx(Z)", "seg(Z)"]
        stored = {"A-": int(prof[12]), "Z=(A+)^-1": int(prof[13]), "LU factor": int(prof[15])}
    else:
        names = ["vtx(A-)", "seg(A-)", "vtx(L^-1)", "seg(L^-1)", "vtx(U^-1)", "seg(U^-1)"]
        stored = {"A-": int(prof[12]), "L^-1": int(prof[13]), "U^-1": int(prof[14]),
                  "LU factor": int(prof[15])}
    nk = len(names)
    kms = prof[:nk]
    kbytes = prof[6:6 + nk]
    if prof[11] == 1.0:
        dom = 1 + int(np.argmax(kms[1:]))
    else:
        dom = 1 if zform == 2 else int(np.argmax(kms))
    peak, peak_src = measured_peaks()
    achieved = kbytes[dom] / (kms[dom] / 1000.0) / 1e9
    step_bytes = float(kbytes.sum())
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if traffic_file and os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(names[dom])
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "peak_source": peak_src, "algorithmic_bytes_per_launch": float(kbytes[dom]),
                "kernel_ms": float(kms[dom]),
                "per_kernel": {nm: {"ms": round(float(kms[i]), 4), "GBps": round(kbytes[i] / (kms[i] / 1e3) / 1e9, 1)}
                               for i, nm in enumerate(names) if kms[i] > 0},
                "step_bytes": step_bytes,
                "step_GBps_sum_of_kernels": round(step_bytes / (kms.sum() / 1e3) / 1e9, 1),
                "step_GBps_timed": round(step_bytes / (ms_per_step / 1e3) / 1e9, 1),
                "stored_scalars": stored,
                "reference_algorithm_bytes_per_step": 8.0 * (prof[12] + prof[15] + 6 * N)}

    return roofline


def run_b200(args, world, rank, local):
    import torch

    import paper_1812_08324_b200 as P

    s, F, Hm, times = build_system(P, n=args.n, method=args.method, world=world)
    for k in ("LEVYH_FUSE_DBG", "LEVYH_H2_DBG"):  # timing experiments on the built operator only
        if os.environ.get("BENCH_" + k):
            os.environ[k] = os.environ["BENCH_" + k]
    ctx = Hm.ctx
    L = P._lib.lib()
    N = s.N
    u0 = np.maximum(np.exp(s.x) - 1.0, 0.0)
    u = torch.from_numpy(u0.copy()).cuda()
    mcode = P.SOLVE_METHODS[args.method]

    def steps(k, vec):
        P._lib.check(L.lh_cn_steps(ctx.h, Hm.handle, F.h.handle, vec.data_ptr(), N, 1, int(k), mcode),
                     ctx.h)

    # warm-up (also captures the CUDA graph of one step)
    steps(args.warmup, u)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        time.sleep(0.3)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        # events on the stream the library launches on
        lib_stream = ctx.torch_stream()
        start.record(lib_stream)
        steps(args.steps, u)
        end.record(lib_stream)
        torch.cuda.synchronize()
        ms = start.elapsed_time(end)
        launches_per_step = int(L.lh_step_graph_kernels(F.h.handle))
        # keep the GPU busy for the clock sampler (extra untimed steps)
        t_load = time.perf_counter()
        while time.perf_counter() - t_load < 1.5:
            steps(50, u)
        torch.cuda.synchronize()
    ms = max_over_ranks(ms, world, "cuda")
    ms_per_step = ms / args.steps
    value = world * args.steps / (ms / 1000.0)

    # ---- end to end through the C ABI with HOST buffers (pinned), one step per call
    # (lh_cn_step_host: u in pinned host memory; every call copies u in and the new u out,
    # overlapped piece by piece with the step's kernels, and returns when u is on the host)
    u_host = torch.from_numpy(u0.copy()).pin_memory()
    e2e_steps = max(1, min(args.steps, 50))

    def host_step():
        P._lib.check(L.lh_cn_step_host(ctx.h, Hm.handle, F.h.handle, u_host.data_ptr(),
                                       u_host.data_ptr(), mcode), ctx.h)

    host_step()  # warm (graph for this buffer)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        host_step()
    t_e2e = time.perf_counter() - t0
    e2e = {"value": world * e2e_steps / t_e2e, "unit": "steps/s", "h2d_bytes_per_step": 8 * N,
           "d2h_bytes_per_step": 8 * N,
           "path": "lh_cn_step_host (C ABI, levy.step_cn) with u in pinned host memory, one call per "
                   "step (copies in and out inside the call)"}

    # ---- the reference algorithm on the GPU (A- matvec + substitution solve on the DAG
    # executor, hops.py:65-70 + :424-432) on the same factors, next to the default path
    if args.method != "substitution" and not args.no_sub:
        usub = torch.from_numpy(u0.copy()).cuda()

        def sub_steps(k):
            P._lib.check(L.lh_cn_steps(ctx.h, Hm.handle, F.h.handle, usub.data_ptr(), N, 1, int(k), 0), ctx.h)

        sub_steps(1)
        torch.cuda.synchronize()
        ks = 3
        lib_stream = ctx.torch_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(lib_stream)
        sub_steps(ks)
        e1.record(lib_stream)
        torch.cuda.synchronize()
        sub_ms = e0.elapsed_time(e1) / ks
        sub_line = {"steps_per_s": round(1000.0 / sub_ms, 3), "ms_per_step": round(sub_ms, 3), "steps": ks,
                    "algorithm": "A- matvec + forward/backward substitution (the reference algorithm) on "
                                 "the persistent DAG executor, same factors"}
    else:
        sub_line = None

    roofline = step_roofline(P, ctx, Hm, F, u0, args.method, ms_per_step, N)

    out = {"metric": METRIC, "value": round(value, 3), "unit": "steps/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (BASELINE.json configs[2]; seeded/closed-form inputs, no dataset)",
           "config": cfg3_config(args, N, world), "algorithm": SOLVE_DESC[args.method],
           "clocks": sampler.summary(), "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
           "gpu_launches_per_step": launches_per_step,
           "substitution_on_gpu": sub_line,
           "roofline": roofline, "phases": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in times.items()}}

    if rank == 0 and world == 1 and not args.no_cpu:
        ucpu, ts, t_exp, kind = cpu_reference_steps(P, s, F, Hm, u0, args.cpu_steps, max_seconds=30)
        ci = cpu_info()
        impl = ("levyh.hops.matvec + levyh.hops.solve of the unmodified reference (baseline/_ref)"
                if kind == "reference" else "oracle/levyh_oracle.py (restated hops.matvec + hops.solve)")
        out["cpu_baseline"] = {"value": round(len(ts) / sum(ts), 5), "unit": "steps/s",
                               "cores": ci["cores"], "blas_threads": ci.get("blas_threads"),
                               "cpu_model": ci.get("cpu_model"), "kind": kind,
                               "sample": f"{len(ts)} CN steps (matvec + substitution solve) of the cfg3 operator "
                                         f"at N=2^20 with {impl} on the GPU-built factors exported "
                                         f"to host ({t_exp:.1f}s export, untimed)"}
        # parity at the headline size: the same k steps from u0 on the GPU (default method and
        # the reference algorithm) against the CPU reference on the same factors
        k = len(ts)
        ug = torch.from_numpy(u0.copy()).cuda()
        steps(k, ug)
        us = torch.from_numpy(u0.copy()).cuda()
        P._lib.check(L.lh_cn_steps(ctx.h, Hm.handle, F.h.handle, us.data_ptr(), N, 1, k, 0), ctx.h)
        torch.cuda.synchronize()
        rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
        out["parity"] = {"steps": k, "rel_l2_vs_oracle": rel(ug.cpu().numpy(), ucpu),
                         "rel_l2_substitution_vs_oracle": rel(us.cpu().numpy(), ucpu),
                         "method": args.method, "tolerance": 1e-8,
                         "oracle": f"{impl} on the same exported factors, from the same u0"}
    if rank == 0:
        print(json.dumps(out), flush=True)


def cfg4_bumps(x, K, seed=0):
    """cfg4 initial conditions: per column a sum of 8 Gaussian bumps exp(-((x-c)/w)^2)."""
    rng = np.random.default_rng(seed)
    U = np.zeros((x.shape[0], K))
    for k in range(K):
        c = rng.uniform(-0.8, 0.8, 8)
        w = rng.uniform(0.02, 0.2, 8)
        a = rng.normal(0.0, 1.0, 8)
        U[:, k] = (a[None, :] * np.exp(-((x[:, None] - c[None, :]) / w[None, :]) ** 2)).sum(1)
    return U


def run_cfg4(args, world, rank, local):
    import torch

    import paper_1812_08324_b200 as P

    cfg = CFG4
    t0 = time.perf_counter()
    s = P.FracCNSystem(P.power_measure(1, 0.5), 0.0, 0.0, 0.0, cfg["n"], 1.0 / cfg["n"])
    s.prepare(P.HConfig(n_min=cfg["leaf"], eps1=cfg["eps1"]), cfg["eps2"], method="propagator")
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    F, Hm = s.factor, s.h_minus
    ctx, L, N = Hm.ctx, P._lib.lib(), s.N
    K = cfg["K"]
    lo, hi = rank * K // world, (rank + 1) * K // world  # this rank's columns
    Kr = hi - lo
    U0 = cfg4_bumps(s.x, K)[:, lo:hi]
    u = torch.from_numpy(np.asfortranarray(U0).T.copy()).cuda()  # (Kr, N): column-major N x Kr

    def steps(k, vec):
        P._lib.check(L.lh_cn_steps(ctx.h, Hm.handle, F.h.handle, vec.data_ptr(), N, Kr, int(k), 2), ctx.h)

    steps(args.warmup, u)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        time.sleep(0.3)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        lib_stream = ctx.torch_stream()
        start.record(lib_stream)
        steps(args.steps, u)
        end.record(lib_stream)
        torch.cuda.synchronize()
        ms = start.elapsed_time(end)
    ms = max_over_ranks(ms, world, "cuda")
    ms_per_step = ms / args.steps
    # e2e: each step through the C ABI with the rank's columns in pinned host memory
    u_host = torch.from_numpy(np.asfortranarray(U0).T.copy()).pin_memory()
    u_dev = torch.empty_like(u)
    e2e_steps = max(1, min(args.steps, 10))
    t1 = time.perf_counter()
    for _ in range(e2e_steps):
        u_dev.copy_(u_host, non_blocking=True)
        steps(1, u_dev)
        u_host.copy_(u_dev, non_blocking=True)
        torch.cuda.synchronize()
    t_e2e = max_over_ranks(time.perf_counter() - t1, world, "cuda")
    # DMMA roofline: the algorithmic flops of the multi-RHS form of Z per step: the nested-basis
    # walk (leaves, transfers, couplings) plus the segment matmat of dense leaves and row bases
    # (h2mm.cu), or 2 x stored scalars for the H-form matmat
    zst = F.propagator_stats()
    flops = float(zst[10]) * K
    S_Z = float(zst[10]) / 2.0
    try:
        pk = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_dmma_peak.json")))
        peak, peak_src = float(pk["tflops"]), "measured (profiles/r01_fp64_dmma_peak.json, tools/ubench_dmma.cu)"
    except Exception:
        peak, peak_src = 45.0, "nominal"
    achieved = flops / (ms_per_step / 1e3) / 1e12
    out = {"metric": METRIC4, "value": round(1000.0 / ms_per_step, 3), "unit": "steps/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (BASELINE.json configs[3]; seeded bumps, no dataset)",
           "config": {"workload": cfg["workload"], "N": N, "rhs": K, "rhs_per_rank": Kr,
                      "parallelism": f"columns sharded {K}/{world}",
                      "solve": SOLVE_DESC["propagator"] + "; K right-hand sides per step through the H2 walk as "
                               "batched DMMA products (h2mm.cu)",
                      "l2": "operator and state larger than L2"},
           "rhs_steps_per_s": round(K * 1000.0 / ms_per_step, 1),
           "clocks": sampler.summary(),
           "e2e": {"value": round(world * e2e_steps / t_e2e / world, 3), "unit": "steps/s",
                   "h2d_bytes_per_step": 8 * N * Kr, "d2h_bytes_per_step": 8 * N * Kr,
                   "path": "lh_cn_steps (C ABI) with pinned host columns per step"},
           "gpu_launches": None,
           "roofline": {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                        "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                        "flops_per_step": flops, "scalars_Z_multi_rhs_form": S_Z,
                        "multi_rhs_form": "nested-basis walk as batched DMMA products" if zst[11] == 2 else
                                          "H-form DMMA matmat"},
           "phases": {"setup_total_s": round(t_setup, 3)}}
    if rank == 0:
        print(json.dumps(out), flush=True)


def run_cfg5(args, world, rank, local):
    """BASELINE configs[4]: the large-N phases.  Assembly (symbol + ACA) is sharded across the
    ranks with an NCCL all-gather of the factors; H-LU and the 50 steps run on every rank.
    The step is u <- 2 Z u - u with the propagator Z = (A+)^-1 (default): A- of the CN pair is
    never read by that step, so it is spilled to pinned host memory (HMatrix.spill) and the HBM
    holds the factor and Z.  --method substitution runs the reference algorithm (A- matvec +
    forward/backward substitution) instead."""
    import torch

    import paper_1812_08324_b200 as P

    cfg = CFG5
    method = args.method if args.method_set else "propagator"
    if method != "propagator":
        os.environ["LEVYH_NO_BG_PROP"] = "1"  # no propagator plan (host and device memory)
    mem = {}

    def used_gb():
        free_b, total_b = torch.cuda.mem_get_info()
        return round((total_b - free_b) / 1e9, 2)
    t0 = time.perf_counter()
    s = P.FracCNSystem(P.power_measure(1, 0.8), 0.1, 0.0, 0.0, cfg["n"], 1.0 / cfg["n"],
                       distributed=world > 1)
    torch.cuda.synchronize()
    t_symbol = time.perf_counter() - t0
    # low-rank capacity 24 (H-LU updates add two ranks of ~7): the factor, A-, and A-'s packed
    # matvec copy then fit one GPU at N = 2^22
    hc = P.HConfig(n_min=cfg["leaf"], eps1=cfg["eps1"], kcap=int(os.environ.get("LEVYH_CFG5_KCAP", "24")))
    t1 = time.perf_counter()
    Hp, Hm = s.build_pair(hc)
    torch.cuda.synchronize()
    t_aca = time.perf_counter() - t1
    mem_p = P.memory_report(Hp)
    mem["after_assembly"] = used_gb()
    t_spill = 0.0
    if method == "propagator":
        ts = time.perf_counter()
        Hm.spill()
        t_spill = time.perf_counter() - ts
        mem["after_spill_of_A-"] = used_gb()
    t2 = time.perf_counter()
    F = P.hlu(Hp, cfg["eps2"])
    torch.cuda.synchronize()
    t_lu = time.perf_counter() - t2
    st = np.zeros(8)
    P._lib.lib().lh_hlu_stats(F.h.handle, P._lib.host_ptr(st))
    t3 = time.perf_counter()
    if method == "propagator":
        F.prepare_propagator()
    elif method == "inverse":
        F.prepare_inverse()
    torch.cuda.synchronize()
    t_prep = time.perf_counter() - t3
    mem["after_prepare"] = used_gb()
    ctx, L, N = Hm.ctx, P._lib.lib(), s.N
    u0 = np.maximum(1.0 - s.x ** 2, 0.0) ** 3
    u = torch.from_numpy(u0.copy()).cuda()
    mcode = P.SOLVE_METHODS[method]
    k = min(args.steps, cfg["steps"])

    def steps(kk):
        P._lib.check(L.lh_cn_steps(ctx.h, Hm.handle, F.h.handle, u.data_ptr(), N, 1, int(kk), mcode), ctx.h)

    steps(1)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        lib_stream = ctx.torch_stream()
        start.record(lib_stream)
        steps(k)
        end.record(lib_stream)
        torch.cuda.synchronize()
        ms = start.elapsed_time(end)
    ms = max_over_ranks(ms, world, "cuda")
    free_b, total_b = torch.cuda.mem_get_info()
    out = {"metric": METRIC5, "value": round(world * k / (ms / 1000.0), 3), "unit": "steps/s",
           "n_gpus": world, "steps": k, "warmup": 1, "ms_per_step": round(ms / k, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (BASELINE.json configs[4]; closed-form inputs, no dataset)",
           "config": {"workload": cfg["workload"], "N": N, "leaf": cfg["leaf"], "solve": method,
                      "parallelism": f"assembly sharded over {world} rank(s); H-LU and steps replicated"},
           "clocks": sampler.summary(),
           "phases": {"symbol_s": round(t_symbol, 3), "aca_s": round(t_aca, 3),
                      "assembly_s": round(t_symbol + t_aca, 3), "hlu_s": round(t_lu, 3),
                      "hlu_plan_s": round(float(st[1]), 3), "hlu_exec_s": round(float(st[3]), 3),
                      "hlu_tasks": int(st[0]), "prepare_s": round(t_prep, 3),
                      "assembly_sharding": (Hp.shard_stats if getattr(Hp, "shard_stats", None)
                                            else "unsharded (1 rank)"),
                      "stored_scalars_plus": mem_p["stored_scalars"],
                      "spill_A-_s": round(t_spill, 3),
                      "device_mem_used_gb": round((total_b - free_b) / 1e9, 2), "device_mem_gb": mem}}
    if method in ("propagator", "inverse"):
        out["roofline"] = step_roofline(P, ctx, Hm, F, u0, method, ms / k, N, traffic_file=False)
    if method == "propagator":
        zs = F.propagator_stats()
        out["phases"]["propagator_form"] = int(zs[6])
        out["phases"]["propagator_form_probe_rel_err"] = f"{zs[7]:.2e}"
    if rank == 0:
        print(json.dumps(out), flush=True)


METRIC_G = ("reference bench system (cli.bench_point: Gaussian jumps, rank 10, leaf 64) at N=2^20: "
            "construct / matvec / H-LU / solve seconds; CN steps/s")


def run_gauss(args, world, rank, local):
    """The reference's own benchmark system (cli.bench_point, cli.py:163-224):
    gaussian_measure(5.0), a=b=c=0, UniformGrid1D(2^20), dt=0.01, HConfig(n_min=64,
    fixed_rank=10, eps1=1e-4), eps2=1e-10.  Times the four bench kinds (construct = series
    H-build of A+, matvec, H-LU, solve by substitution = the reference algorithm) with the
    reference's median-of-repeats convention, plus CN steps/s (one H-matvec of Z per step)."""
    if rank != 0:
        return
    import torch

    import paper_1812_08324_b200 as P

    n = 2 ** 20
    rep = 3

    def med(fn):
        ts = []
        for k in range(rep + 1):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        return float(np.median(ts[1:])), r

    s = P.assemble_cn_1d(P.gaussian_measure(5.0), 0.0, 0.0, 0.0, P.UniformGrid1D(n), 0.01)
    cfg = P.HConfig(n_min=64, fixed_rank=10, eps1=1e-4)
    t_con, H = med(lambda: s.hmatrix("plus", cfg))
    stored = P.memory_report(H)["stored_scalars"]
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
    t_mv, _ = med(lambda: P.matvec(H, x))
    lu_times = []
    Hm = None
    for k in range(rep + 1):
        if k < rep:
            Hk = s.hmatrix("plus", cfg)
        else:  # the pair CNSystem.prepare builds: A- derived from A+ (takes the 2 Z u - u step)
            Hk, Hm = s.build_pair(cfg)
        torch.cuda.synchronize()
        t = time.perf_counter()
        F = P.hlu(Hk, 1e-10)
        torch.cuda.synchronize()
        lu_times.append(time.perf_counter() - t)
    t_lu = float(np.median(lu_times[1:]))
    t_sol, _ = med(lambda: P.solve(F, x, method="substitution"))
    t0 = time.perf_counter()
    F.prepare_propagator()
    torch.cuda.synchronize()
    t_prop = time.perf_counter() - t0
    t_solz, _ = med(lambda: P.solve(F, x, method="propagator"))
    s.h_minus, s.factor, s.method = Hm, F, "propagator"
    u = torch.from_numpy(np.exp(-50 * s.grid.points ** 2)).cuda()
    L, ctx = P._lib.lib(), s.h_minus.ctx

    def steps(k):
        P._lib.check(L.lh_cn_steps(ctx.h, s.h_minus.handle, F.h.handle, u.data_ptr(), n, 1, int(k), 2),
                     ctx.h)

    steps(args.warmup)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib_stream = ctx.torch_stream()
    start.record(lib_stream)
    steps(args.steps)
    end.record(lib_stream)
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / args.steps
    out = {"metric": METRIC_G, "value": round(1000.0 / ms, 3), "unit": "steps/s", "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (the reference bench system, closed-form symbol)",
           "config": {"workload": "cli.bench_point system: gaussian_measure(5.0), a=b=c=0, N=2^20, "
                                  "dt=0.01, leaf 64, fixed_rank 10, eps1 1e-4, eps2 1e-10",
                      "N": n, "repeat": rep, "warmup_repeats": 1},
           "bench_point_seconds": {"construct": round(t_con, 4), "matvec": round(t_mv, 6),
                                   "lu": round(t_lu, 4), "solve": round(t_sol, 6),
                                   "solve_propagator": round(t_solz, 6),
                                   "propagator_prepare": round(t_prop, 4)},
           "stored_scalars": stored,
           "reference_context": {"source": "BASELINE.md 2(a) (reference levyh bench, survey container, "
                                           "8 vCPU; not this run) and BASELINE.md 1 (paper, Julia)",
                                 "reference_cpu_2^20": {"matvec": 2.363, "solve": 2.033, "lu": 239.6},
                                 "paper_julia_2^20": {"construct": 81.86, "matvec": 1.7325,
                                                      "lu": 125.12, "solve": 1.4913}}}
    print(json.dumps(out), flush=True)


def export_factors(args):
    """--export-factors DIR: the reference arm's input preparation, run as a CHILD process so
    the process that times the reference never loads the native library.  Builds the cfg3
    operators on the GPU (the reference cannot assemble them at N = 2^20) and writes
    the exported layouts (oracle/levyh_bridge.py reads them) of A- and of the H-LU factor of A+,
    and with --export-plus also the unfactored A+ (for timing the reference hops.hlu)."""
    import paper_1812_08324_b200 as P

    cfg = CFG3
    n = args.n or cfg["n"]
    s = P.FracCNSystem(P.cgmy_measure(1.0, 5.0, 10.0, 0.5), cfg["a"], cfg["b"], cfg["c"], n, cfg["dt"],
                       L=cfg["L"], L_W=cfg["L_W"], drift_compensation=True)
    Hp, Hm = s.build_pair(P.HConfig(n_min=cfg["leaf"], eps1=cfg["eps1"]))

    def dump(H, name):
        d = os.path.join(args.export_factors, name)
        os.makedirs(d, exist_ok=True)
        for k, v in zip(("recs", "arena", "ranks", "perm"), P.hmatrix.export_layout(H)):
            np.save(os.path.join(d, k + ".npy"), v)

    np.save(os.path.join(args.export_factors, "x.npy"), s.x)
    if args.export_plus:
        dump(Hp, "plus")
    dump(Hm, "minus")
    F = P.hlu(Hp, cfg["eps2"])
    dump(F.h, "factor")


def _scratch_dir(need_gb):
    import shutil
    import tempfile

    for base in ("/dev/shm", None):
        try:
            if base is None or shutil.disk_usage(base).free > need_gb * 1e9:
                return tempfile.mkdtemp(prefix="levyh_ref_", dir=base)
        except Exception:
            continue
    return tempfile.mkdtemp(prefix="levyh_ref_")


def reference_inputs(args, plus=False):
    """Run the export child and load the factors as the REAL reference's block types
    (levyh from baseline/_ref) -- or as the oracle restatement's when levyh is not installed.
    Returns (kind, api, x, Fh, Hm, Hp_or_None, export_seconds)."""
    import shutil

    from oracle import levyh_bridge as LB

    d = _scratch_dir(40 if plus else 30)
    t0 = time.perf_counter()
    try:
        cmd = [sys.executable, os.path.abspath(__file__), "--export-factors", d]
        if args.n:
            cmd += ["--n", str(args.n)]
        if plus:
            cmd += ["--export-plus"]
        env = dict(os.environ)
        for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
            env.pop(k, None)
        subprocess.run(cmd, check=True, env=env)
        t_exp = time.perf_counter() - t0
        x = np.load(os.path.join(d, "x.npy"))
        levyh = LB.import_levyh()
        leaf = CFG3["leaf"]
        if levyh is not None:
            mk = lambda name: LB.hmatrix_from_export(levyh, x, leaf, *LB.load_export(os.path.join(d, name)))
            Fh, Hm = mk("factor"), mk("minus")
            Hp = mk("plus") if plus else None
            return "reference", levyh, x, Fh, Hm, Hp, t_exp
        from oracle import export_bridge as EB

        mk = lambda name: EB.tree_from_export(x, leaf, *LB.load_export(os.path.join(d, name)))
        return "port", None, x, mk("factor"), mk("minus"), (mk("plus") if plus else None), t_exp
    finally:
        shutil.rmtree(d, ignore_errors=True)


def run_reference(args, world, rank, local):
    """--impl reference: the reference's own CPU implementation of the path on the host cores
    (rank 0 only): levyh.hops.matvec + levyh.hops.solve (hops.py:65-70, :424-432) of the
    UNMODIFIED reference installed in baseline/_ref, stepping levyh.levy.run_cn's loop
    (levy.py:309-330) on the cfg3 operators (exported from the GPU build by a child process).
    --ref-phase hlu times levyh.hops.hlu on the exported, unfactored A+ instead."""
    if rank != 0:
        return
    kind, levyh, x, Fh, Hm, Hp, t_exp = reference_inputs(args, plus=args.ref_phase == "hlu")
    N = len(x)
    if kind == "reference":
        hops = levyh.hops
        F = hops.HFactorization(Fh, CFG3["eps2"])
        step = lambda u: hops.solve(F, hops.matvec(Hm, u))
        impl_desc = ("levyh.hops.solve(F, levyh.hops.matvec(H-, u)) of the unmodified reference "
                     "(baseline/_ref, levyh 0.1.0)")
    else:
        from oracle import levyh_oracle as O

        step = lambda u: O.lu_solve(Fh, O.hmatvec(Hm, u))
        impl_desc = "oracle/levyh_oracle.py restatement of hops.matvec + hops.solve (levyh not installed)"
    ci = cpu_info()
    if args.ref_phase == "hlu":
        t = time.perf_counter()
        if kind == "reference":
            levyh.hops.hlu(Hp, CFG3["eps2"])
        else:
            from oracle import levyh_oracle as O

            O.hlu(Hp, CFG3["eps2"])
        t_lu = time.perf_counter() - t
        print(json.dumps({"impl": "reference", "phase": "hlu", "N": N, "hlu_s": round(t_lu, 3),
                          "kind": kind, "cores": ci["cores"], "blas_threads": ci.get("blas_threads"),
                          "cpu_model": ci.get("cpu_model")}), flush=True)
        return
    u = np.maximum(np.exp(x) - 1.0, 0.0)
    warm = min(args.warmup, 1)
    k = max(1, min(args.steps, args.ref_steps))
    ts = []
    for i in range(warm + k):
        t = time.perf_counter()
        u = step(u)
        ts.append(time.perf_counter() - t)
    ts = ts[warm:]
    value = len(ts) / sum(ts)
    out = {"metric": METRIC, "value": round(value, 5), "unit": "steps/s", "n_gpus": world,
           "steps": len(ts), "warmup": warm, "ms_per_step": round(1000 * sum(ts) / len(ts), 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (BASELINE.json configs[2]; seeded/closed-form inputs, no dataset)",
           "impl": "reference", "config": cfg3_config(args, N, world),
           "algorithm": "A- matvec + forward/backward substitution solve per step (hops.py:65-70, :424-432)",
           "cpu_baseline": {"value": round(value, 5), "unit": "steps/s", "cores": ci["cores"],
                            "blas_threads": ci.get("blas_threads"), "cpu_model": ci.get("cpu_model"),
                            "kind": kind,
                            "sample": f"{len(ts)} timed CN steps (+{warm} warm-up) of {impl_desc} on the cfg3 "
                                      f"factors built on the GPU by a child process and exported to host "
                                      f"({t_exp:.1f}s, untimed; the reference cannot assemble at N=2^20, "
                                      f"SURVEY G7); this process never loads the native library"},
           "e2e": {"value": round(value, 5), "unit": "steps/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override half-grid n (N = 2n-1); default 2^19")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--ref-steps", type=int, default=100, help="cap on the reference arm's timed steps")
    ap.add_argument("--ref-phase", default="steps", choices=["steps", "hlu"])
    ap.add_argument("--export-factors", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--export-plus", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the GPU substitution-step timing")
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg4", "cfg5", "gauss"])
    ap.add_argument("--method", default=None, choices=["propagator", "inverse", "substitution"],
                    help="per-step solve: one H-matvec of Z=(A+)^-1 (default; cfg5: substitution)")
    args = ap.parse_args()
    args.method_set = args.method is not None
    if args.method is None:
        args.method = "propagator"
    if args.export_factors:
        export_factors(args)
        return
    if args.warmup < 3:
        log("warning: fewer than 3 warm-up steps")
    if args.impl == "reference":
        # the reference arm runs on host cores only: no CUDA context, no native library
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, world, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")))
        return
    world, rank, local = dist_setup()
    if args.workload == "cfg4":
        run_cfg4(args, world, rank, local)
    elif args.workload == "cfg5":
        run_cfg5(args, world, rank, local)
    elif args.workload == "gauss":
        run_gauss(args, world, rank, local)
    else:
        run_b200(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
