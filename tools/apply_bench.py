"""Times the matrix-free evaluators and the variable-order assembly on the GPU (CUDA events on
the library's stream, warm-up first) and prints one JSON object with each kernel's achieved rate
against the bound that applies: FP64 multiply-add throughput for the window correlations
(2 flops per output x tap; peak = the FP64 rate measured on this pool, profiles/r01_fp64_dmma_peak.json),
HBM writes for the assembly (8 m^2 bytes; peak from MEASURED_PEAKS.json).

    python tools/apply_bench.py > gpurun_out/apply_bench.json
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1812_08324_b200 as P  # noqa: E402


def timed(fn, reps=3):
    ctx = P._lib.Context.get()
    st = ctx.torch_stream()
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 6500.0))
    fp64 = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_dmma_peak.json")))["tflops"]
    out = {"fp64_peak_tflops": fp64, "hbm_peak_gbs": hbm, "cases": []}
    for logk in (14, 17, 19):
        K = 2 ** logk
        cfg = P.FracConfig(s=0.5, h=1.0 / K, L=1.0, L_W=2.0, rho_r=0.2)
        M = cfg.n_window
        u = torch.randn(2 * (M + K) + 1, dtype=torch.float64, device="cuda")
        ms = timed(lambda: P.frac_apply_1d(u, cfg))
        flops = 2.0 * (2 * K + 1) * (2 * M + 1)
        out["cases"].append({"op": "frac_apply_1d", "main_points": 2 * K + 1, "window_taps": 2 * M + 1,
                             "ms": ms, "tflops": flops / ms / 1e9, "frac_of_fp64_peak": flops / ms / 1e9 / fp64})
    for K, M in ((64, 64), (128, 128)):
        h = 1.0 / K
        cfg = P.FracConfig(s=0.5, h=h, L=1.0, L_W=M * h, rho_r=0.2, dim=2)
        side = 2 * (M + K) + 1
        u = torch.randn((side, side), dtype=torch.float64, device="cuda")
        ms = timed(lambda: P.frac_apply_2d(u, cfg))
        flops = 2.0 * (2 * K + 1) ** 2 * (2 * M + 1) ** 2
        out["cases"].append({"op": "frac_apply_2d", "main_points": (2 * K + 1) ** 2, "window_taps": (2 * M + 1) ** 2,
                             "ms": ms, "tflops": flops / ms / 1e9, "frac_of_fp64_peak": flops / ms / 1e9 / fp64})
    for n in (48, 64, 128, 192):
        m = 3 * n * n // 4
        ms = timed(lambda: P.assemble_variable_order(n, device=True), reps=2)
        W = 2 * n + 1
        out["cases"].append({"op": "assemble_variable_order", "n": n, "rows": m, "window_offsets_per_row": W * W,
                             "ms": ms, "matrix_GB": 8.0 * m * m / 1e9, "write_GBps": 8.0 * m * m / ms / 1e6,
                             "frac_of_hbm_peak": 8.0 * m * m / ms / 1e6 / hbm,
                             "kernel_evaluations_per_s": m * W * W / ms * 1e3})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
