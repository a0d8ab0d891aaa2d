"""On-disk formats and measurement helpers around the path: the CSV layout
with '#' metadata lines, the hashed .npy reference-solution cache, and the timing / order-fit
helpers the studies use -- /root/reference/pkg/src/levyh/cli.py:71-135.  Files written here are
readable by the reference's CLI and vice versa (same file names, same number formatting).

The cache holds device results too: ``cache_store`` accepts a torch tensor and ``cache_load``
can return the array on the GPU (``device=...``), so a cached fine-grid reference solution of a
convergence study goes straight back into HBM.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

__all__ = ["write_csv", "read_csv", "median_time", "fit_loglog_slope", "fit_order", "cache_path",
           "cache_load", "cache_store"]


def _cell(v):
    if isinstance(v, (float, np.floating)):
        return f"{float(v):.17g}"
    s = str(v)
    if any(ch in s for ch in ',"\r\n'):
        s = '"' + s.replace('"', '""') + '"'
    return s


def write_csv(path, header, rows, meta=()):
    """cli.py:71-83: '# ' metadata lines, a header row, LF endings; floats as %.17g (they
    round-trip), everything else as str; ``path`` None/'' writes to stdout."""
    fh = open(path, "w", newline="", encoding="utf-8") if path else sys.stdout
    try:
        fh.writelines(f"# {line}\n" for line in meta)
        fh.write(",".join(_cell(h) for h in header) + "\n")
        for row in rows:
            fh.write(",".join(_cell(v) for v in row) + "\n")
    finally:
        if path:
            fh.close()


def read_csv(path):
    """Inverse of write_csv: (meta lines, header, rows of strings)."""
    import csv

    meta, body = [], []
    with open(path, newline="", encoding="utf-8") as fh:
        for line in fh:
            if line.startswith("# ") and not body:
                meta.append(line[2:].rstrip("\n"))
            else:
                body.append(line)
    rows = list(csv.reader(body))
    return meta, rows[0], rows[1:]


def median_time(fn, repeat=3, warmup=1):
    """cli.py:96-106: median wall time of fn() over ``repeat`` runs after ``warmup`` runs; returns
    (seconds, last result).  GPU work inside fn must end synchronised (the C ABI's host-returning
    calls are; for device-resident results pass a fn that calls Context.synchronize())."""
    result = None
    for _ in range(warmup):
        result = fn()
    times = []
    for _ in range(max(1, repeat)):
        t0 = time.perf_counter()
        result = fn()
        times.append(time.perf_counter() - t0)
    return float(np.median(times)), result


def fit_loglog_slope(xs, ys):
    """cli.py:109-113: least-squares slope of log y against log x."""
    lx, ly = np.log(np.asarray(xs, dtype=float)), np.log(np.asarray(ys, dtype=float))
    return float(np.polyfit(lx, ly, 1)[0])


def fit_order(params, errors):
    """cli.py:116-118: convergence order = -slope of log error against log parameter."""
    return -fit_loglog_slope(params, errors)


def cache_path(cache_dir, key):
    """cli.py:124, :134: <cache_dir>/<first 24 hex digits of sha256(key)>.npy."""
    return os.path.join(cache_dir, hashlib.sha256(key.encode()).hexdigest()[:24] + ".npy")


def cache_load(cache_dir, key, device=None):
    """cli.py:121-128: the cached array for ``key`` or None (also None without a cache_dir)."""
    if not cache_dir:
        return None
    path = cache_path(cache_dir, key)
    if not os.path.exists(path):
        return None
    arr = np.load(path)
    if device is None:
        return arr
    import torch

    return torch.from_numpy(arr).to(device)


def cache_store(cache_dir, key, arr):
    """cli.py:131-135: np.save under the hashed name (directory created on demand)."""
    if not cache_dir:
        return
    os.makedirs(cache_dir, exist_ok=True)
    if hasattr(arr, "detach"):
        arr = arr.detach().cpu().numpy()
    np.save(cache_path(cache_dir, key), arr)
