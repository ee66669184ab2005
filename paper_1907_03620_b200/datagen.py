"""The five BASELINE.json workloads as seeded generator specs
(include/raster_datagen.h). x = longitude, y = latitude.

    cfg  points  structure                                         p  tau mu
    1    1M      1,000 Gaussian clusters x 1,000, sigma 0.005      2  5   4
    2    10M     10,000 x 900, sigma 0.005, + 1M uniform noise     2  5   4
    3    100M    100,000 x 1,000, sigma 0.0005                     3  5   4
    4    500M    1,000,000 x 500, sigma 0.0005                     3  4   4
    5    200M    100M blob (sigma 1e-4) + 1,000 walks x 20,000     3  3   4
                 steps of 0.001 (3 points per position) + 40M noise

`scale` shrinks the cluster/walk/noise counts (same shapes and densities) for
parity tests the CPU oracle finishes in seconds.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .raster import Bounds, GridParams

SEEDS = {1: 0x5EED0001, 2: 0x5EED0002, 3: 0x5EED0003, 4: 0x5EED0004, 5: 0x5EED0005}


def spec(config: int, scale: float = 1.0, seed: int | None = None) -> N.rg_gen_spec:
    s = N.rg_gen_spec()
    s.seed = SEEDS[config] if seed is None else seed
    s.x_lo, s.x_hi, s.y_lo, s.y_hi = -180.0, 180.0, -90.0, 90.0

    def k(v):
        return max(1, int(round(v * scale)))

    if config == 1:
        s.n_clusters, s.points_per_cluster, s.sigma = k(1000), 1000, 0.005
    elif config == 2:
        s.n_clusters, s.points_per_cluster, s.sigma = k(10000), 900, 0.005
        s.n_noise = k(1_000_000)
    elif config == 3:
        s.n_clusters, s.points_per_cluster, s.sigma = k(100_000), 1000, 0.0005
    elif config == 4:
        s.n_clusters, s.points_per_cluster, s.sigma = k(1_000_000), 500, 0.0005
    elif config == 5:
        s.blob_points, s.blob_sigma = k(100_000_000), 1e-4
        s.n_walks, s.walk_steps, s.points_per_step, s.step = k(1000), 20000, 3, 0.001
        s.n_noise = k(40_000_000)
    else:
        raise ValueError(f"unknown config {config}")
    return s


def params(config: int) -> GridParams:
    p, tau = {1: (2, 5), 2: (2, 5), 3: (3, 5), 4: (3, 4), 5: (3, 3)}[config]
    return GridParams(precision=float(p), bounds=Bounds.gps(), threshold=tau, distance=1,
                      min_cluster_size=4)


def count(s: N.rg_gen_spec) -> int:
    return int(N.gen().rg_gen_count(C.byref(s)))


def generate_into(s: N.rg_gen_spec, out_ptr: int, threads: int = 0) -> None:
    if N.gen().rg_generate(C.byref(s), out_ptr, threads) != 0:
        raise RuntimeError("generation failed")


def generate(s: N.rg_gen_spec, threads: int = 0, shuffle_seed: int | None = None) -> np.ndarray:
    n = count(s)
    out = np.empty((n, 2), np.float64)
    if n:
        generate_into(s, out.ctypes.data, threads)
    if shuffle_seed is not None and n:
        out = shuffle(out, shuffle_seed, threads)
    return out


def shuffle(pts: np.ndarray, seed: int, threads: int = 0) -> np.ndarray:
    src = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
    out = np.empty_like(src)
    if N.gen().rg_shuffle(src.ctypes.data, out.ctypes.data, src.shape[0], seed, threads) != 0:
        raise RuntimeError("shuffle failed")
    return out
