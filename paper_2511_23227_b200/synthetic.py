"""Synthetic scene generators for BASELINE.json configs 3 and 4, which name
scene types the reference has no generator for ("builder
defines"): a LiDAR-like ring scan and a surface-sampled indoor fragment.
Host-side numpy, seeded.  The reference's own generators (uniform cube,
features, weights: synthetic.hpp, tensors.hpp:142-150) are exported by
libnpcg.so as host functions and wrapped here, so product code never needs
oracle/ (test infrastructure) for its inputs."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def _check(st: int, what: str):
    if st != 0:
        raise ValueError(f"{what}: {L.STATUS_NAMES.get(st, st)}")


def gen_uniform_cube(n: int, extent: float, seed: int) -> np.ndarray:
    """synthetic.cpp:12-23 (the reference's stream, via npcg_gen_uniform_cube)."""
    out = np.empty((n, 3), dtype=np.float64)
    _check(L.lib().npcg_gen_uniform_cube(n, extent, seed, out.ctypes.data_as(C.c_void_p)),
           "gen_uniform_cube")
    return out


def gen_features(n: int, groups: int, channels: int, seed: int, dtype=np.float32) -> np.ndarray:
    """synthetic.hpp:33-40: uniform in [-1, 1) (npcg_gen_features)."""
    out = np.empty((n, groups, channels), dtype=dtype)
    _check(L.lib().npcg_gen_features(n, groups, channels, seed, 0 if dtype == np.float32 else 1,
                                     out.ctypes.data_as(C.c_void_p)), "gen_features")
    return out


def make_weights(t: int, groups: int, c_in: int, c_out: int, seed: int,
                 dtype=np.float32) -> np.ndarray:
    """tensors.hpp:142-150: uniform in [-s, s), s = (G C_in)^(-1/2) (npcg_make_weights)."""
    out = np.empty((t ** 3, groups, c_in, c_out), dtype=dtype)
    _check(L.lib().npcg_make_weights(t, groups, c_in, c_out, seed,
                                     0 if dtype == np.float32 else 1,
                                     out.ctypes.data_as(C.c_void_p)), "make_weights")
    return out


def gen_lidar_scan(n: int, seed: int) -> np.ndarray:
    """64-beam spinning scan from 1.7 m over a ground plane with 40 axis-aligned
    boxes (cars / walls), elevations -25..+3 deg, 60 m max range, 1 cm range
    noise: range-dependent density (rings thin out with distance).  Returns the
    first n hits in azimuth-sweep order (the scan order), float64 metres."""
    rng = np.random.default_rng(seed)
    lo = np.c_[rng.uniform(-40, 40, 40), rng.uniform(-40, 40, 40), np.zeros(40)]
    size = np.c_[rng.uniform(1.5, 6, 40), rng.uniform(1.5, 6, 40), rng.uniform(1.2, 3.5, 40)]
    keep_box = np.hypot(lo[:, 0] + size[:, 0] / 2, lo[:, 1] + size[:, 1] / 2) > 4
    lo, hi = lo[keep_box], lo[keep_box] + size[keep_box]
    elev = np.deg2rad(np.linspace(-25.0, 3.0, 64))
    origin = np.array([0.0, 0.0, 1.7])
    pts = []
    total = 0
    n_az = 2048
    sweep = 0
    while total < n:
        az = (np.arange(n_az) + rng.uniform(0, 1)) * (2 * np.pi / n_az) + sweep * 1e-3
        sweep += 1
        el, a = np.meshgrid(elev, az)  # azimuth-major scan order
        d = np.stack([np.cos(el) * np.cos(a), np.cos(el) * np.sin(a), np.sin(el)], -1).reshape(-1, 3)
        t = np.full(len(d), np.inf)
        down = d[:, 2] < 0
        t[down] = -origin[2] / d[down, 2]
        with np.errstate(divide="ignore", invalid="ignore"):
            inv = 1.0 / d
            for b in range(len(lo)):
                t1 = (lo[b] - origin) * inv
                t2 = (hi[b] - origin) * inv
                tmin = np.nanmax(np.minimum(t1, t2), axis=1)
                tmax = np.nanmin(np.maximum(t1, t2), axis=1)
                hit = (tmax >= np.maximum(tmin, 0)) & (tmin > 0)
                t = np.where(hit & (tmin < t), tmin, t)
        ok = t < 60.0
        p = origin + d[ok] * (t[ok] + rng.normal(0, 0.01, ok.sum()))[:, None]
        pts.append(p)
        total += len(p)
    return np.concatenate(pts)[:n].astype(np.float64)


def gen_indoor_fragment(n: int, seed: int) -> tuple[np.ndarray, float]:
    """Surface-sampled room fragment (6 x 5 x 2.8 m: floor, three walls, no
    ceiling) with 25 furniture boxes (5 faces each), uniform per unit area,
    2 mm noise, random point order.  Returns (xyz, surface area in m^2)."""
    rng = np.random.default_rng(seed)
    rects = []  # (origin, u, v) parallelograms

    def box(o, s):
        x, y, z = o
        a, b, c = s
        rects.extend([((x, y, z + c), (a, 0, 0), (0, b, 0)),   # top
                      ((x, y, z), (a, 0, 0), (0, 0, c)), ((x, y + b, z), (a, 0, 0), (0, 0, c)),
                      ((x, y, z), (0, b, 0), (0, 0, c)), ((x + a, y, z), (0, b, 0), (0, 0, c))])
    rects.append(((0, 0, 0), (6, 0, 0), (0, 5, 0)))           # floor
    rects.append(((0, 0, 0), (6, 0, 0), (0, 0, 2.8)))         # walls
    rects.append(((0, 0, 0), (0, 5, 0), (0, 0, 2.8)))
    rects.append(((6, 0, 0), (0, 5, 0), (0, 0, 2.8)))
    for _ in range(25):
        s = rng.uniform([0.4, 0.4, 0.4], [2.0, 1.2, 1.8])
        o = rng.uniform([0.1, 0.1, 0.0], [6 - s[0] - 0.1, 5 - s[1] - 0.1, 0.0 + 1e-9])
        box(o, s)
    o = np.array([r[0] for r in rects], float)
    u = np.array([r[1] for r in rects], float)
    v = np.array([r[2] for r in rects], float)
    area = np.linalg.norm(np.cross(u, v), axis=1)
    face = rng.choice(len(rects), size=n, p=area / area.sum())
    a, b = rng.random(n), rng.random(n)
    xyz = o[face] + a[:, None] * u[face] + b[:, None] * v[face] + rng.normal(0, 0.002, (n, 3))
    return xyz, float(area.sum())
