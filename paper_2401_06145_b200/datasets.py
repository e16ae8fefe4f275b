"""Synthetic point clouds with the shapes of the BASELINE configs.

No datasets exist offline; these generators produce deterministic clouds (numpy
SplitMix-seeded Generator) with the geometry the configs name:
  * kitti_scan      — 64-beam LiDAR (elevation -24.8..+2 deg, sensor at 1.73 m) ray-cast
                      against a ground plane + random boxes/cylinders, range <= 80 m,
                      voxelised at 5 cm (~120k voxels; 4 channels x, y, z, intensity)
  * s3dis_room      — 8 x 6 x 3 m room (floor, ceiling, walls, furniture boxes),
                      surface-sampled, voxelised at 2.5 cm (~300k voxels; xyz + rgb)
  * shapenet_object — union of random primitives, surface-sampled in a 128^3 grid
                      (~2-5e4 voxels)
`voxelize` follows the reference's semantics (geometry.hpp:184-255: floor to the grid,
duplicates merged by mean, output sorted by packed key).
"""
from __future__ import annotations

import numpy as np

BIAS = 1 << 20


def pack(xyz: np.ndarray) -> np.ndarray:
    x = xyz.astype(np.int64) + BIAS
    return (x[:, 0] << 42) | (x[:, 1] << 21) | x[:, 2]


def voxelize(points: np.ndarray, features: np.ndarray, resolution: float):
    """Floor to the grid, merge duplicates by mean, sort by packed key (reference voxelize)."""
    v = np.floor(points / resolution).astype(np.int64)
    keys = pack(v)
    uniq, inv = np.unique(keys, return_inverse=True)
    counts = np.bincount(inv, minlength=len(uniq)).astype(np.float64)
    feats = np.zeros((len(uniq), features.shape[1]), np.float64)
    np.add.at(feats, inv, features.astype(np.float64))
    feats /= counts[:, None]
    coords = np.stack([(uniq >> 42) & 0x1FFFFF, (uniq >> 21) & 0x1FFFFF, uniq & 0x1FFFFF], 1) - BIAS
    return coords.astype(np.int32), feats.astype(np.float32)


def _ray_box(o, d, lo, hi):
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        t0 = (lo - o) * inv
        t1 = (hi - o) * inv
    tmin = np.nanmax(np.minimum(t0, t1), axis=1)
    tmax = np.nanmin(np.maximum(t0, t1), axis=1)
    hit = (tmax >= np.maximum(tmin, 0)) & (tmax > 0)
    return np.where(hit, np.maximum(tmin, 0), np.inf)


def _ray_cylinder(o, d, cx, cy, r, h):
    ox, oy = o[0] - cx, o[1] - cy
    a = d[:, 0] ** 2 + d[:, 1] ** 2
    b = 2 * (ox * d[:, 0] + oy * d[:, 1])
    c = ox * ox + oy * oy - r * r
    disc = b * b - 4 * a * c
    with np.errstate(invalid="ignore", divide="ignore"):
        t = (-b - np.sqrt(disc)) / (2 * a)
    z = o[2] + t * d[:, 2]
    ok = (disc >= 0) & (t > 0) & (z >= 0) & (z <= h)
    return np.where(ok, t, np.inf)


def kitti_scan(seed: int = 0, n_azimuth: int = 2900, beams: int = 64, max_range: float = 80.0,
               resolution: float = 0.05, raw: bool = False):
    """Simulated 64-beam LiDAR scan; raw=True returns the points (float64) + features before
    voxelization (the input of voxelize)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x4B495454]))
    o = np.array([0.0, 0.0, 1.73])
    el = np.deg2rad(np.linspace(-24.8, 2.0, beams))
    az = np.linspace(0, 2 * np.pi, n_azimuth, endpoint=False)
    E, A = np.meshgrid(el, az, indexing="ij")
    d = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1).reshape(-1, 3)
    t = np.where(d[:, 2] < 0, -o[2] / np.where(d[:, 2] < 0, d[:, 2], -1), np.inf)  # ground plane z = 0
    for _ in range(int(rng.integers(25, 40))):  # cars / buildings / walls
        c = rng.uniform(-60, 60, 2)
        if np.hypot(*c) < 4:
            continue
        size = rng.uniform([1.5, 1.5, 1.2], [12, 6, 6])
        t = np.minimum(t, _ray_box(o, d, np.array([c[0], c[1], 0]) - size * [0.5, 0.5, 0],
                                   np.array([c[0], c[1], 0]) + size * [0.5, 0.5, 1]))
    for _ in range(int(rng.integers(15, 30))):  # poles / trunks
        c = rng.uniform(-50, 50, 2)
        if np.hypot(*c) < 3:
            continue
        t = np.minimum(t, _ray_cylinder(o, d, c[0], c[1], rng.uniform(0.1, 0.6), rng.uniform(2, 8)))
    keep = t <= max_range
    p = o + d[keep] * t[keep, None]
    p += rng.normal(0, 0.01, p.shape)
    inten = rng.random((len(p), 1))
    feats = np.concatenate([p, inten], 1)
    if raw:
        return p, feats.astype(np.float32)
    return voxelize(p, feats, resolution)


def s3dis_room(seed: int = 0, n_points: int = 1_000_000, resolution: float = 0.025):
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x53334453]))
    L, W, H = 8.0, 6.0, 3.0
    quads = [  # (origin, u, v) for floor, ceiling, 4 walls
        ((0, 0, 0), (L, 0, 0), (0, W, 0)), ((0, 0, H), (L, 0, 0), (0, W, 0)),
        ((0, 0, 0), (L, 0, 0), (0, 0, H)), ((0, W, 0), (L, 0, 0), (0, 0, H)),
        ((0, 0, 0), (0, W, 0), (0, 0, H)), ((L, 0, 0), (0, W, 0), (0, 0, H)),
    ]
    for _ in range(int(rng.integers(10, 21))):  # furniture boxes: 5 visible faces
        lo = rng.uniform([0.2, 0.2, 0], [L - 1.5, W - 1.5, 0])
        sz = rng.uniform([0.4, 0.4, 0.4], [1.5, 1.5, 1.8])
        x, y, z = lo
        a, b, c = sz
        quads += [((x, y, z + c), (a, 0, 0), (0, b, 0)), ((x, y, z), (a, 0, 0), (0, 0, c)),
                  ((x, y + b, z), (a, 0, 0), (0, 0, c)), ((x, y, z), (0, b, 0), (0, 0, c)),
                  ((x + a, y, z), (0, b, 0), (0, 0, c))]
    areas = np.array([np.linalg.norm(np.cross(u, v)) for _, u, v in quads])
    counts = rng.multinomial(n_points, areas / areas.sum())
    pts, cols = [], []
    for (org, u, v), n in zip(quads, counts):
        st = rng.random((n, 2))
        pts.append(np.asarray(org) + st[:, :1] * np.asarray(u) + st[:, 1:] * np.asarray(v))
        cols.append(np.tile(rng.random(3), (n, 1)) + rng.normal(0, 0.02, (n, 3)))
    p = np.concatenate(pts)
    feats = np.concatenate([p, np.concatenate(cols)], 1)
    return voxelize(p, feats, resolution)


def shapenet_object(seed: int = 0, n_points: int = 120_000, grid: int = 128, channels: int = 32):
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x5348504E]))
    pts = []
    for _ in range(int(rng.integers(3, 7))):
        kind = rng.integers(0, 3)
        c = rng.uniform(0.25, 0.75, 3)
        n = n_points // 5
        if kind == 0:  # sphere
            v = rng.normal(size=(n, 3))
            pts.append(c + rng.uniform(0.08, 0.25) * v / np.linalg.norm(v, axis=1, keepdims=True))
        elif kind == 1:  # box surface
            s = rng.uniform(0.1, 0.4, 3)
            f = rng.integers(0, 3, n)
            q = rng.random((n, 3)) - 0.5
            q[np.arange(n), f] = np.where(rng.random(n) < 0.5, -0.5, 0.5)
            pts.append(c + q * s)
        else:  # cylinder side
            r, h = rng.uniform(0.05, 0.2), rng.uniform(0.1, 0.5)
            a = rng.uniform(0, 2 * np.pi, n)
            pts.append(c + np.stack([r * np.cos(a), r * np.sin(a), rng.uniform(-h / 2, h / 2, n)], 1))
    p = np.clip(np.concatenate(pts), 0, 1 - 1e-9) * grid
    feats = rng.random((len(p), channels))
    return voxelize(p, feats, 1.0)


def batch_clouds(clouds, spacing=256):
    """Several clouds as ONE sparse tensor (the usual batch-in-coordinates encoding): cloud b is
    shifted by b * spacing along x, so no kernel offset or stride floor can reach across clouds
    when spacing exceeds every cloud's x extent plus the network's reach and is a multiple of its
    largest tensor stride. Returns (coords sorted, feats, row ranges per cloud); sorting keeps the
    clouds contiguous and in order because x is the most significant key field.

    clouds: list of (coords int32 [n, 3], feats float32 [n, c])."""
    xs, fs, ranges, start = [], [], [], 0
    for b, (c, f) in enumerate(clouds):
        cc = c.astype(np.int64).copy()
        if len(c):
            # shift by a multiple of `spacing`: residues modulo every power-of-two stride <= spacing
            # are kept, so Eq. 1 floors group voxels exactly as in the unbatched cloud
            base = (int(c[:, 0].min()) // spacing) * spacing
            if int(c[:, 0].max()) - base >= spacing // 2:
                raise ValueError("cloud x extent too large for the batch spacing")
            cc[:, 0] += b * spacing - base
        order = np.lexsort((cc[:, 2], cc[:, 1], cc[:, 0]))
        xs.append(cc[order])
        fs.append(f[order])
        ranges.append((start, start + len(c)))
        start += len(c)
    coords = np.concatenate(xs).astype(np.int32) if xs else np.zeros((0, 3), np.int32)
    return coords, np.concatenate(fs).astype(np.float32), ranges

