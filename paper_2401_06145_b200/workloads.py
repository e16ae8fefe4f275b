"""The BASELINE.json configurations as concrete inputs (pure Python + numpy; no engine import).

One definition serves bench.py's GPU arm, its CPU reference arm and the full-size parity
tests, so all three see bit-identical scenes, graphs and weights:

  c1_layer_100k          configs[0]  one submanifold 3^3 layer, 32->32, 100k voxels in 400^3
  c2_minkunet42_kitti    configs[1]  MinkUNet42 on one KITTI-shaped scan (scene 0, ~119k voxels)
  c3_resnet21d_s3dis     configs[2]  SparseResNet21D (width x2) on an S3DIS-shaped room (~337k)
  c4_unet_pair_shapenet  configs[3]  K=2 s=2 down + transposed pair on 8 ShapeNet-shaped
                                     objects batched in the coordinates (one sparse tensor)
  c5_minkunet42_batch64  configs[4]  MinkUNet42 on 64 KITTI-shaped scans (scenes 0..63),
                                     scene-sharded: rank r of G runs shard_range(64, G, r)

Weights: graphs.init_weights(g, WEIGHT_SEED, generate) with the SPEC PRNG (the engine's and
the oracle's generators give the same bits).
"""
from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

if __package__:
    from . import datasets as D
    from . import graphs as G
else:  # loaded by path (CPU reference arm): sibling modules by path as well
    import importlib.util
    import sys

    def _sibling(name):
        key = f"_sconv_pure_{name}"
        if key not in sys.modules:
            spec = importlib.util.spec_from_file_location(key, os.path.join(os.path.dirname(__file__), f"{name}.py"))
            mod = importlib.util.module_from_spec(spec)
            sys.modules[key] = mod
            spec.loader.exec_module(mod)
        return sys.modules[key]

    D, G = _sibling("datasets"), _sibling("graphs")

NETWORKS = {
    "c2_minkunet42_kitti": ("MinkUNet42", G.minkunet42),
    "c3_resnet21d_s3dis": ("SparseResNet21D-w2", G.sparse_resnet21d),
    "c4_unet_pair_shapenet": ("UNetPair(K2s2 down+transposed)", G.unet_pair),
    "c5_minkunet42_batch64": ("MinkUNet42", G.minkunet42),
}
WORKLOADS = ["c2_minkunet42_kitti", "c1_layer_100k", "c3_resnet21d_s3dis", "c4_unet_pair_shapenet",
             "c5_minkunet42_batch64"]
WEIGHT_SEED = 1
C4_OBJECTS = 8
C5_SCENES = 64


def shard_range(n_units: int, rank: int, world: int):
    """Contiguous [start, end) of ``n_units`` for ``rank``; the first n_units % world ranks
    take one extra unit (64 scenes over 8 GPUs -> 8 each)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    if n_units < 0:
        raise ValueError("unit count must be nonnegative")
    base, extra = divmod(n_units, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def graph(name: str):
    return NETWORKS[name][1]()


def _kitti(i):
    return D.kitti_scan(i)


def scenes(name: str, world: int = 1, rank: int = 0):
    """This rank's inputs for one step: a list of (coords int32 [n,3] sorted, feats f32)."""
    if name == "c2_minkunet42_kitti":
        return [D.kitti_scan(0)]
    if name == "c3_resnet21d_s3dis":
        return [D.s3dis_room(0, n_points=870_000)]
    if name == "c4_unet_pair_shapenet":
        c, f, _ = D.batch_clouds([D.shapenet_object(i) for i in range(C4_OBJECTS)])
        return [(c, f)]
    if name == "c5_minkunet42_batch64":
        lo, hi = shard_range(C5_SCENES, rank, world)
        ids = list(range(lo, hi))
        workers = min(len(ids), os.cpu_count() or 1, 16)
        if workers <= 1:
            return [D.kitti_scan(i) for i in ids]
        with ProcessPoolExecutor(workers) as ex:
            return list(ex.map(_kitti, ids))
    raise ValueError(name)


def kitti_scene(i: int):
    """Scene i of the 64-scan C5 batch (scene 0 is the C2 scan)."""
    return D.kitti_scan(i)


def total_points(clouds) -> int:
    return int(sum(len(c) for c, _ in clouds))


__all__ = ["NETWORKS", "WORKLOADS", "WEIGHT_SEED", "C4_OBJECTS", "C5_SCENES", "shard_range", "graph", "scenes",
           "kitti_scene", "total_points", "np"]
