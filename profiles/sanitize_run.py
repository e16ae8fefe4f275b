#!/usr/bin/env python3
"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): unsorted-input map (bucket sort + k_search), a strided map (the
cooperative k_floor_unique), the fused row order (cooperative k_mask_sort), the fused
kernels (tile-queue and work-item variants), GMaS (gather, grouped tcgen05 GEMM, scatter),
the hash backend and a small MinkUNet42 forward.

  compute-sanitizer --tool racecheck python profiles/sanitize_run.py [--net]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2401_06145_b200 as sc  # noqa: E402
from paper_2401_06145_b200 import network as N  # noqa: E402
from paper_2401_06145_b200 import datasets as D  # noqa: E402
from paper_2401_06145_b200 import graphs as G  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=3000)
p.add_argument("--net", action="store_true")
a = p.parse_args()
ctx = sc.Context(0)
xyz, F = sc.generate_synthetic(a.n, 20, 32, 3)
for c in (32, 96):
    W = sc.generate_weights(3, 1, 27, 32, c)
    w = sc.Weights(ctx, W)
    m = sc.KernelMap.build(ctx, xyz, False, 3, 1, 1)
    for df in (sc.DATAFLOW_GMAS, sc.DATAFLOW_FUSED):
        out = sc.layer_forward(ctx, m, w, F, sc.exec_cfg(dataflow=df))
        assert np.isfinite(out).all()
    m.free()
ms = sc.KernelMap.build(ctx, xyz, False, 2, 1, 2)  # strided K=2 s=2
ms.read()
mh = sc.KernelMap.build(ctx, xyz, False, 3, 1, 1, backend=sc.MAP_HASH)
mh.read()
# column search on chunks with scattered targets (skip-ahead slices + the direct global path):
# a sparse slice between two dense wall planes (tests/test_gpu_parity.py::test_map_scattered_chunks)
yy, zz = np.meshgrid(np.arange(200), np.arange(64), indexing="ij")
wall = lambda x: np.stack([np.full(yy.size, x), yy.ravel(), zz.ravel()], 1)  # noqa: E731
rg = np.random.default_rng(214)
mid = np.stack([np.ones(128, np.int64), np.sort(rg.choice(200, 128, replace=False)), rg.integers(0, 64, 128)], 1)
walls = np.concatenate([wall(0), mid, wall(2)]).astype(np.int32)
walls = walls[np.lexsort((walls[:, 2], walls[:, 1], walls[:, 0]))]
sc.KernelMap.build(ctx, walls, True, 3, 1, 1).read()
ctx.synchronize()
if a.net:
    coords, feats = D.kitti_scan(0, n_azimuth=120)
    g = G.minkunet42(feats.shape[1])
    net = N.Network(ctx, g, N.init_weights(g, 5), sc.exec_cfg(dataflow=sc.DATAFLOW_FUSED))
    net.forward(coords, feats, True)
    net.forward(coords, feats, True)
    # serving loop: host inputs staged on the net's input stream, results read back
    # asynchronously while the next forward runs (two staging slots each, so both are reused)
    import torch
    scans = [D.kitti_scan(s, n_azimuth=120) for s in (1, 2, 3)]
    outs = []
    for i, (c, f) in enumerate(scans + scans):
        net.forward(c, f, True)
        n, ch, _ = net.info(g.output)
        outs.append(torch.empty((n, ch), dtype=torch.float32, pin_memory=True).numpy())
        if i:
            net.wait_reads()
        net.read_async(g.output, outs[-1])
    net.wait_reads()
    for i in range(3):
        assert np.array_equal(outs[i], outs[i + 3]), "serving loop results differ between rounds"
    net.free()
    ctx.synchronize()
ctx.close()
print("sanitize run ok")
