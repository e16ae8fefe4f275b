#!/usr/bin/env python3
"""GPU voxelize (sconv_voxelize, host buffers in and out) vs the reference's own voxelize
(oracle/_ref: geometry.hpp compiled from the reference headers, one CPU thread) on a raw
KITTI-shaped LiDAR sweep at 5 cm. Checks the outputs are identical."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D
from oracle_lib import load_oracle, load_ref_oracle
ctx = sc.Context(0)
pts, f = D.kitti_scan(0, raw=True)
ref = load_ref_oracle() or load_oracle()
for _ in range(3):
    g = sc.voxelize(ctx, pts, f, 0.05)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); g = sc.voxelize(ctx, pts, f, 0.05); ts.append(time.perf_counter() - t0)
t0 = time.perf_counter(); xyz, of = ref.voxelize(pts, f, 0.05); tr = time.perf_counter() - t0
same = np.array_equal(g.coords, xyz) and np.array_equal(g.features, of)
print(f"points={len(pts)} voxels={len(xyz)} gpu(api, host buffers)={1e3 * np.median(ts):.2f} ms "
      f"reference cpu={1e3 * tr:.1f} ms identical={same}")
