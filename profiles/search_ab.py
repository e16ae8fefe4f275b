#!/usr/bin/env python3
"""Search-stage time (k_search, CUDA events, median of 5 after 1 warm-up) of the sorted Map on
the KITTI / S3DIS level-0 clouds and a uniform 1e6 cloud: for A/B runs of the search kernels
(SCONV_SEARCH_PERSIST, SCONV_SEARCH_CPC)."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D

ctx = sc.Context(0)
rng = np.random.default_rng(0)
flat = rng.choice(150 ** 3, size=1_000_000, replace=False)
clouds = {"kitti": (D.kitti_scan(0)[0], True), "s3dis": (D.s3dis_room(0)[0], True),
          "u1e6": (np.stack(np.unravel_index(flat, (150,) * 3), 1).astype(np.int32), False)}
only = sys.argv[1:]  # optional cloud names
out = []
for name, (xyz, srt) in clouds.items():
    if only and name not in only:
        continue
    ts = []
    for r in range(6):
        ctx.set_profiling(True)
        ctx.profile_reset()
        m = sc.KernelMap.build(ctx, xyz, srt, 3, 1, 1)
        prof = ctx.profile()
        ctx.set_profiling(False)
        ts.append(prof["k_search"][1])
        m.free()
    out.append(f"{name} {1e3 * statistics.median(ts[1:]):7.1f} us")
print(f"[persist={os.environ.get('SCONV_SEARCH_PERSIST', '1')} cpc={os.environ.get('SCONV_SEARCH_CPC', '0')}] " + "  ".join(out))
