#!/usr/bin/env python3
"""Eq. 1 output coordinates (one-launch floor / sort / unique, k_floor_unique*) alone: GPU kernel
duration from CUPTI (torch.profiler; CUDA events around a lone launch would also count the
host's launch latency) of a stride-2 map build over the KITTI scan, the S3DIS room and the C4
object batch, median of 5 after 1 warm-up, for A/B runs (SCONV_FLOOR_CLUSTER, SCONV_COOP_E)."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D
from paper_2401_06145_b200 import workloads as WL

ctx = sc.Context(0)
c4 = WL.scenes("c4_unet_pair_shapenet")[0][0]
clouds = {"kitti": D.kitti_scan(0)[0], "s3dis": D.s3dis_room(0)[0], "c4": c4}
if len(sys.argv) > 1 and sys.argv[1] == "sizes":  # prefixes of the sorted KITTI scan
    k = D.kitti_scan(0)[0]
    k = k[np.lexsort((k[:, 2], k[:, 1], k[:, 0]))]
    clouds = {f"kitti[:{m}]": k[:m] for m in (4000, 12000, 25000, 50000, 80000, 118964)}
out = []
for name, xyz in clouds.items():
    xyz = xyz[np.lexsort((xyz[:, 2], xyz[:, 1], xyz[:, 0]))]
    m = sc.KernelMap.build(ctx, xyz, True, 2, 1, 2)
    m.free()
    ctx.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for r in range(5):
            m = sc.KernelMap.build(ctx, xyz, True, 2, 1, 2)
            m.free()
        ctx.synchronize()
    ts = [e.time_range.end - e.time_range.start for e in prof.events()
          if e.device_type == torch.autograd.DeviceType.CUDA and "k_floor" in e.name]
    out.append(f"{name}({len(xyz)}) {statistics.median(ts) if ts else float('nan'):6.1f} us")
print(f"[coop_e={os.environ.get('SCONV_COOP_E', '1')}] " + "  ".join(out))
