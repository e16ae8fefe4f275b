#!/usr/bin/env python3
"""Steady-state network forwards for clean ncu captures (fixed dataflow, no AUTO tuning).

  ncu --set full -k regex:k_conv_fused -s 1 -c 1 python profiles/run_net.py --dataflow fused --steps 1
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2401_06145_b200 as sc  # noqa: E402
import bench  # noqa: E402
from paper_2401_06145_b200 import network as N  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--workload", default="c2_minkunet42_kitti")
p.add_argument("--dataflow", default="fused", choices=["fused", "gmas", "auto"])
p.add_argument("--steps", type=int, default=1)
p.add_argument("--time", action="store_true", help="print per-kernel event times")
p.add_argument("--profile-last", action="store_true",
               help="cudaProfilerStart/Stop around the last forward (ncu --profile-from-start off)")
a = p.parse_args()
df = {"fused": sc.DATAFLOW_FUSED, "gmas": sc.DATAFLOW_GMAS, "auto": sc.DATAFLOW_AUTO}[a.dataflow]
ctx = sc.Context(0)
g = bench.graph(a.workload)
net = N.Network(ctx, g, N.init_weights(g, 1), sc.exec_cfg(dataflow=df))
coords, feats = bench.scene(a.workload, 0)
xyz_d, f_d = torch.from_numpy(coords).cuda(), torch.from_numpy(feats).cuda()
_stream = torch.cuda.Stream()  # a real stream: the legacy default (handle 0) would not order with the library's
torch.cuda.set_stream(_stream)
ctx.set_stream(_stream.cuda_stream)
if a.time:
    ctx.set_profiling(True)
for step in range(a.steps):
    last = step == a.steps - 1
    if a.profile_last and last:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    net.forward(device_xyz=xyz_d.data_ptr(), device_feats=f_d.data_ptr(), n=len(coords), sorted_=True)
    if a.profile_last and last:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
torch.cuda.synchronize()
if a.time:
    for k, (n, ms) in sorted(ctx.profile().items(), key=lambda kv: -kv[1][1]):
        print(f"{k:24s} {n / a.steps:6.1f} launches/step {1e3 * ms / a.steps:9.1f} us/step")
