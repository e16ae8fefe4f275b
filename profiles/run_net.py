#!/usr/bin/env python3
"""Run a network workload's forward a few times with a fixed dataflow (for ncu captures:
the AUTO tuner's trial launches would otherwise interleave with the measured ones).

  python profiles/run_net.py [workload] [--forwards 2] [--dataflow fused|gmas|auto]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2401_06145_b200 as sc  # noqa: E402
from paper_2401_06145_b200 import network as N  # noqa: E402
from paper_2401_06145_b200 import workloads as WL  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("workload", nargs="?", default="c2_minkunet42_kitti")
p.add_argument("--forwards", type=int, default=2)
p.add_argument("--dataflow", default="fused")
a = p.parse_args()
df = {"fused": sc.DATAFLOW_FUSED, "gmas": sc.DATAFLOW_GMAS, "auto": sc.DATAFLOW_AUTO}[a.dataflow]
ctx = sc.Context(0)
g = WL.graph(a.workload)
coords, feats = WL.scenes(a.workload)[0]
net = N.Network(ctx, g, N.init_weights(g, WL.WEIGHT_SEED), sc.exec_cfg(dataflow=df))
for _ in range(a.forwards):
    net.forward(coords, feats, True)
ctx.synchronize()
print("convs", len(net.conv_stats()))
