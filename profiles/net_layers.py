#!/usr/bin/env python3
"""Per-conv breakdown of a network forward: shape, |M|, and the AUTO tuner's GMaS vs fused
times (CUDA events, warm L2, min of 2 after a warm-up). Used to pick what to optimise.

  python profiles/net_layers.py --workload c2_minkunet42_kitti [--json out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402,F401

import paper_2401_06145_b200 as sc  # noqa: E402
import bench  # noqa: E402
from paper_2401_06145_b200 import network as N  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--workload", default="c2_minkunet42_kitti")
p.add_argument("--json", default=None)
a = p.parse_args()
ctx = sc.Context(0)
g = bench.graph(a.workload)
w = N.init_weights(g, 1)
coords, feats = bench.scene(a.workload, 0)
net = N.Network(ctx, g, w, sc.exec_cfg(dataflow=sc.DATAFLOW_AUTO))
net.forward(coords, feats, True)
st = net.conv_stats()
tm = net.auto_timings()
rows = []
tot = [0.0, 0.0, 0.0]
conv_ops = [i for i, o in enumerate(g.ops) if o.kind == N.CONV]
print(f"{'op':>3} {'K3':>3} {'n_in':>7} {'n_out':>7} {'|M|':>8} {'cin':>4} {'cout':>4} {'gmas_us':>8} {'fused_us':>8} {'res':>3}")
for s, i in zip(st, conv_ops):
    gm, fu = tm[i]
    tot[0] += gm
    tot[1] += fu
    tot[2] += min(gm, fu)
    rows.append(dict(op=i, **s, gmas_ms=gm, fused_ms=fu))
    print(f"{i:>3} {s['K3']:>3} {s['n_in']:>7} {s['n_out']:>7} {s['M']:>8} {s['c_in']:>4} {s['c_out']:>4} "
          f"{1e3 * gm:>8.1f} {1e3 * fu:>8.1f} {s['residual']:>3}")
print(f"total: gmas {tot[0]:.3f} ms, fused {tot[1]:.3f} ms, best-of {tot[2]:.3f} ms")
if a.json:
    with open(a.json, "w") as f:
        json.dump({"workload": a.workload, "convs": rows, "total_ms": tot}, f, indent=1)
