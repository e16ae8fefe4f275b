#!/usr/bin/env python3
"""Debug helper: run a network twice (env A vs env B set by the caller through two processes is
awkward, so this runs FUSED and GMaS, unfolded) and report the first tensor that differs."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D, network as N
ctx = sc.Context(0)
coords, feats = D.kitti_scan(3, n_azimuth=400)
g = N.minkunet42(); w = N.init_weights(g, 7)
nets = {}
for name, df in (("gmas", sc.DATAFLOW_GMAS), ("fused", sc.DATAFLOW_FUSED)):
    net = N.Network(ctx, g, w, sc.exec_cfg(dataflow=df, fuse_residual=0, partial_f16=0))
    net.forward(coords, feats, True)
    nets[name] = net
for i, o in enumerate(g.ops):
    a = nets["gmas"].read(o.out)[1]; b = nets["fused"].read(o.out)[1]
    err = np.abs(a - b).max() / max(np.abs(a).max(), 1e-30)
    tag = "" if err < 1e-2 else "   <-- DIFF"
    print(f"op {i:2d} kind={o.kind} K={o.K} s={o.out_stride} T={o.transposed} {o.c_in}->{o.c_out} n={a.shape[0]} rel={err:.2e}{tag}")
