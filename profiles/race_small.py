#!/usr/bin/env python3
"""One small fused conv (tile-queue kernel) for a detailed compute-sanitizer racecheck report."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2401_06145_b200 as sc  # noqa: E402

ctx = sc.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
c = int(sys.argv[2]) if len(sys.argv) > 2 else 32
xyz, F = sc.generate_synthetic(n, 16, c, 3)
W = sc.generate_weights(3, 1, 27, c, c)
m = sc.KernelMap.build(ctx, xyz, False, 3, 1, 1)
out = sc.layer_forward(ctx, m, sc.Weights(ctx, W), F, sc.exec_cfg(dataflow=sc.DATAFLOW_FUSED))
print("ok", float(np.abs(out).sum()))
ctx.close()
