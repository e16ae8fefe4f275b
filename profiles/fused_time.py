#!/usr/bin/env python3
"""Time the fused kernel on one KITTI-shaped submanifold layer (K=3) per channel width:
device time from CUDA events on a dedicated stream, median of 20 after warm-up."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2401_06145_b200 as sc
from paper_2401_06145_b200 import datasets as D
ctx = sc.Context(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
coords, _ = D.kitti_scan(0)
m = sc.KernelMap.build(ctx, coords, True, 3, 1, 1)
M = m.info().total_matches
for c in [int(x) for x in (sys.argv[1:] or ["32", "96", "256"])]:
    w = sc.Weights(ctx, sc.generate_weights(1, 1, 27, c, c))
    x = torch.rand((len(coords), c), device="cuda").half(); y = torch.empty_like(x)
    cfg = sc.exec_cfg(dataflow=sc.DATAFLOW_FUSED)
    f = lambda: sc.layer_forward_device(ctx, m, w, x.data_ptr(), sc.F16, y.data_ptr(), sc.F16, cfg)
    for _ in range(3): f()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); f(); f(); f(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) / 4 * 1e3)
    t = float(np.median(ts))
    print(f"c={c:3d} n={len(coords)} |M|={M} fused {t:7.1f} us  useful gather {M * c * 2 / t / 1e3:6.0f} GB/s", flush=True)
