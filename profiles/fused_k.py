#!/usr/bin/env python3
"""The fused kernel on the KITTI level-0 coordinates for a given kernel size K (1 = identity
map, 2, 3): device time per launch (CUDA events, median of 20 x 4 launches) per channel width.

  python profiles/fused_k.py K [channels ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_06145_b200 as sc  # noqa: E402
from paper_2401_06145_b200 import datasets as D  # noqa: E402

K = int(sys.argv[1])
chans = [int(x) for x in (sys.argv[2:] or ["32", "96", "256"])]
ctx = sc.Context(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
coords, _ = D.kitti_scan(0)
m = sc.KernelMap.build(ctx, coords, True, K, 1, 1)
M = m.info().total_matches
for c in chans:
    w = sc.Weights(ctx, sc.generate_weights(1, 1, K ** 3, c, c))
    x = torch.rand((len(coords), c), device="cuda").half()
    y = torch.empty_like(x)
    cfg = sc.exec_cfg(dataflow=sc.DATAFLOW_FUSED)
    f = lambda: sc.layer_forward_device(ctx, m, w, x.data_ptr(), sc.F16, y.data_ptr(), sc.F16, cfg)  # noqa: E731
    for _ in range(3):
        f()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f(); f(); f(); f()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 4 * 1e3)
    print(f"K={K} c={c:3d} n={len(coords)} |M|={M} fused {float(np.median(ts)):7.1f} us", flush=True)
