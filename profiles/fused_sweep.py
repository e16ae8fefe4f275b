#!/usr/bin/env python3
"""Fused vs GMaS layer latency sweep on synthetic clouds (device-resident, CUDA events,
median of 10 after warm-up). Separates per-tile fixed costs from per-row/per-offset costs.

  python profiles/fused_sweep.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_06145_b200 as sc  # noqa: E402
from paper_2401_06145_b200 import datasets as D  # noqa: E402

ctx = sc.Context(0)
_stream = torch.cuda.Stream()  # a real stream: the legacy default (handle 0) would not order with the library's
torch.cuda.set_stream(_stream)
ctx.set_stream(_stream.cuda_stream)


def timed(fn, reps=10):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    fn()
    fn()
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


coords, _ = D.kitti_scan(0)
rows = []
for K in (1, 3):
    for n in (16000, 60000, len(coords)):
        xyz = coords[:n] if K == 1 else coords[:n]
        m = sc.KernelMap.build(ctx, xyz, True, K, 1, 1)
        info = m.info()
        for cin, cout in ((32, 32), (96, 96), (256, 256)):
            W = sc.generate_weights(1, 1, K ** 3, cin, cout)
            w = sc.Weights(ctx, W)
            x = torch.rand((n, cin), device="cuda").half()
            y = torch.empty((n, cout), device="cuda", dtype=torch.half)
            res = {}
            for name, df in (("gmas", sc.DATAFLOW_GMAS), ("fused", sc.DATAFLOW_FUSED)):
                cfg = sc.exec_cfg(dataflow=df)
                res[name] = timed(lambda: sc.layer_forward_device(ctx, m, w, x.data_ptr(), sc.F16, y.data_ptr(),
                                                                  sc.F16, cfg))
            useful = info.total_matches * cin * 2
            print(f"K={K} n={n:6d} |M|={info.total_matches:7d} {cin:3d}->{cout:3d}  gmas {res['gmas']:7.1f} us"
                  f"  fused {res['fused']:7.1f} us  fused useful-gather {useful / res['fused'] / 1e3:6.0f} GB/s",
                  flush=True)
        m.free()
