#!/usr/bin/env python3
"""Steady-state C1 layer loop for clean ncu captures (no autotuning launches).

  ncu --set full -k regex:"k_search|k_scatter" -s 20 -c 4 python profiles/run_layer.py --steps 4
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_06145_b200 as sc  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=4)
p.add_argument("--n", type=int, default=100000)
p.add_argument("--extent", type=int, default=400)
p.add_argument("--c", type=int, default=32)
p.add_argument("--tg", type=int, default=8)
p.add_argument("--ts", type=int, default=16)
p.add_argument("--B", type=int, default=256)
p.add_argument("--C", type=int, default=512)
p.add_argument("--time", action="store_true", help="print per-kernel event times")
a = p.parse_args()
ctx = sc.Context(0)
xyz, F = sc.generate_synthetic(a.n, a.extent, a.c, 1)
W = sc.generate_weights(1, 1, 27, a.c, a.c)
w = sc.Weights(ctx, W)
xyz_d = torch.from_numpy(xyz).cuda()
F_d = torch.from_numpy(F).cuda()
out = torch.empty((a.n, a.c), device="cuda")
torch.cuda.synchronize()
cfg = sc.exec_cfg(gather_tile=a.tg, scatter_tile=a.ts)
def step():
    m = sc.KernelMap.build(ctx, None, False, 3, 1, 1, device_ptr=xyz_d.data_ptr(), n=a.n, B=a.B, Cq=a.C)
    sc.layer_forward_device(ctx, m, w, F_d.data_ptr(), sc.F32, out.data_ptr(), sc.F32, cfg)
    m.free()


for _ in range(2):
    step()
ctx.synchronize()
if a.time:
    ctx.set_profiling(True)
    ctx.profile_reset()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
_stream = torch.cuda.Stream()  # a real stream: the legacy default (handle 0) would not order with the library's
torch.cuda.set_stream(_stream)
ctx.set_stream(_stream.cuda_stream)
ev0.record()
for _ in range(a.steps):
    step()
ev1.record()
ctx.synchronize()
torch.cuda.synchronize()
print(f"B={a.B} C={a.C} n={a.n}: {ev0.elapsed_time(ev1) / a.steps * 1e3:.1f} us/step")
if a.time:
    for k, (n, ms) in sorted(ctx.profile().items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:28s} {ms / n * 1e3:8.2f} us x {n // a.steps}")
