#!/usr/bin/env python3
"""Host vs device time of one network forward: if the host enqueue time approaches the device
time the forward is host-bound (GPU idles between launches)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2401_06145_b200 as sc
import bench
from paper_2401_06145_b200 import network as N
ctx = sc.Context(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
g = bench.graph("c2_minkunet42_kitti")
net = N.Network(ctx, g, N.init_weights(g, 1), sc.exec_cfg(dataflow=sc.DATAFLOW_AUTO))
coords, feats = bench.scene("c2_minkunet42_kitti", 0)
x, f = torch.from_numpy(coords).cuda(), torch.from_numpy(feats).cuda()
fwd = lambda: net.forward(device_xyz=x.data_ptr(), device_feats=f.data_ptr(), n=len(coords), sorted_=True)
for _ in range(3): fwd()
torch.cuda.synchronize()
host, dev = [], []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); a.record(); fwd(); t1 = time.perf_counter(); b.record(); b.synchronize()
    host.append((t1 - t0) * 1e3); dev.append(a.elapsed_time(b))
print(f"host enqueue {np.median(host):.3f} ms, device (events) {np.median(dev):.3f} ms")
ctx.set_profiling(True)
fwd(); torch.cuda.synchronize()
tot = sum(ms for _, ms in ctx.profile().values())
print(f"sum of per-kernel event times {tot:.3f} ms over {sum(n for n, _ in ctx.profile().values())} launches")
