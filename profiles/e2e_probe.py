#!/usr/bin/env python3
"""Where the end-to-end (host-buffer) step of a network workload spends its time.

Host-clock per-step times of back-to-back loops (no L2 flush): device inputs; host inputs
without a readback; host inputs + synchronous readback; host inputs + pipelined
sconv_net_read_async; the readback alone; the host time spent inside forward(). Then a
CUPTI trace (torch.profiler) of 3 pipelined steps: copies, the compute stream's idle gaps and
what follows them.

  python profiles/e2e_probe.py [workload]
"""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2401_06145_b200 as sc  # noqa: E402
from paper_2401_06145_b200 import network as N  # noqa: E402
from paper_2401_06145_b200 import workloads as WL  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_minkunet42_kitti"
ctx = sc.Context(0)
g = WL.graph(name)
coords, feats = WL.scenes(name)[0]
net = N.Network(ctx, g, N.init_weights(g, WL.WEIGHT_SEED), sc.exec_cfg(compute_dtype=sc.F16))
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
c_h, f_h = pin(coords), pin(feats)
xyz, f = torch.from_numpy(coords).cuda(), torch.from_numpy(feats).cuda()
net.forward(c_h, f_h, True)
n, ch, _ = net.info(g.output)
outs = [torch.empty((n, ch), dtype=torch.float32, pin_memory=True).numpy() for _ in range(2)]
host_in_fwd = []


def fwd_dev():
    net.forward(device_xyz=xyz.data_ptr(), device_feats=f.data_ptr(), n=xyz.shape[0], sorted_=True)


def fwd_host():
    t = time.perf_counter()
    net.forward(c_h, f_h, True)
    host_in_fwd.append(time.perf_counter() - t)


def seq_read():
    fwd_host()
    net.read(g.output, feats_out=outs[0], coords=False)


state = {"i": 0}


def piped():
    i = state["i"]
    fwd_host()
    if i:
        net.wait_reads()
    net.read_async(g.output, outs[i & 1])
    state["i"] += 1


def read_only():
    net.read(g.output, feats_out=outs[0], coords=False)


def timed(fn, k=20, tail=None):
    for _ in range(3):
        fn()
    (tail or (lambda: None))()
    ctx.synchronize()
    torch.cuda.synchronize()
    host_in_fwd.clear()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    (tail or (lambda: None))()
    ctx.synchronize()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / k


res = {"device inputs": timed(fwd_dev), "host inputs, no readback": timed(fwd_host)}
res["host in forward() (ms, host inputs)"] = 1e3 * sum(host_in_fwd) / max(1, len(host_in_fwd))
res["host inputs + sync readback"] = timed(seq_read)
res["host inputs + read_async pipelined"] = timed(piped, tail=net.wait_reads)
res["host in forward() (ms, pipelined)"] = 1e3 * sum(host_in_fwd) / max(1, len(host_in_fwd))
res["readback alone (%d bytes)" % outs[0].nbytes] = timed(read_only)
for k, v in res.items():
    print(f"{k:45s} {v:8.3f} ms")

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], acc_events=True) as prof:
    for _ in range(3):
        piped()
    net.wait_reads()
    torch.cuda.synchronize()
with tempfile.NamedTemporaryFile(suffix=".json") as tf:
    prof.export_chrome_trace(tf.name)
    trace = json.load(open(tf.name))["traceEvents"]
ev = sorted(({"name": e["name"][:60], "t0": e["ts"], "t1": e["ts"] + e.get("dur", 0),
              "stream": e.get("args", {}).get("stream", e.get("tid", 0)), "cat": e.get("cat")}
             for e in trace if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")), key=lambda e: e["t0"])
host = sorted((e for e in trace if e.get("cat") == "cuda_runtime" and e.get("dur", 0) > 50),
              key=lambda e: e["ts"])
t00 = ev[0]["t0"]
print("copies:")
for e in ev:
    if e["cat"] == "gpu_memcpy" and e["t1"] - e["t0"] > 20:
        print(f"  {e['t0'] - t00:9.1f} {e['t1'] - t00:9.1f} stream {e['stream']} {e['name']}")
conv = [e for e in ev if "k_conv" in e["name"]]
cs = collections_stream = max(set(e["stream"] for e in conv), key=lambda s: sum(1 for e in conv if e["stream"] == s))
on = [e for e in ev if e["stream"] == cs]
print(f"compute stream {cs}: gaps > 30 us")
for a, b in zip(on, on[1:]):
    if b["t0"] - a["t1"] > 30:
        print(f"  gap {b['t0'] - a['t1']:7.1f} us at {a['t1'] - t00:9.1f} before {b['name']}")
print("host runtime calls > 50 us:")
for e in host:
    print(f"  {e['ts'] - t00:9.1f} dur {e['dur']:8.1f} {e['name']}")
