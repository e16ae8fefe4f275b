#!/usr/bin/env python3
"""Kernel timeline of steady-state network forwards (CUPTI through torch.profiler; nsys is not
in the image). Per forward: span, per-stream busy time, the idle gaps of the stream that runs
the convs (the critical path) and what the longest gaps wait for.

  python profiles/timeline.py [workload] [--forwards 3] [--json out.json]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2401_06145_b200 as sc  # noqa: E402
from paper_2401_06145_b200 import network as N  # noqa: E402
from paper_2401_06145_b200 import workloads as WL  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("workload", nargs="?", default="c2_minkunet42_kitti")
p.add_argument("--forwards", type=int, default=3)
p.add_argument("--json", default=None)
p.add_argument("--dataflow", default="auto")
a = p.parse_args()
ctx = sc.Context(0)
g = WL.graph(a.workload)
(coords, feats) = WL.scenes(a.workload)[0]
df = {"fused": sc.DATAFLOW_FUSED, "gmas": sc.DATAFLOW_GMAS, "auto": sc.DATAFLOW_AUTO}[a.dataflow]
net = N.Network(ctx, g, N.init_weights(g, WL.WEIGHT_SEED), sc.exec_cfg(dataflow=df))
xyz = torch.from_numpy(coords).cuda()
f = torch.from_numpy(feats).cuda()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)


def fwd():
    net.forward(device_xyz=xyz.data_ptr(), device_feats=f.data_ptr(), n=xyz.shape[0], sorted_=True)


for _ in range(3):
    fwd()
ctx.synchronize()
torch.cuda.synchronize()
marks = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], acc_events=True) as prof:
    for _ in range(a.forwards):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fwd()
        e1.record(st)
        marks.append((e0, e1))
        ctx.synchronize()
    torch.cuda.synchronize()
# kernels with their host launch time: the chrome trace links each kernel to its runtime /
# driver launch call by correlation id (same time base)
import tempfile  # noqa: E402
with tempfile.NamedTemporaryFile(suffix=".json") as tf:
    prof.export_chrome_trace(tf.name)
    trace = json.load(open(tf.name))["traceEvents"]
api = {}
for e in trace:
    if e.get("cat") in ("cuda_runtime", "cuda_driver") and "correlation" in e.get("args", {}):
        api[e["args"]["correlation"]] = e["ts"]
kern = []
for e in trace:
    if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"):
        c = e.get("args", {}).get("correlation")
        kern.append({"name": e["name"], "start": e["ts"], "end": e["ts"] + e.get("dur", 0),
                     "stream": e.get("args", {}).get("stream", e.get("tid", 0)), "launch": api.get(c)})
kern.sort(key=lambda k: k["start"])
# split into forwards: the first kernel of each forward is k_convert_rows or the first map kernel; use gaps > 200 us
fw, cur = [], []
for k in kern:  # every forward starts by converting its input features (k_convert_rows)
    if cur and "k_convert_rows" in k["name"]:
        fw.append(cur)
        cur = []
    cur.append(k)
if cur:
    fw.append(cur)
out = []
for i, f_ in enumerate(fw):
    t0 = min(k["start"] for k in f_)
    t1 = max(k["end"] for k in f_)
    by = collections.defaultdict(list)
    for k in f_:
        by[k["stream"]].append(k)
    conv_stream = max(by, key=lambda s: sum(("conv" in k["name"] or "gemm" in k["name"]) for k in by[s]))
    cs = sorted(by[conv_stream], key=lambda k: k["start"])
    gaps = []
    prev = t0
    for k in cs:
        if k["start"] - prev > 0:
            gaps.append((k["start"] - prev, k["name"].replace("(anonymous namespace)::", "").replace("sconvb::", "")[:50],
                         prev - t0))
        prev = max(prev, k["end"])
    busy = {s: sum(k["end"] - k["start"] for k in ks) for s, ks in by.items()}
    names = collections.defaultdict(float)
    for k in cs:
        names[k["name"].replace("(anonymous namespace)::", "").replace("sconvb::", "").split("(")[0][-40:]] += k["end"] - k["start"]
    alln = collections.defaultdict(lambda: [0, 0.0])
    for k in f_:
        nm = k["name"].replace("(anonymous namespace)::", "").replace("sconvb::", "").split("(")[0][-40:]
        alln[nm][0] += 1
        alln[nm][1] += k["end"] - k["start"]
    rec = {"forward": i, "all_kernels": {n: {"launches": c, "us": round(t, 1)} for n, (c, t) in
                                         sorted(alln.items(), key=lambda kv: -kv[1][1])}, "span_us": t1 - t0, "launches": len(f_), "conv_stream": conv_stream,
           "busy_us": {str(s): v for s, v in busy.items()},
           "conv_stream_idle_us": sum(g_[0] for g_ in gaps), "conv_stream_gaps": len(gaps),
           "top_gaps": [{"us": round(g_[0], 1), "before": g_[1], "at_us": round(g_[2], 1)}
                        for g_ in sorted(gaps, reverse=True)[:12]],
           "conv_stream_kernels_us": dict(sorted(names.items(), key=lambda kv: -kv[1]))}
    rec["first_kernels"] = [{"t0": round(k["start"] - t0, 1), "t1": round(k["end"] - t0, 1), "stream": k["stream"],
                             "launch": round(k["launch"] - t0, 1) if k.get("launch") is not None else None,
                             "name": k["name"].replace("(anonymous namespace)::", "").replace("sconvb::", "").split("(")[0][-48:]} for k in sorted(f_, key=lambda k: k["start"])[:60]]
    out.append(rec)
    print(f"forward {i}: span {rec['span_us']:.1f} us, {len(f_)} launches, conv stream busy "
          f"{busy[conv_stream]:.1f} us, idle {rec['conv_stream_idle_us']:.1f} us in {len(gaps)} gaps; "
          f"streams busy " + ", ".join(f"{s}:{v:.0f}" for s, v in busy.items()))
    for g_ in rec["top_gaps"][:8]:
        print(f"   gap {g_['us']:7.1f} us at {g_['at_us']:7.1f} before {g_['before']}")
if out:
    print("kernel totals of the last forward (all streams):")
    for n, v in out[-1]["all_kernels"].items():
        print(f"  {n:44s} {v['launches']:3d} {v['us']:8.1f} us")
    print("timeline of the last forward (first 60 kernels): t0 t1 stream host-launch name")
    for k in out[-1]["first_kernels"]:
        la = f"{k['launch']:8.1f}" if k["launch"] is not None else "       -"
        print(f"  {k['t0']:8.1f} {k['t1']:8.1f} {k['stream']:4d} {la} {k['name']}")
for i, (e0, e1) in enumerate(marks):
    print(f"forward {i} event time {e0.elapsed_time(e1) * 1e3:.1f} us")
if a.json:
    with open(a.json, "w") as fh:
        json.dump(out, fh, indent=1)
