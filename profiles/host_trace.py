#!/usr/bin/env python3
"""Host-side phase timestamps of steady network forwards WITHOUT a profiler attached (CUPTI
inflates every API call): SCONV_HOST_TRACE=1 makes the library print per-op host marks at the
end of each forward; this runs a few forwards on device-resident inputs (as bench.py does).

  SCONV_HOST_TRACE=1 python profiles/host_trace.py [workload] > trace.txt
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2401_06145_b200 as sc  # noqa: E402
from paper_2401_06145_b200 import network as N  # noqa: E402
from paper_2401_06145_b200 import workloads as WL  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_minkunet42_kitti"
ctx = sc.Context(0)
g = WL.graph(name)
coords, feats = WL.scenes(name)[0]
net = N.Network(ctx, g, N.init_weights(g, WL.WEIGHT_SEED), sc.exec_cfg(dataflow=sc.DATAFLOW_AUTO))
xyz, f = torch.from_numpy(coords).cuda(), torch.from_numpy(feats).cuda()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
for _ in range(4):
    ctx.flush_l2(256 << 20)
    net.forward(device_xyz=xyz.data_ptr(), device_feats=f.data_ptr(), n=xyz.shape[0], sorted_=True)
    ctx.synchronize()
